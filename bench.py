"""Benchmark: list ranking (default: rs_rank on a random 2^26-node list,
BASELINE.json configs[1]) and connected components on the B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload lr26|lr28|lr28o|cc22|cc26] [--p P]

One JSON line on rank 0.  `value` = device-timed throughput with inputs
resident in HBM (CUDA events on the launching stream, max over ranks);
`e2e` = the same metric through the public API from pinned host buffers
(H2D + kernels + D2H inside the timed region).  `--impl reference` times the
reference algorithm's CPU port (oracle/, the sequential seq_rank /
seq_components restated in C) on the host cores -- rank 0 only.

Multi-GPU (torchrun): list ranking runs one replica per GPU (weak scaling);
cc22/cc26 shard the edge list over the ranks with an NCCL min all-reduce of
the parent array per round (strong scaling).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "List ranking M nodes/s & CC M edges/s vs CPU ref; achieved HBM GB/s"

WORKLOADS = {
    # name: (kind, log2 n, log2 m, list order)
    "lr26": ("list", 26, None, "random"),
    "lr28": ("list", 28, None, "random"),
    "lr28o": ("list", 28, None, "ordered"),
    "cc22": ("cc", 22, 24, None),
    "cc26": ("cc", 26, 28, None),
}

# SURVEY §8(d) algorithmic bytes
LR_BYTES_PER_NODE = {"random": 116, "ordered": 40}       # whole ranking
CC_EDGE_SWEEP_BYTES = 72                                  # 8 B edge + 2 x 32 B parent gathers
CC_VERTEX_SWEEP_BYTES = 40                                # 4 B + 32 B gather + 4 B write

# Algorithmic bytes per unit (node / edge) for each kernel of the step, used
# for the dominant kernel's roofline.  rs3_walk and the CC hooks use SURVEY
# §8(d)'s per-access figures (every data-dependent access to an array >> L2
# charged one 32-B sector); the streaming passes are charged the bytes they
# must move.  out = bytes per output rank (4 device-resident, 8 int64).
def kernel_bytes(kernel, order, out):
    return {
        "rs3_walk": 96 if order == "random" else 20,   # RS3: packed write + succ[cur] + packed read (listrank.py:279-283)
        "rs5_partition": 12 + 8,                       # record {cur, sid|local} in, {cur, rank} pair out
        "rs5_refine": 8 + 8,                           # binned walk record in, {cur, rank} out (IS_1 gather: L2)
        "rs5_scatter": 8 + out,
        "rs3_contract": 4 + 4,                         # succ in, {segment, distance} word out
        "rs5_expand": 4 + out,                         # node word in, rank out
        "rs1_validate": 4,
        "cc_hook_uf": CC_EDGE_SWEEP_BYTES,
        "cc_hook_sv": CC_EDGE_SWEEP_BYTES,
        "cc_partition": 8 + 8 + 8,                     # count pass reads the pairs; scatter reads + writes them
        "wy_jump": 48,
    }.get(kernel)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="lr26")
    ap.add_argument("--p", type=int, default=16384, help="reference splitter count p (rs_rank)")
    ap.add_argument("--variant", default="uf", help="components variant (uf | sv)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU-baseline sample length")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(workload, kernel):
    """DRAM bytes per step of `kernel` from the committed ncu capture
    (profiles/traffic.json, written by tools/ncu_summary.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            w = json.load(f).get(workload, {})
    except Exception:
        return None
    if kernel == "cc_partition" and "cc_partition_scatter" in w:
        return w.get("cc_partition_count", 0) + w["cc_partition_scatter"]
    return w.get(kernel)


class ClockSampler:
    """SM clocks + throttle reasons, polled through NVML every ~2 ms on a
    background thread while the timed region runs (nvidia-smi -lms cannot
    sample a region of a few ms)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.stop_flag = False
        self.thread = None
        self.max_mhz = None
        self.err = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:  # NVML enumerates every GPU of the host: match the CUDA device by UUID
                import torch
                uuid = str(torch.cuda.get_device_properties(self.index).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            except Exception:  # noqa: BLE001
                h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            return

        def run():
            while not self.stop_flag:
                try:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
                    self.samples.append((sm, rs, util))
                except Exception:  # noqa: BLE001
                    pass
                time.sleep(0.002)
        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "not sampled"], "samples": 0}
        self.stop_flag = True
        self.thread.join()
        busy = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = sorted(nm for nm, bit in self.REASONS.items() if any(s[1] & bit for s in busy))
        sm = [s[0] for s in busy]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(busy), "source": "nvml, 2 ms polling during the timed region"}


# ---------------------------------------------------------------------------
# reference arm: the CPU port of the reference's sequential algorithms

def cpu_list_rate(succ_host, threads, seconds):
    """M nodes/s of seq_rank's two dependent walks (core.py:164, :175) on the
    full-size list, `threads` independent walkers, about `seconds` of work."""
    from oracle import orc

    probe = 1 << 18
    t0 = time.perf_counter()
    done = orc.rank_walk_sample(succ_host, probe, threads)
    dt = time.perf_counter() - t0
    rate = done / max(dt, 1e-9)
    hops = int(min(max(rate * seconds / threads, 1 << 16), len(succ_host) // max(threads, 1)))
    t0 = time.perf_counter()
    done = orc.rank_walk_sample(succ_host, hops, threads)
    dt = time.perf_counter() - t0
    return done / dt / 1e6, done, dt


def cpu_cc_rate(n, edges_host, seconds):
    """M edges/s of seq_components (core.py:209-248) on an every-stride-th
    edge sample of the same graph: union time scaled to all m edges, plus the
    full labelling pass."""
    from oracle import orc

    m = len(edges_host)
    used, tu, tl = orc.uf_sample(n, edges_host, 1024)
    per_edge = tu / max(used, 1)
    stride = int(min(max(1, np.ceil(m * per_edge / max(seconds, 1e-3))), 1024))
    used, tu, tl = orc.uf_sample(n, edges_host, stride)
    est = tu * (m / used) + tl
    return m / est / 1e6, used, stride, tu, tl


# ---------------------------------------------------------------------------

def main():
    a = parse()
    kind, logn, logm, order = WORKLOADS[a.workload]
    n = 1 << logn
    m = (1 << logm) if logm else None
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    unit = "M nodes/s" if kind == "list" else "M edges/s"
    config = {"workload": a.workload, "n": n}
    if kind == "list":
        config.update(order=order, p=a.p,
                      algorithm="rs_rank: recursive sparse ruling set (scattered layouts) / tile contraction "
                                "(local layouts)",
                      inputs="device-resident u32 successors",
                      l2="inputs (4n B) > 126 MB L2, no flush" if n >= (1 << 26) else "L2 flushed between steps")
    else:
        config.update(m=m, variant=a.variant, inputs="device-resident u32 edge pairs",
                      l2="edges (8m B) > 126 MB L2, no flush" if m * 8 > (126 << 20) else "L2 flushed between steps")

    if a.impl == "reference":
        return reference_arm(a, kind, n, m, order, unit, config, world, rank)

    import torch
    import torch.distributed as dist

    import paper_1002_4482_b200 as g
    from paper_1002_4482_b200 import dist as sgdist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if "RANK" in os.environ and "WORLD_SIZE" in os.environ:  # launched by torchrun
        dist.init_process_group("nccl", device_id=dev)
    config["parallelism"] = (f"replicas x{world}" if kind == "list" else f"edge-sharded dp{world}")

    def barrier():
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x):
        if not dist.is_initialized():
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    need_flush = "flushed" in config["l2"]

    def flush():
        if need_flush:
            flush_buf.random_(0, 255)

    # ---- inputs (reference generators, bit-exact, built on the device) ----------
    if kind == "list":
        if order == "random":
            sl = g.gen_list(n, seed=rank, device=dev, dtype=torch.int32)
        else:
            sl = g.ordered_list(n, device=dev, dtype=torch.int32)

        def step():
            return g.rs_rank(sl, a.p, seed=0)
    else:
        gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=dev)
        edges32 = gr.edges.to(torch.int32)
        del gr
        gd = g.EdgeGraph(n, edges32)

        def step():
            if not dist.is_initialized():
                return g.sv_components(gd, 1024, variant=a.variant)
            return sgdist.sv_components_dist(gd, 1024, variant=a.variant)
    torch.cuda.synchronize(dev)

    # ---- warm-up ------------------------------------------------------------------
    for _ in range(a.warmup):
        out = step()
    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(2):
        out = step()
    # ---- timed region: exactly K steps ---------------------------------------------
    stream = torch.cuda.current_stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    launches = 0
    kern_ms = {}
    barrier()
    wall0 = time.perf_counter()
    for k in range(a.steps):
        flush()
        evs[k][0].record(stream)
        out, st = step()
        evs[k][1].record(stream)
        launches += len(st.launch_log)
        for rec in st.launch_log:
            kern_ms.setdefault(rec.kernel, []).append(rec.ms)
    barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = total_ms / a.steps
    units = n if kind == "list" else m
    units_job = units * world if kind == "list" else units
    value = units_job / (ms_per_step / 1e3) / 1e6

    # ---- dominant kernel roofline --------------------------------------------------
    peak, peak_src = load_peaks()
    units = n if kind == "list" else m
    step_kern = {k: sum(v) / a.steps for k, v in kern_ms.items()}        # ms per step, per kernel
    launches_per_step = {k: len(v) / a.steps for k, v in kern_ms.items()}
    kname = max(step_kern, key=step_kern.get)
    out_bytes = 4
    bpu = kernel_bytes(kname, order, out_bytes)
    k_units = units // world if (kind == "cc" and world > 1 and kname.startswith("cc_")) else units
    k_ms = step_kern[kname]
    algo_bytes = bpu * k_units if bpu is not None else None
    achieved = (algo_bytes / (k_ms / 1e3) / 1e9) if (algo_bytes and k_ms) else None
    if kind == "list":
        pipe_bytes = LR_BYTES_PER_NODE[order] * n
    else:
        pipe_bytes = st.meta["edge_sweeps"] * CC_EDGE_SWEEP_BYTES * m + st.meta["vertex_sweeps"] * CC_VERTEX_SWEEP_BYTES * n
    traffic = load_traffic(a.workload, kname)
    roofline = {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1) if achieved else None,
                "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4) if achieved else None,
                "traffic": traffic, "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)",
                "algorithmic_bytes_per_unit": bpu, "units_per_step": k_units,
                "algorithmic_bytes_per_step": algo_bytes, "kernel_ms_per_step": round(k_ms, 4),
                "launches_per_step": launches_per_step[kname],
                "kernel_share_of_step": round(k_ms / ms_per_step, 3),
                "traffic_note": "dram__bytes_read+write per step from the committed ncu capture (profiles/)",
                "pipeline": {"algorithmic_bytes": pipe_bytes,
                             "bytes_per_unit": (LR_BYTES_PER_NODE[order] if kind == "list" else None),
                             "achieved": round(pipe_bytes / (ms_per_step / 1e3) / 1e9, 1),
                             "frac": round(pipe_bytes / (ms_per_step / 1e3) / 1e9 / peak, 4),
                             "note": ("SURVEY 8(d) bytes: every parent gather charged a 32-B DRAM sector; "
                                      "frac > 1 means the window partition served them from L2")
                             if kind != "list" else
                             ("SURVEY 8(d) bytes per node" if order == "random" else
                              "SURVEY 8(d) 40 B/node charges the ruling-set streams; the tile contraction "
                              "moves ~20 B/node, so frac can exceed 1")}}
    kernels = {k: round(sum(v) / len(v), 4) for k, v in sorted(kern_ms.items())}

    # ---- e2e through the public API with pinned host buffers -------------------------
    e2e = None
    if not a.no_e2e:
        e2e = e2e_run(a, g, sgdist, torch, dev, kind, n, m, order, world, rank, barrier, max_over_ranks,
                      sl if kind == "list" else gd)

    # ---- secondary: Wyllie vs ruling set (configs[1]) -------------------------------
    secondary = None
    if kind == "list" and not a.no_secondary and logn <= 26:
        w_ms = []
        g.wyllie_rank(sl, 1024)
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.wyllie_rank(sl, 1024)
            e1.record(stream)
            e1.synchronize()
            w_ms.append(e0.elapsed_time(e1))
        wm = statistics.median(w_ms)
        secondary = {"wyllie_rank": {"ms_per_step": round(wm, 3), "value": round(n * world / wm / 1e3, 1),
                                     "unit": unit, "rounds": int(np.ceil(np.log2(n))),
                                     "speedup_of_rs_rank": round(wm / ms_per_step, 2)}}

    # ---- CPU baseline (rank 0, N = 1) ------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline(a, kind, n, m, sl if kind == "list" else gd, torch)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": unit, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
                "scaling": "weak" if kind == "list" else "strong", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic: the reference generators (gen_list / gen_random_graph, seed 0) reproduced "
                        "bit-exactly on the device",
                "config": config, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk, "kernels_ms": kernels,
                "wall_s_timed_region": round(wall, 4)}
        if secondary:
            line["secondary"] = secondary
        if kind == "cc":
            line["cc"] = {"rounds": st.meta["rounds"], "edge_sweeps": st.meta["edge_sweeps"],
                          "vertex_sweeps": st.meta["vertex_sweeps"],
                          "components": st.meta["roots_per_round"][-1]}
        else:
            line["ruling_set"] = {"path": st.meta["path"], "levels": st.meta["levels"],
                                  "level_size": st.meta["level_size"], "fallback": st.meta["fallback"]}
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


def e2e_run(a, g, sgdist, torch, dev, kind, n, m, order, world, rank, barrier, max_over_ranks, dev_input):
    """Same metric through the public API from pinned host int64 buffers:
    every step copies the inputs H2D and reads the int64 result back."""
    if kind == "list":
        host = dev_input.succ.to(torch.int64).cpu().pin_memory()

        def step():
            return g.rs_rank(g.SuccessorList(host), a.p, seed=0)
        h2d = 8 * n
        d2h = 8 * n
    else:
        host = dev_input.edges.to(torch.int64).cpu().pin_memory()

        def step():
            if not torch.distributed.is_initialized():
                return g.sv_components(g.EdgeGraph(n, host), 1024, variant=a.variant)
            return sgdist.sv_components_dist(g.EdgeGraph(n, host), 1024, variant=a.variant)
        h2d = 16 * m // (world if world > 1 else 1)
        d2h = 8 * n
    outs = [step()[0] for _ in range(3)]  # warm: the pinned host-allocator cache fills on the first calls
    del outs
    steps = max(3, min(a.steps, 10))
    barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        out, _ = step()
    barrier()
    dt = max_over_ranks(time.perf_counter() - t0) / steps
    units = (n * world) if kind == "list" else m
    assert isinstance(out, np.ndarray) and out.shape == (n,)
    return {"value": round(units / dt / 1e6, 1), "unit": "M nodes/s" if kind == "list" else "M edges/s",
            "ms_per_step": round(dt * 1e3, 3), "steps": steps, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "rs_rank(SuccessorList(pinned int64)) -> numpy int64" if kind == "list"
            else "sv_components(EdgeGraph(pinned int64)) -> numpy int64"}


def cpu_baseline(a, kind, n, m, inp, torch):
    threads = 1
    if kind == "list":
        succ = inp.succ.to(torch.int64).cpu().numpy()
        rate, done, dt = cpu_list_rate(succ, threads, a.cpu_seconds)
        return {"value": round(rate, 3), "unit": "M nodes/s", "cores": threads, "kind": "port",
                "sample": f"seq_rank's two dependent walks (oracle/orc.c, core.py:122-186) for {done} hops each "
                          f"over the full 2^{int(np.log2(n))}-node list; {dt:.1f} s",
                "algorithm": "seq_rank"}
    edges = inp.edges.to(torch.int64).cpu().numpy()
    rate, used, stride, tu, tl = cpu_cc_rate(n, edges, a.cpu_seconds)
    return {"value": round(rate, 3), "unit": "M edges/s", "cores": threads, "kind": "port",
            "sample": f"seq_components union-find (oracle/orc.c, core.py:209-248) over every {stride}-th edge "
                      f"({used} edges, {tu:.2f} s, scaled to m) + full labelling pass ({tl:.2f} s)",
            "algorithm": "seq_components"}


def reference_arm(a, kind, n, m, order, unit, config, world, rank):
    """Times the reference's CPU implementation (its sequential oracles,
    restated in C under oracle/) on the host cores.  Rank 0 only."""
    if rank != 0:
        return
    import torch  # noqa: F401  (generation runs on the device when one is present)

    import paper_1002_4482_b200 as g

    threads = os.cpu_count() or 1
    have_gpu = torch.cuda.is_available()
    dev = torch.device("cuda", 0) if have_gpu else None
    if kind == "list":
        if order == "random":
            sl = g.gen_list(n, seed=0, device=dev)
        else:
            sl = g.ordered_list(n)
        succ = sl.host_succ()
        per_step = max(1.0, 60.0 / max(a.steps + a.warmup, 1))
        for _ in range(a.warmup):
            cpu_list_rate(succ, threads, min(per_step, 1.0))
        rates = []
        t0 = time.perf_counter()
        for _ in range(a.steps):
            r, done, dt = cpu_list_rate(succ, threads, per_step)
            rates.append(r)
        wall = time.perf_counter() - t0
        value = statistics.median(rates)
        sample = (f"{threads} threads each walking seq_rank's two dependent walks (oracle/orc.c; core.py:122-186) "
                  f"for ~{per_step:.1f} s over the full 2^{int(np.log2(n))}-node list")
        ms_per_step = wall / a.steps * 1e3
    else:
        gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=dev)
        edges = gr.host_edges()
        threads = 1   # union-find is sequential; one core
        rates = []
        t0 = time.perf_counter()
        for _ in range(a.warmup):
            cpu_cc_rate(n, edges, 2.0)
        t0 = time.perf_counter()
        for _ in range(a.steps):
            r, used, stride, tu, tl = cpu_cc_rate(n, edges, 5.0)
            rates.append(r)
        wall = time.perf_counter() - t0
        value = statistics.median(rates)
        sample = (f"seq_components union-find (oracle/orc.c; core.py:209-248) over every {stride}-th edge of the "
                  f"2^{int(np.log2(m))}-edge graph, union time scaled to m + full labelling pass")
        ms_per_step = wall / a.steps * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": unit, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "weak" if kind == "list" else "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic: reference generators, seed 0", "config": config,
            "cpu_baseline": {"value": round(value, 3), "unit": unit, "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": round(value, 3), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
