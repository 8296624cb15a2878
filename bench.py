"""Benchmark: list ranking and connected components on the B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload lr28|lr28o|lr26|cc22|cc26] [--blocks lr28o,lr26,cc22,cc26|none]

Default headline (north_star's target, BASELINE.json configs[2]): `rs_rank`
on the 2^28-node random list (C3).  The same JSON line carries one block per
other config -- `lr28o` (C3 ordered), `lr26` (C2, with Wyllie beside it),
`cc22` (C4) and `cc26` (C5: 2^26 vertices / 2^28 edges) -- each with its own
value, roofline and kernel times; the headline and `cc26` also carry `e2e`
and `cpu_baseline`.

`value` = device-timed throughput with inputs resident in HBM (CUDA events
on the launching stream, max over ranks); `e2e` = the same metric through
the public API from pinned host int64 buffers (H2D + kernels + D2H inside
the timed region).

`--impl reference` times the reference's own CPU algorithm for the headline
config -- its sequential `seq_rank` (core.py:179-186), restated in C under
oracle/ -- on the host, rank 0 only, with inputs made by the oracle's
generators (oracle/orc.c gen_list, gen.py:110-127).  Each step is a bounded
sample (the first H nodes of the chain, seq_rank's full per-node work);
one complete seq_rank over the whole list calibrates the sample and is
checked against the reference's own digest (tests/golden/hashes.json).
Nothing of paper_1002_4482_b200 is imported on that arm.

Multi-GPU (torchrun): list ranking runs one replica per GPU (weak scaling);
the cc blocks shard the edge list over the ranks with an NCCL min
all-reduce of the parent array per round (strong scaling).
"""

import argparse
import gc
import hashlib
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "List ranking M nodes/s & CC M edges/s vs CPU ref; achieved HBM GB/s"

WORKLOADS = {
    # name: (kind, log2 n, log2 m, list order, BASELINE config)
    "lr26": ("list", 26, None, "random", "C2"),
    "lr28": ("list", 28, None, "random", "C3"),
    "lr28o": ("list", 28, None, "ordered", "C3"),
    "cc22": ("cc", 22, 24, None, "C4"),
    "cc26": ("cc", 26, 28, None, "C5"),
}
DEFAULT_BLOCKS = "lr28o,lr26,cc22,cc26"

# SURVEY §8(d) algorithmic bytes
LR_BYTES_PER_NODE = {"random": 116, "ordered": 40}       # whole ranking
CC_EDGE_SWEEP_BYTES = 72                                  # 8 B edge + 2 x 32 B parent gathers
CC_VERTEX_SWEEP_BYTES = 40                                # 4 B + 32 B gather + 4 B write


def kernel_bytes(kernel, order, out):
    """Algorithmic bytes per unit (node / edge) of each kernel of the step,
    for the dominant kernel's roofline.  rs3_walk and the CC hooks use SURVEY
    §8(d)'s per-access figures (every data-dependent access to an array >> L2
    charged one 32-B sector); streaming passes are charged the bytes they
    must move.  out = bytes per output rank (4 device-resident)."""
    return {
        "rs3_walk": 96 if order == "random" else 20,   # RS3: packed write + succ[cur] + packed read (listrank.py:279-283)
        "rs5_refine": 8 + 8,                           # binned walk record in, {cur, rank} out (IS_1 gather: L2)
        "rs5_scatter": 8 + out,
        # contraction: succ in, {segment, distance} word out; the run tiles of an
        # ordered list are settled from the census's flag (no per-node bytes)
        "rs3_contract": 4 + 4 if order != "ordered" else None,
        "rs5_expand": 4 + out if order != "ordered" else out,  # node word in (not for run tiles), rank out
        "rs1_validate": 4,
        "cc_hook_uf": CC_EDGE_SWEEP_BYTES,
        "cc_hook_sv": CC_EDGE_SWEEP_BYTES,
        "cc_partition": 8 + 8,                         # one pass: reads the pairs, writes them by window
        "wy_jump": 48,
    }.get(kernel)


def config_for(name, p):
    """The `config` object of a workload -- identical on both arms."""
    kind, logn, logm, order, cfg = WORKLOADS[name]
    n = 1 << logn
    c = {"workload": name, "baseline_config": cfg, "n": n}
    if kind == "list":
        c.update(order=order, p=p, seed=0,
                 l2="succ (4n B) > 126 MB L2, no flush" if n >= (1 << 26) else "L2 flushed between steps")
    else:
        m = 1 << logm
        c.update(m=m, seed=0,
                 l2="edges (8m B) > 126 MB L2, no flush" if m * 8 > (126 << 20) else "L2 flushed between steps")
    return c


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="lr28")
    ap.add_argument("--blocks", default=None,
                    help=f"comma list of extra workloads in the same line (default {DEFAULT_BLOCKS} for lr28; "
                         "'none' for none)")
    ap.add_argument("--p", type=int, default=16384, help="reference splitter count p (rs_rank)")
    ap.add_argument("--variant", default="uf", help="components variant (uf | sv)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-calibrate", action="store_true", help="reference arm: skip the complete seq_rank run")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU-baseline sample length")
    a = ap.parse_args(argv)
    if a.blocks is None:
        a.blocks = DEFAULT_BLOCKS if a.workload == "lr28" else "none"
    a.blocks = [] if a.blocks in ("", "none") else [b for b in a.blocks.split(",") if b != a.workload]
    for b in a.blocks:
        if b not in WORKLOADS:
            ap.error(f"unknown block {b}")
    return a


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md HBM copy figure)"


def load_traffic(workload, kernel):
    """DRAM bytes per step of `kernel` from the committed ncu capture
    (profiles/traffic.json, written by tools/ncu_summary.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(workload, {}).get(kernel)
    except Exception:
        return None


def load_hashes():
    with open(os.path.join(ROOT, "tests", "golden", "hashes.json")) as f:
        return json.load(f)


def sha256_i64(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


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

    # the sampler polls NVML in a child process (no GIL shared with the timed
    # loop), timestamps each sample on CLOCK_MONOTONIC and the parent keeps the
    # samples inside [start, stop]
    CHILD = r"""
import sys, time, pynvml
pynvml.nvmlInit()
uuid, index, period, util_on = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), sys.argv[4] == "1"
try:
    h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
except Exception:
    h = pynvml.nvmlDeviceGetHandleByIndex(index)
print("max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
import select
while True:
    r, _, _ = select.select([sys.stdin], [], [], period)
    if r:
        break
    try:
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu if util_on else 1
        print(time.monotonic(), sm, rs, util, flush=True)
    except Exception:
        pass
"""

    # NVML queries go through the driver and stall the CUDA calls of the timed
    # process while they run: 2 ms polling cost lr28 ~15 % (measured, r02j),
    # so the sampler polls every PERIOD_MS (still several samples per workload)
    PERIOD_MS = float(os.environ.get("SG_BENCH_POLL_MS", "20"))

    def start(self):
        import subprocess
        if self.PERIOD_MS <= 0:  # diagnostics only: no sampling
            self.err = "sampling disabled (SG_BENCH_POLL_MS=0)"
            return
        try:
            import torch
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            self.proc = subprocess.Popen([sys.executable, "-c", self.CHILD, uuid, str(self.index),
                                          str(self.PERIOD_MS / 1e3), os.environ.get("SG_BENCH_POLL_UTIL", "0")],
                                         stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)
            first = self.proc.stdout.readline().split()
            if not first or first[0] != "max":
                raise RuntimeError("sampler did not start")
            self.max_mhz = int(first[1])
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml unavailable: {e}"
            self.proc = None
            return
        self.thread = True

    def mark(self):
        """Open the sampled window (after warm-up, right before the timed loop)."""
        self.t0 = time.monotonic()

    def stop(self):
        if self.thread is None or self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "not sampled"], "samples": 0}
        t1 = time.monotonic()
        out, _ = self.proc.communicate("stop\n", timeout=30)
        t0 = getattr(self, "t0", 0.0)
        for line in out.splitlines():
            f = line.split()
            if len(f) == 4 and t0 <= float(f[0]) <= t1:
                self.samples.append((int(f[1]), int(f[2]), int(f[3])))
        busy = [s for s in self.samples if s[2] > 0] or self.samples
        reasons = sorted(nm for nm, bit in self.REASONS.items() if any(s[1] & bit for s in busy))
        sm = [s[0] for s in busy]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(busy), "source": f"nvml, {self.PERIOD_MS:g} ms polling in a child process during the timed region"}


# ---------------------------------------------------------------------------
# CPU side: the reference's sequential algorithms, restated in C (oracle/)

def seq_rank_samples(orc, succ, count, seconds_each, warm=1):
    """`count` bounded samples of seq_rank on the full-size list (orc.c
    orc_seq_rank_sample): each ranks the first H nodes of the chain with
    seq_rank's per-node work, H sized for ~seconds_each.  Returns
    (per-sample (hops, seconds) list, H)."""
    smp = orc.SeqRankSampler(succ)
    t0 = time.perf_counter()
    k = smp(1 << 18)
    rate = k / max(time.perf_counter() - t0, 1e-9)
    hops = int(min(max(rate * seconds_each, 1 << 18), len(succ)))
    for _ in range(warm):
        smp(hops)
    out = []
    for _ in range(count):
        t0 = time.perf_counter()
        k = smp(hops)
        out.append((k, time.perf_counter() - t0))
    return out, hops


def cpu_list_baseline(orc, succ, seconds, logn):
    samples, hops = seq_rank_samples(orc, succ, 3, seconds / 3)
    nodes = sum(k for k, _ in samples)
    dt = sum(t for _, t in samples)
    return {"value": round(nodes / dt / 1e6, 3), "unit": "M nodes/s", "cores": 1, "kind": "port",
            "algorithm": "seq_rank (core.py:179-186), oracle/orc.c, single-threaded (sequential algorithm)",
            "sample": f"3 samples, each seq_rank's per-node work (range/self-loop scans, validation walk, "
                      f"position walk, rank fill) for the first {hops} nodes of the 2^{logn}-node chain over "
                      f"the full-size arrays; {dt:.1f} s in total"}


def cpu_cc_baseline(orc, n, edges, logm):
    t0 = time.perf_counter()
    lab = orc.seq_components(n, edges)
    dt = time.perf_counter() - t0
    return {"value": round(len(edges) / dt / 1e6, 3), "unit": "M edges/s", "cores": 1, "kind": "port",
            "algorithm": "seq_components (core.py:240-248): validate_graph + union-find, oracle/orc.c, "
                         "single-threaded (sequential algorithm)",
            "sample": f"one complete run over all 2^{logm} edges ({dt:.1f} s), not a sample",
            "components": int(np.count_nonzero(lab == np.arange(n)))}, lab


# ---------------------------------------------------------------------------
# our arm

class Ctx:
    @staticmethod
    def xfer_bytes(count, bound=None):
        """PCIe bytes the public API moves for `count` int64 host ids: long
        arrays cross as 32-bit ids (paper_1002_4482_b200/_device.py
        NARROW_MIN, sg_xfer.cu), short ones as int64."""
        from paper_1002_4482_b200._device import NARROW_MIN

        return 4 * count if count >= NARROW_MIN else 8 * count


def measure(a, ctx, name, primary):
    """Run one workload: W warm-up steps, K timed steps (CUDA events on the
    launching stream, barrier + synchronize on both sides, max over ranks),
    then the roofline of the dominant kernel, e2e and the CPU baseline."""
    torch, g, sgdist, dist, dev = ctx.torch, ctx.g, ctx.sgdist, ctx.dist, ctx.dev
    kind, logn, logm, order, _ = WORKLOADS[name]
    n = 1 << logn
    m = (1 << logm) if logm else None
    world, rank = ctx.world, ctx.rank
    unit = "M nodes/s" if kind == "list" else "M edges/s"
    config = config_for(name, a.p)
    config["parallelism"] = f"replicas x{world}" if kind == "list" else f"edge-sharded x{world}"

    need_flush = "flushed" in config["l2"]
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if need_flush else None

    if kind == "list":
        if order == "random":
            sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32)
        else:
            sl = g.ordered_list(n, device=dev, dtype=torch.int32)

        def step():
            return g.rs_rank(sl, a.p, seed=0)
        inp = sl
    else:
        gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=dev)
        gd = g.EdgeGraph(n, gr.edges.to(torch.int32))
        del gr

        def step():
            if world == 1:
                return g.sv_components(gd, 1024, variant=a.variant)
            return sgdist.sv_components_dist(gd, 1024, variant=a.variant)
        inp = gd
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(ctx.local)
    clocks.start()
    for _ in range(a.warmup):
        out = step()
    del out
    stream = torch.cuda.current_stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    launches = 0
    kern_ms = {}
    # the cyclic GC is paused over the timed steps (as timeit does): a
    # collection landing between an event record and the call's first launch
    # idles the GPU for milliseconds (measured: single-step outliers of +5-13 ms)
    gc.collect()
    if os.environ.get("SG_BENCH_GC", "0") != "1":
        gc.disable()
    ctx.barrier()
    clocks.mark()
    wall0 = time.perf_counter()
    for k in range(a.steps):
        if need_flush:
            flush_buf.random_(0, 255)
        evs[k][0].record(stream)
        out, st = step()
        evs[k][1].record(stream)
        # per-kernel CUDA-event times (ExecStats resolves them on first read;
        # the call has already synchronised its stream)
        launches += len(st.launch_log)
        for rec in st.launch_log:
            kern_ms.setdefault(rec.kernel, []).append(rec.ms)
    ctx.barrier()
    wall = time.perf_counter() - wall0
    gc.enable()
    clk = clocks.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    ms_per_step = ctx.max_over_ranks(sum(step_ms)) / a.steps
    units = n if kind == "list" else m
    units_job = units * world if kind == "list" else units
    value = units_job / (ms_per_step / 1e3) / 1e6

    # ---- dominant kernel roofline ----------------------------------------------------
    peak, peak_src = load_peaks()
    step_kern = {k: sum(v) / a.steps for k, v in kern_ms.items()}
    launches_per_step = {k: len(v) / a.steps for k, v in kern_ms.items()}
    kname = max((k for k in step_kern if not k.startswith("nccl")), key=step_kern.get)
    bpu = kernel_bytes(kname, order, 4)
    k_units = units // world if (kind == "cc" and world > 1) else units
    k_ms = step_kern[kname]
    algo_bytes = bpu * k_units if bpu is not None else None
    achieved = (algo_bytes / (k_ms / 1e3) / 1e9) if (algo_bytes and k_ms) else None
    if kind == "list":
        pipe_bytes = LR_BYTES_PER_NODE[order] * n
    else:
        pipe_bytes = (st.meta["edge_sweeps"] * CC_EDGE_SWEEP_BYTES * m
                      + st.meta["vertex_sweeps"] * CC_VERTEX_SWEEP_BYTES * n) // world
    traffic = load_traffic(name, kname) if world == 1 else None
    roofline = {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1) if achieved else None,
                "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4) if achieved else None,
                "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_unit": bpu, "units_per_launch_set": k_units,
                "algorithmic_bytes_per_step": algo_bytes, "kernel_ms_per_step": round(k_ms, 4),
                "launches_per_step": launches_per_step[kname],
                "kernel_share_of_step": round(k_ms / ms_per_step, 3),
                "traffic_note": "ncu dram__bytes_read+write of this kernel per step, committed capture "
                                "(profiles/traffic.json)",
                "pipeline": {"algorithmic_bytes": pipe_bytes,
                             "bytes_per_unit": LR_BYTES_PER_NODE[order] if kind == "list" else None,
                             "achieved": round(pipe_bytes / (ms_per_step / 1e3) / 1e9, 1),
                             "frac": round(pipe_bytes / (ms_per_step / 1e3) / 1e9 / peak, 4),
                             "note": ("SURVEY 8(d) 116 B/node" if order == "random" else
                                      "SURVEY 8(d) 40 B/node charges the ruling-set streams; the tile "
                                      "contraction moves ~20 B/node, so frac can exceed 1") if kind == "list"
                             else ("SURVEY 8(d) E*72*m + V*40*n (per rank): every parent gather charged a 32-B "
                                   "DRAM sector although the window partition serves them from L2")}}
    if traffic and k_ms:
        # the same kernel against what it actually moved (ncu DRAM bytes): the
        # honest utilisation where a per-access model over- or under-charges
        meas = traffic / (k_ms / 1e3) / 1e9
        roofline["measured_dram"] = {"achieved": round(meas, 1), "frac": round(meas / peak, 4),
                                     "bytes_per_launch_set": traffic}
    if kname.startswith("cc_hook"):
        roofline["bound_note"] = ("latency-bound, not HBM-bound: union-find finds and root CAS against an "
                                  "L2-resident window of the parent array (ncu L2 hit ~60 %); SURVEY's 72 B/edge "
                                  "charges every parent gather a DRAM sector the window partition never pays, so "
                                  "frac can exceed 1 -- measured_dram is the utilisation")
    elif kname == "rs3_walk" and order == "random":
        roofline["bound_note"] = ("random-access bound: one dependent 4-B succ load per hop, each costing ~97-133 B "
                                  "of DRAM (sector + overfetch, ncu); the walk runs at the measured random-gather "
                                  "ceiling (profiles/r01_ubench_random.txt)")
    srt = sorted(step_ms)
    res = {"value": round(value, 1), "unit": unit, "ms_per_step": round(ms_per_step, 4), "steps": a.steps,
           "timing": "CUDA events on the launching stream around each API call; python cyclic GC paused over "
                     "the timed steps",
           "step_ms_spread": {"min": round(srt[0], 4), "median": round(srt[len(srt) // 2], 4),
                              "max": round(srt[-1], 4), "argmax": int(max(range(len(step_ms)), key=step_ms.__getitem__))},
           "warmup": a.warmup, "config": config,
           "algorithm": ("rs_rank (listrank.py:411): recursive sparse ruling set on scattered layouts, tile "
                         "contraction on local layouts" if kind == "list" else
                         f"sv_components (concomp.py:208), variant {a.variant}"),
           "inputs": "device-resident u32 successors" if kind == "list" else "device-resident u32 edge pairs", "roofline": roofline, "gpu_launches": launches,
           "clocks": clk, "kernels_ms_per_step": {k: round(v, 4) for k, v in sorted(step_kern.items())},
           "wall_s_timed_region": round(wall, 4)}
    if kind == "cc":
        res["cc"] = {"rounds": st.meta["rounds"], "edge_sweeps": st.meta["edge_sweeps"],
                     "vertex_sweeps": st.meta["vertex_sweeps"], "components": st.meta["roots_per_round"][-1]}
        if world > 1:
            res["cc"]["collectives"] = collective_bw(st.meta, step_kern, world)
    else:
        res["ruling_set"] = {"path": st.meta["path"], "levels": st.meta["levels"],
                             "level_size": st.meta["level_size"], "fallback": st.meta["fallback"]}

    # ---- Wyllie beside the ruling set (C2) ---------------------------------------------
    if kind == "list" and logn <= 26 and order == "random":
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
        res["wyllie_rank"] = {"ms_per_step": round(wm, 3), "value": round(n * world / wm / 1e3, 1),
                              "unit": unit, "rounds": int(np.ceil(np.log2(n))),
                              "rs_rank_speedup": round(wm / ms_per_step, 2)}

    # ---- e2e through the public API with pinned host buffers -----------------------------
    full = primary or kind == "cc" and logn >= 26
    if full and not a.no_e2e:
        res["e2e"] = e2e_run(a, ctx, kind, n, m, inp)

    # ---- CPU baseline (rank 0, N = 1) ------------------------------------------------------
    if full and rank == 0 and world == 1 and not a.no_cpu:
        from oracle import orc
        if kind == "list":
            succ = inp.succ.to(torch.int64).cpu().numpy()
            res["cpu_baseline"] = cpu_list_baseline(orc, succ, a.cpu_seconds, logn)
        else:
            edges = inp.edges.to(torch.int64).cpu().numpy()
            cpu, lab = cpu_cc_baseline(orc, n, edges, logm)
            ours, _ = g.sv_components(inp, 1024, variant=a.variant)
            cpu["labels_equal_ours"] = bool(np.array_equal(lab, ours.cpu().numpy()))
            res["cpu_baseline"] = cpu
    return res


def collective_bw(meta, step_kern, world):
    """SURVEY 8(d) multi-GPU figures for the sharded rounds: per step, bytes
    and CUDA-event time of the min all-reduce and the all-gather(s), algbw =
    bytes / time, busbw = algbw * 2(G-1)/G (all-reduce) or (G-1)/G
    (all-gather; its span also holds the 8-B root-count all-reduce)."""
    out = {}
    for name, key, factor, bkey in (("allreduce_min", "nccl_allreduce_min", 2.0 * (world - 1) / world,
                                     "allreduce_bytes"),
                                    ("allgather", "nccl_allgather", (world - 1) / world, "allgather_bytes")):
        ms = step_kern.get(key, 0.0) + (step_kern.get(key + "_changes", 0.0) if name == "allgather" else 0.0)
        nbytes = int(meta.get(bkey, 0))
        algbw = nbytes / (ms / 1e3) / 1e9 if ms > 0 else None
        out[name] = {"bytes_per_step": nbytes, "ms_per_step": round(ms, 4),
                     "algbw_gbs": round(algbw, 1) if algbw else None,
                     "busbw_gbs": round(algbw * factor, 1) if algbw else None}
    return out


def e2e_run(a, ctx, kind, n, m, dev_input):
    """Same metric through the public API from pinned host int64 buffers:
    every step copies the inputs H2D and reads the int64 result back."""
    torch, g, sgdist, world = ctx.torch, ctx.g, ctx.sgdist, ctx.world
    if kind == "list":
        host = dev_input.succ.to(torch.int64).cpu().pin_memory()

        def step():
            return g.rs_rank(g.SuccessorList(host), a.p, seed=0)
        h2d = d2h = ctx.xfer_bytes(n)
    else:
        host = dev_input.edges.to(torch.int64).cpu().pin_memory()

        def step():
            if world == 1:
                return g.sv_components(g.EdgeGraph(n, host), 1024, variant=a.variant)
            return sgdist.sv_components_dist(g.EdgeGraph(n, host), 1024, variant=a.variant)
        h2d = ctx.xfer_bytes(2 * (m // world), bound=n)
        d2h = ctx.xfer_bytes(n)
    outs = [step()[0] for _ in range(3)]  # warm: the pinned host-allocator cache fills on the first calls
    del outs
    steps = max(3, min(a.steps, 10))
    gc.collect()
    if os.environ.get("SG_BENCH_GC", "0") != "1":
        gc.disable()  # as in the device-timed loop
    ctx.barrier()
    t0 = time.perf_counter()
    marks = [t0]
    for _ in range(steps):
        out, _ = step()
        marks.append(time.perf_counter())
    ctx.barrier()
    dt = ctx.max_over_ranks(time.perf_counter() - t0) / steps
    gc.enable()
    per = sorted((b - a_) * 1e3 for a_, b in zip(marks, marks[1:]))
    units = (n * world) if kind == "list" else m
    assert isinstance(out, np.ndarray) and out.shape == (n,)
    return {"value": round(units / dt / 1e6, 1), "unit": "M nodes/s" if kind == "list" else "M edges/s",
            "ms_per_step": round(dt * 1e3, 3), "steps": steps, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "rs_rank(SuccessorList(pinned int64)) -> numpy int64" if kind == "list"
            else "sv_components(EdgeGraph(pinned int64)) -> numpy int64",
            "host_threads": _xfer_threads(),
            "step_ms_spread": {"min": round(per[0], 3), "median": round(per[len(per) // 2], 3),
                               "max": round(per[-1], 3)},
            "timing": "host perf_counter around the API calls, max over ranks"}


def _xfer_threads():
    """Host threads of the boundary conversions (sg_xfer_threads)."""
    from paper_1002_4482_b200 import _native
    return int(_native.lib().sg_xfer_threads())


def ours(a):
    import torch
    import torch.distributed as dist

    import paper_1002_4482_b200 as g
    from paper_1002_4482_b200 import dist as sgdist

    ctx = Ctx()
    ctx.torch, ctx.g, ctx.sgdist, ctx.dist = torch, g, sgdist, dist
    ctx.world = int(os.environ.get("WORLD_SIZE", "1"))
    ctx.rank = int(os.environ.get("RANK", "0"))
    ctx.local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(ctx.local)
    ctx.dev = dev = torch.device("cuda", ctx.local)
    if "RANK" in os.environ and "WORLD_SIZE" in os.environ:  # launched by torchrun
        dist.init_process_group("nccl", device_id=dev)

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
    ctx.barrier, ctx.max_over_ranks = barrier, max_over_ranks

    head = measure(a, ctx, a.workload, primary=True)
    torch.cuda.empty_cache()
    blocks = {}
    for b in a.blocks:
        blocks[b] = measure(a, ctx, b, primary=False)
        torch.cuda.empty_cache()

    if ctx.rank == 0:
        kind = WORKLOADS[a.workload][0]
        line = {"metric": METRIC, "value": head["value"], "unit": head["unit"], "n_gpus": ctx.world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": head["ms_per_step"],
                "higher_is_better": True, "scaling": "weak" if kind == "list" else "strong",
                "vs_baseline": None, "dtype": "u32",
                "data": "synthetic: the reference generators (gen_list / gen_random_graph, seed 0) reproduced "
                        "bit-exactly on the device (digests pinned to the reference in tests/golden/hashes.json)",
                "config": head["config"], "roofline": head["roofline"], "cpu_baseline": head.get("cpu_baseline"),
                "e2e": head.get("e2e"), "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
                "kernels_ms_per_step": head["kernels_ms_per_step"],
                "wall_s_timed_region": head["wall_s_timed_region"]}
        for k in ("timing", "step_ms_spread", "algorithm", "inputs", "ruling_set", "cc", "wyllie_rank"):
            if k in head:
                line[k] = head[k]
        for b, r in blocks.items():
            line[b] = r
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm

def reference_arm(a):
    """The reference's CPU implementation of the headline path: its sequential
    seq_rank (core.py:179-186) -- the paper's "sequential CPU" baseline,
    PAPER.md:679-684 -- restated in C (oracle/orc.c), on inputs from the
    oracle's restatement of gen_list (gen.py:110-127).  Rank 0 only; one
    host thread (the algorithm is a single dependent walk).  Every step is a
    bounded sample; one complete seq_rank calibrates it and is checked
    against the reference's digest."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle import orc

    kind, logn, logm, order, _ = WORKLOADS[a.workload]
    n = 1 << logn
    config = config_for(a.workload, a.p)
    config["parallelism"] = f"replicas x{world}" if kind == "list" else f"edge-sharded x{world}"
    hashes = load_hashes()
    t0 = time.perf_counter()
    calib = None
    if kind == "list":
        succ = orc.gen_list(n, 0) if order == "random" else np.minimum(np.arange(1, n + 1), n - 1)
        t_gen = time.perf_counter() - t0
        per_step = max(0.3, min(1.5, 40.0 / max(a.steps + a.warmup, 1)))
        samples, hops = seq_rank_samples(orc, succ, a.steps, per_step, warm=a.warmup)
        nodes = sum(k for k, _ in samples)
        secs = sum(t for _, t in samples)
        value = nodes / secs / 1e6
        ms_per_step = secs / a.steps * 1e3
        sample = (f"each step = seq_rank's per-node work (range/self-loop scans, validation walk core.py:164, "
                  f"position walk core.py:175, rank fill) for the first {hops} nodes of the 2^{logn}-node chain, "
                  f"over the full-size arrays")
        if not a.no_calibrate:
            t1 = time.perf_counter()
            rank = orc.seq_rank(succ)
            tf = time.perf_counter() - t1
            key = f"seq_rank_{n}_0" if order == "random" else None
            calib = {"complete_seq_rank_s": round(tf, 2), "complete_rate": round(n / tf / 1e6, 3),
                     "unit": "M nodes/s", "sample_over_complete": round(value / (n / tf / 1e6), 3),
                     "digest_matches_reference": (sha256_i64(rank) == hashes[key]) if key in hashes else None}
            del rank
        unit = "M nodes/s"
    else:
        m = 1 << logm
        edges = orc.gen_random_graph(n, m / (n * (n - 1) // 2), 0)
        t_gen = time.perf_counter() - t0
        res = []
        for _ in range(max(1, min(a.steps, 2))):
            cpu, lab = cpu_cc_baseline(orc, n, edges, logm)
            res.append(cpu)
        value = statistics.median(r["value"] for r in res)
        ms_per_step = m / value / 1e3
        key = f"seq_components_{n}_{m}_0"
        calib = {"digest_matches_reference": (sha256_i64(lab) == hashes[key]) if key in hashes else None}
        sample = f"complete seq_components over all 2^{logm} edges, {len(res)} runs"
        unit = "M edges/s"
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": unit, "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "weak" if kind == "list" else "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic: oracle/orc.c restatement of the reference generators, seed 0", "config": config,
            "inputs": "host int64 arrays from the oracle generators (oracle/orc.c)",
            "algorithm": "seq_rank (core.py:179-186)" if kind == "list" else "seq_components (core.py:240-248)",
            "cpu_baseline": {"value": round(value, 3), "unit": unit, "cores": 1, "kind": "port", "sample": sample,
                             "host_cpus": os.cpu_count(), "calibration": calib,
                             "input_generation_s": round(t_gen, 1)},
            "e2e": {"value": round(value, 3), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        return reference_arm(a)
    return ours(a)


if __name__ == "__main__":
    main()
