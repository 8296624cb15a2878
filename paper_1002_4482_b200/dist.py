"""Edge-sharded connected components over several GPUs (one process per GPU,
``torch.distributed`` over NCCL / NVLink).

SURVEY §8e: the stored edge list is cut into G contiguous row blocks; each
rank keeps a full replica of the parent array D (u32, D[i] <= i).  A round is

1. local hook over the rank's edge block (``sg_cc_hook``; UF: CAS root
   hooking on the current forest, SV: conditional min-hook on stars);
2. ``all_reduce(MIN)`` of D -- hooks only ever lower parents, so the
   element-wise minimum of the G proposals is itself a valid forest with
   D[i] <= i; word n carries 1 - changed, so convergence rides the same
   collective;
3. (SV, and the final round) a sharded shortcut: rank g chases roots for its
   n/G slice of the merged D (static during the chase), then
   ``all_gather_into_tensor`` restores the replica.

The loop ends after a round in which no rank hooked anything; then every
edge joins vertices of one tree, so the roots are the component minima.
Round 1 also validates the edge blocks (first bad row reduced with MAX of
~row, as in the single-GPU kernel).

The collective and the kernels are injected (``comm``, ``ops``) so the
orchestration is tested with the gloo backend on CPU (tests/test_dist.py);
the product path uses ``CudaOps`` + NCCL.
"""

import contextlib
import ctypes
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _device, _native
from .concomp import _graph_error_message, sv_round_bound
from .core import EdgeGraph, ExecStats, InvalidGraphError, KernelCounters, LaunchRecord

_NO_ROW = 1 << 62


class TorchDistComm:
    """Collectives over a torch.distributed process group."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce_min_(self, t):
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)

    def allreduce_max_(self, t):
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)

    def allreduce_sum_(self, t):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def allgather_(self, full, chunk):
        dist.all_gather_into_tensor(full, chunk, group=self.group)


class CudaOps:
    """Device kernels of one rank (libsg C ABI on the current CUDA stream).

    The rank's edge block is split once by vertex window (``sg_cc_hook_part``,
    validating rows on the way) into a workspace that later rounds re-hook
    from, so every round's parent gathers stay L2-resident."""

    def __init__(self, device):
        self.device = device
        self.lib = _native.lib()
        self.ws = None
        self.parted = None  # (data_ptr, m) of the block held in ws

    def stream(self):
        return _device.stream_ptr(self.device)

    def parents(self, size):
        return torch.empty(size, dtype=torch.int32, device=self.device)

    def init(self, D, n):
        _native.check(self.lib.sg_cc_init(_device.ptr(D), n, self.stream()), "sg_cc_init")

    def hook(self, edges, row0, n, D, variant, validate, flags):
        code = _native.SG_CC_UF if variant == "uf" else _native.SG_CC_SV
        m = edges.shape[0]
        if self.ws is None:
            self.ws = _device.workspace(self.lib.sg_cc_hook_workspace_bytes(n, m), self.device)
        key = (edges.data_ptr(), m)
        reuse = int(self.parted == key and not validate)
        rc = self.lib.sg_cc_hook_part(_device.ptr(edges), _device.dtype_code(edges), m, row0, n, _device.ptr(D),
                                      code, int(validate), _device.ptr(flags), _device.ptr(self.ws), self.ws.numel(),
                                      reuse, self.stream())
        _native.check(rc, "sg_cc_hook_part")
        self.parted = key

    def compress(self, D, lo, hi, roots):
        _native.check(self.lib.sg_cc_compress(_device.ptr(D), lo, hi, _device.ptr(roots), self.stream()),
                      "sg_cc_compress")

    def changes(self, Dold, D, n, cap):
        """(idx, val, count tensor) of the entries i < n this rank lowered."""
        idx = torch.empty(max(cap, 1), dtype=torch.int32, device=self.device)
        val = torch.empty(max(cap, 1), dtype=torch.int32, device=self.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
        _native.check(self.lib.sg_cc_changes(_device.ptr(Dold), _device.ptr(D), n, _device.ptr(idx), _device.ptr(val),
                                             cap, _device.ptr(cnt), self.stream()), "sg_cc_changes")
        return idx, val, cnt

    def apply_min(self, D, idx, val):
        _native.check(self.lib.sg_cc_apply_min(_device.ptr(D), _device.ptr(idx), _device.ptr(val), idx.numel(),
                                               self.stream()), "sg_cc_apply_min")

    def synchronize(self):
        torch.cuda.synchronize(self.device)


class _NoTrace:
    @contextlib.contextmanager
    def span(self, name):
        yield


class CudaTrace:
    """CUDA events around every kernel / collective of the sharded rounds ->
    ExecStats launch records."""

    def __init__(self):
        self.spans = []

    @contextlib.contextmanager
    def span(self, name):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        yield
        b.record()
        self.spans.append((name, a, b))


def sharded_components(n, edges, row0, comm, ops, variant="uf", round_bound=None, trace=None, sparse_cap=None):
    """Run the sharded rounds.  `edges` is this rank's (m_g, 2) block whose
    first row is global row `row0`.  Returns (D replica as int32 tensor of
    size >= n, info dict)."""
    trace = trace or _NoTrace()
    if variant not in ("uf", "sv"):
        raise ValueError(f"unknown variant {variant!r}")
    G = comm.world
    bound = sv_round_bound(n) if round_bound is None else round_bound
    S = -(-(n + 1) // G)              # slice length; padded replica holds the flag word at index n
    npad = S * G
    D = ops.parents(npad)
    ops.init(D, npad)
    lo = comm.rank * S
    hi = min(lo + S, n)
    flags = torch.zeros(4, dtype=torch.int64, device=D.device)
    roots = torch.zeros(1, dtype=torch.int64, device=D.device)
    info = {"rounds": 0, "roots_per_round": [n], "edge_sweeps": 0, "vertex_sweeps": 0,
            "allreduce_bytes": 0, "allgather_bytes": 0, "comm_s": 0.0}
    # sparse merge while every rank lowered at most n/8/G entries
    cap = max(1, (n // 8) // G) if sparse_cap is None else max(1, int(sparse_cap))
    sparse = hasattr(ops, "changes")
    r = 0
    while True:
        r += 1
        if r > bound:
            raise RuntimeError(f"no convergence after {r - 1} rounds (bound {bound})")
        flags.zero_()
        Dold = D.clone() if (sparse and r > 1 and G > 1) else None
        with trace.span("cc_hook_uf" if variant == "uf" else "cc_hook_sv"):
            ops.hook(edges, row0, n, D, variant, r == 1, flags)
        info["edge_sweeps"] += 1
        if r == 1:
            # kernel flags hold ~row (0 = none); reduce the first bad global row
            f = flags[1:3]
            bad = torch.where(f != 0, torch.bitwise_not(f), torch.full_like(f, _NO_ROW))
            comm.allreduce_min_(bad)
            b = bad.cpu().tolist()
            if b[0] != _NO_ROW or b[1] != _NO_ROW:
                kind, row = (1, b[0]) if b[0] != _NO_ROW else (2, b[1])
                raise InvalidGraphError(_graph_error_message(kind, row))
        # one UF sweep unites every edge of the block, so a single rank is
        # done after round 1 (the single-GPU path's one-sweep argument)
        changed = int(flags[0].item()) and not (variant == "uf" and G == 1)
        t0 = time.perf_counter()
        if Dold is not None:
            # replicas are identical after the previous merge: exchange only
            # the entries this round lowered (hooks and path halving), padded
            # to the largest rank's count; dense if that is too many
            idx, val, cnt = ops.changes(Dold, D, n, cap)
            hdr = torch.stack([cnt[0], torch.tensor(int(changed), dtype=torch.int64, device=D.device)])
            comm.allreduce_max_(hdr)
            kmax, any_changed = (int(x) for x in hdr.cpu().tolist())
            converged = any_changed == 0
            if not converged and kmax <= cap:
                k = int(cnt.item())
                if kmax > k:  # pad: (0, int32 max) is a no-op min on D[0] == 0
                    idx[k:kmax] = 0
                    val[k:kmax] = 0x7FFFFFFF
                gi = torch.empty(G * kmax, dtype=torch.int32, device=D.device)
                gv = torch.empty(G * kmax, dtype=torch.int32, device=D.device)
                with trace.span("nccl_allgather_changes"):
                    comm.allgather_(gi, idx[:kmax].contiguous())
                    comm.allgather_(gv, val[:kmax].contiguous())
                ops.apply_min(D, gi, gv)
                info["sparse_rounds"] = info.get("sparse_rounds", 0) + 1
                info["allgather_bytes"] += 2 * G * kmax * 4
            elif not converged:
                with trace.span("nccl_allreduce_min"):
                    comm.allreduce_min_(D)
                info["allreduce_bytes"] += D.numel() * D.element_size()
        else:
            D[n] = 0 if changed else 1
            with trace.span("nccl_allreduce_min"):
                comm.allreduce_min_(D)
            info["allreduce_bytes"] += D.numel() * D.element_size()
            converged = int(D[n].item()) == 1
        info["comm_s"] += time.perf_counter() - t0
        if variant == "sv" or converged:
            roots.zero_()
            with trace.span("cc_shortcut"):
                ops.compress(D, lo, hi, roots)
            info["vertex_sweeps"] += 1
            t0 = time.perf_counter()
            with trace.span("nccl_allgather"):
                comm.allgather_(D, D[comm.rank * S:(comm.rank + 1) * S].clone())
                comm.allreduce_sum_(roots)
            info["comm_s"] += time.perf_counter() - t0
            info["allgather_bytes"] += D.numel() * D.element_size()
            if variant == "sv" or converged:
                info["roots_per_round"].append(int(roots.item()))
        info["rounds"] = r
        if converged:
            break
    return D, info


def sv_components_dist(graph, p, group=None, variant="uf", backend="simulated", accounting="full",
                       block_size=256, seed=0, workers=None, shard=None, comm=None, sparse_cap=None):
    """Edge-sharded ``sv_components`` across the ranks of `group`.

    Every rank calls it with the same graph (host or its own device copy) --
    or with its own block of rows via ``shard=(row0, edges_block)`` -- and
    gets the full int64 label array (replicated) plus ExecStats.  `comm`
    replaces the group's collectives (any object with TorchDistComm's
    methods); `sparse_cap` overrides the changed-entry exchange's per-rank
    cap (default n/8/G).
    """
    if graph is not None and graph.n <= 0:
        raise InvalidGraphError("graph needs at least one vertex")
    comm = comm or TorchDistComm(group)
    dev = _device.require_cuda()
    n = graph.n
    if shard is None:
        m = graph.m
        per = -(-m // comm.world)
        row0 = min(comm.rank * per, m)
        row1 = min(row0 + per, m)
        edges = graph.edges[row0:row1]
    else:
        row0, edges = shard
    edges, _ = _device.to_device(edges if edges.shape[0] else np.empty((0, 2), np.int64), dev, bound=n)
    if int(p) > n:
        raise ValueError(f"more threads ({p}) than vertices ({n})")
    ops = CudaOps(dev)
    trace = CudaTrace()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    start.record()
    D, info = sharded_components(n, edges, int(row0), comm, ops, variant=variant, trace=trace, sparse_cap=sparse_cap)
    stop.record()
    stop.synchronize()
    labels = D[:n].to(torch.int64)
    stats = ExecStats(backend="sm_100a")
    for k, (name, a, b) in enumerate(trace.spans):
        ms = a.elapsed_time(b)
        stats.launch_log.append(LaunchRecord(kernel=name, counters=KernelCounters(launches=1, ms=ms), round=k, ms=ms))
    stats.barriers = max(0, len(stats.launch_log) - 1)
    stats.rounds = info["rounds"]
    stats.wall_time = start.elapsed_time(stop) / 1e3
    stats.meta.update(n=n, p=int(p), m_stored=graph.m, oriented_m=2 * graph.m, rounds=info["rounds"],
                      round_bound=sv_round_bound(n), roots_per_round=info["roots_per_round"], variant=variant,
                      edge_sweeps=info["edge_sweeps"], vertex_sweeps=info["vertex_sweeps"], world=comm.world,
                      allreduce_bytes=info["allreduce_bytes"], allgather_bytes=info["allgather_bytes"],
                      sparse_rounds=info.get("sparse_rounds", 0))
    if isinstance(graph.edges, torch.Tensor) and graph.edges.is_cuda:
        return labels, stats
    return labels.cpu().numpy(), stats


# ---------------------------------------------------------------------------
# one process, G GPUs: the C ABI's sg_cc_multi

_COMMS = {}


def _nccl_comms(devs):
    """One NCCL clique per device tuple (ncclCommInitAll through libsg),
    created on first use and kept for the process."""
    key = tuple(devs)
    c = _COMMS.get(key)
    if c is None:
        G = len(devs)
        c = (ctypes.c_void_p * G)()
        d = (ctypes.c_int * G)(*devs)
        _native.check(_native.lib().sg_nccl_comms_init(G, d, c), "sg_nccl_comms_init")
        _COMMS[key] = c
    return c


def sv_components_multi(graph, p, devices=None, variant="uf", backend="simulated", accounting="full",
                        block_size=256, seed=0, workers=None):
    """Edge-sharded ``sv_components`` over several GPUs driven by this one
    process (``sg_cc_multi``: per-device hook sweeps, NCCL min all-reduce per
    round, sharded shortcut + all-gather; concomp.py:225-240).  `devices`:
    CUDA device indices (default: all).  Returns the labels like
    ``sv_components`` (numpy int64 for a host graph, a tensor on the first
    device for a device graph) and ExecStats."""
    if graph.n <= 0:
        raise InvalidGraphError("graph needs at least one vertex")
    n, m = graph.n, graph.m
    if int(p) > n:
        raise ValueError(f"more threads ({p}) than vertices ({n})")
    if variant not in ("uf", "sv"):
        raise ValueError(f"unknown variant {variant!r}")
    devs = list(range(torch.cuda.device_count())) if devices is None else [int(d) for d in devices]
    if not devs:
        raise RuntimeError("sv_components_multi needs at least one CUDA device")
    G = len(devs)
    L = _native.lib()
    per = -(-m // G)
    shards, ws, labels, streams = [], [], [], []
    for g, d in enumerate(devs):
        dev = torch.device("cuda", d)
        r0, r1 = min(g * per, m), min((g + 1) * per, m)
        blk = graph.edges[r0:r1]
        if isinstance(blk, torch.Tensor) and blk.is_cuda and blk.device != dev:
            blk = blk.to(dev)
        e, _ = _device.to_device(blk if blk.shape[0] else np.empty((0, 2), np.int64), dev, bound=n)
        shards.append(e)
        ws.append(_device.workspace(L.sg_cc_multi_workspace_bytes(n, r1 - r0, G), dev))
        labels.append(torch.empty(n, dtype=torch.int64, device=dev))
        streams.append(_device.stream_ptr(dev))
    dt = _device.dtype_code(shards[0])
    if any(_device.dtype_code(e) != dt for e in shards):  # one shard fell back to int64: use int64 everywhere
        shards = [e.to(torch.int64) for e in shards]
        dt = _device.dtype_code(shards[0])
    arr = lambda ty, xs: (ty * G)(*xs)  # noqa: E731
    st = _native.Stats()
    viol = _native.Violation()
    rc = L.sg_cc_multi(G, arr(ctypes.c_int, devs), arr(ctypes.c_void_p, [_device.ptr(e) for e in shards]), dt,
                       arr(ctypes.c_uint64, [e.shape[0] for e in shards]), n,
                       arr(ctypes.c_void_p, [_device.ptr(t) for t in labels]), _native.SG_I64,
                       _native.SG_CC_UF if variant == "uf" else _native.SG_CC_SV, sv_round_bound(n),
                       arr(ctypes.c_void_p, [_device.ptr(w) for w in ws]), arr(ctypes.c_size_t, [w.numel() for w in ws]),
                       _nccl_comms(devs), arr(ctypes.c_void_p, streams), ctypes.byref(st), ctypes.byref(viol))
    if rc == _native.SG_ERR_INVALID_GRAPH:
        raise InvalidGraphError(_graph_error_message(viol.kind, int(viol.index)))
    if rc == _native.SG_ERR_RUNTIME:
        raise RuntimeError(f"no convergence within {sv_round_bound(n)} rounds")
    _native.check(rc, "sg_cc_multi")
    stats = ExecStats(backend="sm_100a")
    stats.rounds = int(st.rounds)
    roots = [int(st.roots_per_round[k]) for k in range(st.n_roots)]
    stats.meta.update(n=n, p=int(p), m_stored=m, oriented_m=2 * m, rounds=int(st.rounds), round_bound=sv_round_bound(n),
                      roots_per_round=roots, variant=variant, edge_sweeps=int(st.edge_sweeps),
                      vertex_sweeps=int(st.vertex_sweeps), world=G, devices=devs, backend=backend,
                      accounting=accounting, block_size=block_size, seed=seed, workers=workers)
    if isinstance(graph.edges, torch.Tensor) and graph.edges.is_cuda:
        return labels[0], stats
    return labels[0].cpu().numpy(), stats
