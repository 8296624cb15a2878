"""Connected components on the B200: drop-in for ``simtgraph.concomp``
(``/root/reference/pkg/src/simtgraph/concomp.py``).

``sv_components(graph, p, ...)`` keeps the reference's signature, return
value ``(labels int64[n], ExecStats)`` (labels = smallest vertex of each
component, core.py:240-257), ``meta`` keys and errors.  Underneath
(``csrc/sg_cc.cu``) the stored edge list is streamed as (u, v) pairs with
both orientations handled in registers:

* ``variant="uf"`` (default): one hook sweep of CAS root hooking with path
  halving (every edge is united when the sweep ends) + one shortcut sweep.
* ``variant="sv"``: the Shiloach-Vishkin round structure -- conditional
  min-hooking with atomicMin, then a root-chasing shortcut to stars, until a
  round changes nothing (concomp.py:225-240).

Both keep D[i] <= i, so roots are component minima and no relabel pass is
needed.  Multi-GPU edge sharding lives in ``dist.py``.
"""

import ctypes
from collections import namedtuple

import numpy as np
import torch

from . import _device, _native
from .core import EdgeGraph, InvalidGraphError
from .listrank import _machine_error

VARIANTS = {"uf": _native.SG_CC_UF, "sv": _native.SG_CC_SV}


def sv_round_bound(n):
    """Worst-case rounds: floor(log_{3/2} n) + 2, in integers (concomp.py:27-32)."""
    k = 0
    while 3 ** (k + 1) <= n * 2 ** (k + 1):
        k += 1
    return k + 2


def _graph_error_message(kind, row):
    if kind == 1:
        return f"edge endpoint out of range at row {row}"
    return f"self-loop at edge {row}"


def sv_components(graph, p, backend="simulated", accounting="full", block_size=256, seed=0, workers=None,
                  variant="uf"):
    """Label the connected components; returns (labels, ExecStats)
    (concomp.py:208-246).  Labels are the smallest vertex id of each
    component, bit-identical to ``seq_components``.  ``variant`` selects the
    device algorithm (``"uf"`` or ``"sv"``); the result does not depend on it.
    """
    if graph.n <= 0:
        raise InvalidGraphError("graph needs at least one vertex")
    n = graph.n
    m = graph.m
    p = int(p)
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    err = ValueError(f"more threads ({p}) than vertices ({n})") if p > n else _machine_error(
        p, block_size, backend, accounting)
    if n >= 0x7FFFFFFF:
        from .core import CapabilityError
        raise CapabilityError(f"device vertex ids are 31-bit here: n={n} is too large")
    bound = sv_round_bound(n)
    dev = _device.require_cuda(graph.edges.device if isinstance(graph.edges, torch.Tensor)
                               and graph.edges.is_cuda else None)
    with torch.cuda.device(dev):
        if m:
            edges, host_input = _device.to_device(graph.edges, dev, bound=n)
        else:
            edges, host_input = torch.empty((0, 2), dtype=torch.int64, device=dev), not graph.on_device
        ldt = _device.host_out_dtype(n) if host_input else (torch.int64 if edges.dtype == torch.int64 else edges.dtype)
        labels = torch.empty(n, dtype=ldt, device=dev)
        L = _native.lib()
        ws = _device.workspace(L.sg_cc_workspace_bytes(n, m), dev)
        st = _native.Stats()
        viol = _native.Violation()
        code = VARIANTS[variant] if err is None else _native.SG_CC_UF
        rc = L.sg_cc(_device.ptr(edges), _device.dtype_code(edges), m, n, _device.ptr(labels),
                     _device.dtype_code(labels), code, bound, _device.ptr(ws), ws.numel(),
                     _device.stream_ptr(dev), ctypes.byref(st), ctypes.byref(viol))
        del ws
    if rc == _native.SG_ERR_INVALID_GRAPH:
        raise InvalidGraphError(_graph_error_message(viol.kind, int(viol.index)))
    if err is not None:
        raise err
    if rc == _native.SG_ERR_RUNTIME:
        raise RuntimeError(f"no convergence after {bound} rounds (bound {bound})")
    _native.check(rc, "sg_cc")
    stats = _device.exec_stats(st)
    stats.rounds = int(st.rounds)
    stats.meta.update(n=n, p=p, m_stored=m, oriented_m=2 * m, rounds=int(st.rounds), round_bound=bound,
                      roots_per_round=[int(st.roots_per_round[k]) for k in range(st.n_roots)],
                      variant=variant, edge_sweeps=int(st.edge_sweeps), vertex_sweeps=int(st.vertex_sweeps),
                      backend=backend, accounting=accounting, block_size=block_size, seed=seed, workers=workers)
    if host_input:
        return _device.to_host_numpy(labels), stats
    return labels, stats


RoundProfile = namedtuple("RoundProfile", ["rows", "sv23_read_dominated"])

# global reads per item of each launch, the reference's counting rule
# (concomp.py:249-271 sums ctx.read elements): a hook reads the stored edge
# (2 ids) and both parents; the partition reads the edge; a shortcut or label
# pass reads D[i] and D[D[i]]; collectives read nothing on the SMs
_READS_PER_ITEM = {"cc_hook_uf": 4, "cc_hook_sv": 4, "cc_partition": 2, "cc_shortcut": 2, "cc_labels": 2}


def round_profile(stats):
    """Per-launch table of a components run (concomp.py:249-271): round,
    kernel, reads, writes, transactions (the reference's row keys; reads from
    the per-item model above, writes and transactions live in ncu, 0 here),
    plus items and device ms.  The flag says whether the hooking kernels
    account for the majority of all global reads, as the reference's
    ``sv23_read_dominated`` does for its SV2 + SV3."""
    rows = []
    hook = other = 0
    for rec in stats.launch_log:
        c = rec.counters
        reads = c.reads or _READS_PER_ITEM.get(rec.kernel, 0) * c.items
        rows.append({"round": rec.round, "kernel": rec.kernel, "reads": reads, "writes": c.writes,
                     "transactions": c.transactions, "items": c.items, "ms": rec.ms})
        if rec.kernel.startswith("cc_hook"):
            hook += reads
        else:
            other += reads
    return RoundProfile(rows, hook > other)
