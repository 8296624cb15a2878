"""List ranking on the B200: drop-in for ``simtgraph.listrank``
(``/root/reference/pkg/src/simtgraph/listrank.py``).

Same entry points, signatures, return values ``(rank int64[n], ExecStats)``,
``meta`` keys and error conventions; the work runs in libsg's sm_100a
kernels (``csrc/sg_list.cu``):

* ``wyllie_rank``  -- pointer jumping over packed {rank, succ} words
  (``variant="multi_kernel"``: ceil(log2 n) launches; ``"single_block"``:
  one CTA with block barriers).
* ``rs_rank`` / ``rs_rank_even`` -- sparse ruling set, recursive.  The
  reference's ``p`` is its splitter/thread count on a simulated 2009 GPU; it
  is kept as the splitter set reported in ``meta["splitter_set"]``
  (identical to the reference: same KISS draw, sublist lengths, reduced
  successors, splitter ranks), derived from the device ranks.  The device
  walks its own hashed ruling set, sized for 148 SMs, so performance does
  not hinge on ``p``.

Backend / accounting / workers select the reference's simulator; they are
validated exactly like ``vkm.Machine`` (vkm.py:434-454) and recorded in
``meta``, but execution is always the CUDA path (no CPU fallback).
"""

import ctypes
import functools
import collections
import math
import weakref
from collections import namedtuple
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _native
from .core import (
    P48_MAX_THREADS,
    CapabilityError,
    InvalidListError,
    ListViolation,
    Packing,
    SuccessorList,
    VIOLATION_KINDS,
)
from .gen import kiss_batch, kiss_seed

MAX_BLOCK_SIZE = 768            # vkm.py:41
SM_COUNT = 27                   # the reference's simulated device (core.py:313-314)
CORES_PER_SM = 8
DEFAULT_P = 4 * SM_COUNT * CORES_PER_SM   # vkm.py:46


def _jump_rounds(n):
    """ceil(log2 n), 0 for n <= 1 (listrank.py:38-40)."""
    return max(0, int(n - 1).bit_length()) if n > 1 else 0


@dataclass
class SplitterSet:
    """Everything known about the r splitters (listrank.py:43-50)."""
    r: int
    splitter_node: np.ndarray
    sublist_len: np.ndarray = None
    splitter_succ: np.ndarray = None
    splitter_rank: np.ndarray = None


SublistStats = namedtuple("SublistStats", ["max_len", "mean_len", "histogram"])


def sublist_stats(splitters):
    """Max/mean/histogram of sub-list lengths (listrank.py:64-69)."""
    lens = np.asarray(splitters.sublist_len, dtype=np.int64)
    hist = np.bincount(lens)
    return SublistStats(int(lens.max()), lens.sum() / lens.size, hist)


# ---------------------------------------------------------------------------
# argument checks, in the reference's order

def _machine_error(p, block_size, backend, accounting):
    """The ValueErrors vkm.Machine / GridConfig raise (vkm.py:58-62, 436-439)."""
    if backend not in ("simulated", "threaded"):
        return ValueError(f"unknown backend {backend!r}")
    if accounting not in ("full", "counts"):
        return ValueError(f"unknown accounting mode {accounting!r}")
    if p < 1:
        return ValueError("need at least one thread")
    if not 1 <= block_size <= MAX_BLOCK_SIZE:
        return ValueError(f"block size must be in [1, {MAX_BLOCK_SIZE}]")
    return None


def _as_packing(packing):
    if isinstance(packing, Packing):
        return packing
    return Packing(str(packing).lower())


def _rs_param_error(n, p, packing, block_size, backend, accounting):
    """_rs_pipeline checks (listrank.py:388-393), then Machine's."""
    if packing is Packing.P48 and p > P48_MAX_THREADS:
        return CapabilityError(f"48-bit packing cannot be invoked with more than {P48_MAX_THREADS} threads (got {p})")
    if p > n:
        return ValueError(f"more threads ({p}) than nodes ({n})")
    return _machine_error(p, block_size, backend, accounting)


# ---------------------------------------------------------------------------
# device calls

def _raise_invalid(sl, code, viol):
    """Turn a device-reported invalid list into the reference's exact
    InvalidListError message (the index comes from the host validator)."""
    kind, index = _native.list_violation_host(sl.host_succ())
    if kind == 0:  # device and host disagree -- should not happen
        kind, index = viol.kind, viol.index
    raise InvalidListError(str(ListViolation(VIOLATION_KINDS.get(kind, "unreachable"), int(index))))


class _PinnedPool:
    """Pinned int64 host blocks for meta["splitter_set"], recycled: a block is
    lent to one call, its result arrays are views of it, and it returns to the
    pool when the last of those views is gone (weakref.finalize on the numpy
    array every view hangs off).  A fresh block from torch's caching pinned
    allocator costs a cudaHostAlloc (~1.5 ms) whenever that cache runs dry
    (measured: every few calls), and copying the result out of one shared
    block costs ~100 us per call."""

    def __init__(self):
        # no lock: the finalizer can run inside any allocation of any thread
        # (a lock taken here could be re-entered by it); deque append / pop
        # and dict.setdefault are atomic under the GIL
        self.free = {}

    def take(self, count):
        try:
            return self.free[count].pop()
        except (KeyError, IndexError):
            return torch.empty(count, dtype=torch.int64, pin_memory=True)

    def lend(self, block, count, shape):
        """numpy view of `block` whose death returns `block` to the pool."""
        own = block.numpy()
        weakref.finalize(own, self._give_back, count, block)
        return own[:count].reshape(shape)

    def _give_back(self, count, block):
        q = self.free.setdefault(count, collections.deque())
        if len(q) < 8:
            q.append(block)


_META_POOL = _PinnedPool()


def _run_list(kind, sl, variant_code, seed, reuse_succ, scratch_out=False, meta=None):
    """Rank `sl` on the GPU.  Returns (rank tensor, native stats, status,
    violation, host_input).  `meta` = (spl_nodes, cache key) asks the ruling
    set call for meta["splitter_set"] in the same device pass; its host copy
    is returned through meta_out (a list) as a (3, r) int64 array."""
    n = sl.n
    if n >= 0xFFFFFFFF:
        raise CapabilityError(f"device node ids are 32-bit: n={n} is too large")
    dev = _device.require_cuda(sl.succ.device if isinstance(sl.succ, torch.Tensor) and sl.succ.is_cuda else None)
    with torch.cuda.device(dev):
        succ, host_input = _device.to_device(sl.succ, dev, bound=n)
        if reuse_succ and not scratch_out:
            rank = succ  # ranks overwrite the (device copy of the) successors, listrank.py:186-187
        else:
            odt = _device.host_out_dtype(n) if host_input else (
                torch.int64 if succ.dtype == torch.int64 else succ.dtype)
            rank = torch.empty(n, dtype=odt, device=dev)
        st = _native.Stats()
        viol = _native.Violation()
        L = _native.lib()
        sdt = _device.dtype_code(succ)
        odt = _device.dtype_code(rank)
        stream = _device.stream_ptr(dev)
        if kind == "wyllie":
            ws = _device.workspace(L.sg_wyllie_workspace_bytes(n), dev)
            rc = L.sg_wyllie_rank(_device.ptr(succ), sdt, _device.ptr(rank), odt, n, variant_code, _device.ptr(ws),
                                  ws.numel(), stream, ctypes.byref(st), ctypes.byref(viol))
        else:
            ws = _device.workspace(L.sg_rs_workspace_bytes(n), dev)
            if meta is None:
                rc = L.sg_rs_rank(_device.ptr(succ), sdt, _device.ptr(rank), odt, n, int(seed) & (2**64 - 1),
                                  _device.ptr(ws), ws.numel(), stream, ctypes.byref(st), ctypes.byref(viol))
            else:
                spl_nodes, key, meta_out = meta
                r = len(spl_nodes)
                idx = _device_index(spl_nodes, dev, key)
                res = torch.empty((3, r), dtype=torch.int64, device=dev)
                # a persistent pinned staging block per device: a fresh block from
                # torch's caching pinned allocator costs a cudaHostAlloc (~1.5 ms)
                # whenever its cache runs dry (measured: every few calls); the
                # result is copied out after the call (3r int64, ~20 us)
                mws = _device.workspace(L.sg_splitter_meta_workspace_bytes(r), dev)
                host = _META_POOL.take(3 * r)  # this call's own block (recycled, see _PinnedPool)
                rc = L.sg_rs_rank_meta(_device.ptr(succ), sdt, _device.ptr(rank), odt, n, int(seed) & (2**64 - 1),
                                       _device.ptr(ws), ws.numel(), _device.ptr(idx), r, _device.ptr(res),
                                       ctypes.c_void_p(host.data_ptr()), _device.ptr(mws), mws.numel(), stream,
                                       ctypes.byref(st), ctypes.byref(viol))
                meta_out.append(_META_POOL.lend(host, 3 * r, (3, r)))
        del ws
    if rc not in (_native.SG_OK, _native.SG_ERR_INVALID_LIST):
        _native.check(rc, f"sg_{kind}_rank")
    return rank, st, rc, viol, host_input


def _finish_rank(rank, host_input):
    if host_input:
        return _device.to_host_numpy(rank)
    return rank


# ---------------------------------------------------------------------------
# Wyllie

def wyllie_rank(sl, p, variant="multi_kernel", backend="simulated", accounting="full", block_size=256, seed=0,
                workers=None):
    """Rank a list by pointer jumping; returns (rank array, ExecStats)
    (listrank.py:75-155).

    ``multi_kernel``: init + ceil(log2 n) jump launches over packed 64-bit
    {rank, succ} words; ``single_block``: one CTA, block barriers between
    rounds, requires p <= block_size.
    """
    n = sl.n
    p = int(p)
    err = _machine_error(p, block_size, backend, accounting)
    if err is None:
        if variant == "single_block" and p > block_size:
            err = CapabilityError(f"single-block variant limited to {block_size} threads, got {p}")
        elif variant not in ("multi_kernel", "single_block"):
            err = ValueError(f"unknown variant {variant!r}")
    code = _native.SG_WY_SINGLE_BLOCK if (err is None and variant == "single_block") else _native.SG_WY_MULTI_KERNEL
    rank, st, rc, viol, host_input = _run_list("wyllie", sl, code, seed, False, scratch_out=err is not None)
    if rc == _native.SG_ERR_INVALID_LIST:
        _raise_invalid(sl, rc, viol)
    if err is not None:
        raise err
    stats = _device.exec_stats(st)
    rounds = _jump_rounds(n)
    stats.rounds = rounds
    stats.meta.update(n=n, p=p, variant=variant, rounds=rounds, backend=backend, accounting=accounting,
                      block_size=block_size, seed=seed, workers=workers)
    return _finish_rank(rank, host_input), stats


# ---------------------------------------------------------------------------
# ruling set

# draws and device index copies are cached only up to this many splitters
# (64 cached entries x 512 KiB at most, host and HBM); larger p is redrawn
_CACHE_MAX_R = 1 << 16


def _draw_splitters(n, r, seed):
    """Copy of the reference's splitter draw (deterministic in its
    arguments; cached for r <= _CACHE_MAX_R)."""
    if int(r) > _CACHE_MAX_R:
        return _draw_splitters_uncached(int(n), int(r), int(seed))
    return _draw_splitters_cached(int(n), int(r), int(seed))  # read-only, shared by the calls that drew it


@functools.lru_cache(maxsize=64)
def _draw_splitters_cached(n, r, seed):
    a = _draw_splitters_uncached(n, r, seed)
    a.setflags(write=False)
    return a




def _draw_splitters_uncached(n, r, seed):
    """Head plus r-1 distinct random interior nodes, reproducible by seed
    (listrank.py:211-231): KISS rejection sampling in batches, or a random
    ordering of all interior nodes when more than half of them are needed."""
    if r == 1:
        return np.zeros(1, dtype=np.int64)
    state = kiss_seed(seed)
    if r - 1 > (n - 1) // 2:
        keys, _ = kiss_batch(state, n - 1)
        picks = 1 + np.argsort(keys, kind="stable")[: r - 1]
    else:
        chosen = np.empty(0, dtype=np.int64)
        while chosen.size < r - 1:
            need = (r - 1) - chosen.size
            draws, state = kiss_batch(state, need + need // 3 + 16)
            cand = 1 + (draws % np.uint64(n - 1)).astype(np.int64)
            _, first = np.unique(cand, return_index=True)
            cand = cand[np.sort(first)]
            cand = cand[~np.isin(cand, chosen)]
            chosen = np.concatenate([chosen, cand[:need]])
        picks = chosen
    return np.concatenate([[0], picks]).astype(np.int64)


_IDX_CACHE = {}


def _device_index(spl_nodes, dev, key):
    """Device copy of a splitter-node array; cached when `key` names a
    deterministic draw (n, p, seed)."""
    if key is None or len(spl_nodes) > _CACHE_MAX_R:
        return torch.from_numpy(np.array(spl_nodes, dtype=np.int64)).to(dev)  # (a copy: the cached draw is read-only)
    key = (str(dev),) + tuple(key)
    t = _IDX_CACHE.get(key)
    if t is None:
        if len(_IDX_CACHE) > 32:
            _IDX_CACHE.clear()
        t = torch.from_numpy(np.array(spl_nodes, dtype=np.int64)).to(dev)  # (a copy: the cached draw is read-only)
        _IDX_CACHE[key] = t
    return t


def _splitter_set(rank, spl_nodes, n, key=None):
    """meta["splitter_set"] from the device ranks: splitter ranks are global
    ranks (listrank.py:355-356); in list order (descending rank) each
    sublist runs to the next splitter, the last one to the tail
    (listrank.py:252-299).  One device sort, one D2H copy."""
    dev = rank.device
    r = len(spl_nodes)
    idx = _device_index(spl_nodes, dev, key)
    L = _native.lib()
    res = torch.empty((3, r), dtype=torch.int64, device=dev)   # rank, sublist length, reduced successor
    ws = _device.workspace(L.sg_splitter_meta_workspace_bytes(r), dev)
    _native.check(L.sg_splitter_meta(_device.ptr(rank), _device.dtype_code(rank), n, _device.ptr(idx), r,
                                     _device.ptr(res), _device.ptr(ws), ws.numel(), _device.stream_ptr(dev)),
                  "sg_splitter_meta")
    host = res.cpu().numpy()
    out = SplitterSet(r, np.ascontiguousarray(spl_nodes, dtype=np.int64))
    out.splitter_rank = host[0]
    out.sublist_len = host[1]
    out.splitter_succ = host[2]
    return out


def _rs(sl, p, packing, seed, backend, accounting, block_size, workers, reuse_succ, even):
    n = sl.n
    p = int(p)
    packing = _as_packing(packing)
    err = _rs_param_error(n, p, packing, block_size, backend, accounting)
    meta = None
    if not even and err is None and 0 < p < n and n < 0xFFFFFFFF:
        meta = (_draw_splitters(n, p, seed), (n, p, int(seed)), [])
    rank, st, rc, viol, host_input = _run_list("rs", sl, 0, seed, reuse_succ, scratch_out=err is not None, meta=meta)
    if rc == _native.SG_ERR_INVALID_LIST:
        _raise_invalid(sl, rc, viol)
    if err is not None:
        raise err
    stats = _device.exec_stats(st)
    if p > 1 and p * math.log2(p) > n:
        stats.warnings.append("super-linear work regime: p*lg(p) > n")
        stats.meta["superlinear"] = True
    if p > block_size:
        # the reference's reduced list is wider than one block, so its RS4
        # runs one launch per jump round (listrank.py:343-346); the device
        # ranks its own ruler levels either way, the flag keeps the meta
        stats.meta["rs4_fallback"] = True
    if even:
        # perfect splitters every n/p chain positions (listrank.py:431-436):
        # node at chain position k has rank n-1-k
        # (one streaming pass on the device, sg_even_splitters: p writes instead of an n-long position array)
        dnodes = torch.empty(p, dtype=torch.int64, device=rank.device)
        _native.check(_native.lib().sg_even_splitters(_device.ptr(rank), _device.dtype_code(rank), n, p,
                                                      _device.ptr(dnodes), _device.stream_ptr(rank.device)),
                      "sg_even_splitters")
        spl_nodes = dnodes.cpu().numpy()
        splitters = _splitter_set(rank, spl_nodes, n)
    elif meta is not None and meta[2]:
        host = meta[2][0]
        splitters = SplitterSet(p, np.ascontiguousarray(meta[0], dtype=np.int64))
        splitters.splitter_rank, splitters.sublist_len, splitters.splitter_succ = host[0], host[1], host[2]
    else:
        spl_nodes = _draw_splitters(n, p, seed)
        splitters = _splitter_set(rank, spl_nodes, n, key=(n, p, int(seed)))
    stats.meta.update(n=n, p=p, packing=packing.value, splitter_set=splitters,
                      max_sublist=int(splitters.sublist_len.max()),
                      levels=int(st.levels), level_size=[int(st.level_size[k]) for k in range(st.levels + 1)],
                      fallback=bool(st.fallback),
                      path="wyllie" if st.fallback else ("contract" if st.list_path == 1 else "ruling_set"),
                      backend=backend, accounting=accounting,
                      block_size=block_size, seed=seed, workers=workers)
    return _finish_rank(rank, host_input), stats


def rs_rank(sl, p, packing=Packing.P64, seed=0, backend="simulated", accounting="full", block_size=256,
            workers=None, reuse_succ=False):
    """Random-splitter list ranking; returns (rank array, ExecStats)
    (listrank.py:411-419).  ``meta["splitter_set"]`` holds the reference's p
    KISS-drawn splitters (``_draw_splitters(n, p, seed)``) with their sublist
    lengths, reduced-list successors and global ranks."""
    return _rs(sl, p, packing, seed, backend, accounting, block_size, workers, reuse_succ, even=False)


def rs_rank_even(sl, p, packing=Packing.P64, seed=0, backend="simulated", accounting="full", block_size=256,
                 workers=None, reuse_succ=False):
    """As rs_rank, with perfect splitters every n/p chain positions
    (listrank.py:422-438).  The reference finds them with a sequential
    pre-walk; here they come from the device ranks."""
    n = sl.n
    if n % p != 0:
        raise ValueError(f"even splitters need p | n (p={p}, n={n})")
    return _rs(sl, p, packing, seed, backend, accounting, block_size, workers, reuse_succ, even=True)
