"""Reproducible input generators, bit-identical to the reference's
(``/root/reference/pkg/src/simtgraph/gen.py``), with a device path for the
sizes the benchmark needs.

KISS64 (gen.py:30-64) = multiply-with-carry + xorshift + LCG.  Each part has
a closed-form jump-ahead, which lets the device generate the stream in
independent chunks that agree draw-for-draw with the sequential recurrence:

* LCG  z' = A z + C (mod 2^64): compose the affine map by squaring;
* xorshift: linear over GF(2)^64 -> powers of its 64x64 bit matrix;
* MWC with base b = 2^64 and multiplier a = 2^58 + 1: y = c*b + x satisfies
  y' = a*y mod p with the prime p = a*b - 1, so y_k = a^k y_0 mod p.
"""

from collections import namedtuple

import numpy as np

from . import _native
from .core import EdgeGraph, SuccessorList

MASK64 = (1 << 64) - 1

DEFAULT_X = 1234567890987654321
DEFAULT_Y = 362436362436362436
DEFAULT_Z = 1066149217761810
DEFAULT_C = 123456123456123456

KissState = namedtuple("KissState", ["x", "y", "z", "c"])
DEFAULT_STATE = KissState(DEFAULT_X, DEFAULT_Y, DEFAULT_Z, DEFAULT_C)

_LCG_A = 6906969069
_LCG_C = 1234567
_MWC_A = (1 << 58) + 1
_MWC_P = _MWC_A * (1 << 64) - 1


def kiss_next(state):
    """One KISS step on plain integers: (value, new state) (gen.py:30-48)."""
    x, y, z, c = state
    t = ((x << 58) + c) & MASK64
    c = x >> 6
    x = (x + t) & MASK64
    c += x < t
    y ^= (y << 13) & MASK64
    y ^= y >> 17
    y ^= (y << 43) & MASK64
    z = (_LCG_A * z + _LCG_C) & MASK64
    return (x + y + z) & MASK64, KissState(x, y, z, c)


def kiss_batch(state, n):
    """n draws at once on the host: (uint64 array, new state) (gen.py:67-72)."""
    out, st = _native.kiss_batch_host(tuple(state), int(n))
    return out, KissState(*st)


def _splitmix64(s):
    s = (s + 0x9E3779B97F4A7C15) & MASK64
    z = s
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return s, z ^ (z >> 31)


def kiss_seed(seed):
    """Expand one integer seed into a KissState via splitmix64 (gen.py:83-99)."""
    s = int(seed) & MASK64
    s, x = _splitmix64(s)
    s, y = _splitmix64(s)
    s, z = _splitmix64(s)
    s, c = _splitmix64(s)
    c &= (1 << 58) - 1
    if y == 0:
        y = DEFAULT_Y
    if x == 0 and c == 0:
        x = DEFAULT_X
    return KissState(x, y, z, c)


def kiss_split(seed, stream):
    """Independent state for (seed, stream) pairs (gen.py:102-104)."""
    return kiss_seed((int(seed) ^ ((int(stream) + 1) * 0xD1B54A32D192ED03)) & MASK64)


# ---------------------------------------------------------------------------
# jump-ahead

def _xs_step(y):
    y ^= (y << 13) & MASK64
    y ^= y >> 17
    y ^= (y << 43) & MASK64
    return y


def _mat_apply(cols, y):
    r = 0
    j = 0
    while y:
        if y & 1:
            r ^= cols[j]
        y >>= 1
        j += 1
    return r


def _mat_mul(a, b):
    """columns of a∘b"""
    return [_mat_apply(a, col) for col in b]


_XS_POW = [[_xs_step(1 << j) for j in range(64)]]   # _XS_POW[i] = T^(2^i)


def _xs_pow2(i):
    while len(_XS_POW) <= i:
        m = _XS_POW[-1]
        _XS_POW.append(_mat_mul(m, m))
    return _XS_POW[i]


def _xs_jump(y, k):
    i = 0
    while k:
        if k & 1:
            y = _mat_apply(_xs_pow2(i), y)
        k >>= 1
        i += 1
    return y


def _xs_matrix(k):
    """T^k as columns."""
    cols = [1 << j for j in range(64)]
    i = 0
    while k:
        if k & 1:
            cols = _mat_mul(_xs_pow2(i), cols)
        k >>= 1
        i += 1
    return cols


def _lcg_affine(k):
    """(A_k, C_k) with z_k = A_k z_0 + C_k."""
    a, c = 1, 0
    ba, bc = _LCG_A, _LCG_C
    while k:
        if k & 1:
            a, c = (ba * a) & MASK64, (ba * c + bc) & MASK64
        ba, bc = (ba * ba) & MASK64, (ba * bc + bc) & MASK64
        k >>= 1
    return a, c


def kiss_jump(state, k):
    """State after k steps of the recurrence, in O(log k)."""
    x, y, z, c = state
    k = int(k)
    if k == 0:
        return KissState(x, y, z, c)
    ymwc = (c << 64) | x
    ymwc = (pow(_MWC_A, k, _MWC_P) * ymwc) % _MWC_P
    a, cc = _lcg_affine(k)
    return KissState(ymwc & MASK64, _xs_jump(y, k), (a * z + cc) & MASK64, ymwc >> 64)


def kiss_chunk_states(state, chunks, chunk_len):
    """Start states of `chunks` consecutive chunks of `chunk_len` draws,
    as a (chunks, 4) uint64 array."""
    out = np.empty((chunks, 4), dtype=np.uint64)
    mx = pow(_MWC_A, chunk_len, _MWC_P)
    xs = _xs_matrix(chunk_len)
    la, lc = _lcg_affine(chunk_len)
    x, y, z, c = state
    ymwc = (c << 64) | x
    for k in range(chunks):
        out[k] = (ymwc & MASK64, y, z, ymwc >> 64)
        ymwc = (mx * ymwc) % _MWC_P
        y = _mat_apply(xs, y)
        z = (la * z + lc) & MASK64
    return out


def kiss_batch_device(state, n, device=None):
    """n KISS draws generated on the GPU: (uint64 draws as an int64 CUDA
    tensor holding the same bits, new state)."""
    import torch

    from . import _device

    dev = _device.require_cuda(device)
    n = int(n)
    out = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    if n == 0:
        return out[:0], KissState(*state)
    chunks = int(min(max(1, n // 4096), 16384))
    chunk_len = -(-n // chunks)
    chunks = -(-n // chunk_len)
    states = torch.from_numpy(kiss_chunk_states(state, chunks, chunk_len).view(np.int64)).to(dev)
    rc = _native.lib().sg_kiss_device(_device.ptr(states), chunks, chunk_len, n, _device.ptr(out),
                                      _device.stream_ptr(dev))
    _native.check(rc, "sg_kiss_device")
    return out[:n], kiss_jump(state, n)


# ---------------------------------------------------------------------------
# generators

def gen_list(n, seed=0, device=None, dtype=None):
    """Uniformly shuffled chain over n nodes, head 0, tail self-looped
    (gen.py:110-127).  ``device="cuda"`` builds it in HBM (int64 unless
    ``dtype`` says otherwise) and returns a device-resident SuccessorList."""
    assert n >= 1
    n = int(n)
    if device is None:
        succ = np.empty(n, dtype=np.int64)
        if n == 1:
            succ[0] = 0
            return SuccessorList(succ)
        keys, _ = kiss_batch(kiss_seed(seed), n - 1)
        order = np.empty(n, dtype=np.int64)
        order[0] = 0
        order[1:] = 1 + np.argsort(keys, kind="stable")
        succ[order[:-1]] = order[1:]
        succ[order[-1]] = order[-1]
        return SuccessorList(succ)
    import torch

    from . import _device

    dev = _device.require_cuda(device)
    dtype = dtype or torch.int64
    succ = torch.empty(n, dtype=dtype, device=dev)
    if n == 1:
        succ.zero_()
        return SuccessorList(succ)
    keys, _ = kiss_batch_device(kiss_seed(seed), n - 1, dev)
    # unsigned order == signed order after flipping the sign bit
    keys ^= torch.tensor(-(1 << 63), dtype=torch.int64, device=dev)
    perm = torch.sort(keys, stable=True).indices
    del keys
    rc = _native.lib().sg_list_from_order(_device.ptr(perm), n, _device.ptr(succ), _device.dtype_code(succ),
                                          _device.stream_ptr(dev))
    _native.check(rc, "sg_list_from_order")
    return SuccessorList(succ)


def ordered_list(n, device=None, dtype=None):
    """succ = [1, 2, ..., n-1, n-1]: the coalesced best case."""
    if device is None:
        succ = np.arange(1, n + 1, dtype=np.int64)
        succ[-1] = n - 1
        return SuccessorList(succ)
    import torch

    succ = torch.arange(1, n + 1, dtype=dtype or torch.int64, device=device)
    succ[-1] = n - 1
    return SuccessorList(succ)


TREE_SIZE_TARGET = 10_000


def _build_forest(n, t, k, draws):
    """Attach each vertex to a uniformly chosen parent with a free child slot
    (gen.py:133-159)."""
    edges = np.empty((n - t, 2), dtype=np.int64)
    base, rem = divmod(n, t)
    d = draws.tolist()
    e = 0
    offset = 0
    for ti in range(t):
        size = base + (1 if ti < rem else 0)
        children = [0] * size
        slots = [0]
        for j in range(1, size):
            idx = d[offset + j] % len(slots)
            parent = slots[idx]
            edges[e, 0] = offset + parent
            edges[e, 1] = offset + j
            e += 1
            children[parent] += 1
            if children[parent] == k:
                slots[idx] = slots[-1]
                slots.pop()
            slots.append(j)
        offset += size
    return edges


def gen_tree_graph(n, k, seed=0):
    """Forest of random trees, at most k children per vertex, ids scrambled
    (gen.py:162-180)."""
    assert n >= 1 and k >= 1
    t = max(1, n // TREE_SIZE_TARGET)
    draws, state = kiss_batch(kiss_seed(seed), n)
    edges = _build_forest(n, t, k, draws)
    keys, _ = kiss_batch(state, n)
    perm = np.argsort(keys, kind="stable")
    return EdgeGraph(n, perm[edges])


def _edge_count(n, d):
    if not 0 < d <= 1:
        raise ValueError(f"density must be in (0, 1], got {d}")
    capacity = n * (n - 1) // 2
    m = int(round(d * capacity))
    if m > capacity:
        raise ValueError(f"density {d} asks for {m} edges but only {capacity} exist")
    return m


def gen_random_graph(n, d, seed=0, device=None):
    """m = round(d * n(n-1)/2) distinct undirected non-loop edges, rows sorted
    with u < v (gen.py:183-218).  Batches of KISS pairs are drawn; self-loop
    draws are dropped, repeats keep their first occurrence in draw order, and
    batches are topped up until m distinct edges exist.  ``device="cuda"``
    draws, deduplicates and sorts in HBM and returns a device EdgeGraph."""
    assert n >= 1
    m = _edge_count(n, d)
    state = kiss_seed(seed)
    if device is None:
        un = np.uint64(n)
        seen = np.empty(0, dtype=np.uint64)
        while seen.size < m:
            need = m - seen.size
            draws, state = kiss_batch(state, 2 * (need + need // 4 + 16))
            u = draws[0::2] % un
            v = draws[1::2] % un
            keep = u != v
            lo = np.minimum(u[keep], v[keep])
            hi = np.maximum(u[keep], v[keep])
            keys = lo * un + hi
            _, first = np.unique(keys, return_index=True)
            fresh = keys[np.sort(first)]
            fresh = fresh[~np.isin(fresh, seen)]
            seen = np.concatenate([seen, fresh[:need]])
        keys = np.sort(seen)
        return EdgeGraph(n, np.stack([(keys // un).astype(np.int64), (keys % un).astype(np.int64)], axis=1))
    import torch

    from . import _device

    dev = _device.require_cuda(device)
    seen = torch.empty(0, dtype=torch.int64, device=dev)
    lib = _native.lib()
    while seen.numel() < m:
        need = m - seen.numel()
        ndraw = 2 * (need + need // 4 + 16)
        draws, state = kiss_batch_device(state, ndraw, dev)
        pairs = ndraw // 2
        keys = torch.empty(pairs, dtype=torch.int64, device=dev)
        _native.check(lib.sg_edge_keys(_device.ptr(draws), pairs, n, _device.ptr(keys), _device.stream_ptr(dev)),
                      "sg_edge_keys")
        del draws
        keys = keys[keys >= 0]                      # drop self-loop draws
        sk, idx = torch.sort(keys, stable=True)
        first = torch.ones_like(sk, dtype=torch.bool)
        first[1:] = sk[1:] != sk[:-1]
        keep = torch.zeros_like(first)
        keep[idx[first]] = True                     # first occurrence of each key
        del sk, idx, first
        if seen.numel():
            keep &= ~torch.isin(keys, seen)
        fresh = keys[keep]
        seen = torch.cat([seen, fresh[:need]])
        del keys, keep, fresh
    keys = torch.sort(seen).values
    del seen
    edges = torch.empty((m, 2), dtype=torch.int64, device=dev)
    _native.check(lib.sg_edges_from_keys(_device.ptr(keys), m, n, _device.ptr(edges), _device.stream_ptr(dev)),
                  "sg_edges_from_keys")
    return EdgeGraph(n, edges)
