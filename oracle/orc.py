"""CPU ORACLE -- test infrastructure only.

ctypes wrapper over ``oracle/liborc.so`` (``orc.c``: plain-C restatement of
the reference's sequential algorithms) plus numpy restatements of the
reference's generators and splitter draw.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
use this module, as the checker and as the timed CPU baseline; the product
package never imports it.

Each function cites the reference file:line it restates
(``/root/reference/pkg/src/simtgraph/...``).  Pinned against the reference's
golden outputs in ``tests/golden`` (see ``tests/test_oracle.py``).
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "orc.c")
LIB = os.path.join(HERE, "liborc.so")

MASK64 = (1 << 64) - 1
KINDS = {1: "out-of-range", 2: "no-tail", 3: "multiple-self-loops", 4: "unreachable"}


def build(force=False):
    """Compile liborc.so with gcc (no CUDA involved)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp"
        subprocess.run(["gcc", "-O2", "-fPIC", "-shared", "-o", tmp, SRC], check=True)
        os.replace(tmp, LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P, I64 = ctypes.c_void_p, ctypes.c_int64
        L.orc_kiss_batch.argtypes = [P, ctypes.c_uint64, P]
        L.orc_chain_positions.argtypes = [P, I64, P, P]
        L.orc_chain_positions.restype = ctypes.c_int
        L.orc_validate_list.argtypes = [P, I64, P, P]
        L.orc_validate_list.restype = ctypes.c_int
        L.orc_seq_rank.argtypes = [P, I64, P, P]
        L.orc_seq_rank.restype = ctypes.c_int
        L.orc_seq_components.argtypes = [I64, P, I64, P, P]
        L.orc_validate_graph.argtypes = [I64, P, I64, P]
        L.orc_validate_graph.restype = ctypes.c_int
        L.orc_gen_list.argtypes = [I64, P, P]
        L.orc_gen_list.restype = ctypes.c_int
        L.orc_gen_random_graph.argtypes = [I64, I64, P, P]
        L.orc_gen_random_graph.restype = ctypes.c_int
        L.orc_seq_rank_sample.argtypes = [P, I64, P, P, I64, I64, P]
        L.orc_seq_rank_sample.restype = I64
        _lib = L
    return _lib


class OracleListError(ValueError):
    pass


class OracleGraphError(ValueError):
    pass


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---- lists -----------------------------------------------------------------

def validate_list(succ):
    """(kind, index) of the first violation, (None, -1) if valid (core.py:148-167)."""
    succ = _i64(succ)
    n = succ.shape[0]
    pos = np.empty(n, dtype=np.int64)
    idx = ctypes.c_int64()
    kind = lib().orc_validate_list(succ.ctypes.data, n, ctypes.byref(idx), pos.ctypes.data)
    return (KINDS[kind] if kind else None), idx.value


def chain_positions(succ):
    """Hops from the head per node (core.py:170-176)."""
    succ = _i64(succ)
    kind, index = validate_list(succ)
    if kind:
        raise OracleListError(f"{kind} at index {index}")
    pos = np.empty(succ.shape[0], dtype=np.int64)
    bad = ctypes.c_int64()
    lib().orc_chain_positions(succ.ctypes.data, succ.shape[0], pos.ctypes.data, ctypes.byref(bad))
    return pos


def seq_rank(succ):
    """rank = (n-1) - hops from the head (core.py:179-186)."""
    succ = _i64(succ)
    rank = np.empty(succ.shape[0], dtype=np.int64)
    idx = ctypes.c_int64()
    kind = lib().orc_seq_rank(succ.ctypes.data, succ.shape[0], rank.ctypes.data, ctypes.byref(idx))
    if kind:
        raise OracleListError(f"{KINDS[kind]} at index {idx.value}")
    return rank


# ---- graphs ----------------------------------------------------------------

def validate_graph(n, edges):
    """(kind, row) -- core.py:196-206."""
    e = _i64(edges).reshape(-1, 2)
    idx = ctypes.c_int64()
    kind = lib().orc_validate_graph(int(n), e.ctypes.data, e.shape[0], ctypes.byref(idx))
    return {0: None, 1: "out-of-range", 2: "self-loop"}[kind], idx.value


def seq_components(n, edges):
    """Union-find labels = component minima (core.py:209-248)."""
    if n <= 0:
        raise OracleGraphError("graph needs at least one vertex")
    e = _i64(edges).reshape(-1, 2)
    kind, row = validate_graph(n, e)
    if kind:
        raise OracleGraphError(f"{kind} at row {row}")
    label = np.empty(n, dtype=np.int64)
    parent = np.empty(n, dtype=np.int64)
    lib().orc_seq_components(int(n), e.ctypes.data, e.shape[0], label.ctypes.data, parent.ctypes.data)
    return label


# ---- KISS + generators (gen.py) --------------------------------------------

def _splitmix64(s):
    s = (s + 0x9E3779B97F4A7C15) & MASK64
    z = s
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return s, z ^ (z >> 31)


def kiss_seed(seed):
    """gen.py:83-99"""
    s = int(seed) & MASK64
    s, x = _splitmix64(s)
    s, y = _splitmix64(s)
    s, z = _splitmix64(s)
    s, c = _splitmix64(s)
    c &= (1 << 58) - 1
    if y == 0:
        y = 362436362436362436
    if x == 0 and c == 0:
        x = 1234567890987654321
    return (x, y, z, c)


def kiss_batch(state, n):
    """gen.py:67-72 -> (uint64 draws, new state)"""
    st = np.array([int(v) & MASK64 for v in state], dtype=np.uint64)
    out = np.empty(int(n), dtype=np.uint64)
    if n:
        lib().orc_kiss_batch(st.ctypes.data, int(n), out.ctypes.data)
    return out, tuple(int(v) for v in st)


def _state(seed):
    return np.array(kiss_seed(seed), dtype=np.uint64)


def gen_list(n, seed=0):
    """gen.py:110-127: chain visiting interior nodes in KISS sort-key order
    (orc.c: KISS batch + stable LSD radix argsort)."""
    n = int(n)
    assert 1 <= n < (1 << 32)
    succ = np.empty(n, dtype=np.int64)
    st = _state(seed)
    if lib().orc_gen_list(n, st.ctypes.data, succ.ctypes.data):
        raise MemoryError("orc_gen_list: allocation failed")
    return succ


def gen_random_graph(n, d, seed=0):
    """gen.py:183-218 -> int64 (m,2) edges, rows sorted, u < v (orc.c:
    draw-order rejection sampling with a hash set, then a radix sort)."""
    n = int(n)
    cap = n * (n - 1) // 2
    m = int(round(d * cap))
    if not 0 < d <= 1 or m > cap:
        raise ValueError(f"density {d} out of range")
    edges = np.empty((m, 2), dtype=np.int64)
    st = _state(seed)
    if lib().orc_gen_random_graph(n, m, st.ctypes.data, edges.ctypes.data):
        raise MemoryError("orc_gen_random_graph: allocation failed")
    return edges


def gen_list_np(n, seed=0):
    """numpy restatement of gen.py:110-127 (cross-check of the C generator)."""
    succ = np.empty(n, dtype=np.int64)
    if n == 1:
        succ[0] = 0
        return succ
    keys, _ = kiss_batch(kiss_seed(seed), n - 1)
    order = np.concatenate([[0], 1 + np.argsort(keys, kind="stable")])
    succ[order[:-1]] = order[1:]
    succ[order[-1]] = order[-1]
    return succ


def gen_random_graph_np(n, d, seed=0):
    """numpy restatement of gen.py:183-218 (cross-check of the C generator)."""
    cap = n * (n - 1) // 2
    m = int(round(d * cap))
    state = kiss_seed(seed)
    un = np.uint64(n)
    got = np.empty(0, dtype=np.uint64)
    while got.size < m:
        need = m - got.size
        draws, state = kiss_batch(state, 2 * (need + need // 4 + 16))
        a, b = draws[0::2] % un, draws[1::2] % un
        ok = a != b
        a, b = a[ok], b[ok]
        k = np.minimum(a, b) * un + np.maximum(a, b)
        _, first = np.unique(k, return_index=True)
        k = k[np.sort(first)]
        k = k[~np.isin(k, got)]
        got = np.concatenate([got, k[:need]])
    got = np.sort(got)
    return np.stack([(got // un).astype(np.int64), (got % un).astype(np.int64)], axis=1)


def draw_splitters(n, r, seed):
    """listrank.py:211-231: head + r-1 distinct interior nodes."""
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


def splitter_set(succ, splitter_node):
    """Reference RS3/RS4 outputs for a splitter set (listrank.py:252-357):
    sublist lengths, reduced successors, global splitter ranks -- from the
    oracle ranks."""
    rank = seq_rank(succ)
    sr = rank[splitter_node]
    order = np.argsort(-sr, kind="stable")
    r = len(splitter_node)
    sub_len = np.empty(r, dtype=np.int64)
    red = np.empty(r, dtype=np.int64)
    for j in range(r):
        t = order[j]
        if j + 1 < r:
            sub_len[t] = sr[t] - sr[order[j + 1]]
            red[t] = order[j + 1]
        else:
            sub_len[t] = sr[t] + 1
            red[t] = t
    return sub_len, red, sr


# ---- CPU-baseline timing -----------------------------------------------------

class SeqRankSampler:
    """Bounded samples of seq_rank (core.py:179-186) on a full-size list:
    each call ranks the first `hops` nodes of the chain with seq_rank's
    per-node work (both dependent walks over the n-sized arrays, the scans
    and the rank fill; orc.c orc_seq_rank_sample)."""

    def __init__(self, succ):
        self.succ = _i64(succ)
        n = self.succ.shape[0]
        self.pos = np.zeros(n, dtype=np.int64)
        self.rank = np.empty(n, dtype=np.int64)
        self.pos.fill(0)            # fault the pages in outside any timed sample
        self.rank.fill(0)
        self.epoch = 0

    def __call__(self, hops):
        self.epoch += 1
        an = ctypes.c_int64()
        return int(lib().orc_seq_rank_sample(self.succ.ctypes.data, self.succ.shape[0], self.pos.ctypes.data,
                                             self.rank.ctypes.data, int(hops), self.epoch, ctypes.byref(an)))
