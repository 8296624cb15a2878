"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes tests/golden/golden.npz (small arrays) and tests/golden/hashes.json
(sha256 digests of larger reference outputs).  Nothing here runs on the GPU
box; the fixtures are committed.
"""

import hashlib
import json
import os
import sys

import numpy as np

import simtgraph as ref
from simtgraph.core import chain_positions
from simtgraph.listrank import _draw_splitters

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def main():
    g = {}
    # KISS (gen.py): scalar recurrence and seeding
    st = ref.gen.KissState(1, 2, 3, 4)
    vals = []
    for _ in range(8):
        v, st = ref.gen.kiss_next(st)
        vals.append(v)
    g["kiss_1234_first8"] = np.array(vals, dtype=np.uint64)
    seeds = [0, 1, 42, 2**63, 12345678901234567]
    g["kiss_seed_seeds"] = np.array(seeds, dtype=np.uint64)
    g["kiss_seed_states"] = np.array([list(ref.kiss_seed(s)) for s in seeds], dtype=np.uint64)
    for s in seeds:
        d, st2 = ref.gen.kiss_batch(ref.kiss_seed(s), 4096)
        g[f"kiss_batch_{s}"] = d
        g[f"kiss_batch_state_{s}"] = np.array(list(st2), dtype=np.uint64)

    # lists + oracle ranks
    list_cases = [(1, 0), (2, 0), (3, 1), (10, 0), (17, 3), (300, 7), (1000, 11), (4096, 31), (5000, 21), (1 << 14, 0)]
    g["list_cases"] = np.array(list_cases, dtype=np.int64)
    for n, s in list_cases:
        sl = ref.gen_list(n, seed=s)
        g[f"list_{n}_{s}"] = sl.succ
        g[f"rank_{n}_{s}"] = ref.seq_rank(sl)

    # invalid lists: reference validate_list verdicts
    bad = [[1, 5, 2], [1, 2, 0], [0, 2, 2], [1, 0, 2], [1, 2, 2, 4, 3], [2, 2, 2], [-1, 0], [3, 4, 2, 1, 0],
           [1, 1, 3, 2]]
    g["bad_lists"] = np.array(json.dumps(bad))
    g["bad_verdicts"] = np.array(json.dumps([[v.kind, v.index] if (v := ref.validate_list(ref.SuccessorList(b)))
                                             else None for b in bad]))

    # splitter draws (listrank.py:211-231)
    spl_cases = [(10, 1, 0), (10, 4, 3), (10, 10, 1), (1000, 16, 5), (1000, 250, 9), (4096, 64, 7),
                 (2000, 32, 5), (40000, 16384, 1), (128, 128, 0), (100000, 100, 11)]
    g["spl_cases"] = np.array(spl_cases, dtype=np.int64)
    for n, r, s in spl_cases:
        g[f"spl_{n}_{r}_{s}"] = _draw_splitters(n, r, s)

    # rs_rank meta (splitter_set) for a few runs
    rs_cases = [(3, 1, 0, 0), (2000, 32, 5, 5), (5000, 64, 21, 9), (4096, 64, 31, 31)]
    g["rs_cases"] = np.array(rs_cases, dtype=np.int64)
    for n, p, ls, s in rs_cases:
        sl = ref.gen_list(n, seed=ls) if n > 3 else ref.SuccessorList([1, 2, 2])
        rank, stats = ref.rs_rank(sl, p=p, seed=s, accounting="counts")
        spl = stats.meta["splitter_set"]
        key = f"rs_{n}_{p}_{ls}_{s}"
        g[key + "_node"] = spl.splitter_node
        g[key + "_len"] = spl.sublist_len
        g[key + "_succ"] = spl.splitter_succ
        g[key + "_rank"] = spl.splitter_rank
        g[key + "_max"] = np.array(stats.meta["max_sublist"])
    sl = ref.gen_list(4096, seed=31)
    _, stats = ref.rs_rank_even(sl, p=64, accounting="counts")
    spl = stats.meta["splitter_set"]
    g["rs_even_4096_64_node"] = spl.splitter_node
    g["rs_even_4096_64_len"] = spl.sublist_len
    g["rs_even_4096_64_succ"] = spl.splitter_succ
    g["rs_even_4096_64_rank"] = spl.splitter_rank

    # graphs + oracle labels
    rg_cases = [(4, 1.0, 0), (30, 0.2, 0), (30, 0.2, 1), (200, 0.05, 0), (200, 0.05, 4), (1000, 0.01, 0),
                (1000, 0.002, 6), (3000, 0.0005, 2)]
    g["rg_cases"] = np.array(rg_cases, dtype=np.float64)
    for i, (n, d, s) in enumerate(rg_cases):
        gr = ref.gen_random_graph(n, d, seed=s)
        g[f"rg_{i}_edges"] = gr.edges
        g[f"rg_{i}_labels"] = ref.seq_components(gr)
    tr_cases = [(50, 2, 0), (300, 3, 1), (2000, 10, 2), (20000, 3, 0), (64, 2, 1)]
    g["tr_cases"] = np.array(tr_cases, dtype=np.int64)
    for i, (n, k, s) in enumerate(tr_cases):
        gr = ref.gen_tree_graph(n, k, seed=s)
        g[f"tr_{i}_edges"] = gr.edges
        g[f"tr_{i}_labels"] = ref.seq_components(gr)
    path = ref.list_to_graph(ref.gen_list(3000, seed=2))
    g["path_3000_2_edges"] = path.edges
    g["path_3000_2_labels"] = ref.seq_components(path)
    g["round_bound_n"] = np.array([1, 2, 3, 10, 1000, 10**5, 2**20, 2**22, 2**26], dtype=np.int64)
    g["round_bound"] = np.array([ref.sv_round_bound(int(n)) for n in g["round_bound_n"]], dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, "golden.npz"), **g)

    # digests of larger reference outputs (checked on the GPU box at full size)
    h = {}
    for n, s in [(1 << 20, 0), (1 << 20, 1), (1 << 22, 0)]:
        sl = ref.gen_list(n, seed=s)
        h[f"gen_list_{n}_{s}"] = sha(sl.succ)
        h[f"seq_rank_{n}_{s}"] = sha(ref.seq_rank(sl))
        print("list", n, s, file=sys.stderr)
    for n, m, s in [(1 << 16, 1 << 18, 0), (1 << 20, 1 << 22, 0), (1 << 22, 1 << 24, 0)]:
        gr = ref.gen_random_graph(n, m / (n * (n - 1) // 2), seed=s)
        assert gr.m == m
        h[f"gen_random_graph_{n}_{m}_{s}"] = sha(gr.edges)
        lab = ref.seq_components(gr)
        h[f"seq_components_{n}_{m}_{s}"] = sha(lab)
        h[f"components_{n}_{m}_{s}"] = int(len(np.unique(lab)))
        print("graph", n, m, s, file=sys.stderr)
    spl = _draw_splitters(1 << 20, 4096, 0)
    h["draw_splitters_1048576_4096_0"] = sha(spl)
    with open(os.path.join(OUT, "hashes.json"), "w") as f:
        json.dump(h, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
