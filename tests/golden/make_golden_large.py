"""Digests of the reference's outputs at the benchmark sizes (C2, C3, C5).

Run once in the build container, where /root/reference exists (about 15
minutes and ~35 GB of RAM -- the reference's gen_random_graph at 2^26/2^28):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden_large.py

Merges sha256 digests (int64, C order) of
  gen_list(2^26, 0), gen_list(2^28, 0)            (gen.py:110-127)
  seq_rank of both                                (core.py:179-186)
  gen_random_graph(2^26, m=2^28, 0) edges         (gen.py:183-218)
  seq_components of it + its component count      (core.py:240-248)
into tests/golden/hashes.json.  The GPU tests (tests/test_fullsize_gpu.py)
compare the device generators and the device results with these digests.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

import simtgraph as ref

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def main():
    path = os.path.join(OUT, "hashes.json")
    with open(path) as f:
        h = json.load(f)
    only = set(sys.argv[1:])

    def save():
        with open(path, "w") as f:
            json.dump(h, f, indent=1, sort_keys=True)

    for n, s in [(1 << 26, 0), (1 << 28, 0)]:
        if only and "list" not in only:
            break
        t = time.time()
        sl = ref.gen_list(n, seed=s)
        h[f"gen_list_{n}_{s}"] = sha(sl.succ)
        tg = time.time() - t
        t = time.time()
        rank = ref.seq_rank(sl)
        tr = time.time() - t
        h[f"seq_rank_{n}_{s}"] = sha(rank)
        h[f"seq_rank_{n}_{s}_seconds"] = round(tr, 1)
        print(f"list {n} {s}: gen {tg:.1f} s, seq_rank {tr:.1f} s", file=sys.stderr, flush=True)
        del sl, rank
        save()
    for n, m, s in [(1 << 26, 1 << 28, 0)]:
        if only and "graph" not in only:
            break
        t = time.time()
        gr = ref.gen_random_graph(n, m / (n * (n - 1) // 2), seed=s)
        assert gr.m == m
        tg = time.time() - t
        h[f"gen_random_graph_{n}_{m}_{s}"] = sha(gr.edges)
        t = time.time()
        lab = ref.seq_components(gr)
        tc = time.time() - t
        h[f"seq_components_{n}_{m}_{s}"] = sha(lab)
        h[f"seq_components_{n}_{m}_{s}_seconds"] = round(tc, 1)
        h[f"components_{n}_{m}_{s}"] = int(len(np.unique(lab)))
        print(f"graph {n} {m} {s}: gen {tg:.1f} s, seq_components {tc:.1f} s", file=sys.stderr, flush=True)
        save()


if __name__ == "__main__":
    main()
