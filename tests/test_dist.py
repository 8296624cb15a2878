"""Multi-GPU components orchestration (paper_1002_4482_b200/dist.py) with
world_size 2 on the gloo backend (CPU).  The device kernels are replaced by
a host test double with the same contract (init / hook / compress), so this
checks the sharding, the min all-reduce merge, the folded convergence flag,
the sharded shortcut + all-gather and the global validation reduction."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1002_4482_b200.dist import TorchDistComm, sharded_components


class HostOps:
    """CPU stand-in for CudaOps (test double; not product code)."""

    def parents(self, size):
        return torch.empty(size, dtype=torch.int32)

    def init(self, D, n):
        D[:n] = torch.arange(n, dtype=torch.int32)

    def hook(self, edges, row0, n, D, variant, validate, flags):
        e = edges.numpy().astype(np.int64).reshape(-1, 2)
        d = D.numpy()
        ok = np.ones(len(e), dtype=bool)
        if validate and len(e):
            rng = (e < 0) | (e >= n)
            bad = np.flatnonzero(rng.any(axis=1))
            if bad.size:
                flags[1] = ~torch.tensor(row0 + int(bad[0]), dtype=torch.int64)
            loops = np.flatnonzero((e[:, 0] == e[:, 1]) & ~rng.any(axis=1))
            if loops.size:
                flags[2] = ~torch.tensor(row0 + int(loops[0]), dtype=torch.int64)
            ok = ~rng.any(axis=1) & (e[:, 0] != e[:, 1])
        changed = False
        if variant == "uf":
            def find(x):
                while d[x] != x:
                    d[x] = d[d[x]]
                    x = d[x]
                return x
            for u, v in e[ok]:
                a, b = find(u), find(v)
                if a != b:
                    hi, lo = max(a, b), min(a, b)
                    d[hi] = lo
                    changed = True
        else:
            u, v = e[ok, 0], e[ok, 1]
            du, dv = d[u].astype(np.int64), d[v].astype(np.int64)
            sel = du != dv
            hi, lo = np.maximum(du, dv)[sel], np.minimum(du, dv)[sel]
            before = d.copy()
            np.minimum.at(d, hi, lo.astype(d.dtype))
            changed = bool((d != before).any())
        if changed:
            flags[0] = 1

    def changes(self, Dold, D, n, cap):
        ch = torch.nonzero(D[:n] != Dold[:n]).flatten()
        k = ch.numel()
        idx = torch.zeros(max(cap, 1), dtype=torch.int32)
        val = torch.zeros(max(cap, 1), dtype=torch.int32)
        kk = min(k, cap)
        idx[:kk] = ch[:kk].to(torch.int32)
        val[:kk] = D[ch[:kk]]
        return idx, val, torch.tensor([k], dtype=torch.int64)

    def apply_min(self, D, idx, val):
        np.minimum.at(D.numpy(), idx.numpy().astype(np.int64), val.numpy())

    def compress(self, D, lo, hi, roots):
        d = D.numpy()
        c = 0
        for i in range(lo, hi):
            r = d[i]
            while d[r] != r:
                r = d[r]
            d[i] = r
            c += int(r == i)
        roots += c


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, edges, variant, q, sparse_cap=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = len(edges)
        per = -(-m // world)
        r0 = min(rank * per, m)
        r1 = min(r0 + per, m)
        blk = torch.from_numpy(np.ascontiguousarray(edges[r0:r1]).reshape(-1, 2))
        try:
            D, info = sharded_components(n, blk, r0, TorchDistComm(), HostOps(), variant=variant, sparse_cap=sparse_cap)
            q.put((rank, "ok", D[:n].numpy().copy(), info))
        except Exception as exc:  # report to the parent
            q.put((rank, "err", type(exc).__name__, str(exc)))
    finally:
        dist.destroy_process_group()


def _run(n, edges, variant, world=2, sparse_cap=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, edges, variant, q, sparse_cap)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("variant", ["uf", "sv"])
def test_two_rank_components_match_oracle(orc, variant):
    from paper_1002_4482_b200 import gen_random_graph, gen_tree_graph

    sparse = 0
    for gr in (gen_random_graph(400, 0.004, seed=3), gen_tree_graph(600, 2, seed=1),
               gen_random_graph(3000, 0.0004, seed=5)):
        want = orc.seq_components(gr.n, gr.edges)
        for cap in (None, gr.n):  # default threshold, and always-sparse after round 1
            res = _run(gr.n, gr.edges, variant, sparse_cap=cap)
            for rank, status, D, info in res:
                assert status == "ok", D
                assert np.array_equal(D.astype(np.int64), want), (variant, rank)
                assert info["roots_per_round"][-1] == len(np.unique(want))
                assert info["rounds"] <= 30
                sparse += info.get("sparse_rounds", 0)
    if variant == "uf":
        assert sparse > 0  # rounds after the first merged only the lowered entries


def test_two_rank_edgeless(orc):
    res = _run(5, np.empty((0, 2), dtype=np.int64), "uf")
    for rank, status, D, info in res:
        assert status == "ok" and D.tolist() == [0, 1, 2, 3, 4] and info["rounds"] == 1


def test_two_rank_validation_reports_global_row():
    edges = np.array([[0, 1], [1, 2], [2, 3], [3, 9], [4, 4], [0, 4]], dtype=np.int64)
    res = _run(5, edges, "uf")
    for rank, status, name, msg in res:
        assert status == "err" and name == "InvalidGraphError"
        assert msg == "edge endpoint out of range at row 3"
    edges[3] = [3, 4]
    res = _run(5, edges, "sv")
    for rank, status, name, msg in res:
        assert status == "err" and msg == "self-loop at edge 4"
