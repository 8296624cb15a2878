"""The edge-sharded CUDA path with two ranks (concomp.py:225-240).

Two processes share cuda:0 (NCCL refuses two ranks on one device, and the
box has one GPU), each driving the real ``CudaOps`` -- ``sg_cc_hook_part``,
``sg_cc_changes`` / ``sg_cc_apply_min``, ``sg_cc_compress`` -- through
``sv_components_dist``.  The collectives are gloo's, staged through host
copies of the CUDA tensors (test infrastructure, ``_HostStagedComm``); the
merge semantics are the product's.  Labels must equal the reference's
``seq_components`` (C4 digest, tree family through the oracle), the sparse
changed-entry rounds must run, and a bad row in rank 1's block must be
reported with its global row on both ranks."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sha(a):
    import hashlib

    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    import paper_1002_4482_b200 as g
    from oracle import orc
    from paper_1002_4482_b200 import dist as sgdist

    class _HostStagedComm(sgdist.TorchDistComm):
        """gloo collectives over host copies of CUDA tensors (test only)."""

        def _run(self, t, op):
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)

        def allreduce_min_(self, t):
            self._run(t, dist.ReduceOp.MIN)

        def allreduce_max_(self, t):
            self._run(t, dist.ReduceOp.MAX)

        def allreduce_sum_(self, t):
            self._run(t, dist.ReduceOp.SUM)

        def allgather_(self, full, chunk):
            h = torch.empty(full.shape, dtype=full.dtype)
            dist.all_gather_into_tensor(h, chunk.cpu(), group=self.group)
            full.copy_(h)

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    comm = _HostStagedComm()
    res = {}
    try:
        n, m = 1 << 22, 1 << 24
        gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=dev)
        for variant in ("uf", "sv"):
            # sparse_cap = n: every round after the first exchanges changed entries
            lab, st = sgdist.sv_components_dist(gr, 64, variant=variant, comm=comm, sparse_cap=n)
            res[f"c4_{variant}"] = {"sha": _sha(lab), "rounds": st.meta["rounds"],
                                    "sparse_rounds": st.meta["sparse_rounds"],
                                    "names": sorted({r.kernel for r in st.launch_log}),
                                    "components": int(st.meta["roots_per_round"][-1])}
        tr = g.gen_tree_graph(70_000, 3, seed=2)
        want = orc.seq_components(tr.n, tr.edges)
        for variant in ("uf", "sv"):
            lab, st = sgdist.sv_components_dist(tr, 8, variant=variant, comm=comm, sparse_cap=tr.n)
            res[f"tree_{variant}"] = {"equal": bool(np.array_equal(lab, want)), "rounds": st.meta["rounds"],
                                      "sparse_rounds": st.meta["sparse_rounds"]}
        e = g.gen_random_graph(60_000, 5e-5, seed=4).edges.copy()
        bad_row = len(e) - 10   # in rank 1's block
        e[bad_row] = [9, 9]
        try:
            sgdist.sv_components_dist(g.EdgeGraph(60_000, e), 8, comm=comm)
            res["invalid"] = "no error"
        except g.InvalidGraphError as ex:
            res["invalid"] = str(ex)
        res["bad_row"] = bad_row
    finally:
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
            json.dump(res, f)
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu(cuda, hashes, tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    out = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(world)]
    n, m = 1 << 22, 1 << 24
    for r, res in enumerate(out):
        for variant in ("uf", "sv"):
            c = res[f"c4_{variant}"]
            assert c["sha"] == hashes[f"seq_components_{n}_{m}_0"], (r, variant)
            assert c["components"] == hashes[f"components_{n}_{m}_0"]
            assert c["sparse_rounds"] >= 1, (r, variant, c)
            assert {"nccl_allgather_changes", "nccl_allreduce_min", "cc_shortcut"} <= set(c["names"]), c["names"]
            t = res[f"tree_{variant}"]
            assert t["equal"], (r, variant)
        assert res["invalid"] == f"self-loop at edge {res['bad_row']}", res["invalid"]
    # replicas agree and the round count does not depend on the rank
    assert out[0]["c4_uf"]["rounds"] == out[1]["c4_uf"]["rounds"]
