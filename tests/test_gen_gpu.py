"""Device input generation bit-exact with the reference generators."""

import hashlib

import numpy as np
import pytest
import torch

import paper_1002_4482_b200 as g
from paper_1002_4482_b200 import gen

pytestmark = pytest.mark.gpu


def sha(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


@pytest.mark.parametrize("n", [1, 5, 4095, 4096, 100_003, 1 << 20])
def test_device_kiss_matches_host(cuda, n):
    st = g.kiss_seed(12345)
    d, st_d = gen.kiss_batch_device(st, n, cuda)
    h, st_h = g.kiss_batch(st, n)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), h)
    assert tuple(st_d) == tuple(st_h)


def test_device_gen_list_matches_reference(cuda, golden):
    for n, s in golden["list_cases"].tolist():
        sl = g.gen_list(n, seed=s, device=cuda)
        assert sl.on_device
        assert np.array_equal(sl.succ.cpu().numpy(), golden[f"list_{n}_{s}"]), (n, s)


def test_device_gen_random_graph_matches_reference(cuda, golden, hashes):
    for i, (n, d, s) in enumerate(golden["rg_cases"].tolist()):
        gr = g.gen_random_graph(int(n), d, seed=int(s), device=cuda)
        assert np.array_equal(gr.edges.cpu().numpy(), golden[f"rg_{i}_edges"]), (n, d, s)
    n, m = 1 << 20, 1 << 22
    gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=cuda)
    assert sha(gr.edges) == hashes[f"gen_random_graph_{n}_{m}_0"]


def test_device_gen_list_digest(cuda, hashes):
    sl = g.gen_list(1 << 22, seed=0, device=cuda)
    assert sha(sl.succ) == hashes["gen_list_4194304_0"]
    sl32 = g.gen_list(1 << 20, seed=1, device=cuda, dtype=torch.int32)
    assert sl32.succ.dtype == torch.int32
    assert sha(sl32.succ) == hashes["gen_list_1048576_1"]
