"""The API boundary's 32-bit transfers (sg_xfer.cu): long int64 host
arrays cross PCIe narrowed to 32-bit ids and come back widened, with the
reference's exact errors when a value does not fit (core.py:148-167,
196-206).  Lengths straddle the pipeline's chunk (2^22 elements) and the
NARROW_MIN threshold."""

import ctypes

import numpy as np
import pytest
import torch

import paper_1002_4482_b200 as g
from paper_1002_4482_b200 import _device, _native

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("count", [1 << 20, (1 << 22) + 5, 3 * (1 << 22) + 17])
def test_narrow_widen_round_trip(cuda, count):
    rng = np.random.default_rng(count)
    host = rng.integers(0, 2**31 - 1, count, dtype=np.int64)
    d, was_host = _device.to_device(host, cuda, bound=2**31)
    assert was_host and d.dtype == torch.int32
    assert np.array_equal(d.cpu().numpy().astype(np.int64), host)
    back = _device.to_host_numpy(d)
    assert back.dtype == np.int64 and np.array_equal(back, host)
    # a value at the bound falls back to the int64 copy (exact values kept)
    host[count - 3] = 2**31
    d, _ = _device.to_device(host, cuda, bound=2**31)
    assert d.dtype == torch.int64 and np.array_equal(d.cpu().numpy(), host)
    host[count // 2] = -1
    d, _ = _device.to_device(torch.from_numpy(host), cuda, bound=2**31)
    assert d.dtype == torch.int64 and int(d[count // 2]) == -1


def test_api_results_through_narrow_path(cuda, orc):
    n = (1 << 20) + 11
    sl = g.gen_list(n, seed=21)
    rank, _ = g.rs_rank(sl, 512)
    assert isinstance(rank, np.ndarray) and rank.dtype == np.int64
    assert np.array_equal(rank, orc.seq_rank(sl.succ))
    w, _ = g.wyllie_rank(sl, 64)
    assert np.array_equal(w, rank)
    r2, _ = g.rs_rank(g.SuccessorList(torch.from_numpy(sl.succ.copy()).pin_memory()), 512, reuse_succ=True)
    assert np.array_equal(r2, rank)
    gr = g.gen_random_graph(1 << 20, (1 << 21) / ((1 << 20) * ((1 << 20) - 1) // 2), seed=3)
    lab, _ = g.sv_components(gr, 64)
    assert lab.dtype == np.int64 and np.array_equal(lab, orc.seq_components(gr.n, gr.edges))


def test_api_errors_through_narrow_path(cuda):
    n = (1 << 20) + 3
    base = g.gen_list(n, seed=2).succ
    for i, v in ((77, n + 5), (1000, -4), (n - 9, 2**40)):
        s = base.copy()
        s[i] = v
        want = g.validate_list(g.SuccessorList(s))
        with pytest.raises(g.InvalidListError) as ei:
            g.rs_rank(g.SuccessorList(s), 64)
        assert str(ei.value) == str(want)
    e = g.gen_random_graph(1 << 20, (1 << 21) / ((1 << 20) * ((1 << 20) - 1) // 2), seed=3).edges.copy()
    e[123_456] = [5, (1 << 20) + 1]
    with pytest.raises(g.InvalidGraphError, match="out of range at row 123456"):
        g.sv_components(g.EdgeGraph(1 << 20, e), 64)


@pytest.mark.parametrize("bad", [2**31, 2**31 + 5, 2**32 + 1, 2**40, -1, -(2**31)])
def test_narrow_detects_every_out_of_range_value(cuda, bad):
    """Values outside [0, bound) anywhere (vector body, unaligned head,
    scalar tail) fall back to the exact int64 copy; values just below the
    bound narrow."""
    count = (1 << 22) + 7
    bound = count
    rng = np.random.default_rng(3)
    base = rng.integers(0, bound, count + 1, dtype=np.int64)
    base[5] = bound - 1
    for view in (base[:count], base[1:]):  # 16-B aligned and unaligned starts
        d, _ = _device.to_device(view, cuda, bound=bound)
        assert d.dtype == torch.int32 and np.array_equal(d.cpu().numpy().astype(np.int64), view)
        for pos in (0, 1, 2, 3, 4, 1000, count // 2 + 1, count - 2, count - 1):
            v = view.copy()
            v[pos] = bad
            d, _ = _device.to_device(v, cuda, bound=bound)
            assert d.dtype == torch.int64, (bad, pos)
            assert np.array_equal(d.cpu().numpy(), v)
    v = base[:count].copy()
    v[77] = bound  # exactly the bound
    d, _ = _device.to_device(v, cuda, bound=bound)
    assert d.dtype == torch.int64


def test_widen_into_unaligned_and_odd_arrays(cuda):
    for count in ((1 << 22) + 3, (1 << 21) + 1):
        x = torch.randint(0, 2**31 - 1, (count,), dtype=torch.int32, device=cuda)
        back = _device.to_host_numpy(x)
        assert back.dtype == np.int64 and np.array_equal(back, x.cpu().numpy().astype(np.int64))
