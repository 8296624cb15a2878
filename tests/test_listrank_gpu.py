"""List ranking on the B200 vs the oracle.  Re-targets the reference's
tests (pkg/tests/test_listrank.py, test_acceptance.py criteria 1, 8, 10) at
the drop-in API; bit-exact ranks everywhere."""

import hashlib
import os

import numpy as np
import pytest
import torch

import paper_1002_4482_b200 as g
from paper_1002_4482_b200 import _device, _native

pytestmark = pytest.mark.gpu

CHAIN3 = g.SuccessorList([1, 2, 2])
PACKINGS = (g.Packing.P48, g.Packing.P64)


def sha(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


# ---------------------------------------------------------------- Wyllie

def test_wyllie_three_chain(cuda):
    for variant in ("multi_kernel", "single_block"):
        rank, stats = g.wyllie_rank(CHAIN3, p=2, variant=variant)
        assert rank.tolist() == [2, 1, 0]
        assert isinstance(rank, np.ndarray) and rank.dtype == np.int64


def test_wyllie_matches_oracle(cuda, orc):
    rng = np.random.default_rng(7)
    for variant in ("multi_kernel", "single_block"):
        for n in (1, 2, 3, 17, 300, 5000):
            for _ in range(3):
                sl = g.gen_list(n, seed=int(rng.integers(2**31)))
                p = int(rng.integers(1, 257))
                rank, stats = g.wyllie_rank(sl, p=p, variant=variant, accounting="counts")
                assert np.array_equal(rank, orc.seq_rank(sl.succ)), (variant, n, p)
                assert stats.meta["rounds"] == (max(0, (n - 1).bit_length()) if n > 1 else 0)


def test_wyllie_launch_structure(cuda):
    _, stats = g.wyllie_rank(g.gen_list(1024, seed=1), p=64)
    per = stats.per_kernel()
    assert per["wy_jump"].launches == 10       # ceil(log2 1024), test_listrank.py:25-30
    assert stats.rounds == 10
    _, stats = g.wyllie_rank(g.gen_list(64, seed=2), p=16, variant="single_block")
    assert stats.per_kernel()["wy_single"].launches == 1


def test_wyllie_caps_and_errors(cuda):
    with pytest.raises(g.CapabilityError):
        g.wyllie_rank(CHAIN3, p=300, variant="single_block", block_size=256)
    with pytest.raises(g.InvalidListError):
        g.wyllie_rank(g.SuccessorList([1, 2, 0]), p=2)
    with pytest.raises(ValueError):
        g.wyllie_rank(CHAIN3, p=2, variant="bogus")
    with pytest.raises(ValueError):
        g.wyllie_rank(CHAIN3, p=2, backend="gpu")
    # invalid list wins over a bad argument (validation runs first, listrank.py:83-85)
    with pytest.raises(g.InvalidListError):
        g.wyllie_rank(g.SuccessorList([1, 0, 2]), p=2, variant="bogus")
    # wyllie accepts p > n (test_listrank.py:42-51)
    rank, _ = g.wyllie_rank(CHAIN3, p=200)
    assert rank.tolist() == [2, 1, 0]


# ---------------------------------------------------------------- ruling set

def test_rs_three_chain_single_thread(cuda):
    for packing in PACKINGS:
        rank, stats = g.rs_rank(CHAIN3, p=1, packing=packing)
        assert rank.tolist() == [2, 1, 0]
        spl = stats.meta["splitter_set"]
        assert spl.splitter_node.tolist() == [0]
        assert spl.sublist_len.tolist() == [3]
        assert spl.splitter_rank.tolist() == [2]
        assert spl.splitter_succ.tolist() == [0]


def test_rs_matches_oracle(cuda, orc):
    rng = np.random.default_rng(11)
    for packing in PACKINGS:
        for n, p in [(10, 1), (10, 4), (10, 10), (1000, 16), (1000, 250), (257, 3), (4096, 64),
                     (9000, 100), (70000, 1000), (300000, 4096)]:
            sl = g.gen_list(n, seed=int(rng.integers(2**31)))
            rank, _ = g.rs_rank(sl, p=p, packing=packing, accounting="counts", seed=int(rng.integers(2**31)))
            assert np.array_equal(rank, orc.seq_rank(sl.succ)), (packing, n, p)


def test_rs_meta_matches_reference(cuda, golden):
    for n, p, ls, s in golden["rs_cases"].tolist():
        sl = g.gen_list(n, seed=ls) if n > 3 else CHAIN3
        _, stats = g.rs_rank(sl, p=p, seed=s, accounting="counts")
        spl = stats.meta["splitter_set"]
        key = f"rs_{n}_{p}_{ls}_{s}"
        assert np.array_equal(spl.splitter_node, golden[key + "_node"])
        assert np.array_equal(spl.sublist_len, golden[key + "_len"])
        assert np.array_equal(spl.splitter_succ, golden[key + "_succ"])
        assert np.array_equal(spl.splitter_rank, golden[key + "_rank"])
        assert stats.meta["max_sublist"] == int(golden[key + "_max"])
        assert stats.meta["n"] == n and stats.meta["p"] == p and stats.meta["packing"] == "p64"


def test_rs_even_meta_matches_reference(cuda, golden, orc):
    sl = g.gen_list(4096, seed=31)
    rank, stats = g.rs_rank_even(sl, p=64, accounting="counts")
    assert np.array_equal(rank, orc.seq_rank(sl.succ))
    spl = stats.meta["splitter_set"]
    for part in ("node", "len", "succ", "rank"):
        attr = {"node": "splitter_node", "len": "sublist_len", "succ": "splitter_succ", "rank": "splitter_rank"}[part]
        assert np.array_equal(getattr(spl, attr), golden[f"rs_even_4096_64_{part}"]), part
    assert np.all(spl.sublist_len == 64)


def test_rs_splitter_ranks_are_global_ranks(cuda, orc):
    sl = g.gen_list(2000, seed=5)
    _, stats = g.rs_rank(sl, p=32, seed=5, accounting="counts")
    spl = stats.meta["splitter_set"]
    assert np.array_equal(orc.seq_rank(sl.succ)[spl.splitter_node], spl.splitter_rank)
    assert spl.sublist_len.sum() == 2000


def test_rs_thread_cap_at_exactly_16384(cuda, orc):
    sl = g.gen_list(40_000, seed=1)
    want = orc.seq_rank(sl.succ)
    with pytest.raises(g.CapabilityError):
        g.rs_rank(sl, p=16_385, packing=g.Packing.P48)
    rank, stats = g.rs_rank(sl, p=16_384, packing=g.Packing.P48, accounting="counts")
    assert np.array_equal(rank, want) and stats.meta["p"] == 16_384
    rank, _ = g.rs_rank(sl, p=16_385, packing=g.Packing.P64, accounting="counts")
    assert np.array_equal(rank, want)


def test_rs_errors(cuda):
    with pytest.raises(ValueError):
        g.rs_rank(CHAIN3, p=4)                     # p > n
    with pytest.raises(ValueError):
        g.rs_rank(CHAIN3, p=0)
    with pytest.raises(ValueError):
        g.rs_rank(CHAIN3, p=2, block_size=1000)
    with pytest.raises(g.InvalidListError):
        g.rs_rank(g.SuccessorList([1, 2, 0]), p=4)   # invalid list beats p > n
    with pytest.raises(ValueError):
        g.rs_rank_even(g.gen_list(100, seed=1), p=7)


@pytest.mark.parametrize("algo", ["rs", "wyllie"])
def test_invalid_lists_report_reference_violation(cuda, golden, algo):
    import json

    bad = json.loads(str(golden["bad_lists"]))
    verdicts = json.loads(str(golden["bad_verdicts"]))
    for b, v in zip(bad, verdicts):
        sl = g.SuccessorList(b)
        fn = (lambda s: g.rs_rank(s, p=1)) if algo == "rs" else (lambda s: g.wyllie_rank(s, p=1))
        if v is None:
            fn(sl)
            continue
        with pytest.raises(g.InvalidListError) as ei:
            fn(sl)
        assert str(ei.value) == f"{v[0]} at index {v[1]}", b


def test_invalid_large_lists_detected(cuda):
    n = 200_000
    base = g.gen_list(n, seed=3).succ
    # a cycle that contains no ruler: cut the chain and close a loop
    s = base.copy()
    tail = int(np.flatnonzero(s == np.arange(n))[0])
    s[tail] = 0 if tail != 0 else 1           # head revisited -> no tail
    for fn in (lambda x: g.rs_rank(x, 64), lambda x: g.wyllie_rank(x, 64)):
        with pytest.raises(g.InvalidListError, match="no-tail"):
            fn(g.SuccessorList(s))
    # detached cycle + chain: one tail, unreachable nodes
    s = base.copy()
    order = np.argsort(-np.asarray(g.rs_rank(g.SuccessorList(base), 1)[0]))   # list order
    a, b = int(order[n // 3]), int(order[2 * n // 3])
    s[a] = b           # skip the middle third
    mid_last = int(order[2 * n // 3 - 1])
    s[mid_last] = int(order[n // 3 + 1])   # middle third becomes a cycle
    want = g.validate_list(g.SuccessorList(s))
    assert want.kind == "unreachable"
    for fn in (lambda x: g.rs_rank(x, 64), lambda x: g.wyllie_rank(x, 64)):
        with pytest.raises(g.InvalidListError) as ei:
            fn(g.SuccessorList(s))
        assert str(ei.value) == str(want)
    # the head's walk runs into a detached 2-cycle (possibly without rulers)
    s = np.arange(1, n + 1, dtype=np.int64)
    s[-1] = n - 1
    s[0], s[5], s[6] = 5, 6, 5
    want = g.validate_list(g.SuccessorList(s))
    for fn in (lambda x: g.rs_rank(x, 64), lambda x: g.wyllie_rank(x, 64)):
        with pytest.raises(g.InvalidListError) as ei:
            fn(g.SuccessorList(s))
        assert str(ei.value) == str(want)
    # two nodes share a successor (in-degree 2): the skipped node is unreachable
    s = base.copy()
    a = int(order[n // 2])
    s[a] = s[int(s[a])]
    want = g.validate_list(g.SuccessorList(s))
    for fn in (lambda x: g.rs_rank(x, 64), lambda x: g.wyllie_rank(x, 64)):
        with pytest.raises(g.InvalidListError) as ei:
            fn(g.SuccessorList(s))
        assert str(ei.value) == str(want)
    # out of range
    s = base.copy()
    s[12345] = n + 7
    with pytest.raises(g.InvalidListError, match="out-of-range at index 12345"):
        g.rs_rank(g.SuccessorList(s), 64)


def test_census_full_tile_violations(cuda):
    """Violations inside full 4096-node tiles: the census's branch-free path
    flags the tile and its exact re-scan reports the reference's first
    violation, for host int64 (narrowed to u32 ids) and device int32 input."""
    n = 100_000
    base = g.gen_list(n, seed=5).succ
    cases = []
    s = base.copy()
    s[50_000] = 50_000          # two self-loops in different full tiles
    s[7_000] = 7_000
    cases.append(s)
    s = base.copy()
    s[9_001] = n                # out of range right at n
    s[60_000] = 60_000
    cases.append(s)
    s = base.copy()
    s[4_096 * 3 + 5] = -2       # negative id
    cases.append(s)
    for s in cases:
        want = g.validate_list(g.SuccessorList(s))
        assert want is not None
        for arg in (s, torch.from_numpy(s.astype(np.int32)).cuda()):
            with pytest.raises(g.InvalidListError) as ei:
                g.rs_rank(g.SuccessorList(arg), 64)
            assert str(ei.value) == str(want)


def test_rs_reuse_succ_buffer(cuda, orc):
    sl = g.gen_list(1500, seed=17)
    rank, stats = g.rs_rank(sl, p=32, reuse_succ=True, accounting="counts")
    assert np.array_equal(rank, orc.seq_rank(sl.succ))
    assert stats.meta["splitter_set"].r == 32
    # device input: ranks overwrite the caller's successor tensor in place
    d = torch.from_numpy(g.gen_list(100_000, seed=2).succ).to(cuda)
    want = orc.seq_rank(d.cpu().numpy())
    out, _ = g.rs_rank(g.SuccessorList(d), p=128, reuse_succ=True)
    assert out.data_ptr() == d.data_ptr()
    assert np.array_equal(d.cpu().numpy(), want)


def test_rs_saturation_and_superlinear(cuda, orc):
    sl = g.gen_list(128, seed=23)
    rank, stats = g.rs_rank(sl, p=128, accounting="counts")
    assert np.array_equal(rank, orc.seq_rank(sl.succ))
    assert stats.meta["splitter_set"].sublist_len.max() == 1
    assert stats.meta.get("superlinear") is True
    _, stats = g.rs_rank(g.gen_list(10_000, seed=2), p=16, accounting="counts")
    assert stats.meta.get("superlinear") is None


def test_rs_deterministic(cuda):
    sl = g.gen_list(3000, seed=19)
    a, sa = g.rs_rank(sl, p=64, seed=3)
    b, sb = g.rs_rank(sl, p=64, seed=3)
    assert np.array_equal(a, b)
    assert np.array_equal(sa.meta["splitter_set"].sublist_len, sb.meta["splitter_set"].sublist_len)


def test_sublist_stats(cuda):
    sl = g.gen_list(4096, seed=37)
    _, stats = g.rs_rank(sl, p=64, seed=37, accounting="counts")
    st = g.sublist_stats(stats.meta["splitter_set"])
    assert st.mean_len == 4096 / 64 and st.max_len >= st.mean_len and st.histogram.sum() == 64
    _, stats = g.rs_rank_even(sl, p=64, accounting="counts")
    st = g.sublist_stats(stats.meta["splitter_set"])
    assert st.max_len == st.mean_len == 64


def test_acceptance_criterion_1_sample(cuda, orc):
    # test_acceptance.py:42-75 (5 variants, oracle equality), 10 seeds per size
    for n in (10, 1000, 100_000, 1_000_000):
        p = min(8192, n)
        p_sb = min(768, n)
        even_p = {10: 5, 1000: 100, 100_000: 4000, 1_000_000: 4000}[n]
        for seed in range(10 if n < 1_000_000 else 3):
            sl = g.gen_list(n, seed=seed)
            want = orc.seq_rank(sl.succ)
            outs = [
                g.wyllie_rank(sl, p, variant="multi_kernel", seed=seed)[0],
                g.wyllie_rank(sl, p_sb, variant="single_block", block_size=768, seed=seed)[0],
                g.rs_rank(sl, p, packing=g.Packing.P48, seed=seed)[0],
                g.rs_rank(sl, p, packing=g.Packing.P64, seed=seed)[0],
                g.rs_rank_even(sl, even_p, seed=seed)[0],
            ]
            for got in outs:
                assert g.compare_arrays(want, got) == -1, (n, seed)


def test_splitter_statistics_walk_consistent(cuda, orc):
    # test_acceptance.py:305-344 (exact part): lengths == positional gaps
    n, p = 100_000, 100
    sl = g.gen_list(n, seed=11)
    pos = orc.chain_positions(sl.succ)
    _, stats = g.rs_rank(sl, p, accounting="counts", seed=11)
    spl = stats.meta["splitter_set"]
    lens = spl.sublist_len
    assert lens.sum() == n and lens.size == p
    ps = pos[spl.splitter_node]
    order = np.argsort(ps)
    assert np.array_equal(lens[order], np.diff(np.append(ps[order], n)))


# ---------------------------------------------------------------- device-resident inputs

@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_device_resident_lists(cuda, orc, dtype):
    host = g.gen_list(300_000, seed=9)
    want = orc.seq_rank(host.succ)
    d = g.SuccessorList(torch.from_numpy(host.succ).to(cuda, dtype))
    for fn in (lambda s: g.rs_rank(s, 256), lambda s: g.wyllie_rank(s, 256)):
        out, _ = fn(d)
        assert out.is_cuda and out.dtype == dtype
        assert np.array_equal(out.cpu().numpy(), want)


def test_c_abi_u32_path(cuda, orc):
    """Call the C ABI directly with u32 successors / u32 ranks."""
    import ctypes

    n = 1 << 18
    host = g.gen_list(n, seed=4).succ
    succ = torch.from_numpy(host.astype(np.int32)).to(cuda)
    rank = torch.empty(n, dtype=torch.int32, device=cuda)
    L = _native.lib()
    ws = _device.workspace(L.sg_rs_workspace_bytes(n), cuda)
    st, v = _native.Stats(), _native.Violation()
    rc = L.sg_rs_rank(_device.ptr(succ), _native.SG_U32, _device.ptr(rank), _native.SG_U32, n, 0,
                      _device.ptr(ws), ws.numel(), _device.stream_ptr(cuda), ctypes.byref(st), ctypes.byref(v))
    assert rc == 0
    assert np.array_equal(rank.cpu().numpy().astype(np.int64), orc.seq_rank(host))
    assert st.levels >= 1 and st.level_size[0] == n and st.n_launches > 0
    assert st.total_ms == 0 and st.launch[0].ms == 0      # event times are read on demand
    assert L.sg_stats_resolve(ctypes.byref(st)) == 0
    assert st.total_ms > 0 and all(st.launch[k].ms >= 0 for k in range(st.n_launches))
    assert abs(sum(st.launch[k].ms for k in range(st.n_launches)) - st.total_ms) < 0.05 * st.total_ms + 0.05
    # a call's event set is recycled 64 calls later: resolving then reports it
    st2 = _native.Stats()
    rc = L.sg_rs_rank(_device.ptr(succ), _native.SG_U32, _device.ptr(rank), _native.SG_U32, n, 0,
                      _device.ptr(ws), ws.numel(), _device.stream_ptr(cuda), ctypes.byref(st2), ctypes.byref(v))
    early = g.rs_rank(g.SuccessorList(succ), 64)[1]      # ExecStats not read yet
    for _ in range(64):
        g.rs_rank(g.SuccessorList(succ), 64)
    assert L.sg_stats_resolve(ctypes.byref(st2)) == _native.SG_ERR_RUNTIME
    # the Python layer reports it instead of returning zeros
    assert early.wall_time is None
    assert all(np.isnan(r.ms) for r in early.launch_log)
    assert any("recycled" in w for w in early.warnings)
    assert st2.total_ms == 0


# ---------------------------------------------------------------- scale

def test_rank_against_reference_digests(cuda, hashes):
    for n, s in [(1 << 20, 0), (1 << 20, 1), (1 << 22, 0)]:
        sl = g.gen_list(n, seed=s, device=cuda)
        assert sha(sl.succ) == hashes[f"gen_list_{n}_{s}"]
        for fn in (lambda x: g.rs_rank(x, 4096), lambda x: g.wyllie_rank(x, 4096)):
            rank, _ = fn(sl)
            assert sha(rank) == hashes[f"seq_rank_{n}_{s}"], (n, s)


def _check_rank_properties(succ, rank):
    """Size-independent: rank is a permutation of 0..n-1 that decreases by one
    along every link (rank[succ[i]] == rank[i] - 1 off the tail)."""
    n = succ.numel()
    succ = succ.to(torch.int64)
    rank = rank.to(torch.int64)
    idx = torch.arange(n, device=succ.device)
    tail = succ == idx
    assert int(tail.sum()) == 1
    assert int(rank[0]) == n - 1
    assert torch.all(rank[tail] == 0)
    assert torch.all(rank[succ[~tail]] == rank[~tail] - 1)
    assert int(torch.bincount(rank, minlength=n).max()) == 1


@pytest.mark.parametrize("kind", ["random", "ordered"])
def test_full_size_properties_2_28(cuda, kind):
    """BASELINE configs[2]: 2^28 nodes, random and ordered layouts."""
    n = 1 << 28
    sl = g.gen_list(n, seed=0, device=cuda, dtype=torch.int32) if kind == "random" else \
        g.ordered_list(n, device=cuda, dtype=torch.int32)
    rank, stats = g.rs_rank(sl, 16384)
    assert stats.meta["path"] == ("ruling_set" if kind == "random" else "contract")
    _check_rank_properties(sl.succ, rank)
    assert stats.meta["fallback"] is False


@pytest.mark.parametrize("kind", ["random", "ordered"])
def test_full_size_properties_2_26(cuda, kind):
    n = 1 << 26
    sl = g.gen_list(n, seed=0, device=cuda, dtype=torch.int32) if kind == "random" else \
        g.ordered_list(n, device=cuda, dtype=torch.int32)
    rank, stats = g.rs_rank(sl, 16384)
    _check_rank_properties(sl.succ, rank)
    assert stats.meta["fallback"] is False
    w, _ = g.wyllie_rank(sl, 1024)
    assert torch.equal(w, rank)


def _list_from_order(order):
    succ = np.empty(order.size, dtype=np.int64)
    succ[order[:-1]] = order[1:]
    succ[order[-1]] = order[-1]
    return succ


def test_contraction_run_tiles(cuda, orc):
    """Ordered tiles the census flags as runs (the contraction skips them)
    next to locally shuffled and partial tiles, and defects next to runs."""
    T = 4096
    n = 10 * T + 123
    rng = np.random.default_rng(11)
    order = np.arange(n)
    order[3 * T:4 * T] = 3 * T + rng.permutation(T)       # tile 3 shuffled inside
    order[6 * T + 7:6 * T + 40] = order[6 * T + 7:6 * T + 40][::-1]  # a reversed stretch in tile 6
    succ = _list_from_order(order)
    want = orc.seq_rank(succ)
    for arg in (succ, torch.from_numpy(succ.astype(np.int32)).cuda()):
        rank, stats = g.rs_rank(g.SuccessorList(arg), 64)
        assert stats.meta["path"] == "contract"
        rank = rank.cpu().numpy() if isinstance(rank, torch.Tensor) else rank
        assert np.array_equal(rank, want)
    # defects beside run tiles: a back edge (in-degree 2 + cycle), a jump
    # skipping a node, a tile whose successor leaves to a non-head
    ordered = np.arange(1, n + 1, dtype=np.int64)
    ordered[-1] = n - 1
    bad = []
    s = ordered.copy(); s[5 * T + 10] = 5 * T; bad.append(s)
    s = ordered.copy(); s[7 * T - 1] = 7 * T + 1; bad.append(s)
    s = ordered.copy(); s[2 * T + 5] = 8 * T + 3; bad.append(s)
    for s in bad:
        want = g.validate_list(g.SuccessorList(s))
        assert want is not None
        for arg in (s, torch.from_numpy(s.astype(np.int32)).cuda()):
            with pytest.raises(g.InvalidListError) as ei:
                g.rs_rank(g.SuccessorList(arg), 64)
            assert str(ei.value) == str(want)


def test_walk_cap_fallback(cuda, orc, sg_env):
    """A walk that exceeds the hop cap falls back to pointer jumping."""
    sg_env(SG_RS_WALK_CAP="4")
    sl = g.gen_list(50_000, seed=8)
    rank, stats = g.rs_rank(sl, 32)
    assert stats.meta["fallback"] is True
    assert np.array_equal(rank, orc.seq_rank(sl.succ))


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("n", [5_000, 300_001, 3_000_017])
def test_record_paths_match_oracle(cuda, orc, sg_env, fused, n):
    """Both level-0 record pipelines: the walk that bins its records by output
    window itself (k_rs_walk_bin, default) and the chunked walk followed by
    rs5_partition (SG_RS_FUSED=0)."""
    sg_env(SG_RS_FUSED=fused)
    sl = g.gen_list(n, seed=n % 97)
    rank, _ = g.rs_rank(sl, 256, seed=3)
    assert np.array_equal(rank, orc.seq_rank(sl.succ))


@pytest.mark.parametrize("fused", ["1", "0"])
def test_record_paths_invalid_lists(cuda, sg_env, fused):
    """Invalid lists overfill some output windows of the binned walk: the
    records are dropped and the reference violation is still reported."""
    sg_env(SG_RS_FUSED=fused)
    n = 1_000_003
    base = g.gen_list(n, seed=5).succ
    order = np.argsort(-np.asarray(g.rs_rank(g.SuccessorList(base), 1)[0]))
    s = base.copy()
    a = int(order[n // 2])
    s[a] = s[int(s[a])]                     # in-degree 2
    s2 = base.copy()
    s2[int(order[n // 3])] = int(order[n // 5])   # cycle back into the list
    for bad in (s, s2):
        want = g.validate_list(g.SuccessorList(bad))
        assert want.kind != "ok"
        with pytest.raises(g.InvalidListError) as ei:
            g.rs_rank(g.SuccessorList(bad), 64)
        assert str(ei.value) == str(want)


@pytest.mark.parametrize("topn,coop", [("0", "1"), ("20000", "1"), ("20000", "0"), ("524288", "1")])
def test_top_level_ranking_paths(cuda, orc, sg_env, topn, coop):
    """The ruler list above level 0 is finished either by more walked levels
    and the one-CTA final (SG_RS_TOPN=0), or by multi-CTA in-place pointer
    jumping once it has at most SG_RS_TOPN rulers (default 2^20): one
    cooperative launch with grid barriers (default) or one launch per round
    (SG_RS_COOP=0)."""
    sg_env(SG_RS_TOPN=topn)
    sg_env(SG_RS_COOP=coop)
    if topn == "0":
        sg_env(SG_RS_KBITS="3")  # chains of 8 above level 0: two walked levels end at <= 8192 rulers
    sl = g.gen_list(2_500_003, seed=11)
    rank, st = g.rs_rank(sl, 128, seed=1)
    assert np.array_equal(rank, orc.seq_rank(sl.succ))
    top = [r for r in st.launch_log if r.kernel == "rs4_rank"]
    if topn == "0":
        assert sum(r.kernel == "rs4_walk" for r in st.launch_log) >= 2
        assert len(top) == 1 and top[0].blocks == 1
    elif coop == "1":
        assert len(top) == 1 and top[0].blocks > 1      # init + rounds + extraction in one grid
    else:
        assert len(top) > 10                            # init + ceil(log2 R) + 1 jump rounds
    # an invalid list through the same path still reports the reference violation
    s = sl.succ.copy()
    s[int(np.flatnonzero(s == np.arange(s.size))[0])] = 0   # tail -> head: one big cycle
    with pytest.raises(g.InvalidListError):
        g.rs_rank(g.SuccessorList(s), 64)


@pytest.mark.parametrize("n", [8_193, 65_537, 1_048_575, 2_097_153, (1 << 23) + 1])
def test_plan_boundaries(cuda, orc, n):
    """Sizes around the plan's switch points: the one-CTA final (8192), the
    pointer-jumping top (2^20 rulers), and the coarse-window count (256
    windows of 2^15 int32 ranks at 2^23: one more node doubles the window)."""
    sl = g.gen_list(n, seed=n % 1009)
    want = orc.seq_rank(sl.succ)
    rank, _ = g.rs_rank(sl, 64, seed=2)                                   # int64 ranks (host input)
    assert np.array_equal(rank, want)
    d = torch.from_numpy(sl.succ.astype(np.int32)).to(cuda)
    out, _ = g.rs_rank(g.SuccessorList(d), 64, seed=2)                     # int32 ranks (device input)
    assert np.array_equal(out.cpu().numpy().astype(np.int64), want)


@pytest.mark.parametrize("refine", ["0", "1", "2", "3", "4", "5", "6", "7"])
def test_refine_variants(cuda, orc, sg_env, refine):
    """rs5_refine variants (SG_RS_REFINE: 0 shared-atomic ranking, the
    default; 1 the block multisplit refine; 2 lean + match.any; 3 lean,
    alternating; 4 lean in the tile layout; 5 lean + shared atomics; 6 lean +
    ballots; 7 ranks stored straight from the records, no rs5_scatter) on
    windows shrunk to 8 KiB (SG_RS_WIN_KB=8) so 2^20 nodes already split
    every coarse window into 8 fine bins and 2^25 nodes into 64 (the C3
    fan-out): exact against the oracle, and the size-independent rank
    properties at 2^25."""
    sg_env(SG_RS_REFINE=refine, SG_RS_WIN_KB=8)
    sl = g.gen_list((1 << 20) + 7, seed=13)
    rank, st = g.rs_rank(sl, 256, seed=2)
    assert st.meta["path"] == "ruling_set"
    assert np.array_equal(rank, orc.seq_rank(sl.succ))
    big = g.gen_list((1 << 25) + 3, seed=0, device=cuda, dtype=torch.int32)
    rank, st = g.rs_rank(big, 16384)
    assert st.meta["fallback"] is False
    _check_rank_properties(big.succ, rank)



def test_splitter_meta_blocks_are_not_shared(cuda, orc):
    """meta["splitter_set"] arrays live in pinned blocks lent per call
    (listrank._PinnedPool): results kept from earlier calls stay intact while
    later calls run, and a block returns to the pool once its arrays are gone."""
    import gc

    from paper_1002_4482_b200 import listrank

    sls = [g.gen_list((1 << 18) + k, seed=30 + k) for k in range(3)]
    kept = []
    for sl in sls:
        _, st = g.rs_rank(sl, 512, seed=4)
        kept.append(st.meta["splitter_set"])
    for _ in range(3):  # more calls of the same shape reuse whatever blocks are free
        g.rs_rank(sls[0], 512, seed=4)
    for sl, ss in zip(sls, kept):
        assert np.array_equal(orc.seq_rank(sl.succ)[ss.splitter_node], ss.splitter_rank)
        assert not ss.splitter_node.flags.writeable  # the cached draw is shared read-only
    del kept, ss, st
    gc.collect()
    assert sum(len(v) for v in listrank._META_POOL.free.values()) >= 1


@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_rs_rank_even_splitters_device(cuda, orc, dtype):
    """rs_rank_even's perfect splitters (listrank.py:431-436) come from one
    device pass over the ranks (sg_even_splitters): the node at chain
    position k * n/p, for p = 1, a middle p and p = n."""
    n = 3 * (1 << 16)
    sl = g.gen_list(n, seed=8)
    want_rank = orc.seq_rank(sl.succ)
    node_at = np.empty(n, dtype=np.int64)
    node_at[(n - 1) - want_rank] = np.arange(n)
    d = g.SuccessorList(torch.from_numpy(sl.succ).to(cuda).to(dtype))
    for p in (1, 3 * 256, n):
        rank, st = g.rs_rank_even(d, p)
        ss = st.meta["splitter_set"]
        assert np.array_equal(ss.splitter_node, node_at[:: n // p]), p
        assert np.array_equal(ss.splitter_rank, want_rank[ss.splitter_node])
