"""Host-side logic of the package (no GPU): generators bit-exact with the
reference, KISS jump-ahead, argument checks that precede device work,
packing, ExecStats, fixtures, the splitter-set derivation."""

import numpy as np
import pytest
import torch

import paper_1002_4482_b200 as g
from paper_1002_4482_b200 import gen, listrank
from paper_1002_4482_b200.listrank import _draw_splitters, _splitter_set


# ---- generators ---------------------------------------------------------------

def test_kiss_next_golden(golden):
    st = gen.KissState(1, 2, 3, 4)
    out = []
    for _ in range(8):
        v, st = g.kiss_next(st)
        out.append(v)
    assert out == golden["kiss_1234_first8"].tolist()


def test_kiss_seed_and_batch(golden):
    for s, st in zip(golden["kiss_seed_seeds"].tolist(), golden["kiss_seed_states"].tolist()):
        assert list(g.kiss_seed(s)) == st
        d, st2 = g.kiss_batch(g.kiss_seed(s), 4096)
        assert np.array_equal(d, golden[f"kiss_batch_{s}"])
        assert list(st2) == golden[f"kiss_batch_state_{s}"].tolist()


def test_kiss_batch_carries_state():
    # test_gen.py:56-66: batches agree with the scalar recurrence across splits
    st = g.kiss_seed(42)
    a, st_a = g.kiss_batch(st, 300)
    b1, s1 = g.kiss_batch(st, 120)
    b2, s2 = g.kiss_batch(s1, 180)
    assert np.array_equal(a, np.concatenate([b1, b2])) and s2 == st_a
    s = st
    for i in range(50):
        v, s = g.kiss_next(s)
        assert v == int(a[i])


@pytest.mark.parametrize("k", [0, 1, 2, 63, 64, 1000, 123457])
def test_kiss_jump_ahead(k):
    st = g.kiss_seed(7)
    seq, after = g.kiss_batch(st, k + 5)
    j = gen.kiss_jump(st, k)
    nxt, _ = g.kiss_batch(j, 5)
    assert np.array_equal(nxt, seq[k:k + 5])


def test_kiss_chunk_states():
    st = g.kiss_seed(3)
    seq, _ = g.kiss_batch(st, 10 * 777)
    cs = gen.kiss_chunk_states(st, 10, 777)
    for k in range(10):
        d, _ = g.kiss_batch(gen.KissState(*[int(v) for v in cs[k]]), 777)
        assert np.array_equal(d, seq[k * 777:(k + 1) * 777])


def test_gen_list_matches_reference(golden):
    for n, s in golden["list_cases"].tolist():
        assert np.array_equal(g.gen_list(n, seed=s).succ, golden[f"list_{n}_{s}"]), (n, s)


def test_gen_random_graph_matches_reference(golden):
    for i, (n, d, s) in enumerate(golden["rg_cases"].tolist()):
        e = g.gen_random_graph(int(n), d, seed=int(s)).edges
        assert np.array_equal(e, golden[f"rg_{i}_edges"]), (n, d, s)
    gr = g.gen_random_graph(1000, 0.01, seed=0)
    assert gr.m == 4995                      # test_gen.py:163-165
    with pytest.raises(ValueError):
        g.gen_random_graph(10, 0.0)
    with pytest.raises(ValueError):
        g.gen_random_graph(10, 1.5)


def test_gen_tree_graph_matches_reference(golden):
    for i, (n, k, s) in enumerate(golden["tr_cases"].tolist()):
        assert np.array_equal(g.gen_tree_graph(n, k, seed=s).edges, golden[f"tr_{i}_edges"]), (n, k, s)


def test_draw_splitters_match_reference(golden):
    for n, r, s in golden["spl_cases"].tolist():
        assert np.array_equal(_draw_splitters(n, r, s), golden[f"spl_{n}_{r}_{s}"]), (n, r, s)


# ---- splitter set from ranks (host tensors stand in for device ones) ----------

@pytest.mark.gpu
def test_splitter_set_from_ranks(golden, orc, cuda):
    """meta["splitter_set"] derivation (sg_splitter_meta) from oracle ranks
    vs the reference's own RS3/RS4 outputs."""
    for n, p, ls, s in golden["rs_cases"].tolist():
        key = f"rs_{n}_{p}_{ls}_{s}"
        rank = torch.from_numpy(orc.seq_rank(orc.gen_list(n, ls))) if n > 3 else torch.tensor([2, 1, 0])
        rank = rank.to(cuda)
        spl = _splitter_set(rank, _draw_splitters(n, p, s), n)
        assert spl.r == p
        assert np.array_equal(spl.splitter_node, golden[key + "_node"])
        assert np.array_equal(spl.sublist_len, golden[key + "_len"])
        assert np.array_equal(spl.splitter_succ, golden[key + "_succ"])
        assert np.array_equal(spl.splitter_rank, golden[key + "_rank"])
        assert int(spl.sublist_len.max()) == int(golden[key + "_max"])


# ---- argument checks that precede device work -----------------------------------

def test_rs_rank_even_divisibility_checked_first():
    with pytest.raises(ValueError):
        g.rs_rank_even(g.gen_list(100, seed=1), p=7)     # test_listrank.py:221-223


def test_graph_without_vertices():
    with pytest.raises(g.InvalidGraphError):
        g.sv_components(g.EdgeGraph(0, []), 1)


def test_unknown_cc_variant():
    with pytest.raises(ValueError):
        g.sv_components(g.EdgeGraph(2, [[0, 1]]), 1, variant="nope")


def test_machine_checks_order():
    e = listrank._machine_error
    assert "backend" in str(e(1, 256, "gpu", "full"))
    assert "accounting" in str(e(1, 256, "simulated", "x"))
    assert "thread" in str(e(0, 256, "simulated", "full"))
    assert "block size" in str(e(4, 769, "simulated", "full"))
    assert e(4, 768, "threaded", "counts") is None
    err = listrank._rs_param_error(40000, 16385, g.Packing.P48, 256, "bogus", "full")
    assert isinstance(err, g.CapabilityError)       # capability before Machine checks
    assert isinstance(listrank._rs_param_error(3, 4, g.Packing.P64, 256, "simulated", "full"), ValueError)


def test_round_bound(golden):
    for n, b in zip(golden["round_bound_n"].tolist(), golden["round_bound"].tolist()):
        assert g.sv_round_bound(n) == b
    assert g.sv_round_bound(1000) == 19 and g.sv_round_bound(10 ** 5) == 30


# ---- core types -------------------------------------------------------------------

def test_pack_unpack():
    for p in (g.Packing.P48, g.Packing.P64):
        for mark, rank in [(0, 0), (1, 2**32 - 1), (2**16 - 1, 12345)]:
            assert g.unpack(g.pack(mark, rank, p), p) == (mark, rank)
    assert g.pack(1, 0, g.Packing.P64) == 4294967296
    assert g.pack(3, 5, g.Packing.P48) == 12884901893
    with pytest.raises(g.PackingError):
        g.pack(2**16, 0, g.Packing.P48)
    with pytest.raises(g.PackingError):
        g.unpack(1 << 48, g.Packing.P48)
    assert issubclass(g.CapabilityError, ValueError)


def test_validate_list_host(golden):
    assert g.validate_list(g.SuccessorList([1, 2, 2])) is None
    v = g.validate_list(g.SuccessorList([1, 5, 2]))
    assert v.kind == "out-of-range" and v.index == 1
    assert g.validate_list(g.SuccessorList([1, 2, 0])).kind == "no-tail"
    assert g.validate_list(g.SuccessorList([0, 2, 2])).kind == "multiple-self-loops"
    v = g.validate_list(g.SuccessorList([1, 0, 2]))
    assert v.kind == "unreachable" and v.index == 2


def test_containers_accept_tensors():
    sl = g.SuccessorList(torch.tensor([1, 2, 2], dtype=torch.int32))
    assert sl.n == 3 and not sl.on_device
    assert sl.host_succ().dtype == np.int64
    gr = g.EdgeGraph(3, torch.tensor([[0, 1]], dtype=torch.int64))
    assert gr.m == 1 and gr.host_edges().tolist() == [[0, 1]]
    assert g.EdgeGraph(4, []).m == 0


def test_exec_stats_aggregates():
    st = g.ExecStats()
    st.launch_log.append(g.LaunchRecord("a", g.KernelCounters(launches=1, items=5, ms=1.0)))
    st.launch_log.append(g.LaunchRecord("a", g.KernelCounters(launches=1, items=7, ms=2.0)))
    st.launch_log.append(g.LaunchRecord("b", g.KernelCounters(launches=1, items=1)))
    per = st.per_kernel()
    assert per["a"].launches == 2 and per["a"].items == 12 and per["a"].ms == 3.0
    assert st.kernel_launches == 3 and st.totals().items == 13
    rows = st.csv_rows(7)
    assert rows[-1]["kernel"] == "total" and rows[-1]["launches"] == 3


def test_fixtures_roundtrip(tmp_path):
    sl = g.gen_list(50, seed=3)
    g.save_list(sl, tmp_path / "l.txt")
    assert np.array_equal(g.load_list(tmp_path / "l.txt").succ, sl.succ)
    gr = g.EdgeGraph(6, [(0, 1), (1, 2), (4, 5)])
    g.save_graph(gr, tmp_path / "g.txt")
    back = g.load_graph(tmp_path / "g.txt")
    assert back.n == 6 and back.m == 3 and np.array_equal(back.edges, gr.edges)
    g.save_graph(g.EdgeGraph(3, []), tmp_path / "e.txt")
    assert g.load_graph(tmp_path / "e.txt").m == 0


def test_canonical_and_compare():
    assert g.canonical_labels([4, 4, 2, 2, 3]).tolist() == [0, 0, 2, 2, 4]
    assert g.compare_arrays([1, 2, 3], [1, 2, 3]) == -1
    assert g.compare_arrays([1, 2, 3], [1, 0, 3]) == 1
    assert g.compare_arrays([1, 2], [1, 2, 3]) == 0


def test_list_to_graph():
    gr = g.list_to_graph(g.SuccessorList([1, 2, 2]))
    assert gr.n == 3 and gr.edges.tolist() == [[0, 1], [1, 2]]


def test_exec_stats_has_no_reference_cycle():
    """A dropped ExecStats (and the meta arrays it holds) is freed by
    reference counting alone -- the bench times with the cyclic GC paused,
    and the splitter-meta pinned blocks return to their pool only when their
    arrays die (listrank._PinnedPool)."""
    import gc
    import weakref

    from paper_1002_4482_b200 import _device, _native

    st = _native.Stats()
    st.n_launches = 2
    es = _device.exec_stats(st)
    es.meta["x"] = object()
    ref = weakref.ref(es)
    was = gc.isenabled()
    gc.disable()
    try:
        del es
        assert ref() is None
    finally:
        if was:
            gc.enable()
