"""Pin the CPU oracle (oracle/orc.c, oracle/orc.py) to the reference: golden
vectors produced by the reference itself (tests/golden/make_golden.py) and
the reference's own known-answer tests (test_core.py, test_gen.py)."""

import json

import numpy as np
import pytest


def test_kiss_golden_vectors(orc, golden):
    # test_gen.py:12-23 / :26-37: scalar recurrence from (1,2,3,4) and the default state
    out, _ = orc.kiss_batch((1, 2, 3, 4), 8)
    assert out.tolist() == golden["kiss_1234_first8"].tolist()
    out, _ = orc.kiss_batch((1234567890987654321, 362436362436362436, 1066149217761810, 123456123456123456), 5)
    assert out.tolist() == [8932985056925012148, 5710300428094272059, 18342510866933518593,
                            14303636270573868250, 542381058189297533]


def test_kiss_seed_and_batches(orc, golden):
    for s, st in zip(golden["kiss_seed_seeds"].tolist(), golden["kiss_seed_states"].tolist()):
        assert list(orc.kiss_seed(s)) == st
        d, st2 = orc.kiss_batch(orc.kiss_seed(s), 4096)
        assert np.array_equal(d, golden[f"kiss_batch_{s}"])
        assert list(st2) == golden[f"kiss_batch_state_{s}"].tolist()


def test_seq_rank_known_answers(orc):
    # test_core.py:46-59
    assert orc.seq_rank([0]).tolist() == [0]
    assert orc.seq_rank([1, 2, 2]).tolist() == [2, 1, 0]
    assert orc.seq_rank([3, 4, 2, 1, 2]).tolist() == [4, 2, 0, 3, 1]
    assert orc.chain_positions([3, 4, 2, 1, 2]).tolist() == [0, 2, 4, 1, 3]


def test_gen_list_and_seq_rank_match_reference(orc, golden):
    for n, s in golden["list_cases"].tolist():
        succ = orc.gen_list(n, s)
        assert np.array_equal(succ, golden[f"list_{n}_{s}"]), (n, s)
        assert np.array_equal(orc.seq_rank(succ), golden[f"rank_{n}_{s}"]), (n, s)


def test_validate_list_matches_reference(orc, golden):
    bad = json.loads(str(golden["bad_lists"]))
    verdicts = json.loads(str(golden["bad_verdicts"]))
    for b, v in zip(bad, verdicts):
        kind, idx = orc.validate_list(b)
        if v is None:
            assert kind is None
        else:
            assert [kind, idx] == v, (b, v)


def test_draw_splitters_match_reference(orc, golden):
    for n, r, s in golden["spl_cases"].tolist():
        assert np.array_equal(orc.draw_splitters(n, r, s), golden[f"spl_{n}_{r}_{s}"]), (n, r, s)


def test_splitter_set_matches_reference(orc, golden):
    for n, p, ls, s in golden["rs_cases"].tolist():
        succ = orc.gen_list(n, ls) if n > 3 else np.array([1, 2, 2])
        key = f"rs_{n}_{p}_{ls}_{s}"
        nodes = orc.draw_splitters(n, p, s)
        assert np.array_equal(nodes, golden[key + "_node"])
        ln, red, sr = orc.splitter_set(succ, nodes)
        assert np.array_equal(ln, golden[key + "_len"])
        assert np.array_equal(red, golden[key + "_succ"])
        assert np.array_equal(sr, golden[key + "_rank"])


def test_random_graphs_and_labels_match_reference(orc, golden):
    for i, (n, d, s) in enumerate(golden["rg_cases"].tolist()):
        e = orc.gen_random_graph(int(n), d, int(s))
        assert np.array_equal(e, golden[f"rg_{i}_edges"]), (n, d, s)
        assert np.array_equal(orc.seq_components(int(n), e), golden[f"rg_{i}_labels"])


def test_tree_and_path_labels_match_reference(orc, golden):
    for i, (n, k, s) in enumerate(golden["tr_cases"].tolist()):
        assert np.array_equal(orc.seq_components(n, golden[f"tr_{i}_edges"]), golden[f"tr_{i}_labels"])
    assert np.array_equal(orc.seq_components(3000, golden["path_3000_2_edges"]), golden["path_3000_2_labels"])


def test_seq_components_known_answers(orc):
    # test_core.py:102-108
    assert orc.seq_components(6, [(0, 1), (1, 2), (4, 5)]).tolist() == [0, 0, 0, 3, 4, 4]
    assert orc.seq_components(4, np.empty((0, 2))).tolist() == [0, 1, 2, 3]


def test_seq_components_matches_scipy(orc):
    # test_core.py:112-126
    sp = pytest.importorskip("scipy.sparse")
    from scipy.sparse.csgraph import connected_components

    rng = np.random.default_rng(99)
    for _ in range(20):
        n = int(rng.integers(2, 120))
        m = int(rng.integers(0, 3 * n))
        e = rng.integers(0, n, size=(m, 2))
        e = e[e[:, 0] != e[:, 1]]
        mat = sp.coo_matrix((np.ones(len(e)), (e[:, 0], e[:, 1])), shape=(n, n))
        _, lab = connected_components(mat, directed=False)
        small = np.full(n, n, dtype=np.int64)
        np.minimum.at(small, lab, np.arange(n))
        assert np.array_equal(small[lab], orc.seq_components(n, e))


def test_validate_graph(orc):
    # core.py:196-206 order: range over all endpoints, then self-loops
    assert orc.validate_graph(3, [(0, 1)]) == (None, -1)
    assert orc.validate_graph(3, [(0, 1), (2, 2), (0, 5)]) == ("out-of-range", 2)
    assert orc.validate_graph(3, [(0, 1), (2, 2)]) == ("self-loop", 1)


def test_c_generators_match_numpy_restatement(orc):
    # the C generators (orc.c) against the numpy restatements of gen.py, on
    # sizes / densities that force several rejection batches
    for n, s in [(1, 0), (2, 5), (3, 1), (1000, 3), (65537, 9)]:
        assert np.array_equal(orc.gen_list(n, s), orc.gen_list_np(n, s)), (n, s)
    for n, d, s in [(2, 1.0, 0), (5, 1.0, 3), (40, 0.9, 1), (300, 0.3, 2), (5000, 0.001, 4)]:
        assert np.array_equal(orc.gen_random_graph(n, d, s), orc.gen_random_graph_np(n, d, s)), (n, d, s)


def test_generator_digests_match_reference(orc, hashes):
    import hashlib

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()

    assert sha(orc.gen_list(1 << 20, 0)) == hashes["gen_list_1048576_0"]
    e = orc.gen_random_graph(1 << 16, (1 << 18) / ((1 << 16) * ((1 << 16) - 1) // 2), 0)
    assert sha(e) == hashes["gen_random_graph_65536_262144_0"]
    assert sha(orc.seq_components(1 << 16, e)) == hashes["seq_components_65536_262144_0"]


def test_seq_rank_sampler(orc):
    succ = orc.gen_list(1 << 12, 0)
    smp = orc.SeqRankSampler(succ)
    assert smp(100) == 100
    assert smp(100) == 100          # a fresh epoch: nothing looks visited
    assert smp(1 << 20) == (1 << 12) - 1   # the whole chain: n - 1 hops to the tail
    assert np.array_equal(smp.rank, orc.seq_rank(succ))
