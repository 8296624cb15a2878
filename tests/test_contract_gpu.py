"""Tile contraction (local layouts) of rs_rank: ordered and locally shuffled
lists are ranked by contracting in-tile segments (csrc/sg_list.cu,
k_rs_contract).  Ranks must equal seq_rank (core.py:179-186) bit-exactly,
and invalid local lists must raise the reference's InvalidListError
(core.py:148-167) exactly like the ruling-set path."""

import numpy as np
import pytest
import torch

import paper_1002_4482_b200 as g

pytestmark = pytest.mark.gpu

TILE = 4096


def list_from_order(order):
    """succ for the list visiting `order` (order[0] must be 0)."""
    order = np.asarray(order, dtype=np.int64)
    succ = np.empty(order.size, dtype=np.int64)
    succ[order[:-1]] = order[1:]
    succ[order[-1]] = order[-1]
    return succ


def ordered(n):
    return list_from_order(np.arange(n))


def block_shuffled(n, block, seed):
    """Chain order: blocks of `block` ids in increasing order, each block's
    ids in random order (node 0 stays first)."""
    rng = np.random.default_rng(seed)
    order = np.arange(n)
    for b0 in range(0, n, block):
        seg = order[b0:b0 + block]
        rng.shuffle(seg)
    z = int(np.flatnonzero(order == 0)[0])
    order[[0, z]] = order[[z, 0]]
    return list_from_order(order)


def tiles_permuted(n, seed):
    """Whole tiles visited in random order, each tile in index order."""
    rng = np.random.default_rng(seed)
    nt = (n + TILE - 1) // TILE
    perm = np.concatenate([[0], 1 + rng.permutation(nt - 1)])
    order = np.concatenate([np.arange(t * TILE, min(n, (t + 1) * TILE)) for t in perm])
    return list_from_order(order)


def reversed_list(n):
    """0 -> n-1 -> n-2 -> ... -> 1 (tail 1)."""
    return list_from_order(np.concatenate([[0], np.arange(n - 1, 0, -1)]))


CASES = {
    "ordered": lambda n: ordered(n),
    "reversed": lambda n: reversed_list(n),
    "block7": lambda n: block_shuffled(n, 7, 1),
    "block300": lambda n: block_shuffled(n, 300, 2),
    "tiles": lambda n: tiles_permuted(n, 3),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("n", [8193, 10_000, 65_537, 300_001, 1 << 20])
def test_contraction_matches_oracle(cuda, orc, case, n):
    succ = CASES[case](n)
    want = orc.seq_rank(succ)
    rank, stats = g.rs_rank(g.SuccessorList(succ), 64)
    assert np.array_equal(rank, want), (case, n)
    assert stats.meta["path"] == "contract", stats.meta
    # device-resident int32 in, int32 out; and the reuse_succ alias
    d = torch.from_numpy(succ.astype(np.int32)).to(cuda)
    out, _ = g.rs_rank(g.SuccessorList(d), 64)
    assert np.array_equal(out.cpu().numpy().astype(np.int64), want)
    out, _ = g.rs_rank(g.SuccessorList(d), 64, reuse_succ=True)
    assert out.data_ptr() == d.data_ptr()
    assert np.array_equal(d.cpu().numpy().astype(np.int64), want)


def test_contraction_meta_matches_ruling_set(cuda, orc, sg_env):
    """The splitter meta is path-independent (derived from the ranks)."""
    succ = block_shuffled(200_000, 50, 4)
    a, sa = g.rs_rank(g.SuccessorList(succ), 256, seed=5)
    sg_env(SG_RS_CONTRACT="0")
    b, sb = g.rs_rank(g.SuccessorList(succ), 256, seed=5)
    assert sa.meta["path"] == "contract" and sb.meta["path"] == "ruling_set"
    assert np.array_equal(a, b)
    for f in ("splitter_node", "sublist_len", "splitter_succ", "splitter_rank"):
        assert np.array_equal(getattr(sa.meta["splitter_set"], f), getattr(sb.meta["splitter_set"], f))


def test_scattered_lists_keep_the_ruling_set(cuda):
    _, st = g.rs_rank(g.gen_list(100_000, seed=1), 64)
    assert st.meta["path"] == "ruling_set"


def _expect_invalid(succ):
    want = g.validate_list(g.SuccessorList(succ))
    assert want.kind != "ok"
    for fn in (lambda x: g.rs_rank(x, 64), lambda x: g.wyllie_rank(x, 64)):
        with pytest.raises(g.InvalidListError) as ei:
            fn(g.SuccessorList(succ))
        assert str(ei.value) == str(want)


def test_contraction_invalid_lists(cuda):
    n = 100_000
    # two in-tile predecessors: 9 -> 11 skips 10 (10 -> 11 as well)
    s = ordered(n)
    s[9] = 11
    _expect_invalid(s)
    # cross-tile shared successor: the last node of tile 1 jumps into tile 3
    s = ordered(n)
    s[2 * TILE - 1] = 3 * TILE + 5
    _expect_invalid(s)
    # in-tile cycle without a local ruler: 1 -> 2 -> 3 -> 1, 0 -> 4
    s = ordered(n)
    s[0], s[3] = 4, 1
    _expect_invalid(s)
    # a tile that is one run except that its last id links back into it
    # (not a single-run tile: the fast path must not take it)
    s = ordered(n)
    s[2 * TILE - 1] = TILE + 5
    _expect_invalid(s)
    # in-tile cycle through rulers, reached from the head: ... 40 -> 17
    s = ordered(n)
    s[40] = 17
    _expect_invalid(s)
    # node 0 has an in-tile predecessor: 5 -> 0 -> 1 ... 4 -> 6 (5 unreachable from 0)
    s = ordered(n)
    s[5], s[4] = 0, 6
    _expect_invalid(s)
    # cycle spanning tiles, no tail reachable; a second self-loop; out of range
    s = ordered(n)
    s[n - 1] = 3 * TILE
    s[3 * TILE - 1] = 3 * TILE - 1
    _expect_invalid(s)
    s = ordered(n)
    s[50_000] = 50_000
    _expect_invalid(s)
    s = ordered(n)
    s[77_777] = n + 3
    _expect_invalid(s)


def test_contraction_full_size_2_26_properties(cuda):
    n = 1 << 26
    sl = g.ordered_list(n, device=cuda, dtype=torch.int32)
    rank, st = g.rs_rank(sl, 16384)
    assert st.meta["path"] == "contract"
    want = torch.arange(n - 1, -1, -1, device=cuda, dtype=torch.int32)
    assert torch.equal(rank, want)
