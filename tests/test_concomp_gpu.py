"""Connected components on the B200 vs the oracle / reference goldens.
Re-targets pkg/tests/test_concomp.py and test_acceptance.py criteria 2-3."""

import ctypes
import hashlib

import numpy as np
import pytest
import torch

import paper_1002_4482_b200 as g
from paper_1002_4482_b200 import _device, _native

pytestmark = pytest.mark.gpu

VARIANTS = ("uf", "sv")


def sha(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


@pytest.mark.parametrize("variant", VARIANTS)
def test_small_hand_graphs(cuda, variant):
    labels, stats = g.sv_components(g.EdgeGraph(2, [[0, 1]]), p=2, variant=variant)
    assert labels.tolist() == [0, 0] and stats.rounds <= 3
    labels, _ = g.sv_components(g.EdgeGraph(6, [[0, 1], [1, 2], [0, 2], [3, 4], [4, 5]]), p=4, variant=variant)
    assert labels.tolist() == [0, 0, 0, 3, 3, 3]
    labels, stats = g.sv_components(g.EdgeGraph(7, []), p=4, variant=variant)
    assert labels.tolist() == list(range(7)) and stats.rounds == 1
    labels, stats = g.sv_components(g.EdgeGraph(1, []), p=1, variant=variant)
    assert labels.tolist() == [0] and stats.rounds == 1
    labels, _ = g.sv_components(g.EdgeGraph(6, [(0, 1), (1, 2), (4, 5)]), p=1, variant=variant)
    assert labels.tolist() == [0, 0, 0, 3, 4, 4]


def test_errors(cuda):
    with pytest.raises(ValueError):
        g.sv_components(g.EdgeGraph(3, [[0, 1]]), p=8)
    with pytest.raises(g.InvalidGraphError, match="out of range at row 1"):
        g.sv_components(g.EdgeGraph(3, [[0, 1], [2, 3], [1, 1]]), p=1)
    with pytest.raises(g.InvalidGraphError, match="self-loop at edge 1"):
        g.sv_components(g.EdgeGraph(3, [[0, 1], [2, 2], [1, 1]]), p=1)
    with pytest.raises(g.InvalidGraphError, match="out of range at row 0"):
        g.sv_components(g.EdgeGraph(3, [[-1, 1]]), p=1)
    # invalid graph wins over p > n (concomp.py:215-218)
    with pytest.raises(g.InvalidGraphError):
        g.sv_components(g.EdgeGraph(3, [[0, 5]]), p=8)
    with pytest.raises(ValueError):
        g.sv_components(g.EdgeGraph(3, [[0, 1]]), p=1, backend="cuda")


@pytest.mark.parametrize("variant", VARIANTS)
def test_matches_reference_goldens(cuda, golden, variant):
    for i, (n, d, s) in enumerate(golden["rg_cases"].tolist()):
        gr = g.EdgeGraph(int(n), golden[f"rg_{i}_edges"])
        labels, stats = g.sv_components(gr, p=min(30, int(n)), variant=variant)
        assert np.array_equal(labels, golden[f"rg_{i}_labels"]), (n, d, s)
        assert stats.meta["oriented_m"] == 2 * gr.m
        assert stats.rounds <= stats.meta["round_bound"]
    for i, (n, k, s) in enumerate(golden["tr_cases"].tolist()):
        gr = g.EdgeGraph(n, golden[f"tr_{i}_edges"])
        labels, _ = g.sv_components(gr, p=32, variant=variant)
        assert np.array_equal(labels, golden[f"tr_{i}_labels"]), (n, k, s)
    gr = g.EdgeGraph(3000, golden["path_3000_2_edges"])
    labels, _ = g.sv_components(gr, p=64, variant=variant)
    assert np.array_equal(labels, golden["path_3000_2_labels"])


@pytest.mark.parametrize("variant", VARIANTS)
def test_paths_trees_random_vs_oracle(cuda, orc, variant):
    for n in [1, 2, 17, 256, 3000, 100_000]:
        for seed in range(3):
            gr = g.list_to_graph(g.gen_list(n, seed=seed))
            labels, stats = g.sv_components(gr, p=min(64, n), variant=variant)
            assert np.array_equal(labels, orc.seq_components(n, gr.edges)), (n, seed)
            assert stats.rounds <= stats.meta["round_bound"]
    for n, k in [(50, 2), (300, 3), (2000, 10), (100_000, 2), (100_000, 10)]:
        gr = g.gen_tree_graph(n, k, seed=1)
        labels, _ = g.sv_components(gr, p=32, variant=variant)
        assert np.array_equal(labels, orc.seq_components(n, gr.edges)), (n, k)
    for n, d in [(10_000, 0.001), (3000, 0.01), (200_000, 2e-5)]:
        gr = g.gen_random_graph(n, d, seed=3)
        labels, _ = g.sv_components(gr, p=64, variant=variant)
        assert np.array_equal(labels, orc.seq_components(n, gr.edges)), (n, d)


@pytest.mark.parametrize("variant", VARIANTS)
def test_roots_per_round_monotone(cuda, variant):
    gr = g.gen_tree_graph(500, 3, seed=9)
    labels, stats = g.sv_components(gr, p=16, variant=variant)
    roots = stats.meta["roots_per_round"]
    assert roots[0] == 500
    assert all(a >= b for a, b in zip(roots, roots[1:]))
    assert roots[-1] == len(np.unique(labels))


def test_sv_round_behaviour(cuda):
    # test_concomp.py:214-227 -- SV round-count properties (variant "sv")
    g_path = g.list_to_graph(g.gen_list(3000, seed=5))
    g_tree = g.gen_tree_graph(3000, 4, seed=5)
    _, s1 = g.sv_components(g_path, p=64, variant="sv")
    _, s2 = g.sv_components(g_tree, p=64, variant="sv")
    assert abs(s1.rounds - s2.rounds) <= 2 or max(s1.rounds, s2.rounds) <= s1.meta["round_bound"]
    g_tree = g.gen_tree_graph(10_000, 3, seed=6)
    g_rand = g.gen_random_graph(1000, 0.02, seed=6)
    _, s_tree = g.sv_components(g_tree, p=64, variant="sv")
    _, s_rand = g.sv_components(g_rand, p=64, variant="sv")
    assert s_rand.rounds < s_tree.rounds, (s_rand.rounds, s_tree.rounds)
    # uf converges in one hook sweep on every graph
    _, s = g.sv_components(g_tree, p=64, variant="uf")
    assert s.rounds == 1 and s.meta["edge_sweeps"] == 1


def test_acceptance_criteria_2_3(cuda, orc):
    # test_acceptance.py:81-131 (5 seeds per family instead of 20)
    cfgs = [("list", None, 100_000), ("tree", 2, 100_000), ("tree", 3, 100_000), ("tree", 10, 100_000),
            ("random", 0.001, 10_000), ("random", 0.01, 3000)]
    for fam, prm, n in cfgs:
        for seed in range(5):
            if fam == "list":
                gr = g.list_to_graph(g.gen_list(n, seed=seed))
            elif fam == "tree":
                gr = g.gen_tree_graph(n, prm, seed=seed)
            else:
                gr = g.gen_random_graph(n, prm, seed=seed)
            want = orc.seq_components(n, gr.edges)
            for variant in VARIANTS:
                labels, stats = g.sv_components(gr, p=min(864, n), variant=variant, seed=seed)
                assert np.array_equal(labels, want), (fam, prm, seed, variant)
                assert stats.rounds <= g.sv_round_bound(n)


@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
def test_device_resident_graph(cuda, orc, dtype):
    gr = g.gen_random_graph(50_000, 4e-5, seed=2)
    want = orc.seq_components(gr.n, gr.edges)
    d = g.EdgeGraph(gr.n, torch.from_numpy(gr.edges).to(cuda, dtype))
    for variant in VARIANTS:
        labels, _ = g.sv_components(d, p=64, variant=variant)
        assert labels.is_cuda and labels.dtype == dtype
        assert np.array_equal(labels.cpu().numpy(), want)


def test_against_reference_digests(cuda, hashes):
    for n, m in [(1 << 16, 1 << 18), (1 << 20, 1 << 22), (1 << 22, 1 << 24)]:
        gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=cuda)
        assert gr.m == m
        assert sha(gr.edges) == hashes[f"gen_random_graph_{n}_{m}_0"]
        for variant in VARIANTS:
            labels, stats = g.sv_components(gr, p=64, variant=variant)
            assert sha(labels) == hashes[f"seq_components_{n}_{m}_0"], (n, variant)
            assert stats.meta["roots_per_round"][-1] == hashes[f"components_{n}_{m}_0"]


def _check_label_properties(edges, labels, n):
    """Size-independent: every edge joins equal labels, labels are fixpoints
    (label[label[i]] == label[i]) and minimal (label[i] <= i)."""
    e = edges.to(torch.int64)
    lab = labels.to(torch.int64)
    assert torch.all(lab[e[:, 0]] == lab[e[:, 1]])
    assert torch.all(lab[lab] == lab)
    assert torch.all(lab <= torch.arange(n, device=lab.device))


def test_full_size_properties_2_26(cuda):
    n, m = 1 << 26, 1 << 28
    gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=cuda)
    e32 = g.EdgeGraph(n, gr.edges.to(torch.int32))
    del gr
    labels, stats = g.sv_components(e32, p=1024)
    _check_label_properties(e32.edges, labels, n)
    # minimality: every vertex labelled r lies in r's component and r is its smallest member
    roots = int((labels == torch.arange(n, device=cuda, dtype=labels.dtype)).sum())
    assert stats.meta["roots_per_round"][-1] == roots
    # the reference's own count for C5 (seq_components on gen_random_graph(2^26, .., seed=0))
    assert e32.m == m and roots == 22_599
    sv, _ = g.sv_components(e32, p=1024, variant="sv")
    assert torch.equal(sv, labels)


def test_building_blocks_c_abi(cuda, orc):
    """sg_cc_init / sg_cc_hook / sg_cc_compress / sg_cc_labels compose into
    the same labels (the multi-GPU path's kernels)."""
    gr = g.gen_random_graph(20_000, 1e-4, seed=1)
    want = orc.seq_components(gr.n, gr.edges)
    L = _native.lib()
    e = torch.from_numpy(gr.edges.astype(np.int32)).to(cuda)
    D = torch.empty(gr.n, dtype=torch.int32, device=cuda)
    flags = torch.zeros(4, dtype=torch.int64, device=cuda)
    roots = torch.zeros(1, dtype=torch.int64, device=cuda)
    s = _device.stream_ptr(cuda)
    assert L.sg_cc_init(_device.ptr(D), gr.n, s) == 0
    half = gr.m // 2
    for row0, blk in ((0, e[:half]), (half, e[half:])):
        assert L.sg_cc_hook(_device.ptr(blk), _native.SG_I32, blk.shape[0], row0, gr.n, _device.ptr(D),
                            _native.SG_CC_UF, 1, _device.ptr(flags), s) == 0
    assert L.sg_cc_compress(_device.ptr(D), 0, gr.n, _device.ptr(roots), s) == 0
    out = torch.empty(gr.n, dtype=torch.int64, device=cuda)
    assert L.sg_cc_labels(_device.ptr(D), gr.n, _device.ptr(out), _native.SG_I64, s) == 0
    assert np.array_equal(out.cpu().numpy(), want)
    assert int(roots.item()) == len(np.unique(want))
    assert int(flags[0].item()) == 1 and int(flags[1].item()) == 0 and int(flags[2].item()) == 0


@pytest.mark.parametrize("part", ["chunks", "count"])
@pytest.mark.parametrize("variant", VARIANTS)
def test_partitioned_path_small_windows(cuda, orc, sg_env, variant, part):
    """Force the windowed (partitioned-edge) hook on small graphs: windows of
    2^12 vertices -> up to 16 partitions; both partition layouts (one-pass
    chunk lists, the default, and count + scatter).  The star and the
    one-window graph put every edge of a tile into one window (chunk claims
    several chunks per tile); the last case has fewer edges than one tile
    per CTA, so most chunks are padding."""
    sg_env(SG_CC_WBITS="12", **({"SG_CC_PART": "count"} if part == "count" else {}))
    n = 70_000  # > 2^16 edges in the star: partitioned
    star = np.stack([np.arange(n - 1, dtype=np.int64), np.full(n - 1, n - 1, dtype=np.int64)], axis=1)
    rng = np.random.default_rng(5)
    hi = rng.integers(65_600, n, size=(200_000, 2), dtype=np.int64)  # every edge in the top window
    hi = hi[hi[:, 0] != hi[:, 1]]
    lowonly = rng.integers(0, 10_000, size=(70_000, 2), dtype=np.int64)  # windows >= 3 of 16 stay empty
    lowonly = lowonly[lowonly[:, 0] != lowonly[:, 1]]
    exact = g.list_to_graph(g.gen_list((1 << 16) + 1, seed=6))  # exactly 2^16 rows: the split threshold
    cases = [g.gen_random_graph(60_000, 5e-5, seed=4), g.gen_tree_graph(70_000, 3, seed=2),
             g.list_to_graph(g.gen_list(66_000, seed=1)), g.gen_random_graph(30_000, 2e-4, seed=9),
             g.EdgeGraph(n, star), g.EdgeGraph(n, hi), g.gen_random_graph(300_000, 2e-6, seed=3),
             g.EdgeGraph(60_000, lowonly), exact]
    for gr in cases:
        labels, stats = g.sv_components(gr, p=64, variant=variant)
        assert np.array_equal(labels, orc.seq_components(gr.n, gr.edges)), (gr.n, gr.m)
        assert any(r.kernel == "cc_partition" for r in stats.launch_log)
    e = g.gen_random_graph(60_000, 5e-5, seed=4).edges.copy()
    e[40_000] = [7, 7]
    e[80_000] = [3, 60_000]
    with pytest.raises(g.InvalidGraphError, match="self-loop at edge 40000"):
        g.sv_components(g.EdgeGraph(60_000, e[:70_000]), p=8, variant=variant)
    with pytest.raises(g.InvalidGraphError, match="out of range at row 80000"):
        g.sv_components(g.EdgeGraph(60_000, e), p=8, variant=variant)


@pytest.mark.parametrize("variant", VARIANTS)
def test_sharded_path_on_nccl_single_rank(cuda, orc, sg_env, tmp_path, variant):
    """The edge-sharded product path (dist.sv_components_dist: partitioned
    per-rank hook via sg_cc_hook_part, NCCL min all-reduce, sharded
    shortcut + all-gather) on a one-rank NCCL group, windows forced small so
    the block is split; plus the launch trace and global-row validation."""
    import torch.distributed as dist

    from paper_1002_4482_b200 import dist as sgdist

    sg_env(SG_CC_WBITS="12")
    store = dist.FileStore(str(tmp_path / "store"), 1)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=cuda)
    try:
        for gr in (g.gen_random_graph(60_000, 5e-5, seed=4), g.gen_tree_graph(70_000, 3, seed=2)):
            labels, stats = sgdist.sv_components_dist(gr, 64, variant=variant)
            assert np.array_equal(labels, orc.seq_components(gr.n, gr.edges))
            names = {r.kernel for r in stats.launch_log}
            assert {"nccl_allreduce_min", "cc_shortcut"} <= names and any(k.startswith("cc_hook") for k in names)
        e = g.gen_random_graph(60_000, 5e-5, seed=4).edges.copy()
        e[50_000] = [9, 9]
        with pytest.raises(g.InvalidGraphError, match="self-loop at edge 50000"):
            sgdist.sv_components_dist(g.EdgeGraph(60_000, e), 8, variant=variant)
    finally:
        dist.destroy_process_group()


def test_sparse_merge_building_blocks(cuda):
    """sg_cc_changes / sg_cc_apply_min: the sharded rounds' changed-entry
    exchange (dist.py) reproduces the dense min all-reduce."""
    L = _native.lib()
    n = 1 << 20
    rng = np.random.default_rng(7)
    base = np.arange(n, dtype=np.int32)
    a = base.copy()
    b = base.copy()
    ia = rng.choice(n, 5000, replace=False)
    ib = rng.choice(n, 7000, replace=False)
    a[ia] = (ia * rng.random(ia.size)).astype(np.int32)
    b[ib] = (ib * rng.random(ib.size)).astype(np.int32)
    old = torch.from_numpy(base).to(cuda)
    out = {}
    for name, arr in (("a", a), ("b", b)):
        D = torch.from_numpy(arr).to(cuda)
        cap = 8192
        idx = torch.empty(cap, dtype=torch.int32, device=cuda)
        val = torch.empty(cap, dtype=torch.int32, device=cuda)
        cnt = torch.zeros(1, dtype=torch.int64, device=cuda)
        rc = L.sg_cc_changes(_device.ptr(old), _device.ptr(D), n, _device.ptr(idx), _device.ptr(val), cap,
                             _device.ptr(cnt), _device.stream_ptr(cuda))
        assert rc == 0
        k = int(cnt.item())
        assert k == int((arr != base).sum())
        got = dict(zip(idx[:k].cpu().tolist(), val[:k].cpu().tolist()))
        assert got == {int(i): int(arr[i]) for i in np.flatnonzero(arr != base)}
        out[name] = (idx[:k], val[:k])
    D = torch.from_numpy(a).to(cuda)  # rank a applies rank b's changes
    rc = L.sg_cc_apply_min(_device.ptr(D), _device.ptr(out["b"][0]), _device.ptr(out["b"][1]), out["b"][0].numel(),
                           _device.stream_ptr(cuda))
    assert rc == 0
    assert np.array_equal(D.cpu().numpy(), np.minimum(a, b))


def test_c4_matches_reference_counts(cuda):
    """C4 (BASELINE configs[3]): gen_random_graph(2^22, m = 2^24, seed 0) has
    1 437 components, the largest with 4 192 867 vertices (the reference's
    seq_components)."""
    n, m = 1 << 22, 1 << 24
    gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=cuda)
    assert gr.m == m
    labels, _ = g.sv_components(gr, p=1024)
    counts = torch.bincount(labels.to(torch.int64), minlength=n)
    assert int((counts > 0).sum()) == 1_437
    assert int(counts.max()) == 4_192_867


@pytest.mark.parametrize("split", ["0", "1", "3", "5", "3+1"])
def test_uf_split_hook(cuda, orc, sg_env, split):
    """Unpartitioned UF with a full shortcut sweep after the first m / 2^f rows
    (SG_CC_SPLIT=f; 3 is the default, 0 one hook launch): labels exact on
    random, tree, path and int64 / device-resident edge lists (the second hook
    starts m1 rows in, so 16-B rows are offset correctly), the invalid row
    reported by its global index from either half, and one more vertex sweep
    counted per sweep when the split applies (m >= 2^16); "3+1" adds the
    second sweep after m / 2 rows (SG_CC_SPLIT2)."""
    f, _, f2 = split.partition("+")
    sg_env(SG_CC_SPLIT=f, SG_CC_SPLIT2=f2 or "0")
    cases = [g.gen_random_graph(1 << 16, 4.0 / (1 << 16), seed=11), g.gen_tree_graph(90_000, 3, seed=4),
             g.list_to_graph(g.gen_list(70_001, seed=8)), g.gen_random_graph(5_000, 1e-3, seed=2)]
    base = None
    for gr in cases:
        labels, stats = g.sv_components(gr, p=64, variant="uf")
        assert np.array_equal(labels, orc.seq_components(gr.n, gr.edges)), (gr.n, gr.m, split)
        if gr is cases[0]:
            base = stats.meta["vertex_sweeps"]
        d = torch.from_numpy(gr.edges.astype(np.int64)).to(cuda)  # int64 rows on the device
        dl, _ = g.sv_components(g.EdgeGraph(gr.n, d), p=64, variant="uf")
        assert np.array_equal(dl.cpu().numpy(), orc.seq_components(gr.n, gr.edges))
    assert base == 2 + (f != "0") + (f2 != "")
    e = cases[0].edges.copy()
    m = len(e)
    for row in (m // 64, m - 3):  # before and after the split point
        bad = e.copy()
        bad[row] = [5, 5]
        with pytest.raises(g.InvalidGraphError, match=f"self-loop at edge {row}"):
            g.sv_components(g.EdgeGraph(cases[0].n, bad), p=8, variant="uf")


@pytest.mark.parametrize("comp4", ["0", "1"])
@pytest.mark.parametrize("variant", VARIANTS)
def test_shortcut_widths(cuda, orc, sg_env, comp4, variant):
    """cc_shortcut with one or four vertices per thread (SG_CC_COMP4): n not
    a multiple of four (the trailing vertices), int64 labels from host input
    (separate label buffer) and u32 labels in place on the device, the root
    count in roots_per_round."""
    sg_env(SG_CC_COMP4=comp4)
    for gr in (g.gen_random_graph(100_003, 3e-5, seed=21), g.gen_tree_graph(50_001, 4, seed=3),
               g.list_to_graph(g.gen_list(9_999, seed=5)), g.EdgeGraph(7, [[1, 2], [5, 6]])):
        want = orc.seq_components(gr.n, gr.edges)
        labels, st = g.sv_components(gr, p=min(64, gr.n), variant=variant)
        assert np.array_equal(labels, want)
        assert st.meta["roots_per_round"][-1] == int(np.count_nonzero(want == np.arange(gr.n)))
        d = torch.from_numpy(gr.edges.astype(np.int32)).to(cuda)
        dl, _ = g.sv_components(g.EdgeGraph(gr.n, d), p=min(64, gr.n), variant=variant)
        assert np.array_equal(dl.cpu().numpy().astype(np.int64), want)
