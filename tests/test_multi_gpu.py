"""Components over several GPUs from one process (dist.sv_components_multi
-> the C ABI's sg_cc_multi): per-device hook sweeps over the
row blocks, NCCL min all-reduce per round, sharded shortcut + all-gather
(concomp.py:225-240).  The box has one GPU, so the clique is devices=[0];
the per-device loops, the NCCL calls, the global-row validation and the
round logic all run."""
import numpy as np
import pytest
import torch

import paper_1002_4482_b200 as g
from paper_1002_4482_b200 import dist as sgdist

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", ["uf", "sv"])
@pytest.mark.parametrize("wbits", [None, "12"])
def test_multi_matches_oracle(cuda, orc, sg_env, variant, wbits):
    if wbits:
        sg_env(SG_CC_WBITS=wbits)  # windows of 2^12 vertices: the split, chunked hook path
    for gr in (g.gen_random_graph(60_000, 5e-5, seed=4), g.gen_tree_graph(70_000, 3, seed=2),
               g.gen_random_graph(1 << 18, 3.0 / (1 << 18), seed=7)):
        labels, stats = sgdist.sv_components_multi(gr, 64, devices=[0], variant=variant)
        assert labels.dtype == np.int64
        assert np.array_equal(labels, orc.seq_components(gr.n, gr.edges)), (gr.n, variant)
        assert stats.meta["world"] == 1 and stats.rounds >= 1
        assert stats.meta["roots_per_round"][-1] == len(np.unique(labels))


def test_multi_device_graph_and_errors(cuda, orc):
    gr = g.gen_random_graph(1 << 20, (1 << 21) / ((1 << 20) * ((1 << 20) - 1) // 2), seed=3)
    d = g.EdgeGraph(gr.n, torch.from_numpy(gr.edges).to(cuda).to(torch.int32))
    labels, _ = sgdist.sv_components_multi(d, 64, devices=[0])
    assert labels.is_cuda and np.array_equal(labels.cpu().numpy(), orc.seq_components(gr.n, gr.edges))
    e = gr.edges.copy()
    e[123_456] = [5, 5]
    with pytest.raises(g.InvalidGraphError, match="self-loop at edge 123456"):
        sgdist.sv_components_multi(g.EdgeGraph(gr.n, e), 64, devices=[0])
    e[100_000] = [gr.n + 3, 1]
    with pytest.raises(g.InvalidGraphError, match="out of range at row 100000"):
        sgdist.sv_components_multi(g.EdgeGraph(gr.n, e), 64, devices=[0])
    with pytest.raises(ValueError):
        sgdist.sv_components_multi(gr, gr.n + 1, devices=[0])
