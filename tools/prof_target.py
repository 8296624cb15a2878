"""One call of a hot path on device-resident inputs, for ncu captures:
    python tools/prof_target.py lr26|lr28|lr28o|cc22|cc26|wy26 [variant]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402

w = sys.argv[1]
dev = torch.device("cuda", 0)
if w.startswith(("lr", "wy")):
    logn = int(w[2:4])
    sl = g.ordered_list(1 << logn, device=dev, dtype=torch.int32) if w.endswith("o") else \
        g.gen_list(1 << logn, seed=0, device=dev, dtype=torch.int32)
    torch.cuda.synchronize()
    if w.startswith("wy"):
        g.wyllie_rank(sl, 1024)
    else:
        g.rs_rank(sl, 16384)
else:
    logn = int(w[2:4])
    n, m = 1 << logn, 1 << (logn + 2)
    gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=dev)
    e = g.EdgeGraph(n, gr.edges.to(torch.int32))
    del gr
    torch.cuda.synchronize()
    g.sv_components(e, 1024, variant=sys.argv[2] if len(sys.argv) > 2 else "uf")
torch.cuda.synchronize()
