"""cProfile of rs_rank on a device-resident 2^26 list (host-side overhead)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402

dev = torch.device("cuda", 0)
w = sys.argv[1] if len(sys.argv) > 1 else "lr26"
n = 1 << int(w[2:4])
sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32) if not w.endswith("o") else \
    g.ordered_list(n, device=dev, dtype=torch.int32)
for _ in range(3):
    g.rs_rank(sl, 16384)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    g.rs_rank(sl, 16384)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
