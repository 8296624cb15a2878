"""cProfile of back-to-back rs_rank calls (device-resident lr26): where the
host time of a call goes outside the native pipeline."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 26
sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32)
for _ in range(5):
    g.rs_rank(sl, 16384)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    out, st = g.rs_rank(sl, 16384)
pr.disable()
ps = pstats.Stats(pr).sort_stats("tottime")
ps.print_stats(25)
