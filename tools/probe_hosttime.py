"""Host-side phases of rs_rank calls (SG_HOST_TIMING=1 prints them from libsg)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402

dev = torch.device("cuda", 0)
w = sys.argv[1] if len(sys.argv) > 1 else "lr26"
n = 1 << int(w[2:4])
sl = g.ordered_list(n, device=dev, dtype=torch.int32) if w.endswith("o") else \
    g.gen_list(n, seed=0, device=dev, dtype=torch.int32)
for _ in range(3):
    g.rs_rank(sl, 16384)
torch.cuda.synchronize()
os.environ["SG_HOST_TIMING"] = "1"
for _ in range(2):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    out, st = g.rs_rank(sl, 16384)
    t1 = time.perf_counter()
    b.record()
    b.synchronize()
    print(f"api {a.elapsed_time(b):.3f} ms (host {1e3 * (t1 - t0):.3f}); device pipeline {st.wall_time * 1e3:.3f} ms",
          file=sys.stderr, flush=True)
