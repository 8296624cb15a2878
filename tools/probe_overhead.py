"""Host-side overhead of one rs_rank / sv_components call on device-resident
input: event time of the whole API call vs the sum of its kernels, and the
splitter-meta tail.  python tools/probe_overhead.py lr26"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402
from paper_1002_4482_b200 import listrank  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "lr26"
dev = torch.device("cuda", 0)
n = 1 << int(w[2:4])
sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32)
for _ in range(3):
    g.rs_rank(sl, 16384)
torch.cuda.synchronize()
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    out, st = g.rs_rank(sl, 16384)
    t1 = time.perf_counter()
    b.record()
    b.synchronize()
    ksum = sum(r.ms for r in st.launch_log)
    print(f"api event {a.elapsed_time(b):.3f} ms  host {1e3 * (t1 - t0):.3f} ms  kernels {ksum:.3f} ms  "
          f"pipeline(device total) {st.wall_time * 1e3:.3f} ms  launches {len(st.launch_log)}")
# the native call alone
t0 = time.perf_counter()
rank, nst, rc, viol, hi = listrank._run_list("rs", sl, 0, 0, False)
t1 = time.perf_counter()
print(f"native call {1e3 * (t1 - t0):.3f} ms (includes status sync)")
t0 = time.perf_counter()
spl = listrank._draw_splitters(n, 16384, 0)
ss = listrank._splitter_set(rank, spl, n, key=(n, 16384, 0))
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"splitter meta {1e3 * (t1 - t0):.3f} ms")
