"""Per-call timeline of back-to-back rs_rank calls on device-resident input:
CUDA-event time of each call, host time, and the native call's own phases
(SG_HOST_TIMING=1 prints them to stderr).  python tools/probe_steps.py lr26 40"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "lr26"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 40
dev = torch.device("cuda", 0)
n = 1 << int(w[2:4])
sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32)
torch.cuda.synchronize()
stream = torch.cuda.current_stream(dev)
for i in range(calls):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(stream)
    out, st = g.rs_rank(sl, 16384)
    b.record(stream)
    t1 = time.perf_counter()
    b.synchronize()
    ks = sum(r.ms for r in st.launch_log)
    print(f"call {i:3d}  event {a.elapsed_time(b):8.3f} ms  host {1e3 * (t1 - t0):8.3f} ms  kernels {ks:7.3f} ms",
          flush=True)
