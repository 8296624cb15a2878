"""Host time of one rs_rank call split into: Python before the native call,
the native call (enqueue + its one synchronisation), Python after it.
python tools/probe_host_split.py lr26 30"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402
from paper_1002_4482_b200 import _native  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "lr26"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 30
dev = torch.device("cuda", 0)
n = 1 << int(w[2:4])
sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32)
L = _native.lib()
orig = L.sg_rs_rank_meta
marks = {}


def wrapped(*args):
    marks["n0"] = time.perf_counter()
    rc = orig(*args)
    marks["n1"] = time.perf_counter()
    return rc


L.sg_rs_rank_meta = wrapped
for _ in range(5):
    g.rs_rank(sl, 16384)
torch.cuda.synchronize()
pre, nat, post = [], [], []
for _ in range(calls):
    t0 = time.perf_counter()
    out, st = g.rs_rank(sl, 16384)
    t1 = time.perf_counter()
    pre.append(marks["n0"] - t0)
    nat.append(marks["n1"] - marks["n0"])
    post.append(t1 - marks["n1"])
med = lambda v: sorted(v)[len(v) // 2] * 1e6  # noqa: E731
print(f"{w}: python before {med(pre):.1f} us, native call {med(nat):.1f} us, python after {med(post):.1f} us "
      f"(device pipeline {st.wall_time * 1e6:.1f} us)")
