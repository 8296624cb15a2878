"""Where the end-to-end time of rs_rank / sv_components goes (pinned int64 host
input -> numpy int64 output).  python tools/probe_e2e.py lr26|cc26"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "lr26"
dev = torch.device("cuda", 0)
logn = int(w[2:4])
n = 1 << logn
if w.startswith("lr"):
    sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32)
    host = sl.succ.to(torch.int64).cpu().pin_memory()
    call = lambda x: g.rs_rank(g.SuccessorList(x), 16384)  # noqa: E731
else:
    m = 4 * n
    gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=dev)
    host = gr.edges.to(torch.int64).cpu().pin_memory()
    call = lambda x: g.sv_components(g.EdgeGraph(n, x), 1024)  # noqa: E731
call(host)


def t(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


d = host.to(dev)
out_dev = torch.empty(n, dtype=torch.int64, device=dev)
pin_out = torch.empty(n, dtype=torch.int64, pin_memory=True)
print(w, "bytes in", host.numel() * 8, "out", n * 8)
print("h2d pinned ms", t(lambda: host.to(dev, non_blocking=True)))
print("d2h pinned ms", t(lambda: pin_out.copy_(out_dev, non_blocking=True)))
print("api device-resident int64 ms", t(lambda: call(d)))
print("api host pinned (e2e) ms", t(lambda: call(host)))
npin = host.numpy().copy()
print("api host numpy pageable ms", t(lambda: call(npin), reps=3))
