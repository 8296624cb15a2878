"""Phases of the e2e call at C3 (2^28 nodes, pinned int64 host list):
boundary H2D (narrowed vs int64), the device call, boundary D2H (widened vs
int64), each timed with a device sync around it."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1002_4482_b200 as g  # noqa: E402
from paper_1002_4482_b200 import _device  # noqa: E402

n = 1 << 28
dev = torch.device("cuda", 0)
sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32)
host = sl.succ.to(torch.int64).cpu().pin_memory()
hnp = host.numpy()
nppage = np.array(hnp)  # pageable copy


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print("to_device narrowed (pinned torch)  %.1f ms" % t(lambda: _device.to_device(host, dev, bound=n)))
print("to_device narrowed (pageable np)   %.1f ms" % t(lambda: _device.to_device(nppage, dev, bound=n)))
print("to_device int64 (pinned torch)     %.1f ms" % t(lambda: _device.to_device(host, dev)))
d32 = _device.to_device(host, dev, bound=n)[0]
r32 = torch.empty(n, dtype=torch.int32, device=dev)
print("rs_rank device int32               %.1f ms" % t(lambda: g.rs_rank(g.SuccessorList(d32), 16384)))
print("to_host_numpy widened              %.1f ms" % t(lambda: _device.to_host_numpy(d32)))
d64 = d32.to(torch.int64)
print("to_host_numpy int64                %.1f ms" % t(lambda: _device.to_host_numpy(d64)))
print("e2e rs_rank(pinned int64)          %.1f ms" % t(lambda: g.rs_rank(g.SuccessorList(host), 16384)))
print("e2e rs_rank(pageable numpy)        %.1f ms" % t(lambda: g.rs_rank(g.SuccessorList(nppage), 16384)))
