"""Where does the per-call time go?  Device time of the raw C-ABI call vs the
full Python API call (meta derivation, stats), on a device-resident list."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402
from paper_1002_4482_b200 import _device, _native, listrank  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32)
L = _native.lib()
rank = torch.empty(n, dtype=torch.int32, device=dev)
ws = _device.workspace(L.sg_rs_workspace_bytes(n), dev)
st, v = _native.Stats(), _native.Violation()


def raw():
    return L.sg_rs_rank(_device.ptr(sl.succ), _native.SG_I32, _device.ptr(rank), _native.SG_I32, n, 0,
                        _device.ptr(ws), ws.numel(), _device.stream_ptr(dev), ctypes.byref(st), ctypes.byref(v))


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


print("raw C-ABI call   ms:", round(timed(raw), 3), " (device pipeline total", round(st.total_ms, 3), ")")
print("raw, no stats    ms:", round(timed(lambda: L.sg_rs_rank(_device.ptr(sl.succ), _native.SG_I32, _device.ptr(rank),
                                                               _native.SG_I32, n, 0, _device.ptr(ws), ws.numel(),
                                                               _device.stream_ptr(dev), None, None)), 3))
print("rs_rank API      ms:", round(timed(lambda: g.rs_rank(sl, 16384)), 3))
out = g.rs_rank(sl, 16384)[0]
print("splitter meta    ms:", round(timed(lambda: listrank._splitter_set(out, listrank._draw_splitters(n, 16384, 0), n)), 3))
print("per kernel:", {k: round(x.ms, 4) for k, x in g.rs_rank(sl, 16384)[1].per_kernel().items()})

# PCIe: pinned H2D / D2H of the e2e payloads
host = sl.succ.to(torch.int64).cpu().pin_memory()
dst = torch.empty_like(host, device=dev)
print("H2D 8n pinned    ms:", round(timed(lambda: dst.copy_(host, non_blocking=True)), 3), "for", host.numel() * 8 / 2**20, "MiB")
hb = torch.empty(host.shape, dtype=torch.int64, pin_memory=True)
print("D2H 8n pinned    ms:", round(timed(lambda: hb.copy_(dst, non_blocking=True)), 3))
hs = g.SuccessorList(host)
print("e2e API (pinned) ms:", round(timed(lambda: g.rs_rank(hs, 16384), reps=3), 3))
import numpy as np
hn = g.SuccessorList(host.numpy())
print("e2e API (numpy)  ms:", round(timed(lambda: g.rs_rank(hn, 16384), reps=3), 3))
