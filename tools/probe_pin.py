"""D2H options for a 2^26 int64 result: pinned alloc + copy vs pageable."""
import time
import numpy as np
import torch

n = 1 << 26
dev = torch.device("cuda", 0)
d = torch.arange(n, dtype=torch.int64, device=dev)
torch.cuda.synchronize()


def t(label, fn, reps=6):
    ts = []
    keep = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        keep.append(fn())
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
        if len(keep) > 2:
            keep.pop(0)
    print(f"{label:40s} " + " ".join(f"{x:7.2f}" for x in ts))


def pinned():
    h = torch.empty(n, dtype=torch.int64, pin_memory=True)
    h.copy_(d, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


def pageable():
    a = np.empty(n, dtype=np.int64)
    torch.from_numpy(a).copy_(d)
    return a


t("pinned alloc+copy (torch.empty pin)", pinned)
t("pageable np.empty + copy", pageable)
t("pinned alloc only", lambda: torch.empty(n, dtype=torch.int64, pin_memory=True))
