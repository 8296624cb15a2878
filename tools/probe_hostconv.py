"""Probe: can host-side int64 <-> u32 conversion feed PCIe faster than
moving int64?  Times (a) pinned int64 H2D / D2H of 2^28 elements, (b)
multi-threaded narrowing int64 -> pinned int32 and widening pinned int32 ->
int64 (torch CPU copy kernels, all host threads), (c) int32 H2D / D2H."""
import time

import torch

n = 1 << 28
torch.set_num_threads(torch.get_num_threads())
print("host threads", torch.get_num_threads())
dev = torch.device("cuda", 0)
h64 = torch.randint(0, n, (n,), dtype=torch.int64).pin_memory()
p32 = torch.empty(n, dtype=torch.int32).pin_memory()
o64 = torch.empty(n, dtype=torch.int64).pin_memory()
d64 = torch.empty(n, dtype=torch.int64, device=dev)
d32 = torch.empty(n, dtype=torch.int32, device=dev)


def t(f, reps=3):
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print("H2D int64 pinned   %.1f ms" % t(lambda: d64.copy_(h64, non_blocking=True)))
print("D2H int64 pinned   %.1f ms" % t(lambda: o64.copy_(d64, non_blocking=True)))
print("H2D int32 pinned   %.1f ms" % t(lambda: d32.copy_(p32, non_blocking=True)))
print("D2H int32 pinned   %.1f ms" % t(lambda: p32.copy_(d32, non_blocking=True)))
for th in (1, 4, 8, 16, torch.get_num_threads()):
    torch.set_num_threads(th)
    print("threads %2d narrow i64->pinned i32 %.1f ms   widen pinned i32->i64 %.1f ms   memcpy i64 %.1f ms" % (
        th, t(lambda: p32.copy_(h64)), t(lambda: o64.copy_(p32)), t(lambda: o64.copy_(h64))))
