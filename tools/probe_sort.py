"""Reference point: torch.sort (CUB onesweep radix sort) throughput on this GPU."""
import torch
dev = torch.device("cuda", 0)
for logn in (26, 28):
    n = 1 << logn
    k32 = torch.randint(0, 1 << 31, (n,), dtype=torch.int32, device=dev)
    k64 = torch.randint(0, 1 << 62, (n,), dtype=torch.int64, device=dev)
    for name, k in (("int32 keys + idx", k32), ("int64 keys + idx", k64)):
        torch.sort(k, stable=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        torch.sort(k, stable=True)
        b.record()
        b.synchronize()
        print(f"2^{logn} {name}: {a.elapsed_time(b):.3f} ms")
