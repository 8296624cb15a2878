"""Time one workload (device-resident inputs) and print per-kernel ms as JSON.
    python tools/probe_one.py lr26|lr28|lr28o|cc22|cc26[:variant] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_4482_b200 as g  # noqa: E402

w = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda", 0)
variant = w.split(":")[1] if ":" in w else "uf"
w = w.split(":")[0]
logn = int(w[2:4])
if w.startswith(("lr", "wy")):
    sl = g.ordered_list(1 << logn, device=dev, dtype=torch.int32) if w.endswith("o") else \
        g.gen_list(1 << logn, seed=0, device=dev, dtype=torch.int32)
    fn = (lambda: g.wyllie_rank(sl, 1024)) if w.startswith("wy") else (lambda: g.rs_rank(sl, 16384))
else:
    n, m = 1 << logn, 1 << (logn + 2)
    gr = g.gen_random_graph(n, m / (n * (n - 1) // 2), seed=0, device=dev)
    e = g.EdgeGraph(n, gr.edges.to(torch.int32))
    del gr
    fn = lambda: g.sv_components(e, 1024, variant=variant)  # noqa: E731
fn()
best = None
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    out, st = fn()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b)
    if best is None or ms < best[0]:
        best = (ms, {k: round(v.ms, 4) for k, v in st.per_kernel().items()})
print(json.dumps({"workload": sys.argv[1], "env": {k: v for k, v in os.environ.items() if k.startswith("SG_")},
                  "ms": round(best[0], 4), "kernels": best[1]}), flush=True)
