"""Quick device-time probe of the hot paths (development aid, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1002_4482_b200 as g

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); out = fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts), out

dev = torch.device("cuda", 0)
for logn in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["20", "24", "26", "28"])]:
    n = 1 << logn
    t0 = time.time(); sl = g.gen_list(n, seed=0, device=dev, dtype=torch.int32); torch.cuda.synchronize()
    print(f"gen_list 2^{logn}: {time.time()-t0:.2f}s", flush=True)
    ms, (rank, st) = timeit(lambda: g.rs_rank(sl, 16384))
    per = {k: round(v.ms, 3) for k, v in st.per_kernel().items()}
    print(f"rs_rank 2^{logn} random: {ms:.3f} ms  {n/ms/1e6:.2f} Gnodes/s  levels={st.meta['levels']} sizes={st.meta['level_size']} fb={st.meta['fallback']} per={per}", flush=True)
    if logn <= 26:
        ms, (rank, st) = timeit(lambda: g.wyllie_rank(sl, 1024), reps=2)
        print(f"wyllie 2^{logn} random: {ms:.3f} ms  {n/ms/1e6:.2f} Gnodes/s", flush=True)
    so = g.ordered_list(n, device=dev, dtype=torch.int32)
    ms, (rank, st) = timeit(lambda: g.rs_rank(so, 16384))
    per = {k: round(v.ms, 3) for k, v in st.per_kernel().items()}
    print(f"rs_rank 2^{logn} ordered: {ms:.3f} ms  {n/ms/1e6:.2f} Gnodes/s per={per}", flush=True)
    del sl, so, rank
for logn, logm in [(22, 24), (26, 28)]:
    n, m = 1 << logn, 1 << logm
    t0 = time.time(); gr = g.gen_random_graph(n, m / (n*(n-1)//2), seed=0, device=dev); torch.cuda.synchronize()
    print(f"gen_random_graph 2^{logn}/2^{logm}: {time.time()-t0:.2f}s", flush=True)
    e32 = g.EdgeGraph(n, gr.edges.to(torch.int32)); del gr
    for variant in ("uf", "sv"):
        ms, (lab, st) = timeit(lambda: g.sv_components(e32, 1024, variant=variant))
        per = {k: round(v.ms, 3) for k, v in st.per_kernel().items()}
        print(f"cc {variant} 2^{logn}/2^{logm}: {ms:.3f} ms {m/ms/1e6:.2f} Gedges/s rounds={st.rounds} per={per}", flush=True)
    del e32
