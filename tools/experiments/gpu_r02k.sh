#!/bin/bash
# refine atom (new default), partition pre-claim, NVML poll period vs step time, NT-store boundary copies
TAG=${TAG:-r02k}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_concomp_gpu.py tests/test_listrank_gpu.py tests/test_boundary_gpu.py -q -x > $O/pytest.log 2>&1
timeout 300 python bench.py --workload cc26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc26.json 2>$O/cc26.err
for pm in 2 20 100; do
  SG_BENCH_POLL_MS=$pm timeout 300 python bench.py --workload lr28 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr28_poll$pm.json 2>$O/lr28_poll$pm.err
done
SG_BENCH_POLL_MS=20 SG_BENCH_POLL_UTIL=1 timeout 300 python bench.py --workload lr28 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr28_poll20u.json 2>$O/lr28_poll20u.err
timeout 300 python bench.py --workload lr26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr26.json 2>$O/lr26.err
timeout 300 python tools/probe_overhead.py lr28 > $O/overhead_lr28.txt 2>&1
timeout 600 python tools/probe_e2e2.py > $O/e2e_phases.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'part_chunks' -s 0 -c 1 \
    -o $O/ncu_cc26_part python bench.py --workload cc26 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_cc.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine -s 2 -c 1 \
    -o $O/ncu_refine_atom python bench.py --workload lr28 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_refine.log 2>&1
lscpu > $O/lscpu.txt 2>&1
tail -n 3 $O/pytest.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], round(sum(k.values()),4), {a:b for a,b in k.items() if b>0.1}, d['clocks']['samples'], d['clocks']['sm_mhz'])"; done
cat $O/overhead_lr28.txt $O/e2e_phases.txt
