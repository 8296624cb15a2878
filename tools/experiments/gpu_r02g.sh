#!/bin/bash
# round-2 re-entry measurement pass: build, full GPU suite, default bench
# (lr28 + blocks), the reference arm, refine variants, the launch list
TAG=${TAG:-r02g}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for v in 0 1 2 4; do
  SG_RS_REFINE=$v timeout 300 python bench.py --workload lr28 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr28_ref$v.json 2>$O/lr28_ref$v.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_lr28.csv \
    python bench.py --workload lr28 --steps 2 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_launch.log 2>&1
tail -3 $O/pytest_gpu.log
tail -2 $O/smoke.log
for f in $O/lr28_ref*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], 'refine', k.get('rs5_refine'), 'scatter', k.get('rs5_scatter'))"; done
