#!/bin/bash
# step spread with GC paused vs running
TAG=${TAG:-r02o}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
for i in 1 2 3; do
for gcm in 0 1; do
  SG_BENCH_GC=$gcm timeout 300 python bench.py --workload lr26 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/lr26_gc${gcm}_$i.json 2>$O/lr26_gc${gcm}_$i.err
done
done
timeout 300 python bench.py --workload cc26 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/cc26.json 2>$O/cc26.err
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], round(sum(k.values()),4), d['clocks']['samples'], d.get('step_ms_spread'), k.get('cc_partition'), k.get('rs5_refine'))"; done
