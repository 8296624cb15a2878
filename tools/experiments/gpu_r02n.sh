#!/bin/bash
# step-time spread with / without the NVML sampler
TAG=${TAG:-r02n}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
for i in 1 2 3; do
for pm in 0 20; do
  SG_BENCH_POLL_MS=$pm timeout 300 python bench.py --workload lr26 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/lr26_p${pm}_$i.json 2>$O/lr26_p${pm}_$i.err
done
done
for pm in 0 20; do
  SG_BENCH_POLL_MS=$pm timeout 300 python bench.py --workload lr28 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/lr28_p${pm}.json 2>$O/lr28_p${pm}.err
  SG_BENCH_POLL_MS=$pm timeout 300 python bench.py --workload cc26 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/cc26_p${pm}.json 2>$O/cc26_p${pm}.err
done
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], round(sum(k.values()),4), d['clocks']['samples'], d.get('step_ms_spread'), k.get('cc_partition'), k.get('rs5_refine'))"; done
