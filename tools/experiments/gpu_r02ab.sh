#!/bin/bash
TAG=${TAG:-r02ao}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_listrank_gpu.py tests/test_fullsize_gpu.py -q -x > $O/pytest.log 2>&1
for i in 1 2; do
timeout 300 python bench.py --workload lr28 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/lr28_$i.json 2>$O/lr28_$i.err
done
timeout 300 python bench.py --workload lr26 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/lr26.json 2>$O/lr26.err
tail -n 2 $O/pytest.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d.get('step_ms_spread',{}).get('median'), round(sum(k.values()),4), k.get('rs5_refine'))"; done
