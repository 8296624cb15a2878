#!/bin/bash
# refine: block-scan prefix + branch-free atomics
TAG=${TAG:-r02r}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_listrank_gpu.py tests/test_fullsize_gpu.py -q -x > $O/pytest.log 2>&1
timeout 300 python bench.py --workload lr28 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr28.json 2>$O/lr28.err
timeout 300 python bench.py --workload lr26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr26.json 2>$O/lr26.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine -s 2 -c 1 \
    -o $O/ncu_refine python bench.py --workload lr28 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_refine.log 2>&1
tail -n 3 $O/pytest.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], round(sum(k.values()),4), d.get('step_ms_spread'), k.get('rs5_refine'), k.get('rs5_scatter'))"; done
