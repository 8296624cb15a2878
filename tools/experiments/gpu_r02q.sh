#!/bin/bash
# refine: flat write-out (0) vs warp-autonomous (7)
TAG=${TAG:-r02q}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_listrank_gpu.py -q -x -k "refine or full or rs_rank" > $O/pytest.log 2>&1
for v in 0 7; do
  SG_RS_REFINE=$v timeout 300 python bench.py --workload lr28 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr28_r$v.json 2>$O/lr28_r$v.err
  SG_RS_REFINE=$v timeout 300 python bench.py --workload lr26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr26_r$v.json 2>$O/lr26_r$v.err
done
for v in 0 7; do
SG_RS_REFINE=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine -s 2 -c 1 \
    -o $O/ncu_refine_r$v python bench.py --workload lr28 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_refine_r$v.log 2>&1
done
tail -n 3 $O/pytest.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], round(sum(k.values()),4), d.get('step_ms_spread'), k.get('rs5_refine'), k.get('rs5_scatter'))"; done
