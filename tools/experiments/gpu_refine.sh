#!/bin/bash
# refine experiment: parity of every refine variant, lr28/lr26 per variant,
# ncu --set full of the default refine
TAG=${TAG:-r02d}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_listrank_gpu.py tests/test_concomp_gpu.py tests/test_contract_gpu.py tests/test_abi.py -q -x > $O/pytest_sel.log 2>&1
for v in 0 1 2 3; do
  for w in lr28 lr26; do
    SG_RS_REFINE=$v timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/${w}_ref$v.json 2>$O/${w}_ref$v.err
  done
done
SG_RS_REFINE=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine -s 2 -c 1 \
    -o $O/ncu_refine_lean python bench.py --workload lr28 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_lean.log 2>&1
tail -3 $O/pytest_sel.log
for f in $O/lr2*_ref*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], 'refine', k.get('rs5_refine'))"; done
