#!/bin/bash
# CC partition rows in flight; window size
TAG=${TAG:-r02aa}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
SG_CC_PG=3 timeout 600 python -m pytest tests/test_concomp_gpu.py -q -x -k partitioned > $O/pytest_pg3.log 2>&1
for pg in 2 3; do
  SG_CC_PG=$pg timeout 300 python bench.py --workload cc26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc26_pg$pg.json 2>$O/cc26_pg$pg.err
done
for wb in 22 24; do
  SG_CC_WBITS=$wb timeout 300 python bench.py --workload cc26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc26_wb$wb.json 2>$O/cc26_wb$wb.err
done
tail -n 2 $O/pytest_pg3.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d.get('step_ms_spread',{}).get('median'), {a:b for a,b in k.items() if b>0.1})"; done
