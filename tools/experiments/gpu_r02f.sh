#!/bin/bash
TAG=${TAG:-r02f}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
SG_RS_REFINE=4 timeout 900 python -m pytest tests/test_listrank_gpu.py tests/test_fullsize_gpu.py -q -x > $O/pytest_tiles.log 2>&1
for v in 0 4; do
  for w in lr28 lr26; do
    SG_RS_REFINE=$v timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/${w}_ref$v.json 2>$O/${w}_ref$v.err
  done
done
timeout 600 python tools/probe_e2e2.py > $O/e2e_phases.txt 2>&1
SG_XFER_THREADS=8 timeout 600 python tools/probe_e2e2.py > $O/e2e_phases_t8.txt 2>&1
tail -3 $O/pytest_tiles.log
for f in $O/lr2*_ref*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], 'refine', k.get('rs5_refine'), 'scatter', k.get('rs5_scatter'))"; done
cat $O/e2e_phases.txt $O/e2e_phases_t8.txt
