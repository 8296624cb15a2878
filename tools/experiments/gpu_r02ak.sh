#!/bin/bash
# UF hook: lockstep path-splitting finds vs serial halving
TAG=${TAG:-r02ak}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_concomp_gpu.py tests/test_dist_gpu.py -q -x > $O/pytest.log 2>&1
SG_CC_FIND_SERIAL=1 timeout 900 python -m pytest tests/test_concomp_gpu.py -q -x > $O/pytest_serial.log 2>&1
for fs in 0 1; do
for w in cc26 cc22; do
  SG_CC_FIND_SERIAL=$fs timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/${w}_s$fs.json 2>$O/${w}_s$fs.err
done
done
tail -n 2 $O/pytest.log $O/pytest_serial.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d.get('step_ms_spread',{}).get('median'), k)"; done
