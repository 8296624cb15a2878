#!/bin/bash
# UF hook: hook a root larger endpoint straight under the other endpoint's parent
TAG=${TAG:-r02au}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_concomp_gpu.py tests/test_dist_gpu.py tests/test_multi_gpu.py tests/test_fullsize_gpu.py -q -x > $O/pytest.log 2>&1
for i in 1 2; do
for w in cc26 cc22; do
  timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/${w}_$i.json 2>$O/${w}_$i.err
done
done
tail -n 2 $O/pytest.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d.get('step_ms_spread',{}).get('median'), k)"; done
