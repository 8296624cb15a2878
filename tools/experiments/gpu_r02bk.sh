#!/bin/bash
# CC: shortcut each window's slice of D right after its hook (SG_CC_WCOMP=1) vs not
TAG=${TAG:-r02bk}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
SG_CC_WCOMP=1 timeout 600 python -m pytest tests/test_concomp_gpu.py -q -x > $O/pytest.log 2>&1
for i in 1 2; do
  for c in 0 1; do
    SG_CC_WCOMP=$c timeout 300 python bench.py --workload cc26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc26_c${c}_$i.json 2>$O/cc26_c${c}_$i.err
  done
done
tail -1 $O/pytest.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], {a: round(b,3) for a,b in k.items()})"; done
