#!/bin/bash
TAG=${TAG:-r02v}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
for f in 5 6; do
  SG_RS_SCATTER_FUSE=$f timeout 300 python bench.py --workload lr26 --steps 5 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr26_f$f.json 2>$O/lr26_f$f.err
done
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], k.get('rs5_refine'), k.get('rs5_scatter'))"; done
tail -3 $O/*.err
