#!/bin/bash
# CC window size sweep at C5 / C4 (SG_CC_WBITS: 2^w vertices per hook window)
TAG=${TAG:-r02bj}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
for i in 1 2; do
  for w in 21 22 23 24; do
    SG_CC_WBITS=$w timeout 300 python bench.py --workload cc26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc26_w${w}_$i.json 2>$O/cc26_w${w}_$i.err
  done
done
for w in 19 20 21 22; do
  SG_CC_WBITS=$w timeout 300 python bench.py --workload cc22 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc22_w${w}.json 2>$O/cc22_w${w}.err
done
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], {a: round(b,3) for a,b in k.items()})"; done
