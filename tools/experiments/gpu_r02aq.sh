#!/bin/bash
TAG=${TAG:-r02aq}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
run() { env $1 timeout 300 python bench.py --workload $2 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/$3.json 2>$O/$3.err; }
for i in 1 2; do
run "SG_RS_KBITS=3" lr28 k3_$i
run "SG_RS_KBITS=4 SG_RS_TOPN=1048576" lr28 k4t20_$i
run "SG_RS_KBITS=3" lr26 k3_26_$i
run "SG_RS_KBITS=4 SG_RS_TOPN=1048576" lr26 k4t20_26_$i
done
run "SG_RS_KBITS=4 SG_RS_TOPN=1048576" lr28o k4t20_28o
run "SG_RS_KBITS=3" lr28o k3_28o
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d['step_ms_spread']['median'], round(sum(k.values()),4), d['ruling_set']['level_size'])"; done
