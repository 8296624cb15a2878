#!/bin/bash
TAG=${TAG:-r02ar}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
run() { env $1 timeout 300 python bench.py --workload $2 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/$3.json 2>$O/$3.err; }
run "SG_RS_KBITS=4" lr28 d
run "SG_RS_KBITS=5" lr28 k5
run "SG_RS_KBITS=5 SG_RS_TOPN=524288" lr28 k5t19
run "SG_RS_KBITS=4 SG_RS_TOPN=2097152" lr28 k4t21
run "SG_RS_KBITS0=6" lr28 k06
run "SG_RS_KBITS0=4" lr28 k04
run "SG_RS_KBITS=4" lr28 d2
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d['step_ms_spread']['median'], round(sum(k.values()),4), {a:k.get(a) for a in ('rs3_walk','rs4_walk','rs4_rank','rs5_refine')}, d['ruling_set']['level_size'])"; done
