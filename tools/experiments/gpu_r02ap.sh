#!/bin/bash
# upper ruling-set levels: ruler density above level 0 and the pointer-jumping threshold
TAG=${TAG:-r02ap}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
run() { env $1 timeout 300 python bench.py --workload $2 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/$3.json 2>$O/$3.err; }
run "SG_RS_KBITS=3" lr28 k3_def
run "SG_RS_KBITS=3 SG_RS_TOPN=1048576" lr28 k3_t20
run "SG_RS_KBITS=4" lr28 k4_def
run "SG_RS_KBITS=4 SG_RS_TOPN=1048576" lr28 k4_t20
run "SG_RS_KBITS=2" lr28 k2_def
run "SG_RS_KBITS=3 SG_RS_TOPN=1048576" lr26 k3_t20_26
run "SG_RS_KBITS=3" lr26 k3_def_26
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d['step_ms_spread']['median'], round(sum(k.values()),4), {a:k[a] for a in ('rs4_walk','rs4_rank','rs4_expand','rs4_select','rs4_count')}, d['ruling_set']['level_size'])"; done
