#!/bin/bash
# CC_HOOK_HU sweep (pass x13): one build per value through SG_NVCC_DEFS
O=gpurun_out/x13; mkdir -p $O
for hu in 2 1 3 4 2; do
  SG_NVCC_DEFS="-DCC_HOOK_HU=$hu" python -c "import __graft_entry__ as e; e.build()" > $O/build_$hu.log 2>&1
  for wl in cc26 cc22; do
    timeout 300 python bench.py --workload $wl --no-cpu --no-e2e --blocks none > $O/b_${hu}_$wl.json 2>&1
    python -c "import json; d=json.loads(open('$O/b_${hu}_$wl.json').read().strip().splitlines()[-1]); print('HU=$hu', '$wl', d['ms_per_step'], d['kernels_ms_per_step'].get('cc_hook_uf'))"
  done
done
