#!/bin/bash
# CC partition launch shape sweep (pass x14): CTAs per SM x 16-B row groups per lane
O=gpurun_out/x14; mkdir -p $O
for cfg in 5:4 6:4 4:4 5:3 6:3 5:4; do
  IFS=: read -r c g <<< "$cfg"
  SG_NVCC_DEFS="-DCC_PD_CTAS=$c -DCC_PD_G16=$g" python -c "import __graft_entry__ as e; e.build()" > $O/build_${c}_$g.log 2>&1
  timeout 300 python bench.py --workload cc26 --no-cpu --no-e2e --blocks none > $O/b_${c}_$g.json 2>&1
  python -c "import json; d=json.loads(open('$O/b_${c}_$g.json').read().strip().splitlines()[-1]); print('ctas=$c g=$g', d['ms_per_step'], d['kernels_ms_per_step'].get('cc_partition'))" 2>&1 | tail -1
done
