#!/bin/bash
# census (k_rs_count0) grid: resident CTAs per SM (occupancy query) vs 8 per SM
TAG=${TAG:-r02bd}
O=gpurun_out/$TAG
mkdir -p $O
for cfg in occ grid8; do
  D=""; [ $cfg = grid8 ] && D="-DSG_COUNT0_GRID8"
  SG_NVCC_DEFS="$D" python -c "import __graft_entry__ as e; e.build()" > $O/build_$cfg.log 2>&1
  [ $cfg = occ ] && timeout 900 python -m pytest tests/test_listrank_gpu.py -q -x > $O/pytest_$cfg.log 2>&1
  for i in 1 2; do
    for wl in lr28 lr26 lr28o; do
      SG_NVCC_DEFS="$D" timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/${wl}_${cfg}_$i.json 2>$O/${wl}_${cfg}_$i.err
    done
  done
done
tail -n 1 $O/pytest_*.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d['step_ms_spread']['median'], k.get('rs1_validate'))"; done
