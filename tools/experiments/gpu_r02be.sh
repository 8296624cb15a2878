#!/bin/bash
# census (k_rs_count0): branch-free full-tile path vs the exact per-node path only
TAG=${TAG:-r02be}
O=gpurun_out/$TAG
mkdir -p $O
for cfg in fast exact; do
  D=""; [ $cfg = exact ] && D="-DSG_COUNT0_EXACT_ONLY"
  SG_NVCC_DEFS="$D" python -c "import __graft_entry__ as e; e.build()" > $O/build_$cfg.log 2>&1
  [ $cfg = fast ] && timeout 900 python -m pytest tests/test_listrank_gpu.py -q -x > $O/pytest_$cfg.log 2>&1
  SG_NVCC_DEFS="$D" timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:k_rs_count0 -c 1 python tools/prof_target.py lr28 > $O/ncu_$cfg.txt 2>&1
  for i in 1 2; do
    for wl in lr28 lr26 lr28o; do
      SG_NVCC_DEFS="$D" timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/${wl}_${cfg}_$i.json 2>$O/${wl}_${cfg}_$i.err
    done
  done
done
tail -n 1 $O/pytest_*.log
grep -E 'duration|dram__|issue_active|inst_executed|warps_active' $O/ncu_*.txt
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d['step_ms_spread']['median'], k.get('rs1_validate'))"; done
