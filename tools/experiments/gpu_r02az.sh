#!/bin/bash
# rs5_refine: 256-thread CTAs x 4 vs 512-thread CTAs x 2 (tile 2048 vs 4096)
TAG=${TAG:-r02az}
O=gpurun_out/$TAG
mkdir -p $O
for cfg in 256 512; do
  SG_NVCC_DEFS="-DRA_THREADS_CFG=$cfg" python -c "import __graft_entry__ as e; e.build()" > $O/build_$cfg.log 2>&1
  SG_NVCC_DEFS="-DRA_THREADS_CFG=$cfg" timeout 600 python -m pytest tests/test_listrank_gpu.py -q -x -k "refine or full or rs_rank" > $O/pytest_$cfg.log 2>&1
  for i in 1 2; do
    SG_NVCC_DEFS="-DRA_THREADS_CFG=$cfg" timeout 300 python bench.py --workload lr28 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/lr28_${cfg}_$i.json 2>$O/lr28_${cfg}_$i.err
  done
  SG_NVCC_DEFS="-DRA_THREADS_CFG=$cfg" timeout 300 python bench.py --workload lr26 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/lr26_${cfg}.json 2>$O/lr26_${cfg}.err
done
tail -n 1 $O/pytest_*.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d['step_ms_spread']['median'], k.get('rs5_refine'))"; done
