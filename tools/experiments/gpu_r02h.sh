#!/bin/bash
# CC chunk-list partition vs count + scatter; ncu of the partition and of rs5_refine (v0 lean, v1 ms_split_fn)
TAG=${TAG:-r02h}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_concomp_gpu.py tests/test_dist_gpu.py -q -x > $O/pytest_cc.log 2>&1
for part in chunks count; do
  for w in cc26 cc22; do
    SG_CC_PART=$part timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/${w}_$part.json 2>$O/${w}_$part.err
  done
done
SG_CC_PART=chunks timeout 300 python bench.py --workload cc26 --variant sv --steps 5 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc26sv_chunks.json 2>$O/cc26sv_chunks.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'part_chunks|hook_uf' -s 0 -c 9 \
    -o $O/ncu_cc26_chunks python bench.py --workload cc26 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_cc.log 2>&1
for v in 0 1; do
SG_RS_REFINE=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine -s 2 -c 1 \
    -o $O/ncu_refine_v$v python bench.py --workload lr28 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_refine_v$v.log 2>&1
done
tail -3 $O/pytest_cc.log
for f in $O/cc*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], k)"; done
