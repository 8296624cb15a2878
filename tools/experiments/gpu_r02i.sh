#!/bin/bash
# CC direct chunk partition; host overhead probe of lr28
TAG=${TAG:-r02i}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_concomp_gpu.py tests/test_dist_gpu.py -q -x > $O/pytest_cc.log 2>&1
for part in chunks count; do
  SG_CC_PART=$part timeout 300 python bench.py --workload cc26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc26_$part.json 2>$O/cc26_$part.err
done
timeout 300 python bench.py --workload cc22 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc22.json 2>$O/cc22.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'part_chunks' -s 0 -c 1 \
    -o $O/ncu_cc26_part python bench.py --workload cc26 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_cc.log 2>&1
timeout 300 python tools/probe_overhead.py lr28 > $O/overhead_lr28.txt 2>&1
SG_HOST_TIMING=1 timeout 300 python tools/probe_overhead.py lr28 > $O/overhead_lr28_host.txt 2>&1
tail -3 $O/pytest_cc.log
for f in $O/cc*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], k)"; done
cat $O/overhead_lr28.txt
