#!/bin/bash
# partition fast path; refine with shared atomics (SG_RS_REFINE=5); bench clocks in a child process
TAG=${TAG:-r02j}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_concomp_gpu.py tests/test_listrank_gpu.py -q -x > $O/pytest.log 2>&1
SG_RS_REFINE=5 timeout 900 python -m pytest tests/test_listrank_gpu.py -q -x > $O/pytest_ref5.log 2>&1
timeout 300 python bench.py --workload cc26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc26.json 2>$O/cc26.err
for v in 0 1 5; do
  SG_RS_REFINE=$v timeout 300 python bench.py --workload lr28 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr28_ref$v.json 2>$O/lr28_ref$v.err
done
SG_RS_REFINE=5 timeout 300 python bench.py --workload lr26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr26_ref5.json 2>$O/lr26_ref5.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'part_chunks' -s 0 -c 1 \
    -o $O/ncu_cc26_part python bench.py --workload cc26 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_cc.log 2>&1
SG_RS_REFINE=5 timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine -s 2 -c 1 \
    -o $O/ncu_refine_v5 python bench.py --workload lr28 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_refine_v5.log 2>&1
tail -2 $O/pytest.log $O/pytest_ref5.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], round(sum(k.values()),4), {a:b for a,b in k.items() if b>0.1}, d['clocks'])"; done
