#!/bin/bash
# pipelined refine atom; chunk partition match.any vs ballots; per-step spread
TAG=${TAG:-r02l}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_concomp_gpu.py tests/test_listrank_gpu.py tests/test_boundary_gpu.py -q -x > $O/pytest.log 2>&1
SG_CC_RANK=ballot timeout 600 python -m pytest tests/test_concomp_gpu.py -q -x -k partitioned > $O/pytest_ballot.log 2>&1
for r in match ballot; do
  SG_CC_RANK=$r timeout 300 python bench.py --workload cc26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/cc26_$r.json 2>$O/cc26_$r.err
done
for i in 1 2; do
timeout 300 python bench.py --workload lr28 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr28_$i.json 2>$O/lr28_$i.err
done
timeout 300 python bench.py --workload lr26 --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/lr26.json 2>$O/lr26.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:'part_chunks' -s 0 -c 1 \
    -o $O/ncu_cc26_part python bench.py --workload cc26 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_cc.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine -s 2 -c 1 \
    -o $O/ncu_refine_atom python bench.py --workload lr28 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_refine.log 2>&1
tail -n 3 $O/pytest.log $O/pytest_ballot.log
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], round(sum(k.values()),4), {a:b for a,b in k.items() if b>0.1}, d['clocks']['samples'], d.get('step_ms_spread'))"; done
