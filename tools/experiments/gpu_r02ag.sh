#!/bin/bash
# boundary transfers: direct int64 lane share
TAG=${TAG:-r02ag}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_boundary_gpu.py tests/test_listrank_gpu.py -q -x -k "boundary or narrow or widen or api" > $O/pytest.log 2>&1
for d in 0 1 2 3 4; do
  SG_XFER_DIRECT=$d timeout 600 python tools/probe_e2e2.py > $O/e2e_d$d.txt 2>&1
done
for d in 0 2 3; do
  SG_XFER_DIRECT=$d timeout 600 python bench.py --workload lr28 --steps 5 --warmup 3 --no-cpu --blocks none > $O/lr28_d$d.json 2>$O/lr28_d$d.err
done
tail -n 2 $O/pytest.log
for d in 0 1 2 3 4; do echo "== direct $d"; cat $O/e2e_d$d.txt; done
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['e2e'])"; done
