#!/bin/bash
TAG=${TAG:-r02ad}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_listrank_gpu.py tests/test_host_api.py tests/test_contract_gpu.py -q -x > $O/pytest.log 2>&1
python tools/probe_host_split.py lr26 30 > $O/split.txt 2>&1; python tools/probe_host_split.py lr28 20 >> $O/split.txt 2>&1
timeout 300 python bench.py --workload lr28 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/lr28.json 2>$O/lr28.err
timeout 300 python bench.py --workload lr26 --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/lr26.json 2>$O/lr26.err
tail -n 2 $O/pytest.log; cat $O/split.txt
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], d.get('step_ms_spread',{}).get('median'), round(sum(k.values()),4), k.get('rs5_refine'))"; done
