#!/bin/bash
# census flags run tiles; the contraction skips them, the expand recomputes their words
TAG=${TAG:-r02bm}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_listrank_gpu.py tests/test_cli.py tests/test_boundary_gpu.py -m gpu -q -x > $O/pytest.log 2>&1
timeout 600 compute-sanitizer --tool memcheck --kernel-name kns=sg:: python tools/sanitize_driver.py list > $O/memcheck_list.txt 2>&1
timeout 600 compute-sanitizer --tool initcheck python tools/sanitize_driver.py list > $O/initcheck_list.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --kernel-name kns=sg:: python tools/sanitize_driver.py list > $O/racecheck_list.txt 2>&1
for i in 1 2; do
  for wl in lr28o lr28 lr26; do
    timeout 300 python bench.py --workload $wl --steps 20 --warmup 5 --no-e2e --no-cpu --blocks none > $O/${wl}_$i.json 2>$O/${wl}_$i.err
  done
done
tail -n 2 $O/pytest.log; tail -n 1 $O/memcheck_list.txt $O/initcheck_list.txt $O/racecheck_list.txt
for f in $O/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); k=d['kernels_ms_per_step']; print('$f', d['ms_per_step'], k.get('rs1_validate'), k.get('rs3_contract'), k.get('rs5_expand'))"; done
