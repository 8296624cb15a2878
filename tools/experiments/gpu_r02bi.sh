#!/bin/bash
# e2e after the GPU test suite (the driver's order: pytest, smoke, bench)
TAG=${TAG:-r02bi}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 600 python bench.py --no-cpu --blocks none > $O/bench_before.json 2> $O/bench_before.err
(free -m; cat /proc/meminfo | grep -E "Huge|Dirty|Writeback|Mlocked|Unevict|Cached") > $O/mem_before.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
(free -m; cat /proc/meminfo | grep -E "Huge|Dirty|Writeback|Mlocked|Unevict|Cached") > $O/mem_after.txt
for i in 1 2; do
  timeout 600 python bench.py --no-cpu --blocks none > $O/bench_after_$i.json 2> $O/bench_after_$i.err
  timeout 600 python tools/probe_e2e2.py > $O/e2e_probe_$i.txt 2>&1
done
tail -1 $O/pytest_gpu.log
paste $O/mem_before.txt $O/mem_after.txt
for f in $O/e2e_probe*.txt; do echo "== $f"; grep -E 'narrowed \(pinned|widened|e2e rs_rank\(pinned' $f | tr '\n' ' '; echo; done
for f in $O/bench*.json; do echo "$f $(python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['e2e']['ms_per_step'])")"; done
