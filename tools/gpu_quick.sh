#!/bin/bash
# Quick GPU pass: build, gpu tests, smoke, every bench workload (no ncu).
O=gpurun_out/q
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_lr26.json 2> $O/bench_lr26.err
for w in lr28 lr28o cc22 cc26 wy26; do timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_lr26.json 2>&1
tail -n 3 $O/*.log $O/*.json
