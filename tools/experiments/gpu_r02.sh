#!/bin/bash
# Round-2 GPU pass: build, GPU tests (incl. full-size digests), smoke, the
# default bench line (lr28 + blocks) and the reference arm, as the driver runs them.
TAG=${TAG:-r02a}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > $O/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.log 2>&1
fi
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
if [ -z "$NO_REF" ]; then
( time timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > $O/bench_ref.json 2> $O/bench_ref.err
fi
tail -n 5 $O/pytest_gpu.log $O/smoke.log $O/bench.err $O/bench_ref.err 2>/dev/null
