#!/bin/bash
O=gpurun_out/sweep4.jsonl
: > $O
./tools/ubench_random > gpurun_out/ubench.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu4.log 2>&1
tail -3 gpurun_out/pytest_gpu4.log
for w in lr26 lr26o lr28 lr28o cc26:uf; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep4.err; done
