#!/bin/bash
O=gpurun_out/sweep14.jsonl
: > $O
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu14.log 2>&1
tail -3 gpurun_out/pytest_gpu14.log
for w in lr26 lr28 cc26:uf; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep14.err; done
