#!/bin/bash
O=gpurun_out/sweep16.jsonl
: > $O
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu16.log 2>&1
tail -3 gpurun_out/pytest_gpu16.log
for w in lr26 lr28 lr26o; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep16.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rs_walk_stage|k_rs_rec_refine_st" -c 2 -o gpurun_out/prof_stage28 python tools/prof_target.py lr28 > /dev/null 2>&1
