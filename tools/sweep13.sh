#!/bin/bash
O=gpurun_out/sweep13.jsonl
: > $O
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu13.log 2>&1
tail -3 gpurun_out/pytest_gpu13.log
for w in lr26 lr28 cc26:uf; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep13.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rs_rec_part" -c 1 -o gpurun_out/prof_rec28f python tools/prof_target.py lr28 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_cc_hook_uf" -s 5 -c 1 -o gpurun_out/prof_hookuf5 python tools/prof_target.py cc26 > /dev/null 2>&1
