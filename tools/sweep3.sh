#!/bin/bash
O=gpurun_out/sweep3.jsonl
: > $O
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu3.log 2>&1
tail -3 gpurun_out/pytest_gpu3.log
for w in lr26 lr26o lr28 cc22:uf cc22:sv cc26:uf cc26:sv; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep3.err; done
for wb in 22 24; do SG_CC_WBITS=$wb timeout 120 python tools/probe_one.py cc26:uf 3 >> $O 2>>gpurun_out/sweep3.err; SG_CC_WBITS=$wb timeout 120 python tools/probe_one.py cc26:sv 3 >> $O 2>>gpurun_out/sweep3.err; done
timeout 300 ncu --set full --clock-control none -k regex:k_rs_walk0 -c 1 -o gpurun_out/prof_walk0b_26 python tools/prof_target.py lr26 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"k_cc_hook_uf|k_cc_part|k_scan" -c 12 -o gpurun_out/prof_cc26b python tools/prof_target.py cc26 > /dev/null 2>&1
