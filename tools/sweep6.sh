#!/bin/bash
O=gpurun_out/sweep6.jsonl
: > $O
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu6.log 2>&1
tail -3 gpurun_out/pytest_gpu6.log
for w in lr26 lr28 lr26o; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep6.err; done
for wb in 19 20 21 22; do SG_RS_WBITS=$wb timeout 120 python tools/probe_one.py lr26 5 >> $O 2>>gpurun_out/sweep6.err; done
for wb in 21 22; do SG_RS_WBITS=$wb timeout 120 python tools/probe_one.py lr28 3 >> $O 2>>gpurun_out/sweep6.err; done
for k in 4 6; do SG_RS_KBITS0=$k timeout 120 python tools/probe_one.py lr28 3 >> $O 2>>gpurun_out/sweep6.err; done
SG_RS_KBITS=3 timeout 120 python tools/probe_one.py lr28 3 >> $O 2>>gpurun_out/sweep6.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rs_walk_rec -c 1 -o gpurun_out/prof_walkrec28b python tools/prof_target.py lr28 > /dev/null 2>&1
