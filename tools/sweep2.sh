#!/bin/bash
O=gpurun_out/sweep2.jsonl
: > $O
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu2.log 2>&1
tail -3 gpurun_out/pytest_gpu2.log
for w in lr26 lr26o lr28 cc22:uf cc22:sv cc26:uf cc26:sv; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep2.err; done
for k0 in 4 5 6; do for k1 in 3 4 5; do
  SG_RS_KBITS0=$k0 SG_RS_KBITS=$k1 timeout 120 python tools/probe_one.py lr26 5 >> $O 2>>gpurun_out/sweep2.err
done; done
for wb in 22 24 25 31; do SG_CC_WBITS=$wb timeout 120 python tools/probe_one.py cc26:uf 3 >> $O 2>>gpurun_out/sweep2.err; done
timeout 300 ncu --set full --clock-control none -k regex:k_rs_walk0 -c 1 -o gpurun_out/prof_walk0_26 python tools/prof_target.py lr26 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_cc_hook_uf -c 1 -o gpurun_out/prof_hookuf_part26 python tools/prof_target.py cc26 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_cc_part -c 3 -o gpurun_out/prof_part26 python tools/prof_target.py cc26 > /dev/null 2>&1
