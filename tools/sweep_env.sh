#!/bin/bash
# env sweep on the GPU box: L2 fetch granularity x walk load mode
O=gpurun_out/sweep.jsonl
: > $O
for f in "" 32 64 128; do
  for wl in 0 1 3; do
    SG_DEBUG=1 SG_L2_FETCH=$f SG_WALK_LOAD=$wl timeout 120 python tools/probe_one.py lr26 >> $O 2>>gpurun_out/sweep.err
  done
  SG_DEBUG=1 SG_L2_FETCH=$f timeout 120 python tools/probe_one.py lr26o >> $O 2>>gpurun_out/sweep.err
  SG_L2_FETCH=$f timeout 120 python tools/probe_one.py cc26:uf 3 >> $O 2>>gpurun_out/sweep.err
  SG_L2_FETCH=$f timeout 120 python tools/probe_one.py cc26:sv 3 >> $O 2>>gpurun_out/sweep.err
  SG_L2_FETCH=$f timeout 120 python tools/probe_one.py wy26 2 >> $O 2>>gpurun_out/sweep.err
done
SG_L2_FETCH=32 timeout 300 ncu --set full --clock-control none -k regex:k_rs_walk -c 1 -o gpurun_out/prof_walk26_f32 python tools/prof_target.py lr26 > /dev/null 2>&1
SG_L2_FETCH=32 timeout 300 ncu --set full --clock-control none -k regex:k_cc_hook_uf -c 1 -o gpurun_out/prof_hookuf26_f32 python tools/prof_target.py cc26 > /dev/null 2>&1
