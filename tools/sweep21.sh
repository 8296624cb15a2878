#!/bin/bash
O=gpurun_out/sweep21.jsonl
: > $O
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu21.log 2>&1
tail -5 gpurun_out/pytest_gpu21.log
for w in lr26 lr28 lr28o cc22 cc26 cc26:sv; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep21.err; done
cat $O
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_cc_part" -c 3 -o gpurun_out/prof_ccpart26 python tools/prof_target.py cc26 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_rs_rec_partition2|k_rs_rec_refine2|k_rs_rec_scatter" -c 3 -o gpurun_out/prof_ms2_28d python tools/prof_target.py lr28 > /dev/null 2>&1
