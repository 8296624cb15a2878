#!/bin/bash
O=gpurun_out/sweep19.jsonl
: > $O
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu19.log 2>&1
tail -15 gpurun_out/pytest_gpu19.log
for w in lr26o lr28o lr26 lr28; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep19.err; done
cat $O
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_rs_contract|k_rs_count0|k_rs_scan0" -c 4 -o gpurun_out/prof_contract28o_b python tools/prof_target.py lr28o > /dev/null 2>&1
ls gpurun_out
