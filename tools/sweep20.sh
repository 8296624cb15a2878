#!/bin/bash
O=gpurun_out/sweep20.jsonl
: > $O
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu20.log 2>&1
tail -5 gpurun_out/pytest_gpu20.log
for w in lr26 lr28 cc26; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep20.err; done
for w in lr26 lr28; do SG_RS_MS=1 timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep20.err; done
cat $O
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_rs_rec_partition2|k_rs_rec_refine2" -c 2 -o gpurun_out/prof_ms2_28c python tools/prof_target.py lr28 > /dev/null 2>&1
