#!/bin/bash
O=gpurun_out/sweep12.jsonl
: > $O
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu12.log 2>&1
tail -3 gpurun_out/pytest_gpu12.log
for w in lr26 lr28 lr26o cc26:uf cc26:sv cc22:uf; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep12.err; done
timeout 120 python tools/probe_host.py 26 > gpurun_out/probe_host26b.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rs_rec" -c 3 -o gpurun_out/prof_rec28e python tools/prof_target.py lr28 > /dev/null 2>&1
