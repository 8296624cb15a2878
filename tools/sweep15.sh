#!/bin/bash
timeout 300 python tools/probe_sort.py > gpurun_out/probe_sort.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu15.log 2>&1
tail -3 gpurun_out/pytest_gpu15.log
timeout 200 python tools/probe_one.py cc26:uf 5 >> gpurun_out/sweep15.jsonl 2>>gpurun_out/sweep15.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rs_rec_refine" -c 1 -o gpurun_out/prof_refine28 python tools/prof_target.py lr28 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sort.csv python tools/probe_sort.py > /dev/null 2>&1
