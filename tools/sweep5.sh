#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu5.log 2>&1
tail -3 $O/pytest_gpu5.log
timeout 120 python tools/probe_host.py 26 > $O/probe_host26.txt 2>&1
for spec in "lr26:k_rs_walk_rec:walkrec26" "lr28:k_rs_walk_rec:walkrec28" "lr26:k_rs_rec_scatter:recscatter26" "lr26:k_rs_rec_partition:recpart26" "lr28:k_rs_rec_scatter:recscatter28"; do
  IFS=: read -r wl kern name <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 -o $O/prof_$name \
      python tools/prof_target.py $wl > $O/ncu_$name.log 2>&1
done
