#!/bin/bash
./tools/ubench_random > gpurun_out/ubench2.txt 2>&1
for kk in chase chase_cg chase_na chase32 chase32_cg; do
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"^${kk}\$" -c 1 ./tools/ubench_random > gpurun_out/ncu_ub_$kk.txt 2>&1
done
for m in 0 1 3; do SG_WALK_LOAD=$m timeout 200 python tools/probe_one.py lr28 3 >> gpurun_out/sweep10.jsonl 2>>gpurun_out/sweep10.err; done
