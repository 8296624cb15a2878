#!/bin/bash
# Round-2 measurement pass (final code): GPU suite, smoke, the default bench
# line (lr28 + lr28o/lr26/cc22/cc26 blocks), the reference arm (lr28, cc26),
# the ncu launch lists of lr28 and cc26 steps.  NCU=1: the ncu --set full
# captures instead (summarise here with tools/ncu_summary.py).
TAG=${TAG:-r02final7}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
if [ -z "$NCU" ]; then
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.log 2>&1
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference > $O/bench_ref_lr28.json 2> $O/bench_ref_lr28.err
timeout 900 python bench.py --impl reference --workload cc26 > $O/bench_ref_cc26.json 2> $O/bench_ref_cc26.err
timeout 300 python bench.py --workload cc26 --variant sv --no-cpu --no-e2e --blocks none > $O/bench_cc26sv.json 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload cc26 --no-cpu --no-e2e --blocks none > $O/bench_cc26_torchrun1.json 2> $O/bench_cc26_torchrun1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lr28.csv \
    python bench.py --workload lr28 --steps 3 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_launch_lr28.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cc26.csv \
    python bench.py --workload cc26 --steps 3 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_launch_cc26.log 2>&1
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
else
for spec in lr28:'k_rs_count0|k_rs_select|k_rs_walk_bin|k_rs_refine_atom|k_rs_rec_scatter':lr28:7 \
            cc26:'k_cc_part_chunks|k_cc_hook_uf|k_cc_compress':cc26:10 \
            lr28o:'k_rs_count0|k_rs_contract|k_rs_contract_expand':lr28o:4 cc22:'k_cc_hook_uf':cc22:1; do
  IFS=: read -r wl kern name cnt <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kern" -c $cnt -o $O/prof_$name \
      python tools/prof_target.py $wl > $O/ncu_$name.log 2>&1
  # summarise on the box (the reports together exceed gpurun's 64 MiB return limit)
  python tools/ncu_summary.py $O/prof_$name.ncu-rep $wl r02_ncu_$name >> $O/ncu_$name.log 2>&1
  cp profiles/r02_ncu_$name.txt $O/
  case $name in cc*) rm -f $O/prof_$name.ncu-rep ;; esac
done
cp profiles/traffic.json $O/traffic.json
fi
ls -la $O
