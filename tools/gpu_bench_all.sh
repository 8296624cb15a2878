#!/bin/bash
# Full measurement pass: every bench workload, the reference arm, the ncu
# launch list of the default bench command and one `ncu --set full` capture
# per dominant kernel.  Output: gpurun_out/$TAG (summarise with tools/ncu_summary.py).
TAG=${TAG:-r01}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
if [ -z "$ONLY_NCU" ]; then
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench_lr26.json 2> $O/bench_lr26.err
for w in lr28 lr28o cc22 cc26; do timeout 600 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 300 python bench.py --workload cc26 --variant sv --no-cpu --no-e2e > $O/bench_cc26sv.json 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref_lr26.json 2>&1
timeout 300 python bench.py --impl reference --workload cc26 --steps 3 --warmup 3 > $O/bench_ref_cc26.json 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload cc26 --no-cpu --no-e2e > $O/bench_cc26_torchrun1.json 2> $O/bench_cc26_torchrun1.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lr26.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary > $O/ncu_launch_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cc26.csv \
    python bench.py --workload cc26 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch_cc.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lr28o.csv \
    python bench.py --workload lr28o --steps 3 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch_lr28o.log 2>&1
fi
# ncu captures: a separate call per batch (gpurun_out is capped at 64 MiB)
if [ -n "$NCU_BATCH" ]; then
  for spec in $NCU_BATCH; do
    IFS=: read -r wl kern name cnt <<< "$spec"
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kern" -c $cnt -o $O/prof_$name \
        python tools/prof_target.py $wl > $O/ncu_$name.log 2>&1
  done
fi
ls $O
