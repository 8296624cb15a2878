#!/bin/bash
# Profiling pass on the GPU box (one GPU): launch list of the bench command,
# then one `ncu --set full` capture per hot kernel.  Output: gpurun_out/.
set -x
O=gpurun_out
python -c "import __graft_entry__ as e; e.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_lr26.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-secondary > $O/ncu_launch_bench.log 2>&1
for spec in "lr26:k_rs_walk:walk26" "lr26:k_rs_expand0:expand26" "lr26:k_rs_count:count26" "lr28:k_rs_walk:walk28" \
            "cc26:k_cc_hook_uf:hookuf26" "cc26 sv:k_cc_hook_sv:hooksv26" "wy26:k_wy_jump:wyjump26"; do
  IFS=: read -r wl kern name <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$kern -c 1 -o $O/prof_$name \
      python tools/prof_target.py $wl > $O/ncu_$name.log 2>&1
done
