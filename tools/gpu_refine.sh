#!/bin/bash
# refine experiment: parity of the counter-ranked refine, lr28/lr26 with both
# refines, one ncu --set full capture of each refine kernel, host conversion probe
TAG=${TAG:-r02c}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_listrank_gpu.py tests/test_fullsize_gpu.py -q -x > $O/pytest_list.log 2>&1
for v in 1 0; do
  for w in lr28 lr26; do
    SG_RS_REFINE_CNT=$v timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu --blocks none > $O/${w}_cnt$v.json 2>$O/${w}_cnt$v.err
  done
done
for v in 1 0; do
  SG_RS_REFINE_CNT=$v timeout 600 ncu --set full --import-source on --clock-control none -k regex:refine -s 2 -c 1 \
    -o $O/ncu_refine_cnt$v python bench.py --workload lr28 --steps 1 --warmup 3 --no-e2e --no-cpu --blocks none > $O/ncu_cnt$v.log 2>&1
done
timeout 120 ./tools/_ubench_l2 > $O/ubench_l2.txt 2>&1
timeout 300 python tools/probe_hostconv.py > $O/hostconv.txt 2>&1
tail -3 $O/pytest_list.log
