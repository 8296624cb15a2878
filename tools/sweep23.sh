#!/bin/bash
O=gpurun_out/sweep23.jsonl
: > $O
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu23.log 2>&1
tail -3 gpurun_out/pytest_gpu23.log
for w in lr26o lr28o lr26 lr28; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep23.err; done
cat $O
./tools/ubench_random > gpurun_out/ubench_default.txt 2>&1
UB_FETCH=32 ./tools/ubench_random > gpurun_out/ubench_fetch32.txt 2>&1
UB_FETCH=64 ./tools/ubench_random > gpurun_out/ubench_fetch64.txt 2>&1
for f in "" 32; do
  UB_FETCH=$f timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:"chase32_cg|chase32" -c 2 ./tools/ubench_random > gpurun_out/ncu_ub_fetch$f.txt 2>&1
done
