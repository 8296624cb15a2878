#!/bin/bash
# tile contraction: parity + timing
O=gpurun_out/sweep18.jsonl
: > $O
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu18.log 2>&1
tail -15 gpurun_out/pytest_gpu18.log
for w in lr26o lr28o lr26 lr28; do timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep18.err; done
cat $O
