#!/bin/bash
# L2 window scatter vs refine+smem scatter; coarse window size sweep
O=gpurun_out/sweep17.jsonl
: > $O
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
SG_RS_SCATTER=1 timeout 600 python -m pytest tests -x -q -m gpu -k "listrank" > gpurun_out/pytest_gpu17.log 2>&1
tail -3 gpurun_out/pytest_gpu17.log
for w in lr26 lr28; do
  timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep17.err
  for c in 18 19 20 21 22 23; do SG_RS_SCATTER=1 SG_RS_CSHIFT=$c timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep17.err; done
done
cat $O
