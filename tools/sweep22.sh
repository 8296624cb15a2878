#!/bin/bash
O=gpurun_out/sweep22.jsonl
: > $O
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu22.log 2>&1
tail -3 gpurun_out/pytest_gpu22.log
for pm in 0 1; do for w in lr26 lr28 cc26; do SG_MS_PEERS=$pm timeout 200 python tools/probe_one.py $w 5 >> $O 2>>gpurun_out/sweep22.err; done; done
cat $O
