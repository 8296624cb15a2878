#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu27.log 2>&1
tail -3 gpurun_out/pytest_gpu27.log
for w in cc26 cc22 lr26 lr28o; do timeout 200 python tools/probe_one.py $w 5; done
