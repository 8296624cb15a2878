#!/bin/bash
TAG=${TAG:-r02p}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
SG_HOST_TIMING=1 timeout 300 python tools/probe_steps.py lr26 40 > $O/steps_lr26.txt 2> $O/steps_lr26_host.txt
timeout 300 python tools/probe_steps.py lr26 40 > $O/steps_lr26_b.txt 2>&1
cat $O/steps_lr26.txt $O/steps_lr26_b.txt
