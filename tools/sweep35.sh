#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
for mb in 0 40 80 100; do for w in lr26 lr28; do SG_L2_PERSIST_MB=$mb timeout 200 python tools/probe_one.py $w 5; done; done
