#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
for k0 in 4 6 7; do for w in lr26 lr28; do SG_RS_KBITS0=$k0 timeout 200 python tools/probe_one.py $w 5; done; done
