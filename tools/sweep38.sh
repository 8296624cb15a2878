#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
for cb in 256 128 64; do for w in lr26 lr28; do SG_RS_CBINS=$cb timeout 200 python tools/probe_one.py $w 5; done; done
