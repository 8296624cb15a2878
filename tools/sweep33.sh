#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for pk in 1 0; do for w in lr26 lr28; do SG_RS_PACKED=$pk timeout 200 python tools/probe_one.py $w 5; done; done
