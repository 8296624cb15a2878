#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
for it in 8 16; do for w in lr26 lr28; do SG_MS_ITEMS=$it timeout 200 python tools/probe_one.py $w 5; done; done
SG_MS_ITEMS=8 timeout 900 python -m pytest tests -x -q -m gpu -k "listrank" 2>&1 | tail -2
