#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
for kb in 32 64 128; do for w in lr26 lr28; do SG_RS_WIN_KB=$kb timeout 200 python tools/probe_one.py $w 5; done; done
SG_RS_WIN_KB=64 timeout 900 python -m pytest tests -x -q -m gpu -k "listrank" 2>&1 | tail -1
