#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
for pm in 2 1 0; do for w in lr28 cc26; do SG_MS_PEERS=$pm timeout 200 python tools/probe_one.py $w 5; done; done
