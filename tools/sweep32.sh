#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "concomp or cc or components" 2>&1 | tail -2
for w in cc26 cc26:sv; do timeout 200 python tools/probe_one.py $w 5; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:"k_cc_part" -c 3 python tools/prof_target.py cc26 2>&1 | grep -E "k_cc_part|duration|dram" | head -12
