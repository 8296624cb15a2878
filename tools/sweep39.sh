#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
for kb in 2 3; do for fin in 4096 8192 32768; do SG_RS_KBITS=$kb SG_RS_FINAL=$fin timeout 200 python tools/probe_one.py lr28 5; done; done
