#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu24.log 2>&1
tail -3 gpurun_out/pytest_gpu24.log
python tools/probe_pin.py
python tools/probe_overhead.py lr26
for kb in 3 4; do SG_RS_KBITS=$kb timeout 200 python tools/probe_one.py lr26 5; SG_RS_KBITS=$kb timeout 200 python tools/probe_one.py lr28 3; done
timeout 200 python tools/probe_one.py lr26 5; timeout 200 python tools/probe_one.py lr28 3
