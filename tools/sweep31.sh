#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for t in 1 0; do SG_CC_TILESORT=$t timeout 200 python tools/probe_one.py cc26 5; SG_CC_TILESORT=$t timeout 200 python tools/probe_one.py cc26:sv 3; done
