#!/bin/bash
# boundary transfers: chunk size
TAG=${TAG:-r02aw}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_boundary_gpu.py -q -x > $O/pytest.log 2>&1
for i in 1 2; do
for c in 4 1 2 8; do
  SG_XFER_CHUNK_MI=$c timeout 600 python tools/probe_e2e2.py > $O/e2e_c${c}_$i.txt 2>&1
done
done
tail -n 2 $O/pytest.log
for f in $O/e2e_*.txt; do echo "== $f"; grep -E 'narrowed \(pinned|widened|e2e rs_rank\(pinned' $f | tr '\n' ' '; echo; done
