#!/bin/bash
# boundary transfers: AVX-512 vs SSE2 conversions
TAG=${TAG:-r02ay}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_boundary_gpu.py -q -x > $O/pytest.log 2>&1
SG_XFER_NO_AVX512=1 timeout 600 python -m pytest tests/test_boundary_gpu.py -q -x > $O/pytest_sse.log 2>&1
for i in 1 2 3; do
  timeout 600 python tools/probe_e2e2.py > $O/e2e_avx_$i.txt 2>&1
  SG_XFER_NO_AVX512=1 timeout 600 python tools/probe_e2e2.py > $O/e2e_sse_$i.txt 2>&1
done
tail -n 2 $O/pytest.log $O/pytest_sse.log
for f in $O/e2e_*.txt; do echo "== $f"; grep -E 'narrowed \(pinned|widened|e2e rs_rank\(pinned' $f | tr '\n' ' '; echo; done
