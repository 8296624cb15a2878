#!/bin/bash
# boundary copies: chunk size x cached / non-temporal staging stores
TAG=${TAG:-r02bc}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
lscpu | grep -E "L3|L2|Model name" > $O/cpu.txt
SG_XFER_NT_STAGE=0 SG_XFER_CHUNK_KI=256 timeout 600 python -m pytest tests/test_boundary_gpu.py -q -x > $O/pytest.log 2>&1
for i in 1 2; do
  for ki in 256 1024 4096; do
    for nt in 1 0; do
      SG_XFER_NT_STAGE=$nt SG_XFER_CHUNK_KI=$ki timeout 600 python tools/probe_e2e2.py > $O/e2e_k${ki}_nt${nt}_$i.txt 2>&1
    done
  done
done
tail -n 2 $O/pytest.log; cat $O/cpu.txt
for f in $O/e2e_*.txt; do echo "== $f"; grep -E 'narrowed \(pinned|widened|e2e rs_rank\(pinned' $f | tr '\n' ' '; echo; done
