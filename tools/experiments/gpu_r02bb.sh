#!/bin/bash
# boundary narrowing: software prefetch distance (SG_XFER_PF, ids; 0 = off)
TAG=${TAG:-r02bb}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
cat /sys/fs/cgroup/cpu.max > $O/cgroup.txt 2>&1; lscpu >> $O/cgroup.txt 2>&1
SG_XFER_PF=512 timeout 600 python -m pytest tests/test_boundary_gpu.py -q -x > $O/pytest_pf.log 2>&1
for i in 1 2; do
  for pf in 0 256 1024 4096; do
    SG_XFER_PF=$pf timeout 600 python tools/probe_e2e2.py > $O/e2e_pf${pf}_$i.txt 2>&1
  done
done
tail -n 2 $O/pytest_pf.log; grep -E "Thread|Core|Socket|NUMA node\(|Model name" $O/cgroup.txt; head -1 $O/cgroup.txt
for f in $O/e2e_*.txt; do echo "== $f"; grep -E 'narrowed \(pinned|widened|e2e rs_rank\(pinned' $f | tr '\n' ' '; echo; done
