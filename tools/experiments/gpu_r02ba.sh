#!/bin/bash
# e2e variance: probe vs bench on the same box, spin pool on/off, thread counts
TAG=${TAG:-r02ba}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
nproc > $O/nproc.txt; cat /proc/cpuinfo | grep "model name" | head -1 >> $O/nproc.txt; free -g >> $O/nproc.txt
for i in 1 2; do
  timeout 600 python tools/probe_e2e2.py > $O/e2e_probe_$i.txt 2>&1
  SG_XFER_SPIN=0 timeout 600 python tools/probe_e2e2.py > $O/e2e_probe_nospin_$i.txt 2>&1
  timeout 600 python bench.py --no-cpu --blocks none > $O/bench_$i.json 2> $O/bench_$i.err
  SG_XFER_SPIN=0 timeout 600 python bench.py --no-cpu --blocks none > $O/bench_nospin_$i.json 2> $O/bench_nospin_$i.err
  SG_XFER_THREADS=8 timeout 600 python bench.py --no-cpu --blocks none > $O/bench_t8_$i.json 2> $O/bench_t8_$i.err
done
cat $O/nproc.txt
for f in $O/e2e_probe*.txt; do echo "== $f"; grep -E 'narrowed \(pinned|widened|e2e rs_rank\(pinned' $f | tr '\n' ' '; echo; done
for f in $O/bench*.json; do echo "$f $(python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['e2e']['ms_per_step'])")"; done
