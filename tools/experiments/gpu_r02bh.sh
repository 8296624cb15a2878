#!/bin/bash
# e2e on the box that read 91.6 ms in r02final4: phases and repeated bench e2e
TAG=${TAG:-r02bh}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
(nproc; lscpu | grep -E "Model name|L3|MHz"; cat /sys/kernel/mm/transparent_hugepage/enabled; uptime; free -g) > $O/host.txt 2>&1
for i in 1 2; do
  timeout 600 python tools/probe_e2e2.py > $O/e2e_probe_$i.txt 2>&1
  timeout 600 python bench.py --no-cpu --blocks none > $O/bench_$i.json 2> $O/bench_$i.err
done
cat $O/host.txt
for f in $O/e2e_probe*.txt; do echo "== $f"; cat $f | tr '\n' ' '; echo; done
for f in $O/bench*.json; do echo "$f $(python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['e2e'])")"; done
