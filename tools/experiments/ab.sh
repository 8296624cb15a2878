#!/bin/bash
# A/B driver: SG_* variants of bench workloads, e.g.
#   TAG=x8 RUNS="SG_CC_COMP4=0:cc26 SG_CC_COMP4=1:cc26" bash tools/experiments/ab.sh
# (passes x1-x12 of DESIGN.md §9: RUNS lists env[,env]:workload; TESTK runs a pytest -k subset first)
O=gpurun_out/${TAG:-x1}; mkdir -p $O
python -c "import __graft_entry__ as e; e.build()" > $O/build.log 2>&1
[ -n "$TESTK" ] && timeout 600 python -m pytest tests -m gpu -q -k "$TESTK" > $O/t.log 2>&1
for spec in $RUNS; do
  IFS=: read -r env wl <<< "$spec"
  f=$O/b_${env//[=,]/_}_$wl.json
  env ${env//,/ } timeout 300 python bench.py --workload $wl --no-cpu --no-e2e --blocks none > $f 2>&1
  python - "$f" "$env" "$wl" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    k = d["kernels_ms_per_step"]
    print(sys.argv[2], sys.argv[3], d["ms_per_step"], {a: round(b, 3) for a, b in k.items() if b > 0.05})
except Exception as e:
    print(sys.argv[2], sys.argv[3], "FAILED", e, open(sys.argv[1]).read()[-500:])
PY
done
if [ -n "$TESTK" ]; then tail -3 $O/t.log; fi
