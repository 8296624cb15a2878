O=gpurun_out/fz22; mkdir -p $O
for t in 0 65536 262144 524288 1048576; do for w in lr26 lr28; do SG_RS_TOPN=$t timeout 300 python bench.py --workload $w --no-cpu --no-e2e > $O/b_${w}_$t.json 2> $O/b_${w}_$t.err; done; done
for x in $O/b_*.json; do echo $x; python -c "
import json,sys;d=json.loads(open('$x').read().strip().splitlines()[-1]);k=d['kernels_ms'];print(d['ms_per_step'],'walk',k['rs3_walk'],d['roofline']['pipeline']['frac'])"; done
SG_RS_TOPN=262144 timeout 900 python -m pytest tests/test_listrank_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
