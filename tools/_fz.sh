O=gpurun_out/fz9; mkdir -p $O
timeout 600 python -m pytest tests/test_listrank_gpu.py tests/test_contract_gpu.py -x -q > $O/pytest.log 2>&1
for w in lr26 lr28; do timeout 300 python bench.py --workload $w --no-e2e --no-cpu > $O/b_${w}.json 2> $O/b_${w}.err; done
tail -n 2 $O/pytest*.log
for x in $O/b_*.json; do echo $x; python -c "import json,sys;d=json.loads(open('$x').read().strip().splitlines()[-1]);k=d['kernels_ms'];print(d['ms_per_step'],k['rs3_walk'],k['rs5_refine'],k['rs5_scatter'])"; done
