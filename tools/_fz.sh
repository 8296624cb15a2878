O=gpurun_out/fz27; mkdir -p $O
timeout 900 python -m pytest tests/test_listrank_gpu.py tests/test_host_api.py -m gpu -x -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
PYTHONPATH=. ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"spl_meta_block|spl_keys" -c 6 python tools/_p.py > $O/ncu.txt 2>&1; grep -E "duration" $O/ncu.txt | head -6
timeout 300 python bench.py --no-cpu > $O/b.json 2>/dev/null; python -c "import json;d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['e2e']['value'])"
