#!/bin/bash
python -c "import __graft_entry__ as e; e.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu25.log 2>&1
tail -3 gpurun_out/pytest_gpu25.log
python tools/probe_overhead.py lr26
timeout 600 python bench.py > gpurun_out/b25_lr26.json 2> gpurun_out/b25_lr26.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --workload cc26 --no-cpu > gpurun_out/b25_cc26_tr1.json 2> gpurun_out/b25_cc26_tr1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --workload lr26 --no-cpu --no-secondary > gpurun_out/b25_lr26_tr1.json 2> gpurun_out/b25_lr26_tr1.err
tail -c 1500 gpurun_out/b25_cc26_tr1.err
