#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "backward or golden or config1 or smoke" > gpurun_out/pt_ib.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ib.log
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_sp.py tests/test_gpu_sp_procs.py -q -s -x > gpurun_out/pt_ib2.log 2>&1; echo "rc=$?" >> gpurun_out/pt_ib2.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ib.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ib.log
