#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -s -x -k "p4 or bf16_matches" > gpurun_out/pt_t4.log 2>&1; echo "rc=$?" >> gpurun_out/pt_t4.log
timeout 600 python bench.py --workload cfg3 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/bench_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
   python bench.py --workload cfg3 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_cfg3.log 2>&1
