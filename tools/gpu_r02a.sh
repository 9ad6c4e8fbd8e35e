#!/bin/bash
# Round-2 GPU session A: full gpu test suite, smoke, default bench, extra workloads.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --workload cfg3 --steps 3 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg3.log
timeout 300 python bench.py --workload cfg1 --steps 10 --warmup 3 > gpurun_out/bench_cfg1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg1.log
timeout 600 python bench.py --workload sp1m --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_sp1m.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sp1m.log
tail -3 gpurun_out/*.log
