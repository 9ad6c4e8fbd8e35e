#!/bin/bash
# Round-2 final: the whole gpu test suite, smoke, and the bench lines of every workload.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -s -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg3.log
timeout 300 python bench.py --workload cfg1 --steps 10 --warmup 3 > gpurun_out/bench_cfg1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg1.log
timeout 600 python bench.py --workload sp1m --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_sp1m.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sp1m.log
timeout 900 python bench.py --workload lm124m --steps 5 --warmup 3 > gpurun_out/bench_lm.log 2>&1; echo "rc=$?" >> gpurun_out/bench_lm.log
echo done > gpurun_out/final_done.txt
