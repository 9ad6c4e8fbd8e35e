#!/bin/bash
# new-kernel check: targeted backward tests, full gpu suite, bench (new and old state VJP)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "backward_tensor_core" -x -q > gpurun_out/z_test.log 2>&1; echo "rc=$?" >> gpurun_out/z_test.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
PA_DPHI_OLD=1 timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_old.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_old.log
tail -n 25 gpurun_out/z_test.log; tail -n 3 gpurun_out/pytest_gpu.log
for f in bench bench_old; do python -c "
import json,sys
for line in open('gpurun_out/$f.log'):
    if line.startswith('{'):
        d=json.loads(line); print('$f', d['ms_per_step'], {k: round(v,3) for k,v in d['stages_ms'].items()})
"; done
