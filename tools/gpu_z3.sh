#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/zdbg.py > gpurun_out/zdbg.txt 2>&1; tail -2 gpurun_out/zdbg.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench.log 2>&1
python -c "
import json,sys
for line in open('gpurun_out/bench.log'):
    if line.startswith('{'):
        d=json.loads(line); print(d['ms_per_step'], {k: round(v,3) for k,v in d['stages_ms'].items()})
"
timeout 300 python tools/trace_zv.py > gpurun_out/trace_zv.txt 2>&1
grep -A11 side gpurun_out/trace_zv.txt | grep -v stage
