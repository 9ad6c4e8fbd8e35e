#!/bin/bash
# GPU tests + a quick bench line (stage times), used between kernel changes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench.log 2>&1
python -c "
import json,sys
for line in open('gpurun_out/bench.log'):
    if line.startswith('{'):
        d=json.loads(line); print(round(d['ms_per_step'],3), d['clocks'], {k: round(v,3) for k,v in d['stages_ms'].items()})
"
