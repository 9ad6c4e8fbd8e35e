#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for mode in overlap serial; do
  if [ $mode == serial ]; then export PA_BWD_SERIAL=1; fi
  timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench_$mode.log 2>&1
  python -c "
import json,sys
for line in open('gpurun_out/bench_$mode.log'):
    if line.startswith('{'):
        d=json.loads(line); print('$mode', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms'].items()})
"
done
