#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -k "backward_tensor_core or bf16" -q 2>&1 | tail -5 > gpurun_out/z_new.log
timeout 600 python bench.py --no-e2e --no-cpu > gpurun_out/bench.log 2>&1
timeout 300 python tools/trace_zv.py > gpurun_out/trace_zv.txt 2>&1
cat gpurun_out/z_new.log
python -c "
import json,sys
for line in open('gpurun_out/bench.log'):
    if line.startswith('{'):
        d=json.loads(line); print(d['ms_per_step'], {k: round(v,3) for k,v in d['stages_ms'].items()})
"
