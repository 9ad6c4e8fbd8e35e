#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
   python bench.py --workload cfg3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_cfg3.log 2>&1
echo done >> gpurun_out/ncu_cfg3.log
