#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc4_vjp" -c 1 -o gpurun_out/t4v2_full \
  python bench.py --workload cfg3 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_t4v2.log 2>&1
echo done >> gpurun_out/ncu_t4v2.log
