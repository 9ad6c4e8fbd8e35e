#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc4_state|k_tc4_tok" -c 2 -o gpurun_out/t4s_full \
  python bench.py --workload cfg3 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_t4s.log 2>&1
echo done >> gpurun_out/ncu_t4s.log
