#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tc_zvjp --launch-skip 1 -c 1 -o gpurun_out/r02b_zv1 \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_zv1.log 2>&1
echo done >> gpurun_out/ncu_zv1.log
