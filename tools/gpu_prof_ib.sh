#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ib.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tc_intra_bwd -c 1 -o gpurun_out/ib_full \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_ib.log 2>&1
echo done >> gpurun_out/ncu_ib.log
