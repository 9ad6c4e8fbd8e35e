#!/bin/bash
# Round-2 evidence after the fused-scan / degree-4 work: bench lines, launch lists, ncu of the top kernels.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --workload cfg3 --steps 5 --warmup 3 > gpurun_out/bench_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg3.log
timeout 300 python bench.py --workload cfg1 --steps 10 --warmup 3 > gpurun_out/bench_cfg1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg1.log
timeout 600 python bench.py --workload sp1m --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_sp1m.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sp1m.log
timeout 900 python bench.py --workload lm124m --steps 5 --warmup 3 > gpurun_out/bench_lm.log 2>&1; echo "rc=$?" >> gpurun_out/bench_lm.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv \
   python bench.py --workload cfg3 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_launch3.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_tc_intra_bwd|k_tc_zvjp|k_tc_out2|k_tc_featscan" -c 5 \
   -o gpurun_out/r02b_top python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/ncu_top.log 2>&1
echo done > gpurun_out/evidence_done.txt
