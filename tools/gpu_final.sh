#!/bin/bash
# round-end evidence: gpu tests, smoke, full bench (e2e + cpu baseline), sp1m bench,
# ncu launch list with DRAM bytes, ncu --set full of the dominant kernels
mkdir -p gpurun_out
nvidia-smi -q -d POWER,CLOCK > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | cut -c1-200
timeout 900 python bench.py --workload sp1m --steps 3 --warmup 1 --no-cpu > gpurun_out/bench_sp1m.log 2>&1; tail -1 gpurun_out/bench_sp1m.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu \
  > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_tc_zvjp|k_tc_ib|k_tc_out|k_tc_featmajor|k_tc_scan" \
  -c 9 -o gpurun_out/prof_full python tools/time_fwd.py --b 1 --iters 1 --bwd > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?"
