#!/bin/bash
# Round evidence: full bench line, per-launch device time + DRAM bytes of one
# step (ncu, cold-cache/serialised), and an ncu --set full capture of the
# dominant kernels at b=1.  Summaries are built locally by tools/summarize_profiles.py.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_full.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu \
  > gpurun_out/ncu_launch_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_tc_zvjp|k_tc_ib|k_tc_out|k_tc_featmajor}" \
  -c ${NCU_C:-7} -o gpurun_out/prof_full python tools/time_fwd.py --b 1 --iters 1 --bwd > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
