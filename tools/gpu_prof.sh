#!/bin/bash
# smoke + ncu --set full of the tensor-core kernels at b=1 (one replay set each)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"${NCU_K:-k_tc_}" -c ${NCU_C:-9} \
  -o gpurun_out/prof_full python tools/time_fwd.py --b 1 --iters 1 --bwd > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
