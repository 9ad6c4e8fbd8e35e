#!/bin/bash
# fused forward update + scan: parity and step time with / without it
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -s -k "not expansion and not zero_den" > gpurun_out/fs_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fs_tests.log
grep -E "max_rel|norm-wise|passed|failed" gpurun_out/fs_tests.log | tail -30
for f in 1 0; do
  PA_FUSED_SCAN=$f PA_STAGE_TIMING=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/fs_bench_$f.log 2>&1
  python - "$f" <<'PY'
import json, sys
for line in open(f"gpurun_out/fs_bench_{sys.argv[1]}.log"):
    if line.startswith("{"):
        d = json.loads(line)
        print("fused", sys.argv[1], round(d["ms_per_step"], 3), "ms", {k: round(v, 3) for k, v in d.get("stages_ms", {}).items()}, d.get("clocks"))
PY
done
