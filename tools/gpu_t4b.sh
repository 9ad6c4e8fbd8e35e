#!/bin/bash
# degree-4 path: parity and configs[2] step time
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -x -s -m gpu -k "p4 or config2 or fixture or config0 or configs0 or f32" > gpurun_out/t4b_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t4b_tests.log
grep -E "max_rel|passed|failed|Error" gpurun_out/t4b_tests.log | tail -12
PA_STAGE_TIMING=1 timeout 600 python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu > gpurun_out/t4b_bench.log 2>&1
python - <<'PY'
import json
for line in open("gpurun_out/t4b_bench.log"):
    if line.startswith("{"):
        d = json.loads(line)
        print("cfg3", round(d["ms_per_step"], 2), "ms", d.get("clocks"))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t4b_launches.csv python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/summarize_profiles.py gpurun_out/t4b_launches.csv 2>/dev/null | head -30 || true
