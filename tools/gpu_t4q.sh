#!/bin/bash
# quick degree-4 check: p=4 parity + configs[2] bench + launch shares
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu -k "p4 or config2" > gpurun_out/t4q_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t4q_tests.log
tail -2 gpurun_out/t4q_tests.log
PA_STAGE_TIMING=1 timeout 600 python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/t4q_bench.log 2>&1
python - <<'PY'
import json
for line in open("gpurun_out/t4q_bench.log"):
    if line.startswith("{"):
        d = json.loads(line)
        print("cfg3", round(d["ms_per_step"], 2), "ms", d.get("clocks"))
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t4q_launches.csv python bench.py --workload cfg3 --steps 1 --warmup 0 --no-cpu --no-e2e > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/t4q_launches.csv')))
hdr=None; agg=collections.defaultdict(float)
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr is None or len(r)!=len(hdr): continue
    d=dict(zip(hdr,r))
    if d.get('Metric Name')!='gpu__time_duration.sum': continue
    agg[d['Kernel Name'][:40]] += float(d['Metric Value'].replace(',',''))
tot=sum(agg.values())
for n,v in sorted(agg.items(), key=lambda x:-x[1])[:6]: print(f"{n:40s} {100*v/tot:5.1f}%")
PY
