"""Summarise the ncu launch list of one bench step (tools/gpu_evidence.sh) into
profiles/: a per-kernel table (device time, DRAM bytes, share of the step) and
profiles/ncu_traffic.json (DRAM bytes per launch keyed by bench stage, read by
bench.py for roofline.traffic).

    python tools/summarize_profiles.py gpurun_out/launches.csv r01
"""

from __future__ import annotations

import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# bench stage -> kernel-name fragments (pa_tc*.cu)
STAGES = {
    "fwd_prep": ["k_tc_prep_gates", "k_tc_prep_xt#fwd", "k_tc_prep_rows#fwd"],
    "fwd_update_state": ["k_tc_featscan<", "k_tc_featmajor<0"],
    "fwd_discumsum": ["k_tc_scan_fwd"],
    "fwd_attn_query": ["k_tc_out"],
    "bwd_prep": ["k_tc_bwd_prep", "k_tc_prep_xt#bwd", "k_tc_prep_rows#bwd"],
    "bwd_query_state_dA": ["k_tc_featscan_bwd", "k_tc_featmajor<1"],
    "bwd_discumsum": ["k_tc_scan_bwd"],
    "bwd_intra": ["k_tc_intra_bwd", "k_tc_ib"],
    "bwd_query_state_dq": ["k_tc_zvjp<0", "k_tc_dq_chunk0"],
    "bwd_update_state": ["k_tc_zvjp<1"],
    "bwd_finish": ["k_tc_gate_finish"],
}


def short(name: str) -> str:
    n = name.replace("void ", "").replace("pa::", "").replace("(bool)", "").replace("(int)", "")
    return n.split("(")[0].replace(", ", ",")


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    recs = {}
    order = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        if key not in recs:
            recs[key] = {"name": short(d["Kernel Name"]), "grid": d.get("Grid Size", "")}
            order.append(key)
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        m = d["Metric Name"]
        if m == "gpu__time_duration.sum":
            recs[key]["ms"] = v / 1e6 if unit == "ns" else (v / 1e3 if unit == "us" else v)
        elif m.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            recs[key][m] = v * scale
    return [recs[k] for k in order]


def stage_of(name: str, phase: str) -> str | None:
    for st, frags in STAGES.items():
        for f in frags:
            frag, _, ph = f.partition("#")
            if frag in name and (not ph or ph == phase):
                return st
    return None


def main():
    path = sys.argv[1]
    tag = sys.argv[2] if len(sys.argv) > 2 else "r01"
    recs = load(path)
    # the last forward+backward step: from the last k_tc_prep_gates launch on
    start = max(i for i, r in enumerate(recs) if "k_tc_prep_gates" in r["name"])
    step = recs[start:]
    tot = sum(r.get("ms", 0.0) for r in step)
    lines = [f"ncu launch list, one fwd+bwd step of configs[1] (b=4 h=16 t=65536 c=1024 p=2 d=64, bf16);",
             "gpu__time_duration.sum and dram bytes per launch, --clock-control none (cold-cache, serialised:",
             "compare shares, not absolutes, with the CUDA-event bench line)", ""]
    traffic = {}
    phase = "fwd"
    for r in step:
        if "k_tc_bwd_prep" in r["name"] or "featmajor<1" in r["name"] or "featscan_bwd" in r["name"]:
            phase = "bwd"
        if r["name"].startswith("k_tc_prep_xt") and phase == "fwd" and any(
                "k_tc_out" in x["name"] for x in step[: step.index(r)]):
            phase = "bwd"
        st = stage_of(r["name"], phase)
        rb = r.get("dram__bytes_read.sum", 0.0)
        wb = r.get("dram__bytes_write.sum", 0.0)
        lines.append(f"{r['name'][:44]:44s} grid {r['grid']:>14s} {r.get('ms', 0):8.3f} ms "
                     f"{100 * r.get('ms', 0) / tot:5.1f}%  DRAM rd {rb / 1e9:7.3f} GB wr {wb / 1e9:7.3f} GB  [{st}]")
        if st:
            t = traffic.setdefault(st, {"bytes": 0.0, "launches": 0})
            t["bytes"] += rb + wb
            t["launches"] += 1
    lines.append(f"total {tot:.3f} ms")
    out = os.path.join(ROOT, "profiles", f"{tag}_launches.txt")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    per_launch = {k: v["bytes"] / max(v["launches"], 1) for k, v in traffic.items()}
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w") as f:
        json.dump({"source": f"profiles/{tag}_launches.txt", "unit": "bytes per launch", **per_launch}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
