"""Print the key metrics of an ncu report (details page) compactly."""
import csv, io, subprocess, sys
rep = sys.argv[1]
pat = [s.lower() for s in (sys.argv[2:] or ["duration", "tensor", "issue slots", "warp cycles per issued", "no eligible",
       "eligible warps", "shared memory", "l2 hit", "dram throughput", "memory throughput", "compute (sm) throughput",
       "registers", "achieved occupancy", "stall"])]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki, si, mi, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Section Name", "Metric Name", "Metric Unit", "Metric Value"))
for r in rows[1:]:
    name = r[mi].lower()
    if any(p in name for p in pat):
        print(f"{r[ki][:28]:28s} | {r[si][:26]:26s} | {r[mi][:48]:48s} | {r[vi]:>14s} {r[ui]}")
