"""Summarise an ncu --page source --print-source sass CSV: hot instructions with
their top stall reasons, and per-region sample totals."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 200
hdr = rows[1]
si = hdr.index('Warp Stall Sampling (All Samples)')
src = hdr.index('Source')
ie = hdr.index('Instructions Executed')
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
sidx = [hdr.index(h) for h in stalls]


def I(x):
    try:
        return int(x)
    except ValueError:
        return 0


seen, out = set(), []
for r in rows[2:]:
    if len(r) <= si or r[0] in seen:
        continue
    seen.add(r[0])
    out.append(r)
tot = sum(I(r[si]) for r in out)
print('total samples', tot)
for i, r in enumerate(out):
    n = I(r[si])
    if n > thr or 'UTC' in r[src] and 'HMMA' in r[src]:
        top = sorted([(I(r[j]), h[6:]) for j, h in zip(sidx, stalls)], reverse=True)[:3]
        print(f"{i:5d} {n:6d} {100*n/max(tot,1):5.1f}% ex={r[ie]:>8s} {r[src][:60]:60s} {top}")
