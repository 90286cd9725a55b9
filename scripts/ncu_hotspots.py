"""Summarise an `ncu --page source --csv --print-source sass` dump: top instructions by stall samples.

    python scripts/ncu_hotspots.py src.csv [top]
"""
import csv
import sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[2:]:
    if len(r) != len(hdr):
        continue
    try:
        samp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = {k: int(r[ix[k]] or 0) for k in stall_cols}
    data.append((r[ix["Address"]], r[ix["Source"]], samp, st, r[ix["Instructions Executed"]]))
tot = sum(d[2] for d in data)
print(f"total samples {tot}")
agg = Counter()
for d in data:
    for k, v in d[3].items():
        agg[k] += v
print("by reason:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in agg.most_common(10)))
op = Counter()
for d in data:
    op[d[1].split()[0] if d[1].split() else "?"] += d[2]
print("by opcode:", ", ".join(f"{k} {v / tot:.1%}" for k, v in op.most_common(15)))
print()
for i, d in sorted(enumerate(data), key=lambda t: -t[1][2])[:top]:
    reasons = ", ".join(f"{k[6:]}={v}" for k, v in sorted(d[3].items(), key=lambda t: -t[1])[:3] if v)
    print(f"{i:5d} {d[0]} {d[2] / tot:6.2%} {d[1][:60]:60s} {reasons}")
