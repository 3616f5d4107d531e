"""Hot SASS lines and stall reasons from an ncu source-page CSV export.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_hot.py src.csv [top]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
S = ix["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[S] or 0) for r in data)
print(f"total samples {tot:.0f}")
agg = Counter()
for r in data:
    for h in stalls:
        agg[h] += float(r[ix[h]] or 0)
print("stall totals:", ", ".join(f"{k[6:]} {v/tot:.1%}" for k, v in agg.most_common(10)))
by = sorted(data, key=lambda r: -float(r[S] or 0))[:top]
for r in by:
    st = sorted(((float(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:3]
    print(f"{r[ix['Address']]:>6} {float(r[S] or 0)/tot:6.2%} {r[ix['Source']][:70]:70s} "
          + " ".join(f"{n}:{v/tot:.1%}" for v, n in st if v > 0))
