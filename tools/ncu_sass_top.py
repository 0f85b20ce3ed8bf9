"""Summarise an `ncu --page source --csv --print-source sass` dump: total
stall reasons and the hottest SASS instructions (by warp-stall samples)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
def num(r, k):
    try:
        return float(r[ix[k]] or 0)
    except ValueError:
        return 0.0
tot = Counter()
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in data:
    for s in stalls:
        tot[s] += num(r, s)
S = sum(tot.values())
print("total samples", S)
for s, v in tot.most_common(12):
    print(f"  {s:28s} {100*v/S:5.1f}%")
ninst = sum(num(r, "Instructions Executed") for r in data)
print("instructions executed", ninst)
top = sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for r in top:
    st = sorted(((num(r, s), s) for s in stalls), reverse=True)[:2]
    print(f"{r[ix['Address']]:>6} {100*num(r,'Warp Stall Sampling (All Samples)')/S:5.2f}% "
          f"exec={num(r,'Instructions Executed'):.3g} thr={num(r,'Avg. Threads Executed'):4.1f} "
          f"{r[ix['Source']][:48]:48s} " + " ".join(f"{s[6:]}:{100*v/S:.2f}" for v, s in st))
