"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum
--csv): us per step (divided by argv[2] steps), launches, share."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    agg[r[ki][:90]][0] += 1
    agg[r[ki][:90]][1] += v
tot = sum(v[1] for v in agg.values())
print("kernel,launches,us_per_step,share")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f'"{k}",{v[0]},{v[1] / steps / 1e3:.1f},{v[1] / tot:.4f}')
