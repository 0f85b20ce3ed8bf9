"""Print `Section | Metric | Unit | Value` rows of an ncu report."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout.splitlines()
r = csv.reader(out)
h = next(r)
ix = [h.index(x) for x in ["Section Name", "Metric Name", "Metric Unit", "Metric Value"]]
want = sys.argv[2].split(",") if len(sys.argv) > 2 else None
for row in r:
    if len(row) <= max(ix) or not row[ix[1]]:
        continue
    if want and not any(w.lower() in (row[ix[0]] + row[ix[1]]).lower() for w in want):
        continue
    print(" | ".join(row[i] for i in ix))
