"""Attribute ncu SASS-level samples/instruction counts to CUDA source lines.

usage: ncu_lines.py <sass.csv from `ncu --page source --csv --print-source sass`>
                    <lib.so> <mangled kernel name> [top]
Uses nvdisasm -g line tables (build with -lineinfo)."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile

sass_csv, lib, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubins = [f for f in os.listdir(tmp) if f.endswith(".cubin")]
line_of = {}
for cb in cubins:
    out = subprocess.run(["nvdisasm", "-g", "-c", cb], cwd=tmp, capture_output=True, text=True).stdout
    cur_fn, cur_line = None, None
    for ln in out.splitlines():
        m = re.match(r"\.text\.(\S+):", ln.strip())
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn == fn:
            line_of[int(m.group(1), 16)] = cur_line
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[ix["Address"]] != "Address"]
# (a capture with several launches lists the kernel once per launch: keep the first)
base = int(data[0][ix["Address"]], 16)
seen, first = set(), []
for r in data:
    a = r[ix["Address"]]
    if a in seen:
        break
    seen.add(a)
    first.append(r)
data = first
def f(r, k):
    try:
        return float(r[ix[k]] or 0)
    except ValueError:
        return 0.0
agg = collections.defaultdict(lambda: [0.0, 0.0, collections.Counter()])
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in data:
    off = int(r[ix["Address"]], 16) - base
    key = line_of.get(off, "?")
    a = agg[key]
    a[0] += f(r, "Warp Stall Sampling (All Samples)")
    a[1] += f(r, "Instructions Executed")
    for s in stalls:
        a[2][s] += f(r, s)
S = sum(v[0] for v in agg.values())
E = sum(v[1] for v in agg.values())
src = {}
for k in agg:
    if ":" in k:
        fnm, ln = k.split(":")
        src[k] = fnm
print(f"total samples {S:.0f}, instructions {E:.3g}")
for k, (s, e, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    st = ", ".join(f"{n[6:]}={100*v/S:.1f}" for n, v in c.most_common(2))
    print(f"{k:28s} samples {100*s/S:5.1f}%  instr {100*e/E:5.1f}%  [{st}]")
