"""Summarise a tools/gpu_round.sh capture (gpurun_out/) into profiles/<tag>_*.

usage: python tools/profile_round.py <tag> [gpurun_out]

  <tag>_launches_summary.csv  per-kernel launches / us per step / share of the
                              ncu launch list (gpu__time_duration.sum,
                              --clock-control none: cold-cache, serialised —
                              compare shares, not absolutes)
  <tag>_<kernel>_ncu.txt      selected details + raw counters of the
                              `ncu --set full` capture of one measured run
  r2_kernel_counts.json       per kernel of that run: launches, duration,
                              DRAM bytes, warp instructions — with the sha256
                              of the library that was profiled (bench.py uses
                              the counts only for the same build)
"""
import collections
import csv
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
out = os.path.join(ROOT, "profiles")
LIB = os.path.join(ROOT, "paper_2210_07297_b200", "libamp_search.so")
KERNELS = ["k_trie_dp", "k_trie_build", "k_trie_back", "k_est_t", "k_place_t", "k_run_pipe"]


def short(name):
    for k in KERNELS:
        if k in name:
            return k
    return None


# ---- launch list ---------------------------------------------------------
rows = [r for r in csv.reader(open(os.path.join(src, "launches.csv"))) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    a = agg.setdefault(r[ki], [0, 0.0])
    a[0] += 1
    a[1] += v / 1e3
tot = sum(v[1] for v in agg.values())
steps = float(os.environ.get("PROFILE_STEPS", "2"))
with open(os.path.join(out, f"{tag}_launches_summary.csv"), "w") as f:
    f.write("# ncu launch list: python tools/prof_eval.py 100000000 (2 runs of the bench workload: "
            "100M candidates) — tools/gpu_round.sh\n")
    f.write("# metric gpu__time_duration.sum, --clock-control none (cold-cache, serialised; compare "
            "shares, not absolutes)\n")
    f.write("kernel,launches,us_per_run,share\n")
    for k, (n, us) in sorted(agg.items(), key=lambda t: -t[1][1]):
        f.write(f'"{k[:120]}",{n},{us / steps:.1f},{us / tot:.4f}\n')

# ---- full capture of one run ----------------------------------------------
rep = os.path.join(src, "pe_full.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
raw = [r for r in csv.reader(raw.splitlines()) if r]
h, units, data = raw[0], raw[1], raw[2:]
ix = {k: i for i, k in enumerate(h)}


def num(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except (KeyError, ValueError):
        return 0.0


counts = {"source": f"profiles/r2_kernel_counts.json from ncu --set full of one measured run "
                    f"(tools/gpu_round.sh, capture {tag})",
          "workload": "hetero_cluster sweep, 100M candidates (tools/prof_eval.py): every launch of "
                      "the second run, summed per kernel",
          "lib_sha256": hashlib.sha256(open(LIB, "rb").read()).hexdigest()}
for r in data:
    k = short(r[ix["Kernel Name"]])
    if not k:
        continue
    c = counts.setdefault(k, {"launches": 0, "runs": 1, "duration_ms": 0.0, "dram_bytes": 0.0,
                              "warp_inst": 0.0, "fp64_pipe_pct": []})
    c["launches"] += 1
    c["duration_ms"] += num(r, "gpu__time_duration.sum") * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
                                                             "second": 1e3}.get(units[ix["gpu__time_duration.sum"]], 1e-6)
    mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        c["dram_bytes"] += num(r, m) * mul.get(units[ix[m]], 1)
    c["warp_inst"] += num(r, "smsp__inst_executed.sum")
    c["fp64_pipe_pct"].append(num(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"))
with open(os.path.join(out, "r2_kernel_counts.json"), "w") as f:
    json.dump(counts, f, indent=1)

details = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_details.py"), rep,
                          "Duration,Compute (SM) Throughput,Memory Throughput,DRAM Throughput,"
                          "Executed Ipc Active,Issue Slots Busy,Eligible Warps,No Eligible,"
                          "Warp Cycles Per Issued,Registers Per Thread,Dynamic Shared Memory,"
                          "Theoretical Occupancy,Achieved Occupancy,L1/TEX Hit,L2 Hit,Block Size,Grid Size"],
                         capture_output=True, text=True).stdout
with open(os.path.join(out, f"{tag}_kernels_ncu.txt"), "w") as f:
    f.write("# ncu --set full --clock-control none -k regex:'k_trie_dp|k_trie_build|k_est_t|k_place_t' of the "
            "second run of tools/prof_eval.py 100000000 (tools/gpu_round.sh)\n")
    f.write("# kernels in launch order: " + ", ".join(short(r[ix['Kernel Name']]) or r[ix['Kernel Name']][:40]
                                                      for r in data) + "\n\n")
    f.write(details)
    f.write("\n## per-kernel sums (r2_kernel_counts.json)\n")
    for k, v in counts.items():
        if isinstance(v, dict):
            f.write(f"{k}: {json.dumps(v)}\n")
print(json.dumps({k: v for k, v in counts.items() if isinstance(v, dict)}, indent=1))
