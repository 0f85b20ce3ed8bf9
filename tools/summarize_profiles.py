"""Summarise a gpu_round.sh capture (gpurun_out/) into profiles/<tag>_*.

usage: python tools/summarize_profiles.py <tag> [gpurun_out]

  <tag>_launches_summary.csv  per-kernel launches / total time / share of the
                              ncu launch list (gpu__time_duration.sum,
                              --clock-control none: cold-cache, serialised —
                              compare shares, not absolutes)
  <tag>_k_dp_multi_ncu.txt    selected details + raw counters of the one
                              `ncu --set full` capture, and the hottest source
                              lines (tools/ncu_lines.py)
"""
import collections
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
mangled = sys.argv[3] if len(sys.argv) > 3 else "_ZN3amp12k_trie_stageENS_10TrieParamsEimPy"
kname_short = sys.argv[4] if len(sys.argv) > 4 else "k_trie_stage"
out = os.path.join(ROOT, "profiles")


def rows(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    return list(csv.DictReader(lines))


# ---- launch list ---------------------------------------------------------
L = rows(os.path.join(src, "launches.csv"))
agg = collections.OrderedDict()
for r in L:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    a = agg.setdefault(r["Kernel Name"], [0, 0.0])
    a[0] += 1
    a[1] += float(r["Metric Value"]) / 1e3
tot = sum(v[1] for v in agg.values())
with open(os.path.join(out, f"{tag}_launches_summary.csv"), "w") as f:
    f.write("# ncu launch list: python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-dense "
            "--no-e2e (tools/gpu_round.sh)\n")
    f.write("# metric gpu__time_duration.sum, --clock-control none (cold-cache, serialised; compare "
            "shares, not absolutes)\n")
    f.write("kernel,launches,total_us,share\n")
    for k, (n, us) in sorted(agg.items(), key=lambda t: -t[1][1]):
        f.write(f'"{k}",{n},{us:.1f},{us / tot:.4f}\n')

# ---- full capture --------------------------------------------------------
want_details = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
                "Executed Ipc Active", "Issue Slots Busy", "Eligible Warps Per Scheduler",
                "No Eligible", "Warp Cycles Per Issued Instruction", "Registers Per Thread",
                "Dynamic Shared Memory Per Block", "Block Size", "Grid Size",
                "Theoretical Occupancy", "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate"]
det = rows(os.path.join(src, "kdp_full_details.csv"))
raw = list(csv.reader(open(os.path.join(src, "kdp_full_raw.csv"))))
raw = [r for r in raw if r and not r[0].startswith("==")]
hdr, unit, val = raw[0], raw[1], raw[2]
want_raw = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__grid_size", "launch__block_size"]
kname = det[0]["Kernel Name"] if det else "?"
lines_txt = ""
try:
    lib = os.path.join(ROOT, "paper_2210_07297_b200", "libamp_search.so")
    lines_txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"),
                                os.path.join(src, "kdp_full_sass.csv"), lib, mangled, "25"],
                               capture_output=True, text=True).stdout
except Exception as e:  # noqa: BLE001
    lines_txt = f"(ncu_lines failed: {e})"
with open(os.path.join(out, f"{tag}_{kname_short}_ncu.txt"), "w") as f:
    f.write(f"# ncu --set full --clock-control none --import-source on -k regex:{kname_short} "
            "(tools/gpu_round.sh) python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-dense "
            "--no-e2e --no-wall-time\n")
    f.write(f"# kernel: {kname}\n\n## details\n")
    for r in det:
        if r["Metric Name"] in want_details:
            f.write(f'{r["Section Name"]} | {r["Metric Name"]} | {r["Metric Unit"]} | '
                    f'{r["Metric Value"]}\n')
    f.write("\n## raw\n")
    for name in want_raw:
        if name in hdr:
            i = hdr.index(name)
            f.write(f"{name} {unit[i]} {val[i]}\n")
    f.write("\n## hottest source lines (tools/ncu_lines.py)\n")
    f.write(lines_txt)
print("wrote", tag)

# ---- per-candidate kernels: instructions and DRAM bytes per item ----------
# (tools/gpu_round.sh's pe_full capture: the first chunk of the measured run
#  of prof_eval.py 100000000 — 67,108,864 items, of which the 45,714,304 of
#  the pp >= 3 classes go through K_place; K_est covers the whole chunk)
pe = os.path.join(src, "pe_full_raw.csv")
if os.path.exists(pe):
    import json
    raw = [r for r in csv.reader(open(pe)) if r and not r[0].startswith("==")]
    hdr, unit = raw[0], raw[1]
    n_cls, P = 70, -(-100_000_000 // 70)
    heavy = 32 * P  # pp >= 3 items: K_place's work (K_est: every item)
    items = {"k_place_t": heavy, "k_est_t": 100_000_000}
    out_j = {"source": f"profiles/{tag}_kernel_counts.json from ncu --set full (tools/gpu_round.sh)",
             "workload": "hetero_cluster sweep, 100M candidates: every launch of one measured run "
                         "(2 chunks), summed per kernel"}
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    acc = {}
    for row in raw[2:]:
        d = dict(zip(hdr, row))
        name = d["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1].split()[-1]
        if name not in items:
            continue
        rd = float(d["dram__bytes_read.sum"]) * scale[unit[hdr.index("dram__bytes_read.sum")]]
        wr = float(d["dram__bytes_write.sum"]) * scale[unit[hdr.index("dram__bytes_write.sum")]]
        tu = unit[hdr.index("gpu__time_duration.sum")]
        ms = float(d["gpu__time_duration.sum"]) * {"ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(tu, 1.0)
        a = acc.setdefault(name, [0.0, 0.0, 0.0, 0])
        a[0] += float(d["smsp__inst_executed.sum"])
        a[1] += rd + wr
        a[2] += ms
        a[3] += 1
    for name, (inst, byts, ms, nl) in acc.items():
        n = items[name]
        out_j[name] = {"items": n, "launches": nl, "warp_inst_per_item": inst / n,
                       "dram_bytes_per_item": byts / n, "duration_ms": ms}
    with open(os.path.join(out, f"{tag}_kernel_counts.json"), "w") as f:
        json.dump(out_j, f, indent=1)
    print("kernel counts", out_j)

# ---- per-candidate kernels: details + hottest source lines ---------------
rep = os.path.join(src, "pe_full.ncu-rep")
if os.path.exists(rep):
    import re
    pdet = rows(os.path.join(src, "pe_full_details.csv"))
    syms = subprocess.run(["cuobjdump", "-symbols", os.path.join(ROOT, "paper_2210_07297_b200",
                                                               "libamp_search.so")],
                          capture_output=True, text=True).stdout
    for short in ("k_est_t", "k_place_t"):
        mine = [r for r in pdet if re.search(rf"\b{short}<", r["Kernel Name"])]
        if not mine:
            continue
        kname = mine[0]["Kernel Name"]
        sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                               "-k", f"regex:{short}", "--launch-count", "1"],
                              capture_output=True, text=True).stdout.splitlines()
        heads = [i for i, l in enumerate(sass) if l.startswith('"Kernel Name"')]
        block = sass[heads[0]:heads[1] if len(heads) > 1 else len(sass)] if heads else []
        tmpf = os.path.join(src, f"{short}_sass.csv")
        with open(tmpf, "w") as f:
            f.write("\n".join(block) + "\n")
        # the launched instantiation (FAST shape kernels when present)
        cands = re.findall(rf"_ZN3amp\d+{short}ILi16ELb[01]EEEvNS_10EvalParamsE", syms)
        fast = "true" in kname or ", 1>" in kname
        mang = next((c for c in cands if ("Lb1" in c) == fast), cands[0] if cands else "")
        lines_txt = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmpf,
                                    os.path.join(ROOT, "paper_2210_07297_b200", "libamp_search.so"),
                                    mang, "25"], capture_output=True, text=True).stdout
        with open(os.path.join(out, f"{tag}_{short}_ncu.txt"), "w") as f:
            f.write(f"# ncu --set full --clock-control none --import-source on -k regex:'k_est_t|k_place_t' "
                    f"(tools/gpu_round.sh) python tools/prof_eval.py 100000000 — first 64M-item chunk of "
                    f"the measured run\n# kernel: {kname}\n\n## details\n")
            seen = set()
            for r in mine:
                if r["Metric Name"] in want_details and r["Metric Name"] not in seen:
                    seen.add(r["Metric Name"])
                    f.write(f'{r["Section Name"]} | {r["Metric Name"]} | {r["Metric Unit"]} | '
                            f'{r["Metric Value"]}\n')
            f.write("\n## hottest source lines (tools/ncu_lines.py)\n")
            f.write(lines_txt)
        print("wrote", f"{tag}_{short}_ncu.txt")
