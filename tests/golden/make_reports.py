"""Regenerate tests/golden/reports/: the reference CLI `plan` outputs.

Runs oracle/_ref/gen_report (reference plan() + write_report +
print_candidate_table, compiled from /root/reference by oracle/Makefile) on
the reference configs.  Needs /root/reference; the fixtures travel.

  <case>.json   report.json (report.cpp:85-91)
  <case>.txt    stdout: ranked table + "best by simulation" line
  <case>.rc     exit code (and <case>.err stderr when non-zero)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_2210_07297_b200 import problem as P  # noqa: E402

REF = "/root/reference/proj/configs"
BIN = os.path.join(ROOT, "oracle", "_ref", "gen_report")
OUT = os.path.join(HERE, "reports")

# case -> (config dir, gbs, budget, profile override)
CASES = {
    "C1_b10": ("homogeneous", 32, 10, None),
    "C1_b5": ("homogeneous", 32, 5, None),
    "C2_b10": ("hetero_cluster", 32, 10, None),
    "C3_b10": ("hetero_model", 64, 10, None),
    "C1_partial_b3": ("homogeneous", 32, 3, "partial"),  # test_cli.cpp:131-160
    "C1_allmiss_b1": ("homogeneous", 32, 1, "empty"),    # test_cli.cpp:100-115
    # CLI `baseline` (megatron_baseline), test_cli.cpp:267-281
    "C1_baseline_layer": ("homogeneous", 32, 1, None),
    "C1_baseline_param": ("homogeneous", 32, 1, None),
    "C2_baseline_layer": ("hetero_cluster", 32, 1, None),
    "C3_baseline_param": ("hetero_model", 64, 1, None),
    "C1_partial_baseline_layer": ("homogeneous", 32, 1, "partial"),
    # CLI `anneal` (acceptance criterion 9: --budget 5 --iterations 60 --seed 17)
    "C1_anneal_i60_s17": ("homogeneous", 32, 5, None),
    "C2_anneal_i200_s3": ("hetero_cluster", 32, 10, None),
    "C3_anneal_i120_s11": ("hetero_model", 64, 10, None),
}


def profile_variant(kind, src, dst):
    """The test_cli.cpp profile variants, written with our json_io mirror."""
    full = P.load_profile(src)
    t = P.ProfileTable()
    if kind == "partial":
        for (l, tmp, mbs), v in full.entries():
            if tmp == 1:
                t.set(l, tmp, mbs, v)
    P.write_json_file(P.profile_to_json(t), dst)


def main():
    subprocess.run(["make", "-C", ROOT, "-f", os.path.join(ROOT, "oracle", "Makefile"), BIN],
                   check=True)
    os.makedirs(OUT, exist_ok=True)
    for case, (cfg, gbs, budget, variant) in CASES.items():
        d = os.path.join(REF, cfg)
        prof = os.path.join(d, "profile.json")
        if variant:
            prof = f"/tmp/parplan_{variant}_profile.json"
            profile_variant(variant, os.path.join(d, "profile.json"), prof)
        rep = os.path.join(OUT, case + ".json")
        if os.path.exists(rep):
            os.remove(rep)
        env = dict(os.environ)
        if "baseline" in case:
            env["GEN_MODE"] = "param-balance" if case.endswith("param") else "layer-balance"
        if "anneal" in case:  # C?_anneal_i<iters>_s<seed>, with the trace
            it, sd = case.split("_i")[1].split("_s")
            env["GEN_MODE"] = f"anneal:{it}:{sd}:trace"
        r = subprocess.run([BIN, os.path.join(d, "model.json"), os.path.join(d, "cluster.json"), prof,
                            str(gbs), str(budget), rep], capture_output=True, text=True, env=env)
        with open(os.path.join(OUT, case + ".txt"), "w") as f:
            f.write(r.stdout)
        with open(os.path.join(OUT, case + ".rc"), "w") as f:
            f.write(f"{r.returncode}\n")
        if r.returncode:
            with open(os.path.join(OUT, case + ".err"), "w") as f:
                f.write(r.stderr)
        print(case, "rc", r.returncode)
    # the reference's profile.json bytes (json_io.cpp write_file), pinned by hash
    import hashlib
    for cfg in ("homogeneous", "hetero_cluster", "hetero_model"):
        with open(os.path.join(REF, cfg, "profile.json"), "rb") as f:
            h = hashlib.sha256(f.read()).hexdigest()
        with open(os.path.join(OUT, f"profile_{cfg}.sha256"), "w") as f:
            f.write(f"{h}  configs/{cfg}/profile.json\n")


if __name__ == "__main__":
    main()
