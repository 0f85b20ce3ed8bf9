"""Regenerate the golden fixtures under tests/golden/ from the reference.

Run in the build container (needs /root/reference and oracle/_ref built):
    make -f oracle/Makefile all oracle/_ref/gen_golden
    ./oracle/_ref/gen_golden tests/golden          # dp_*.json
    python tests/golden/make_golden.py             # scenarios + plan/sweep goldens

scenarios/<name>.json  the reference's three config directories
                       (proj/configs/*/{model,cluster,profile}.json) in the
                       compact SoA form of paper_2210_07297_b200.problem
plan_<name>.json       reference parplan::plan() (budget 10) ranked output
sweep_<name>.json      reference call chain over the C5 placement sweep
All doubles are stored as C99 hex strings (float.hex) so they are exact.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import bindings as B  # noqa: E402
from paper_2210_07297_b200 import problem as P  # noqa: E402

REF_CONFIGS = "/root/reference/proj/configs"
SCEN = {"homogeneous": 32, "hetero_cluster": 32, "hetero_model": 64}


def hx(v):
    return float(v).hex()


def plan_golden(sc, budget=10):
    enc = P.EncodedProblem.from_scenario(sc)
    max_pp = max(c[0] for c in P.candidate_classes(sc.cluster.device_count(), sc.gbs))
    r = B.ref_plan(enc, max_pp, budget=budget, workers=8)
    out = []
    for i, rec in enumerate(r["records"]):
        pp = int(rec["pp"])
        e = {"rank": i + 1, "index": int(rec["index"]),
             "degrees": [pp, int(rec["dp"]), int(rec["tmp"])], "mbs": int(rec["mbs"]),
             "failure": r["failures"][i] or None}
        if not e["failure"]:
            e.update(total=hx(rec["total"]), pipeline_time=hx(rec["pipeline_time"]),
                     dpsync_time=hx(rec["dpsync_time"]),
                     cuts=[int(x) for x in r["cuts"][i][: pp + 1]],
                     per_stage_times=[hx(x) for x in r["stage_times"][i][:pp]],
                     per_edge_times=[hx(x) for x in r["edge_times"][i][: pp - 1]])
            sim = r["simulated"][i]
            e["simulated"] = None if sim != sim else hx(sim)
        out.append(e)
    return {"scenario": sc.name, "gbs": sc.gbs, "budget": budget, "best_index": r["best_index"],
            "candidates": out}


def sweep_golden(sc, P_, seed, n):
    enc = P.EncodedProblem.from_scenario(sc)
    max_pp = max(c[0] for c in P.candidate_classes(sc.cluster.device_count(), sc.gbs))
    r = B.ref_sweep(enc, P_, seed, 0, n, 8, max_pp, details=True)
    out = []
    for i, rec in enumerate(r["records"]):
        pp = int(rec["pp"])
        e = {"index": int(rec["index"]), "fail_code": int(rec["fail_code"])}
        if rec["fail_code"] == 0:
            e.update(total=hx(rec["total"]), cuts=[int(x) for x in r["cuts"][i][: pp + 1]])
        out.append(e)
    return {"scenario": sc.name, "placements_per_class": P_, "seed": seed, "n": n, "records": out}


def main():
    os.makedirs(os.path.join(HERE, "scenarios"), exist_ok=True)
    scen = {}
    for name, gbs in SCEN.items():
        d = os.path.join(REF_CONFIGS, name)
        sc = P.Scenario(name, P.load_model(os.path.join(d, "model.json")),
                        P.load_cluster(os.path.join(d, "cluster.json")),
                        P.load_profile(os.path.join(d, "profile.json")), gbs)
        scen[name] = sc
        with open(os.path.join(HERE, "scenarios", name + ".json"), "w") as f:
            json.dump(P.scenario_to_dict(sc), f, separators=(",", ":"))
        print("scenario", name)
    for name, sc in scen.items():
        g = plan_golden(sc)
        with open(os.path.join(HERE, f"plan_{name}.json"), "w") as f:
            json.dump(g, f, indent=0)
        print("plan", name, len(g["candidates"]), "best_index", g["best_index"])
    g = plan_golden(P.synthetic_c4(), budget=10)
    with open(os.path.join(HERE, "plan_synthetic96.json"), "w") as f:
        json.dump(g, f, indent=0)
    print("plan synthetic96", len(g["candidates"]))
    for name in ("hetero_cluster", "hetero_model"):
        g = sweep_golden(scen[name], 50, 0, 50 * (70 if name == "hetero_cluster" else 85))
        with open(os.path.join(HERE, f"sweep_{name}.json"), "w") as f:
            json.dump(g, f, separators=(",", ":"))
        print("sweep", name, g["n"])


if __name__ == "__main__":
    main()
