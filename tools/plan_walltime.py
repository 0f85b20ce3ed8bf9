"""AMP search wall time of plan() (the metric's second half): the GPU
drop-in (planner.plan: context create + K0/K0b + evaluate + rank + simulate
top budget) vs the reference parplan::plan on the host cores (oracle/_ref),
same inputs, same outputs, for C1-C4."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import scenario  # noqa: E402
from oracle import bindings as B  # noqa: E402
from paper_2210_07297_b200 import planner, problem as P  # noqa: E402

out = {}
for name in ["homogeneous", "hetero_cluster", "hetero_model", "synthetic96"]:
    sc = scenario(name)
    for budget in (0, 10):
        opts = P.PlanOptions(budget=budget, cost_options=sc.options.cost_options,
                             max_params_per_device=sc.options.max_params_per_device)
        planner.plan(sc.model, sc.cluster, sc.profile, sc.gbs, opts)  # warm-up
        ts = []
        for _ in range(5 if name != "synthetic96" else 3):
            t0 = time.perf_counter()
            res = planner.plan(sc.model, sc.cluster, sc.profile, sc.gbs, opts)
            ts.append(time.perf_counter() - t0)
        gpu = min(ts)
        ref = None
        if B.ref_available():
            enc = P.EncodedProblem.from_scenario(sc, opts)
            max_pp = max(c[0] for c in P.candidate_classes(sc.cluster.device_count(), sc.gbs))
            rs = []
            for _ in range(3 if name != "synthetic96" else 1):
                t0 = time.perf_counter()
                r = B.ref_plan(enc, max_pp, budget=budget, workers=os.cpu_count() or 1)
                rs.append(time.perf_counter() - t0)
            ref = min(rs)
            assert r["best_index"] == res.best_index
            assert [int(x) for x in r["records"]["index"]] == [c.index for c in res.candidates]
        out[f"{name}/budget{budget}"] = {"gpu_s": gpu, "ref_s": ref, "ref_threads": os.cpu_count(),
                                         "candidates": len(res.candidates)}
        print(name, budget, out[f"{name}/budget{budget}"], flush=True)
print(json.dumps(out))
