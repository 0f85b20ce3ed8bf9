"""Debug helper: one sweep run (scenario, P, seed) on cuda:0, printing stats
and (optionally, P small) the record comparison with the memoised oracle.
  python tools/dbg_run.py hetero_cluster 30000 6 [--oracle]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07297_b200 import planner, problem as P  # noqa: E402

name, P_, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
K = int(os.environ.get("DBG_K", "10"))
sc = P.synthetic_c4() if name == "synthetic96" else P.load_scenario(
    os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                 "scenarios", name + ".json"))
enc = P.EncodedProblem.from_scenario(sc)
with planner.Searcher(enc, placements_per_class=P_, seed=seed) as s:
    want_all = "--oracle" in sys.argv
    top, allr, _ = s.run(0, s.num_candidates, k=K, want_all=want_all, details=False)
    st = s.stats()
print({k: st[k] for k in ("dp_instances", "dp_inner", "dp_ms", "dp_stage_ms", "dp_stage_launches",
                          "dp_fallback", "place_ms", "est_ms", "total_ms")})
print("top", [(int(r["index"]), float(r["total"])) for r in top[:3]])
if want_all:
    from oracle import bindings as B
    o = B.Oracle(enc, P_, seed)
    orec, _ = o.run(threads=os.cpu_count() or 8, details=False, memo=True)
    ok = orec["fail_code"] == 0
    bad = np.nonzero((allr["fail_code"] != orec["fail_code"]) |
                     (ok & (allr["total"] != orec["total"])))[0]
    print("mismatches", len(bad), bad[:10])
