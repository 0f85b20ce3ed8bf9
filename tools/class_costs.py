"""Per-class device time of the sweep's kernels (K_place / K_dp / K_est
events) — which (pp, dp, tmp) shapes the step's time goes to."""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_07297_b200 import problem as P  # noqa: E402
from paper_2210_07297_b200.planner import Searcher  # noqa: E402
from oracle import bindings as B  # noqa: E402

sc = P.load_scenario(os.path.join(ROOT, "tests", "golden", "scenarios", "hetero_cluster.json"))
enc = P.EncodedProblem.from_scenario(sc)
Pp = 1428572
cls = B.Oracle(enc, 1, 0).classes()
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0])
with Searcher(enc, placements_per_class=Pp, seed=0) as s:
    for c in range(len(cls)):
        for it in range(2):
            s.run(c * Pp, (c + 1) * Pp, k=10)
            st = s.stats()
        a = agg[cls[c][:3]]
        a[0] += st["place_ms"]
        a[1] += st["dp_ms"]
        a[2] += st["est_ms"]
        a[3] += 1
tot = [sum(v[i] for v in agg.values()) for i in range(3)]
print(f"total place/dp/est {tot[0]:.2f}/{tot[1]:.2f}/{tot[2]:.2f} ms (classes run one at a time)")
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][0] + kv[1][1] + kv[1][2])):
    print(f"(pp,dp,tmp)={k}  classes {v[3]}  place {v[0]:.3f}  dp {v[1]:.3f}  est {v[2]:.3f} ms")
