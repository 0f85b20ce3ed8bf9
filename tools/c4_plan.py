"""One plan() of the synthetic 96-layer / 1024-GPU scenario (C4), for ncu."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import scenario  # noqa: E402
from paper_2210_07297_b200 import planner, problem as P  # noqa: E402

sc = scenario("synthetic96")
res = planner.plan(sc.model, sc.cluster, sc.profile, sc.gbs,
                   P.PlanOptions(budget=0, cost_options=sc.options.cost_options))
print("best", res.candidates[0].strategy.degrees, res.candidates[0].estimated.total)
