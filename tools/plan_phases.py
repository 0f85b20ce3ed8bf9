"""plan() phase times (AMP_TIMING=1: host encode / create (+ create phases
on stderr) / run / decode / simulate) for C2 and C4, after a warm-up."""
import os
import sys

os.environ["AMP_TIMING"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import scenario  # noqa: E402
from paper_2210_07297_b200 import planner, problem as P  # noqa: E402

for name in sys.argv[1:] or ["hetero_cluster", "synthetic96"]:
    sc = scenario(name)
    opts = P.PlanOptions(budget=10, cost_options=sc.options.cost_options,
                         max_params_per_device=sc.options.max_params_per_device)
    for it in range(3):
        print(f"== {name} {it}", flush=True)
        planner.plan(sc.model, sc.cluster, sc.profile, sc.gbs, opts,
                     dense_dp=os.environ.get("PLAN_DENSE") == "1")
        sys.stdout.flush()
