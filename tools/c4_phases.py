"""C4 plan() phase breakdown (run on a GPU box with AMP_TIMING=1 for the
create-internal phases): python tools/c4_phases.py [reps] [n_gpus]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07297_b200 import planner, problem as P  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n_gpus = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sc = P.synthetic_c4()
for r in range(reps):
    tm = {}
    t = time.perf_counter()
    res = planner.plan(sc.model, sc.cluster, sc.profile, sc.gbs, sc.options, timing=tm, n_gpus=n_gpus)
    print(f"n_gpus {n_gpus} rep {r}: total {1e3 * (time.perf_counter() - t):.2f} ms",
          {k: round(1e3 * v, 3) for k, v in tm.items()}, flush=True)
