"""Debug helper: one |D| = 1024 sweep (tests/test_gpu_parity.py LARGE_D) on cuda:0."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_07297_b200 import planner, problem as P  # noqa: E402

nodes, per, P_ = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (128, 8, 3)))
sc = P.synthetic_cluster(nodes, per, 24, 1024, 64)
enc = P.EncodedProblem.from_scenario(sc)
with planner.Searcher(enc, placements_per_class=P_, seed=5) as s:
    top, allr, _ = s.run(0, s.num_candidates, k=10, want_all=True, details=False)
    print(s.stats())
