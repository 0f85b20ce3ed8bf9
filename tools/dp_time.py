"""Experiment helper: K_dp stage / span times of the bench sweep (1e8
candidates, hetero_cluster) under the current environment switches; never a
bench number (no L2 flush, no clocks check)."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_07297_b200 import problem as P  # noqa: E402
from paper_2210_07297_b200.planner import Searcher  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000000
sc = P.load_scenario(os.path.join(ROOT, "tests", "golden", "scenarios", "hetero_cluster.json"))
enc = P.EncodedProblem.from_scenario(sc)
with Searcher(enc, placements_per_class=-(-n // 70), seed=0) as s:
    st, best = [], None
    for it in range(6):
        top, _, _ = s.run(0, n, k=10)
        st.append(s.stats())
        best = (int(top[0]["index"]), float(top[0]["total"]))
    st = st[1:]
    med = lambda k: statistics.median(x[k] for x in st)  # noqa: E731
    frac = med("fp64_ops") / (med("dp_stage_ms") * 1e-3) / 18.5e12
    print(f"{os.environ.get('TAG', '')}: stage {med('dp_stage_ms'):.3f} ms span {med('dp_ms'):.3f} "
          f"est {med('est_ms'):.3f} place {med('place_ms'):.3f} total {med('kernel_ms'):.3f} "
          f"frac {frac:.3f} best {best}")
