"""Profiling driver: one hetero_cluster sweep run of N candidates through the
C-ABI (used under ncu; never a bench number)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_07297_b200 import problem as P  # noqa: E402
from paper_2210_07297_b200.planner import Searcher  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
scen = sys.argv[2] if len(sys.argv) > 2 else "hetero_cluster"
dense = len(sys.argv) > 3 and sys.argv[3] == "dense"
sc = P.load_scenario(os.path.join(ROOT, "tests", "golden", "scenarios", scen + ".json"))
enc = P.EncodedProblem.from_scenario(sc)
n_cls = 70 if scen != "hetero_model" else 85
Pp = -(-n // n_cls)
with Searcher(enc, placements_per_class=Pp, seed=0, dense_dp=dense) as s:
    for it in range(2):
        t0 = time.perf_counter()
        top, _, _ = s.run(0, n, k=int(os.environ.get("PE_K", "10")))
        st = s.stats()
        print(f"run {it}: {n} candidates in {st['kernel_ms']:.3f} ms kernel, "
              f"{(time.perf_counter()-t0)*1e3:.1f} ms wall, place/dp/est {st['place_ms']:.2f}/{st['dp_ms']:.2f}/{st['est_ms']:.2f} ms, inner={st['dp_inner']:.3e} "
              f"fp64={st['fp64_ops']:.3e} best={(top[0]['total'] if len(top) else None)!r}")
