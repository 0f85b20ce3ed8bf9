"""Phase timing of one end-to-end search through the public API (the bench's
e2e leg): amp_search_create (AMP_TIMING phases), run to a host top-k, destroy."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_07297_b200 import problem as P  # noqa: E402
from paper_2210_07297_b200.planner import Searcher  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
sc = P.load_scenario(os.path.join(ROOT, "tests", "golden", "scenarios", "hetero_cluster.json"))
enc = P.EncodedProblem.from_scenario(sc)
Pp = -(-n // 70)
for it in range(4):
    t0 = time.perf_counter()
    s = Searcher(enc, placements_per_class=Pp, seed=0)
    t1 = time.perf_counter()
    top, _, _ = s.run(0, s.num_candidates, k=10)
    t2 = time.perf_counter()
    st = s.stats()
    s.close()
    t3 = time.perf_counter()
    print(f"iter {it}: create {1e3*(t1-t0):.2f} ms  run {1e3*(t2-t1):.2f} ms (device {st['total_ms']:.2f})"
          f"  destroy {1e3*(t3-t2):.2f} ms  total {1e3*(t3-t0):.2f} ms", flush=True)
