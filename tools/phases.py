"""Per-phase cycle split of the evaluate kernel (instrumented build)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_07297_b200 import _native as N  # noqa: E402

N.LIB_PATH = os.path.join(ROOT, "paper_2210_07297_b200", "libamp_search_phases.so")
lib = N.load(N.LIB_PATH)
lib.amp_debug_phase_cycles.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong)]
from paper_2210_07297_b200 import problem as P  # noqa: E402
from paper_2210_07297_b200.planner import Searcher  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
scen = sys.argv[2] if len(sys.argv) > 2 else "hetero_cluster"
sc = P.load_scenario(os.path.join(ROOT, "tests", "golden", "scenarios", scen + ".json"))
enc = P.EncodedProblem.from_scenario(sc)
Pp = -(-n // (70 if scen != "hetero_model" else 85))
names = ["fetch+decode", "placement", "tables+bw", "DP", "stage/ceiling", "estimate", "record",
         "tail"]
with Searcher(enc, placements_per_class=Pp, seed=0) as s:
    for it in range(2):
        s.run(0, n, k=10)
    st = s.stats()
    out = (C.c_ulonglong * 8)()
    lib.amp_debug_phase_cycles(s.ctx, out)
    tot = sum(out)
    print(f"{n} candidates, kernel {st['kernel_ms']:.3f} ms, ctas {st['ctas']}")
    for nm, v in zip(names, out):
        print(f"  {nm:14s} {100*v/tot:5.1f}%  {v/n:9.0f} cycles/candidate (per CTA)")
