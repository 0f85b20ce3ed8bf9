"""ctypes bindings of the oracle — TEST INFRASTRUCTURE ONLY.

  liboracle.so          plain-C restatement (oracle/amp_oracle.c)
  _ref/libparplan_ref.so the reference library itself (oracle/ref_bridge.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's CPU arm import this.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_2210_07297_b200 import _native as N  # noqa: E402  (struct layouts only)
from paper_2210_07297_b200.planner import RECORD_DTYPE  # noqa: E402

ORACLE_PATH = os.path.join(_HERE, "liboracle.so")
REF_PATH = os.path.join(_HERE, "_ref", "libparplan_ref.so")

_dp, _ip, _u64p = N._dp, N._ip, N._u64p
_recp = C.POINTER(N.AmpRecord)
_i64p = C.POINTER(C.c_int64)

_oracle = None
_ref = None


def load_oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_PATH)
        sig = {
            "oracle_create": (C.c_void_p, [C.POINTER(N.AmpProblem), C.c_uint64, C.c_uint64]),
            "oracle_destroy": (None, [C.c_void_p]),
            "oracle_num_candidates": (C.c_uint64, [C.c_void_p]),
            "oracle_num_classes": (C.c_int32, [C.c_void_p]),
            "oracle_max_pp": (C.c_int32, [C.c_void_p]),
            "oracle_class": (C.c_int, [C.c_void_p, C.c_int32, _ip, _ip, _ip, _ip]),
            "oracle_layer_time": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, _dp]),
            "oracle_optimal_assignment": (C.c_int, [_dp, C.c_int32, C.c_int32, C.c_int32, _dp, _ip, _dp,
                                                    _ip, _dp]),
            "oracle_tolerance_domain": (C.c_int32, [_dp, C.c_int32, _dp]),
            "oracle_placement": (None, [C.c_void_p, C.c_uint64, _ip]),
            "oracle_evaluate": (None, [C.c_void_p, C.c_uint64, _recp, _ip, _dp, _dp]),
            "oracle_run": (None, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int32, _recp, _ip, _dp, _dp]),
            "oracle_run_memo": (None, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int32, _recp, _ip, _dp, _dp]),
            "oracle_rank": (None, [_recp, C.c_int64, _i64p]),
            "oracle_splitmix64": (C.c_uint64, [C.c_uint64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def load_ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_PATH)
        sig = {
            "ref_plan": (C.c_int, [C.POINTER(N.AmpProblem), C.c_int32, C.c_int32, _recp, _ip, _dp, _dp, _dp,
                                   _ip, C.c_char_p, C.c_int32, C.c_int32]),
            "ref_num_classes": (C.c_int, [C.POINTER(N.AmpProblem)]),
            "ref_sweep": (C.c_int, [C.POINTER(N.AmpProblem), C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                    C.c_int32, _recp, _ip, _dp, _dp, C.c_char_p, C.c_int32, C.c_int32]),
            "ref_sweep_indices": (C.c_int, [C.POINTER(N.AmpProblem), C.c_uint64, C.c_uint64, _u64p, C.c_int64,
                                            C.c_int32, _recp, C.c_int32]),
            "ref_optimal_assignment": (C.c_int, [_dp, C.c_int32, C.c_int32, C.c_int32, _dp, _ip, _dp]),
            "ref_anneal": (C.c_int, [C.POINTER(N.AmpProblem), C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                     _dp, _dp, _ip]),
            "ref_brute_force": (C.c_int, [_dp, C.c_int32, C.c_int32, C.c_int32, _dp, _ip, _dp]),
            "ref_tolerance_domain": (C.c_int, [_dp, C.c_int32, _dp]),
            "ref_estimate": (C.c_int, [C.POINTER(N.AmpProblem), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       _ip, _ip, _dp, _dp, _dp, _dp, _dp, C.c_char_p, C.c_int32]),
            "ref_simulate": (C.c_int, [C.POINTER(N.AmpProblem), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       _ip, _ip, _dp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _ref = lib
    return _ref


def _recs(n):
    a = np.zeros(n, dtype=RECORD_DTYPE)
    return a, a.ctypes.data_as(_recp)


# --------------------------------------------------------------------------
# plain-C oracle
# --------------------------------------------------------------------------

class Oracle:
    def __init__(self, enc, placements_per_class: int = 1, seed: int = 0):
        self.lib = load_oracle()
        self.enc = enc
        self.h = self.lib.oracle_create(enc.ref(), placements_per_class, seed & (2**64 - 1))
        if not self.h:
            raise ValueError("oracle_create failed")
        self.num_candidates = int(self.lib.oracle_num_candidates(self.h))
        self.num_classes = int(self.lib.oracle_num_classes(self.h))
        self.max_pp = int(self.lib.oracle_max_pp(self.h))

    def classes(self):
        out = []
        a, b, c, d = (C.c_int32() for _ in range(4))
        for k in range(self.num_classes):
            self.lib.oracle_class(self.h, k, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
            out.append((a.value, b.value, c.value, d.value))
        return out

    def run(self, begin=0, end=None, threads=1, details=True, memo=False):
        """Evaluate [begin, end); memo=True memoises the DP per worker by
        (class, boundary bandwidths) — identical outputs, for large N."""
        end = self.num_candidates if end is None else end
        n = end - begin
        recs, rp = _recs(n)
        mp = self.max_pp
        cuts = np.full((n, mp + 1), -1, dtype=np.int32) if details else None
        st = np.full((n, mp), np.nan) if details else None
        ed = np.full((n, mp), np.nan) if details else None
        fn = self.lib.oracle_run_memo if memo else self.lib.oracle_run
        fn(self.h, begin, end, threads, rp,
                            cuts.ctypes.data_as(_ip) if details else None,
                            st.ctypes.data_as(_dp) if details else None,
                            ed.ctypes.data_as(_dp) if details else None)
        return recs, {"cuts": cuts, "stage_times": st, "edge_times": ed} if details else {}

    def placement(self, index: int):
        out = np.zeros(self.enc.D, dtype=np.int32)
        self.lib.oracle_placement(self.h, index, out.ctypes.data_as(_ip))
        return out

    def close(self):
        if self.h:
            self.lib.oracle_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def oracle_dp(times, k, gas, edges):
    lib = load_oracle()
    t = np.ascontiguousarray(times, dtype=np.float64)
    e = np.ascontiguousarray(edges if len(edges) else [0.0], dtype=np.float64)
    cuts = np.zeros(k + 1, dtype=np.int32)
    cost = C.c_double()
    M = C.c_int32()
    inner = C.c_double()
    st = lib.oracle_optimal_assignment(t.ctypes.data_as(_dp), len(t), k, gas, e.ctypes.data_as(_dp),
                                       cuts.ctypes.data_as(_ip), C.byref(cost), C.byref(M), C.byref(inner))
    if st:
        raise ValueError("invalid DP instance")
    return cuts.tolist(), cost.value, M.value, inner.value


def oracle_rank(recs):
    lib = load_oracle()
    order = np.zeros(len(recs), dtype=np.int64)
    lib.oracle_rank(recs.ctypes.data_as(_recp), len(recs), order.ctypes.data_as(_i64p))
    return order


# --------------------------------------------------------------------------
# the reference itself
# --------------------------------------------------------------------------

def ref_plan(enc, max_pp: int, budget: int = 0, workers: int = 0, n_max: int = 100000):
    lib = load_ref()
    recs, rp = _recs(n_max)
    cuts = np.full((n_max, max_pp + 1), -1, dtype=np.int32)
    st = np.full((n_max, max_pp), np.nan)
    ed = np.full((n_max, max_pp), np.nan)
    sim = np.full(n_max, np.nan)
    best = C.c_int32(-1)
    stride = 160
    text = C.create_string_buffer(n_max * stride)
    n = lib.ref_plan(enc.ref(), budget, workers, rp, cuts.ctypes.data_as(_ip), st.ctypes.data_as(_dp),
                     ed.ctypes.data_as(_dp), sim.ctypes.data_as(_dp), C.byref(best), text, stride, max_pp)
    if n < 0:
        raise RuntimeError("ref_plan failed")
    texts = [text.raw[i * stride:(i + 1) * stride].split(b"\0", 1)[0].decode() for i in range(n)]
    return {"records": recs[:n], "cuts": cuts[:n], "stage_times": st[:n], "edge_times": ed[:n],
            "simulated": sim[:n], "best_index": best.value, "failures": texts}


def ref_sweep(enc, P, seed, begin, end, threads, max_pp, details=True, texts=False):
    lib = load_ref()
    n = end - begin
    recs, rp = _recs(n)
    cuts = np.full((n, max_pp + 1), -1, dtype=np.int32) if details else None
    st = np.full((n, max_pp), np.nan) if details else None
    ed = np.full((n, max_pp), np.nan) if details else None
    stride = 160 if texts else 0
    text = C.create_string_buffer(max(1, n * stride))
    rc = lib.ref_sweep(enc.ref(), P, seed & (2**64 - 1), begin, end, threads, rp,
                       cuts.ctypes.data_as(_ip) if details else None,
                       st.ctypes.data_as(_dp) if details else None,
                       ed.ctypes.data_as(_dp) if details else None,
                       text if texts else None, stride, max_pp)
    if rc:
        raise RuntimeError("ref_sweep failed")
    out = {"records": recs, "cuts": cuts, "stage_times": st, "edge_times": ed}
    if texts:
        out["failures"] = [text.raw[i * stride:(i + 1) * stride].split(b"\0", 1)[0].decode()
                           for i in range(n)]
    return out


def ref_sweep_indices(enc, P, seed, indices, threads, max_pp):
    lib = load_ref()
    idx = np.ascontiguousarray(indices, dtype=np.uint64)
    recs, rp = _recs(len(idx))
    if lib.ref_sweep_indices(enc.ref(), P, seed & (2**64 - 1), idx.ctypes.data_as(_u64p), len(idx), threads,
                             rp, max_pp):
        raise RuntimeError("ref_sweep_indices failed")
    return recs


def ref_dp(times, k, gas, edges, brute=False):
    lib = load_ref()
    t = np.ascontiguousarray(times, dtype=np.float64)
    e = np.ascontiguousarray(edges if len(edges) else [0.0], dtype=np.float64)
    cuts = np.zeros(k + 1, dtype=np.int32)
    cost = C.c_double()
    fn = lib.ref_brute_force if brute else lib.ref_optimal_assignment
    if fn(t.ctypes.data_as(_dp), len(t), k, gas, e.ctypes.data_as(_dp), cuts.ctypes.data_as(_ip),
          C.byref(cost)):
        raise ValueError("reference refused the instance")
    return cuts.tolist(), cost.value


def ref_simulate(enc, pp, dp, tmp, mbs, placement, cuts):
    lib = load_ref()
    pl = np.ascontiguousarray(placement, dtype=np.int32)
    cu = np.ascontiguousarray(cuts, dtype=np.int32)
    out = C.c_double()
    if lib.ref_simulate(enc.ref(), pp, dp, tmp, mbs, pl.ctypes.data_as(_ip), cu.ctypes.data_as(_ip),
                        C.byref(out)):
        raise ValueError("invalid strategy")
    return out.value


def ref_anneal(enc, iterations: int, seed: int, budget: int = 10, record_all: bool = False):
    """The reference anneal chain (parplan::anneal): (initial cost, best cost,
    recorded states)."""
    lib = load_ref()
    ic, bc, nr = C.c_double(), C.c_double(), C.c_int32()
    if lib.ref_anneal(enc.ref(), iterations, seed & (2**64 - 1), budget, int(record_all), C.byref(ic),
                      C.byref(bc), C.byref(nr)):
        raise RuntimeError("ref_anneal failed")
    return ic.value, bc.value, nr.value
