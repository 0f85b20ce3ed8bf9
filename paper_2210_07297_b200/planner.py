"""Host API over the C-ABI: the reference's plan() surface, plus the sweep.

`plan()` mirrors parplan::plan (reference proj/src/optimizer.cpp:200-251,
declared optimizer.hpp:74-75): same candidate list, same ranking, same
CandidateRecord/PlanResult shapes and failure texts.  The worker pool +
evaluate_candidate + rank_records region runs on the GPU through
libamp_search.so; the simulator validation of the top `budget` runs on the
device too (the engine's batched simulator, simulator.cpp:75-198).

`Searcher` is the thin object over an amp_ctx for the large placement sweep
 and for multi-GPU sharding.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .problem import (Cluster, EncodedProblem, ModelGraph, PlanOptions, ProfileTable,
                      ValidationError)

RECORD_DTYPE = np.dtype([
    ("index", "<u8"), ("total", "<f8"), ("pipeline_time", "<f8"), ("dpsync_time", "<f8"),
    ("pp", "<i4"), ("dp", "<i4"), ("tmp", "<i4"), ("mbs", "<i4"),
    ("fail_code", "<i4"), ("fail_layer", "<i4"), ("fail_value", "<f8"),
])
assert RECORD_DTYPE.itemsize == 64


def cpp_to_string(v: float) -> str:
    """std::to_string(double) == printf("%f")."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%f" % v


def failure_text(rec, n_layers: int) -> Optional[str]:
    """Rebuild the reference's exception text from a failure code."""
    code = int(rec["fail_code"])
    if code == N.AMP_FAIL_NONE:
        return None
    if code == N.AMP_FAIL_PP_GT_L:  # optimizer.cpp:149-152
        return f"infeasible: pp = {int(rec['pp'])} exceeds layer count {n_layers}"
    if code == N.AMP_FAIL_PROFILE_MISS:  # types.cpp:106-110
        return (f"profile miss: no entry for (layer={int(rec['fail_layer'])}, tmp={int(rec['tmp'])}, "
                f"mbs={int(rec['mbs'])}) and analytic fallback is disabled")
    if code == N.AMP_FAIL_CEILING:  # optimizer.cpp:165-167
        return "exceeds per-device parameter ceiling"
    if code == N.AMP_FAIL_P2P_BANDWIDTH:  # cost_model.cpp:54-59
        return "invalid p2p bandwidth " + cpp_to_string(float(rec["fail_value"]))
    if code == N.AMP_FAIL_ALLREDUCE_BANDWIDTH:  # cost_model.cpp:47-50
        return "invalid bandwidth " + cpp_to_string(float(rec["fail_value"])) + " in all-reduce group"
    return f"unknown failure code {code}"


@dataclass
class Strategy:
    pp: int
    dp: int
    tmp: int
    mbs: int
    placement: List[int] = field(default_factory=list)   # rank -> device id
    cut_boundaries: List[int] = field(default_factory=list)

    @property
    def degrees(self) -> Tuple[int, int, int]:
        return (self.pp, self.dp, self.tmp)

    def device_at(self, stage: int, replica: int, shard: int) -> int:
        """Placement::device_at (types.hpp:117-120)."""
        return self.placement[(stage * self.dp + replica) * self.tmp + shard]


@dataclass
class CostBreakdown:
    pipeline_time: float = 0.0
    dpsync_time: float = 0.0
    total: float = 0.0
    per_stage_times: List[float] = field(default_factory=list)
    per_edge_times: List[float] = field(default_factory=list)


@dataclass
class CandidateRecord:
    strategy: Strategy
    estimated: CostBreakdown
    rank: int = 0
    simulated: Optional[float] = None
    failure: Optional[str] = None
    index: int = 0


@dataclass
class PlanResult:
    candidates: List[CandidateRecord]
    best_index: int = -1
    simulated_all: Optional[List[Optional[float]]] = None  # plan(simulate_all=True)


class Searcher:
    """One amp_ctx: problem tables resident on one GPU."""

    def __init__(self, problem: EncodedProblem, placements_per_class: int = 1, seed: int = 0,
                 device: int = 0, max_ctas: int = 0, dense_dp: bool = False,
                 dedup: bool = True, n_gpus: int = 1):
        self.lib = N.load()
        self.problem = problem
        cfg = N.AmpSearchConfig(int(placements_per_class), int(seed) & (2**64 - 1), int(device),
                                int(max_ctas),
                                (N.AMP_FLAG_DENSE_DP if dense_dp else 0) |
                                (0 if dedup else N.AMP_FLAG_NO_DEDUP), int(n_gpus))
        h = C.c_void_p()
        N.check(self.lib.amp_search_create(C.byref(h), problem.ref(), C.byref(cfg)))
        self.ctx = h
        self.P = int(placements_per_class)
        self.num_candidates = int(self.lib.amp_search_num_candidates(h))
        self.num_classes = int(self.lib.amp_search_num_classes(h))
        self.max_pp = int(self.lib.amp_search_max_pp(h))
        self.n_devices = problem.D
        self.n_layers = problem.L

    # -- queries ---------------------------------------------------------
    def classes(self) -> List[Tuple[int, int, int, int]]:
        out = []
        a, b, c, d = (C.c_int32() for _ in range(4))
        for k in range(self.num_classes):
            N.check(self.lib.amp_search_class(self.ctx, k, C.byref(a), C.byref(b), C.byref(c),
                                              C.byref(d)), self.ctx)
            out.append((a.value, b.value, c.value, d.value))
        return out

    def partition(self, n_parts: int) -> List[int]:
        b = (C.c_uint64 * (n_parts + 1))()
        N.check(self.lib.amp_search_partition(self.ctx, n_parts, b), self.ctx)
        return [int(x) for x in b]

    def stats(self) -> dict:
        s = N.AmpStats()
        N.check(self.lib.amp_search_last_stats(self.ctx, C.byref(s)), self.ctx)
        return {f: getattr(s, f) for f, _ in N.AmpStats._fields_}

    # -- evaluation --------------------------------------------------------
    def _details(self, n: int, details: bool, placement: bool, simulate: bool = False):
        if not (details or placement or simulate):
            return None, None
        mp = self.max_pp
        bufs = {}
        d = N.AmpDetails()
        if details:
            bufs["cuts"] = np.full((n, mp + 1), -1, dtype=np.int32)
            bufs["stage_times"] = np.full((n, mp), np.nan)
            bufs["edge_times"] = np.full((n, mp), np.nan)
            d.cuts = bufs["cuts"].ctypes.data_as(N._ip)
            d.stage_times = bufs["stage_times"].ctypes.data_as(N._dp)
            d.edge_times = bufs["edge_times"].ctypes.data_as(N._dp)
        if placement:
            bufs["placement"] = np.full((n, self.n_devices), -1, dtype=np.int32)
            d.placement = bufs["placement"].ctypes.data_as(N._ip)
        if simulate:  # batched device simulator (simulator.cpp:140-198)
            bufs["simulated"] = np.full(n, np.nan)
            d.simulated = bufs["simulated"].ctypes.data_as(N._dp)
        return d, bufs

    def run(self, begin: int = 0, end: Optional[int] = None, k: int = 10, want_all: bool = False,
            details: bool = False, placement: bool = False, simulate: bool = False):
        """Evaluate [begin, end); returns (topk records, all records | None, detail arrays)."""
        end = self.num_candidates if end is None else int(end)
        n = end - begin
        top = np.zeros(max(k, 1), dtype=RECORD_DTYPE)
        ntop = C.c_int32(0)
        allr = np.zeros(n, dtype=RECORD_DTYPE) if want_all else None
        d, bufs = self._details(n, details and want_all, placement and want_all,
                                simulate and want_all)
        N.check(self.lib.amp_search_run(
            self.ctx, begin, end, k, top.ctypes.data_as(C.POINTER(N.AmpRecord)), C.byref(ntop),
            allr.ctypes.data_as(C.POINTER(N.AmpRecord)) if allr is not None else None,
            C.byref(d) if d is not None else None), self.ctx)
        return top[:ntop.value], allr, bufs or {}

    def evaluate(self, indices: Sequence[int], details: bool = True, placement: bool = True,
                 simulate: bool = False):
        idx = np.ascontiguousarray(indices, dtype=np.uint64)
        n = len(idx)
        out = np.zeros(n, dtype=RECORD_DTYPE)
        d, bufs = self._details(n, details, placement, simulate)
        N.check(self.lib.amp_search_evaluate(
            self.ctx, idx.ctypes.data_as(N._u64p), n, out.ctypes.data_as(C.POINTER(N.AmpRecord)),
            C.byref(d) if d is not None else None), self.ctx)
        return out, bufs or {}

    def estimate(self, indices: Sequence[int], cuts: np.ndarray, details: bool = True,
                 placement: bool = True, simulate: bool = False):
        """Estimate only, with the caller's cuts ([n][max_pp+1]); no DP."""
        idx = np.ascontiguousarray(indices, dtype=np.uint64)
        n = len(idx)
        c = np.full((n, self.max_pp + 1), -1, dtype=np.int32)
        for i, row in enumerate(cuts):
            c[i, :len(row)] = row
        out = np.zeros(n, dtype=RECORD_DTYPE)
        d, bufs = self._details(n, details, placement, simulate)
        N.check(self.lib.amp_search_estimate(
            self.ctx, idx.ctypes.data_as(N._u64p), c.ctypes.data_as(N._ip), n,
            out.ctypes.data_as(C.POINTER(N.AmpRecord)), C.byref(d) if d is not None else None),
            self.ctx)
        return out, bufs or {}

    def evaluate_placed(self, classes: Sequence[int], placements: np.ndarray,
                        cuts: Optional[np.ndarray] = None, details: bool = True,
                        placement: bool = True, simulate: bool = False):
        """Caller placements ([n][|D|]) of classes[i]; DP when cuts is None."""
        ci = np.ascontiguousarray(classes, dtype=np.int32)
        n = len(ci)
        pl = np.ascontiguousarray(placements, dtype=np.int32).reshape(n, self.n_devices)
        cu = None if cuts is None else np.ascontiguousarray(cuts, dtype=np.int32)
        out = np.zeros(n, dtype=RECORD_DTYPE)
        d, bufs = self._details(n, details, placement, simulate)
        N.check(self.lib.amp_search_evaluate_placed(
            self.ctx, ci.ctypes.data_as(N._ip), pl.ctypes.data_as(N._ip),
            cu.ctypes.data_as(N._ip) if cu is not None else None, n,
            out.ctypes.data_as(C.POINTER(N.AmpRecord)), C.byref(d) if d is not None else None),
            self.ctx)
        return out, bufs or {}

    def run_device(self, begin: int, end: int, k: int, d_topk_ptr: int, stream_ptr: int = 0):
        N.check(self.lib.amp_search_run_device(self.ctx, begin, end, k, C.c_void_p(d_topk_ptr),
                                               C.c_void_p(stream_ptr)), self.ctx)

    def run_device_shard(self, shard: int, n_shards: int, k: int, d_topk_ptr: int,
                         stream_ptr: int = 0):
        """Placements [P*shard/n, P*(shard+1)/n) of every class (multi-GPU shard)."""
        N.check(self.lib.amp_search_run_device_shard(self.ctx, shard, n_shards, k,
                                                     C.c_void_p(d_topk_ptr), C.c_void_p(stream_ptr)),
                self.ctx)

    def shard_ranges(self, shard: int, n_shards: int):
        """Index ranges of shard `shard` (the engine's LPT shard plan)."""
        n = C.c_int32()
        N.check(self.lib.amp_search_shard_ranges(self.ctx, shard, n_shards, None, 0, C.byref(n)), self.ctx)
        r = np.zeros(2 * max(1, n.value), dtype=np.uint64)
        N.check(self.lib.amp_search_shard_ranges(self.ctx, shard, n_shards, r.ctypes.data_as(N._u64p),
                                                 n.value, C.byref(n)), self.ctx)
        return [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(n.value)]

    def shard_size(self, shard: int, n_shards: int) -> int:
        return int(self.lib.amp_search_shard_size(self.ctx, shard, n_shards))

    def merge_device(self, d_in_ptr: int, n_in: int, k: int, d_out_ptr: int, stream_ptr: int = 0):
        N.check(self.lib.amp_search_merge_topk_device(self.ctx, C.c_void_p(d_in_ptr), n_in, k,
                                                      C.c_void_p(d_out_ptr), C.c_void_p(stream_ptr)),
                self.ctx)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.amp_search_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def records_to_candidates(recs: np.ndarray, bufs: dict, n_layers: int,
                          rows: Optional[Sequence[int]] = None) -> List[CandidateRecord]:
    out = []
    rows = range(len(recs)) if rows is None else rows
    for i in rows:
        r = recs[i]
        pp, dp, tmp, mbs = int(r["pp"]), int(r["dp"]), int(r["tmp"]), int(r["mbs"])
        fail = failure_text(r, n_layers)
        st = Strategy(pp, dp, tmp, mbs)
        est = CostBreakdown()
        if fail is None:  # (ndarray.tolist: C-speed conversion of the detail rows)
            if "placement" in bufs:
                st.placement = bufs["placement"][i][: pp * dp * tmp].tolist()
            if "cuts" in bufs:
                st.cut_boundaries = bufs["cuts"][i][: pp + 1].tolist()
            est = CostBreakdown(float(r["pipeline_time"]), float(r["dpsync_time"]), float(r["total"]),
                                bufs["stage_times"][i][:pp].tolist() if "stage_times" in bufs else [],
                                bufs["edge_times"][i][:pp - 1].tolist() if "edge_times" in bufs else [])
        out.append(CandidateRecord(st, est, 0, None, fail, int(r["index"])))
    return out


def rank_order(recs: np.ndarray) -> np.ndarray:
    """rank_records key (optimizer.cpp:178-196): (failed, total, index)."""
    failed = (recs["fail_code"] != 0).astype(np.int64)
    total = np.where(failed == 1, 0.0, recs["total"])
    return np.lexsort((recs["index"], total, failed))


def plan(model: ModelGraph, cluster: Cluster, profile: ProfileTable, gbs: int,
         options: Optional[PlanOptions] = None, device: int = 0, dense_dp: bool = False,
         simulate_all: bool = False, n_gpus: int = 1, timing: Optional[dict] = None) -> PlanResult:
    """parplan::plan on the GPU (optimizer.cpp:200-251).  simulate_all: also
    return every candidate's simulated time (result.simulated_all, in rank
    order) — acceptance criterion 5's rank agreement in one pass.  timing:
    a dict filled with the host phase times (s): encode, create, run,
    destroy, decode, simulate."""
    import os
    import time

    tm = timing if timing is not None else ({} if os.environ.get("AMP_TIMING") else None)
    t = time.perf_counter()
    options = options or PlanOptions()
    enc = EncodedProblem(model, cluster, profile, gbs, options)
    if tm is not None:
        tm["encode"] = time.perf_counter() - t
        t = time.perf_counter()
    with Searcher(enc, placements_per_class=1, device=device, dense_dp=dense_dp, n_gpus=n_gpus) as s:
        if tm is not None:
            tm["create"] = time.perf_counter() - t
            t = time.perf_counter()
        # the batched device simulator runs in the same pass (K_est), so the
        # top-`budget` validation needs no host simulation
        _, allr, bufs = s.run(0, s.num_candidates, k=0, want_all=True, details=True, placement=True,
                              simulate=options.budget > 0 or simulate_all)
        if tm is not None:
            tm["run"] = time.perf_counter() - t
            t = time.perf_counter()
    if tm is not None:
        tm["destroy"] = time.perf_counter() - t
        t = time.perf_counter()
    order = rank_order(allr)
    cands = records_to_candidates(allr, bufs, model.layer_count(), rows=order)
    for i, c in enumerate(cands):
        c.rank = i + 1
    result = PlanResult(cands, -1)
    if tm is not None:
        tm["decode"] = time.perf_counter() - t
        t = time.perf_counter()
    # validate the top `budget` with the simulator (optimizer.cpp:235-249):
    # values from the device simulator (bit-identical to simulate(),
    # tests/test_gpu_parity.py); best_index is the first strict minimum in
    # rank order, as in the reference's sequential loop
    sims = bufs.get("simulated")
    for i in range(min(len(cands), max(0, options.budget))):
        if cands[i].failure is not None:
            continue
        v = float(sims[order[i]])
        cands[i].simulated = v
        if result.best_index < 0 or v < cands[result.best_index].simulated:
            result.best_index = i
    if simulate_all and sims is not None:
        result.simulated_all = [None if c.failure is not None else float(sims[order[i]])
                                for i, c in enumerate(cands)]
    if tm is not None:
        tm["simulate"] = time.perf_counter() - t
        if timing is None:
            print("plan timing (ms):", {k: round(v * 1e3, 3) for k, v in tm.items()})
    return result
