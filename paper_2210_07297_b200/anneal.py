"""Annealing search (reference placement.cpp:299-398, the paper's
Algorithm 2) on the engine.

The chain runs in the library (amp_anneal.cpp): the reference's
mt19937_64 draws, domino tilings, temperatures and acceptances, bit for
bit, with every proposal's layer-partition DP and estimate on the GPU.  The
top `budget` states are validated with the device simulator, as the
reference CLI does (parplan_main.cpp:219-240).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from .planner import CostBreakdown, RECORD_DTYPE, Searcher, Strategy, failure_text
from .problem import (Cluster, CostModelOptions, EncodedProblem, ModelGraph, PlanOptions,
                      ProfileTable, ValidationError)


class ProfileMissError(ValidationError):
    """ProfileMissError of the reference (types.hpp:163-178)."""


@dataclass
class AnnealOptions:  # placement.hpp:76-87
    iterations: int = 200
    seed: int = 0
    budget: int = 10
    initial_temperature: float = 1.0
    cooling: float = 0.97
    min_temperature: float = 1e-3
    record_all: bool = False
    neighbor_retries: int = 20
    cost_options: CostModelOptions = field(default_factory=CostModelOptions)


@dataclass
class AnnealEntry:  # placement.hpp:89-94
    strategy: Strategy
    estimated: CostBreakdown
    iteration: int = 0
    accepted: bool = True
    simulated: Optional[float] = None


@dataclass
class AnnealResult:  # placement.hpp:96-104
    top: List[AnnealEntry]
    record: List[AnnealEntry]
    initial_cost: float = 0.0
    best_cost: float = 0.0


def anneal(model: ModelGraph, cluster: Cluster, profile: ProfileTable, gbs: int,
           options: Optional[AnnealOptions] = None, device: int = 0,
           simulate_top: bool = True) -> AnnealResult:
    o = options or AnnealOptions()
    if o.iterations < 1:
        raise ValidationError("anneal needs at least one iteration")
    enc = EncodedProblem(model, cluster, profile, gbs, PlanOptions(cost_options=o.cost_options))
    cap = o.iterations + 1
    with Searcher(enc, placements_per_class=1, device=device) as s:
        D, mp = s.n_devices, s.max_pp
        cfg = N.AmpAnnealConfig(o.iterations, o.budget, o.seed, o.initial_temperature, o.cooling,
                                o.min_temperature, int(o.record_all), o.neighbor_retries)
        rec = (N.AmpAnnealEntry * cap)()
        place = np.full((cap, D), -1, dtype=np.int32)
        cuts = np.full((cap, mp + 1), -1, dtype=np.int32)
        top = np.zeros(max(1, o.budget), dtype=np.int32)
        n_rec, n_top = C.c_int32(0), C.c_int32(0)
        init = C.c_double(0.0)
        failed = N.AmpRecord()
        st = s.lib.amp_search_anneal(s.ctx, enc.ref(), C.byref(cfg), rec,
                                     place.ctypes.data_as(N._ip), cuts.ctypes.data_as(N._ip), cap,
                                     C.byref(n_rec), top.ctypes.data_as(N._ip), C.byref(n_top),
                                     C.byref(init), C.byref(failed))
        if st == N.AMP_E_CANDIDATE:
            r = np.frombuffer(bytes(failed), dtype=RECORD_DTYPE)[0]
            msg = failure_text(r, model.layer_count())
            if int(r["fail_code"]) == N.AMP_FAIL_PROFILE_MISS:
                raise ProfileMissError(msg)
            raise ValidationError(msg)
        N.check(st, s.ctx)
        entries = []
        for i in range(n_rec.value):
            e = rec[i]
            r = e.estimated
            stg = Strategy(r.pp, r.dp, r.tmp, r.mbs, [int(x) for x in place[i][: r.pp * r.dp * r.tmp]],
                           [int(x) for x in cuts[i][: r.pp + 1]])
            entries.append(AnnealEntry(stg, CostBreakdown(r.pipeline_time, r.dpsync_time, r.total),
                                       int(e.iteration), bool(e.accepted)))
        tops = [entries[int(i)] for i in top[: n_top.value]]
        if simulate_top and tops:  # device simulator, caller placements and cuts
            cls = {s.classes()[c]: c for c in range(len(s.classes()))}
            ci = np.array([cls[(t.strategy.pp, t.strategy.dp, t.strategy.tmp, t.strategy.mbs)]
                           for t in tops], dtype=np.int32)
            pl = np.array([t.strategy.placement for t in tops], dtype=np.int32)
            cu = np.full((len(tops), mp + 1), -1, dtype=np.int32)
            for j, t in enumerate(tops):
                cu[j, : len(t.strategy.cut_boundaries)] = t.strategy.cut_boundaries
            _, bufs = s.evaluate_placed(ci, pl, cu, details=False, placement=False, simulate=True)
            for t, v in zip(tops, bufs["simulated"]):
                t.simulated = float(v)
    best = tops[0].estimated.total if tops else init.value
    return AnnealResult(tops, entries, float(init.value), float(best))
