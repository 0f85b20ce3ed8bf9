"""Simulator validation of plan()'s top `budget` (optimizer.cpp:235-249),
through the engine's host simulator (amp_simulate, restating
reference proj/src/simulator.cpp:140-198)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .problem import Cluster, CostModelOptions, EncodedProblem, ModelGraph, PlanOptions, ProfileTable


def simulate(strategy, model: ModelGraph, cluster: Cluster, profile: ProfileTable, gbs: int,
             cost_options: CostModelOptions, encoded: EncodedProblem = None) -> float:
    lib = N.load()
    enc = encoded or EncodedProblem(model, cluster, profile, gbs, PlanOptions(cost_options=cost_options))
    place = np.ascontiguousarray(strategy.placement, dtype=np.int32)
    cuts = np.ascontiguousarray(strategy.cut_boundaries, dtype=np.int32)
    out = C.c_double(0.0)
    st = lib.amp_simulate(enc.ref(), strategy.pp, strategy.dp, strategy.tmp, strategy.mbs,
                          place.ctypes.data_as(N._ip), cuts.ctypes.data_as(N._ip), C.byref(out))
    if st != N.AMP_OK:
        raise N.AmpError(st, "cannot simulate an invalid strategy")
    return out.value


def rank_correlation(estimates, simulated) -> float:
    """Spearman rank correlation with average ranks for ties (reference
    simulator.cpp:200-258, same summation order)."""
    import math
    if len(estimates) != len(simulated):
        raise ValueError("rank correlation needs equally sized inputs")
    n = len(estimates)
    if n < 3:
        raise ValueError("rank correlation needs at least 3 samples")

    def average_ranks(values):
        order = sorted(range(n), key=lambda i: values[i])
        ranks = [0.0] * n
        i = 0
        while i < n:
            j = i
            while j + 1 < n and values[order[j + 1]] == values[order[i]]:
                j += 1
            rank = (float(i) + float(j)) / 2.0 + 1.0
            for k in range(i, j + 1):
                ranks[order[k]] = rank
            i = j + 1
        return ranks

    rx, ry = average_ranks(list(estimates)), average_ranks(list(simulated))
    mx = my = 0.0
    for i in range(n):
        mx += rx[i]
        my += ry[i]
    mx /= float(n)
    my /= float(n)
    cov = vx = vy = 0.0
    for i in range(n):
        cov += (rx[i] - mx) * (ry[i] - my)
        vx += (rx[i] - mx) * (rx[i] - mx)
        vy += (ry[i] - my) * (ry[i] - my)
    if vx == 0.0 or vy == 0.0:
        return 0.0
    return cov / math.sqrt(vx * vy)
