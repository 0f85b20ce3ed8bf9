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
