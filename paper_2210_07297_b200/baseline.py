"""Megatron-style baseline on the B200 engine.

Mirrors the reference's `megatron_baseline` (optimizer.cpp:253-279):
* one candidate per micro-batch size in divisors(gbs);
* degrees from `megatron_degree_choice` (optimizer.cpp:64-79);
* heuristic placement;
* cuts from `uniform_assignment` (81-95) or `param_balance_assignment`
  (97-123), computed on the host (integer work plus one cumulative-sum
  comparison);
* costs from the engine's estimate-only path `amp_search_estimate`
  (K_place -> K_est, no DP), then `rank_records`.

The candidate index is the plan() class index: the context has
placements_per_class = 1, so p = 0 is the heuristic placement.
"""
from __future__ import annotations

from typing import List, Optional, Tuple

import numpy as np

from .planner import CandidateRecord, Searcher, rank_order, records_to_candidates
from .problem import (Cluster, CostModelOptions, EncodedProblem, ModelGraph, PlanOptions,
                      ProfileTable, ValidationError, candidate_classes, divisors, enumerate_degrees)

LAYER_BALANCE = "layer-balance"
PARAM_BALANCE = "param-balance"


def min_node_size(cluster: Cluster) -> int:
    """Cluster::min_node_size (types.cpp:52-58)."""
    sizes = {}
    for d in cluster.devices:
        sizes[d.node_id] = sizes.get(d.node_id, 0) + 1
    return min([cluster.device_count()] + list(sizes.values()))


def megatron_degree_choice(cluster: Cluster, gbs: int, mbs: int,
                           layer_count: int) -> Optional[Tuple[int, int, int]]:
    """optimizer.cpp:64-79: the smallest (tmp*pp, tmp) among the feasible
    degrees (tmp within the smallest node, pp <= L, gbs/dp divisible by mbs);
    the first one wins ties, in enumerate_degrees order."""
    best = None
    mn = min_node_size(cluster)
    for pp, dp, tmp in enumerate_degrees(cluster.device_count()):
        if tmp > mn or pp > layer_count:
            continue
        if gbs % dp != 0 or (gbs // dp) % mbs != 0:
            continue
        if best is None or (tmp * pp, tmp) < (best[2] * best[0], best[2]):
            best = (pp, dp, tmp)
    return best


def uniform_assignment(layer_count: int, stages: int) -> List[int]:
    """optimizer.cpp:81-95"""
    if stages < 1 or stages > layer_count:
        raise ValidationError(f"infeasible: cannot split {layer_count} layers into {stages} "
                              "non-empty stages")
    base, extra = divmod(layer_count, stages)
    cuts, nxt = [], 0
    for j in range(stages):
        cuts.append(nxt)
        nxt += base + (1 if j < extra else 0)
    cuts.append(layer_count)
    return cuts


def param_balance_assignment(model: ModelGraph, stages: int) -> List[int]:
    """optimizer.cpp:97-123: cut j at the boundary whose cumulative parameter
    count is closest to total*j/stages (the first one on ties), keeping every
    stage non-empty."""
    L = model.layer_count()
    if stages < 1 or stages > L:
        raise ValidationError(f"infeasible: cannot split {L} layers into {stages} "
                              "non-empty stages")
    cum = [0.0] * (L + 1)
    for i in range(L):
        cum[i + 1] = cum[i] + float(model.layers[i].param_count)
    cuts = [0]
    for j in range(1, stages):
        target = cum[L] * j / stages
        lo, hi = cuts[-1] + 1, L - (stages - j)
        best = lo
        for c in range(lo, hi + 1):
            if abs(cum[c] - target) < abs(cum[best] - target):
                best = c
        cuts.append(best)
    cuts.append(L)
    return cuts


def megatron_baseline(model: ModelGraph, cluster: Cluster, profile: ProfileTable, gbs: int,
                      mode: str = LAYER_BALANCE, cost_options: Optional[CostModelOptions] = None,
                      device: int = 0) -> List[CandidateRecord]:
    """optimizer.cpp:253-279 through amp_search_estimate; ranked."""
    opts = PlanOptions(cost_options=cost_options or CostModelOptions())
    enc = EncodedProblem(model, cluster, profile, gbs, opts)
    cls_index = {c: i for i, c in enumerate(candidate_classes(cluster.device_count(), gbs))}
    idx, cuts = [], []
    for mbs in divisors(gbs):
        deg = megatron_degree_choice(cluster, gbs, mbs, model.layer_count())
        if deg is None:
            continue
        pp, dp, tmp = deg
        idx.append(cls_index[(pp, dp, tmp, mbs)])
        cuts.append(uniform_assignment(model.layer_count(), pp) if mode == LAYER_BALANCE
                    else param_balance_assignment(model, pp))
    if not idx:
        return []
    with Searcher(enc, placements_per_class=1, device=device) as s:
        recs, bufs = s.estimate(idx, cuts, details=True, placement=True)
    order = rank_order(recs)
    cands = records_to_candidates(recs, bufs, model.layer_count(), rows=order)
    for i, c in enumerate(cands):
        c.rank = i + 1
    return cands
