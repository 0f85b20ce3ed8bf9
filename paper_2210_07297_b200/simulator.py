"""Rank agreement of the estimate with the simulator (acceptance criterion 5).

The simulator itself (reference proj/src/simulator.cpp:75-198) runs on the
device, batched, inside the engine's estimate kernel (amp_pipeline.cuh
sim_iteration; `Searcher.run(..., details=True)` / planner.plan's top-`budget`
validation).  This module keeps the Spearman statistic the acceptance check
applies to it.
"""
from __future__ import annotations


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
