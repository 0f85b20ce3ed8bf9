"""Multi-GPU search: one process per GPU, candidates sharded across ranks.

SURVEY.md §8(e): candidates are independent, so each rank evaluates its own
part of the class-major index space and keeps its local top-k on the
device.  Two splits: the LPT shard plan (`search_gpu_sharded`,
amp_search_run_device_shard, mirrored by `lpt_shards`: every class cut into
min(P, n) placement blocks weighted by its work, longest first to the
least-loaded rank — with P >= n and enough pp <= 2 work the DP classes stay
whole, so the ranks solve disjoint signatures and the pp <= 2 blocks balance
the load; with P = 1 an LPT split of the plan() DP instances) and the
contiguous work-weighted index range (`search_gpu`, amp_search_partition).
The only
exchange is one all-gather of the k records per rank (NCCL over NVLink on
GPUs, gloo in the CPU tests) followed by a deterministic merge under the
reference ranking key (failed, total, index) — identical for any world size.

`search()` is written against two small hooks so the exchange logic is the
same with the CUDA engine and with the CPU oracle used by the gloo tests.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import numpy as np

from .planner import RECORD_DTYPE, rank_order


def merge_topk_host(records: np.ndarray, k: int) -> np.ndarray:
    """Host merge under the rank_records key; drops empty slots."""
    records = records[records["fail_code"] >= 0]
    return records[rank_order(records)[:k]]


def shard_bounds(n_total: int, world: int, weights: Optional[Sequence[int]] = None) -> List[int]:
    """Equal-count contiguous split (the engine's amp_search_partition gives
    the work-weighted one)."""
    if weights is not None:
        return list(weights)
    return [n_total * r // world for r in range(world + 1)]


def search_gpu(searcher, k: int, bounds: Sequence[int], rank: int, world: int, group=None):
    """Evaluate this rank's slice on the GPU; all-gather the device top-k
    (NCCL) and merge on the device.  Returns the global top-k (host)."""
    import torch
    import torch.distributed as dist

    stream = torch.cuda.current_stream()
    local = torch.empty(k * RECORD_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    searcher.run_device(bounds[rank], bounds[rank + 1], k, local.data_ptr(), stream.cuda_stream)
    if world == 1:
        out = local
    else:
        gathered = torch.empty(world * k * RECORD_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        dist.all_gather_into_tensor(gathered, local, group=group)
        out = torch.empty_like(local)
        searcher.merge_device(gathered.data_ptr(), world * k, k, out.data_ptr(), stream.cuda_stream)
    recs = np.frombuffer(out.cpu().numpy().tobytes(), dtype=RECORD_DTYPE)
    return recs[recs["fail_code"] >= 0]


def search_gpu_sharded(searcher, k: int, rank: int, world: int, group=None):
    """Evaluate this rank's per-class placement slice on the GPU, all-gather
    the device top-k (NCCL) and merge on the device.  Returns the global
    top-k (host)."""
    import torch
    import torch.distributed as dist

    stream = torch.cuda.current_stream()
    local = torch.empty(k * RECORD_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    searcher.run_device_shard(rank, world, k, local.data_ptr(), stream.cuda_stream)
    if world == 1:
        out = local
    else:
        gathered = torch.empty(world * k * RECORD_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        dist.all_gather_into_tensor(gathered, local, group=group)
        out = torch.empty_like(local)
        searcher.merge_device(gathered.data_ptr(), world * k, k, out.data_ptr(), stream.cuda_stream)
    recs = np.frombuffer(out.cpu().numpy().tobytes(), dtype=RECORD_DTYPE)
    return recs[recs["fail_code"] >= 0]


def lpt_shards(class_weights: Sequence[float], P: int, n_shards: int,
               heavy: Optional[Sequence[bool]] = None) -> List[List[tuple]]:
    """The shard plan of amp_search_run_device_shard (amp_search.cu
    shard_plan): each class c cut into min(P, n) placement blocks of weight
    class_weights[c] * size, blocks longest-first (stable) to the
    least-loaded shard (lowest on ties).  With `heavy` (the DP classes,
    pp >= 3) the signature-disjoint variant applies when n > 1, P >= n and
    the pp <= 2 candidates are at least n times the largest DP class's
    doubled size: every DP class is one unit of weight 2 * P (dealt first,
    the largest class_weights first), the others min(P, n) blocks of weight
    1 * size.  Returns each shard's index ranges (in assignment order; the
    engine dispatches them heaviest class first)."""
    nb = min(P, n_shards)
    disjoint = False
    if heavy is not None and n_shards > 1 and P >= n_shards and any(heavy):
        light = sum(P for h in heavy if not h)
        disjoint = light >= 2.0 * P * n_shards
    units = []
    for c, wc in enumerate(class_weights):
        whole = disjoint and heavy[c]
        nbc = 1 if whole else nb
        key = (1e12 + wc) if whole else (1.0 if disjoint else wc)
        for b in range(nbc):
            p0, p1 = P * b // nbc, P * (b + 1) // nbc
            if p1 > p0:
                wu = (2.0 if whole else 1.0) if disjoint else wc
                units.append((wu * (p1 - p0), key, c, p0, p1))
    # longest first by the class weight, a class's blocks adjacent (stable)
    units.sort(key=lambda u: -u[1])
    load = [0.0] * n_shards
    out: List[List[tuple]] = [[] for _ in range(n_shards)]
    for w, _, c, p0, p1 in units:
        s = min(range(n_shards), key=lambda r: (load[r], r))
        load[s] += w
        out[s].append((c * P + p0, c * P + p1))
    return out


def search_host(evaluate: Callable[[int, int], np.ndarray], k: int, bounds: Sequence[int], rank: int,
                world: int, group=None) -> np.ndarray:
    """Same exchange with a host evaluator (tests / gloo): each rank ranks its
    slice, all-gathers k fixed-size records and merges."""
    import torch
    import torch.distributed as dist

    if isinstance(bounds[0], (list, tuple)):  # a list of ranges per rank (class slices)
        parts = [evaluate(lo, hi) for lo, hi in bounds[rank]]
        recs = np.concatenate(parts) if parts else np.zeros(0, dtype=RECORD_DTYPE)
    else:
        recs = evaluate(bounds[rank], bounds[rank + 1])
    local = np.zeros(k, dtype=RECORD_DTYPE)
    local["fail_code"] = -1
    local["index"] = np.iinfo(np.uint64).max
    top = merge_topk_host(recs, k)
    local[: len(top)] = top
    t = torch.from_numpy(np.frombuffer(local.tobytes(), dtype=np.uint8).copy())
    if world == 1:
        return merge_topk_host(local, k)
    out = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(out, t, group=group)
    allr = np.frombuffer(b"".join(o.numpy().tobytes() for o in out), dtype=RECORD_DTYPE)
    return merge_topk_host(allr, k)
