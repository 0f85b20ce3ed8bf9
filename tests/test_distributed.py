"""Multi-process exchange of the sharded search on CPU (gloo, world_size 2):
each rank evaluates its index range (oracle evaluator), the k best records
are all-gathered and merged; the result must equal the single-process top-k
for any split (output identical for any n_gpus)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, scenario


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, bounds, k, out_path):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from conftest import scenario as sc_
    from oracle import bindings as B
    from paper_2210_07297_b200 import distributed as Dd
    from paper_2210_07297_b200 import problem as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = sc_("hetero_model")
    enc = P.EncodedProblem.from_scenario(sc)
    o = B.Oracle(enc, placements_per_class=6, seed=9)

    def evaluate(lo, hi):
        recs, _ = o.run(lo, hi, threads=2, details=False)
        return recs

    top = Dd.search_host(evaluate, k, bounds, rank, world)
    if rank == 0:
        np.save(out_path, top)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("split", ["even", "skewed", "lpt", "lpt-p1"])
def test_gloo_two_rank_merge_matches_single_process(tmp_path, split):
    from oracle import bindings as B
    from paper_2210_07297_b200 import distributed as Dd
    from paper_2210_07297_b200 import problem as P

    sc = scenario("hetero_model")
    enc = P.EncodedProblem.from_scenario(sc)
    o = B.Oracle(enc, placements_per_class=6, seed=9)
    n = o.num_candidates
    recs, _ = o.run(0, n, threads=4, details=False)
    k = 12
    want = Dd.merge_topk_host(recs, k)
    if split == "lpt":  # the engine's shard plan (amp_search_run_device_shard), uneven weights
        w = [1.0 + (c % 7) * 3.5 for c in range(n // 6)]
        bounds = Dd.lpt_shards(w, 6, 2)
    elif split == "lpt-p1":  # P = 1 would be pure LPT over classes: blocks of one placement
        w = [float((c * 37) % 11 + 1) for c in range(n)]
        bounds = Dd.lpt_shards(w, 1, 2)
    else:
        bounds = [0, n // 2, n] if split == "even" else [0, 37, n]
    out = str(tmp_path / "top.npy")
    mp.spawn(_worker, args=(2, _free_port(), bounds, k, out), nprocs=2, join=True)
    got = np.load(out)
    assert got["index"].tolist() == want["index"].tolist()
    assert np.array_equal(got["total"], want["total"])


def test_lpt_shards_cover_space_and_balance():
    """The shard plan covers every index exactly once for any (P, n) and
    balances the shards within the largest block, also for uneven
    single-placement classes (P = 1: the C4 plan() case)."""
    from paper_2210_07297_b200 import distributed as Dd
    for n_cls, P_, n in [(70, 100, 8), (440, 1, 8), (35, 3, 4), (5, 1, 8), (12, 7, 3)]:
        w = [float((c * 2654435761) % 1000 + 1) for c in range(n_cls)]
        plan = Dd.lpt_shards(w, P_, n)
        seen = np.zeros(n_cls * P_, dtype=np.int32)
        for rngs in plan:
            for lo, hi in rngs:
                seen[lo:hi] += 1
        assert (seen == 1).all()
        loads = [sum(w[lo // P_] * (hi - lo) for lo, hi in r) for r in plan]
        assert max(loads) - min(loads) <= max(w) * -(-P_ // n) + 1e-9  # greedy: <= the largest block


def test_signature_disjoint_shards():
    """The signature-disjoint plan (P >= n, enough pp <= 2 work): every DP
    class lies in exactly one shard (no signature is solved twice), every
    index is covered once, and the per-candidate load (2 per DP-class
    candidate, 1 otherwise) is balanced within one pp <= 2 block."""
    from paper_2210_07297_b200 import distributed as Dd
    for n_cls, n_heavy, P_, n in [(70, 32, 1000, 4), (70, 32, 1000, 8), (40, 6, 64, 2), (20, 2, 9, 3)]:
        heavy = [c >= n_cls - n_heavy for c in range(n_cls)]
        w = [float(c) for c in range(n_cls)]
        plan = Dd.lpt_shards(w, P_, n, heavy)
        seen = np.zeros(n_cls * P_, dtype=np.int32)
        owner = {}
        for r, rngs in enumerate(plan):
            for lo, hi in rngs:
                seen[lo:hi] += 1
                c = lo // P_
                assert (hi - 1) // P_ == c
                if heavy[c]:
                    assert c not in owner
                    owner[c] = r
                    assert hi - lo == P_
        assert (seen == 1).all() and len(owner) == n_heavy
        loads = [sum((2.0 if heavy[lo // P_] else 1.0) * (hi - lo) for lo, hi in r) for r in plan]
        assert max(loads) - min(loads) <= -(-P_ // n) + 1e-9
    # not enough pp <= 2 work: the block plan (every class in min(P, n) blocks)
    plan = Dd.lpt_shards([1.0] * 10, 100, 4, [c < 8 for c in range(10)])
    assert sum(len(r) for r in plan) == 40
