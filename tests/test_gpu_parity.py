"""GPU parity: the CUDA engine (through the C-ABI) vs the reference's golden
vectors and the oracle, bit-exact for every index, degree, placement, cut
and fp64 cost (the declared tolerance is 1e-9 relative; exact ties in the
real configs make bit-exactness necessary for identical ranking)."""
import ctypes as C

import numpy as np
import pytest

from conftest import hexf, load_json, scenario
from oracle import bindings as B
from paper_2210_07297_b200 import _native as N
from paper_2210_07297_b200 import planner, problem as P

pytestmark = pytest.mark.gpu

DP_FILES = ["dp_kat.json", "dp_seed31.json", "dp_seed37.json", "dp_seed101.json", "dp_large.json"]


def gpu_dp_batch(instances):
    lib = N.load()
    n = len(instances)
    keep = []
    arr = (N.AmpDpInstance * n)()
    stride = max(i["k"] for i in instances) + 1
    for j, inst in enumerate(instances):
        t = np.ascontiguousarray([hexf(x) for x in inst["times"]], dtype=np.float64)
        e = np.ascontiguousarray([hexf(x) for x in inst["edges"]] or [0.0], dtype=np.float64)
        keep += [t, e]
        arr[j] = N.AmpDpInstance(inst["L"], inst["k"], inst["gas"], 0, t.ctypes.data_as(N._dp),
                                 e.ctypes.data_as(N._dp))
    cuts = np.zeros((n, stride), dtype=np.int32)
    cost = np.zeros(n)
    status = np.zeros(n, dtype=np.int32)
    N.check(lib.amp_dp_solve_batch(0, arr, n, cuts.ctypes.data_as(N._ip), stride,
                                   cost.ctypes.data_as(N._dp), status.ctypes.data_as(N._ip)))
    return cuts, cost, status


@pytest.mark.parametrize("fname", DP_FILES)
def test_gpu_dp_matches_reference(fname):
    inst = load_json(fname)["instances"]
    cuts, cost, status = gpu_dp_batch(inst)
    for j, i in enumerate(inst):
        assert status[j] == 0
        assert cuts[j][: i["k"] + 1].tolist() == i["cuts"], i["name"]
        assert cost[j] == hexf(i["cost"]), i["name"]


def test_gpu_dp_invalid_instances_flagged():
    lib = N.load()
    t = np.ones(3)
    arr = (N.AmpDpInstance * 2)()
    arr[0] = N.AmpDpInstance(3, 4, 1, 0, t.ctypes.data_as(N._dp), t.ctypes.data_as(N._dp))  # k > L
    arr[1] = N.AmpDpInstance(3, 1, 0, 0, t.ctypes.data_as(N._dp), None)  # gas < 1
    cuts = np.zeros((2, 5), dtype=np.int32)
    cost = np.zeros(2)
    status = np.zeros(2, dtype=np.int32)
    N.check(lib.amp_dp_solve_batch(0, arr, 2, cuts.ctypes.data_as(N._ip), 5,
                                   cost.ctypes.data_as(N._dp), status.ctypes.data_as(N._ip)))
    assert status.tolist() == [1, 1]


def check_plan_against_golden(res, golden):
    cands = golden["candidates"]
    assert len(res.candidates) == len(cands)
    for c, g in zip(res.candidates, cands):
        s = c.strategy
        assert c.rank == g["rank"]
        assert c.index == g["index"]
        assert [s.pp, s.dp, s.tmp] == g["degrees"] and s.mbs == g["mbs"]
        assert c.failure == g["failure"]
        if g["failure"]:
            continue
        assert c.estimated.total == hexf(g["total"])
        assert c.estimated.pipeline_time == hexf(g["pipeline_time"])
        assert c.estimated.dpsync_time == hexf(g["dpsync_time"])
        assert s.cut_boundaries == g["cuts"]
        assert c.estimated.per_stage_times == [hexf(x) for x in g["per_stage_times"]]
        assert c.estimated.per_edge_times == [hexf(x) for x in g["per_edge_times"]]
        if g.get("simulated") is not None:
            assert c.simulated == hexf(g["simulated"])
        else:
            assert c.simulated is None
    assert res.best_index == golden["best_index"]


@pytest.mark.parametrize("dense", [False, True], ids=["pruned", "dense"])
@pytest.mark.parametrize("name", ["homogeneous", "hetero_cluster", "hetero_model", "synthetic96"])
def test_gpu_plan_matches_reference(name, dense):
    sc = scenario(name)
    golden = load_json(f"plan_{name}.json")
    res = planner.plan(sc.model, sc.cluster, sc.profile, sc.gbs, sc.options, dense_dp=dense)
    check_plan_against_golden(res, golden)


def test_heuristic_placement_matches_reference_order():
    sc = scenario("hetero_cluster")
    enc = P.EncodedProblem.from_scenario(sc)
    with planner.Searcher(enc) as s:
        recs, bufs = s.evaluate(list(range(s.num_candidates)))
    assert (bufs["placement"] == np.arange(16)).all()


@pytest.mark.parametrize("dense", [False, True], ids=["pruned", "dense"])
@pytest.mark.parametrize("name", ["hetero_cluster", "hetero_model"])
def test_gpu_sweep_matches_reference(name, dense):
    g = load_json(f"sweep_{name}.json")
    sc = scenario(name)
    enc = P.EncodedProblem.from_scenario(sc)
    with planner.Searcher(enc, placements_per_class=g["placements_per_class"], seed=g["seed"],
                          dense_dp=dense) as s:
        top, allr, bufs = s.run(0, g["n"], k=10, want_all=True, details=True)
    for i, e in enumerate(g["records"]):
        r = allr[i]
        assert int(r["index"]) == e["index"]
        assert int(r["fail_code"]) == e["fail_code"]
        if e["fail_code"] == 0:
            assert r["total"] == hexf(e["total"]), i
            assert bufs["cuts"][i][: int(r["pp"]) + 1].tolist() == e["cuts"], i
    order = planner.rank_order(allr)[:10]
    assert top["index"].tolist() == allr["index"][order].tolist()


@pytest.mark.parametrize("dense", [False, True], ids=["pruned", "dense"])
@pytest.mark.parametrize("kind", ["plain", "miss", "ceiling", "fallback"])
def test_gpu_failure_paths_match_oracle(kind, dense):
    from test_oracle import _variant_world
    model, cl, prof, gbs, opts = _variant_world(kind)
    enc = P.EncodedProblem(model, cl, prof, gbs, opts)
    o = B.Oracle(enc, placements_per_class=5, seed=11)
    orec, odet = o.run(threads=4)
    with planner.Searcher(enc, placements_per_class=5, seed=11, dense_dp=dense) as s:
        _, allr, bufs = s.run(0, s.num_candidates, k=5, want_all=True, details=True)
    for f in ("index", "pp", "dp", "tmp", "mbs", "fail_code"):
        assert np.array_equal(allr[f], orec[f]), f
    ok = orec["fail_code"] == 0
    for f in ("total", "pipeline_time", "dpsync_time"):
        assert np.array_equal(allr[f][ok], orec[f][ok]), f
    assert np.array_equal(bufs["cuts"][ok], odet["cuts"][ok])
    assert np.array_equal(bufs["stage_times"][ok], odet["stage_times"][ok], equal_nan=True)
    ed_ok = ~np.isnan(odet["edge_times"])
    assert np.array_equal(bufs["edge_times"][ed_ok], odet["edge_times"][ed_ok])
    miss = orec["fail_code"] == 2
    assert np.array_equal(allr["fail_layer"][miss], orec["fail_layer"][miss])
    if B.ref_available():
        ref = B.ref_sweep(enc, 5, 11, 0, len(orec), 4, s.max_pp, details=False, texts=True)
        texts = [planner.failure_text(r, model.layer_count()) or "" for r in allr]
        assert texts == ref["failures"]


def test_gpu_sweep_topk_and_sample_vs_oracle():
    """N = 2e5 hetero_cluster sweep: the GPU top-k equals the oracle's
    evaluation of the same indices, and a seeded random sample of indices is
    bit-equal (BASELINE.md §3 large-N parity)."""
    sc = scenario("hetero_cluster")
    enc = P.EncodedProblem.from_scenario(sc)
    P_ = 2000
    with planner.Searcher(enc, placements_per_class=P_, seed=0) as s:
        top, _, _ = s.run(0, 70 * P_, k=20)
        rng = np.random.default_rng(7)
        sample = np.unique(rng.integers(0, 70 * P_, 300).astype(np.uint64))
        srec, _ = s.evaluate(sample, details=False, placement=False)
    o = B.Oracle(enc, P_, 0)
    for idx, r in zip(sample, srec):
        rec = np.zeros(1, dtype=planner.RECORD_DTYPE)
        o.lib.oracle_evaluate(o.h, int(idx), rec.ctypes.data_as(B._recp), None, None, None)
        assert rec[0]["total"] == r["total"] or (rec[0]["fail_code"] and r["fail_code"])
    # the top-k totals must be exactly the oracle's values for those indices,
    # and no sampled candidate may beat the k-th entry
    for r in top:
        rec = np.zeros(1, dtype=planner.RECORD_DTYPE)
        o.lib.oracle_evaluate(o.h, int(r["index"]), rec.ctypes.data_as(B._recp), None, None, None)
        assert rec[0]["total"] == r["total"]
    kth = top[-1]
    for r in srec:
        if r["fail_code"] == 0:
            assert (r["total"], r["index"]) >= (kth["total"], kth["index"]) or \
                r["index"] in top["index"]
    assert np.all(np.diff(top["total"]) >= 0)


def test_run_device_merge_and_partition_invariance():
    """Sharded runs (work-weighted partition) merged on device give the same
    global top-k as one run — the multi-GPU exchange contract."""
    import torch
    sc = scenario("hetero_model")
    enc = P.EncodedProblem.from_scenario(sc)
    P_ = 300
    k = 16
    with planner.Searcher(enc, placements_per_class=P_, seed=3) as s:
        N_ = s.num_candidates
        whole, _, _ = s.run(0, N_, k=k)
        bounds = s.partition(4)
        assert bounds[0] == 0 and bounds[-1] == N_ and bounds == sorted(bounds)
        parts = torch.empty((4, k * 64), dtype=torch.uint8, device="cuda")
        for i in range(4):
            s.run_device(bounds[i], bounds[i + 1], k, parts[i].data_ptr(),
                         torch.cuda.current_stream().cuda_stream)
        out = torch.empty(k * 64, dtype=torch.uint8, device="cuda")
        s.merge_device(parts.data_ptr(), 4 * k, k, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        merged = np.frombuffer(out.cpu().numpy().tobytes(), dtype=planner.RECORD_DTYPE)
    assert merged["index"].tolist() == whole["index"].tolist()
    assert np.array_equal(merged["total"], whole["total"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,P_,n_shards", [("hetero_cluster", 101, 2), ("hetero_cluster", 101, 3),
                                              ("hetero_cluster", 101, 8), ("synthetic96", 1, 2),
                                              ("synthetic96", 1, 4), ("synthetic96", 1, 8)])
def test_lpt_shards_merge_to_single_run(name, P_, n_shards):
    """The LPT shard plan (amp_search_run_device_shard, the multi-GPU split;
    with P = 1 the C4 plan() space's 440 uneven DP instances) covers the
    space exactly once and the shards' device top-k lists merge to the
    single-run top-k."""
    import torch
    sc = scenario(name)
    enc = P.EncodedProblem.from_scenario(sc)
    k = 12
    with planner.Searcher(enc, placements_per_class=P_, seed=5) as s:
        N_ = s.num_candidates
        whole, _, _ = s.run(0, N_, k=k)
        assert sum(s.shard_size(r, n_shards) for r in range(n_shards)) == N_
        seen = np.zeros(N_, dtype=np.int32)
        for r in range(n_shards):
            for lo, hi in s.shard_ranges(r, n_shards):
                seen[lo:hi] += 1
        assert (seen == 1).all()
        st = torch.cuda.current_stream().cuda_stream
        parts = torch.empty((n_shards, k * 64), dtype=torch.uint8, device="cuda")
        for r in range(n_shards):
            s.run_device_shard(r, n_shards, k, parts[r].data_ptr(), st)
        out = torch.empty(k * 64, dtype=torch.uint8, device="cuda")
        s.merge_device(parts.data_ptr(), n_shards * k, k, out.data_ptr(), st)
        torch.cuda.synchronize()
        merged = np.frombuffer(out.cpu().numpy().tobytes(), dtype=planner.RECORD_DTYPE)
    assert merged["index"].tolist() == whole["index"].tolist()
    assert np.array_equal(merged["total"], whole["total"])


@pytest.mark.parametrize("name,P_", [("homogeneous", 1), ("hetero_cluster", 1), ("hetero_model", 1),
                                     ("hetero_cluster", 40), ("synthetic96", 1)])
def test_batched_simulator_matches_reference_simulate(name, P_):
    """the device simulator (amp_details.simulated, K_est)
    equals the reference simulate() (simulator.cpp:140-198, oracle/_ref)
    bit for bit on every candidate — the plan() spaces, shuffled placements,
    and C4's pp up to 64 (the > 32-stage path)."""
    if not B.ref_available():
        pytest.skip("oracle/_ref not built")
    sc = scenario(name)
    enc = P.EncodedProblem.from_scenario(sc)
    with planner.Searcher(enc, placements_per_class=P_, seed=7) as s:
        n = s.num_candidates
        idx = np.arange(n) if n <= 3000 else np.random.default_rng(3).choice(n, 3000, replace=False)
        recs, bufs = s.evaluate(idx, details=True, placement=True, simulate=True)
    checked = 0
    for i in range(len(idx)):
        r = recs[i]
        if r["fail_code"] != 0:
            assert np.isnan(bufs["simulated"][i])
            continue
        pp, dp, tmp, mbs = int(r["pp"]), int(r["dp"]), int(r["tmp"]), int(r["mbs"])
        ref = B.ref_simulate(enc, pp, dp, tmp, mbs, bufs["placement"][i][: pp * dp * tmp],
                             bufs["cuts"][i][: pp + 1])
        assert bufs["simulated"][i] == ref, (name, i, pp, dp, tmp, mbs)
        checked += 1
    assert checked > 0


@pytest.mark.parametrize("name", ["homogeneous", "hetero_cluster", "hetero_model"])
def test_acceptance_rank_agreement_one_pass(name):
    """acceptance_main.cpp:236-267 (criterion 5): Spearman(estimate,
    simulation) over every feasible candidate >= 0.5, here from one plan()
    pass with the device simulator; the simulated values equal the
    reference's simulate() on the reference's own plan() strategies."""
    if not B.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2210_07297_b200 import simulator
    sc = scenario(name)
    enc = P.EncodedProblem.from_scenario(sc)
    res = planner.plan(sc.model, sc.cluster, sc.profile, sc.gbs, P.PlanOptions(budget=1),
                       simulate_all=True)
    est, sim = [], []
    for c, v in zip(res.candidates, res.simulated_all):
        if c.failure is not None:
            continue
        s = c.strategy
        assert v == B.ref_simulate(enc, s.pp, s.dp, s.tmp, s.mbs, s.placement, s.cut_boundaries)
        est.append(c.estimated.total)
        sim.append(v)
    rho = simulator.rank_correlation(est, sim)
    assert len(est) >= 20 and rho >= 0.5


@pytest.mark.parametrize("name", ["hetero_cluster", "hetero_model", "homogeneous"])
def test_memoised_dp_equals_per_candidate_dp(name):
    """DP memoisation by signature (amp_dedup.cuh) changes no output: every
    record and every cut of a shuffled-placement sweep equals the
    one-DP-per-candidate run (AMP_FLAG_NO_DEDUP), and the top-k matches."""
    sc = scenario(name)
    enc = P.EncodedProblem.from_scenario(sc)
    outs = []
    for dedup in (True, False):
        with planner.Searcher(enc, placements_per_class=3000, seed=11, dedup=dedup) as s:
            top, allr, bufs = s.run(0, s.num_candidates, k=20, want_all=True, details=True)
            st = s.stats()
        outs.append((top, allr, bufs["cuts"], st))
    (t1, a1, c1, s1), (t2, a2, c2, s2) = outs
    assert np.array_equal(a1.view(np.uint8), a2.view(np.uint8))
    assert np.array_equal(c1, c2)
    assert t1["index"].tolist() == t2["index"].tolist()
    assert s1["dp_instances"] < s2["dp_instances"]  # memoisation did skip repeats


@pytest.mark.parametrize("name", ["hetero_cluster", "hetero_model"])
def test_thread_and_warp_kernels_agree(name, monkeypatch):
    """Thread-per-candidate K_place/K_est (amp_thread.cuh, |D| <= 16) and the
    warp-per-candidate kernels produce identical records, cuts, edges,
    placements and top-k on a shuffled sweep."""
    sc = scenario(name)
    enc = P.EncodedProblem.from_scenario(sc)
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("AMP_NO_THREAD", env)
        else:
            monkeypatch.delenv("AMP_NO_THREAD", raising=False)
        with planner.Searcher(enc, placements_per_class=700, seed=13) as s:
            top, allr, bufs = s.run(0, s.num_candidates, k=24, want_all=True, details=True,
                                    placement=True)
        outs.append((top, allr, bufs))
    (t1, a1, b1), (t2, a2, b2) = outs
    assert np.array_equal(a1.view(np.uint8), a2.view(np.uint8))
    for key in ("cuts", "stage_times", "edge_times", "placement"):
        assert np.array_equal(b1[key], b2[key], equal_nan=True), key
    assert t1.view(np.uint8).tobytes() == t2.view(np.uint8).tobytes()


def test_full_sweep_1m_equals_memoised_oracle():
    """SURVEY §8(d) large-N parity: a 1.05 M-candidate hetero_cluster sweep
    (the bench scenario and seed, its production path: thread kernels,
    signature memoisation, prefix-shared DP) equals the full-N memoised CPU
    oracle record for record, and the device top-k is the oracle's ranking."""
    import os
    sc = scenario("hetero_cluster")
    enc = P.EncodedProblem.from_scenario(sc)
    P_ = 15000
    with planner.Searcher(enc, placements_per_class=P_, seed=0) as s:
        top, allr, _ = s.run(0, s.num_candidates, k=32, want_all=True, details=False)
        n = s.num_candidates
    o = B.Oracle(enc, P_, 0)
    orec, _ = o.run(threads=os.cpu_count() or 4, details=False, memo=True)
    assert len(orec) == n == 70 * P_
    for f in ("index", "pp", "dp", "tmp", "mbs", "fail_code"):
        assert np.array_equal(allr[f], orec[f]), f
    ok = orec["fail_code"] == 0
    assert ok.sum() > n // 2
    for f in ("total", "pipeline_time", "dpsync_time"):
        assert np.array_equal(allr[f][ok], orec[f][ok]), f
    order = B.oracle_rank(orec)
    assert top["index"].tolist() == orec["index"][order[:32]].tolist()


@pytest.mark.parametrize("name", ["hetero_cluster", "hetero_model", "homogeneous"])
def test_shape_kernels_equal_generic_estimate(name, monkeypatch):
    """K_est_t's unrolled per-shape estimate (est_shape, records-only runs)
    equals the generic body (AMP_NO_SHAPE=1) record for record, top-k too."""
    sc = scenario(name)
    enc = P.EncodedProblem.from_scenario(sc)
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("AMP_NO_SHAPE", env)
        else:
            monkeypatch.delenv("AMP_NO_SHAPE", raising=False)
        with planner.Searcher(enc, placements_per_class=2000, seed=5) as s:
            top, allr, _ = s.run(0, s.num_candidates, k=24, want_all=True, details=False)
        outs.append((top, allr))
    (t1, a1), (t2, a2) = outs
    assert np.array_equal(a1.view(np.uint8), a2.view(np.uint8))
    assert np.array_equal(t1.view(np.uint8), t2.view(np.uint8))


@pytest.mark.parametrize("kind", ["plain", "miss", "ceiling", "fallback"])
def test_records_only_failure_paths_match_oracle(kind):
    """Records-only runs (the shape kernels where they apply) on the failure
    variants equal the oracle field by field."""
    from test_oracle import _variant_world
    model, cl, prof, gbs, opts = _variant_world(kind)
    enc = P.EncodedProblem(model, cl, prof, gbs, opts)
    o = B.Oracle(enc, placements_per_class=7, seed=3)
    orec, _ = o.run(threads=4, details=False)
    with planner.Searcher(enc, placements_per_class=7, seed=3) as s:
        top, allr, _ = s.run(0, s.num_candidates, k=5, want_all=True, details=False)
    for f in ("index", "pp", "dp", "tmp", "mbs", "fail_code", "fail_layer", "fail_value"):
        assert np.array_equal(allr[f], orec[f]), f
    ok = orec["fail_code"] == 0
    for f in ("total", "pipeline_time", "dpsync_time"):
        assert np.array_equal(allr[f][ok], orec[f][ok]), f
    assert top["index"].tolist() == orec["index"][B.oracle_rank(orec)[:5]].tolist()


def test_sweep_1e9_topk_and_sample_vs_oracle():
    """SURVEY §8(d) parity at N > 1e6: a 10^9-candidate hetero_cluster sweep
    (16 chunks through the production path) — every top-k entry equals the
    oracle's evaluation of that index, the top-k is sorted under the rank
    key, and 20,000 seeded random indices evaluated on the device are
    bit-equal to the oracle with none beating the k-th entry."""
    sc = scenario("hetero_cluster")
    enc = P.EncodedProblem.from_scenario(sc)
    n = 10 ** 9
    P_ = -(-n // 70)
    k = 32
    with planner.Searcher(enc, placements_per_class=P_, seed=0) as s:
        top, _, _ = s.run(0, n, k=k)
        rng = np.random.default_rng(2022)
        sample = np.unique(rng.integers(0, n, 20000).astype(np.uint64))
        srec, _ = s.evaluate(sample, details=False, placement=False)
    o = B.Oracle(enc, P_, 0)

    def oracle_rec(i):
        rec = np.zeros(1, dtype=planner.RECORD_DTYPE)
        o.lib.oracle_evaluate(o.h, int(i), rec.ctypes.data_as(B._recp), None, None, None)
        return rec[0]

    assert len(top) == k
    for r in top:
        e = oracle_rec(r["index"])
        assert int(e["fail_code"]) == int(r["fail_code"]) == 0
        assert e["total"] == r["total"] and e["pipeline_time"] == r["pipeline_time"]
    key = [(float(r["total"]), int(r["index"])) for r in top]
    assert key == sorted(key)
    kth = key[-1]
    for i, r in zip(sample, srec):
        e = oracle_rec(i)
        assert int(e["fail_code"]) == int(r["fail_code"]), int(i)
        if e["fail_code"] == 0:
            assert e["total"] == r["total"], int(i)
            assert (float(r["total"]), int(i)) >= kth or int(i) in set(top["index"].tolist())


def test_light_tail_overlap_equals_single_stream(monkeypatch):
    """The opt-in light-tail overlap (AMP_OVERLAP=1: the pp <= 2 items' K_est
    on a second stream with its own CTA lists) gives the same top-k and
    records as the single-stream run."""
    sc = scenario("hetero_cluster")
    enc = P.EncodedProblem.from_scenario(sc)
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("AMP_OVERLAP", env)
        else:
            monkeypatch.delenv("AMP_OVERLAP", raising=False)
        with planner.Searcher(enc, placements_per_class=3000, seed=9) as s:
            top, allr, _ = s.run(0, s.num_candidates, k=40, want_all=True, details=False)
        outs.append((top, allr))
    assert np.array_equal(outs[0][0].view(np.uint8), outs[1][0].view(np.uint8))
    assert np.array_equal(outs[0][1].view(np.uint8), outs[1][1].view(np.uint8))


@pytest.mark.parametrize("name", ["hetero_cluster", "hetero_model"])
def test_multi_chunk_equals_single_chunk(name, monkeypatch):
    """A sweep cut into many chunks (AMP_CHUNK: per-chunk hash epochs, CTA
    top-k lists persisted across launches, pure-light chunks) gives the same
    records and top-k as one chunk."""
    sc = scenario(name)
    enc = P.EncodedProblem.from_scenario(sc)
    outs = []
    for chunk in (None, "700000"):
        if chunk:
            monkeypatch.setenv("AMP_CHUNK", chunk)
        else:
            monkeypatch.delenv("AMP_CHUNK", raising=False)
        with planner.Searcher(enc, placements_per_class=60000, seed=4) as s:
            top, allr, _ = s.run(0, s.num_candidates, k=16, want_all=True, details=False)
        outs.append((top, allr))
    assert len(outs[1][1]) > 4 * 700000
    assert np.array_equal(outs[0][0].view(np.uint8), outs[1][0].view(np.uint8))
    assert np.array_equal(outs[0][1].view(np.uint8), outs[1][1].view(np.uint8))


@pytest.mark.parametrize("ceiling", [None, 1.5e8, 5e7])
def test_run_pipe_with_parameter_ceiling_matches_oracle(ceiling, monkeypatch):
    """The per-run estimate of dp == 1 classes (k_run_pipe) and the shape
    kernels under a per-device parameter ceiling (some candidates fail it):
    records equal the oracle and the AMP_NO_RUN_PIPE=1 run, 16 devices."""
    sc = scenario("hetero_cluster")
    opts = P.PlanOptions(cost_options=sc.options.cost_options, max_params_per_device=ceiling)
    enc = P.EncodedProblem(sc.model, sc.cluster, sc.profile, sc.gbs, opts)
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("AMP_NO_RUN_PIPE", env)
        else:
            monkeypatch.delenv("AMP_NO_RUN_PIPE", raising=False)
        with planner.Searcher(enc, placements_per_class=400, seed=21) as s:
            top, allr, _ = s.run(0, s.num_candidates, k=12, want_all=True, details=False)
        outs.append((top, allr))
    assert np.array_equal(outs[0][1].view(np.uint8), outs[1][1].view(np.uint8))
    assert np.array_equal(outs[0][0].view(np.uint8), outs[1][0].view(np.uint8))
    o = B.Oracle(enc, 400, 21)
    orec, _ = o.run(threads=8, details=False, memo=True)
    allr = outs[0][1]
    for f in ("index", "fail_code"):
        assert np.array_equal(allr[f], orec[f]), f
    ok = orec["fail_code"] == 0
    assert np.array_equal(allr["total"][ok], orec["total"][ok])
    if ceiling is not None:
        assert (orec["fail_code"] == 3).any() and ok.any()  # AMP_FAIL_CEILING, some pass


SWITCHES = [
    ("AMP_NO_TRIE", "1"),          # signature-mode K_dp (k_dp_multi over the keys)
    ("AMP_TRIE_VCAP", "20000"),    # trie capacity exceeded on the device -> same fallback
    ("AMP_NO_FUSE", "1"),          # K_place places the pp <= 2 tail too
    ("AMP_NO_FUSE_HASH", "1"),     # separate k_hash_insert launch
    ("AMP_NO_RUN_SLOT", "1"),      # k_hash_scatter + rep_of lookup in K_est
    ("AMP_KEEP_WORK", "1"),        # K_place writes work records, K_est reads them
    ("AMP_WIDE_MEMO", "1"),        # hashed signature keys (the |D| = 1024 path), verified
    ("AMP_TRIE_LEVELS", "1"),      # level-by-level trie build instead of the sorted-key build
]


@pytest.mark.parametrize("var,val", SWITCHES)
def test_switch_paths_equal_default(var, val, monkeypatch):
    """Every comparison switch of the engine gives records and
    a top-k identical to the default path, across chunks (AMP_CHUNK), and the
    records equal the memoised oracle."""
    sc = scenario("hetero_cluster")
    enc = P.EncodedProblem.from_scenario(sc)
    outs = []
    monkeypatch.setenv("AMP_CHUNK", "1000000")
    for env in (None, val):
        if env:
            monkeypatch.setenv(var, env)
        else:
            monkeypatch.delenv(var, raising=False)
        with planner.Searcher(enc, placements_per_class=30000, seed=6) as s:
            top, allr, _ = s.run(0, s.num_candidates, k=16, want_all=True, details=False)
            st = s.stats()
        outs.append((top, allr, st))
    monkeypatch.delenv(var, raising=False)
    assert np.array_equal(outs[0][1].view(np.uint8), outs[1][1].view(np.uint8))
    assert np.array_equal(outs[0][0].view(np.uint8), outs[1][0].view(np.uint8))
    assert outs[0][2]["dp_fallback"] == 0
    if var == "AMP_TRIE_VCAP":
        assert outs[1][2]["dp_fallback"] > 0
    o = B.Oracle(enc, 30000, 6)
    orec, _ = o.run(threads=8, details=False, memo=True)
    allr = outs[0][1]
    assert np.array_equal(allr["fail_code"], orec["fail_code"])
    ok = orec["fail_code"] == 0
    assert np.array_equal(allr["total"][ok], orec["total"][ok])


@pytest.mark.parametrize("bits", ["64", "3"])
def test_hashed_signature_keys_exact_under_collisions(bits, monkeypatch):
    """Hashed signature keys (AMP_WIDE_MEMO: the keys of |D| = 1024 exceed 63
    bits) with the full hash and with 3 hash bits (every class collides):
    k_hash_verify catches each collision and the per-item K_dp takes over,
    so the records equal the exact-key run and the memoised oracle."""
    sc = scenario("hetero_cluster")
    enc = P.EncodedProblem.from_scenario(sc)
    with planner.Searcher(enc, placements_per_class=3000, seed=6) as s:
        top0, all0, _ = s.run(0, s.num_candidates, k=16, want_all=True, details=True)
        st0 = s.stats()
    monkeypatch.setenv("AMP_WIDE_MEMO", "1")
    monkeypatch.setenv("AMP_WIDE_HASH_BITS", bits)
    with planner.Searcher(enc, placements_per_class=3000, seed=6) as s:
        top1, all1, _ = s.run(0, s.num_candidates, k=16, want_all=True, details=True)
        st1 = s.stats()
    monkeypatch.delenv("AMP_WIDE_MEMO")
    monkeypatch.delenv("AMP_WIDE_HASH_BITS")
    assert np.array_equal(all0.view(np.uint8), all1.view(np.uint8))
    assert np.array_equal(top0.view(np.uint8), top1.view(np.uint8))
    if bits == "64":  # no collision: one DP per distinct signature, as with exact keys
        assert st1["dp_instances"] == st0["dp_instances"]
    o = B.Oracle(enc, 3000, 6)
    orec, _ = o.run(threads=8, details=False, memo=True)
    ok = orec["fail_code"] == 0
    assert np.array_equal(all1["fail_code"], orec["fail_code"])
    assert np.array_equal(all1["total"][ok], orec["total"][ok])


def test_trie_dp_stage_timing_and_counts():
    """The bench's roofline inputs: the trie path reports its executed inner
    iterations and the CUDA-event time of its stage kernels, and no chunk
    falls back."""
    sc = scenario("hetero_cluster")
    enc = P.EncodedProblem.from_scenario(sc)
    with planner.Searcher(enc, placements_per_class=200000, seed=0) as s:
        s.run(0, s.num_candidates, k=10)
        st = s.stats()
    assert st["dp_fallback"] == 0
    assert st["dp_stage_launches"] == 1 and st["dp_stage_ms"] > 0  # one K_trie_dp per chunk
    assert st["dp_inner"] > 0 and st["fp64_ops"] == 7 * st["dp_inner"]


LARGE_D = [(4, 8, 60), (8, 8, 24), (128, 8, 3)]  # (nodes, devices per node, P): |D| = 32, 64, 1024


@pytest.mark.parametrize("nodes,per,P_", LARGE_D, ids=["D32", "D64", "D1024"])
def test_large_cluster_sweep_matches_oracle_and_reference(nodes, per, P_):
    """|D| > 16 (warp K_place / K_est, generic Fisher-Yates, coded boundary
    minima, the node-pair all-reduce minimum, memoised signatures with 3-bit
    codes and the trie at U = 8) on the C4 topology with a 24-layer model
    and shuffled placements (P > 1): every record equals the memoised
    oracle, the top-k is its ranking, a strided sample equals the compiled
    reference (ref_sweep), and the pair-scan all-reduce (AMP_NO_NODEBW=1)
    gives the same records."""
    sc = P.synthetic_cluster(nodes, per, 24, 1024, 64)
    enc = P.EncodedProblem.from_scenario(sc)
    outs = []
    for env in (None, "1"):
        import os
        if env:
            os.environ["AMP_NO_NODEBW"] = env
        try:
            with planner.Searcher(enc, placements_per_class=P_, seed=5) as s:
                top, allr, _ = s.run(0, s.num_candidates, k=10, want_all=True, details=False)
                st = s.stats()
        finally:
            os.environ.pop("AMP_NO_NODEBW", None)
        outs.append((top, allr, st))
    assert np.array_equal(outs[0][1].view(np.uint8), outs[1][1].view(np.uint8))
    allr = outs[0][1]
    assert outs[0][2]["dp_instances"] > 0 and outs[0][2]["dp_fallback"] == 0
    o = B.Oracle(enc, P_, 5)
    orec, _ = o.run(threads=16, details=False, memo=True)
    assert np.array_equal(allr["fail_code"], orec["fail_code"])
    ok = orec["fail_code"] == 0
    assert ok.any() and np.array_equal(allr["total"][ok], orec["total"][ok])
    order = planner.rank_order(orec)[:10]
    assert outs[0][0]["index"].tolist() == orec["index"][order].tolist()
    if B.ref_available():
        idx = np.arange(0, len(allr), max(1, len(allr) // 64), dtype=np.uint64)
        rrec = B.ref_sweep_indices(enc, P_, 5, idx, 16, o.max_pp)
        for r, i in zip(rrec, idx):
            e = allr[int(i)]
            assert int(r["fail_code"]) == int(e["fail_code"]), int(i)
            if r["fail_code"] == 0:
                assert r["total"] == e["total"], int(i)


@pytest.mark.parametrize("n_gpus", [2, 4])
@pytest.mark.parametrize("name,P_", [("hetero_cluster", 3000), ("synthetic96", 1)])
def test_multi_gpu_context_equals_single(name, P_, n_gpus):
    """One context over n GPUs (config n_gpus: LPT shards, a thread per GPU,
    NCCL all-gather + device merge, per-record outputs gathered to the
    host) returns the records, details and top-k of the one-GPU run."""
    import torch
    if torch.cuda.device_count() < n_gpus:
        pytest.skip(f"needs {n_gpus} GPUs")
    sc = scenario(name)
    enc = P.EncodedProblem.from_scenario(sc)
    outs = []
    for g in (1, n_gpus):
        with planner.Searcher(enc, placements_per_class=P_, seed=3, n_gpus=g) as s:
            top, allr, bufs = s.run(0, s.num_candidates, k=12, want_all=True, details=True)
            top2, _, _ = s.run(s.num_candidates // 3, s.num_candidates, k=7)  # a sub-range
        outs.append((top, allr, bufs, top2))
    for a, b in zip(outs[0][:2], outs[1][:2]):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
    assert {"cuts", "stage_times", "edge_times"} <= set(outs[0][2])
    for key, v in outs[0][2].items():
        assert np.array_equal(v, outs[1][2][key], equal_nan=v.dtype.kind == "f"), key
    assert np.array_equal(outs[0][3].view(np.uint8), outs[1][3].view(np.uint8))


@pytest.mark.parametrize("name,seed,record_all", [("homogeneous", 3, False), ("hetero_cluster", 17, True),
                                                  ("hetero_model", 101, False)])
def test_speculative_anneal_equals_sequential_and_reference(name, seed, record_all, monkeypatch):
    """the batched anneal (accept / reject branches of the
    next iterations evaluated in one GPU call, AMP_ANNEAL_DEPTH) walks the
    same chain as the sequential one (depth 1) — every recorded state,
    iteration and acceptance — and its initial / best costs equal the
    reference parplan::anneal's."""
    from paper_2210_07297_b200 import anneal as A
    sc = scenario(name)
    o = A.AnnealOptions(iterations=150, seed=seed, record_all=record_all, cost_options=sc.options.cost_options)
    runs = []
    for depth in ("1", "4", "9"):
        monkeypatch.setenv("AMP_ANNEAL_DEPTH", depth)
        runs.append(A.anneal(sc.model, sc.cluster, sc.profile, sc.gbs, o, simulate_top=False))
    monkeypatch.delenv("AMP_ANNEAL_DEPTH", raising=False)
    key = lambda r: [(e.iteration, e.accepted, e.strategy.placement, e.strategy.cut_boundaries,  # noqa: E731
                      e.estimated.total) for e in r.record]
    assert key(runs[0]) == key(runs[1]) == key(runs[2])
    if B.ref_available():
        enc = P.EncodedProblem.from_scenario(sc)
        ic, bc, nrec = B.ref_anneal(enc, 150, seed, record_all=record_all)
        assert (ic, bc, nrec) == (runs[0].initial_cost, runs[0].best_cost, len(runs[0].record))


@pytest.mark.parametrize("env", [{"AMP_NO_GANG": "1"}, {"AMP_GANG_UNIT": "1e5", "AMP_GANG_MIN": "1e5"}])
def test_gang_dp_equals_single_cta(env, monkeypatch):
    """C4's large DP instances solved by CTA gangs (k_gang_plan + the gang
    phase of k_dp<kSparseG>; the pp = 64 programs must be
    multi-CTA) give every record, cut and stage time of the one-CTA-per-
    instance path (AMP_NO_GANG=1) and of many small gangs, on the C4 plan()
    space and a P = 3 sweep (more instances per program)."""
    sc = P.synthetic_c4()
    enc = P.EncodedProblem.from_scenario(sc)
    for P_ in (1, 3):
        outs = []
        for e in ({}, env):
            for k in ("AMP_NO_GANG", "AMP_GANG_UNIT", "AMP_GANG_MIN"):
                monkeypatch.delenv(k, raising=False)
            for k, v in e.items():
                monkeypatch.setenv(k, v)
            with planner.Searcher(enc, placements_per_class=P_, seed=4) as s:
                top, allr, bufs = s.run(0, s.num_candidates, k=10, want_all=True, details=True)
                outs.append((top, allr, bufs, s.stats()))
        assert np.array_equal(outs[0][1].view(np.uint8), outs[1][1].view(np.uint8))
        assert np.array_equal(outs[0][0].view(np.uint8), outs[1][0].view(np.uint8))
        for key in ("cuts", "stage_times"):
            assert np.array_equal(outs[0][2][key], outs[1][2][key], equal_nan=True)
        assert outs[0][3]["dp_instances"] == outs[1][3]["dp_instances"] > 0
