"""The drop-in CLI (paper_2210_07297_b200.cli) against the reference CLI's
own outputs (tests/golden/reports/, made by tests/golden/make_reports.py
from the compiled reference: plan() + write_report + print_candidate_table).

CPU: the report/table writers reproduce the golden bytes from the golden
records (serializer parity).  GPU: `cli plan` end to end writes the same
report.json and table byte for byte, and the exit-code contract of
parplan_main.cpp:71-82 / test_cli.cpp:95-160 holds.
"""
import io
import os
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT, scenario

REPORTS = os.path.join(GOLDEN, "reports")
CASES = {
    "C1_b10": ("homogeneous", 32, 10, None),
    "C1_b5": ("homogeneous", 32, 5, None),
    "C2_b10": ("hetero_cluster", 32, 10, None),
    "C3_b10": ("hetero_model", 64, 10, None),
    "C1_partial_b3": ("homogeneous", 32, 3, "partial"),
    "C1_baseline_layer": ("homogeneous", 32, "layer-balance", None),
    "C1_baseline_param": ("homogeneous", 32, "param-balance", None),
    "C2_baseline_layer": ("hetero_cluster", 32, "layer-balance", None),
    "C3_baseline_param": ("hetero_model", 64, "param-balance", None),
    "C1_partial_baseline_layer": ("homogeneous", 32, "layer-balance", "partial"),
}


def _read(name):
    with open(os.path.join(REPORTS, name)) as f:
        return f.read()


def _write_inputs(tmp, name, variant=None):
    """model/cluster/profile JSON of a scenario, written with the json_io mirror."""
    from paper_2210_07297_b200 import problem as P
    sc = scenario(name)
    paths = {k: str(tmp / f"{k}.json") for k in ("model", "cluster", "profile")}
    P.write_json_file(P.model_to_json(sc.model), paths["model"])
    P.write_json_file(P.cluster_to_json(sc.cluster), paths["cluster"])
    prof = sc.profile
    if variant is not None:
        t = P.ProfileTable()
        if variant == "partial":  # test_cli.cpp:131-160: tmp = 1 entries only
            for (l, tmp_, mbs), v in prof.entries():
                if tmp_ == 1:
                    t.set(l, tmp_, mbs, v)
        prof = t
    P.write_json_file(P.profile_to_json(prof), paths["profile"])
    return paths


@pytest.mark.parametrize("case", sorted(CASES))
def test_report_writer_reproduces_reference_bytes(case):
    import json

    from paper_2210_07297_b200 import jsonfmt, report as R
    recs = R.report_from_json(json.loads(_read(case + ".json")))
    text = jsonfmt.dumps(R.report_to_json(recs)) + "\n"
    assert text == _read(case + ".json")
    out = io.StringIO()
    R.print_candidate_table(out, recs)
    best = -1
    for i, r in enumerate(recs):
        if r.simulated is not None and (best < 0 or r.simulated < recs[best].simulated):
            best = i
    line = R.best_line(recs, best)
    assert out.getvalue() + (line + "\n" if line else "") == _read(case + ".txt")


def test_profile_writer_reproduces_reference_config_bytes():
    """json_io.cpp profile_to_json + write_file == the reference's profile.json."""
    from paper_2210_07297_b200 import jsonfmt, problem as P
    for name in ("homogeneous", "hetero_cluster", "hetero_model"):
        sc = scenario(name)
        text = jsonfmt.dumps(P.profile_to_json(sc.profile)) + "\n"
        ref = os.path.join(GOLDEN, "reports", f"profile_{name}.sha256")
        import hashlib
        with open(ref) as f:
            assert hashlib.sha256(text.encode()).hexdigest() == f.read().split()[0]


def _cli(args, cwd):
    return subprocess.run([sys.executable, "-m", "paper_2210_07297_b200.cli"] + args,
                          capture_output=True, text=True, cwd=cwd,
                          env={**os.environ, "PYTHONPATH": ROOT})


def test_budget_zero_is_a_usage_error(tmp_path):
    p = _write_inputs(tmp_path, "homogeneous")
    r = _cli(["plan", "--model", p["model"], "--cluster", p["cluster"], "--profile", p["profile"],
              "--gbs", "32", "--budget", "0"], ROOT)
    assert r.returncode != 0


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES))
def test_cli_plan_matches_reference_report_bytes(case, tmp_path):
    name, gbs, budget, variant = CASES[case]
    p = _write_inputs(tmp_path, name, variant)
    rep = str(tmp_path / "report.json")
    common = ["--model", p["model"], "--cluster", p["cluster"], "--profile", p["profile"],
              "--gbs", str(gbs), "--report", rep]
    if "baseline" in case:  # CLI `baseline` (megatron_baseline through amp_search_estimate)
        r = _cli(["baseline"] + common + ["--mode", budget], ROOT)
    else:
        r = _cli(["plan"] + common + ["--budget", str(budget)], ROOT)
    assert r.returncode == 0, r.stderr
    with open(rep) as f:
        assert f.read() == _read(case + ".json")
    assert r.stdout == _read(case + ".txt")


@pytest.mark.gpu
def test_cli_all_profile_miss_exits_3(tmp_path):
    """test_cli.cpp:100-115: empty profile, every candidate misses -> exit 3,
    the reference's message on stderr, no report written."""
    p = _write_inputs(tmp_path, "homogeneous", "empty")
    rep = str(tmp_path / "allmiss.json")
    r = _cli(["plan", "--model", p["model"], "--cluster", p["cluster"], "--profile", p["profile"],
              "--gbs", "32", "--budget", "1", "--report", rep], ROOT)
    assert r.returncode == int(_read("C1_allmiss_b1.rc"))
    assert r.stderr == _read("C1_allmiss_b1.err")
    assert not os.path.exists(rep)


def test_megatron_host_rules_match_reference_unit_cases():
    """test_optimizer.cpp:126-155 (degree rule) and the assignment helpers."""
    from paper_2210_07297_b200 import baseline as Bl, problem as P
    sc = scenario("homogeneous")  # 4 nodes x 4 devices
    # largest dp that fits: tmp*pp minimal -> (1, 16, 1) for mbs 1
    assert Bl.megatron_degree_choice(sc.cluster, 32, 1, 24) == (1, 16, 1)
    # mbs 4: dp must divide 32/4*... -> gbs/dp % 4 == 0 -> dp <= 8
    assert Bl.megatron_degree_choice(sc.cluster, 32, 4, 24) == (2, 8, 1)
    for mbs in (1, 2, 4, 8):
        pp, dp, tmp = Bl.megatron_degree_choice(sc.cluster, 32, mbs, 4)
        assert tmp <= Bl.min_node_size(sc.cluster) and pp <= 4
    assert Bl.uniform_assignment(30, 4) == [0, 8, 16, 23, 30]
    assert Bl.uniform_assignment(24, 1) == [0, 24]
    with pytest.raises(P.ValidationError):
        Bl.uniform_assignment(3, 4)
    m = scenario("hetero_model").model
    assert Bl.param_balance_assignment(m, 4) == [0, 3, 6, 9, 24]


ANNEAL = {"C1_anneal_i60_s17": ("homogeneous", 32, 5, 60, 17),
          "C2_anneal_i200_s3": ("hetero_cluster", 32, 10, 200, 3),
          "C3_anneal_i120_s11": ("hetero_model", 64, 10, 120, 11)}


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(ANNEAL))
def test_cli_anneal_reproduces_reference_chain(case, tmp_path):
    """`anneal` (placement.cpp:299-398) with every
    proposal's DP + estimate on the GPU reproduces the reference chain bit
    for bit: the same report.json (top states, estimates, simulated times),
    table and the whole recorded trace (JSON lines)."""
    name, gbs, budget, iters, seed = ANNEAL[case]
    p = _write_inputs(tmp_path, name)
    rep, trace = str(tmp_path / "anneal.json"), str(tmp_path / "anneal.trace")
    r = _cli(["anneal", "--model", p["model"], "--cluster", p["cluster"], "--profile", p["profile"],
              "--gbs", str(gbs), "--budget", str(budget), "--iterations", str(iters),
              "--seed", str(seed), "--report", rep, "--trace", trace], ROOT)
    assert r.returncode == 0, r.stderr
    with open(rep) as f:
        assert f.read() == _read(case + ".json")
    assert r.stdout == _read(case + ".txt")
    with open(trace) as f:
        assert f.read() == _read(case + ".json.trace")
