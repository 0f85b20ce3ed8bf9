"""CPU tests of the C-ABI boundary: the library loads, exports every symbol
include/amp_search.h declares, struct layouts agree, and host-side helpers
(failure texts, scenario round trip) behave like the reference."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, scenario
from paper_2210_07297_b200 import _native as N
from paper_2210_07297_b200 import planner, problem as P

HEADER = os.path.join(ROOT, "include", "amp_search.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(amp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    names = header_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert {s[0] for s in N.SIGNATURES} == set(names)
    assert lib.amp_search_abi_version() == 1


def test_struct_layouts():
    assert C.sizeof(N.AmpRecord) == 64
    assert planner.RECORD_DTYPE.itemsize == 64
    assert C.sizeof(N.AmpSearchConfig) == 32
    # amp_problem: 4 ints, 6 ptrs, int64, 4 ptrs, 3 doubles, 2 ints, 1 double
    assert C.sizeof(N.AmpProblem) == 16 + 48 + 8 + 32 + 24 + 8 + 8


def test_no_cpu_fallback_without_device(has_gpu):
    """Without an sm_100a device the engine fails loudly (no CPU path)."""
    if has_gpu:
        pytest.skip("device present")
    sc = scenario("homogeneous")
    enc = P.EncodedProblem.from_scenario(sc)
    with pytest.raises(N.AmpError):
        planner.Searcher(enc)


def test_failure_texts_match_reference_formats():
    rec = np.zeros(1, dtype=planner.RECORD_DTYPE)[0]
    rec["pp"], rec["tmp"], rec["mbs"] = 128, 2, 4
    rec["fail_code"] = N.AMP_FAIL_PP_GT_L
    assert planner.failure_text(rec, 96) == "infeasible: pp = 128 exceeds layer count 96"
    rec["fail_code"], rec["fail_layer"] = N.AMP_FAIL_PROFILE_MISS, 0
    assert planner.failure_text(rec, 4) == (
        "profile miss: no entry for (layer=0, tmp=2, mbs=4) and analytic fallback is disabled")
    rec["fail_code"] = N.AMP_FAIL_CEILING
    assert planner.failure_text(rec, 4) == "exceeds per-device parameter ceiling"
    rec["fail_code"], rec["fail_value"] = N.AMP_FAIL_P2P_BANDWIDTH, 0.0
    assert planner.failure_text(rec, 4) == "invalid p2p bandwidth 0.000000"
    rec["fail_code"], rec["fail_value"] = N.AMP_FAIL_ALLREDUCE_BANDWIDTH, -1.5
    assert planner.failure_text(rec, 4) == "invalid bandwidth -1.500000 in all-reduce group"


def test_scenario_round_trip():
    sc = scenario("hetero_cluster")
    d = P.scenario_to_dict(sc)
    sc2 = P.scenario_from_dict(d)
    assert np.array_equal(sc.cluster.bandwidth, sc2.cluster.bandwidth)
    assert sc.profile.seconds == sc2.profile.seconds
    assert [l.param_count for l in sc.model.layers] == [l.param_count for l in sc2.model.layers]
    assert sc.cluster.bandwidth[12, 13] == 50e9 and sc.cluster.bandwidth[0, 4] == 10e9
    assert math.isinf(sc.cluster.bandwidth[3, 3])


def test_reference_json_loaders_validate():
    with pytest.raises(P.ParseError):
        P.model_from_json({"layers": []})
    with pytest.raises(P.ValidationError):
        P.model_from_json({"layers": [{"id": 1, "kind": "x", "param_count": 1}],
                           "activation_volumes": []})
    with pytest.raises(P.ValidationError):
        P.cluster_from_json({"devices": [{"id": 0, "node_id": 0, "device_type": "a"},
                                         {"id": 1, "node_id": 0, "device_type": "a"}],
                             "bandwidth": [[0, 1], [2, 0]]})
    with pytest.raises(P.ValidationError):
        P.profile_from_json({"entries": [{"layer": 0, "tmp": 1, "mbs": 1, "seconds": -1}]})


def test_rank_order_key():
    r = np.zeros(5, dtype=planner.RECORD_DTYPE)
    r["index"] = [0, 1, 2, 3, 4]
    r["total"] = [3.0, 1.0, np.nan, 1.0, 0.5]
    r["fail_code"] = [0, 0, 2, 0, 1]
    assert planner.rank_order(r).tolist() == [1, 3, 0, 2, 4]


def test_synthetic_c4_shape():
    sc = P.synthetic_c4()
    assert sc.model.layer_count() == 96 and sc.cluster.device_count() == 1024
    bw = sc.cluster.bandwidth
    assert bw[0, 1] == 900e9 and bw[8, 9] == 600e9 and bw[16, 17] == 300e9
    assert bw[0, 8] == 50e9 and bw[0, 16] == 25e9
