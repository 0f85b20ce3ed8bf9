"""ctypes bindings of include/amp_search.h (the C-ABI of libamp_search.so).

The shared library is built in-tree (``make lib`` / ``__graft_entry__.build()``)
and loaded from this package directory.  There is deliberately no fallback:
if the library or an sm_100a device is missing, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# AMP_SEARCH_LIB overrides the library (A/B builds in tools/)
LIB_PATH = os.environ.get("AMP_SEARCH_LIB", os.path.join(_HERE, "libamp_search.so"))

AMP_OK = 0
AMP_E_INVALID = -1
AMP_E_CUDA = -2
AMP_E_OOM = -3
AMP_E_UNSUPPORTED = -4
AMP_E_NOT_BUILT = -5
AMP_E_CANDIDATE = -6

AMP_FAIL_NONE = 0
AMP_FAIL_PP_GT_L = 1
AMP_FAIL_PROFILE_MISS = 2
AMP_FAIL_CEILING = 3
AMP_FAIL_P2P_BANDWIDTH = 4
AMP_FAIL_ALLREDUCE_BANDWIDTH = 5

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


class AmpProblem(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32),
        ("n_devices", C.c_int32),
        ("gbs", C.c_int32),
        ("fallback_enabled", C.c_int32),
        ("param_count", _dp),
        ("flops_per_sample", _dp),
        ("flops_present", _u8p),
        ("activation_volumes", _dp),
        ("node_id", _ip),
        ("bandwidth", _dp),
        ("n_profile_entries", C.c_int64),
        ("profile_layer", _ip),
        ("profile_tmp", _ip),
        ("profile_mbs", _ip),
        ("profile_seconds", _dp),
        ("bytes_per_param", C.c_double),
        ("fallback_device_flops", C.c_double),
        ("fallback_tmp_bandwidth", C.c_double),
        ("has_max_params_per_device", C.c_int32),
        ("reserved0", C.c_int32),
        ("max_params_per_device", C.c_double),
    ]


class AmpSearchConfig(C.Structure):
    _fields_ = [
        ("placements_per_class", C.c_uint64),
        ("seed", C.c_uint64),
        ("device", C.c_int32),
        ("max_ctas", C.c_int32),
        ("flags", C.c_int32),
        ("n_gpus", C.c_int32),
    ]


AMP_FLAG_DENSE_DP = 1
AMP_FLAG_NO_DEDUP = 2


class AmpRecord(C.Structure):
    _fields_ = [
        ("index", C.c_uint64),
        ("total", C.c_double),
        ("pipeline_time", C.c_double),
        ("dpsync_time", C.c_double),
        ("pp", C.c_int32),
        ("dp", C.c_int32),
        ("tmp", C.c_int32),
        ("mbs", C.c_int32),
        ("fail_code", C.c_int32),
        ("fail_layer", C.c_int32),
        ("fail_value", C.c_double),
    ]


assert C.sizeof(AmpRecord) == 64


class AmpAnnealConfig(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("budget", C.c_int32),
        ("seed", C.c_uint64),
        ("initial_temperature", C.c_double),
        ("cooling", C.c_double),
        ("min_temperature", C.c_double),
        ("record_all", C.c_int32),
        ("neighbor_retries", C.c_int32),
    ]


class AmpAnnealEntry(C.Structure):
    _fields_ = [
        ("estimated", AmpRecord),
        ("iteration", C.c_int32),
        ("accepted", C.c_int32),
        ("reserved", C.c_int32 * 2),
    ]


class AmpDetails(C.Structure):
    _fields_ = [
        ("cuts", _ip),
        ("stage_times", _dp),
        ("edge_times", _dp),
        ("placement", _ip),
        ("simulated", _dp),
    ]


class AmpStats(C.Structure):
    _fields_ = [
        ("kernel_ms", C.c_double),
        ("total_ms", C.c_double),
        ("dp_cells", C.c_double),
        ("dp_inner", C.c_double),
        ("dp_inner_lt", C.c_double),
        ("fp64_ops", C.c_double),
        ("bytes", C.c_double),
        ("candidates", C.c_uint64),
        ("dp_instances", C.c_uint64),
        ("launches", C.c_int32),
        ("ctas", C.c_int32),
        ("place_ms", C.c_double),
        ("dp_ms", C.c_double),
        ("est_ms", C.c_double),
        ("dp_items", C.c_uint64),
        ("dp_launches", C.c_int32),
        ("dp_group", C.c_int32),
        ("dp_stage_ms", C.c_double),
        ("dp_stage_launches", C.c_int32),
        ("dp_fallback", C.c_int32),
    ]


class AmpDpInstance(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32),
        ("stages", C.c_int32),
        ("gas", C.c_int32),
        ("reserved", C.c_int32),
        ("layer_times", _dp),
        ("edge_costs", _dp),
    ]


# (name, restype, argtypes) for every symbol the header declares
SIGNATURES = [
    ("amp_search_create", C.c_int, [C.POINTER(C.c_void_p), C.POINTER(AmpProblem), C.POINTER(AmpSearchConfig)]),
    ("amp_search_destroy", None, [C.c_void_p]),
    ("amp_search_last_error", C.c_char_p, [C.c_void_p]),
    ("amp_last_error", C.c_char_p, []),
    ("amp_search_abi_version", C.c_int, []),
    ("amp_search_num_candidates", C.c_uint64, [C.c_void_p]),
    ("amp_search_num_classes", C.c_int32, [C.c_void_p]),
    ("amp_search_shard_ranges", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, _u64p, C.c_int32, _ip]),
    ("amp_search_max_pp", C.c_int32, [C.c_void_p]),
    ("amp_search_class", C.c_int, [C.c_void_p, C.c_int32, _ip, _ip, _ip, _ip]),
    ("amp_search_partition", C.c_int, [C.c_void_p, C.c_int32, _u64p]),
    ("amp_search_run", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int32,
                                 C.POINTER(AmpRecord), _ip, C.POINTER(AmpRecord), C.POINTER(AmpDetails)]),
    ("amp_search_evaluate", C.c_int, [C.c_void_p, _u64p, C.c_int32, C.POINTER(AmpRecord),
                                      C.POINTER(AmpDetails)]),
    ("amp_search_estimate", C.c_int, [C.c_void_p, _u64p, _ip, C.c_int32, C.POINTER(AmpRecord),
                                      C.POINTER(AmpDetails)]),
    ("amp_search_evaluate_placed", C.c_int, [C.c_void_p, _ip, _ip, _ip, C.c_int32,
                                             C.POINTER(AmpRecord), C.POINTER(AmpDetails)]),
    ("amp_search_anneal", C.c_int, [C.c_void_p, C.POINTER(AmpProblem), C.POINTER(AmpAnnealConfig),
                                    C.POINTER(AmpAnnealEntry), _ip, _ip, C.c_int32, _ip, _ip, _ip,
                                    _dp, C.POINTER(AmpRecord)]),
    ("amp_search_run_device", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int32, C.c_void_p,
                                        C.c_void_p]),
    ("amp_search_run_device_shard", C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                              C.c_void_p, C.c_void_p]),
    ("amp_search_shard_size", C.c_uint64, [C.c_void_p, C.c_int32, C.c_int32]),
    ("amp_search_merge_topk_device", C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                               C.c_void_p, C.c_void_p]),
    ("amp_search_last_stats", C.c_int, [C.c_void_p, C.POINTER(AmpStats)]),
    ("amp_dp_solve_batch", C.c_int, [C.c_int32, C.POINTER(AmpDpInstance), C.c_int32, _ip, C.c_int32,
                                     _dp, _ip]),
    ("amp_fp64_peak", C.c_int, [C.c_int32, _dp, _dp]),
]

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libamp_search.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} not found: the CUDA engine is not built (run `make lib` or "
            "__graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class AmpError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"amp_search status {status}: {message}")
        self.status = status


def check(status: int, ctx=None) -> None:
    if status == AMP_OK:
        return
    lib = load()
    msg = lib.amp_search_last_error(ctx) if ctx else lib.amp_last_error()
    raise AmpError(status, (msg or b"").decode(errors="replace"))
