"""Host data model mirroring the reference's inputs, plus their SoA encoding.

Mirrors reference proj/include/parplan/types.hpp (ModelGraph 41-54, Cluster
67-79, ProfileTable 91-100), cost_model.hpp:41-52 (CostModelOptions) and
optimizer.hpp:56-63 (PlanOptions).  Loaders read the reference's JSON file
formats (proj/src/json_io.cpp, proj/README.md "File formats"), including its
validation rules and error texts for the cases a planner run can hit.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N

INF = math.inf


class ParseError(RuntimeError):
    """types.hpp:163-166"""


class ValidationError(RuntimeError):
    """types.hpp:168-171"""


@dataclass
class LayerSpec:
    id: int
    kind: str
    param_count: float
    flops_per_sample: Optional[float] = None


@dataclass
class ModelGraph:
    layers: List[LayerSpec]
    activation_volumes: List[float]

    def layer_count(self) -> int:
        return len(self.layers)


@dataclass
class DeviceSpec:
    id: int
    node_id: int
    device_type: str = "gpu"


@dataclass
class Cluster:
    devices: List[DeviceSpec]
    bandwidth: np.ndarray  # [D, D] float64, +inf diagonal

    def device_count(self) -> int:
        return len(self.devices)

    def link(self, i: int, j: int) -> float:
        return float(self.bandwidth[i, j])


class ProfileTable:
    """(layer, tmp, mbs) -> seconds; set() overwrites (types.cpp:82-84)."""

    def __init__(self):
        self.layer: List[int] = []
        self.tmp: List[int] = []
        self.mbs: List[int] = []
        self.seconds: List[float] = []

    def set(self, layer: int, tmp: int, mbs: int, seconds: float) -> None:
        self.layer.append(int(layer))
        self.tmp.append(int(tmp))
        self.mbs.append(int(mbs))
        self.seconds.append(float(seconds))

    def __len__(self) -> int:
        return len(self.layer)

    def entries(self):
        """std::map<ProfileKey, double> view: last set() wins, ordered by
        (layer, tmp, mbs) (types.hpp:81-100)."""
        d = {}
        for l, t, m, v in zip(self.layer, self.tmp, self.mbs, self.seconds):
            d[(l, t, m)] = v
        return sorted(d.items())


@dataclass
class AnalyticFallback:
    enabled: bool = False
    device_flops: float = 0.0
    tmp_bandwidth: float = INF


@dataclass
class CostModelOptions:
    bytes_per_param: float = 2.0
    fallback: AnalyticFallback = field(default_factory=AnalyticFallback)


@dataclass
class PlanOptions:
    budget: int = 10
    workers: int = 0
    cost_options: CostModelOptions = field(default_factory=CostModelOptions)
    max_params_per_device: Optional[float] = None


# --------------------------------------------------------------------------
# validation (types.cpp:119-188), raised as ValidationError like json_io
# --------------------------------------------------------------------------

def validate_model(model: ModelGraph) -> List[str]:
    out = []
    L = model.layer_count()
    if L < 1:
        return ["model must have at least one layer"]
    if len(model.activation_volumes) != L - 1:
        out.append(f"activation_volumes has {len(model.activation_volumes)} entries, "
                   f"expected L-1 = {L - 1}")
    for i, layer in enumerate(model.layers):
        if layer.id != i:
            out.append(f"layer ids must be contiguous 0..L-1; position {i} has id {layer.id}")
            break
    for layer in model.layers:
        if layer.param_count < 0:
            out.append(f"layer {layer.id} has negative param_count")
        if layer.flops_per_sample is not None and layer.flops_per_sample < 0:
            out.append(f"layer {layer.id} has negative flops_per_sample")
    for i, v in enumerate(model.activation_volumes):
        if v < 0:
            out.append(f"activation_volumes[{i}] is negative")
    return out


def validate_cluster(cluster: Cluster) -> List[str]:
    n = cluster.device_count()
    if n < 1:
        return ["cluster must have at least one device"]
    seen = [False] * n
    for d in cluster.devices:
        if d.id < 0 or d.id >= n or seen[d.id]:
            return [f"device ids must be a permutation of 0..|D|-1; bad id {d.id}"]
        seen[d.id] = True
    bw = cluster.bandwidth
    if bw.shape != (n, n):
        return [f"bandwidth matrix has shape {bw.shape}, expected ({n}, {n})"]
    out = []
    iu = np.triu_indices(n, 1)
    a, b = bw[iu], bw.T[iu]
    for k in np.nonzero(a != b)[0]:
        out.append(f"bandwidth matrix is asymmetric at ({iu[0][k]},{iu[1][k]})")
    for k in np.nonzero(~(a > 0))[0]:
        out.append(f"bandwidth[{iu[0][k]}][{iu[1][k]}] must be > 0")
    return out


def _require(violations: List[str], what: str) -> None:
    if violations:
        raise ValidationError(what + ":" + "".join("\n  - " + v for v in violations))


# --------------------------------------------------------------------------
# reference JSON formats (json_io.cpp:58-148)
# --------------------------------------------------------------------------

def model_from_json(j: dict) -> ModelGraph:
    layers = j.get("layers", [])
    if not isinstance(layers, list) or not layers:
        raise ParseError("model.layers: must be a non-empty array")
    specs = []
    for l in layers:
        specs.append(LayerSpec(int(l["id"]), str(l["kind"]), float(l["param_count"]),
                               float(l["flops_per_sample"]) if "flops_per_sample" in l else None))
    model = ModelGraph(specs, [float(v) for v in j["activation_volumes"]])
    _require(validate_model(model), "invalid model")
    return model


def cluster_from_json(j: dict) -> Cluster:
    devs = j.get("devices", [])
    if not isinstance(devs, list) or not devs:
        raise ParseError("cluster.devices: must be a non-empty array")
    devices = sorted((DeviceSpec(int(d["id"]), int(d["node_id"]), str(d["device_type"]))
                      for d in devs), key=lambda d: d.id)
    bw = np.array(j["bandwidth"], dtype=np.float64)
    n = min(bw.shape) if bw.ndim == 2 else 0
    for i in range(n):  # json_io.cpp:119-123: diagonal is the +inf sentinel
        bw[i, i] = INF
    cluster = Cluster(devices, bw)
    _require(validate_cluster(cluster), "invalid cluster")
    return cluster


def profile_from_json(j: dict) -> ProfileTable:
    t = ProfileTable()
    for i, e in enumerate(j.get("entries", [])):
        seconds = float(e["seconds"])
        if seconds < 0:
            raise ValidationError(f"entries[{i}].seconds: profile times must be >= 0")
        t.set(int(e["layer"]), int(e["tmp"]), int(e["mbs"]), seconds)
    return t


def model_to_json(model: ModelGraph) -> dict:
    """json_io.cpp:177-187"""
    layers = []
    for l in model.layers:
        e = {"id": int(l.id), "kind": l.kind, "param_count": float(l.param_count)}
        if l.flops_per_sample is not None:
            e["flops_per_sample"] = float(l.flops_per_sample)
        layers.append(e)
    return {"layers": layers, "activation_volumes": [float(v) for v in model.activation_volumes]}


def cluster_to_json(cluster: Cluster) -> dict:
    """json_io.cpp:189-199: the +inf self-link is written as 0.0."""
    bw = np.array(cluster.bandwidth, dtype=np.float64).copy()
    for i in range(min(bw.shape)):
        bw[i, i] = 0.0
    return {"devices": [{"id": d.id, "node_id": d.node_id, "device_type": d.device_type}
                        for d in cluster.devices],
            "bandwidth": [[float(x) for x in row] for row in bw]}


def profile_to_json(profile: ProfileTable) -> dict:
    """json_io.cpp:201-208"""
    return {"entries": [{"layer": l, "tmp": t, "mbs": m, "seconds": float(v)}
                        for (l, t, m), v in profile.entries()]}


def write_json_file(obj, path: str) -> None:
    """write_file (json_io.cpp:49-55): nlohmann dump(2) + newline."""
    from .jsonfmt import dumps
    try:
        with open(path, "w") as f:
            f.write(dumps(obj) + "\n")
    except OSError:
        raise ParseError(f"cannot open file for writing: {path}")


def layer_activation_volume(model: ModelGraph, layer: int) -> float:
    """ModelGraph::layer_activation_volume (types.cpp:42-50)."""
    n = model.layer_count()
    if n <= 1:
        return 0.0
    return float(model.activation_volumes[layer if layer < n - 1 else layer - 1])


def allreduce_time(workers: int, message_size: float, bandwidth: float) -> float:
    """cost_model.cpp:40-52: ((2.0*(n-1))*M)/(n*B)."""
    if workers < 1:
        raise ValidationError("all-reduce needs at least one worker")
    if workers == 1:
        return 0.0
    if not bandwidth > 0:
        raise ValidationError(f"invalid bandwidth {bandwidth:f} in all-reduce group")
    return 2.0 * (workers - 1) * message_size / (workers * bandwidth)


def analytic_layer_time(layer: LayerSpec, tmp: int, mbs: int, device_flops: float,
                        message_size: float, bandwidth: float) -> float:
    """cost_model.cpp:61-68 (raises ProfileMissError-like ValidationError
    when the layer has no flops)."""
    if layer.flops_per_sample is None:
        raise ValidationError(f"profile miss: layer={layer.id} tmp={tmp} mbs={mbs}")
    compute = mbs * layer.flops_per_sample / (tmp * device_flops)
    return compute + allreduce_time(tmp, message_size, bandwidth)


def load_model(path: str) -> ModelGraph:
    with open(path) as f:
        return model_from_json(json.load(f))


def load_cluster(path: str) -> Cluster:
    with open(path) as f:
        return cluster_from_json(json.load(f))


def load_profile(path: str) -> ProfileTable:
    with open(path) as f:
        return profile_from_json(json.load(f))


# --------------------------------------------------------------------------
# compact scenario fixtures (tests/golden/scenarios/*.json)
# --------------------------------------------------------------------------

@dataclass
class Scenario:
    name: str
    model: ModelGraph
    cluster: Cluster
    profile: ProfileTable
    gbs: int
    options: PlanOptions = field(default_factory=PlanOptions)


def scenario_to_dict(s: Scenario) -> dict:
    bw = s.cluster.bandwidth.copy()
    np.fill_diagonal(bw, 0.0)
    fo = s.options.cost_options.fallback
    return {
        "name": s.name, "gbs": s.gbs,
        "param_count": [l.param_count for l in s.model.layers],
        "flops_per_sample": [l.flops_per_sample for l in s.model.layers],
        "activation_volumes": list(s.model.activation_volumes),
        "node_id": [d.node_id for d in s.cluster.devices],
        "bandwidth": bw.tolist(),
        "profile": {"layer": s.profile.layer, "tmp": s.profile.tmp, "mbs": s.profile.mbs,
                    "seconds": s.profile.seconds},
        "fallback": {"enabled": fo.enabled, "device_flops": fo.device_flops,
                     "tmp_bandwidth": None if math.isinf(fo.tmp_bandwidth) else fo.tmp_bandwidth},
        "bytes_per_param": s.options.cost_options.bytes_per_param,
        "max_params_per_device": s.options.max_params_per_device,
    }


def scenario_from_dict(d: dict) -> Scenario:
    layers = [LayerSpec(i, "layer", float(p), None if f is None else float(f))
              for i, (p, f) in enumerate(zip(d["param_count"], d["flops_per_sample"]))]
    model = ModelGraph(layers, [float(v) for v in d["activation_volumes"]])
    devices = [DeviceSpec(i, int(n)) for i, n in enumerate(d["node_id"])]
    bw = np.array(d["bandwidth"], dtype=np.float64)
    np.fill_diagonal(bw, INF)
    prof = ProfileTable()
    pr = d["profile"]
    prof.layer, prof.tmp, prof.mbs = list(pr["layer"]), list(pr["tmp"]), list(pr["mbs"])
    prof.seconds = [float(x) for x in pr["seconds"]]
    fb = d.get("fallback", {})
    opts = PlanOptions(cost_options=CostModelOptions(
        bytes_per_param=float(d.get("bytes_per_param", 2.0)),
        fallback=AnalyticFallback(bool(fb.get("enabled", False)), float(fb.get("device_flops", 0.0)),
                                  INF if fb.get("tmp_bandwidth") is None else float(fb["tmp_bandwidth"]))),
        max_params_per_device=d.get("max_params_per_device"))
    return Scenario(d["name"], model, Cluster(devices, bw), prof, int(d["gbs"]), opts)


def load_scenario(path: str) -> Scenario:
    with open(path) as f:
        return scenario_from_dict(json.load(f))


def synthetic_c4() -> Scenario:
    """96-layer h=12288 transformer on 1024 GPUs
    (128 nodes x 8, three device types), gbs 512, analytic fallback."""
    return synthetic_cluster(128, 8, 96, 12288, 512, "synthetic96")


def synthetic_cluster(nodes: int, per: int, L: int, h: int, gbs: int, name: str = "") -> Scenario:
    """The C4 topology at any size: `nodes` x `per`
    devices, node type = node mod 3, intra {900, 600, 300} GB/s, inter 50
    GB/s (25 if either node is type 2); an L-layer h-wide transformer chain
    (s = 2048) on the analytic fallback."""
    s = 2048
    layers = [LayerSpec(i, "transformer", float(12 * h * h), float(72 * s * h * h)) for i in range(L)]
    model = ModelGraph(layers, [float(2 * s * h)] * (L - 1))
    D = nodes * per
    node = np.arange(D) // per
    ntype = node % 3
    intra = np.array([900e9, 600e9, 300e9])
    bw = np.where(node[:, None] == node[None, :], intra[ntype][:, None],
                  np.where((ntype[:, None] == 2) | (ntype[None, :] == 2), 25e9, 50e9))
    bw = bw.astype(np.float64)
    np.fill_diagonal(bw, INF)
    devices = [DeviceSpec(i, int(node[i]), ["b200", "h100", "a100"][int(ntype[i])]) for i in range(D)]
    opts = PlanOptions(cost_options=CostModelOptions(
        fallback=AnalyticFallback(True, 1e15, 900e9)))
    return Scenario(name or f"synthetic{L}_d{D}", model, Cluster(devices, bw), ProfileTable(), gbs, opts)


# --------------------------------------------------------------------------
# SoA encoding -> amp_problem
# --------------------------------------------------------------------------

class EncodedProblem:
    """Owns the arrays an amp_problem points to (kept alive with it)."""

    def __init__(self, model: ModelGraph, cluster: Cluster, profile: ProfileTable, gbs: int,
                 options: Optional[PlanOptions] = None):
        options = options or PlanOptions()
        co = options.cost_options
        L = model.layer_count()
        D = cluster.device_count()
        self.L, self.D, self.gbs = L, D, int(gbs)
        self.param = np.ascontiguousarray([l.param_count for l in model.layers], dtype=np.float64)
        self.flops = np.ascontiguousarray(
            [l.flops_per_sample if l.flops_per_sample is not None else 0.0 for l in model.layers],
            dtype=np.float64)
        self.flops_ok = np.ascontiguousarray(
            [l.flops_per_sample is not None for l in model.layers], dtype=np.uint8)
        self.act = np.ascontiguousarray(model.activation_volumes if L > 1 else [0.0], dtype=np.float64)
        node = np.zeros(D, dtype=np.int32)
        for d in cluster.devices:
            node[d.id] = d.node_id
        self.node = node
        self.bw = np.ascontiguousarray(cluster.bandwidth, dtype=np.float64).reshape(D * D).copy()
        self.p_layer = np.ascontiguousarray(profile.layer, dtype=np.int32)
        self.p_tmp = np.ascontiguousarray(profile.tmp, dtype=np.int32)
        self.p_mbs = np.ascontiguousarray(profile.mbs, dtype=np.int32)
        self.p_sec = np.ascontiguousarray(profile.seconds, dtype=np.float64)
        s = N.AmpProblem()
        s.n_layers, s.n_devices, s.gbs = L, D, int(gbs)
        s.fallback_enabled = int(co.fallback.enabled)
        s.param_count = self.param.ctypes.data_as(N._dp)
        s.flops_per_sample = self.flops.ctypes.data_as(N._dp)
        s.flops_present = self.flops_ok.ctypes.data_as(N._u8p)
        s.activation_volumes = self.act.ctypes.data_as(N._dp)
        s.node_id = self.node.ctypes.data_as(N._ip)
        s.bandwidth = self.bw.ctypes.data_as(N._dp)
        s.n_profile_entries = len(self.p_layer)
        s.profile_layer = self.p_layer.ctypes.data_as(N._ip)
        s.profile_tmp = self.p_tmp.ctypes.data_as(N._ip)
        s.profile_mbs = self.p_mbs.ctypes.data_as(N._ip)
        s.profile_seconds = self.p_sec.ctypes.data_as(N._dp)
        s.bytes_per_param = float(co.bytes_per_param)
        s.fallback_device_flops = float(co.fallback.device_flops)
        s.fallback_tmp_bandwidth = float(co.fallback.tmp_bandwidth)
        s.has_max_params_per_device = int(options.max_params_per_device is not None)
        s.max_params_per_device = float(options.max_params_per_device or 0.0)
        self.struct = s

    def ref(self):
        return C.byref(self.struct)

    @classmethod
    def from_scenario(cls, sc: Scenario, options: Optional[PlanOptions] = None) -> "EncodedProblem":
        return cls(sc.model, sc.cluster, sc.profile, sc.gbs, options or sc.options)


def divisors(n: int) -> List[int]:
    """optimizer.cpp:29-41"""
    out = set()
    d = 1
    while d * d <= n:
        if n % d == 0:
            out.add(d)
            out.add(n // d)
        d += 1
    return sorted(out)


def enumerate_degrees(device_count: int):
    """optimizer.cpp:43-51: (pp, dp, tmp) with pp asc, dp asc."""
    return [(pp, dp, device_count // (pp * dp)) for pp in divisors(device_count)
            for dp in divisors(device_count // pp)]


def enumerate_mbs(gbs: int, dp: int) -> List[int]:
    """optimizer.cpp:57-62"""
    if dp < 1 or gbs % dp != 0:
        return []
    return divisors(gbs // dp)


def candidate_classes(device_count: int, gbs: int):
    """plan() candidate list (optimizer.cpp:202-207)."""
    return [(pp, dp, tmp, mbs) for (pp, dp, tmp) in enumerate_degrees(device_count)
            for mbs in enumerate_mbs(gbs, dp)]
