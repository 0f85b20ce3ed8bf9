"""Benchmark of the B200 AMP strategy-search hot path.

One "step" = evaluating one batch of candidate strategies end to end on the
GPU: placement, stage-boundary bandwidths, the layer-partition DP, the cost
estimate, and the global top-k (CTA lists -> device merge; across ranks an
NCCL all-gather of the per-GPU top-k followed by a device merge).

Workload (BASELINE.json configs[1] + configs[4]): the hetero_cluster scenario
(30-layer GPT-2-like chain, 16 devices: 3 fast V100 nodes + 1 T4 node,
asymmetric intra/inter bandwidth, gbs 32) swept over its 70 plan() classes
x P placements, N_PER_GPU candidates per GPU per step
(weak scaling).  Inputs (problem tables) are resident in HBM; the per-step
outputs are a k-record top-k.

Roofline: the DP is the FP64 part of the path; its
headline figure is 7 FP64 ops per executed (cell, cut) iteration of the
memoised, prefix-shared DP over the CUDA-event time of the DP stage kernel
(k_trie_dp), against the measured FP64 DADD peak.  The per-candidate
kernels (K_place / K_est: integer placement shuffle + estimate) are reported
by their HBM fraction and, secondarily, their issue-slot utilisation from
the ncu counts of THIS build (profiles/<round>_kernel_counts.json, checked
against the library's sha256; stale counts are dropped, not used).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SCENARIO = "hetero_cluster"
DEFAULT_N_PER_GPU = 100_000_000
TOPK = 10
METRIC = "candidate strategies/sec"
UNIT = "candidates/s"
LIB = os.path.join(ROOT, "paper_2210_07297_b200", "libamp_search.so")
# ncu counts of this build's kernels on this workload (tools/profile_round.py)
KERNEL_COUNTS = os.path.join(ROOT, "profiles", "r2_kernel_counts.json")
SWEEP_N = [10_000, 100_000, 1_000_000, 10_000_000, 100_000_000, 1_000_000_000]
CPU_FULL_MAX = 1_000_000  # the CPU arm runs the sweep in full up to here, then extrapolates


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-per-gpu", type=int, default=DEFAULT_N_PER_GPU)
    ap.add_argument("--cpu-sample", type=int, default=300000,
                    help="candidates in the bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense-DP comparison leg")
    ap.add_argument("--no-wall-time", action="store_true",
                    help="skip the C1-C4 plan() wall-time leg (ours vs the reference)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the configs[4] N sweep")
    return ap.parse_args()


def load_scenario():
    from paper_2210_07297_b200 import problem as P
    return P.load_scenario(os.path.join(ROOT, "tests", "golden", "scenarios", SCENARIO + ".json"))


def workload(n_per_gpu, world):
    n_total = n_per_gpu * world
    n_cls = 70
    P_ = -(-n_total // n_cls)
    return n_total, P_


def lib_sha256():
    h = hashlib.sha256()
    with open(LIB, "rb") as f:
        h.update(f.read())
    return h.hexdigest()


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every
    millisecond while the timed region runs (nvidia-smi's 100 ms loop would
    see no sample of a ~25 ms region)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, index=0, period_s=0.001):
        self.index = index
        self.period = period_s
        self.rows = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.stop = threading.Event()
        self.t = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self):
        nv, h = self.nv, self.h
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while True:
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx, get_reasons(h)))
            except Exception:
                pass
            if self.stop.wait(self.period):
                break

    def __enter__(self):
        try:
            self.nv, self.h = self._handle()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        reasons = set()
        for _, _, m in self.rows:
            for bit, name in self.REASONS.items():
                if m & bit:
                    reasons.add(name)
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])),
                "sm_max_mhz": float(max(r[1] for r in self.rows)), "reasons": sorted(reasons),
                "samples": len(self.rows), "source": "nvml, 1 ms"}


def cpu_sample_indices(n_total, sample):
    """Strided sample across the whole class-major range (all classes)."""
    stride = max(1, n_total // sample)
    return np.arange(0, n_total, stride, dtype=np.uint64)[:sample]


def run_cpu_reference(sc, n_total, P_, sample, threads):
    """The reference's own CPU call chain (oracle/_ref, compiled from the
    unmodified reference sources) over a bounded strided sample, or over
    the full range when sample >= n_total."""
    from oracle import bindings as B
    from paper_2210_07297_b200 import problem as P
    enc = P.EncodedProblem.from_scenario(sc)
    idx = np.arange(n_total, dtype=np.uint64) if sample >= n_total else cpu_sample_indices(n_total, sample)
    max_pp = 16
    if B.ref_available():
        t0 = time.perf_counter()
        B.ref_sweep_indices(enc, P_, 0, idx, threads, max_pp)
        dt = time.perf_counter() - t0
        kind = "reference"
    else:  # the plain-C port of the same path
        from paper_2210_07297_b200.planner import RECORD_DTYPE
        o = B.Oracle(enc, P_, 0)
        rec = np.zeros(1, dtype=RECORD_DTYPE)
        t0 = time.perf_counter()
        for i in idx:
            o.lib.oracle_evaluate(o.h, int(i), rec.ctypes.data_as(B._recp), None, None, None)
        dt = time.perf_counter() - t0
        kind = "port"
        threads = 1
    return len(idx) / dt, dt, kind, threads, len(idx)


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sc = load_scenario()
    n_total, P_ = workload(args.n_per_gpu, args.gpus)
    threads = os.cpu_count() or 1
    # keep the whole K + W run to ~1-2 minutes of CPU time
    per_step = max(1000, min(args.cpu_sample, args.cpu_sample * 8 // max(1, args.steps + args.warmup)))
    vals = []
    for i in range(args.warmup + args.steps):
        v, dt, kind, th, ns = run_cpu_reference(sc, n_total, P_, per_step, threads)
        if i >= args.warmup:
            vals.append(v)
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * ns / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{SCENARIO} sweep (C2 classes x placements)", "scenario": SCENARIO,
                   "candidates_per_step": n_total, "placements_per_class": P_,
                   "sample": f"{ns} strided candidates of the {n_total}-candidate space"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": th, "kind": kind, "cpu": cpu_model(),
                         "sample": f"{ns} strided candidates, reference call chain "
                                   "(heuristic/shuffled placement, optimal_assignment, estimate)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def search_wall_time(budget=10, runs=10, ref_runs_c4=5):
    """The metric's second half: AMP search wall time of plan() for C1-C4 —
    the drop-in (planner.plan: create from host arrays, K0/K0b, evaluate,
    rank, simulate the top `budget`) vs the reference parplan::plan
    (oracle/_ref, all host threads), same inputs; median of `runs` after a
    warm-up; the argmin and the whole ranking must be identical.  C4 also
    reports its plan() phase times."""
    from oracle import bindings as B
    from paper_2210_07297_b200 import planner, problem as P
    out = {}
    names = {"C1": "homogeneous", "C2": "hetero_cluster", "C3": "hetero_model", "C4": "synthetic96"}
    for tag, name in names.items():
        sc = P.synthetic_c4() if name == "synthetic96" else P.load_scenario(
            os.path.join(ROOT, "tests", "golden", "scenarios", name + ".json"))
        opts = P.PlanOptions(budget=budget, cost_options=sc.options.cost_options,
                             max_params_per_device=sc.options.max_params_per_device)
        planner.plan(sc.model, sc.cluster, sc.profile, sc.gbs, opts)  # warm-up
        ts, phases = [], []
        for _ in range(runs):
            tm = {}
            t0 = time.perf_counter()
            res = planner.plan(sc.model, sc.cluster, sc.profile, sc.gbs, opts, timing=tm)
            ts.append(time.perf_counter() - t0)
            phases.append(tm)
        e = {"workload": name, "candidates": len(res.candidates), "budget": budget, "runs": runs,
             "ours_s": float(np.median(ts)), "ours_min_s": float(min(ts)),
             "best": list(res.candidates[res.best_index].strategy.degrees) if res.best_index >= 0 else None}
        if tag == "C4":
            e["ours_phases_ms"] = {k: round(1e3 * float(np.median([p[k] for p in phases])), 3)
                                   for k in phases[0]}
        if B.ref_available():
            enc = P.EncodedProblem.from_scenario(sc, opts)
            max_pp = max(c[0] for c in P.candidate_classes(sc.cluster.device_count(), sc.gbs))
            rs = []
            n_ref = ref_runs_c4 if tag == "C4" else runs
            B.ref_plan(enc, max_pp, budget=budget, workers=os.cpu_count() or 1)  # warm-up
            for _ in range(n_ref):
                t0 = time.perf_counter()
                r = B.ref_plan(enc, max_pp, budget=budget, workers=os.cpu_count() or 1)
                rs.append(time.perf_counter() - t0)
            e["reference_s"] = float(np.median(rs))
            e["reference_runs"] = n_ref
            e["reference_threads"] = os.cpu_count()
            e["same_argmin"] = bool(r["best_index"] == res.best_index)
            e["same_ranking"] = bool([int(x) for x in r["records"]["index"]] ==
                                     [c.index for c in res.candidates])
            e["speedup"] = e["reference_s"] / e["ours_s"]
        out[tag] = e
    return out


def anneal_wall_time(iterations=200, seed=17, runs=5):
    """the annealing chain (placement.cpp:299-398) —
    ours (anneal.anneal: the chain on the host, every proposal's DP +
    estimate on the GPU, speculative accept/reject branches batched per
    call) vs the reference parplan::anneal (oracle/_ref), C1-C3, median of
    `runs`; the initial and best costs must be identical."""
    from oracle import bindings as B
    from paper_2210_07297_b200 import anneal as A, problem as P
    out = {}
    for tag, name in {"C1": "homogeneous", "C2": "hetero_cluster", "C3": "hetero_model"}.items():
        sc = P.load_scenario(os.path.join(ROOT, "tests", "golden", "scenarios", name + ".json"))
        o = A.AnnealOptions(iterations=iterations, seed=seed, cost_options=sc.options.cost_options)
        A.anneal(sc.model, sc.cluster, sc.profile, sc.gbs, o, simulate_top=False)  # warm-up
        ts = []
        for _ in range(runs):
            t0 = time.perf_counter()
            r = A.anneal(sc.model, sc.cluster, sc.profile, sc.gbs, o, simulate_top=False)
            ts.append(time.perf_counter() - t0)
        e = {"iterations": iterations, "ours_s": float(np.median(ts)), "initial_cost": r.initial_cost,
             "best_cost": r.best_cost}
        if B.ref_available():
            enc = P.EncodedProblem.from_scenario(sc)
            rs = []
            for _ in range(runs):
                t0 = time.perf_counter()
                ic, bc, _ = B.ref_anneal(enc, iterations, seed)
                rs.append(time.perf_counter() - t0)
            e["reference_s"] = float(np.median(rs))
            e["same_result"] = bool(ic == r.initial_cost and bc == r.best_cost)
            e["speedup"] = e["reference_s"] / e["ours_s"]
        out[tag] = e
    return out


def l2_flush(buf):
    buf.add_(1)  # write a buffer larger than L2 (126 MB)


def kernel_counts():
    """ncu counts of this build (None when absent or for another build)."""
    try:
        with open(KERNEL_COUNTS) as f:
            kc = json.load(f)
    except OSError:
        return None, "absent"
    if kc.get("lib_sha256") != lib_sha256():
        return None, f"stale ({os.path.relpath(KERNEL_COUNTS, ROOT)} is for another build)"
    return kc, os.path.relpath(KERNEL_COUNTS, ROOT)


def our_arm(args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_2210_07297_b200 import _native as N
    from paper_2210_07297_b200 import problem as P
    from paper_2210_07297_b200.planner import RECORD_DTYPE, Searcher

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    distributed = world > 1
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc = load_scenario()
    n_total, P_ = workload(args.n_per_gpu, world)
    enc = P.EncodedProblem.from_scenario(sc)
    s = Searcher(enc, placements_per_class=P_, seed=0, device=local)
    # the whole class-major space (70 classes x P_ placements, >= n_total);
    # rank r evaluates its LPT shard (amp_search_run_device_shard: one block
    # of every class when P >= world)
    n_total = s.num_candidates
    n_mine = s.shard_size(rank, world)
    stream = torch.cuda.current_stream()
    k = TOPK
    local_top = torch.empty(k * 64, dtype=torch.uint8, device="cuda")
    gathered = torch.empty(world * k * 64, dtype=torch.uint8, device="cuda")
    final = torch.empty(k * 64, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step():
        s.run_device_shard(rank, world, k, local_top.data_ptr(), stream.cuda_stream)
        if distributed:
            dist.all_gather_into_tensor(gathered, local_top)
            s.merge_device(gathered.data_ptr(), world * k, k, final.data_ptr(), stream.cuda_stream)
        else:
            final.copy_(local_top)

    for _ in range(args.warmup):
        l2_flush(flush)
        step()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kstats = []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            l2_flush(flush)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            kstats.append(s.stats())  # per-kernel events on the engine stream
        torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in ev]
    my_ms = float(sum(times))
    if distributed:
        t = torch.tensor([my_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        my_ms = float(t.item())
        dist.barrier()
    ms_per_step = my_ms / args.steps
    value = n_total / (ms_per_step * 1e-3)
    st = kstats[-1]
    top = np.frombuffer(final.cpu().numpy().tobytes(), dtype=RECORD_DTYPE)

    # ---- rooflines ---------------------------------------------------------
    peak = C.c_double()
    pms = C.c_double()
    N.check(N.load().amp_fp64_peak(local, C.byref(peak), C.byref(pms)))
    peak_t = peak.value / 1e12
    med = lambda key: float(np.median([x[key] for x in kstats]))  # noqa: E731
    dp_stage_ms, dp_ms, place_ms, est_ms = med("dp_stage_ms"), med("dp_ms"), med("place_ms"), med("est_ms")
    fp64 = st["fp64_ops"]  # 7 per executed (cell, cut) iteration, this step's DP (device counters)
    ach_stage = fp64 / (dp_stage_ms * 1e-3) / 1e12
    ach_span = fp64 / (dp_ms * 1e-3) / 1e12
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6537.0))
    kc, kc_src = kernel_counts()
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    csum = clk.summary()
    mhz = csum.get("sm_mhz") or csum.get("sm_max_mhz") or 1965.0
    issue_peak = sms * 4 * mhz * 1e6

    def counted(name, ms):
        c = (kc or {}).get(name)
        if not c:
            return {}
        per_launch = c["dram_bytes"] / c["launches"]
        gbs = c["dram_bytes"] / c["runs"] / (ms * 1e-3) / 1e9
        return {"traffic_per_launch": per_launch, "dram_gbs": gbs, "hbm_frac": gbs / hbm_peak,
                "issue_frac": c["warp_inst"] / c["runs"] / (ms * 1e-3) / issue_peak,
                "counts": kc_src}

    k_dp = {"bound": "fp64", "kernel": "k_trie_dp (layer-partition DP, all stages: memoised by signature, "
                                       "prefix-shared trie, smem-staged parent tables)",
            "achieved": ach_stage, "peak": peak_t, "unit": "TFLOP/s", "frac": ach_stage / peak_t,
            "ms_per_step": dp_stage_ms, "launches_per_step": int(st["dp_stage_launches"]),
            "traffic": None,
            "def": "7 FP64 ops per executed (cell, cut) iteration (SURVEY.md 8(d)), device-counted, over "
                   "the CUDA-event time of k_trie_dp; peak = measured DADD throughput (amp_fp64_peak)"}
    c = (kc or {}).get("k_trie_dp")
    if c:
        k_dp["traffic"] = c["dram_bytes"] / c["launches"]
        k_dp["traffic_unit"] = "bytes per launch (ncu dram__bytes_read+write, " + kc_src + ")"
    rooflines = {
        "k_dp": k_dp,
        "k_dp_span": {"bound": "fp64", "achieved": ach_span, "peak": peak_t, "unit": "TFLOP/s",
                      "frac": ach_span / peak_t, "ms_per_step": dp_ms,
                      "note": "the whole DP phase: signature list + trie build + k_trie_dp + backtrack + "
                              "per-signature estimate"},
        "k_est": dict({"bound": "hbm/issue", "ms_per_step": est_ms}, **counted("k_est_t", est_ms)),
        "k_place": dict({"bound": "hbm/issue", "ms_per_step": place_ms}, **counted("k_place_t", place_ms)),
    }

    # ---- e2e through the C-ABI with host buffers ------------------------
    e2e = None
    if not args.no_e2e:
        e2e = e2e_arm(args, enc, P_, n_total, world, rank, local, distributed)

    dense = per_cand = sweep = None
    if world == 1 and not args.no_dense:
        dense = dense_leg(enc, local)
        per_cand = per_candidate_leg(enc, local, P_, n_total)
    if world == 1 and not args.no_sweep:
        sweep = sweep_leg(sc, enc, local, args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{SCENARIO} sweep (C2 classes x placements)",
                       "scenario": SCENARIO, "candidates_per_step": n_total,
                       "candidates_per_gpu": args.n_per_gpu, "placements_per_class": P_,
                       "topk": k, "l2": "flushed (256 MiB write) before every timed step",
                       "candidates_this_rank": n_mine,
                       "parallelism": f"LPT shards x{world} (amp_search_run_device_shard), NCCL "
                                      "all-gather of the k-record top-k + device merge"},
            "roofline": rooflines["k_dp"],
            "rooflines": rooflines,
            "dp_detail": {
                "dp_memoisation": {"candidates": n_total, "dp_instances_solved": st["dp_instances"]},
                "pipeline_ms_per_step": {"k_place": place_ms, "k_dp_span": dp_ms, "k_dp_stage": dp_stage_ms,
                                         "k_est": est_ms},
                "fp64_ops_per_step": fp64, "dp_inner_per_step": st["dp_inner"],
                "dp_fallback_chunks": st["dp_fallback"],
                "peak_source": "measured live: amp_fp64_peak DADD throughput (MEASURED_PEAKS.json has "
                               "no FP64 entry)"},
            "gpu_launches": int(args.steps * (st["launches"] + (1 if distributed else 0))),
            "best": {"index": int(top[0]["index"]), "total": float(top[0]["total"]),
                     "degrees": [int(top[0]["pp"]), int(top[0]["dp"]), int(top[0]["tmp"])],
                     "mbs": int(top[0]["mbs"])},
            "clocks": csum,
            "lib_sha256": lib_sha256(),
        }
        if e2e:
            line["e2e"] = e2e
        if per_cand:
            line["per_candidate_dp"] = per_cand
        if dense:
            line["dense_dp"] = dense
        if sweep:
            line["sweep"] = sweep
        if world == 1 and not args.no_wall_time:
            line["search_wall_time"] = search_wall_time()
            line["anneal_wall_time"] = anneal_wall_time()
        if world == 1 and not args.no_cpu_baseline:
            th = os.cpu_count() or 1
            v, dt, kind, th, ns = run_cpu_reference(sc, n_total, P_, args.cpu_sample, th)
            v1, dt1, _, _, ns1 = run_cpu_reference(sc, n_total, P_, max(2000, args.cpu_sample // 40), 1)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": th, "kind": kind, "cpu": cpu_model(),
                                    "sample": f"{ns} strided candidates of the same sweep, "
                                              f"{dt:.1f} s on {th} host threads",
                                    "one_thread": {"value": v1, "sample": f"{ns1} strided candidates, "
                                                                          f"{dt1:.1f} s on 1 thread"}}
        print(json.dumps(line), flush=True)
    s.close()
    if distributed:
        dist.destroy_process_group()


def sweep_leg(sc, enc, local, args):
    """configs[4]: N in 1e4 .. 1e9 candidates (C2 classes x placements): the
    device figure (one run's CUDA-event time, warm context), the e2e figure
    (create from host arrays + run + host top-k + destroy, wall clock), and
    the reference CPU path on all host threads — in full up to 1e6
    candidates, a >= 1e6 prefix-equivalent strided sample beyond that,
    labelled extrapolated."""
    from paper_2210_07297_b200.planner import Searcher
    out = []
    th = os.cpu_count() or 1
    cpu_rate = None
    for n in SWEEP_N:
        P_ = -(-n // 70)
        with Searcher(enc, placements_per_class=P_, seed=0, device=local) as s:
            s.run(0, n, k=TOPK)  # warm
            ms = []
            for _ in range(3 if n >= 10**9 else 5):
                s.run(0, n, k=TOPK)
                ms.append(s.stats()["total_ms"])
        dev = float(np.median(ms))
        walls = []
        for _ in range(3):
            t0 = time.perf_counter()
            with Searcher(enc, placements_per_class=P_, seed=0, device=local) as s:
                s.run(0, n, k=TOPK)
            walls.append(time.perf_counter() - t0)
        e = {"n": n, "placements_per_class": P_, "device_ms": dev, "device_value": n / (dev * 1e-3),
             "e2e_s": float(np.median(walls)), "e2e_value": n / float(np.median(walls))}
        if not args.no_cpu_baseline:
            if n <= CPU_FULL_MAX:
                v, dt, kind, thr, ns = run_cpu_reference(sc, n, P_, n, th)
                cpu_rate = (v, kind, thr)
                e["cpu"] = {"value": v, "s": dt, "kind": kind, "cores": thr, "measured": "full"}
            else:
                v, kind, thr = cpu_rate
                e["cpu"] = {"value": v, "s": n / v, "kind": kind, "cores": thr,
                            "measured": f"extrapolated from the full N={CPU_FULL_MAX} run's rate"}
        out.append(e)
    return {"points": out, "unit": UNIT, "workload": f"{SCENARIO}: 70 classes x P placements"}


def per_candidate_leg(enc, local, P_, n):
    """The same sweep with one DP per candidate (AMP_FLAG_NO_DEDUP): the
    K_dp kernel's own efficiency without memoisation (identical results,
    tests/test_gpu_parity.py::test_memoised_dp_equals_per_candidate_dp)."""
    import ctypes as C

    from paper_2210_07297_b200 import _native as N
    from paper_2210_07297_b200.planner import Searcher
    s = Searcher(enc, placements_per_class=P_, seed=0, device=local, dedup=False)
    s.run(0, n, k=TOPK)
    sts = []
    for _ in range(3):
        s.run(0, n, k=TOPK)
        sts.append(s.stats())
    s.close()
    peak = C.c_double()
    pms = C.c_double()
    N.check(N.load().amp_fp64_peak(local, C.byref(peak), C.byref(pms)))
    tot = float(np.median([x["total_ms"] for x in sts]))
    dp_ms = float(np.median([x["dp_ms"] for x in sts]))
    ach = sts[-1]["fp64_ops"] / (dp_ms * 1e-3) / 1e12
    return {"value": n / (tot * 1e-3), "unit": UNIT, "candidates": n, "ms_per_step": tot,
            "pipeline_ms": {"k_place": float(np.median([x["place_ms"] for x in sts])),
                            "k_dp": dp_ms, "k_est": float(np.median([x["est_ms"] for x in sts]))},
            "dp_inner": sts[-1]["dp_inner"],
            "roofline": {"bound": "fp64", "kernel": f"k_dp_multi<{sts[-1]['dp_group']}>",
                         "achieved": ach, "peak": peak.value / 1e12, "unit": "TFLOP/s",
                         "frac": ach / (peak.value / 1e12)}}


def dense_leg(enc, local, n=1_000_000):
    """The reference's full-table DP on the same sweep (AMP_FLAG_DENSE_DP):
    same results, ~36x more DP work; its FP64-pipe roofline is reported
    separately from the production (pruned) path."""
    import ctypes as C

    from paper_2210_07297_b200 import _native as N
    from paper_2210_07297_b200.planner import Searcher
    P_ = -(-n // 70)
    s = Searcher(enc, placements_per_class=P_, seed=0, device=local, dense_dp=True)
    s.run(0, n, k=TOPK)
    ms = []
    for _ in range(3):
        s.run(0, n, k=TOPK)
        ms.append(s.stats()["kernel_ms"])
    st = s.stats()
    s.close()
    peak = C.c_double()
    pms = C.c_double()
    N.check(N.load().amp_fp64_peak(local, C.byref(peak), C.byref(pms)))
    k_ms = float(np.median(ms))
    ach = st["fp64_ops"] / (k_ms * 1e-3) / 1e12
    return {"value": n / (k_ms * 1e-3), "unit": UNIT, "candidates": n, "kernel_ms": k_ms,
            "dp_inner": st["dp_inner"],
            "roofline": {"bound": "fp64", "achieved": ach, "peak": peak.value / 1e12,
                         "unit": "TFLOP/s", "frac": ach / (peak.value / 1e12)}}


def e2e_arm(args, enc, P_, n_total, world, rank, local, distributed):
    """Same metric through the public API per step, from HOST arrays to a
    HOST top-k: amp_search_create (H2D of the problem, K0 tables), the
    sharded run + NCCL all-gather + device merge (distributed.search_gpu_sharded),
    the D2H of the k-record result, destroy — wall clock, max over ranks;
    median of the timed steps after one warm-up step, the first (cold-context)
    call reported separately."""
    import torch
    import torch.distributed as dist

    from paper_2210_07297_b200 import distributed as Dd
    from paper_2210_07297_b200.planner import Searcher
    k = TOPK
    h2d = (enc.param.nbytes + enc.flops.nbytes + enc.flops_ok.nbytes + enc.act.nbytes +
           enc.node.nbytes + enc.bw.nbytes + enc.p_layer.nbytes * 3 + enc.p_sec.nbytes)
    d2h = k * 64
    steps = max(1, min(args.steps, 5))
    walls = []
    for i in range(1 + steps):
        if distributed:
            dist.barrier()
        t0 = time.perf_counter()
        s = Searcher(enc, placements_per_class=P_, seed=0, device=local)
        top = Dd.search_gpu_sharded(s, k, rank, world)
        s.close()
        dt = time.perf_counter() - t0
        if distributed:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        walls.append(dt)
    med = float(np.median(walls[1:]))
    return {"value": n_total / med, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "s_per_step": med, "steps": steps,
            "first_call_s": walls[0],
            "best_index": int(top[0]["index"]) if len(top) else None,
            "note": "wall clock per step: amp_search_create (host arrays -> HBM, K0 tables) + "
                    "sharded run + all-gather/merge + host top-k + destroy; median of the steps "
                    "after the first (first_call_s: the first context of the measurement, in a "
                    "process whose CUDA context and memory pool are already up)"}


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        our_arm(args)


if __name__ == "__main__":
    main()
