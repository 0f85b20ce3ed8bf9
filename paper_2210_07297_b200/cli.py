"""`parplan`-compatible command line over the B200 engine.

    python -m paper_2210_07297_b200.cli plan --model M --cluster C --profile P --gbs N
        [--budget 10] [--workers 0] [--report report.json] [--max-params-per-device X]
        [--bytes-per-param 2] [--fallback-device-flops F] [--fallback-tmp-bandwidth B]
    ... simulate --strategy S.json [--trace T.jsonl]
    ... baseline [--mode layer-balance|param-balance] [--report R]
    ... anneal [--iterations 200] [--seed 0] [--budget 10] [--report R] [--trace T] [--record-all]
    ... gen-profile --model M --device-flops F --tmp 1 2 --mbs 1 2 [--tmp-bandwidth B] [--out P]

Same subcommands, options, outputs and exit codes as the reference CLI
(tools/parplan_main.cpp): 0 ok, 1 error, 3 every candidate failed on a
profile miss (or a profile miss in `simulate`).  `plan` runs the GPU search
(planner.plan) and writes the reference's report.json byte for byte.
"""
from __future__ import annotations

import argparse
import sys
from typing import List, Optional

from . import planner, problem as P, report as R

EXIT_FAILURE = 1
EXIT_PROFILE_MISS = 3


class ProfileMissError(RuntimeError):
    pass


def _positive_int(v: str) -> int:
    x = int(v)
    if x <= 0:
        raise argparse.ArgumentTypeError(f"Value {v} not in range 1 to 2147483647")
    return x


def _positive_float(v: str) -> float:
    x = float(v)
    if x <= 0:
        raise argparse.ArgumentTypeError(f"Value {v} not in range")
    return x


def _add_common(p: argparse.ArgumentParser) -> None:
    """parplan_main.cpp:42-55"""
    p.add_argument("--model", required=True, help="model JSON file")
    p.add_argument("--cluster", required=True, help="cluster JSON file")
    p.add_argument("--profile", required=True, help="profile JSON file")
    p.add_argument("--gbs", required=True, type=_positive_int, help="global batch size")
    p.add_argument("--bytes-per-param", type=float, default=2.0,
                   help="gradient bytes per parameter (default 2, half precision)")
    p.add_argument("--fallback-device-flops", type=float, default=0.0,
                   help="enable the analytic layer-time fallback with this device speed (flops/s)")
    p.add_argument("--fallback-tmp-bandwidth", type=float, default=0.0,
                   help="bandwidth assumed for the fallback's tensor-parallel all-reduce "
                        "(default: infinite)")


def _cost_options(a) -> P.CostModelOptions:
    """parplan_main.cpp:57-69"""
    o = P.CostModelOptions()
    o.bytes_per_param = a.bytes_per_param
    if a.fallback_device_flops > 0:
        o.fallback.enabled = True
        o.fallback.device_flops = a.fallback_device_flops
        if a.fallback_tmp_bandwidth > 0:
            o.fallback.tmp_bandwidth = a.fallback_tmp_bandwidth
    return o


def _abort_if_all_failed(cands) -> int:
    """parplan_main.cpp:71-82"""
    if any(c.failure is None for c in cands):
        return 0
    why = "no candidates" if not cands else cands[0].failure
    sys.stderr.write(f"error: every candidate failed; first failure: {why}\n")
    return EXIT_PROFILE_MISS if "profile miss" in why else EXIT_FAILURE


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(
        prog="parplan",
        description="parplan: searches 3D-parallel training strategies over a layer-graph model "
                    "and a heterogeneous cluster, ranking them with an analytic cost model and "
                    "validating the top picks in a pipeline simulator (B200 engine)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("plan", help="rank all (degrees, mbs) candidates")
    _add_common(p)
    p.add_argument("--budget", type=_positive_int, default=10,
                   help="top candidates validated in the simulator")
    p.add_argument("--workers", type=int, default=0,
                   help="simulation threads (0 = all cores)")
    p.add_argument("--report", default="report.json", help="output report path")
    p.add_argument("--max-params-per-device", type=float, default=0.0,
                   help="fail candidates whose per-device parameter count exceeds this")
    p.add_argument("--device", type=int, default=0, help="CUDA device (engine option)")
    p.add_argument("--gpus", type=int, default=1,
                   help="GPUs driven by the one engine context (devices --device .. +gpus-1)")
    b = sub.add_parser("baseline", help="Megatron-style heuristic candidates")
    _add_common(b)
    b.add_argument("--mode", default="layer-balance", choices=["layer-balance", "param-balance"])
    b.add_argument("--report", default="report.json", help="output report path")
    b.add_argument("--device", type=int, default=0, help="CUDA device (engine option)")
    an = sub.add_parser("anneal", help="simulated-annealing search over domino-tiling placements")
    _add_common(an)
    an.add_argument("--iterations", type=_positive_int, default=200, help="annealing iterations")
    an.add_argument("--seed", type=int, default=0, help="random seed")
    an.add_argument("--budget", type=_positive_int, default=10,
                    help="top recorded strategies to keep and simulate")
    an.add_argument("--report", default="report.json", help="output report path")
    an.add_argument("--trace", default="", help="dump accepted states as JSON lines")
    an.add_argument("--record-all", action="store_true", help="record rejected evaluated states too")
    an.add_argument("--device", type=int, default=0, help="CUDA device (engine option)")
    g = sub.add_parser("gen-profile", help="generate a synthetic profile table from per-layer flops")
    g.add_argument("--model", required=True)
    g.add_argument("--device-flops", required=True, type=_positive_float)
    g.add_argument("--tmp", required=True, type=int, nargs="+")
    g.add_argument("--mbs", required=True, type=int, nargs="+")
    g.add_argument("--tmp-bandwidth", type=float, default=0.0)
    g.add_argument("--out", default="profile.json")
    return ap


def cmd_plan(a) -> int:
    model = P.load_model(a.model)
    cluster = P.load_cluster(a.cluster)
    profile = P.load_profile(a.profile)
    opts = P.PlanOptions(budget=a.budget, workers=a.workers, cost_options=_cost_options(a),
                         max_params_per_device=a.max_params_per_device
                         if a.max_params_per_device > 0 else None)
    res = planner.plan(model, cluster, profile, a.gbs, opts, device=a.device, n_gpus=a.gpus)
    st = _abort_if_all_failed(res.candidates)
    if st:
        return st
    R.write_report(res.candidates, a.report)
    R.print_candidate_table(sys.stdout, res.candidates)
    line = R.best_line(res.candidates, res.best_index)
    if line:
        sys.stdout.write(line + "\n")
    return 0


def cmd_baseline(a) -> int:
    """parplan_main.cpp:285-296 over baseline.megatron_baseline."""
    from . import baseline
    model = P.load_model(a.model)
    cluster = P.load_cluster(a.cluster)
    profile = P.load_profile(a.profile)
    cands = baseline.megatron_baseline(model, cluster, profile, a.gbs, a.mode, _cost_options(a),
                                       device=a.device)
    st = _abort_if_all_failed(cands)
    if st:
        return st
    R.write_report(cands, a.report)
    R.print_candidate_table(sys.stdout, cands)
    return 0


def cmd_anneal(a) -> int:
    """parplan_main.cpp:219-256 over anneal.anneal (chain on the engine)."""
    from . import anneal as A
    from .jsonfmt import dumps_compact
    model = P.load_model(a.model)
    cluster = P.load_cluster(a.cluster)
    profile = P.load_profile(a.profile)
    opts = A.AnnealOptions(iterations=a.iterations, seed=a.seed, budget=a.budget,
                           record_all=a.record_all, cost_options=_cost_options(a))
    try:
        res = A.anneal(model, cluster, profile, a.gbs, opts, device=a.device)
    except A.ProfileMissError as e:
        raise ProfileMissError(str(e))
    cands = []
    for i, t in enumerate(res.top):
        cands.append(planner.CandidateRecord(t.strategy, t.estimated, i + 1, t.simulated))
    R.write_report(cands, a.report)
    R.print_candidate_table(sys.stdout, cands)
    if a.trace:
        try:
            with open(a.trace, "w") as f:
                for e in res.record:
                    line = R.strategy_to_json(e.strategy)
                    line["iteration"] = e.iteration
                    line["accepted"] = e.accepted
                    line["estimated_total"] = float(e.estimated.total)
                    f.write(dumps_compact(line) + "\n")
        except OSError:
            raise P.ParseError(f"cannot open trace file for writing: {a.trace}")
    return 0


def cmd_gen_profile(a) -> int:
    """parplan_main.cpp:170-188 with analytic_layer_time (cost_model.cpp:61-68)."""
    model = P.load_model(a.model)
    t = P.ProfileTable()
    inf = float("inf")
    for l in model.layers:
        for tmp in a.tmp:
            for mbs in a.mbs:
                vol = P.layer_activation_volume(model, l.id) * mbs
                bw = a.tmp_bandwidth if a.tmp_bandwidth > 0 else inf
                t.set(l.id, tmp, mbs, P.analytic_layer_time(l, tmp, mbs, a.device_flops, vol, bw))
    P.write_json_file(P.profile_to_json(t), a.out)
    sys.stdout.write(f"wrote {len(t.entries())} entries to {a.out}\n")
    return 0


def main(argv: Optional[List[str]] = None) -> int:
    a = _parser().parse_args(argv)
    try:
        if a.cmd == "plan":
            return cmd_plan(a)
        if a.cmd == "anneal":
            return cmd_anneal(a)
        if a.cmd == "baseline":
            return cmd_baseline(a)
        if a.cmd == "gen-profile":
            return cmd_gen_profile(a)
    except ProfileMissError as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_PROFILE_MISS
    except (P.ParseError, P.ValidationError, ValueError, OSError) as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_FAILURE
    return EXIT_FAILURE


if __name__ == "__main__":
    sys.exit(main())
