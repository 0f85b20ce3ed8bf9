"""report.json and the ranked table of the CLI (reference report.cpp).

`report_to_json` / `report_from_json` mirror report.cpp:28-83,
`write_report` report.cpp:85-91 and `print_candidate_table`
report.cpp:101-128, so the drop-in CLI's outputs match the reference
byte for byte (tests/golden/reports/).
"""
from __future__ import annotations

import json
from typing import List, Optional, TextIO

from .jsonfmt import dumps
from .planner import CandidateRecord, CostBreakdown, Strategy
from .problem import ParseError


def strategy_to_json(s: Strategy) -> dict:
    """json_io.cpp:210-227: placement nested [stage][replica][shard]."""
    placement = [[[int(s.device_at(i, r, sh)) for sh in range(s.tmp)] for r in range(s.dp)]
                 for i in range(s.pp)]
    return {"degrees": {"pp": s.pp, "dp": s.dp, "tmp": s.tmp}, "placement": placement,
            "mbs": s.mbs, "assignment": [int(c) for c in s.cut_boundaries]}


def strategy_from_json(j: dict) -> Strategy:
    """json_io.cpp:148-175"""
    try:
        deg = j.get("degrees", {})
        pp, dp, tmp = int(deg["pp"]), int(deg["dp"]), int(deg["tmp"])
        flat = [int(d) for stage in j["placement"] for rep in stage for d in rep]
        return Strategy(pp, dp, tmp, int(j["mbs"]), flat, [int(c) for c in j["assignment"]])
    except (KeyError, TypeError, ValueError) as e:
        raise ParseError(f"strategy: {e}")


def report_to_json(candidates: List[CandidateRecord]) -> dict:
    out = []
    for rec in candidates:
        s = rec.strategy
        if rec.failure is not None:
            # a failed candidate never got a placement or assignment
            e = {"degrees": {"pp": s.pp, "dp": s.dp, "tmp": s.tmp}, "mbs": s.mbs,
                 "failure": rec.failure}
        else:
            e = strategy_to_json(s)
            e["estimated"] = {"total": float(rec.estimated.total),
                              "pipeline_time": float(rec.estimated.pipeline_time),
                              "dpsync_time": float(rec.estimated.dpsync_time)}
        e["rank"] = int(rec.rank)
        if rec.simulated is not None:
            e["simulated"] = float(rec.simulated)
        out.append(e)
    return {"candidates": out}


def report_from_json(j: dict) -> List[CandidateRecord]:
    out = []
    for e in j["candidates"]:
        if "failure" in e:
            d = e["degrees"]
            rec = CandidateRecord(Strategy(int(d["pp"]), int(d["dp"]), int(d["tmp"]), int(e["mbs"])),
                                  CostBreakdown(), failure=str(e["failure"]))
        else:
            est = e["estimated"]
            rec = CandidateRecord(strategy_from_json(e),
                                  CostBreakdown(float(est["pipeline_time"]), float(est["dpsync_time"]),
                                                float(est["total"])))
        rec.rank = int(e["rank"])
        if "simulated" in e:
            rec.simulated = float(e["simulated"])
        out.append(rec)
    return out


def write_report(candidates: List[CandidateRecord], path: str) -> None:
    try:
        with open(path, "w") as f:
            f.write(dumps(report_to_json(candidates)) + "\n")
    except OSError:
        raise ParseError(f"cannot open report for writing: {path}")


def load_report(path: str) -> List[CandidateRecord]:
    try:
        with open(path) as f:
            return report_from_json(json.load(f))
    except OSError:
        raise ParseError(f"cannot open report: {path}")


def _w(v, width: int) -> str:  # std::left << std::setw(width)
    return str(v).ljust(width)


def print_candidate_table(out: TextIO, candidates: List[CandidateRecord]) -> None:
    out.write(_w("rank", 5) + _w("pp", 4) + _w("dp", 4) + _w("tmp", 5) + _w("mbs", 5) +
              _w("est_total", 13) + _w("pipeline", 13) + _w("dpsync", 13) + _w("simulated", 13) +
              "assignment\n")
    for rec in candidates:
        s = rec.strategy
        out.write(_w(rec.rank, 5) + _w(s.pp, 4) + _w(s.dp, 4) + _w(s.tmp, 5) + _w(s.mbs, 5))
        if rec.failure is not None:
            out.write("failed: " + rec.failure + "\n")
            continue

        def fmt(v: float) -> str:  # std::fixed << std::setprecision(6)
            return f"{v:.6f}"
        out.write(_w(fmt(rec.estimated.total), 13) + _w(fmt(rec.estimated.pipeline_time), 13) +
                  _w(fmt(rec.estimated.dpsync_time), 13) +
                  _w(fmt(rec.simulated) if rec.simulated is not None else "-", 13))
        out.write("[" + ",".join(str(int(c)) for c in s.cut_boundaries) + "]\n")


def best_line(candidates: List[CandidateRecord], best_index: int) -> Optional[str]:
    if best_index >= 0:
        return f"best by simulation: rank {candidates[best_index].rank}"
    return None
