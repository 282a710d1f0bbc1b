"""Solver report / trace files in the reference's formats (io.cpp:598-694):
JSON (ordered keys, pose as angle-axis + rotation matrix + translation, stats,
trace, config echo) and the trace CSV with 17 significant digits (fmt17,
io.cpp:409-413), so tools that read the reference's outputs read these."""
from __future__ import annotations

import dataclasses
import json
from typing import Optional

import numpy as np

from .host import rotation_matrix

EPSILON_INTERPRETATION = ("absolute gap on the objective value (weights are normalized, so the "
                          "objective is scale-free)")  # solver.cpp:332-334

TRACE_FIELDS = ("wave", "bound_evaluations", "best_upper", "global_lower", "queue_size",
                "unexplored_volume_fraction", "pruned_volume_fraction",
                "resolved_volume_fraction")


def fmt17(v: float) -> str:
    return "%.17g" % v


def _config_echo(config) -> dict:
    if config is None:
        return {}
    if dataclasses.is_dataclass(config):
        return {k: v for k, v in dataclasses.asdict(config).items()}
    return dict(config)


def write_report(report, path: str, fmt: str = "json", config: Optional[object] = None):
    """write_report (io.cpp:598-652): fmt "json" or "trace_csv"."""
    if fmt == "trace_csv":
        with open(path, "w", newline="\n") as f:
            f.write(",".join(TRACE_FIELDS) + "\n")
            for (w, e, ub, lb, q, fu, fp, fr) in report.trace:
                f.write(f"{int(w)},{int(e)},{fmt17(ub)},{fmt17(lb)},{int(q)},{fmt17(fu)},"
                        f"{fmt17(fp)},{fmt17(fr)}\n")
        return
    if fmt != "json":
        raise ValueError(f"unknown report format {fmt!r}")
    R = rotation_matrix(report.r)
    j = {
        "best_value": float(report.best_value),
        "global_lower": float(report.global_lower),
        "gap": float(report.gap),
        "status": report.status,
        "epsilon_interpretation": EPSILON_INTERPRETATION,
        "pose": {"angle_axis": [float(x) for x in report.r],
                 "rotation_matrix": [[float(x) for x in row] for row in R],
                 "translation": [float(x) for x in report.t]},
        "stats": {"branches_expanded": int(report.branches_expanded),
                  "sma_invocations": int(report.sma_invocations),
                  "bound_evaluations": int(report.bound_evaluations),
                  "wall_time_seconds": float(report.wall_time_seconds)},
        "trace": [dict(zip(TRACE_FIELDS, (int(t[0]), int(t[1]), float(t[2]), float(t[3]),
                                          int(t[4]), float(t[5]), float(t[6]), float(t[7]))))
                  for t in report.trace],
        "config": _config_echo(config),
    }
    with open(path, "w") as f:
        f.write(json.dumps(j, indent=2) + "\n")


def read_report(path: str) -> dict:
    """read_report (io.cpp:654-694): the JSON report as a dict (pose arrays as numpy)."""
    with open(path) as f:
        j = json.load(f)
    j["pose"]["angle_axis"] = np.array(j["pose"]["angle_axis"])
    j["pose"]["translation"] = np.array(j["pose"]["translation"])
    j["pose"]["rotation_matrix"] = np.array(j["pose"]["rotation_matrix"])
    return j
