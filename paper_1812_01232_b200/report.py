"""Solver report / trace files in the reference's formats (io.cpp:598-694):
JSON (ordered keys, pose as angle-axis + rotation matrix + translation, stats,
trace, config echo) and the trace CSV with 17 significant digits (fmt17,
io.cpp:409-413), so tools that read the reference's outputs read these."""
from __future__ import annotations

import dataclasses
import json
import math
from typing import Dict, List, Optional

import numpy as np

from .host import rotation_matrix

EPSILON_INTERPRETATION = ("absolute gap on the objective value (weights are normalized, so the "
                          "objective is scale-free)")  # solver.cpp:332-334

TRACE_FIELDS = ("wave", "bound_evaluations", "best_upper", "global_lower", "queue_size",
                "unexplored_volume_fraction", "pruned_volume_fraction",
                "resolved_volume_fraction")


def fmt17(v: float) -> str:
    return "%.17g" % v


@dataclasses.dataclass
class RunConfig:
    """The effective settings of one run (io.hpp:22-55): the config-file keys
    after defaulting, angles in radians."""
    points_path: str = ""
    bearings_path: str = ""
    output_path: str = "smalign_report.json"
    focal: Optional[float] = None
    principal: tuple = (0.0, 0.0)
    lambda_p: float = 0.25
    lambda_f: float = 2.0 * math.pi / 180.0
    epsilon: float = 0.1
    zeta: float = 0.5
    torus_major: Optional[float] = None
    torus_minor: Optional[float] = None
    translation_boxes: List[tuple] = dataclasses.field(default_factory=list)
    rotation_center: tuple = (0.0, 0.0, 0.0)
    rotation_half_width: float = math.pi
    class_weights: Dict[str, float] = dataclasses.field(default_factory=dict)
    max_evaluations: Optional[int] = None
    time_limit_seconds: Optional[float] = None
    queue_capacity: Optional[int] = None
    batch_size: int = 1024
    threads: int = 0
    seed: int = 0


def config_echo(cfg: RunConfig) -> dict:
    """The report's config block (io.cpp:422-462): keyed and scaled like the
    config file (angles in degrees), optional keys only when set, so the block
    reproduces the run."""
    deg = math.pi / 180.0
    j = {}
    if cfg.points_path:
        j["points"] = cfg.points_path
    if cfg.bearings_path:
        j["bearings"] = cfg.bearings_path
    j["output"] = cfg.output_path
    if cfg.focal is not None:
        j["focal"] = float(cfg.focal)
        j["principal_x"] = float(cfg.principal[0])
        j["principal_y"] = float(cfg.principal[1])
    j["lambda_p"] = float(cfg.lambda_p)
    j["lambda_f"] = cfg.lambda_f / deg
    j["epsilon"] = float(cfg.epsilon)
    j["zeta"] = float(cfg.zeta)
    if cfg.torus_major is not None:
        j["torus_major"] = float(cfg.torus_major)
    if cfg.torus_minor is not None:
        j["torus_minor"] = float(cfg.torus_minor)
    if cfg.translation_boxes:
        j["translation_box"] = [[float(x) for x in b] for b in cfg.translation_boxes]
    j["rotation_center"] = [float(x) for x in cfg.rotation_center]
    j["rotation_half_width"] = cfg.rotation_half_width / deg
    if cfg.class_weights:
        j["class_weight"] = {k: float(cfg.class_weights[k]) for k in sorted(cfg.class_weights)}
    if cfg.max_evaluations is not None:
        j["max_evaluations"] = int(cfg.max_evaluations)
    if cfg.time_limit_seconds is not None:
        j["time_limit"] = float(cfg.time_limit_seconds)
    j["batch_size"] = int(cfg.batch_size)
    if cfg.queue_capacity is not None:
        j["queue_capacity"] = int(cfg.queue_capacity)
    j["threads"] = int(cfg.threads)
    j["seed"] = int(cfg.seed)
    return j


def _config_echo(config) -> dict:
    if config is None:
        return {}
    if isinstance(config, RunConfig):
        return config_echo(config)
    if dataclasses.is_dataclass(config):
        return {k: v for k, v in dataclasses.asdict(config).items()}
    return dict(config)


def _num(v: float):
    """JSON number, or null for a non-finite value (nlohmann's encoding)."""
    v = float(v)
    return v if math.isfinite(v) else None


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
        "best_value": _num(report.best_value),
        "global_lower": _num(report.global_lower),
        "gap": _num(report.gap),
        "status": report.status,
        "epsilon_interpretation": EPSILON_INTERPRETATION,
        "pose": {"angle_axis": [float(x) for x in report.r],
                 "rotation_matrix": [[float(x) for x in row] for row in R],
                 "translation": [float(x) for x in report.t]},
        "stats": {"branches_expanded": int(report.branches_expanded),
                  "sma_invocations": int(report.sma_invocations),
                  "bound_evaluations": int(report.bound_evaluations),
                  "wall_time_seconds": float(report.wall_time_seconds)},
        "trace": [dict(zip(TRACE_FIELDS, (int(t[0]), int(t[1]), _num(t[2]), _num(t[3]),
                                          int(t[4]), _num(t[5]), _num(t[6]), _num(t[7]))))
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
