"""Report / trace files in the reference's formats (io.cpp:598-694)."""
import csv
import json
import math

import numpy as np

from paper_1812_01232_b200 import SolverConfig, SolverReport
from paper_1812_01232_b200.report import TRACE_FIELDS, read_report, write_report


def fake_report():
    return SolverReport(r=np.array([0.1, -0.2, 0.3]), t=np.array([1.0, 2.0, -0.5]),
                        best_value=-2.3196510724049677, global_lower=-2.7624255547532943,
                        gap=0.44277448235, status="epsilon_optimal", branches_expanded=12,
                        sma_invocations=4, bound_evaluations=17788906,
                        wall_time_seconds=0.119, waves=2,
                        trace=[(0, 100, -2.1, -9.0, 44, 1.0, 0.0, 0.0),
                               (1, 900, -2.3196510724049677, -2.7624255547532943, 300,
                                0.5, 0.25, 0.25)])


def test_json_report_round_trips_with_reference_keys(tmp_path):
    rep = fake_report()
    p = tmp_path / "r.json"
    write_report(rep, str(p), "json", SolverConfig(epsilon=0.1, zeta=0.5))
    j = json.loads(p.read_text())
    assert list(j) == ["best_value", "global_lower", "gap", "status", "epsilon_interpretation",
                       "pose", "stats", "trace", "config"]
    assert j["best_value"] == rep.best_value  # exact round trip
    r = read_report(str(p))
    R = r["pose"]["rotation_matrix"]
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-12)
    assert list(j["trace"][1]) == list(TRACE_FIELDS)
    assert j["config"]["epsilon"] == 0.1


def test_trace_csv_17_digits(tmp_path):
    rep = fake_report()
    p = tmp_path / "t.csv"
    write_report(rep, str(p), "trace_csv")
    rows = list(csv.reader(open(p)))
    assert tuple(rows[0]) == TRACE_FIELDS
    assert rows[2][2] == "%.17g" % -2.3196510724049677
    assert float(rows[2][3]) == -2.7624255547532943 and not math.isnan(float(rows[1][5]))


def _ref_report_tool():
    import os
    from oracle.bind import HERE
    exe = os.path.join(HERE, "_ref", "ref_report")
    return exe if os.path.exists(exe) else None


def test_reports_match_the_reference_writer(tmp_path):
    """f4: the reference's own write_report (io.cpp:598-652, config_echo
    422-462, compiled into oracle/_ref) and this package's writer produce the
    same JSON document (same keys in the same order, same values; the rotation
    matrix to 1e-15, it is recomputed from the angle-axis on each side) and a
    byte-identical trace CSV, for the same report and config."""
    import subprocess
    import pytest
    from paper_1812_01232_b200.report import EPSILON_INTERPRETATION, RunConfig
    tool = _ref_report_tool()
    if tool is None:
        pytest.skip("reference report writer not built (oracle/_ref/ref_report, needs io.cpp)")
    cfg_text = """points = scene.ply
bearings = pixels.txt
output = out.json
focal = 800
principal_x = 320
principal_y = 240
lambda_p = 0.25
lambda_f = 2
epsilon = 0.1
zeta = 0.5
torus_major = 3.5
torus_minor = 0.5
translation_box = 0.5 -1 2 0.25 0.25 0.5
rotation_center = 0.1 0.2 0.3
rotation_half_width = 90
class_weight = wall 2
class_weight = chair 1
max_evaluations = 1000000
time_limit = 60
batch_size = 512
queue_capacity = 100000
threads = 8
seed = 7
"""
    cfg_path = tmp_path / "run.cfg"
    cfg_path.write_text(cfg_text)
    deg = math.pi / 180.0
    cfg = RunConfig(points_path="scene.ply", bearings_path="pixels.txt", output_path="out.json",
                    focal=800.0, principal=(320.0, 240.0), lambda_p=0.25, lambda_f=2.0 * deg,
                    epsilon=0.1, zeta=0.5, torus_major=3.5, torus_minor=0.5,
                    translation_boxes=[(0.5, -1.0, 2.0, 0.25, 0.25, 0.5)],
                    rotation_center=(0.1, 0.2, 0.3), rotation_half_width=90.0 * deg,
                    class_weights={"wall": 2.0, "chair": 1.0}, max_evaluations=1000000,
                    time_limit_seconds=60.0, batch_size=512, queue_capacity=100000, threads=8,
                    seed=7)
    rep = fake_report()
    rep.trace.insert(0, (0, 44, math.inf, -math.inf, 44, 1.0, 0.0, 0.0))
    f17 = lambda xs: " ".join("%.17g" % float(x) for x in xs)  # noqa: E731
    vals_path = tmp_path / "values.txt"
    vals_path.write_text(
        f17([rep.best_value, rep.global_lower, rep.gap, *rep.r, *rep.t, rep.wall_time_seconds])
        + "\n" + f"0 {rep.branches_expanded} {rep.sma_invocations} {rep.bound_evaluations}\n"
        + EPSILON_INTERPRETATION + "\n" + "".join(f17(t) + "\n" for t in rep.trace))
    for csv_mode, name in ((0, "json"), (1, "csv")):
        ref_path = tmp_path / f"ref.{name}"
        ours_path = tmp_path / f"ours.{name}"
        rc = subprocess.run([tool, str(cfg_path), str(vals_path), str(ref_path), name],
                            timeout=60).returncode
        assert rc == 0
        write_report(rep, str(ours_path), "trace_csv" if csv_mode else "json", cfg)
        if csv_mode:
            assert ours_path.read_bytes() == ref_path.read_bytes()
            continue
        a, b = json.loads(ours_path.read_text()), json.loads(ref_path.read_text())
        Ra, Rb = np.array(a["pose"].pop("rotation_matrix")), np.array(b["pose"].pop("rotation_matrix"))
        assert np.max(np.abs(Ra - Rb)) <= 1e-15
        assert list(a) == list(b) and list(a["config"]) == list(b["config"])
        assert a == b
