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
