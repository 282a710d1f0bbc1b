"""Pins the C oracle against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py via oracle/_ref). CPU only.

The restatement follows the reference's evaluation order without FMA
contraction, so agreement is exact up to libm/ulp-level noise (1e-13 rel)."""
import math

import numpy as np
import pytest

from oracle.bind import Mixture, Oracle, reference_available


def close(a, b, rel=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    both_inf = np.isinf(a) & np.isinf(b) & (np.sign(a) == np.sign(b))
    ok = both_inf | (np.abs(a - b) <= rel * np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))
    return ok


def test_bounds_match_reference(golden_bounds):
    for case in golden_bounds["cases"]:
        o = Oracle(Mixture.from_dict(case["mixture"]))
        nodes = np.array(case["nodes"])
        for res in case["results"]:
            lo, up, lm, um, split = o.eval_bounds(nodes, skip=res["skip"])
            assert close(lo, res["lower"]).all(), case["name"]
            assert close(up, res["upper"]).all(), case["name"]
        ok = (np.array(case["split"]) == split)
        assert ok.all(), case["name"]


def test_children_match_reference(golden_bounds):
    for case in golden_bounds["cases"]:
        o = Oracle(Mixture.from_dict(case["mixture"]))
        flag, kids = o.subdivide(np.array(case["nodes"][0]))
        assert np.array_equal(kids, np.array(case["children0"])), case["name"]


def test_objective_matches_reference(golden_objective):
    for case in golden_objective["cases"]:
        o = Oracle(Mixture.from_dict(case["mixture"]))
        assert close(o.self_energy, case["self_energy"]).all()
        for p in case["poses"]:
            assert close(o.objective(p["r"], p["t"]), p["f"]).all(), case["name"]


def test_threaded_batch_is_order_preserving(golden_bounds):
    # test_solver.cpp:281-310: batch == per-branch evaluation for any thread count
    case = golden_bounds["cases"][0]
    o = Oracle(Mixture.from_dict(case["mixture"]))
    nodes = np.array(case["nodes"])
    a = o.eval_bounds(nodes, threads=1)
    b = o.eval_bounds(nodes, threads=4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_oracle_equals_live_reference_on_fresh_inputs():
    from oracle.bind import Reference
    rng = np.random.default_rng(99)
    for n1, n2, kc in [(4, 3, 40.0), (6, 5, 1e4)]:
        mu = rng.normal(size=(n1, 3)) * 1.5 + np.array([0, 0, 3.0])
        s2 = rng.uniform(0.01, 0.3, n1)
        d = rng.normal(size=(n2, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        mix = Mixture([n1], [n2], [1.0], mu, s2, np.full(n1, 1 / n1), d, rng.uniform(1, kc, n2),
                      np.full(n2, 1 / n2), 0.3)
        nodes = np.zeros((200, 11))
        nodes[:, 0:3] = rng.uniform(-2, 2, (200, 3))
        nodes[:, 3] = rng.uniform(0, 1, 200)
        nodes[:, 4:7] = rng.uniform(-1.5, 1.5, (200, 3))
        nodes[:, 7:10] = rng.uniform(0, 1.2, (200, 3))
        nodes[:, 10] = -math.inf
        lo, up, *_ = Oracle(mix).eval_bounds(nodes)
        rlo, rup = Reference(mix).eval_bounds(nodes)
        assert close(lo, rlo).all() and close(up, rup).all()
