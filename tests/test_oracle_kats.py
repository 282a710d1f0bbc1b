"""Pins the C oracle (oracle/gosma_oracle.c) against the known-answer values
held by the reference's own tests. CPU only."""
import math

import numpy as np
import pytest

from oracle.bind import Mixture, Oracle


def approx(a, b, eps):
    # doctest::Approx rule: |a-b| < eps * (1 + max(|a|, |b|))
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


def toy(kappa1_var=1.0, dir_=(0, 0, 1), kappa2=5.0, zeta=0.5):
    return Oracle(Mixture([1], [1], [1.0], [[0, 0, 2]], [kappa1_var], [1.0], [dir_], [kappa2],
                          [1.0], zeta))


def zref(k):
    return 2.0 if k == 0 else (math.exp(k) - math.exp(-k)) / k


def test_log_z_known_values():
    o = toy()
    # test_sphere_stats.cpp:43-55
    assert approx(math.exp(o.log_z(1.0)), 2.350402387287603, 1e-14)
    assert approx(o.log_z(800.0), 793.315388272332, 1e-12)
    assert approx(math.exp(o.log_z(1e-9)), 2.0, 1e-15)
    # test_sphere_stats.cpp:75-82: log and linear forms agree on [1, 30]
    for i in range(0, 1001, 7):
        k = 1.0 + 29.0 * i / 1000.0
        assert abs(math.log(zref(k)) - o.log_z(k)) < 1e-10


def test_log_z_strictly_increasing():
    o = toy()
    prev = o.log_z(1e-3)
    for i in range(1, 2001):
        k = 1e-3 * (1e6 / 1e-3) ** (i / 2000)
        cur = o.log_z(k)
        assert cur > prev
        prev = cur


def test_psi_trans_known_values():
    o = toy()
    # test_se3.cpp:117-120
    assert approx(o.psi_trans([0, 0, 0], [1, 1, 1], [0, 0, 10]), math.atan2(math.sqrt(2), 9), 1e-14)
    assert approx(o.psi_trans([0, 0, 0], [1, 1, 1], [0.2, 0.9, -0.3]), math.pi, 1.2e-5)


def test_objective_toy_values():
    # test_objective.cpp:121-142
    o = toy()
    f = o.objective([0, 0, 0], [0, 0, 0])
    assert approx(f, -zref(10.0) / (zref(5.0) ** 2), 1e-12)
    assert approx(f, -2.5002, 2e-4)
    oa = toy(dir_=(0, 0, -1))
    fa = oa.objective([0, 0, 0], [0, 0, 0])
    assert approx(fa, zref(10.0) / zref(5.0) ** 2 - 2.0 * 2.0 / zref(5.0) ** 2, 1e-12)
    # standoff: inside zeta -> +inf (the reference throws InfeasiblePoseError)
    assert math.isinf(o.objective([0, 0, 0], [0, 0, 1.7]))


def test_aligned_toy_optimum_value():
    # test_solver.cpp:112-126: f* = -Z(4)/Z(2)^2 at the identity
    o = toy(kappa1_var=4.0, kappa2=2.0)
    z2 = (math.exp(2) - math.exp(-2)) / 2
    z4 = (math.exp(4) - math.exp(-4)) / 4
    assert abs(o.objective([0, 0, 0], [0, 0, 0]) - (-z4 / z2 ** 2)) < 1e-12


def test_kappa_interval_via_zero_rotation_bound():
    # test_bounds.cpp:134-141: kappa in [82, 124] for mu=(0,0,10), sigma2=1, unit box.
    # The oracle's LB on a single-pair context uses exactly these endpoints; the
    # diagonal term phi^2 * klo/2 * coth(klo) exposes klo.
    o = Oracle(Mixture([1], [1], [1.0], [[0, 0, 10]], [1.0], [1.0], [[0, 0, 1]], [1.0], [1.0], 0.5))
    node = np.array([0, 0, 0, 0, 0, 0, 0, 1, 1, 1, -np.inf])
    lo, up, lm, um, sr = o.eval_bounds(node)
    # lm = diag + 2*cross; cross <= ... ; diag alone = 0.5*82*coth(82) = 41
    assert lm[0] >= 41.0 - 1e-9


def test_zero_size_branch_collapses(golden_bounds):
    # test_bounds.cpp:278-295: zero-size branch -> upper == f(centre), lower ~ f
    for case in golden_bounds["cases"]:
        mix = Mixture.from_dict(case["mixture"])
        o = Oracle(mix)
        nodes = np.array(case["nodes"])
        z = (nodes[:, 3] == 0) & (np.all(nodes[:, 7:10] == 0, axis=1))
        for node in nodes[z]:
            lo, up, *_ = o.eval_bounds(node)
            f = o.objective(node[0:3], node[4:7])
            if math.isinf(f):
                continue
            assert up[0] == f
            assert abs(lo[0] - f) <= 1e-12 * (1 + abs(f))


def test_subdivision_geometry():
    # test_se3.cpp:168-214
    o = Oracle(Mixture([1], [1], [1.0], [[0, 0, 5]], [1.0], [1.0], [[0, 0, 1]], [1.0], [1.0], 0.5))
    parent = np.array([0, 0, 0, math.pi, 0, 0, 0, 0.01, 0.01, 0.01, -3.5])
    flag, kids = o.subdivide(parent)
    assert flag == 1
    assert np.allclose(kids[:, 3], math.pi / 2)
    assert np.all(kids[:, 10] == -3.5)
    parent2 = np.array([0, 0, 0, 1e-4, 0, 0, 0, 2, 2, 2, -1.0])
    flag, kids = o.subdivide(parent2)
    assert flag == 0 and np.all(kids[:, 7:10] == 1.0)
    vol = lambda n: (2 * n[3]) ** 3 * np.prod(2 * n[7:10])  # noqa: E731
    assert abs(sum(vol(k) for k in kids) - vol(parent2)) < 1e-12 * vol(parent2)
    flag, _ = o.subdivide(np.array([0, 0, 0, 1e-12, 0, 0, 0, 1e-12, 1e-12, 1e-12, 0.0]))
    assert flag == -1


def test_context_validation():
    with pytest.raises(ValueError):
        Oracle(Mixture([1], [1], [1.0], [[0, 0, 2]], [1.0], [0.9], [[0, 0, 1]], [5.0], [1.0], 0.5))
    with pytest.raises(ValueError):
        Oracle(Mixture([1], [1], [1.0], [[0, 0, 2]], [1.0], [1.0], [[0, 0, 2]], [5.0], [1.0], 0.5))
    with pytest.raises(ValueError):
        Oracle(Mixture([1], [1], [1.0], [[0, 0, 2]], [1.0], [1.0], [[0, 0, 1]], [5.0], [1.0], 0.0))
