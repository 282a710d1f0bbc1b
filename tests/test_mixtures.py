"""Mixture construction (host C++ port of mixtures.cpp:49-362) against the
unmodified reference (oracle/_ref) — bit-identical clusterings and mixtures —
plus the reference's own test_mixtures.cpp scenarios. CPU only."""
import math

import numpy as np
import pytest

import paper_1812_01232_b200 as g
from oracle.bind import reference_available, reference_build_mixtures, reference_dp_means

needs_ref = pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")


def unit(v):
    v = np.asarray(v, float)
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def scene(rng, n_pts=60, n_brg=50, spread=1.0, clusters=5):
    centres = rng.normal(size=(clusters, 3)) * 2.0
    pts = centres[rng.integers(0, clusters, n_pts)] + rng.normal(size=(n_pts, 3)) * 0.1 * spread
    axes = unit(rng.normal(size=(clusters, 3)))
    brg = unit(axes[rng.integers(0, clusters, n_brg)] + rng.normal(size=(n_brg, 3)) * 0.02)
    return pts, brg


@needs_ref
@pytest.mark.parametrize("seed", [None, 0, 7, 12345])
def test_dp_means_bit_identical(seed):
    rng = np.random.default_rng(3 if seed is None else seed + 1)
    for lam in (0.05, 0.3, 1.5, 10.0):
        pts, brg = scene(rng, 120, 90)
        a, c, it = g.dp_means(pts, lam, seed)
        ra, rc, rit = reference_dp_means(pts, lam, seed)
        assert np.array_equal(a, ra) and np.array_equal(c, rc) and it == rit
        for lf in (0.01, 0.2, 1.0):
            a, c, it = g.dp_vmf_means(brg, lf, seed)
            ra, rc, rit = reference_dp_means(brg, lf, seed, vmf=True)
            assert np.array_equal(a, ra) and np.array_equal(c, rc) and it == rit


def same_classes(mine, ref):
    assert len(mine) == len(ref)
    for m, r in zip(mine, ref):
        assert m["id"] == r["id"] and m["weight"] == r["weight"]
        for k in ("mu", "sigma2", "phi1", "dir", "kappa2", "phi2"):
            assert np.array_equal(np.asarray(m[k]), np.asarray(r[k])), k


@needs_ref
def test_build_semantic_mixtures_unlabeled_bit_identical():
    rng = np.random.default_rng(11)
    for _ in range(5):
        pts, brg = scene(rng)
        for lp, lf in ((0.25, math.radians(2.0)), (0.5, 0.1), (2.0, 0.5)):
            mine, w = g.build_semantic_mixtures(pts, brg, lp, lf)
            ref, rw = reference_build_mixtures(pts, brg, lp, lf)
            same_classes(mine, ref)
            assert w == rw == [] and mine[0]["id"] == "all" and mine[0]["weight"] == 1.0


@needs_ref
def test_build_semantic_mixtures_labeled_weights_and_warnings():
    rng = np.random.default_rng(12)
    pts, brg = scene(rng, 200, 150, clusters=8)
    plab = [["chair", "table", "lamp", "10", "9"][i % 5] for i in range(len(pts))]
    blab = [["chair", "table", "door", "10", "9"][i % 5] for i in range(len(brg))]
    mine, w = g.build_semantic_mixtures(pts, brg, 0.3, 0.05, plab, blab)
    ref, rw = reference_build_mixtures(pts, brg, 0.3, 0.05, plab, blab)
    same_classes(mine, ref)
    assert w == rw and len(w) == 2  # lamp has no bearings, door has no points
    assert [c["id"] for c in mine] == ["10", "9", "chair", "table"]  # std::map order
    weights = {"chair": 2.0, "table": 1.0, "10": 0.5, "9": 0.5}
    mine, _ = g.build_semantic_mixtures(pts, brg, 0.3, 0.05, plab, blab, weights)
    ref, _ = reference_build_mixtures(pts, brg, 0.3, 0.05, plab, blab, weights)
    same_classes(mine, ref)
    assert abs(sum(c["weight"] for c in mine) - 1.0) < 1e-12


def test_mixtures_feed_objective_context_shape():
    rng = np.random.default_rng(13)
    pts, brg = scene(rng)
    classes, _ = g.build_semantic_mixtures(pts, brg, 0.25, math.radians(2.0))
    c = classes[0]
    assert c["mu"].shape[1] == 3 and c["dir"].shape[1] == 3
    assert abs(c["phi1"].sum() - 1.0) < 1e-12 and abs(c["phi2"].sum() - 1.0) < 1e-12
    assert np.all(c["sigma2"] >= (0.25 / 10) ** 2)
    assert np.all((c["kappa2"] >= 1e-3) & (c["kappa2"] <= 1e5))


def test_reference_scenarios_from_test_mixtures_cpp():
    # dp_means blob separation (test_mixtures.cpp:63-109)
    blobs = np.array([[0, 0, 0], [0.1, 0, 0], [0, 0.1, 0], [5, 5, 5], [5.1, 5, 5], [5, 5.1, 5]],
                     float)
    a, c, _ = g.dp_means(blobs, 100.0)
    assert len(c) == 1
    a, c, _ = g.dp_means(blobs, 1.0)
    assert len(c) == 2 and a[0] == a[1] == a[2] and a[3] == a[4] == a[5] and a[0] != a[3]
    for b in range(2):
        assert np.linalg.norm(c[a[3 * b]] - blobs[3 * b:3 * b + 3].mean(0)) < 1e-12
    a1, c1, _ = g.dp_means(blobs, 1.0, 42)
    a2, c2, _ = g.dp_means(blobs, 1.0, 42)
    assert np.array_equal(a1, a2) and np.array_equal(c1, c2)
    with pytest.raises(ValueError):
        g.dp_means(np.zeros((0, 3)), 1.0)
    with pytest.raises(ValueError):
        g.dp_means(blobs, 0.0)
    # dp_vmf_means (test_mixtures.cpp:136-186)
    one = unit([[0.0, 0.0, 1.0]])
    a, c, _ = g.dp_vmf_means(np.repeat(one, 3, 0), 0.1)
    assert len(c) == 1 and np.linalg.norm(c[0] - [0, 0, 1]) < 1e-12
    with pytest.raises(ValueError):
        g.dp_vmf_means(one, 0.0)
    with pytest.raises(ValueError):
        g.dp_vmf_means(one, 4.0)
    with pytest.raises(ValueError):
        g.dp_vmf_means(np.array([[0.0, 0.0, 1.1]]), 0.1)  # UnitVector3: |v| off by > 1e-6
    # assembly errors (test_mixtures.cpp:261-330)
    pts = np.array([[0.0, 0.0, 1.0], [1.0, 0.0, 1.0]])
    brg = unit([[0.0, 0.0, 1.0], [0.1, 0.0, 1.0]])
    with pytest.raises(ValueError):
        g.build_semantic_mixtures(pts, brg, 0.25, 0.05, ["a", "b"], None)
    with pytest.raises(ValueError):
        g.build_semantic_mixtures(pts, brg, 0.25, 0.05, ["a", "a"], ["b", "b"])
    with pytest.raises(ValueError):
        g.build_semantic_mixtures(pts, brg, 0.25, 0.05, ["a", "a"], ["a", "a"], {"a": -1.0})
    with pytest.raises(ValueError):
        g.build_semantic_mixtures(pts, brg, 0.25, 0.05, ["a", "a"], ["a", "a"], {"b": 1.0})
    cls, w = g.build_semantic_mixtures(pts, brg, 0.25, 0.05, ["chair", "chair"],
                                       ["chair", "chair"])
    assert len(cls) == 1 and cls[0]["id"] == "chair" and cls[0]["weight"] == 1.0 and not w


def room_cloud(rng, n, size=(8.0, 6.0, 3.0), noise=0.01):
    """Points on the six faces of a box room (a real-data-like surface cloud,
    the paper's 100k-point setting)."""
    size = np.asarray(size)
    face = rng.integers(0, 6, n)
    p = rng.uniform(0, 1, (n, 3)) * size
    axis = face // 2
    p[np.arange(n), axis] = np.where(face % 2 == 0, 0.0, size[axis])
    return p - size / 2 + rng.normal(size=(n, 3)) * noise


@pytest.mark.gpu
@needs_ref
def test_dp_means_at_scale_gpu_bit_identical(gosma):
    """(f)3 mixture construction at scale: 100k room points (lambda_p = 0.25)
    and 100k bearings (lambda_f = 2 deg). The sweeps score the fixed centres
    on the GPU (auto from 4e6 scores per sweep) and admit new centres in
    visit order on the host: the clustering is bit-identical to the
    unmodified reference's dp_means / dp_vmf_means."""
    import time
    rng = np.random.default_rng(2024)
    pts = room_cloud(rng, 100_000)
    t0 = time.perf_counter()
    a, c, it = g.dp_means(pts, 0.25, 7)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    ra, rc, rit = reference_dp_means(pts, 0.25, 7)
    t_ref = time.perf_counter() - t0
    print(f"dp_means 100k points: {len(c)} centres, {it} sweeps, GPU-assisted {t_gpu:.2f} s, "
          f"reference {t_ref:.2f} s")
    assert np.array_equal(a, ra) and np.array_equal(c, rc) and it == rit
    brg = unit(pts - np.array([0.3, -0.2, 0.1]))
    a, c, it = g.dp_vmf_means(brg, math.radians(2.0), None)
    ra, rc, rit = reference_dp_means(brg, math.radians(2.0), None, vmf=True)
    assert np.array_equal(a, ra) and np.array_equal(c, rc) and it == rit
