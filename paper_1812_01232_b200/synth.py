"""Synthetic workloads for the bound-kernel microbench and the parity tests
(BASELINE.json configs[1]; SURVEY.md §8(d) "Config 2").

Mixtures (seeded numpy, uniform weights):
* ``moderate``  — the reference's random_context recipe
  (tests/test_bounds.cpp:18-34): means 1.5·N(0,I) resampled until |mu| >= 0.8,
  sigma^2 = d^2/(0.8·cap - 1)·U(1,3) with d = |mu| + 3, kappa2 ~ U(1, 0.8·cap).
* ``realistic`` — what fitted scenes produce (mixtures.cpp:256-257, 289):
  means U[-1,1]^3, sigma^2 log-uniform in [6.25e-4, 0.05], image directions
  within a 40° cone, kappa2 log-uniform in [1e2, 1e5].

Nodes: rotation cubes at octree levels 1-6 of [-pi, pi]^3 (random cells),
translation cuboids from torus_cover(3.5, 0.5) (se3.cpp:155-175) subdivided
0-3 levels (random cells), parent lower bound -inf.
"""
from __future__ import annotations

import math

import numpy as np

from . import NODE_DTYPE


def torus_cover(major: float = 3.5, minor: float = 0.5) -> np.ndarray:
    """torus_cover (se3.cpp:155-175): rows {center[3], half_widths[3]}."""
    if not (major > 0.0 and minor > 0.0 and minor < major):
        raise ValueError("torus_cover: need 0 < minor < major")
    n = int(math.ceil(2.0 * math.pi * major / minor))
    hw = minor + 2.0 * major * math.sin(math.pi / (2.0 * n))
    boxes = np.zeros((n, 6))
    for k in range(n):
        a = 2.0 * math.pi * k / n
        boxes[k, :3] = (major * math.cos(a), major * math.sin(a), 0.0)
        boxes[k, 3:] = hw
    return boxes


def mixture(n1: int, n2: int, regime: str = "realistic", seed: int = 2026,
            kappa_cap: float = 150.0, n_classes: int = 1):
    """Returns a list of class dicts for ObjectiveContext (uniform class weights)."""
    rng = np.random.default_rng(seed)
    classes = []
    for _ in range(n_classes):
        if regime == "moderate":
            mu = np.empty((n1, 3))
            for i in range(n1):
                m = rng.normal(size=3) * 1.5
                while np.linalg.norm(m) < 0.8:
                    m = rng.normal(size=3) * 1.5
                mu[i] = m
            d = np.linalg.norm(mu, axis=1) + 3.0
            sigma2 = d * d / (0.8 * kappa_cap - 1.0) * rng.uniform(1.0, 3.0, n1)
            dirs = rng.normal(size=(n2, 3))
            dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
            kappa2 = rng.uniform(1.0, 0.8 * kappa_cap, n2)
        elif regime == "realistic":
            mu = rng.uniform(-1.0, 1.0, (n1, 3))
            sigma2 = np.exp(rng.uniform(np.log(6.25e-4), np.log(0.05), n1))
            axis = np.array([0.0, 0.0, 1.0])
            cosmax = math.cos(math.radians(40.0))
            ct = rng.uniform(cosmax, 1.0, n2)
            ph = rng.uniform(0.0, 2 * math.pi, n2)
            st = np.sqrt(1.0 - ct * ct)
            dirs = np.stack([st * np.cos(ph), st * np.sin(ph), ct * axis[2]], axis=1)
            dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
            kappa2 = np.exp(rng.uniform(np.log(1e2), np.log(1e5), n2))
        else:
            raise ValueError(f"unknown regime {regime!r}")
        classes.append({"mu": mu, "sigma2": sigma2, "phi1": np.full(n1, 1.0 / n1), "dir": dirs,
                        "kappa2": kappa2, "phi2": np.full(n2, 1.0 / n2),
                        "weight": 1.0 / n_classes})
    return classes


def nodes(n: int, seed: int = 2026, rot_levels=(1, 6), trans_levels=(0, 3),
          major: float = 3.5, minor: float = 0.5) -> np.ndarray:
    """n random sub-cubes: rotation octree cells x subdivided torus boxes."""
    rng = np.random.default_rng(seed)
    out = np.empty(n, dtype=NODE_DTYPE)
    kr = rng.integers(rot_levels[0], rot_levels[1] + 1, n)
    cells = 2 ** kr
    hw = math.pi / cells
    idx = rng.integers(0, cells[:, None], (n, 3))
    out["rc"] = -math.pi + (2 * idx + 1) * hw[:, None]
    out["rhw"] = hw
    boxes = torus_cover(major, minor)
    b = rng.integers(0, boxes.shape[0], n)
    kt = rng.integers(trans_levels[0], trans_levels[1] + 1, n)
    tcells = 2 ** kt
    thw = boxes[b, 3:] / tcells[:, None]
    tidx = rng.integers(0, tcells[:, None], (n, 3))
    out["tc"] = boxes[b, :3] - boxes[b, 3:] + (2 * tidx + 1) * thw
    out["thw"] = thw
    out["lower"] = -np.inf
    return out


def pair_terms_per_node(classes) -> int:
    """P = sum_c n1c*n2c + n1c(n1c-1)/2 (SURVEY.md §8 notation)."""
    p = 0
    for c in classes:
        a, b = len(c["sigma2"]), len(c["kappa2"])
        p += a * b + a * (a - 1) // 2
    return p


def to_mixture_arrays(classes, zeta):
    """Flat class-concatenated arrays (the oracle's Mixture layout)."""
    return dict(
        n1=[len(c["sigma2"]) for c in classes], n2=[len(c["kappa2"]) for c in classes],
        class_weight=[c.get("weight", 1.0) for c in classes],
        mu=np.concatenate([np.asarray(c["mu"]).reshape(-1, 3) for c in classes]),
        sigma2=np.concatenate([c["sigma2"] for c in classes]),
        phi1=np.concatenate([c["phi1"] for c in classes]),
        dir_=np.concatenate([np.asarray(c["dir"]).reshape(-1, 3) for c in classes]),
        kappa2=np.concatenate([c["kappa2"] for c in classes]),
        phi2=np.concatenate([c["phi2"] for c in classes]), zeta=zeta)
