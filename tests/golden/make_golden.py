"""Generates tests/golden/*.json from the UNMODIFIED reference, compiled in
place from /root/reference by oracle/Makefile (oracle/_ref/libsmalign_ref.so).
Run here (where /root/reference exists):  python tests/golden/make_golden.py

Fixtures (all values printed with 17 significant digits via json/repr):
* bounds_golden.json — contexts x nodes -> evaluate_branch_batch lower/upper
  and subdivide_adaptive split decisions; edge cases included (zero-size
  branches, infeasible cuboids, means inside the cuboid, centres inside a
  standoff ball, parent floors, psi_r = pi).
* objective_golden.json — objective_value at poses, image self-energy.
* solver_golden.json — solve() on the reference toys (test_solver.cpp:105-140,
  test_bench.cpp:222-239) and the ref scene mixtures (test_bench.cpp:241-250).
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.bind import Mixture, Reference, reference_scene_mixtures, reference_torus_cover  # noqa: E402


def random_context(rng, n1, n2, kappa_cap, zeta, n_classes=1):
    """The reference's test_bounds.cpp:18-34 recipe, numpy-seeded."""
    mus, s2, p1, dirs, k2, p2 = [], [], [], [], [], []
    for _ in range(n_classes):
        for _i in range(n1):
            mu = rng.normal(size=3) * 1.5
            while np.linalg.norm(mu) < 0.8:
                mu = rng.normal(size=3) * 1.5
            d = np.linalg.norm(mu) + 3.0
            mus.append(mu)
            s2.append(d * d / (0.8 * kappa_cap - 1.0) * rng.uniform(1.0, 3.0))
            p1.append(1.0 / n1)
        for _j in range(n2):
            v = rng.normal(size=3)
            dirs.append(v / np.linalg.norm(v))
            k2.append(rng.uniform(1.0, 0.8 * kappa_cap))
            p2.append(1.0 / n2)
    return Mixture([n1] * n_classes, [n2] * n_classes, [1.0 / n_classes] * n_classes, mus, s2, p1,
                   dirs, k2, p2, zeta)


def realistic_context(rng, n1, n2, zeta=0.5):
    mu = rng.uniform(-1, 1, (n1, 3))
    s2 = np.exp(rng.uniform(np.log(6.25e-4), np.log(0.05), n1))
    ct = rng.uniform(math.cos(math.radians(40)), 1.0, n2)
    ph = rng.uniform(0, 2 * math.pi, n2)
    st = np.sqrt(1 - ct * ct)
    dirs = np.stack([st * np.cos(ph), st * np.sin(ph), ct], 1)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    k2 = np.exp(rng.uniform(np.log(1e2), np.log(1e5), n2))
    return Mixture([n1], [n2], [1.0], mu, s2, np.full(n1, 1 / n1), dirs, k2, np.full(n2, 1 / n2),
                   zeta)


def random_nodes(rng, n):
    """test_bounds.cpp:36-46 random_branch recipe."""
    N = np.zeros((n, 11))
    N[:, 0:3] = rng.uniform(-2, 2, (n, 3))
    N[:, 3] = rng.uniform(0, 1, n)
    N[:, 4:7] = rng.uniform(-1.5, 1.5, (n, 3))
    N[:, 7:10] = rng.uniform(0, 1.2, (n, 3))
    N[:, 10] = -np.inf
    return N


def edge_nodes(mix, rng):
    mu = mix.mu
    rows = []
    def node(rc, rhw, tc, thw, lower=-np.inf):
        rows.append(list(rc) + [rhw] + list(tc) + list(thw) + [lower])
    node([0.3, -0.2, 0.1], 0.0, [0.0, 0.0, -3.0], [0, 0, 0])          # zero-size branch
    node([1.0, 0.5, -0.7], 0.0, [0.2, 2.5, -1.0], [0, 0, 0])
    node([0, 0, 0], math.pi, [0.0, 0.0, -3.0], [0.5, 0.5, 0.5])        # psi_r = pi
    node([0, 0, 0], 2.0, [0.0, 0.0, -3.0], [0.5, 0.5, 0.5])            # sqrt(3)*2 > pi
    node([0.1, 0.1, 0.1], 0.1, mu[0], [0.01, 0.01, 0.01])               # swallowed: infeasible
    node([0.1, 0.1, 0.1], 0.1, mu[0], [1.0, 1.0, 1.0])                 # mean inside, centre infeasible
    node([0.1, 0.1, 0.1], 0.1, mu[0] + [0.6 * mix.zeta, 0, 0], [0.8, 0.8, 0.8])  # centre in ball
    node([0.4, -0.2, 0.8], 0.1, [0.3, 0.1, -2.0], [0.1, 0.1, 0.1], 5.0)   # parent floor wins
    node([0.4, -0.2, 0.8], 0.1, [0.3, 0.1, -2.0], [0.1, 0.1, 0.1], -1e9)  # parent floor loses
    node([0.4, -0.2, 0.8], 1e-6, [0.3, 0.1, -2.0], [1e-6, 1e-6, 1e-6])    # tiny box
    node([2.5, -2.5, 2.5], 0.3, [0.0, 0.0, 4.0], [2.0, 0.1, 0.1])      # anisotropic cuboid
    node([0.0, 0.0, 0.0], 1e-12, [0.0, 0.0, -3.0], [1e-12, 1e-12, 1e-12])  # below split floor
    return np.array(rows, dtype=np.float64)


def bounds_case(name, mix, nodes, skips=(float("inf"),)):
    ref = Reference(mix)
    out = {"name": name, "mixture": mix.to_dict(), "nodes": nodes.tolist(), "results": []}
    for skip in skips:
        lo, up = ref.eval_bounds(nodes, skip=skip, threads=1)
        out["results"].append({"skip": skip, "lower": lo.tolist(), "upper": up.tolist()})
    out["split"] = [int(ref.subdivide(n)[0]) for n in nodes]
    out["children0"] = ref.subdivide(nodes[0])[1].tolist()
    return out


def main():
    rng = np.random.default_rng(20261018)
    cases = []
    # Moderate contexts (test_bounds recipes): fused-vs-op (4x3, cap 40, zeta .2),
    # soundness (3x3, cap 150, zeta .15), zero-size (3x3, cap 80), random (8x5, cap 150).
    for (n1, n2, cap, zeta, nb) in [(4, 3, 40.0, 0.2, 60), (3, 3, 150.0, 0.15, 60),
                                    (3, 3, 80.0, 0.2, 40), (8, 5, 150.0, 0.2, 60)]:
        mix = random_context(rng, n1, n2, cap, zeta)
        nodes = np.concatenate([random_nodes(rng, nb), edge_nodes(mix, rng)])
        cases.append(bounds_case(f"moderate_{n1}x{n2}_cap{int(cap)}", mix, nodes,
                                 skips=(float("inf"), 0.0)))
    # Semantic: 3 classes.
    mix = random_context(rng, 5, 4, 60.0, 0.2, n_classes=3)
    cases.append(bounds_case("semantic_3x(5x4)", mix,
                             np.concatenate([random_nodes(rng, 60), edge_nodes(mix, rng)])))
    # Extreme concentrations (test_bounds.cpp:161-196).
    mix = Mixture([2], [2], [1.0], [[0.4, -0.2, 0.1], [-0.5, 0.3, -0.2]], [6.25e-4, 6.25e-4],
                  [0.5, 0.5], [np.array([0.1, 0.0, 1.0]) / np.linalg.norm([0.1, 0.0, 1.0]),
                               np.array([-0.1, 0.1, 1.0]) / np.linalg.norm([-0.1, 0.1, 1.0])],
                  [1e5, 1e5], [0.5, 0.5], 0.5)
    en = np.zeros((60, 11))
    en[:, 0:3] = rng.uniform(-2, 2, (60, 3))
    en[:, 3] = rng.uniform(0.1, math.pi, 60)
    en[:, 4:7] = rng.uniform(-4, 4, (60, 3))
    en[:, 7:10] = rng.uniform(0.1, 1.0, (60, 3))
    en[:, 10] = -np.inf
    cases.append(bounds_case("extreme_kappa_1e5", mix, np.concatenate([en, edge_nodes(mix, rng)])))
    # Realistic (config 2 regime), 16x8, nodes from the torus prior.
    mix = realistic_context(rng, 16, 8)
    boxes = reference_torus_cover(3.5, 0.5)
    tn = np.zeros((80, 11))
    for k in range(80):
        lvl = rng.integers(1, 7)
        hw = math.pi / 2 ** lvl
        tn[k, 0:3] = -math.pi + (2 * rng.integers(0, 2 ** lvl, 3) + 1) * hw
        tn[k, 3] = hw
        b = boxes[rng.integers(0, len(boxes))]
        tl = rng.integers(0, 4)
        th = b[3:] / 2 ** tl
        tn[k, 4:7] = b[:3] - b[3:] + (2 * rng.integers(0, 2 ** tl, 3) + 1) * th
        tn[k, 7:10] = th
        tn[k, 10] = -np.inf
    cases.append(bounds_case("realistic_16x8", mix, np.concatenate([tn, edge_nodes(mix, rng)])))
    # Toy contexts of test_solver.cpp:16-20 and test_bench.cpp:17-23.
    toy = Mixture([1], [1], [1.0], [[0, 0, 2]], [1.0], [1.0], [[0, 0, 1]], [5.0], [1.0], 0.5)
    tn = random_nodes(rng, 30)
    cases.append(bounds_case("toy_single_pair", toy, np.concatenate([tn, edge_nodes(toy, rng)])))
    pair = Mixture([2], [2], [1.0], [[0.3, 0.0, 2.2], [-0.4, 0.2, 1.8]], [0.5, 0.7], [0.6, 0.4],
                   [np.array([0.12, 0.0, 1.0]) / np.linalg.norm([0.12, 0.0, 1.0]),
                    np.array([-0.2, 0.1, 1.0]) / np.linalg.norm([-0.2, 0.1, 1.0])],
                   [6.0, 4.0], [0.55, 0.45], 0.4)
    cases.append(bounds_case("toy_pair", pair, np.concatenate([random_nodes(rng, 40),
                                                               edge_nodes(pair, rng)])))
    with open(os.path.join(HERE, "bounds_golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py via oracle/_ref (unmodified reference)",
                   "cases": cases}, f)

    # Objective values.
    obj = []
    for c in cases:
        mix = Mixture.from_dict(c["mixture"])
        ref = Reference(mix)
        poses = []
        for _ in range(12):
            r = rng.uniform(-2, 2, 3)
            t = rng.uniform(-3, 3, 3)
            poses.append({"r": r.tolist(), "t": t.tolist(), "f": ref.objective(r, t)})
        obj.append({"name": c["name"], "mixture": c["mixture"], "self_energy": ref.self_energy,
                    "poses": poses})
    with open(os.path.join(HERE, "objective_golden.json"), "w") as f:
        json.dump({"cases": obj}, f)

    # Solver toys.
    sol = []
    aligned = Mixture([1], [1], [1.0], [[0, 0, 2]], [4.0], [1.0], [[0, 0, 1]], [2.0], [1.0], 0.5)
    r = Reference(aligned, single_ctor=True).solve([0, 0, 0], 0.4,
                                                   [[0.05, -0.03, 0.02, 0.4, 0.4, 0.4]], 0.3, 0.5,
                                                   max_evaluations=3000000, trace_cap=10)
    sol.append({"name": "aligned_toy", "mixture": aligned.to_dict(), "rot_c": [0, 0, 0],
                "rot_hw": 0.4, "boxes": [[0.05, -0.03, 0.02, 0.4, 0.4, 0.4]], "epsilon": 0.3,
                **{k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in r.items()
                   if k != "trace"}})
    r = Reference(pair, single_ctor=True).solve([0, 0, 0], 0.3,
                                                [[0.05, -0.05, 0.1, 0.25, 0.25, 0.25]], 0.05, 0.4,
                                                batch_size=256, max_evaluations=60000,
                                                trace_cap=10)
    sol.append({"name": "toy_pair_grid", "mixture": pair.to_dict(), "rot_c": [0, 0, 0],
                "rot_hw": 0.3, "boxes": [[0.05, -0.05, 0.1, 0.25, 0.25, 0.25]], "epsilon": 0.05,
                **{k: (v.tolist() if isinstance(v, np.ndarray) else v) for k, v in r.items()
                   if k != "trace"}})
    scenes = []
    for seed in (7, 8):
        mix, truth = reference_scene_mixtures(12, 0.0, 0.0, 1.0, seed, zeta=0.5)
        scenes.append({"seed": seed, "n_inliers": 12, "omega": 0.0, "noise_px": 1.0,
                       "mixture": mix.to_dict(), "true_r": truth["r"].tolist(),
                       "true_t": truth["t"].tolist(), "points": truth["points"].tolist(),
                       "pixels": truth["pixels"].tolist()})
    for seed in (1, 2):
        mix, truth = reference_scene_mixtures(30, 0.5, 0.5, 2.0, seed, zeta=0.5)
        scenes.append({"seed": seed, "n_inliers": 30, "omega": 0.5, "noise_px": 2.0,
                       "mixture": mix.to_dict(), "true_r": truth["r"].tolist(),
                       "true_t": truth["t"].tolist(), "points": truth["points"].tolist(),
                       "pixels": truth["pixels"].tolist()})
    with open(os.path.join(HERE, "solver_golden.json"), "w") as f:
        json.dump({"solves": sol, "scenes": scenes,
                   "torus_cover_3.5_0.5": reference_torus_cover(3.5, 0.5).tolist()}, f)
    print("wrote", len(cases), "bound cases,", len(sol), "solves,", len(scenes), "scenes")


if __name__ == "__main__":
    main()
