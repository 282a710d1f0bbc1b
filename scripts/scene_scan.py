"""Time-to-certified-optimum of the GPU solver over the configs[2] / configs[3]
scenes of tests/golden/scenes_golden.json (generate_scene seeds 1..25, N_I =
30, omega = 0.5, 2 px; MODE=semantic uses the octant-labelled classes):
full rotation ball, 44-box torus prior, epsilon EPS, TL seconds per seed.
Prints one JSON line per seed."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1812_01232_b200 as g  # noqa: E402

G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests",
                                "golden", "scenes_golden.json")))
mode = os.environ.get("MODE", "plain")
eps = float(os.environ.get("EPS", "0.1"))
tl = float(os.environ.get("TL", "60"))
seeds = []
for part in os.environ.get("SEEDS", "1-25").split(","):
    a, _, b = part.partition("-")
    seeds += list(range(int(a), int(b or a) + 1))


def classes_of(m):
    out, o1, o2 = [], 0, 0
    for c in range(len(m["n1"])):
        a, b = m["n1"][c], m["n2"][c]
        out.append({"mu": m["mu"][o1:o1 + a], "sigma2": m["sigma2"][o1:o1 + a],
                    "phi1": m["phi1"][o1:o1 + a], "dir": m["dir"][o2:o2 + b],
                    "kappa2": m["kappa2"][o2:o2 + b], "phi2": m["phi2"][o2:o2 + b],
                    "weight": m["class_weight"][c]})
        o1, o2 = o1 + a, o2 + b
    return out


dom = g.PoseDomain(np.zeros(3), math.pi, np.array(G["torus_cover_3.5_0.5"]))
for sc in G["scenes"]:
    if sc["seed"] not in seeds:
        continue
    m = sc["semantic"] if mode == "semantic" else sc["mixture"]
    ctx = g.ObjectiveContext(classes_of(m), m["zeta"], single_mixture=(mode != "semantic"))
    cfg = g.SolverConfig(epsilon=eps, zeta=m["zeta"], time_limit=tl)
    t0 = time.perf_counter()
    r = g.solve(ctx, dom, cfg)
    dt = time.perf_counter() - t0
    tr = np.array(sc["true_r"])
    print(json.dumps({"seed": sc["seed"], "mode": mode, "n1": m["n1"], "n2": m["n2"],
                      "status": r.status, "seconds": dt, "best_value": r.best_value,
                      "global_lower": r.global_lower, "gap": r.gap,
                      "evals": r.bound_evaluations, "waves": r.waves,
                      "r": r.r.tolist(), "t": r.t.tolist(),
                      "t_err": float(np.linalg.norm(r.t - np.array(sc["true_t"])))}), flush=True)
