"""Long certification attempt on a configs[2] scene (generate_scene seed SEED,
N_I=30, omega=0.5, 2 px): full rotation ball, 44-box torus prior, epsilon EPS.
Drives the stepwise solver and prints, every ~PRINT seconds, wall time,
evaluations, live nodes, d*, certified LB and the volume fractions, so a
failure to certify can be diagnosed (bound looseness vs memory folding vs
wave selection).  GOSMA_PROFILE=1 adds per-phase times at the end."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1812_01232_b200 as g  # noqa: E402

seed = int(os.environ.get("SEED", "1"))
eps = float(os.environ.get("EPS", "0.1"))
tl = float(os.environ.get("TL", "300"))
every = float(os.environ.get("PRINT", "5"))
mode = os.environ.get("MODE", "plain")
G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests",
                              "golden", "scenes_golden.json")))
sc = next((s for s in G["scenes"] if s["seed"] == seed), None)
if sc is None:  # configs[0] scenes (generate_scene N_I = 12) live in solver_golden.json
    G2 = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests",
                                     "golden", "solver_golden.json")))
    sc = next(s for s in G2["scenes"] if s["seed"] == seed)
m = sc["semantic"] if mode == "semantic" else sc["mixture"]
cls, o1, o2 = [], 0, 0
for c in range(len(m["n1"])):
    a, b = m["n1"][c], m["n2"][c]
    cls.append({"mu": m["mu"][o1:o1 + a], "sigma2": m["sigma2"][o1:o1 + a],
                "phi1": m["phi1"][o1:o1 + a], "dir": m["dir"][o2:o2 + b],
                "kappa2": m["kappa2"][o2:o2 + b], "phi2": m["phi2"][o2:o2 + b],
                "weight": m["class_weight"][c]})
    o1, o2 = o1 + a, o2 + b
ctx = g.ObjectiveContext(cls, m["zeta"], single_mixture=(mode != "semantic"))
dom = g.PoseDomain(np.zeros(3), math.pi, np.array(G["torus_cover_3.5_0.5"]))
cfg = g.SolverConfig(epsilon=eps, zeta=m["zeta"], wave_nodes=int(os.environ.get("WAVE", "0")))
t0 = time.perf_counter()
S = g.ShardSolver(ctx, dom, cfg)
t_init = time.perf_counter() - t0
cert = -math.inf
last = -1e9
rows = []
status = "time_limit"
while True:
    st = S.status()
    d = st["best_value"]
    cert = max(cert, min(d, st["frontier_min"], st["floor_lower"]))
    now = time.perf_counter() - t0
    row = {"t": round(now, 3), "evals": st["bound_evaluations"], "live": st["live_nodes"],
           "dstar": d, "lb": cert, "frontier_min": st["frontier_min"],
           "floor": st["floor_lower"],
           "pruned": st["pruned_volume"] / st["total_volume"],
           "resolved": st["resolved_volume"] / st["total_volume"]}
    if now - last >= every:
        print(json.dumps(row), flush=True)
        rows.append(row)
        last = now
    if d - cert <= eps:
        status = "epsilon_optimal"
        break
    if st["live_nodes"] == 0:
        status = "queue_exhausted"
        break
    if now >= tl:
        break
    S.expand(d - eps)
res = S.result()
out = {"seed": seed, "mode": mode, "eps": eps, "status": status, "seconds": time.perf_counter() - t0,
       "init_seconds": t_init, "best_value": res["value"], "global_lower": cert,
       "evals": res["bound_evaluations"], "waves": res["waves"], "r": res["r"].tolist(),
       "t": res["t"].tolist(), "last": row}
print(json.dumps(out), flush=True)
del S
