"""Depth-first (drain) mode under a tiny pool budget, for tests/test_solver_gpu.py:
runs in its own process because GOSMA_POOL_FRAC is read once per process.
MODE=certify: the hardest certify_golden.json instance (2 GMM x 2 vMF) to its
certificate; MODE=ledger: 80 waves of the solver_golden 12x12 scene with the
volume ledger checked every wave. Prints one JSON line."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_1812_01232_b200 as g  # noqa: E402
from oracle.bind import Mixture  # noqa: E402


def ctx_of(mix):
    return g.ObjectiveContext([{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1,
                                "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2}],
                              mix.zeta, single_mixture=True)


mode = os.environ.get("MODE", "certify")
wave = int(os.environ.get("WAVE", "256"))
out = {"mode": mode}
if mode == "certify":
    G = json.load(open(os.path.join(ROOT, "tests", "golden", "certify_golden.json")))
    inst = max(G["instances"], key=lambda x: x["bound_evaluations"])
    mix = Mixture.from_dict(inst["mixture"])
    dom = g.PoseDomain(np.array(inst["rot_c"]), inst["rot_hw"], np.array(inst["boxes"]))
    shard = g.ShardSolver(ctx_of(mix), dom, g.SolverConfig(epsilon=inst["epsilon"], zeta=mix.zeta,
                                                           wave_nodes=wave), 0, 1)
    cert, eps, status, waves = -math.inf, inst["epsilon"], "time_limit", 0
    while waves < 20000:
        st = shard.status()
        cert = max(cert, min(st["best_value"], st["frontier_min"], st["floor_lower"]))
        if st["best_value"] - cert <= eps:
            status = "epsilon_optimal"
            break
        if st["live_nodes"] == 0:
            status = "queue_exhausted"
            break
        shard.expand(st["best_value"] - eps)
        waves += 1
    out.update({"status": status, "best_value": st["best_value"], "global_lower": cert,
                "waves": waves, "golden_best": inst["best_value"], "epsilon": eps})
else:
    G = json.load(open(os.path.join(ROOT, "tests", "golden", "solver_golden.json")))
    mix = Mixture.from_dict(G["scenes"][0]["mixture"])
    dom = g.PoseDomain(np.zeros(3), math.pi, np.array(G["torus_cover_3.5_0.5"]))
    shard = g.ShardSolver(ctx_of(mix), dom, g.SolverConfig(epsilon=0.1, zeta=mix.zeta,
                                                           wave_nodes=wave), 0, 1)
    worst, lows = 0.0, []
    for w in range(80):
        st = shard.status()
        tot = st["total_volume"]
        worst = max(worst, abs(st["pruned_volume"] + st["resolved_volume"] + shard.live_volume()
                               - tot) / tot)
        lows.append(min(st["frontier_min"], st["floor_lower"]))
        shard.expand(st["best_value"] - 0.1)
    out.update({"ledger_worst_rel": worst,
                "monotone": all(b >= a - 1e-12 for a, b in zip(lows, lows[1:]))})
del shard
print(json.dumps(out), flush=True)
