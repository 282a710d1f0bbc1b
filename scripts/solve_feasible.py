"""Time-to-certified-optimum on instances the BnB can certify (dev script)."""
import os, sys, json, time, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from oracle.bind import Mixture
G = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "solver_golden.json")))
s = G["solves"][1]
mix = Mixture.from_dict(s["mixture"])
cls = [{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2}]
ctx = g.ObjectiveContext(cls, mix.zeta, single_mixture=True)
dom = g.PoseDomain(np.array(s["rot_c"], float), s["rot_hw"], np.array(s["boxes"], float))
for W in [0]:
    cfg = g.SolverConfig(epsilon=0.05, zeta=mix.zeta, wave_nodes=W, time_limit=60.0)
    t0 = time.time(); r = g.solve(ctx, dom, cfg); dt = time.time() - t0
    print(f"toy_pair eps=0.05 W={W}: d*={r.best_value:.8f} LB={r.global_lower:.6f} status={r.status} evals={r.bound_evaluations} waves={r.waves} {dt:.2f}s", flush=True)
sc = G["scenes"][0]
mix = Mixture.from_dict(sc["mixture"])
cls = [{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2}]
ctx = g.ObjectiveContext(cls, 0.5, single_mixture=True)
dom = g.PoseDomain(np.zeros(3), math.pi, np.array(G["torus_cover_3.5_0.5"]))
cfg = g.SolverConfig(epsilon=0.1, zeta=0.5, time_limit=30.0)
t0 = time.time(); r = g.solve(ctx, dom, cfg); dt = time.time() - t0
print(f"scene7 auto-W: d*={r.best_value:.4f} LB={r.global_lower:.4f} status={r.status} evals={r.bound_evaluations} waves={r.waves} {dt:.2f}s rate {r.bound_evaluations/dt:.3e}/s", flush=True)
