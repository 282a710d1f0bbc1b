"""Time-to-certified-optimum on a generate_scene instance (config-1 style)."""
import os, sys, json, time, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from oracle.bind import Mixture
G = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "solver_golden.json")))
k = int(os.environ.get("SCENE", "0"))
sc = G["scenes"][k]
mix = Mixture.from_dict(sc["mixture"])
cls = [{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2}]
ctx = g.ObjectiveContext(cls, 0.5, single_mixture=True)
dom = g.PoseDomain(np.zeros(3), math.pi, np.array(G["torus_cover_3.5_0.5"]))
cfg = g.SolverConfig(epsilon=0.1, zeta=0.5, time_limit=float(os.environ.get("TL", "300")))
t0 = time.time(); r = g.solve(ctx, dom, cfg); dt = time.time() - t0
print(f"scene seed {sc['seed']} {mix.n1[0]}x{mix.n2[0]}: d*={r.best_value:.6f} LB={r.global_lower:.6f} gap={r.gap:.4f} status={r.status} evals={r.bound_evaluations} waves={r.waves} {dt:.2f}s rate {r.bound_evaluations/dt:.3e}/s", flush=True)
for t in r.trace[::max(1, len(r.trace)//15)]: print("  ", t)
