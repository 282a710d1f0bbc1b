import os, sys, json, time, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from oracle.bind import Mixture
G = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "solver_golden.json")))
s = G["solves"][int(os.environ.get("K", "0"))]
mix = Mixture.from_dict(s["mixture"])
cls = [{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2}]
ctx = g.ObjectiveContext(cls, mix.zeta, single_mixture=True)
dom = g.PoseDomain(np.array(s["rot_c"], float), s["rot_hw"], np.array(s["boxes"], float))
cfg = g.SolverConfig(epsilon=s["epsilon"], zeta=mix.zeta, wave_nodes=int(os.environ.get("W", "2048")), time_limit=float(os.environ.get("TL", "10")), discovery_dive=bool(int(os.environ.get("DIVE", "1"))))
print("start", flush=True)
t0 = time.time(); r = g.solve(ctx, dom, cfg); dt = time.time() - t0
print(f"{s['name']}: d*={r.best_value:.10f} LB={r.global_lower:.6f} status={r.status} evals={r.bound_evaluations} waves={r.waves} sma={r.sma_invocations} {dt:.2f}s ref d*={s['best_value']:.10f}", flush=True)
for t in r.trace[:5] + r.trace[-5:]: print(t)
