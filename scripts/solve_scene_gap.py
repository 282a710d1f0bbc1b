"""Scene solve to a given certified gap (EPS), timed after a warm-up solve;
GOSMA_PROFILE=1 prints the solver's per-phase times."""
import os, sys, json, time, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from oracle.bind import Mixture
G = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "solver_golden.json")))
sc = next(s for s in G["scenes"] if s["seed"] == int(os.environ.get("SEED", "1")))
mix = Mixture.from_dict(sc["mixture"])
cls = [{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2}]
ctx = g.ObjectiveContext(cls, mix.zeta, single_mixture=True)
dom = g.PoseDomain(np.zeros(3), math.pi, np.array(G["torus_cover_3.5_0.5"]))
cfg = g.SolverConfig(epsilon=float(os.environ.get("EPS", "19154.6")), zeta=mix.zeta, time_limit=60)
for rep in range(int(os.environ.get("REPS", "3"))):
    t0 = time.perf_counter(); r = g.solve(ctx, dom, cfg); dt = time.perf_counter() - t0
    print(f"rep {rep}: {dt*1e3:.1f} ms d*={r.best_value:.9f} LB={r.global_lower:.3f} status={r.status} evals={r.bound_evaluations} waves={r.waves}", flush=True)
