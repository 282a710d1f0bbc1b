"""Time-to-certified-optimum on the hardest tests/golden/certify_golden.json
instance (bench.py's solve_certified, GPU side only; GOSMA_PROFILE=1 for phases)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from oracle.bind import Mixture
G = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "certify_golden.json")))
inst = max(G["instances"], key=lambda x: x["bound_evaluations"])
mix = Mixture.from_dict(inst["mixture"])
ctx = g.ObjectiveContext([{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir,
                           "kappa2": mix.kappa2, "phi2": mix.phi2}], mix.zeta, single_mixture=True)
dom = g.PoseDomain(np.array(inst["rot_c"]), inst["rot_hw"], np.array(inst["boxes"]))
cfg = g.SolverConfig(epsilon=inst["epsilon"], zeta=mix.zeta, time_limit=120)
for k in range(int(os.environ.get("REPS", "3"))):
    t0 = time.perf_counter()
    r = g.solve(ctx, dom, cfg)
    dt = time.perf_counter() - t0
    print(f"solve {k}: {dt*1e3:.1f} ms status {r.status} d*={r.best_value:.9f} LB={r.global_lower:.9f} "
          f"evals={r.bound_evaluations} waves={r.waves} sma={r.sma_invocations}", flush=True)
