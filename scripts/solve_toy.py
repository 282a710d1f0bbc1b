"""GPU solve of the reference's grid-oracle toy (test_bench.cpp:222-239) to a gap."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from oracle.bind import Mixture
inst = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "solver_golden.json")))["solves"][1]
mix = Mixture.from_dict(inst["mixture"])
ctx = g.ObjectiveContext([{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2}], mix.zeta, single_mixture=True)
dom = g.PoseDomain(np.array(inst["rot_c"]), inst["rot_hw"], np.array(inst["boxes"]))
for gap in [float(x) for x in os.environ.get("GAPS", "0.44,0.3,0.2").split(",")]:
    t0 = time.perf_counter(); r = g.solve(ctx, dom, g.SolverConfig(epsilon=gap, zeta=mix.zeta, time_limit=float(os.environ.get("TL", "60")))); dt = time.perf_counter() - t0
    print(f"gap {gap}: {dt:.3f}s status {r.status} d*={r.best_value:.6f} LB={r.global_lower:.6f} evals={r.bound_evaluations} waves={r.waves}", flush=True)
