"""Solver init (discovery dive + SMA) and wave costs on synthetic mixtures."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from paper_1812_01232_b200 import synth
n1, n2 = int(os.environ.get("N1", "64")), int(os.environ.get("N2", "32"))
cls = synth.mixture(n1, n2, os.environ.get("REGIME", "realistic"), seed=5)
ctx = g.ObjectiveContext(cls, 0.5)
dom = g.PoseDomain(np.zeros(3), np.pi, synth.torus_cover(3.5, 0.5))
t0 = time.perf_counter()
r = g.solve(ctx, dom, g.SolverConfig(epsilon=0.1, zeta=0.5, time_limit=float(os.environ.get("TL", "5"))))
print(f"{n1}x{n2}: {time.perf_counter()-t0:.2f}s status {r.status} d*={r.best_value:.5f} LB={r.global_lower:.5f} evals={r.bound_evaluations} sma={r.sma_invocations} waves={r.waves}", flush=True)
