"""Solver throughput on a semantic (multi-class) synthetic mixture (BASELINE
configs[3]): NC classes of N1 GMM x N2 vMF components, full 6-DoF domain."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from paper_1812_01232_b200 import synth
nc = int(os.environ.get("NC", "8"))
n1, n2 = int(os.environ.get("N1", "8")), int(os.environ.get("N2", "4"))
cls = synth.mixture(n1, n2, "realistic", seed=5, n_classes=nc)
ctx = g.ObjectiveContext(cls, 0.5)
dom = g.PoseDomain(np.zeros(3), np.pi, synth.torus_cover(3.5, 0.5))
t0 = time.perf_counter()
r = g.solve(ctx, dom, g.SolverConfig(epsilon=0.1, zeta=0.5, time_limit=float(os.environ.get("TL", "5"))))
dt = time.perf_counter() - t0
print(f"{nc}x({n1}x{n2}) [{os.environ.get('GOSMA_WAVE_MODE', 'siblings')}]: {dt:.2f}s status {r.status} "
      f"d*={r.best_value:.5f} LB={r.global_lower:.5f} evals={r.bound_evaluations} "
      f"rate {r.bound_evaluations / dt:.3e}/s waves={r.waves}", flush=True)
