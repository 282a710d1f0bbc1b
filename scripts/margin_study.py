"""Signed FP32 error of the LB core (margin 0) relative to |term| mass, across regimes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from paper_1812_01232_b200 import synth
from oracle.bind import Mixture, Oracle
from tests.golden.make_golden import random_context, random_nodes
worst = 0.0
rng = np.random.default_rng(7)
cases = []
for (n1, n2, kc, z, nc) in [(4,3,40,.2,1),(3,3,150,.15,1),(8,6,1e4,.2,1),(16,8,1e3,.2,1),(5,4,60,.2,3),(2,2,1e5,.5,1),(1,1,20,.2,1)]:
    for rep in range(4):
        cases.append((random_context(rng, n1, n2, kc, z, nc), random_nodes(rng, 3000), f"mod{n1}x{n2}k{kc}"))
for (n1, n2) in [(8,6),(16,8),(64,32),(12,12),(40,36)]:
    for rep in range(3):
        cl = synth.mixture(n1, n2, "realistic", seed=rep*100+n1)
        cases.append((Mixture(**synth.to_mixture_arrays(cl, 0.5)), synth.nodes(3000, seed=rep+n2).view(np.float64).reshape(-1,11), f"real{n1}x{n2}"))
for mix, nodes, name in cases:
    o = Oracle(mix)
    cl, o1, o2 = [], 0, 0
    for c in range(len(mix.n1)):
        a, b = int(mix.n1[c]), int(mix.n2[c])
        cl.append({"mu": mix.mu[o1:o1+a], "sigma2": mix.sigma2[o1:o1+a], "phi1": mix.phi1[o1:o1+a], "dir": mix.dir[o2:o2+b], "kappa2": mix.kappa2[o2:o2+b], "phi2": mix.phi2[o2:o2+b], "weight": float(mix.class_weight[c])})
        o1 += a; o2 += b
    ctx = g.ObjectiveContext(cl, mix.zeta)
    if os.environ.get("NOMARGIN"): ctx.set_lb_margin(-1.0)
    lo, up = g.evaluate_branch_batch(ctx, nodes)
    rlo, rup, lm, um, _ = o.eval_bounds(nodes, threads=8)
    f = np.isfinite(rlo)
    e = (lo[f] - rlo[f]) / lm[f]
    eu = np.abs(up[f] - rup[f]) / np.maximum(um[f], 1e-300)
    worst = max(worst, e.max())
    print(f"{name:14s} signed LB err/mass max {e.max():+.3e} min {e.min():+.3e} | UB abs max {eu.max():.3e}")
print("WORST positive", worst)
