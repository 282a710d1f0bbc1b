import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from oracle.bind import Mixture, Oracle
from tests.golden.make_golden import random_context, random_nodes
rng = np.random.default_rng(7)
for rep in range(3):
    mix = random_context(rng, 1, 1, 20.0, 0.2)
    nodes = random_nodes(rng, 3000)
    o = Oracle(mix)
    ctx = g.ObjectiveContext([{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2}], mix.zeta)
    ctx.set_lb_margin(0.0)
    lo, up = g.evaluate_branch_batch(ctx, nodes)
    rlo, rup, lm, um, _ = o.eval_bounds(nodes)
    f = np.isfinite(rlo)
    e = np.where(f, (lo - rlo) / np.where(f, lm, 1), 0)
    k = np.argsort(-np.abs(e))[:4]
    for i in k:
        nd = nodes[i]
        mu = mix.mu[0]; s2 = mix.sigma2[0]
        d = np.abs(mu - nd[4:7]); ob = np.maximum(d - nd[7:10], 0)
        dlo = max(np.linalg.norm(ob), mix.zeta); dhi = np.linalg.norm(d + nd[7:10])
        klo = dlo**2/s2 + 1; khi = dhi**2/s2+1
        diag = 0.5*klo/math.tanh(klo)
        cross_ref = (diag - rlo[i]) / 2; cross_gpu = (diag - lo[i]) / 2
        print(f"node {i} err/mass {e[i]:+.3e} lo {lo[i]:.9g} ref {rlo[i]:.9g} mass {lm[i]:.4g} klo {klo:.4g} khi {khi:.4g} k2 {mix.kappa2[0]:.4g} cross ref {cross_ref:.9g} gpu {cross_gpu:.9g} rel {(cross_gpu-cross_ref)/cross_ref:+.2e} rhw {nd[3]:.3f}")
