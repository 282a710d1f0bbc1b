import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from oracle.bind import Mixture, Oracle
from tests.golden.make_golden import random_context, random_nodes
from paper_1812_01232_b200 import synth
out = []
def run(mix, nodes, name):
    o = Oracle(mix)
    cl, o1, o2 = [], 0, 0
    for c in range(len(mix.n1)):
        a, b = int(mix.n1[c]), int(mix.n2[c])
        cl.append({"mu": mix.mu[o1:o1+a], "sigma2": mix.sigma2[o1:o1+a], "phi1": mix.phi1[o1:o1+a], "dir": mix.dir[o2:o2+b], "kappa2": mix.kappa2[o2:o2+b], "phi2": mix.phi2[o2:o2+b], "weight": float(mix.class_weight[c])})
        o1 += a; o2 += b
    ctx = g.ObjectiveContext(cl, mix.zeta); ctx.set_lb_margin(0.0)
    lo, up = g.evaluate_branch_batch(ctx, nodes)
    rlo, rup, lm, um, _ = o.eval_bounds(nodes, threads=8)
    f = np.isfinite(rlo)
    e = np.where(f, (lo - rlo) / np.where(f, lm, 1), 0)
    for k in np.argsort(-np.abs(e))[:3]:
        out.append({"name": name, "mix": mix.to_dict(), "node": nodes[k].tolist(), "lo": lo[k], "ref": rlo[k], "mass": lm[k], "err": e[k]})
rng = np.random.default_rng(11)
for rep in range(3):
    run(random_context(rng, 2, 2, 1e5, 0.5), random_nodes(rng, 3000), "mod2x2k1e5")
cl = synth.mixture(8, 6, "realistic", seed=200 + 8)
run(Mixture(**synth.to_mixture_arrays(cl, 0.5)), synth.nodes(3000, seed=2+6).view(np.float64).reshape(-1, 11), "real8x6")
json.dump(out, open("gpurun_out/worst.json", "w"))
for r in out: print(r["name"], r["err"], r["lo"], r["ref"], r["mass"])
