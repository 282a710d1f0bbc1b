import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json, numpy as np, paper_1812_01232_b200 as g
from oracle.bind import Mixture
from paper_1812_01232_b200.host import angular_distance
G = json.load(open('tests/golden/solver_golden.json'))
s = G['solves'][1]
mix = Mixture.from_dict(s['mixture'])
ctx = g.ObjectiveContext([{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2}], mix.zeta, single_mixture=True)
dom = g.PoseDomain(np.array(s['rot_c']), s['rot_hw'], np.array(s['boxes']))
for ev in (60000, 2000000):
    r = g.solve(ctx, dom, g.SolverConfig(epsilon=0.05, zeta=mix.zeta, batch_size=256, max_evaluations=ev))
    print(ev, r.best_value, r.r, r.t, angular_distance(r.r, s['r']), np.linalg.norm(r.t - np.array(s['t'])))
