"""Dev script: GPU solve() on the reference toys and scenes vs golden results."""
import os, sys, json, time, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from oracle.bind import Mixture
G = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "solver_golden.json")))
def ctx_of(md, single=False):
    mix = Mixture.from_dict(md)
    cls = [{"mu": mix.mu, "sigma2": mix.sigma2, "phi1": mix.phi1, "dir": mix.dir, "kappa2": mix.kappa2, "phi2": mix.phi2, "weight": 1.0}]
    return g.ObjectiveContext(cls, mix.zeta, single_mixture=True), mix
for s in G["solves"]:
    ctx, mix = ctx_of(s["mixture"])
    dom = g.PoseDomain(np.array(s["rot_c"], float), s["rot_hw"], np.array(s["boxes"], float))
    cfg = g.SolverConfig(epsilon=s["epsilon"], zeta=mix.zeta, wave_nodes=int(os.environ.get("W", "2048")),
                         max_evaluations=(60000 if s["name"] == "toy_pair_grid" else 3000000), time_limit=60.0)
    t0 = time.time(); r = g.solve(ctx, dom, cfg); dt = time.time() - t0
    print(flush=True); print(f"{s['name']}: gpu d*={r.best_value:.10f} LB={r.global_lower:.6f} status={r.status} evals={r.bound_evaluations} waves={r.waves} sma={r.sma_invocations} {dt:.2f}s | ref d*={s['best_value']:.10f} LB={s['global_lower']:.6f} status={s['status']} evals={s['bound_evaluations']}")
boxes = np.array(G["torus_cover_3.5_0.5"])
for sc in G["scenes"][:2]:
    ctx, mix = ctx_of(sc["mixture"])
    dom = g.PoseDomain(np.zeros(3), math.pi, boxes)
    cfg = g.SolverConfig(epsilon=0.1, zeta=0.5, wave_nodes=int(os.environ.get("W", "16384")), time_limit=float(os.environ.get("TL", "60")))
    t0 = time.time(); r = g.solve(ctx, dom, cfg); dt = time.time() - t0
    print(f"scene seed {sc['seed']} ({mix.n1[0]}x{mix.n2[0]}): d*={r.best_value:.6f} LB={r.global_lower:.6f} gap={r.gap:.4f} status={r.status} evals={r.bound_evaluations} waves={r.waves} sma={r.sma_invocations} {dt:.2f}s")
    print("   pose r", r.r, "t", r.t, " truth r", sc["true_r"], "t", sc["true_t"])
    print("   trace tail", r.trace[-3:] if r.trace else None, flush=True)
