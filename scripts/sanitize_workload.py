"""Small workload touching every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck; see DESIGN.md §10 for why no run is kept):
K1 in its full, class-streamed, translation-cached and siblings modes (with
tail chunks and CTA groups), the precise cross pass, the frontier (select,
expand, route, compaction, depth-first selection), the device dive beam, the
GPU refiner and the DP-means scorer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1812_01232_b200 as g  # noqa: E402
from paper_1812_01232_b200 import synth  # noqa: E402


def k1(n1, n2, ncls, regime, n=512):
    cls = synth.mixture(n1, n2, regime, seed=n1 + n2, n_classes=ncls)
    ctx = g.ObjectiveContext(cls, 0.5)
    nodes = synth.nodes(n, seed=3)
    lo, up = g.evaluate_branch_batch(ctx, nodes)
    assert np.isfinite(lo).any()
    # siblings mode: 8 rotation children per parent
    d_par = torch.from_numpy(nodes.view(np.uint8)).cuda()
    d_split = torch.ones(n, dtype=torch.int8, device="cuda")
    d_lo = torch.empty(8 * n, dtype=torch.float64, device="cuda")
    d_up = torch.empty_like(d_lo)
    s = torch.cuda.Stream()
    g.evaluate_children_device(ctx, d_par.data_ptr(), d_split.data_ptr(), n, d_lo.data_ptr(),
                               d_up.data_ptr(), 0, float("inf"), s.cuda_stream)
    s.synchronize()


for args in ((8, 6, 1, "realistic"), (41, 36, 1, "realistic"), (64, 32, 1, "moderate"),
             (33, 17, 3, "realistic"), (128, 64, 1, "realistic"), (2, 2, 1, "realistic")):
    k1(*args)
    print("k1", args, flush=True)

# solver: a 12x12 scene with a tiny pool budget (forces depth-first waves)
import json  # noqa: E402
G = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests",
                                "golden", "solver_golden.json")))
m = G["scenes"][0]["mixture"]
ctx = g.ObjectiveContext([{"mu": m["mu"], "sigma2": m["sigma2"], "phi1": m["phi1"],
                           "dir": m["dir"], "kappa2": m["kappa2"], "phi2": m["phi2"]}],
                         m["zeta"], single_mixture=True)
dom = g.PoseDomain(np.zeros(3), np.pi, np.array(G["torus_cover_3.5_0.5"]))
r = g.solve(ctx, dom, g.SolverConfig(epsilon=0.1, zeta=0.5, max_evaluations=3_000_000,
                                     wave_nodes=4096))
print("solve", r.status, r.best_value, r.global_lower, flush=True)
# GPU refiner
cls = synth.mixture(40, 24, "moderate", seed=9)
ctx = g.ObjectiveContext(cls, 0.5)
v, rr, tt = g.local_refine_batch(ctx, np.zeros((4, 3)) + 0.1,
                                 np.array([[0.0, 0.0, -3.0]] * 4),
                                 g.PoseDomain(np.zeros(3), 1.0,
                                              np.array([[0.0, 0.0, -3.0, 0.5, 0.5, 0.5]])))
print("refine", v, flush=True)
# DP-means scorer on the GPU
os.environ["GOSMA_DPMEANS"] = "gpu"
pts = np.random.default_rng(1).uniform(-1, 1, (3000, 3))
a, c, it = g.dp_means(pts, 0.25)
print("dp_means", len(c), it, flush=True)
print("sanitize workload ok")
