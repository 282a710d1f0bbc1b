"""Certified-vs-certified probe: a configs[0]-style scene (solver_golden.json
seed SEED, generate_scene N_I = 12) on a domain restricted around the true
pose (rotation cube half-width RHW around true_r, one translation box of
half-width THW around true_t), epsilon EPS: the GPU solver, then (REF=1) the
unmodified reference solve() on all host cores, through bench.solve_compare."""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1812_01232_b200 as g  # noqa: E402
from oracle.bind import Mixture  # noqa: E402
from tests.test_bounds_gpu import mix_classes  # noqa: E402

G = json.load(open(os.path.join(ROOT, "tests", "golden", "solver_golden.json")))
seed = int(os.environ.get("SEED", "7"))
sc = next(s for s in G["scenes"] if s["seed"] == seed)
mix = Mixture.from_dict(sc["mixture"])
ctx = g.ObjectiveContext(mix_classes(mix), mix.zeta, single_mixture=True)
for spec in os.environ.get("DOMS", "0.3:0.3,0.6:0.5,1.0:0.75").split(","):
    rhw, thw = (float(x) for x in spec.split(":"))
    eps = float(os.environ.get("EPS", "0.1"))
    rc = np.zeros(3) if os.environ.get("RC0") else np.asarray(sc["true_r"], float)
    box = np.array([list(sc["true_t"]) + [thw] * 3])
    dom = g.PoseDomain(rc, rhw, box)
    bench.timed_solve(g, ctx, dom, eps, mix.zeta, 0.3)
    r, _ = bench.timed_solve(g, ctx, dom, eps, mix.zeta, float(os.environ.get("GPU_LIMIT", "30")))
    print(json.dumps({"rhw": rhw, "thw": thw, "eps": eps,
                      "gpu": {k: r[k] for k in ("status", "seconds", "best_value", "gap",
                                                "bound_evaluations")}}), flush=True)
    if os.environ.get("REF"):
        out = bench.solve_compare(g, "restricted", mix, True, rc, rhw, box, eps, 30.0,
                                  float(os.environ.get("REF_LIMIT", "60")))
        print(json.dumps({"rhw": rhw, "thw": thw, "compare": {k: out[k] for k in out
                                                              if k != "gosma"}}), flush=True)
