"""Largest-epsilon certification probe on the configs[3] semantic scene
(seed 19): the GPU solver at each EPS (GPU_LIMIT s), then the unmodified
reference solve() on all host cores (REF_LIMIT s) at the EPS values listed in
REF_EPS, through bench.solve_compare. Finds an epsilon both solvers certify,
for a time-to-certified-optimum comparison on a BASELINE config."""
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

G = bench.scene_instances()
sem = next(x for x in G["scenes"] if x["seed"] == bench.SEMANTIC_SEED)["semantic"]
mix = Mixture.from_dict(sem)
boxes = np.array(G["torus_cover_3.5_0.5"])
ctx = g.ObjectiveContext(mix_classes(mix), mix.zeta, single_mixture=False)
dom = g.PoseDomain(np.zeros(3), math.pi, boxes)
bench.timed_solve(g, ctx, dom, 1.0, mix.zeta, 0.5)
for eps in [float(x) for x in os.environ.get("EPS", "1000,300,100,30,10,3").split(",")]:
    r, _ = bench.timed_solve(g, ctx, dom, eps, mix.zeta, float(os.environ.get("GPU_LIMIT", "30")))
    print(json.dumps({"eps": eps, "gpu": {k: r[k] for k in ("status", "seconds", "best_value",
                                                              "gap", "bound_evaluations")}}),
          flush=True)
for eps in [float(x) for x in os.environ.get("REF_EPS", "").split(",") if x]:
    out = bench.solve_compare(g, "semantic probe", mix, False, np.zeros(3), math.pi, boxes, eps,
                              30.0, float(os.environ.get("REF_LIMIT", "120")))
    print(json.dumps({"eps": eps, "compare": out}), flush=True)
