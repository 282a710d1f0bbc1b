"""The unmodified reference solve() on the configs[2]-style scene
(solver_golden.json "scenes", generate_scene seed 1: N_I = 30, omega = 0.5,
2 px noise; 41 GMM x 36 vMF), full rotation ball, the 44-box torus prior,
epsilon 0.1, stopped by an evaluation budget: its incumbent, certified lower
bound and gap -> tests/golden/scene_gap_golden.json. The GPU solver must
certify the same gap with the same d* (tests/test_solver_gpu.py).

  python tests/golden/make_scene_gap.py      (needs oracle/_ref)
"""
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.bind import Mixture, Reference  # noqa: E402


def main():
    G = json.load(open(os.path.join(HERE, "solver_golden.json")))
    sc = next(s for s in G["scenes"] if s["seed"] == 1)
    mix = Mixture.from_dict(sc["mixture"])
    boxes = np.array(G["torus_cover_3.5_0.5"])
    budget = 400_000
    t0 = time.perf_counter()
    rep = Reference(mix, single_ctor=True).solve(np.zeros(3), math.pi, boxes, 0.1, mix.zeta,
                                                 batch_size=1024, max_evaluations=budget,
                                                 threads=os.cpu_count() or 1)
    dt = time.perf_counter() - t0
    out = {"scene_seed": 1, "epsilon": 0.1, "max_evaluations": budget,
           "status": int(rep["status"]), "best_value": float(rep["best_value"]),
           "global_lower": float(rep["global_lower"]),
           "gap": float(rep["best_value"] - rep["global_lower"]),
           "bound_evaluations": int(rep["bound_evaluations"]), "seconds": dt,
           "r": [float(v) for v in rep["r"]], "t": [float(v) for v in rep["t"]]}
    json.dump(out, open(os.path.join(HERE, "scene_gap_golden.json"), "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
