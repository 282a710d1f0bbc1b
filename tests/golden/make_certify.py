"""Tiny random instances the unmodified reference certifies (status
epsilon_optimal) in well under a minute, with the reference's own result:
tests/golden/certify_golden.json. Used by tests/test_solver_gpu.py (certified
optimum parity) and bench.py (time-to-certified-optimum vs the CPU reference).

  python tests/golden/make_certify.py      (needs oracle/_ref)
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.bind import Reference  # noqa: E402
from tests.golden.make_golden import random_context  # noqa: E402


def main():
    rng = np.random.default_rng(5)
    out = []
    for trial in range(14):
        # trials 10-13: two semantic classes (block-diagonal pair terms)
        ncls = 2 if trial >= 10 else 1
        mix = random_context(rng, int(rng.integers(1, 3)), int(rng.integers(1, 3)), 20.0, 0.3,
                             n_classes=ncls)
        c = rng.uniform(-0.2, 0.2, 3)
        box = np.array([[*rng.uniform(-0.3, 0.3, 3), 0.3, 0.3, 0.3]])
        eps = 0.05
        t0 = time.perf_counter()
        rep = Reference(mix).solve(c, 0.3, box, eps, mix.zeta, batch_size=1024, time_limit=60,
                                   threads=8)
        dt = time.perf_counter() - t0
        if rep["status"] != 0:
            continue
        out.append({"mixture": mix.to_dict(), "rot_c": c.tolist(), "rot_hw": 0.3,
                    "boxes": box.tolist(), "epsilon": eps,
                    "best_value": float(rep["best_value"]),
                    "global_lower": float(rep["global_lower"]),
                    "bound_evaluations": int(rep["bound_evaluations"]),
                    "seconds_8_threads": dt})
        print(trial, mix.n1, mix.n2, f"{dt:.2f}s", rep["bound_evaluations"])
        out[-1]["classes"] = ncls
    with open(os.path.join(HERE, "certify_golden.json"), "w") as f:
        json.dump({"instances": out}, f)


if __name__ == "__main__":
    main()
