"""GPU-resident refiner (local_refine_batch) vs the host local_refine: time
for 44 starts (the discovery dive's start count) on synthetic mixtures."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from paper_1812_01232_b200 import synth

host = os.environ.get("HOST", "0") == "1"
for n1, n2 in [(12, 12), (41, 36), (64, 32), (256, 128)]:
    cls = synth.mixture(n1, n2, "realistic", seed=5)
    ctx = g.ObjectiveContext(cls, 0.5)
    dom = g.PoseDomain(np.zeros(3), np.pi, synth.torus_cover(3.5, 0.5))
    rng = np.random.default_rng(1)
    boxes = synth.torus_cover(3.5, 0.5)
    pick = boxes[rng.integers(0, len(boxes), 44)]
    r0 = rng.uniform(-1.0, 1.0, (44, 3))
    t0 = pick[:, :3] + rng.uniform(-1, 1, (44, 3)) * pick[:, 3:]
    g.local_refine_batch(ctx, r0[:2], t0[:2], dom)  # warm-up (module load)
    t = time.perf_counter()
    v, r, tt = g.local_refine_batch(ctx, r0, t0, dom)
    dt = time.perf_counter() - t
    line = f"{n1}x{n2}: GPU {dt*1e3:.1f} ms best {np.nanmin(v):.5f}"
    if host:
        t = time.perf_counter()
        vh = [g.local_refine(ctx, r0[k], t0[k], dom)[0] for k in range(44)]
        dh = time.perf_counter() - t
        line += f" | host 1 thread {dh*1e3:.1f} ms best {np.nanmin(vh):.5f} max|dv| {np.nanmax(np.abs(np.array(vh) - v)):.2e}"
    print(line, flush=True)
