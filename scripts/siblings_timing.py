"""Siblings-mode K1 time (the solver's wave step: 8 rotation children per
parent) on synthetic parents, per workload; ONLY / NODES as kernel_timing.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1812_01232_b200 as g  # noqa: E402
from paper_1812_01232_b200 import synth  # noqa: E402

n = int(os.environ.get("NODES", "125000"))  # parents (8 children each)
W = [("realistic", 64, 32), ("realistic", 8, 4, 8), ("realistic", 12, 12), ("realistic", 41, 36),
     ("realistic", 32, 16, 8)]
only = os.environ.get("ONLY")
for regime, n1, n2, *rest in ([W[int(k)] for k in only.split(",")] if only else W):
    nc = rest[0] if rest else 1
    cls = synth.mixture(n1, n2, regime, seed=2026, n_classes=nc)
    ctx = g.ObjectiveContext(cls, 0.5)
    par = synth.nodes(n, seed=2027)
    d_par = torch.from_numpy(par.view(np.uint8)).cuda()
    d_split = torch.ones(n, dtype=torch.int8, device="cuda")  # rotation splits
    d_lo = torch.empty(8 * n, dtype=torch.float64, device="cuda")
    d_up = torch.empty_like(d_lo)
    st = torch.cuda.Stream()
    P = nc * (n1 * n2 + n1 * (n1 - 1) // 2)

    def run():
        g.evaluate_children_device(ctx, d_par.data_ptr(), d_split.data_ptr(), n, d_lo.data_ptr(),
                                   d_up.data_ptr(), 0, float("inf"), st.cuda_stream)

    with torch.cuda.stream(st):
        for _ in range(2):
            run()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(3):
            run()
        e1.record(st)
    st.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"siblings {regime:9s} {nc}x({n1}x{n2}) parents {n} children {8 * n}  {ms:7.3f} ms  "
          f"{8 * n / ms * 1e3:.3e} bounds/s  {8 * n * P / ms * 1e3:.3e} pairs/s", flush=True)
