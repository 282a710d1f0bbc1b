"""Bound-kernel time per workload (config-2 style batches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_01232_b200 as g
from paper_1812_01232_b200 import synth
n = int(os.environ.get("NODES", "1000000"))
W = [("realistic", 64, 32), ("moderate", 64, 32), ("realistic", 256, 128), ("realistic", 12, 12),
     ("realistic", 41, 36), ("realistic", 45, 40), ("realistic", 8, 4, 8), ("realistic", 32, 16, 8),
     ("realistic", 2, 2), ("realistic", 4, 4), ("realistic", 6, 6), ("realistic", 8, 8),
     ("realistic", 16, 16), ("realistic", 24, 20), ("realistic", 32, 32)]
only = os.environ.get("ONLY")
for regime, n1, n2, *rest in ([W[int(k)] for k in only.split(",")] if only else W):
    nc = rest[0] if rest else 1  # semantic classes (block-sparse pair terms, BASELINE configs[3])
    cls = synth.mixture(n1, n2, regime, seed=2026, n_classes=nc)
    ctx = g.ObjectiveContext(cls, 0.5)
    nn = n if n1 < 256 else n // 16
    nodes = synth.nodes(nn, seed=2027)
    st = torch.cuda.Stream()
    dn = torch.from_numpy(nodes.view(np.uint8)).cuda()
    lo = torch.empty(nn, dtype=torch.float64, device="cuda"); up = torch.empty_like(lo)
    P = nc * (n1 * n2 + n1 * (n1 - 1) // 2)
    for rep in range(1):
        with torch.cuda.stream(st):
            for _ in range(2):
                g.evaluate_branch_batch_device(ctx, dn.data_ptr(), nn, lo.data_ptr(), up.data_ptr(), 0, float("inf"), st.cuda_stream)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(3):
                g.evaluate_branch_batch_device(ctx, dn.data_ptr(), nn, lo.data_ptr(), up.data_ptr(), 0, float("inf"), st.cuda_stream)
            e1.record(st)
        st.synchronize()
        ms = e0.elapsed_time(e1) / 3
        print(f"{regime:9s} {nc}x({n1}x{n2}) nodes {nn} {ms:8.3f} ms  {nn/ms*1e3:.3e} bounds/s  {nn*P/ms*1e3:.3e} pairs/s", flush=True)
