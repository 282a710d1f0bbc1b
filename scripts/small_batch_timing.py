"""Latency of small bound batches (the discovery dive beam): device-resident launch vs the host API."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1812_01232_b200 as g
from paper_1812_01232_b200 import synth
for (n1, n2) in [(2, 2), (12, 12), (64, 32)]:
    cls = synth.mixture(n1, n2, "realistic", seed=2026)
    ctx = g.ObjectiveContext(cls, 0.5)
    for n in [32, 512, 4096]:
        nodes = synth.nodes(n, seed=2027)
        st = torch.cuda.Stream()
        dn = torch.from_numpy(nodes.view(np.uint8)).cuda()
        lo = torch.empty(n, dtype=torch.float64, device="cuda"); up = torch.empty_like(lo)
        for _ in range(5):
            g.evaluate_branch_batch_device(ctx, dn.data_ptr(), n, lo.data_ptr(), up.data_ptr(), 0, float("inf"), st.cuda_stream)
        st.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(100):
            g.evaluate_branch_batch_device(ctx, dn.data_ptr(), n, lo.data_ptr(), up.data_ptr(), 0, float("inf"), st.cuda_stream)
        e1.record(st); st.synchronize()
        dev_us = e0.elapsed_time(e1) * 10
        t = time.perf_counter()
        for _ in range(100):
            g.evaluate_branch_batch(ctx, nodes)
        host_us = (time.perf_counter() - t) * 1e4
        print(f"{n1}x{n2} n={n}: device-resident {dev_us:.1f} us/launch, host API {host_us:.1f} us/call", flush=True)
