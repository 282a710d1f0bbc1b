"""Two launches of K1 on the same configs[1] batch: counts and shows the nodes
whose bounds differ bitwise (the kernel is meant to be deterministic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1812_01232_b200 as g  # noqa: E402
from paper_1812_01232_b200 import synth  # noqa: E402

n1, n2 = int(os.environ.get("N1", 64)), int(os.environ.get("N2", 32))
classes = synth.mixture(n1, n2, os.environ.get("REGIME", "realistic"), seed=2026)
ctx = g.ObjectiveContext(classes, 0.5)
n = int(os.environ.get("NODES", 1_000_000))
nodes = synth.nodes(n, seed=2027)
d_nodes = torch.from_numpy(nodes.view(np.uint8)).cuda()
outs = []
s = torch.cuda.Stream()
d_lo = torch.empty(n, dtype=torch.float64, device="cuda")
d_up = torch.empty_like(d_lo)
d_sp = torch.empty(n, dtype=torch.int8, device="cuda")
for rep in range(3):
    if not os.environ.get("REUSE"):
        d_lo = torch.empty(n, dtype=torch.float64, device="cuda")
        d_up = torch.empty_like(d_lo)
        d_sp = torch.empty(n, dtype=torch.int8, device="cuda")
    with torch.cuda.stream(s):
        g.evaluate_branch_batch_device(ctx, d_nodes.data_ptr(), n, d_lo.data_ptr(), d_up.data_ptr(),
                                       d_sp.data_ptr() if os.environ.get("SPLIT") else 0,
                                       float("inf"), s.cuda_stream)
    s.synchronize()
    outs.append((d_lo.cpu().numpy(), d_up.cpu().numpy()))
for k in (1, 2):
    dl = np.flatnonzero(~((outs[0][0] == outs[k][0]) | (np.isnan(outs[0][0]) & np.isnan(outs[k][0]))))
    du = np.flatnonzero(~((outs[0][1] == outs[k][1]) | (np.isnan(outs[0][1]) & np.isnan(outs[k][1]))))
    print(f"launch {k}: {len(dl)} LB and {len(du)} UB differ")
    for i in dl[:5]:
        print("  ", i, outs[0][0][i], outs[k][0][i], nodes.view(np.float64).reshape(-1, 11)[i])
