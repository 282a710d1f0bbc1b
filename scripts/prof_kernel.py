"""Profiling driver: a few bound-kernel launches on the config-2 workload."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_01232_b200 as g
from paper_1812_01232_b200 import synth
n = int(os.environ.get("NODES", "1000000"))
n1, n2 = int(os.environ.get("N1", "64")), int(os.environ.get("N2", "32"))
cls = synth.mixture(n1, n2, os.environ.get("REGIME", "realistic"), seed=2026)
ctx = g.ObjectiveContext(cls, 0.5)
nodes = synth.nodes(n, seed=2027)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
dn = torch.from_numpy(nodes.view(np.uint8)).cuda()
lo = torch.empty(n, dtype=torch.float64, device="cuda"); up = torch.empty_like(lo)
for _ in range(int(os.environ.get("LAUNCHES", "3"))):
    g.evaluate_branch_batch_device(ctx, dn.data_ptr(), n, lo.data_ptr(), up.data_ptr(), 0, float("inf"), st.cuda_stream)
torch.cuda.synchronize()
print("ok", float(lo.min()), float(up.min()))
