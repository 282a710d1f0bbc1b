"""Dev script: GPU vs oracle on seeded inputs + a quick microbench timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_01232_b200 as g
from paper_1812_01232_b200 import synth
from oracle.bind import Oracle, Mixture

def run(regime, n1, n2, n, seed, zeta, kcap=150.0, ncls=1, **kw):
    cls = synth.mixture(n1, n2, regime, seed=seed, kappa_cap=kcap, n_classes=ncls)
    ctx = g.ObjectiveContext(cls, zeta)
    ctx.set_lb_margin(-1.0)
    nodes = synth.nodes(n, seed=seed + 1, **kw)
    lo, up, sp = g.evaluate_branch_batch(ctx, nodes, return_split=True)
    o = Oracle(Mixture(**synth.to_mixture_arrays(cls, zeta)))
    rlo, rup, lm, um, rsp = o.eval_bounds(nodes.view(np.float64).reshape(-1, 11), threads=8)
    fin = np.isfinite(rlo)
    e_lo = np.abs(lo[fin] - rlo[fin]) / lm[fin]
    fu = np.isfinite(rup)
    e_up = np.abs(up[fu] - rup[fu]) / um[fu]
    print(f"{regime:9s} {n1}x{n2} c{ncls} n={n}: feasible {fin.sum()} inf-match lo {np.array_equal(np.isinf(lo), np.isinf(rlo))} up {np.array_equal(np.isinf(up), np.isinf(rup))} "
          f"| lo err/mass max {e_lo.max():.3e} p99 {np.quantile(e_lo,0.99):.3e} | up err/mass max {e_up.max():.3e} p99 {np.quantile(e_up,0.99):.3e} | split agree {np.mean(sp==rsp):.4f}")
    bad = np.argsort(-e_lo)[:3]
    for b in bad:
        k = np.flatnonzero(fin)[b]
        print("   worst lo", k, lo[k], rlo[k], lm[k], nodes[k])

for args in [] or [("moderate",4,3,2000,31,0.2,40.0), ("moderate",3,3,2000,42,0.15,150.0), ("moderate",64,32,300,7,0.2,150.0),
             ("realistic",64,32,300,2026,0.5), ("realistic",8,6,2000,5,0.5), ("moderate",5,4,1000,9,0.2,60.0,3)]:
    run(*args)

# microbench timing (1M nodes, 64x32 realistic)
import torch
cls = synth.mixture(64, 32, "realistic", seed=2026)
ctx = g.ObjectiveContext(cls, 0.5)
nodes = synth.nodes(1_000_000, seed=2027)
dn = torch.from_numpy(nodes.view(np.uint8)).cuda()
lo = torch.empty(len(nodes), dtype=torch.float64, device="cuda")
up = torch.empty_like(lo)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
s = st.cuda_stream
for _ in range(2):
    g.evaluate_branch_batch_device(ctx, dn.data_ptr(), len(nodes), lo.data_ptr(), up.data_ptr(), stream=s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    g.evaluate_branch_batch_device(ctx, dn.data_ptr(), len(nodes), lo.data_ptr(), up.data_ptr(), stream=s)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
P = synth.pair_terms_per_node(cls)
print(f"1M nodes 64x32: {ms:.2f} ms/launch -> {1e6/ms*1e3:.3e} nodes/s, {P*1e6/ms*1e3:.3e} pair-terms/s")
