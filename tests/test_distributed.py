"""The frontier-sharded driver (paper_1812_01232_b200/distributed.py) on CPU:
world-size-2 gloo process groups running the exact exchange code the GPU ranks
run (min-allreduce of the incumbent and frontier minimum, the stop rules,
rebalancing by point-to-point node transfer). The shards here are a host-side
1-D branch-and-bound with the same interface as ShardSolver, so the test needs
no GPU; the GPU shard itself is covered by tests/test_solver_gpu.py."""
import heapq
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1812_01232_b200.distributed import Comm, plan_rebalance, solve_sharded

A = np.array([1.0, 0.6, 0.35, 0.2])
W = np.array([3.1, 7.3, 13.9, 29.0])
P = np.array([0.3, 1.1, 2.0, 0.7])
LIP = float(np.sum(np.abs(A * W)))
L = 6.0
N_ROOTS = 24


def f(x):
    return float(np.sum(A * np.cos(W * x + P)))


def brute_min():
    xs = np.linspace(0, L, 2_000_001)
    return float(np.min(np.sum(A[:, None] * np.cos(W[:, None] * xs[None, :] + P[:, None]), 0)))


class ToyShard:
    """1-D Lipschitz branch-and-bound with ShardSolver's interface. Nodes are
    rows of the 11-double gosma_node layout (rc[0] = centre, rhw = half width,
    lower in slot 10) so packing/transfer is exercised for real."""

    def __init__(self, rank, world, roots=None):
        h = L / N_ROOTS / 2
        owned = roots if roots is not None else range(rank, N_ROOTS, world)
        self.heap = []
        self.inc = math.inf
        self.x = None
        self.external = math.inf
        self.evals = 0
        self.floor = math.inf
        for k in owned:
            self._push(self._node((2 * k + 1) * h, h, -math.inf), 1.0)

    def _node(self, c, h, parent_lower):
        n = np.zeros(11)
        n[0], n[3] = c, h
        lo = max(f(c) - LIP * h, parent_lower)
        n[10] = lo
        self.evals += 1
        v = f(c)
        if v < self.inc:
            self.inc, self.x = v, c
        return n

    def _push(self, n, vol):
        heapq.heappush(self.heap, (n[10], n[0], n.tolist(), vol))

    def dstar(self):
        return min(self.inc, self.external)

    def status(self):
        live = [e for e in self.heap if e[0] < self.dstar()]
        return {"best_value": self.inc, "frontier_min": self.heap[0][0] if self.heap else math.inf,
                "floor_lower": self.floor, "live_nodes": len(live),
                "bound_evaluations": self.evals}

    def set_incumbent(self, v):
        self.external = min(self.external, v)

    def expand(self, limit, max_evals=0):
        for _ in range(16):
            if not self.heap or self.heap[0][0] >= limit:
                break
            lo, c, n, vol = heapq.heappop(self.heap)
            h = n[3] / 2
            for cc in (c - h, c + h):
                kid = self._node(cc, h, lo)
                if kid[10] < self.dstar():
                    if h < 1e-9:
                        self.floor = min(self.floor, kid[10])
                    else:
                        self._push(kid, vol / 2)

    def export(self, n):
        out = [heapq.heappop(self.heap) for _ in range(min(n, len(self.heap)))]
        nodes = np.array([e[2] for e in out]).reshape(-1, 11)
        vol = np.array([e[3] for e in out])
        return nodes, np.zeros(len(out), dtype=np.int8), vol

    def import_(self, nodes, split, vol):
        for n, v in zip(nodes, vol):
            self._push(np.asarray(n), float(v))

    def result(self):
        return {"value": self.inc, "r": np.array([self.x if self.x is not None else 0.0, 0, 0]),
                "t": np.zeros(3), "bound_evaluations": self.evals}


def test_plan_rebalance_is_balanced_and_conservative():
    assert plan_rebalance([10, 10]) == []
    assert plan_rebalance([100]) == []
    plan = plan_rebalance([100, 0, 0, 20])
    counts = [100, 0, 0, 20]
    for s, d, n in plan:
        counts[s] -= n
        counts[d] += n
    assert sum(counts) == 120
    assert max(counts) - min(counts) <= 2
    assert all(s == 0 or s == 3 for s, _, _ in plan)


def test_single_rank_matches_brute_force():
    comm = Comm()
    rep = solve_sharded(ToyShard(0, 1), 1e-3, comm)
    assert rep.status == "epsilon_optimal"
    m = brute_min()
    assert rep.global_lower <= m + 1e-9
    assert rep.best_value <= m + 1e-3
    assert abs(rep.best_value - f(rep.r[0])) < 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, skew, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        roots = (range(N_ROOTS) if rank == 0 else []) if skew else None
        shard = ToyShard(rank, world, roots)
        rep = solve_sharded(shard, 1e-3, Comm(), rebalance_every=1, max_migrate=64)
        q.put((rank, rep.best_value, rep.global_lower, rep.status, float(rep.r[0]),
               rep.migrated_nodes, rep.bound_evaluations))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("skew", [False, True])
def test_two_ranks_gloo_same_certified_optimum(skew):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, skew, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(2))
    m = brute_min()
    for rank, best, lower, status, x, migrated, evals in res:
        assert status == "epsilon_optimal"
        assert lower <= m + 1e-9 and best <= m + 1e-3
        assert abs(best - f(x)) < 1e-12
    # both ranks agree on the result
    assert res[0][1] == res[1][1] and res[0][2] == res[1][2]
    if skew:
        assert res[0][5] > 0  # rank 0 owned every root: work had to migrate
