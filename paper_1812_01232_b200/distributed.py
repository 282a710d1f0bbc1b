"""Frontier-sharded branch-and-bound across GPUs.

One process per GPU (torchrun), one ``ShardSolver`` per rank. Every rank runs
wave 0 and the discovery dive on all roots (the same d* everywhere), expands
the roots deterministically to >= 8 x SMs nodes and keeps every world-th
(SURVEY.md §8(e)). Every wave:

1. each rank contributes one 5-double record {d*_local, min(frontier min,
   resolved floor), elapsed, live nodes, evaluations} to ONE tiny all-gather
   (NCCL over NVLink for CUDA tensors, gloo on CPU); every rank reduces the
   records identically (min, min, max, sum, sum);
2. certified = max(prev, min(d*, global min)) (solver.cpp:626-627); the stop
   rules (solver.cpp:629-645) are evaluated identically on every rank;
3. the global d* is pushed into every shard (it prunes there, soundly);
4. each shard expands its best nodes below d* - eps;
5. every ``rebalance_every`` waves, when the gathered live-frontier sizes
   differ by more than ``imbalance``, donors hand their best nodes to
   receivers (point-to-point, deterministic pairing; no extra collective).

The shard interface (status / set_incumbent / expand / export / import_ /
result) is duck-typed, so the exchange logic is tested on CPU with gloo and a
host-side toy shard (tests/test_distributed.py).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None
    dist = None


@dataclass
class ShardedReport:
    best_value: float
    global_lower: float
    gap: float
    status: str
    r: np.ndarray
    t: np.ndarray
    bound_evaluations: int
    waves: int
    migrated_nodes: int
    wall_time_seconds: float
    trace: List[tuple] = field(default_factory=list)


class Comm:
    """Collectives of the driver over a torch.distributed process group."""

    def __init__(self, device=None, group=None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.device = device if device is not None else torch.device("cpu")

    def _t(self, values, dtype=torch.float64):
        return torch.tensor(values, dtype=dtype, device=self.device)

    def allreduce(self, values, op="min"):
        t = self._t(values)
        if self.world > 1:
            dist.all_reduce(t, op={"min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX,
                                   "sum": dist.ReduceOp.SUM}[op], group=self.group)
        return t.cpu().numpy()

    def allgather(self, value: float):
        return self.allgather_rows([value])[:, 0]

    def allgather_rows(self, values):
        """All ranks' equal-length records as a (world, len) array (one collective)."""
        t = self._t(values)
        if self.world == 1:
            return t.cpu().numpy().reshape(1, -1)
        out = torch.empty(self.world * t.numel(), dtype=t.dtype, device=self.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy().reshape(self.world, -1)

    def send_array(self, arr: np.ndarray, dst: int):
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(self.device)
        n = self._t([t.shape[0]], torch.int64)
        dist.send(n, dst, group=self.group)
        if t.shape[0]:
            dist.send(t.reshape(-1), dst, group=self.group)

    # node records as device tensors (uint8 node bytes, int8 split, f64 volume)
    def send_tensors(self, tensors, dst: int):
        nodes, split, vol = tensors
        n = self._t([split.numel()], torch.int64)
        dist.send(n, dst, group=self.group)
        if split.numel():
            for t in (nodes, split, vol):
                dist.send(t.contiguous(), dst, group=self.group)

    def recv_tensors(self, src: int):
        n = self._t([0], torch.int64)
        dist.recv(n, src, group=self.group)
        k = int(n.item())
        nodes = torch.empty(k * NODE_BYTES, dtype=torch.uint8, device=self.device)
        split = torch.empty(k, dtype=torch.int8, device=self.device)
        vol = torch.empty(k, dtype=torch.float64, device=self.device)
        if k:
            for t in (nodes, split, vol):
                dist.recv(t, src, group=self.group)
        if self.device.type == "cuda":
            # NCCL receives are ordered on torch's current stream only; the
            # solver's import copies on its own stream, so wait here
            torch.cuda.current_stream(self.device).synchronize()
        return nodes, split, vol

    def recv_array(self, src: int, width: int) -> np.ndarray:
        n = self._t([0], torch.int64)
        dist.recv(n, src, group=self.group)
        k = int(n.item())
        if k == 0:
            return np.zeros((0, width))
        t = torch.empty(k * width, dtype=torch.float64, device=self.device)
        dist.recv(t, src, group=self.group)
        return t.cpu().numpy().reshape(k, width)


def plan_rebalance(counts, imbalance: float = 1.5, min_move: int = 1):
    """Deterministic transfer plan [(src, dst, n)] that moves the live-frontier
    sizes toward their mean when max/min exceeds ``imbalance``. Pure function:
    every rank computes the same plan from the all-gathered counts."""
    counts = [int(c) for c in counts]
    world = len(counts)
    if world < 2:
        return []
    hi, lo = max(counts), min(counts)
    if hi < min_move or hi <= imbalance * max(lo, 1):
        return []
    mean = sum(counts) / world
    donors = [[r, c - int(math.floor(mean))] for r, c in enumerate(counts) if c > mean]
    takers = [[r, int(math.ceil(mean)) - c] for r, c in enumerate(counts) if c < mean]
    plan = []
    di = ti = 0
    while di < len(donors) and ti < len(takers):
        n = min(donors[di][1], takers[ti][1])
        if n >= min_move:
            plan.append((donors[di][0], takers[ti][0], n))
        donors[di][1] -= n
        takers[ti][1] -= n
        if donors[di][1] <= 0:
            di += 1
        if takers[ti][1] <= 0:
            ti += 1
    return plan


NODE_WIDTH = 13  # 11 node doubles + volume + split flag
NODE_BYTES = 88  # gosma_node


def _pack(nodes, split, vol):
    a = np.empty((len(nodes), NODE_WIDTH))
    if len(nodes):
        a[:, :11] = np.asarray(nodes).view(np.float64).reshape(-1, 11)
        a[:, 11] = vol
        a[:, 12] = split
    return a


def _unpack(a):
    nodes = np.ascontiguousarray(a[:, :11])
    return nodes, a[:, 12].astype(np.int8), np.ascontiguousarray(a[:, 11])


def solve_sharded(shard, epsilon: float, comm: Comm, time_limit: Optional[float] = None,
                  max_evaluations: Optional[int] = None, rebalance_every: int = 4,
                  imbalance: float = 1.5, max_migrate: int = 65536,
                  trace: bool = True) -> ShardedReport:
    """Runs the sharded branch-and-bound to the certified gap ``epsilon``."""
    t0 = time.perf_counter()
    certified = -math.inf
    status = "queue_exhausted"
    wave = 0
    migrated = 0
    tr = []
    while True:
        st = shard.status()
        local_min = min(st["frontier_min"], st["floor_lower"])
        rows = comm.allgather_rows([st["best_value"], local_min, time.perf_counter() - t0,
                                    float(st["live_nodes"]), float(st["bound_evaluations"])])
        dstar, gmin = float(rows[:, 0].min()), float(rows[:, 1].min())
        elapsed = float(rows[:, 2].max())
        counts = rows[:, 3]
        live, evals = int(counts.sum()), int(rows[:, 4].sum())
        certified = max(certified, min(dstar, gmin))
        if trace:
            tr.append((wave, evals, dstar, certified, live, elapsed))
        if dstar - certified <= epsilon:
            status = "epsilon_optimal"
            break
        if live == 0:
            status = "queue_exhausted"
            break
        if time_limit is not None and elapsed >= time_limit:
            status = "time_limit"
            break
        if max_evaluations is not None and evals >= max_evaluations:
            status = "time_limit"
            break
        shard.set_incumbent(dstar)
        budget = 0
        if max_evaluations is not None:
            budget = max(1, (max_evaluations - evals) // comm.world)
        shard.expand(dstar - epsilon, budget)
        wave += 1
        if comm.world > 1 and rebalance_every > 0 and wave % rebalance_every == 0:
            # the sizes gathered at the top of this wave (no extra collective)
            device_path = comm.device.type == "cuda" and hasattr(shard, "export_device")
            for src, dst, n in plan_rebalance(counts, imbalance):
                n = min(n, max_migrate)
                if device_path:
                    # node records move GPU -> GPU over NCCL, no host staging
                    if comm.rank == src:
                        comm.send_tensors(shard.export_device(n, comm.device), dst)
                    elif comm.rank == dst:
                        shard.import_device(*comm.recv_tensors(src))
                elif comm.rank == src:
                    comm.send_array(_pack(*shard.export(n)), dst)
                elif comm.rank == dst:
                    nodes, split, vol = _unpack(comm.recv_array(src, NODE_WIDTH))
                    shard.import_(nodes, split, vol)
                migrated += n
    # The rank holding the best incumbent publishes its pose.
    res = shard.result()
    best = comm.allreduce([res["value"]], "min")[0]
    owner = comm.allreduce([comm.rank if res["value"] == best else comm.world], "min")[0]
    pose = np.concatenate([res["r"], res["t"]]) if comm.rank == owner else np.zeros(6)
    pose = comm.allreduce(list(pose), "sum")
    evals = int(comm.allreduce([float(res["bound_evaluations"])], "sum")[0])
    return ShardedReport(best_value=float(best), global_lower=certified,
                         gap=float(best) - certified, status=status, r=pose[:3], t=pose[3:],
                         bound_evaluations=evals, waves=wave, migrated_nodes=migrated,
                         wall_time_seconds=time.perf_counter() - t0, trace=tr)
