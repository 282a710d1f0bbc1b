"""B200-native GOSMA bound evaluation — Python host mirror of the reference
solver API (/root/reference/proj/core/include/smalign/*.hpp) over the C ABI
in include/gosma_capi.h (libgosma.so, built in-tree by csrc/Makefile).

There is no CPU fallback: the first call into the package without a built
libgosma.so raises ImportError, and a compute entry point without a CUDA
device raises GosmaError. The library is mapped on first use, so the pure
data helpers (NODE_DTYPE, synth) load nothing native (bench.py's reference
arm relies on that: it must not map libgosma.so).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

__all__ = [
    "GosmaError", "InfeasiblePoseError", "ObjectiveContext", "NODE_DTYPE", "make_nodes",
    "evaluate_branch_batch", "evaluate_bounds", "objective_value", "objective_gradient",
    "SolverConfig", "SolverReport", "PoseDomain", "solve", "local_refine", "local_refine_batch", "lib", "library_path",
    "kernel_launches", "evaluate_branch_batch_device", "evaluate_branch_batch_cached_device",
    "evaluate_children_device", "objective_batch", "ShardSolver", "build_semantic_mixtures",
    "dp_means", "dp_vmf_means", "release_cached_memory", "calibrate_pipes", "device_info",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# GOSMA_LIBRARY selects an alternative in-tree build (kernel-variant A/B runs).
library_path = os.environ.get("GOSMA_LIBRARY") or os.path.join(_HERE, "libgosma.so")

GOSMA_OK, GOSMA_EINVAL, GOSMA_EINFEASIBLE, GOSMA_EBUDGET = 0, 1, 2, 3


class GosmaError(RuntimeError):
    """A C-ABI failure (CUDA or internal)."""


class InfeasiblePoseError(ValueError):
    """Mirrors smalign::InfeasiblePoseError (errors.hpp:16-21)."""


class _ClassView(C.Structure):
    _fields_ = [("n1", C.c_int), ("n2", C.c_int), ("class_weight", C.c_double),
                ("mu", C.POINTER(C.c_double)), ("sigma2", C.POINTER(C.c_double)),
                ("phi1", C.POINTER(C.c_double)), ("dir", C.POINTER(C.c_double)),
                ("kappa2", C.POINTER(C.c_double)), ("phi2", C.POINTER(C.c_double))]


class _Domain(C.Structure):
    _fields_ = [("rot_center", C.c_double * 3), ("rot_half_width", C.c_double),
                ("boxes", C.POINTER(C.c_double)), ("n_boxes", C.c_int)]


class _Config(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("zeta", C.c_double), ("batch_size", C.c_int),
                ("time_limit", C.c_double), ("max_evaluations", C.c_longlong),
                ("queue_capacity", C.c_longlong), ("threads", C.c_int),
                ("seed", C.c_ulonglong), ("wave_nodes", C.c_int), ("discovery_dive", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("best_r", C.c_double * 3), ("best_t", C.c_double * 3),
                ("best_value", C.c_double), ("global_lower", C.c_double), ("gap", C.c_double),
                ("status", C.c_int), ("branches_expanded", C.c_ulonglong),
                ("sma_invocations", C.c_ulonglong), ("bound_evaluations", C.c_ulonglong),
                ("wall_time_seconds", C.c_double), ("waves", C.c_ulonglong)]


class _WaveStatus(C.Structure):
    _fields_ = [("best_value", C.c_double), ("frontier_min", C.c_double),
                ("floor_lower", C.c_double), ("live_nodes", C.c_ulonglong),
                ("bound_evaluations", C.c_ulonglong), ("pruned_volume", C.c_double),
                ("resolved_volume", C.c_double), ("total_volume", C.c_double),
                ("elapsed_seconds", C.c_double)]


_TRACE_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_ulonglong, C.c_ulonglong, C.c_double, C.c_double,
                        C.c_ulonglong, C.c_double, C.c_double, C.c_double)

_dp = C.POINTER(C.c_double)


def _load():
    if not os.path.exists(library_path):
        raise ImportError(
            f"{library_path} is missing: build it with `make -C {_HERE}/csrc` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    lib = C.CDLL(library_path)
    vp = C.c_void_p
    lib.gosma_last_error.restype = C.c_char_p
    lib.gosma_ctx_create.argtypes = [C.c_int, C.POINTER(_ClassView), C.c_int, C.c_double,
                                     C.c_uint, C.POINTER(vp)]
    lib.gosma_ctx_blurred.argtypes = [vp, C.c_double, C.c_double, C.POINTER(vp)]
    lib.gosma_ctx_destroy.argtypes = [vp]
    lib.gosma_ctx_image_self_energy.restype = C.c_double
    lib.gosma_ctx_image_self_energy.argtypes = [vp]
    lib.gosma_ctx_zeta.restype = C.c_double
    lib.gosma_ctx_zeta.argtypes = [vp]
    lib.gosma_ctx_set_lb_margin.argtypes = [vp, C.c_double]
    lib.gosma_eval_bounds.argtypes = [vp, vp, C.c_size_t, C.c_double, _dp, _dp, vp]
    lib.gosma_eval_bounds_device.argtypes = [vp, vp, C.c_size_t, C.c_double, vp, vp, vp, vp]
    lib.gosma_eval_bounds_cached_device.argtypes = [vp, vp, C.c_size_t, vp, vp, C.c_size_t,
                                                    C.c_double, vp, vp, vp, vp]
    lib.gosma_objective_value.argtypes = [vp, _dp, _dp, _dp]
    lib.gosma_objective_gradient.argtypes = [vp, _dp, _dp, _dp]
    lib.gosma_local_refine.argtypes = [vp, _dp, _dp, C.POINTER(_Domain), _dp, _dp, _dp]
    lib.gosma_local_refine_batch.argtypes = [vp, C.c_size_t, _dp, _dp, C.POINTER(_Domain), _dp,
                                             _dp, _dp]
    lib.gosma_solve.argtypes = [vp, C.POINTER(_Domain), C.POINTER(_Config), C.POINTER(_Report),
                                _TRACE_CB, vp]
    lib.gosma_device_info.argtypes = [C.c_int] + [C.POINTER(C.c_int)] * 4
    lib.gosma_kernel_launches.restype = C.c_ulonglong
    lib.gosma_calibrate_pipes.argtypes = [C.c_int, _dp, _dp]
    lib.gosma_solver_create.argtypes = [vp, C.POINTER(_Domain), C.POINTER(_Config), C.c_int,
                                        C.c_int, C.POINTER(vp)]
    lib.gosma_solver_destroy.argtypes = [vp]
    lib.gosma_solver_status.argtypes = [vp, C.POINTER(_WaveStatus)]
    lib.gosma_solver_set_incumbent.argtypes = [vp, C.c_double]
    lib.gosma_solver_expand.argtypes = [vp, C.c_double, C.c_ulonglong]
    lib.gosma_solver_export.argtypes = [vp, C.c_size_t, vp, vp, vp, C.POINTER(C.c_size_t)]
    lib.gosma_solver_import.argtypes = [vp, vp, vp, vp, C.c_size_t]
    lib.gosma_solver_result.argtypes = [vp, C.POINTER(_Report)]
    lib.gosma_solver_export_device.argtypes = [vp, C.c_size_t, vp, vp, vp,
                                               C.POINTER(C.c_size_t)]
    lib.gosma_solver_import_device.argtypes = [vp, vp, vp, vp, C.c_size_t]
    lib.gosma_solver_live_volume.argtypes = [vp, _dp]
    lib.gosma_objective_batch.argtypes = [vp, _dp, C.c_size_t, _dp, _dp]
    lib.gosma_eval_children_device.argtypes = [vp, vp, vp, C.c_size_t, C.c_double, vp, vp, vp,
                                               vp]
    lib.gosma_release_cached_memory.argtypes = [C.c_int]
    cpp = C.POINTER(C.c_char_p)
    lib.gosma_mixtures_build.argtypes = [_dp, cpp, C.c_size_t, _dp, cpp, C.c_size_t, C.c_double,
                                         C.c_double, cpp, _dp, C.c_size_t, C.POINTER(vp)]
    lib.gosma_mixtures_class_count.argtypes = [vp]
    lib.gosma_mixtures_class.argtypes = [vp, C.c_int, C.POINTER(_ClassView),
                                         C.POINTER(C.c_char_p)]
    lib.gosma_mixtures_warning_count.argtypes = [vp]
    lib.gosma_mixtures_warning.argtypes = [vp, C.c_int]
    lib.gosma_mixtures_warning.restype = C.c_char_p
    lib.gosma_mixtures_destroy.argtypes = [vp]
    for fn in (lib.gosma_dp_means, lib.gosma_dp_vmf_means):
        fn.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_ulonglong,
                       C.POINTER(C.c_int), _dp, C.c_size_t, C.POINTER(C.c_size_t),
                       C.POINTER(C.c_int)]
    return lib


class _LazyLib:
    """libgosma.so, mapped on first attribute access (then cached)."""

    def __init__(self):
        self._lib = None

    def __getattr__(self, name):
        if name == "_lib":
            raise AttributeError(name)
        if self._lib is None:
            self._lib = _load()
        return getattr(self._lib, name)

    @property
    def loaded(self) -> bool:
        return self._lib is not None


lib = _LazyLib()


def kernel_launches() -> int:
    """Bound-kernel launches issued by this process (gpu_launches evidence)."""
    return int(lib.gosma_kernel_launches())


def calibrate_pipes(device: int = 0):
    """(MUFU ops/s, FP32 FMA flop/s) measured on the device right now."""
    m, f = C.c_double(), C.c_double()
    _check(lib.gosma_calibrate_pipes(device, C.byref(m), C.byref(f)), "calibrate_pipes")
    return m.value, f.value


def device_info(device: int = 0):
    sm, clk, ma, mi = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    _check(lib.gosma_device_info(device, C.byref(sm), C.byref(clk), C.byref(ma), C.byref(mi)),
           "device_info")
    return {"sm_count": sm.value, "sm_clock_khz": clk.value, "cc": (ma.value, mi.value)}


def _check(rc: int, what: str):
    if rc == GOSMA_OK:
        return
    msg = lib.gosma_last_error().decode()
    if rc == GOSMA_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == GOSMA_EINFEASIBLE:
        raise InfeasiblePoseError(f"{what}: {msg}")
    raise GosmaError(f"{what} failed ({rc}): {msg}")


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a.reshape(shape) if shape is not None else a


# gosma_node / BranchRegion record (se3.hpp:38-45): 11 doubles.
NODE_DTYPE = np.dtype([("rc", "<f8", 3), ("rhw", "<f8"), ("tc", "<f8", 3), ("thw", "<f8", 3),
                       ("lower", "<f8")])


def make_nodes(rc, rhw, tc, thw, lower=None) -> np.ndarray:
    """Array of BranchRegion records (rotation cube x translation cuboid)."""
    rc = np.atleast_2d(_f64(rc))
    n = rc.shape[0]
    out = np.empty(n, dtype=NODE_DTYPE)
    out["rc"] = rc
    out["rhw"] = np.broadcast_to(_f64(rhw), (n,))
    out["tc"] = np.broadcast_to(_f64(tc), (n, 3))
    out["thw"] = np.broadcast_to(_f64(thw), (n, 3))
    out["lower"] = -np.inf if lower is None else np.broadcast_to(_f64(lower), (n,))
    return out


def _as_nodes(nodes) -> np.ndarray:
    if isinstance(nodes, np.ndarray) and nodes.dtype == NODE_DTYPE:
        return np.ascontiguousarray(nodes)
    a = _f64(nodes)
    if a.ndim == 1:
        a = a.reshape(-1, 11)
    if a.shape[-1] != 11:
        raise ValueError("nodes must be NODE_DTYPE records or (n, 11) float64")
    return np.ascontiguousarray(a).view(NODE_DTYPE).reshape(-1)


class ObjectiveContext:
    """Mirrors smalign::ObjectiveContext (objective.hpp:17-62).

    ``classes`` is a sequence of dicts with keys mu (n1,3), sigma2 (n1),
    phi1 (n1), dir (n2,3), kappa2 (n2), phi2 (n2) and optionally weight
    (the SemanticMixturePair constructor). With ``single_mixture=True`` it is
    the (Gmm, Vmfmm, zeta) constructor: one class of weight 1.
    """

    def __init__(self, classes: Sequence[dict], zeta: float, device: int = 0,
                 single_mixture: bool = False):
        self._keep = []
        views = (_ClassView * len(classes))()
        for k, c in enumerate(classes):
            mu = _f64(c["mu"]).reshape(-1, 3)
            dirs = _f64(c["dir"]).reshape(-1, 3)
            arrs = [mu, _f64(c["sigma2"]), _f64(c["phi1"]), dirs, _f64(c["kappa2"]),
                    _f64(c["phi2"])]
            self._keep += arrs
            views[k] = _ClassView(mu.shape[0], dirs.shape[0], float(c.get("weight", 1.0)),
                                  *[a.ctypes.data_as(_dp) for a in arrs])
        h = C.c_void_p()
        _check(lib.gosma_ctx_create(device, views, len(classes), float(zeta),
                                    1 if single_mixture else 0, C.byref(h)), "ObjectiveContext")
        self._h = h
        self.device = device
        self.zeta = float(zeta)
        self.classes = [dict(c) for c in classes]
        self._keep = []

    @classmethod
    def _wrap(cls, handle, device, zeta, classes):
        o = cls.__new__(cls)
        o._h, o.device, o.zeta, o.classes, o._keep = handle, device, zeta, classes, []
        return o

    @classmethod
    def from_mixture(cls, mix, device: int = 0):
        """From a flat class-concatenated mixture (oracle.bind.Mixture layout:
        n1, n2, class_weight, mu, sigma2, phi1, dir, kappa2, phi2, zeta)."""
        classes, o1, o2 = [], 0, 0
        for c in range(len(mix.n1)):
            a, b = int(mix.n1[c]), int(mix.n2[c])
            classes.append({"mu": mix.mu[o1:o1 + a], "sigma2": mix.sigma2[o1:o1 + a],
                            "phi1": mix.phi1[o1:o1 + a], "dir": mix.dir[o2:o2 + b],
                            "kappa2": mix.kappa2[o2:o2 + b], "phi2": mix.phi2[o2:o2 + b],
                            "weight": float(mix.class_weight[c])})
            o1, o2 = o1 + a, o2 + b
        return cls(classes, mix.zeta, device=device, single_mixture=False)

    def blurred(self, w: float, reference_distance: float) -> "ObjectiveContext":
        """ObjectiveContext::blurred (objective.cpp:70-101)."""
        h = C.c_void_p()
        _check(lib.gosma_ctx_blurred(self._h, float(w), float(reference_distance), C.byref(h)),
               "blurred")
        return ObjectiveContext._wrap(h, self.device, self.zeta, self.classes)

    @property
    def image_self_energy(self) -> float:
        return lib.gosma_ctx_image_self_energy(self._h)

    @property
    def handle(self):
        return self._h

    def set_lb_margin(self, rel: float):
        _check(lib.gosma_ctx_set_lb_margin(self._h, float(rel)), "set_lb_margin")

    @property
    def all_means(self) -> np.ndarray:
        return np.concatenate([_f64(c["mu"]).reshape(-1, 3) for c in self.classes])

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # lib is None during interpreter shutdown
            lib.gosma_ctx_destroy(h)
            self._h = None


def evaluate_branch_batch(ctx: ObjectiveContext, branches, threads: int = 0,
                          skip_upper_at: float = float("inf"), return_split: bool = False):
    """evaluate_branch_batch (solver.hpp:87-95): (lower, upper) per branch, in
    input order. ``threads`` is accepted for signature parity and ignored (the
    GPU decides its own launch geometry; results do not depend on it)."""
    nodes = _as_nodes(branches)
    n = nodes.shape[0]
    lower = np.empty(n)
    upper = np.empty(n)
    split = np.empty(n, dtype=np.int8) if return_split else None
    if n:
        _check(lib.gosma_eval_bounds(ctx.handle, nodes.ctypes.data, n, float(skip_upper_at),
                                     lower.ctypes.data_as(_dp), upper.ctypes.data_as(_dp),
                                     split.ctypes.data if split is not None else None),
               "evaluate_branch_batch")
    return (lower, upper, split) if return_split else (lower, upper)


def evaluate_bounds(ctx: ObjectiveContext, branch, skip_upper_at: float = float("inf")):
    """evaluate_bounds (bounds.hpp:63-69) for one branch: (lower, upper)."""
    lo, up = evaluate_branch_batch(ctx, [branch] if not isinstance(branch, np.ndarray)
                                   else branch, skip_upper_at=skip_upper_at)
    return float(lo[0]), float(up[0])


def evaluate_branch_batch_device(ctx: ObjectiveContext, d_nodes_ptr: int, n: int,
                                 d_lower_ptr: int, d_upper_ptr: int, d_split_ptr: int = 0,
                                 skip_upper_at: float = float("inf"), stream: int = 0):
    """Device-pointer variant (asynchronous on ``stream``)."""
    _check(lib.gosma_eval_bounds_device(ctx.handle, d_nodes_ptr, n, float(skip_upper_at),
                                        d_lower_ptr, d_upper_ptr, d_split_ptr or None,
                                        stream or None), "evaluate_branch_batch_device")


def evaluate_branch_batch_cached_device(ctx, d_nodes_ptr, n, d_tindex_ptr, d_tboxes_ptr,
                                        n_tboxes, d_lower_ptr, d_upper_ptr, d_split_ptr=0,
                                        skip_upper_at=float("inf"), stream=0):
    """Translation-cached device variant (self terms once per cuboid)."""
    _check(lib.gosma_eval_bounds_cached_device(ctx.handle, d_nodes_ptr, n, d_tindex_ptr,
                                               d_tboxes_ptr, n_tboxes, float(skip_upper_at),
                                               d_lower_ptr, d_upper_ptr, d_split_ptr or None,
                                               stream or None),
           "evaluate_branch_batch_cached_device")


def evaluate_children_device(ctx, d_parents_ptr, d_split_ptr, n, d_lower_ptr, d_upper_ptr,
                             d_child_split_ptr=0, skip_upper_at=float("inf"), stream=0):
    """Branch + bound: bounds of the 8 subdivide_adaptive children of each
    parent (slot 8i+c), rotation-split parents sharing their cuboid work."""
    _check(lib.gosma_eval_children_device(ctx.handle, d_parents_ptr, d_split_ptr, n,
                                          float(skip_upper_at), d_lower_ptr, d_upper_ptr,
                                          d_child_split_ptr or None, stream or None),
           "evaluate_children_device")


def objective_value(ctx: ObjectiveContext, r, t) -> float:
    """objective_value (objective.hpp:79-82), host FP64."""
    v = C.c_double()
    _check(lib.gosma_objective_value(ctx.handle, _f64(r).ctypes.data_as(_dp),
                                     _f64(t).ctypes.data_as(_dp), C.byref(v)), "objective_value")
    return v.value


def release_cached_memory(device: int = 0):
    """Frees the device buffers finished solvers left cached on `device`
    (the parked frontier pool and the exact-size block cache)."""
    _check(lib.gosma_release_cached_memory(device), "release_cached_memory")


def objective_batch(ctx: ObjectiveContext, poses):
    """objective_value + objective_gradient for n poses {r[3], t[3]} on the GPU
    (FP64 batched kernel): (f[n], g[n, 6]); f = +inf where infeasible."""
    x = _f64(poses).reshape(-1, 6)
    f = np.empty(len(x))
    g = np.empty((len(x), 6))
    _check(lib.gosma_objective_batch(ctx.handle, x.ctypes.data_as(_dp), len(x),
                                     f.ctypes.data_as(_dp), g.ctypes.data_as(_dp)),
           "objective_batch")
    return f, g


def objective_gradient(ctx: ObjectiveContext, r, t) -> np.ndarray:
    g = np.empty(6)
    _check(lib.gosma_objective_gradient(ctx.handle, _f64(r).ctypes.data_as(_dp),
                                        _f64(t).ctypes.data_as(_dp), g.ctypes.data_as(_dp)),
           "objective_gradient")
    return g


@dataclass
class PoseDomain:
    """PoseDomain (se3.hpp:32-36): rotation cube + translation cuboids
    ({center[3], half_widths[3]} rows)."""
    rot_center: np.ndarray = field(default_factory=lambda: np.zeros(3))
    rot_half_width: float = float(np.pi)
    boxes: np.ndarray = field(default_factory=lambda: np.zeros((0, 6)))

    def _c(self):
        b = _f64(self.boxes).reshape(-1, 6)
        d = _Domain()
        for k in range(3):
            d.rot_center[k] = float(self.rot_center[k])
        d.rot_half_width = float(self.rot_half_width)
        d.boxes = b.ctypes.data_as(_dp)
        d.n_boxes = b.shape[0]
        return d, b


@dataclass
class SolverConfig:
    """SolverConfig (solver.hpp:14-37)."""
    epsilon: float = 0.1
    zeta: float = 0.5
    batch_size: int = 1024
    time_limit: Optional[float] = None
    queue_capacity: Optional[int] = None
    max_evaluations: Optional[int] = None
    threads: int = 0
    seed: int = 0
    wave_nodes: int = 0
    discovery_dive: bool = True


@dataclass
class SolverReport:
    """SolverReport (solver.hpp:64-73)."""
    r: np.ndarray
    t: np.ndarray
    best_value: float
    global_lower: float
    gap: float
    status: str
    branches_expanded: int
    sma_invocations: int
    bound_evaluations: int
    wall_time_seconds: float
    waves: int
    trace: list


_STATUS = {0: "epsilon_optimal", 1: "time_limit", 2: "queue_exhausted"}


def local_refine(ctx: ObjectiveContext, r0, t0, domain: PoseDomain):
    """local_refine (solver.hpp:80-85): (value, r, t)."""
    d, keep = domain._c()
    r, t, v = np.empty(3), np.empty(3), C.c_double()
    _check(lib.gosma_local_refine(ctx.handle, _f64(r0).ctypes.data_as(_dp),
                                  _f64(t0).ctypes.data_as(_dp), C.byref(d),
                                  r.ctypes.data_as(_dp), t.ctypes.data_as(_dp), C.byref(v)),
           "local_refine")
    return v.value, r, t


def local_refine_batch(ctx: ObjectiveContext, r0, t0, domain: PoseDomain):
    """n local refinements on the GPU (one CTA each):
    (values (n,), r (n, 3), t (n, 3)); values are host FP64 objectives."""
    r0 = np.ascontiguousarray(r0, dtype=np.float64).reshape(-1, 3)
    t0 = np.ascontiguousarray(t0, dtype=np.float64).reshape(-1, 3)
    if r0.shape != t0.shape:
        raise ValueError("r0 and t0 must both be (n, 3)")
    n = r0.shape[0]
    d, keep = domain._c()
    r, t, v = np.empty((n, 3)), np.empty((n, 3)), np.empty(n)
    _check(lib.gosma_local_refine_batch(ctx.handle, n, r0.ctypes.data_as(_dp),
                                        t0.ctypes.data_as(_dp), C.byref(d),
                                        r.ctypes.data_as(_dp), t.ctypes.data_as(_dp),
                                        v.ctypes.data_as(_dp)), "local_refine_batch")
    return v, r, t


def solve(ctx: ObjectiveContext, domain: PoseDomain, config: SolverConfig) -> SolverReport:
    """solve (solver.hpp:97-103) on the GPU-resident frontier."""
    d, keep = domain._c()
    cfg = _Config(config.epsilon, config.zeta, config.batch_size,
                  -1.0 if config.time_limit is None else float(config.time_limit),
                  -1 if config.max_evaluations is None else int(config.max_evaluations),
                  -1 if config.queue_capacity is None else int(config.queue_capacity),
                  config.threads, config.seed, config.wave_nodes, int(config.discovery_dive))
    rep = _Report()
    trace = []

    def cb(_u, wave, evals, ub, lb, q, fu, fp, fr):
        trace.append((wave, evals, ub, lb, q, fu, fp, fr))

    ccb = _TRACE_CB(cb)
    rc = lib.gosma_solve(ctx.handle, C.byref(d), C.byref(cfg), C.byref(rep), ccb, None)
    if rc not in (GOSMA_OK, GOSMA_EBUDGET):
        _check(rc, "solve")
    return SolverReport(np.array(rep.best_r[:]), np.array(rep.best_t[:]), rep.best_value,
                        rep.global_lower, rep.gap, _STATUS.get(rep.status, "?"),
                        rep.branches_expanded, rep.sma_invocations, rep.bound_evaluations,
                        rep.wall_time_seconds, rep.waves, trace)


def _config_struct(config: SolverConfig) -> _Config:
    return _Config(config.epsilon, config.zeta, config.batch_size,
                   -1.0 if config.time_limit is None else float(config.time_limit),
                   -1 if config.max_evaluations is None else int(config.max_evaluations),
                   -1 if config.queue_capacity is None else int(config.queue_capacity),
                   config.threads, config.seed, config.wave_nodes, int(config.discovery_dive))


class ShardSolver:
    """One rank's share of the branch-and-bound (gosma_solver_*): the frontier
    of the translation roots rank, rank+world, ... on this GPU. Driven by
    distributed.solve_sharded; world=1 reproduces solve()."""

    def __init__(self, ctx: ObjectiveContext, domain: PoseDomain, config: SolverConfig,
                 rank: int = 0, world: int = 1):
        self._ctx = ctx  # keeps the context alive
        d, self._boxes = domain._c()
        self._dom = d
        self.config = config
        h = C.c_void_p()
        _check(lib.gosma_solver_create(ctx.handle, C.byref(d), C.byref(_config_struct(config)),
                                       rank, world, C.byref(h)), "solver_create")
        self._h = h

    def status(self) -> dict:
        st = _WaveStatus()
        _check(lib.gosma_solver_status(self._h, C.byref(st)), "solver_status")
        return {k: getattr(st, k) for k, _ in _WaveStatus._fields_}

    def live_volume(self) -> float:
        """Volume of the live frontier (ledger check: total = pruned + resolved + live)."""
        v = C.c_double()
        _check(lib.gosma_solver_live_volume(self._h, C.byref(v)), "solver_live_volume")
        return v.value

    def set_incumbent(self, value: float):
        _check(lib.gosma_solver_set_incumbent(self._h, float(value)), "solver_set_incumbent")

    def expand(self, limit: float, max_evals: int = 0):
        _check(lib.gosma_solver_expand(self._h, float(limit), int(max(0, max_evals))),
               "solver_expand")

    def export(self, max_nodes: int):
        nodes = np.empty(max_nodes, dtype=NODE_DTYPE)
        split = np.empty(max_nodes, dtype=np.int8)
        vol = np.empty(max_nodes)
        n = C.c_size_t(0)
        _check(lib.gosma_solver_export(self._h, max_nodes, nodes.ctypes.data, split.ctypes.data,
                                       vol.ctypes.data, C.byref(n)), "solver_export")
        k = n.value
        return nodes[:k], split[:k], vol[:k]

    def import_(self, nodes, split, vol):
        nodes = _as_nodes(nodes)
        split = np.ascontiguousarray(split, dtype=np.int8)
        vol = np.ascontiguousarray(vol, dtype=np.float64)
        _check(lib.gosma_solver_import(self._h, nodes.ctypes.data, split.ctypes.data,
                                       vol.ctypes.data, len(nodes)), "solver_import")

    def export_device(self, max_nodes: int, device):
        """Best live nodes into torch CUDA tensors (node bytes uint8[n*88],
        split int8[n], volume float64[n]) for device-to-device rebalancing."""
        import torch
        nodes = torch.empty(max_nodes * NODE_DTYPE.itemsize, dtype=torch.uint8, device=device)
        split = torch.empty(max_nodes, dtype=torch.int8, device=device)
        vol = torch.empty(max_nodes, dtype=torch.float64, device=device)
        # the solver writes them on its own stream: let torch's stream finish
        # any work on the recycled allocations first (the export itself
        # synchronises its stream before returning)
        torch.cuda.current_stream(device).synchronize()
        n = C.c_size_t(0)
        _check(lib.gosma_solver_export_device(self._h, max_nodes, nodes.data_ptr(),
                                              split.data_ptr(), vol.data_ptr(), C.byref(n)),
               "solver_export_device")
        k = n.value
        return nodes[:k * NODE_DTYPE.itemsize], split[:k], vol[:k]

    def import_device(self, nodes, split, vol):
        """Import node records held in torch CUDA tensors (see export_device)."""
        n = split.numel()
        _check(lib.gosma_solver_import_device(self._h, nodes.data_ptr(), split.data_ptr(),
                                              vol.data_ptr(), n), "solver_import_device")

    def result(self) -> dict:
        rep = _Report()
        _check(lib.gosma_solver_result(self._h, C.byref(rep)), "solver_result")
        return {"value": rep.best_value, "r": np.array(rep.best_r[:]),
                "t": np.array(rep.best_t[:]), "branches_expanded": rep.branches_expanded,
                "sma_invocations": rep.sma_invocations,
                "bound_evaluations": rep.bound_evaluations, "waves": rep.waves}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            lib.gosma_solver_destroy(h)
            self._h = None


# ---- mixture construction (host C++; mixtures.hpp:55-98) ---------------------

def _labels(labels, n):
    if labels is None:
        return None, None
    enc = [str(x).encode() for x in labels]
    if len(enc) != n:
        raise ValueError("build_semantic_mixtures: label count mismatch")
    return (C.c_char_p * len(enc))(*enc), enc


def _clustering(fn, data, lam, shuffle_seed, what):
    x = _f64(data).reshape(-1, 3)
    n = len(x)
    asg = np.zeros(n, dtype=np.int32)
    cen = np.zeros((max(n, 1), 3))
    nc, it = C.c_size_t(0), C.c_int(0)
    _check(fn(x.ctypes.data_as(_dp), n, float(lam), int(shuffle_seed is not None),
              int(shuffle_seed or 0), asg.ctypes.data_as(C.POINTER(C.c_int)),
              cen.ctypes.data_as(_dp), len(cen), C.byref(nc), C.byref(it)), what)
    return asg, cen[:nc.value].copy(), it.value


def dp_means(points, lambda_p: float, shuffle_seed: Optional[int] = None):
    """dp_means (mixtures.cpp:49-109): (assignment, centers, iterations)."""
    return _clustering(lib.gosma_dp_means, points, lambda_p, shuffle_seed, "dp_means")


def dp_vmf_means(bearings, lambda_f: float, shuffle_seed: Optional[int] = None):
    """dp_vmf_means (mixtures.cpp:111-182): (assignment, centers, iterations)."""
    return _clustering(lib.gosma_dp_vmf_means, bearings, lambda_f, shuffle_seed, "dp_vmf_means")


def build_semantic_mixtures(points, bearings, lambda_p: float, lambda_f: float,
                            point_labels=None, bearing_labels=None, class_weights=None):
    """build_semantic_mixtures (mixtures.cpp:269-362): returns (classes,
    warnings); each class is a dict {id, weight, mu, sigma2, phi1, dir, kappa2,
    phi2} accepted by ObjectiveContext."""
    p = _f64(points).reshape(-1, 3)
    b = _f64(bearings).reshape(-1, 3)
    pl, _k1 = _labels(point_labels, len(p))
    bl, _k2 = _labels(bearing_labels, len(b))
    wl = w = None
    keep = None
    if class_weights is not None:
        keys = list(class_weights)
        wl, keep = _labels(keys, len(keys))
        w = np.array([float(class_weights[k]) for k in keys])
    h = C.c_void_p()
    _check(lib.gosma_mixtures_build(p.ctypes.data_as(_dp), pl, len(p), b.ctypes.data_as(_dp), bl,
                                    len(b), float(lambda_p), float(lambda_f), wl,
                                    None if w is None else w.ctypes.data_as(_dp),
                                    0 if w is None else len(w), C.byref(h)),
           "build_semantic_mixtures")
    try:
        classes = []
        for k in range(lib.gosma_mixtures_class_count(h)):
            v, cid = _ClassView(), C.c_char_p()
            _check(lib.gosma_mixtures_class(h, k, C.byref(v), C.byref(cid)), "mixtures_class")
            a, bb = v.n1, v.n2
            arr = lambda ptr, m: np.ctypeslib.as_array(ptr, shape=(m,)).copy()  # noqa: E731
            classes.append({"id": cid.value.decode(), "weight": v.class_weight,
                            "mu": arr(v.mu, 3 * a).reshape(-1, 3), "sigma2": arr(v.sigma2, a),
                            "phi1": arr(v.phi1, a), "dir": arr(v.dir, 3 * bb).reshape(-1, 3),
                            "kappa2": arr(v.kappa2, bb), "phi2": arr(v.phi2, bb)})
        warnings = [lib.gosma_mixtures_warning(h, k).decode()
                    for k in range(lib.gosma_mixtures_warning_count(h))]
    finally:
        lib.gosma_mixtures_destroy(h)
    return classes, warnings
