"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU checkers.

* ``Oracle``: oracle/liboracle.so, the plain-C restatement (gosma_oracle.c).
* ``Reference``: oracle/_ref/libsmalign_ref.so, the unmodified reference
  compiled in place (oracle/Makefile, ref_capi.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsmalign_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def _d(a):
    return a.ctypes.data_as(_dp)


def _i(a):
    return a.ctypes.data_as(_ip)


def build_oracle() -> str:
    """Compile liboracle.so if missing (gcc is present on every box of this image)."""
    src = os.path.join(HERE, "gosma_oracle.c")
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "oracle"])
    return ORACLE_SO


class Mixture:
    """Flat, class-concatenated mixture description shared by both checkers and
    by the product ABI (gosma_class_view)."""

    def __init__(self, n1, n2, class_weight, mu, sigma2, phi1, dir_, kappa2, phi2, zeta):
        self.n1 = np.ascontiguousarray(n1, dtype=np.int32)
        self.n2 = np.ascontiguousarray(n2, dtype=np.int32)
        self.class_weight = np.ascontiguousarray(class_weight, dtype=np.float64)
        self.mu = np.ascontiguousarray(mu, dtype=np.float64).reshape(-1, 3)
        self.sigma2 = np.ascontiguousarray(sigma2, dtype=np.float64)
        self.phi1 = np.ascontiguousarray(phi1, dtype=np.float64)
        self.dir = np.ascontiguousarray(dir_, dtype=np.float64).reshape(-1, 3)
        self.kappa2 = np.ascontiguousarray(kappa2, dtype=np.float64)
        self.phi2 = np.ascontiguousarray(phi2, dtype=np.float64)
        self.zeta = float(zeta)

    @property
    def n_classes(self):
        return int(self.n1.shape[0])

    def to_dict(self):
        return {k: (v.tolist() if isinstance(v, np.ndarray) else v)
                for k, v in self.__dict__.items()}

    @staticmethod
    def from_dict(d):
        return Mixture(d["n1"], d["n2"], d["class_weight"], d["mu"], d["sigma2"], d["phi1"],
                       d["dir"], d["kappa2"], d["phi2"], d["zeta"])


class Oracle:
    """The C restatement. ``eval_bounds`` returns (lower, upper, lb_mass,
    ub_mass, split_rot)."""

    def __init__(self, mix: Mixture):
        lib = C.CDLL(build_oracle())
        self._lib = lib
        lib.oracle_ctx_create.restype = C.c_void_p
        lib.oracle_ctx_create.argtypes = [C.c_int, _ip, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                          C.c_double]
        lib.oracle_ctx_blurred.restype = C.c_void_p
        lib.oracle_ctx_blurred.argtypes = [C.c_void_p, C.c_double, C.c_double]
        lib.oracle_ctx_destroy.argtypes = [C.c_void_p]
        lib.oracle_last_error.restype = C.c_char_p
        lib.oracle_ctx_self_energy.restype = C.c_double
        lib.oracle_ctx_self_energy.argtypes = [C.c_void_p]
        lib.oracle_eval_bounds.argtypes = [C.c_void_p, _dp, C.c_long, C.c_double, _dp, _dp, _dp,
                                           _dp, _ip, C.c_int]
        lib.oracle_objective_value.restype = C.c_double
        lib.oracle_objective_value.argtypes = [C.c_void_p, _dp, _dp]
        lib.oracle_feasible_center.argtypes = [C.c_void_p, _dp, _dp]
        lib.oracle_subdivide.argtypes = [C.c_void_p, _dp, _dp]
        lib.oracle_log_z.restype = C.c_double
        lib.oracle_log_z.argtypes = [C.c_double]
        lib.oracle_psi_trans.restype = C.c_double
        lib.oracle_psi_trans.argtypes = [_dp, _dp, _dp]
        self.mix = mix
        self._ctx = lib.oracle_ctx_create(mix.n_classes, _i(mix.n1), _i(mix.n2),
                                          _d(mix.class_weight), _d(mix.mu), _d(mix.sigma2),
                                          _d(mix.phi1), _d(mix.dir), _d(mix.kappa2),
                                          _d(mix.phi2), mix.zeta)
        if not self._ctx:
            raise ValueError(lib.oracle_last_error().decode())

    def __del__(self):
        if getattr(self, "_ctx", None):
            self._lib.oracle_ctx_destroy(self._ctx)
            self._ctx = None

    def blurred(self, w, ref_dist):
        o = Oracle.__new__(Oracle)
        o._lib = self._lib
        o.mix = None
        o._ctx = self._lib.oracle_ctx_blurred(self._ctx, w, ref_dist)
        return o

    @property
    def self_energy(self):
        return self._lib.oracle_ctx_self_energy(self._ctx)

    def log_z(self, k):
        return self._lib.oracle_log_z(float(k))

    def psi_trans(self, tc, thw, p):
        a = [np.ascontiguousarray(x, dtype=np.float64) for x in (tc, thw, p)]
        return self._lib.oracle_psi_trans(_d(a[0]), _d(a[1]), _d(a[2]))

    def eval_bounds(self, nodes, skip=float("inf"), threads=1):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 11)
        n = nodes.shape[0]
        lo, up, lm, um = (np.empty(n) for _ in range(4))
        sr = np.empty(n, dtype=np.int32)
        self._lib.oracle_eval_bounds(self._ctx, _d(nodes), n, skip, _d(lo), _d(up), _d(lm),
                                     _d(um), _i(sr), threads)
        return lo, up, lm, um, sr

    def objective(self, r, t):
        r = np.ascontiguousarray(r, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        return self._lib.oracle_objective_value(self._ctx, _d(r), _d(t))

    def feasible_center(self, node):
        node = np.ascontiguousarray(node, dtype=np.float64)
        t = np.empty(3)
        rc = self._lib.oracle_feasible_center(self._ctx, _d(node), _d(t))
        return t if rc == 0 else None

    def subdivide(self, node):
        node = np.ascontiguousarray(node, dtype=np.float64)
        kids = np.empty((8, 11))
        flag = self._lib.oracle_subdivide(self._ctx, _d(node), _d(kids))
        return flag, kids


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The unmodified reference (oracle/_ref/libsmalign_ref.so)."""

    def __init__(self, mix: Mixture, single_ctor=False):
        if not reference_available():
            raise FileNotFoundError(REF_SO)
        lib = C.CDLL(REF_SO)
        self._lib = lib
        lib.ref_ctx_create.argtypes = [C.c_int, _ip, _ip, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                       C.c_double, C.c_int, C.POINTER(C.c_void_p)]
        lib.ref_ctx_blurred.argtypes = [C.c_void_p, C.c_double, C.c_double,
                                        C.POINTER(C.c_void_p)]
        lib.ref_ctx_destroy.argtypes = [C.c_void_p]
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_ctx_self_energy.restype = C.c_double
        lib.ref_ctx_self_energy.argtypes = [C.c_void_p]
        lib.ref_ctx_image_cache.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_eval_bounds.argtypes = [C.c_void_p, _dp, C.c_long, C.c_int, C.c_double, _dp, _dp]
        lib.ref_objective_value.restype = C.c_double
        lib.ref_objective_value.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_objective_gradient.argtypes = [C.c_void_p, _dp, _dp, _dp]
        lib.ref_upper_bound_pose.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_subdivide.argtypes = [C.c_void_p, _dp, _dp]
        lib.ref_local_refine.argtypes = [C.c_void_p, _dp, _dp, _dp, C.c_double, _dp, C.c_int,
                                         _dp, _dp, _dp]
        lib.ref_solve.argtypes = [C.c_void_p, _dp, C.c_double, _dp, C.c_int, C.c_double,
                                  C.c_double, C.c_int, C.c_double, C.c_longlong, C.c_longlong,
                                  C.c_int, _dp, C.POINTER(C.c_long), _dp, C.c_long]
        self.mix = mix
        ctx = C.c_void_p()
        rc = lib.ref_ctx_create(mix.n_classes, _i(mix.n1), _i(mix.n2), _d(mix.class_weight),
                                _d(mix.mu), _d(mix.sigma2), _d(mix.phi1), _d(mix.dir),
                                _d(mix.kappa2), _d(mix.phi2), mix.zeta, int(single_ctor),
                                C.byref(ctx))
        if rc != 0:
            raise ValueError(lib.ref_last_error().decode())
        self._ctx = ctx

    def __del__(self):
        if getattr(self, "_ctx", None):
            self._lib.ref_ctx_destroy(self._ctx)
            self._ctx = None

    def blurred(self, w, ref_dist):
        o = Reference.__new__(Reference)
        o._lib = self._lib
        o.mix = None
        ctx = C.c_void_p()
        if self._lib.ref_ctx_blurred(self._ctx, w, ref_dist, C.byref(ctx)) != 0:
            raise ValueError(self._lib.ref_last_error().decode())
        o._ctx = ctx
        return o

    @property
    def self_energy(self):
        return self._lib.ref_ctx_self_energy(self._ctx)

    def image_cache(self, n2_total):
        b = np.empty((n2_total, 3))
        lz = np.empty(n2_total)
        self._lib.ref_ctx_image_cache(self._ctx, _d(b), _d(lz))
        return b, lz

    def eval_bounds(self, nodes, skip=float("inf"), threads=1):
        nodes = np.ascontiguousarray(nodes, dtype=np.float64).reshape(-1, 11)
        n = nodes.shape[0]
        lo, up = np.empty(n), np.empty(n)
        rc = self._lib.ref_eval_bounds(self._ctx, _d(nodes), n, threads, skip, _d(lo), _d(up))
        if rc != 0:
            raise RuntimeError(self._lib.ref_last_error().decode())
        return lo, up

    def objective(self, r, t):
        r = np.ascontiguousarray(r, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        return self._lib.ref_objective_value(self._ctx, _d(r), _d(t))

    def gradient(self, r, t):
        r = np.ascontiguousarray(r, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        g = np.empty(6)
        if self._lib.ref_objective_gradient(self._ctx, _d(r), _d(t), _d(g)) != 0:
            return None
        return g

    def upper_bound_pose(self, node):
        node = np.ascontiguousarray(node, dtype=np.float64)
        t = np.empty(3)
        return t if self._lib.ref_upper_bound_pose(self._ctx, _d(node), _d(t)) == 0 else None

    def subdivide(self, node):
        node = np.ascontiguousarray(node, dtype=np.float64)
        kids = np.empty((8, 11))
        flag = self._lib.ref_subdivide(self._ctx, _d(node), _d(kids))
        return flag, kids

    def local_refine(self, r0, t0, rot_c, rot_hw, boxes):
        r0, t0, rot_c = (np.ascontiguousarray(x, dtype=np.float64) for x in (r0, t0, rot_c))
        boxes = np.ascontiguousarray(boxes, dtype=np.float64).reshape(-1, 6)
        r, t, v = np.empty(3), np.empty(3), np.empty(1)
        rc = self._lib.ref_local_refine(self._ctx, _d(r0), _d(t0), _d(rot_c), rot_hw, _d(boxes),
                                        boxes.shape[0], _d(r), _d(t), _d(v))
        if rc != 0:
            raise RuntimeError(self._lib.ref_last_error().decode())
        return float(v[0]), r, t

    def solve(self, rot_c, rot_hw, boxes, epsilon, zeta, batch_size=1024, time_limit=None,
              max_evaluations=None, queue_capacity=None, threads=0, trace_cap=100000):
        rot_c = np.ascontiguousarray(rot_c, dtype=np.float64)
        boxes = np.ascontiguousarray(boxes, dtype=np.float64).reshape(-1, 6)
        rep = np.zeros(14)
        ntr = C.c_long(0)
        trace = np.zeros((trace_cap, 8))
        rc = self._lib.ref_solve(self._ctx, _d(rot_c), rot_hw, _d(boxes), boxes.shape[0], epsilon,
                                 zeta, batch_size, -1.0 if time_limit is None else time_limit,
                                 -1 if max_evaluations is None else max_evaluations,
                                 -1 if queue_capacity is None else queue_capacity, threads,
                                 _d(rep), C.byref(ntr), _d(trace), trace_cap)
        if rc != 0:
            raise RuntimeError(f"ref_solve rc={rc}: {self._lib.ref_last_error().decode()}")
        n = min(ntr.value, trace_cap)
        return {
            "best_value": rep[0], "global_lower": rep[1], "gap": rep[2], "status": int(rep[3]),
            "branches_expanded": int(rep[4]), "sma_invocations": int(rep[5]),
            "bound_evaluations": int(rep[6]), "wall_time": rep[7], "r": rep[8:11].copy(),
            "t": rep[11:14].copy(), "trace": trace[:n].copy(),
        }


def reference_scene_mixtures(n_inliers, omega_3d, omega_2d, noise_px, seed, lambda_p=0.25,
                             lambda_f=2.0 * np.pi / 180.0, zeta=0.5, cap=4096):
    """generate_scene + build_semantic_mixtures through the reference."""
    lib = C.CDLL(REF_SO)
    lib.ref_scene_mixtures.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double,
                                       C.c_ulonglong, C.c_double, C.c_double, C.c_int, _ip, _ip,
                                       _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _ip, _dp, _ip, _dp]
    lib.ref_last_error.restype = C.c_char_p
    n1, n2, npt, npx = (np.zeros(1, dtype=np.int32) for _ in range(4))
    mu, dir_ = np.zeros((cap, 3)), np.zeros((cap, 3))
    s2, p1, k2, p2 = (np.zeros(cap) for _ in range(4))
    tr, tt = np.zeros(3), np.zeros(3)
    pts, pxs = np.zeros((cap, 3)), np.zeros((cap, 2))
    rc = lib.ref_scene_mixtures(n_inliers, omega_3d, omega_2d, noise_px, seed, lambda_p, lambda_f,
                                cap, _i(n1), _i(n2), _d(mu), _d(s2), _d(p1), _d(dir_), _d(k2),
                                _d(p2), _d(tr), _d(tt), _i(npt), _d(pts), _i(npx), _d(pxs))
    if rc != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    a, b = int(n1[0]), int(n2[0])
    mix = Mixture([a], [b], [1.0], mu[:a], s2[:a], p1[:a], dir_[:b], k2[:b], p2[:b], zeta)
    return mix, {"r": tr, "t": tt, "points": pts[:int(npt[0])], "pixels": pxs[:int(npx[0])]}


def reference_torus_cover(major=3.5, minor=0.5, cap=1024):
    lib = C.CDLL(REF_SO)
    lib.ref_torus_cover.argtypes = [C.c_double, C.c_double, _dp, C.c_int]
    boxes = np.zeros((cap, 6))
    n = lib.ref_torus_cover(major, minor, _d(boxes), cap)
    return boxes[:n].copy()


def _cstrs(labels):
    if labels is None:
        return None, None
    enc = [str(x).encode() for x in labels]
    arr = (C.c_char_p * len(enc))(*enc)
    return arr, enc


def reference_dp_means(points, lam, seed=None, vmf=False, cap=100000):
    """dp_means / dp_vmf_means of the reference: (assignment, centers, iterations)."""
    lib = C.CDLL(REF_SO)
    fn = lib.ref_dp_vmf_means if vmf else lib.ref_dp_means
    fn.argtypes = [_dp, C.c_long, C.c_double, C.c_int, C.c_ulonglong, _ip, _dp, C.c_long,
                   C.POINTER(C.c_long), _ip]
    lib.ref_last_error.restype = C.c_char_p
    p = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    n = len(p)
    asg = np.zeros(n, dtype=np.int32)
    cen = np.zeros((min(cap, max(n, 1)), 3))
    nc, it = C.c_long(0), np.zeros(1, dtype=np.int32)
    rc = fn(_d(p), n, float(lam), int(seed is not None), int(seed or 0), _i(asg), _d(cen),
            len(cen), C.byref(nc), _i(it))
    if rc != 0:
        raise ValueError(lib.ref_last_error().decode())
    return asg, cen[:nc.value].copy(), int(it[0])


def reference_build_mixtures(points, bearings, lambda_p, lambda_f, point_labels=None,
                             bearing_labels=None, class_weights=None, cap_classes=256,
                             cap_comp=100000):
    """build_semantic_mixtures of the reference: (classes, warnings); classes
    are dicts {id, weight, mu, sigma2, phi1, dir, kappa2, phi2}."""
    lib = C.CDLL(REF_SO)
    lib.ref_build_mixtures.restype = C.c_int
    lib.ref_last_error.restype = C.c_char_p
    p = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    b = np.ascontiguousarray(bearings, dtype=np.float64).reshape(-1, 3)
    pl, _k1 = _cstrs(point_labels)
    bl, _k2 = _cstrs(bearing_labels)
    wl, _k3 = _cstrs(list(class_weights) if class_weights else None)
    w = np.array([class_weights[k] for k in class_weights], float) if class_weights else None
    n1 = np.zeros(cap_classes, dtype=np.int32)
    n2 = np.zeros(cap_classes, dtype=np.int32)
    cw = np.zeros(cap_classes)
    mu, dr = np.zeros((cap_comp, 3)), np.zeros((cap_comp, 3))
    s2, p1, k2, p2 = (np.zeros(cap_comp) for _ in range(4))
    ids = C.create_string_buffer(1 << 16)
    warns = C.create_string_buffer(1 << 16)
    nc = lib.ref_build_mixtures(_d(p), pl, C.c_long(len(p)), _d(b), bl, C.c_long(len(b)),
                                C.c_double(lambda_p), C.c_double(lambda_f), wl,
                                None if w is None else _d(w), C.c_long(0 if w is None else len(w)),
                                cap_classes, cap_comp, _i(n1), _i(n2), _d(cw), _d(mu), _d(s2),
                                _d(p1), _d(dr), _d(k2), _d(p2), ids, len(ids), warns, len(warns))
    if nc < 0:
        raise ValueError(lib.ref_last_error().decode())
    names = ids.value.decode().split("\n")[:nc]
    out, o1, o2 = [], 0, 0
    for c in range(nc):
        a, bb = int(n1[c]), int(n2[c])
        out.append({"id": names[c], "weight": float(cw[c]), "mu": mu[o1:o1 + a].copy(),
                    "sigma2": s2[o1:o1 + a].copy(), "phi1": p1[o1:o1 + a].copy(),
                    "dir": dr[o2:o2 + bb].copy(), "kappa2": k2[o2:o2 + bb].copy(),
                    "phi2": p2[o2:o2 + bb].copy()})
        o1, o2 = o1 + a, o2 + bb
    warnings = [x for x in warns.value.decode().split("\n") if x]
    return out, warnings
