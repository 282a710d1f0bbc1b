"""Host-side SE(3) helpers (numpy, FP64) mirroring the reference's
se3.hpp / bench.hpp utilities that callers use around solve()."""
from __future__ import annotations

import math

import numpy as np


def rotation_matrix(r) -> np.ndarray:
    """Rodrigues rotation for an axis-angle vector (se3.cpp:21-31)."""
    r = np.asarray(r, dtype=np.float64)
    th2 = float(r @ r)
    K = np.array([[0.0, -r[2], r[1]], [r[2], 0.0, -r[0]], [-r[1], r[0], 0.0]])
    if th2 < 1e-16:
        return np.eye(3) + K + 0.5 * (K @ K)
    th = math.sqrt(th2)
    return np.eye(3) + (math.sin(th) / th) * K + ((1.0 - math.cos(th)) / th2) * (K @ K)


def angular_distance(r1, r2) -> float:
    """Geodesic angle between two rotations (se3.cpp:43-48)."""
    R = rotation_matrix(r1).T @ rotation_matrix(r2)
    s = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    return math.atan2(0.5 * np.linalg.norm(s), 0.5 * (np.trace(R) - 1.0))


def pose_errors(est_r, est_t, true_r, true_t, centroid=(0.0, 0.0, 0.0)):
    """Rotation error, translation error and relative translation error
    (bench.cpp:144-157)."""
    rel = rotation_matrix(est_r) @ rotation_matrix(true_r).T
    rot = math.acos(max(-1.0, min(1.0, 0.5 * (np.trace(rel) - 1.0))))
    te = float(np.linalg.norm(np.asarray(est_t) - np.asarray(true_t)))
    dist = float(np.linalg.norm(np.asarray(true_t) - np.asarray(centroid)))
    return rot, te, (te / dist if dist > 0 else math.inf)


def is_success(rot_err: float, rel_trans_err: float) -> bool:
    """Strict thresholds of bench.cpp:159-161."""
    return rot_err < 0.1 and rel_trans_err < 0.05
