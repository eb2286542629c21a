"""Rotation differences resolved below acos's ~2e-8 floor near the identity:
the angle of R from its skew part, atan2(|vee(R - R^T)| / 2, (tr R - 1) / 2)."""
import numpy as np


def angle_between(Ra, Rb) -> float:
    R = np.asarray(Ra) @ np.asarray(Rb).T
    v = np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])
    return float(np.arctan2(0.5 * np.linalg.norm(v), 0.5 * (np.trace(R) - 1.0)))
