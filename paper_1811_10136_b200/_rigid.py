"""Rigid FilterReg EM on the GPU: device pass wrapper + closed-form host math.

One EM iteration is ONE fused kernel sweep over the model points
(`fr_rigid_pass`): forward transform, lattice slice, moments epilogue and the
per-point residual statistics, reduced deterministically to a handful of
float64 sums.  Everything after that is 6-parameter host math:

point_to_point (mstep.py:102-210 with S = diag(1/sigma)) -- the pass returns
the weighted sufficient statistics of the centred current positions
y = x - c (c = R c_ref + t) and residuals r = x - target:

    sums[0]      S0 = sum w
    sums[1:4]    S1 = sum w y
    sums[4:10]   S2 = sum w y y^T      (xx, xy, xz, yy, yz, zz)
    sums[10:13]  R1 = sum w r
    sums[13:22]  RX = sum w r y^T      (row-major, RX[j, k] = sum w r_j y_k)
    sums[22:25]  Q  = sum w r_j^2      (per axis)
    [sums[25:27] sigma-update numerator / mass, when |y|^2 is splatted]

From these, H and g of the Gauss-Newton system, the objective at the current
pose and the objective change of ANY candidate pose x' = D x + delta follow in
closed form (all rows are affine in y), so step halving and extra GN
iterations need no further pass over the points.

point_to_plane (per-point normal rows are not low-rank in y):
    sums[0] mass, sums[1:22] upper-triangular H, sums[22:28] g,
    sums[28] sum w r^2, [sums[29:31] sigma update]
and halving candidates are evaluated by `fr_rigid_objective` over the
weight/target/normal planes the pass stored.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .estep import outlier_constant
from .geometry import skew
from .permutohedral import PermutohedralLattice

_E = [skew(e) for e in np.eye(3)]   # K_k = [e_k]x


def _sym3(v6) -> np.ndarray:
    xx, xy, xz, yy, yz, zz = v6
    return np.array([[xx, xy, xz], [xy, yy, yz], [xz, yz, zz]])


@dataclass
class RigidMoments:
    """Point-to-point sufficient statistics about a fixed centre c."""

    S0: float
    S1: np.ndarray
    S2: np.ndarray
    R1: np.ndarray
    RX: np.ndarray
    Q: np.ndarray

    @classmethod
    def from_sums(cls, s) -> "RigidMoments":
        s = np.asarray(s, dtype=float)
        return cls(float(s[0]), s[1:4].copy(), _sym3(s[4:10]), s[10:13].copy(),
                   s[13:22].reshape(3, 3).copy(), s[22:25].copy())

    def energy(self, s2) -> float:
        """E = 1/2 sum ||S (x - t)||^2 (mstep.py:132-138)."""
        return 0.5 * float(np.dot(s2, self.Q))

    def normal_equations(self, c, s2):
        """H = sum w J^T S^2 J, g = sum w J^T S^2 r with J = [-[x]x | I]
        (geometry.py:192-204, mstep.py:179-210), x = y + c."""
        c = np.asarray(c, dtype=float)
        X1 = self.S1 + c * self.S0
        X2 = self.S2 + np.outer(c, self.S1) + np.outer(self.S1, c) + self.S0 * np.outer(c, c)
        XR = self.RX + np.outer(self.R1, c)          # XR[:, k] = sum w r x_k
        Ssq = np.diag(s2)
        H = np.zeros((6, 6))
        tl = np.zeros((3, 3))
        for k in range(3):
            for l in range(3):
                tl += X2[k, l] * (_E[k].T @ Ssq @ _E[l])
        H[:3, :3] = tl
        H[:3, 3:] = skew(X1) @ Ssq
        H[3:, :3] = H[:3, 3:].T
        H[3:, 3:] = self.S0 * Ssq
        g = np.zeros(6)
        for k in range(3):
            g[:3] += _E[k] @ (Ssq @ XR[:, k])
        g[3:] = Ssq @ self.R1
        return H, g

    def _motion_terms(self, D, delta, c):
        A = D - np.eye(3)
        dt = A @ c + delta                            # y' = D y + dt
        su2 = np.array([A[j] @ self.S2 @ A[j] + 2.0 * dt[j] * (A[j] @ self.S1)
                        + dt[j] ** 2 * self.S0 for j in range(3)])
        sur = np.array([A[j] @ self.RX[j] + dt[j] * self.R1[j] for j in range(3)])
        return A, dt, su2, sur

    def delta_energy(self, D, delta, c, s2) -> float:
        """E(D x + delta) - E(x) with the same weights / targets."""
        _, _, su2, sur = self._motion_terms(D, delta, c)
        return 0.5 * float(np.dot(s2, su2 + 2.0 * sur))

    def moved(self, D, delta, c) -> "RigidMoments":
        """Statistics after x -> D x + delta, same centre c and targets."""
        A, dt, su2, sur = self._motion_terms(D, delta, c)
        DS1 = D @ self.S1
        S1n = DS1 + dt * self.S0
        S2n = D @ self.S2 @ D.T + np.outer(DS1, dt) + np.outer(dt, DS1) \
            + self.S0 * np.outer(dt, dt)
        AS1 = A @ self.S1
        R1n = self.R1 + AS1 + dt * self.S0
        U = A @ self.S2 @ D.T + np.outer(AS1, dt) + np.outer(dt, DS1) + self.S0 * np.outer(dt, dt)
        RXn = self.RX @ D.T + np.outer(self.R1, dt) + U
        Qn = self.Q + 2.0 * sur + su2
        return RigidMoments(self.S0, S1n, S2n, R1n, RXn, Qn)


def unpack_upper6(v21) -> np.ndarray:
    H = np.zeros((6, 6))
    o = 0
    for i in range(6):
        for j in range(i, 6):
            H[i, j] = H[j, i] = v21[o]
            o += 1
    return H


class RigidDevicePath:
    """HBM-resident state of one rigid registration: float32 SoA reference
    planes, the observation lattice, and the reduction buffers."""

    def __init__(self, reference, observation, gmm, residual_mode: str):
        import torch
        self.dev = _lib.device()
        self.lib = _lib.load()
        self.mode = _lib.FR_POINT_TO_PLANE if residual_mode == "point_to_plane" \
            else _lib.FR_POINT_TO_POINT
        self.gmm = gmm
        P = np.asarray(reference.positions, dtype=float)
        self.M = len(P)
        self.c_ref = P.mean(axis=0)
        self.ref = torch.from_numpy(np.ascontiguousarray(P.T, dtype=np.float32)).to(self.dev)
        Y = np.asarray(observation.positions, dtype=float)
        self.N = len(Y)
        self.obs = torch.from_numpy(np.ascontiguousarray(Y.T, dtype=np.float32)).to(self.dev)
        self.obs_n = None
        if self.mode == _lib.FR_POINT_TO_PLANE:
            if observation.normals is None:
                raise ValueError("observation cloud has no normals")
            self.obs_n = torch.from_numpy(
                np.ascontiguousarray(observation.normals.T, dtype=np.float32)).to(self.dev)
        self.with_sigma = bool(gmm.update_sigma)
        self.value_mode = (_lib.FR_VALUES_M2 if self.with_sigma else 0) | \
            (_lib.FR_VALUES_NORMALS if self.obs_n is not None else 0)
        self.m2_col = 4 if self.with_sigma else -1
        self.normal_col = (5 if self.with_sigma else 4) if self.obs_n is not None else -1
        self.width = self.lib.fr_rigid_pass_width(self.mode, int(self.with_sigma))
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.sums = torch.empty(max(self.width, 16), **f64)
        self.scratch = torch.empty(
            self.lib.fr_rigid_scratch_doubles(self.mode, int(self.with_sigma), self.M), **f64)
        self.host = torch.empty(max(self.width, 16), dtype=torch.float64, pin_memory=True)
        self.wtn = torch.empty((7, self.M), dtype=torch.float32, device=self.dev) \
            if self.mode == _lib.FR_POINT_TO_PLANE else None
        self.lattice = None
        self.sigma = None
        self.build(gmm.sigma)

    def build(self, sigma) -> None:
        """(Re)build the observation lattice at kernel width sigma."""
        s = np.atleast_1d(np.asarray(sigma, dtype=float))
        if s.size == 1:
            s = np.full(3, s[0])
        lat = PermutohedralLattice(3, s)
        lat.splat_points(self.obs, self.obs_n, self.value_mode)
        lat.blur()
        self.lattice, self.sigma = lat, s
        self.c_prime = outlier_constant(self.gmm.outlier_ratio, self.N, self.M, s)

    def run_pass(self, R, t) -> np.ndarray:
        """One fused E + assembly sweep at pose (R, t); returns the host sums."""
        R = np.asarray(R, dtype=float)
        p = _lib.RigidPassParams()
        p.R[:] = list(R.reshape(-1))
        p.c_ref[:] = list(self.c_ref)
        p.c_world[:] = list(R @ self.c_ref + np.asarray(t, dtype=float))
        p.sigma[:] = list(self.sigma)
        p.c_prime = self.c_prime
        p.mode = self.mode
        p.m2_col = self.m2_col
        p.normal_col = self.normal_col
        _lib.check(self.lib.fr_rigid_pass(self.lattice.handle, _lib.ptr(self.ref), self.M,
                                          ctypes.byref(p), _lib.ptr(self.sums),
                                          _lib.ptr(self.wtn), _lib.ptr(self.scratch),
                                          _lib.stream_handle()))
        self.host[:self.width].copy_(self.sums[:self.width])   # synchronising D2H
        return self.host[:self.width].numpy().copy()

    def centre(self, R, t) -> np.ndarray:
        return np.asarray(R, dtype=float) @ self.c_ref + np.asarray(t, dtype=float)

    def candidate_objectives(self, poses) -> np.ndarray:
        """0.5 * sum r^2 at each (R, t) under the stored point_to_plane spec."""
        k = len(poses)
        Rs = np.ascontiguousarray(np.stack([np.asarray(R, dtype=float).reshape(9)
                                            for R, _ in poses]))
        cs = np.ascontiguousarray(np.stack([self.centre(R, t) for R, t in poses]))
        cr, _k1 = _lib.dptr(self.c_ref)
        rp, _k2 = _lib.dptr(Rs)
        cp, _k3 = _lib.dptr(cs)
        _lib.check(self.lib.fr_rigid_objective(_lib.ptr(self.ref), _lib.ptr(self.wtn), self.M,
                                               cr, k, rp, cp, _lib.ptr(self.sums),
                                               _lib.ptr(self.scratch), _lib.stream_handle()))
        self.host[:16].copy_(self.sums[:16])
        return 0.5 * self.host[:k].numpy().copy()
