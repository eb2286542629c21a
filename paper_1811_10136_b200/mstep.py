"""Weighted Gauss-Newton over twist-parameterised kinematics (drop-in for
mstep.py, pkg/src/twistreg/mstep.py:1-459).

The per-point work (residual rows, J^T J / J^T r reductions, objectives) runs
in device kernels; the (6+DOF)^2 solves with the reference's damping
escalation stay float64 on the host (they are microseconds).  Inside
`register` the rigid M step never re-reads the points: the fused EM pass
returns sufficient statistics from which assembly, step halving and extra GN
iterations follow in closed form (see _rigid.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse
import scipy.sparse.linalg

from . import _lib
from .errors import SolverError
from .geometry import PointCloud, point_twist_jacobian
from .kinematics import RigidModel, forward_points

RESIDUAL_MODES = ("point_to_point", "point_to_plane")
_DENSE_SOLVE_MAX = 360
# block-sparse systems up to this size are factored densely on the GPU
# (cuSOLVER Cholesky through torch) instead of SuperLU on the host: the damped
# normal equations are symmetric positive definite, so the solution agrees to
# round-off and the escalation path is the same (factorization failure)
_GPU_DENSE_MAX = 8192


@dataclass(frozen=True)
class ResidualSpec:
    """Per-point correspondence residuals for one M step (mstep.py:39-84)."""

    weights: np.ndarray
    targets: np.ndarray
    sigma_inv: np.ndarray
    mode: str = "point_to_point"
    normals: np.ndarray | None = None
    normal_valid: np.ndarray | None = None

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=float).reshape(-1)
        t = np.asarray(self.targets, dtype=float)
        if t.shape != (len(w), 3):
            raise ValueError(f"targets must be ({len(w)}, 3), got {t.shape}")
        if np.any(w < 0) or np.any(w > 1) or not np.all(np.isfinite(w)):
            raise ValueError("weights must lie in [0, 1]")
        if not np.all(np.isfinite(t)):
            raise ValueError("non-finite targets")
        s = np.atleast_1d(np.asarray(self.sigma_inv, dtype=float))
        if s.size == 1:
            s = np.full(3, s[0])
        if s.shape != (3,) or np.any(s <= 0) or not np.all(np.isfinite(s)):
            raise ValueError("sigma_inv must be a positive scalar or 3-vector")
        if self.mode not in RESIDUAL_MODES:
            raise ValueError(f"unknown residual mode {self.mode!r}")
        object.__setattr__(self, "weights", w)
        object.__setattr__(self, "targets", t)
        object.__setattr__(self, "sigma_inv", s)
        if self.mode == "point_to_plane":
            if self.normals is None:
                raise ValueError("point-to-plane residuals need normals")
            n = np.asarray(self.normals, dtype=float)
            if n.shape != t.shape:
                raise ValueError("normals must match targets")
            valid = (np.ones(len(w), dtype=bool) if self.normal_valid is None
                     else np.asarray(self.normal_valid, dtype=bool).reshape(len(w)))
            lengths = np.linalg.norm(n[valid], axis=1)
            if len(lengths) and np.max(np.abs(lengths - 1.0)) > 1e-6:
                raise ValueError("normals must be unit length where valid")
            object.__setattr__(self, "normals", n)
            object.__setattr__(self, "normal_valid", valid)

    def __len__(self) -> int:
        return len(self.weights)


def residuals_from_moments(moments, sigma, mode: str = "point_to_point") -> ResidualSpec:
    """mstep.py:87-99"""
    s = np.atleast_1d(np.asarray(sigma, dtype=float))
    if s.size == 1:
        s = np.full(3, s[0])
    normals = valid = None
    if mode == "point_to_plane":
        if moments.normal is None:
            raise ValueError("moments were computed without the normal channel")
        normals, valid = moments.normal, moments.normal_valid
    return ResidualSpec(moments.weight, moments.target, 1.0 / s, mode, normals, valid)


@dataclass
class NormalEquations:
    """Dense or 6x6-block-sparse A and b (mstep.py:154-176).  A block system
    is a dict {(k, l): block} (k <= l) or, as the device assemblies produce
    it, `block_arrays` = (keys (m, 2) with k <= l, values (m, 6, 6)), repeated
    keys adding up."""

    n_params: int
    b: np.ndarray
    A: np.ndarray | None = None
    blocks: dict | None = None
    block_arrays: tuple | None = None

    @property
    def is_block(self) -> bool:
        return self.A is None and (self.blocks is not None or self.block_arrays is not None)

    def arrays(self):
        """(keys, values) of the block system."""
        if self.block_arrays is not None:
            return self.block_arrays
        keys = np.array(list(self.blocks.keys()), dtype=np.int64).reshape(-1, 2)
        vals = np.stack(list(self.blocks.values())) if len(keys) else np.zeros((0, 6, 6))
        return keys, vals

    def to_dense(self) -> np.ndarray:
        if self.A is not None:
            return self.A
        return _dense_blocks(self)

    def trace(self) -> float:
        if self.A is not None:
            return float(np.trace(self.A))
        keys, vals = self.arrays()
        d = keys[:, 0] == keys[:, 1]
        return float(np.trace(vals[d], axis1=1, axis2=2).sum())


def _device_rigid_sums(spec: ResidualSpec, x) -> np.ndarray:
    """fr_assemble_rigid over an explicit spec: [H upper 21 | g 6 | sum r^2]."""
    import torch
    from .permutohedral import _to_device
    lib = _lib.load()
    m = len(spec)
    dev = _lib.device()
    sums = torch.empty(28, dtype=torch.float64, device=dev)
    scratch = torch.empty(lib.fr_rigid_scratch_doubles(0, 0, m), dtype=torch.float64, device=dev)
    dX = _to_device(np.asarray(x, dtype=float))
    dW = _to_device(spec.weights)
    dT = _to_device(spec.targets)
    pl = spec.mode == "point_to_plane"
    dN = _to_device(spec.normals) if pl else None
    dV = _to_device(spec.normal_valid, np.uint8) if pl else None
    si, _keep = _lib.dptr(spec.sigma_inv)
    _lib.check(lib.fr_assemble_rigid(_lib.ptr(dX), _lib.ptr(dW), _lib.ptr(dT), m, si,
                                     int(pl), _lib.ptr(dN), _lib.ptr(dV), _lib.ptr(sums),
                                     _lib.ptr(scratch), _lib.stream_handle()))
    return sums.cpu().numpy()


def objective(spec: ResidualSpec, current_positions) -> float:
    """E = 1/2 sum ||r||^2 (mstep.py:132-138), on the device."""
    x = np.asarray(current_positions, dtype=float)
    if len(x) != len(spec):
        raise ValueError("residual count does not match point count")
    return 0.5 * float(_device_rigid_sums(spec, x)[27])


def assemble_rigid(spec: ResidualSpec, current_positions) -> NormalEquations:
    """mstep.py:205-210, reduction on the device."""
    from ._rigid import unpack_upper6
    x = np.asarray(current_positions, dtype=float)
    if len(x) != len(spec):
        raise ValueError("residual count does not match point count")
    s = _device_rigid_sums(spec, x)
    return NormalEquations(6, b=s[21:27].copy(), A=unpack_upper6(s[:21]))


def _dense_blocks(eq: NormalEquations) -> np.ndarray:
    """Dense A of a 6x6-block system (both triangles), one scatter."""
    P, nb = eq.n_params, eq.n_params // 6
    keys, vals = eq.arrays()
    F = np.zeros((nb, nb, 6, 6))
    np.add.at(F, (keys[:, 0], keys[:, 1]), vals)
    off = keys[:, 0] != keys[:, 1]
    np.add.at(F, (keys[off, 1], keys[off, 0]), np.transpose(vals[off], (0, 2, 1)))
    return F.transpose(0, 2, 1, 3).reshape(P, P)


def _gpu_block_cholesky_solve(eq: NormalEquations, lam: float) -> np.ndarray:
    """(A + lam I) x = b for a 6x6-block system: the blocks (not the dense
    matrix) go to the device, which scatters them into the dense A and factors
    it (cuSOLVER Cholesky through torch)."""
    import torch
    dev = _lib.device()
    P, nb = eq.n_params, eq.n_params // 6
    keys, vals = eq.arrays()
    k = torch.from_numpy(np.ascontiguousarray(keys)).to(dev)
    v = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).to(dev)
    F = torch.zeros((nb, nb, 6, 6), dtype=torch.float64, device=dev)
    F.index_put_((k[:, 0], k[:, 1]), v, accumulate=True)
    off = k[:, 0] != k[:, 1]
    F.index_put_((k[off, 1], k[off, 0]), v[off].transpose(1, 2), accumulate=True)
    A = F.permute(0, 2, 1, 3).reshape(P, P)
    A.diagonal().add_(lam)
    L, info = torch.linalg.cholesky_ex(A)
    if int(info.item()) != 0:
        raise scipy.linalg.LinAlgError("normal equations not positive definite")
    x = torch.cholesky_solve(torch.from_numpy(np.ascontiguousarray(eq.b)).to(dev)[:, None], L)
    sol = x[:, 0].cpu().numpy()
    if not np.all(np.isfinite(sol)):
        raise scipy.linalg.LinAlgError("factorization produced non-finite values")
    return sol


def _factor_solve(eq: NormalEquations, lam: float, method: str) -> np.ndarray:
    """mstep.py:317-345"""
    if method == "auto" and eq.is_block and _DENSE_SOLVE_MAX < eq.n_params <= _GPU_DENSE_MAX:
        return _gpu_block_cholesky_solve(eq, lam)
    sparse = method == "sparse" or (method == "auto" and eq.A is None
                                    and eq.n_params > _DENSE_SOLVE_MAX)
    if sparse and eq.is_block:
        keys, vals = eq.arrays()
        rr, cc = np.meshgrid(np.arange(6), np.arange(6), indexing="ij")
        off = keys[:, 0] != keys[:, 1]
        rows = np.concatenate([(6 * keys[:, 0, None, None] + rr).ravel(),
                               (6 * keys[off, 1, None, None] + rr).ravel(),
                               np.arange(eq.n_params)])
        cols = np.concatenate([(6 * keys[:, 1, None, None] + cc).ravel(),
                               (6 * keys[off, 0, None, None] + cc).ravel(),
                               np.arange(eq.n_params)])
        data = np.concatenate([vals.ravel(), np.transpose(vals[off], (0, 2, 1)).ravel(),
                               np.full(eq.n_params, lam)])
        A = scipy.sparse.csc_matrix((data, (rows, cols)), shape=(eq.n_params, eq.n_params))
        sol = scipy.sparse.linalg.splu(A).solve(eq.b)
        if not np.all(np.isfinite(sol)):
            raise scipy.linalg.LinAlgError("sparse factorization produced non-finite values")
        return sol
    A = eq.to_dense() + lam * np.eye(eq.n_params)
    return scipy.linalg.cho_solve(scipy.linalg.cho_factor(A), eq.b)


def gn_solve(eq: NormalEquations, damping: float | None = None, method: str = "auto",
             _stats: dict | None = None) -> np.ndarray:
    """(A + lam I) step = -b with tenfold escalation (mstep.py:348-369)."""
    if method not in ("auto", "dense", "sparse"):
        raise ValueError(f"unknown solve method {method!r}")
    if not np.any(eq.b):
        if _stats is not None:
            _stats.update(damping=0.0, attempts=0)
        return np.zeros(eq.n_params)
    tr = eq.trace()
    lam = damping if damping is not None else 1e-6 * tr / eq.n_params
    for attempt in range(6):
        try:
            sol = _factor_solve(eq, lam, method)
        except (scipy.linalg.LinAlgError, RuntimeError):
            lam = lam * 10.0 if lam > 0 else max(tr / eq.n_params, 1.0) * 1e-10
            continue
        if _stats is not None:
            _stats.update(damping=lam, attempts=attempt + 1)
        return -sol
    raise SolverError(f"normal equations not factorizable after damping escalation "
                      f"(final damping {lam:.3e})")


@dataclass(frozen=True)
class MStepOptions:
    """mstep.py:372-379"""

    max_gn_iters: int = 1
    damping: float | None = None
    max_halvings: int = 10
    step_tolerance: float = 0.0
    lambda_reg: float = 0.0
    solve_method: str = "auto"


@dataclass
class MStepDiagnostics:
    objectives: list = field(default_factory=list)
    step_norms: list = field(default_factory=list)
    halvings: list = field(default_factory=list)
    dampings: list = field(default_factory=list)


def _accepts(cand: float, value: float) -> bool:
    """Non-increase test of mstep.py:446."""
    return cand <= value * (1.0 + 1e-12) + 1e-300


def m_step(spec: ResidualSpec, reference: PointCloud, model, options: MStepOptions | None = None):
    """Damped GN with step halving over an explicit spec (mstep.py:421-459).

    Rigid models run every point reduction on the device; articulated and
    node-graph models are dispatched by their own modules.
    """
    opts = options if options is not None else MStepOptions()
    if not isinstance(model, RigidModel):
        from . import kinematics
        return kinematics.m_step_model(spec, reference, model, opts)
    current = model
    value = objective(spec, forward_points(reference, current).positions)
    diag = MStepDiagnostics(objectives=[value])
    for _ in range(opts.max_gn_iters):
        x = forward_points(reference, current).positions
        eq = assemble_rigid(spec, x)
        if not np.any(eq.b):
            break
        stats: dict = {}
        step = gn_solve(eq, opts.damping, opts.solve_method, _stats=stats)
        diag.dampings.append(stats.get("damping", 0.0))
        scale = 1.0
        accepted = None
        for halving in range(opts.max_halvings + 1):
            cand = current.updated(scale * step)
            cv = objective(spec, forward_points(reference, cand).positions)
            if _accepts(cv, value):
                accepted = (cand, cv, halving)
                break
            scale *= 0.5
        if accepted is None:
            break
        current, value, halvings = accepted
        diag.objectives.append(value)
        diag.halvings.append(halvings)
        sn = float(np.linalg.norm(scale * step))
        diag.step_norms.append(sn)
        if sn <= opts.step_tolerance:
            break
    return current, diag


def _device_point_rows(spec: ResidualSpec, x):
    """fr_point_rows: per-point [E^T E | E^T r] (m x 28) on the device."""
    import torch
    from .permutohedral import _to_device
    lib = _lib.load()
    m = len(spec)
    dev = _lib.device()
    ete = torch.empty((m, 28), dtype=torch.float64, device=dev)
    pl = spec.mode == "point_to_plane"
    dX, dW, dT = _to_device(np.asarray(x, dtype=float)), _to_device(spec.weights), \
        _to_device(spec.targets)
    dN = _to_device(spec.normals) if pl else None
    dV = _to_device(spec.normal_valid, np.uint8) if pl else None
    si, _keep = _lib.dptr(spec.sigma_inv)
    _lib.check(lib.fr_point_rows(_lib.ptr(dX), _lib.ptr(dW), _lib.ptr(dT), _lib.ptr(dN),
                                 _lib.ptr(dV), m, int(pl), si, _lib.ptr(ete),
                                 _lib.stream_handle()))
    return ete


def _device_blocks(ete, weights, indices, n_nodes, pair_codes=None):
    """fr_graph_blocks over (point, slot) lists built from a skinning-like
    (indices, weights) table: diag (n x 27) and pair blocks (p x 21)."""
    import torch
    from ._nodegraph import gather_lists
    lib = _lib.load()
    dev = ete.device
    K = indices.shape[1]
    L = gather_lists(indices, weights, n_nodes)
    t = {k: torch.from_numpy(v).to(dev) for k, v in L.items() if isinstance(v, np.ndarray)}
    swt = torch.from_numpy(np.ascontiguousarray(np.where(indices >= 0, weights, 0.0))).to(dev)
    diag = torch.zeros((n_nodes, 27), dtype=torch.float64, device=dev)
    off = torch.zeros((max(L["n_pairs"], 1), 21), dtype=torch.float64, device=dev)
    _lib.check(lib.fr_graph_blocks(_lib.ptr(ete), _lib.ptr(swt), K, _lib.ptr(t["dptr"]),
                                   _lib.ptr(t["dent"]), n_nodes, _lib.ptr(t["pptr"]),
                                   _lib.ptr(t["pent"]), L["n_pairs"], _lib.ptr(diag),
                                   _lib.ptr(off), _lib.stream_handle()))
    return diag.cpu().numpy(), off[:L["n_pairs"]].cpu().numpy(), L


def assemble_articulated(spec: ResidualSpec, current_positions, tree) -> NormalEquations:
    """Two-phase assembly (mstep.py:213-229): per-body 6x6 blocks reduced on the
    device (points grouped by body), projected through the spatial velocity
    Jacobians on the host."""
    from ._rigid import unpack_upper6
    x = np.asarray(current_positions, dtype=float)
    if len(x) != len(spec):
        raise ValueError("residual count does not match point count")
    if tree.point_bodies is None:
        raise ValueError("articulated assembly needs the tree's point binding")
    if len(tree.point_bodies) != len(spec):
        raise ValueError("point binding does not match the residual count")
    nb = tree.n_bodies
    ete = _device_point_rows(spec, x)
    idx = np.asarray(tree.point_bodies, dtype=np.int64)[:, None]
    diag, _, _ = _device_blocks(ete, np.ones(idx.shape), idx, nb)
    H = np.stack([unpack_upper6(diag[b, :21]) for b in range(nb)])
    g = diag[:, 21:27]
    live = np.flatnonzero(H.any(axis=(1, 2)) | g.any(axis=1))
    S = tree.spatial_velocity_jacobians()[live]
    A = np.einsum("bip,bij,bjq->pq", S, H[live], S, optimize=True)
    b = np.einsum("bip,bi->p", S, g[live])
    return NormalEquations(tree.n_params, b=b, A=A)


def assemble_nodegraph(spec: ResidualSpec, current_positions, graph,
                       lambda_reg: float = 0.0) -> NormalEquations:
    """Block-sparse assembly (mstep.py:232-314): data blocks on the device,
    ARAP regulariser on the host."""
    from ._nodegraph import normal_equations_from
    x = np.asarray(current_positions, dtype=float)
    if len(x) != len(spec):
        raise ValueError("residual count does not match point count")
    if len(graph.skinning.indices) != len(spec):
        raise ValueError("skinning does not match the residual count")
    if lambda_reg < 0:
        raise ValueError("lambda_reg must be nonnegative")
    ete = _device_point_rows(spec, x)
    diag, off, L = _device_blocks(ete, graph.skinning.weights, graph.skinning.indices,
                                  graph.n_nodes)
    return normal_equations_from(graph, diag, off, L["pair_lo"], L["pair_hi"], lambda_reg)


def _assemble(spec, x, model, lambda_reg) -> NormalEquations:
    from .kinematics import ArticulatedTree, NodeGraph
    if isinstance(model, RigidModel):
        return assemble_rigid(spec, x)
    if isinstance(model, ArticulatedTree):
        return assemble_articulated(spec, x, model)
    if isinstance(model, NodeGraph):
        return assemble_nodegraph(spec, x, model, lambda_reg)
    raise TypeError(f"unsupported kinematic model {type(model).__name__}")


def _total_objective(spec, reference, model, lambda_reg) -> float:
    """mstep.py:404-408"""
    from ._nodegraph import regularizer_objective
    from .kinematics import NodeGraph
    value = objective(spec, forward_points(reference, model).positions)
    if isinstance(model, NodeGraph):
        value += regularizer_objective(model, lambda_reg)
    return value


def m_step_general(spec, reference, model, opts):
    """m_step for articulated trees and node graphs over an explicit spec."""
    current = model
    value = _total_objective(spec, reference, current, opts.lambda_reg)
    diag = MStepDiagnostics(objectives=[value])
    for _ in range(opts.max_gn_iters):
        x = forward_points(reference, current).positions
        eq = _assemble(spec, x, current, opts.lambda_reg)
        if not np.any(eq.b):
            break
        stats: dict = {}
        step = gn_solve(eq, opts.damping, opts.solve_method, _stats=stats)
        diag.dampings.append(stats.get("damping", 0.0))
        scale = 1.0
        accepted = None
        for halving in range(opts.max_halvings + 1):
            cand = current.updated(scale * step)
            cv = _total_objective(spec, reference, cand, opts.lambda_reg)
            if _accepts(cv, value):
                accepted = (cand, cv, halving)
                break
            scale *= 0.5
        if accepted is None:
            break
        current, value, halvings = accepted
        diag.objectives.append(value)
        diag.halvings.append(halvings)
        sn = float(np.linalg.norm(scale * step))
        diag.step_norms.append(sn)
        if sn <= opts.step_tolerance:
            break
    return current, diag


__all__ = ["assemble_articulated", "assemble_nodegraph", "RESIDUAL_MODES", "ResidualSpec", "residuals_from_moments", "NormalEquations",
           "objective", "assemble_rigid", "gn_solve", "MStepOptions", "MStepDiagnostics",
           "m_step", "point_twist_jacobian"]
