"""Articulated FilterReg EM on the GPU (mstep.py:213-229, kinematics.py:76-229).

Model points are sorted by body once; one device pass per EM iteration
(`fr_body_pass`) returns per-body statistics -- the rigid pass layout
(_rigid.py) about each body's own centre -- so the point loop never sees the
joint count (Algorithm 1 of PAPER.md:289-308).  The host then forms each body's
6x6 H_b, g_b, projects A = sum S_b^T H_b S_b, b = sum S_b^T g_b through the
spatial velocity Jacobians, solves, and (point_to_point) evaluates every
halving candidate in closed form from the per-body statistics.
point_to_plane candidates use `fr_body_objective`.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._rigid import FAST_QUERY, RigidDevicePath, RigidMoments, unpack_upper6


class BodyPose(ctypes.Structure):
    _fields_ = [("R", ctypes.c_double * 9), ("c_ref", ctypes.c_double * 3),
                ("c_world", ctypes.c_double * 3)]


class ArticulatedDevicePath(RigidDevicePath):
    """Body-sorted float32 model planes + chunk table + the observation lattice."""

    CHUNK = 4096

    def __init__(self, reference, observation, gmm, residual_mode, tree, process_group=None):
        import torch
        from .geometry import PointCloud
        if tree.point_bodies is None:
            raise ValueError("articulated model has no point binding")
        labels = np.asarray(tree.point_bodies, dtype=np.int64)
        if len(labels) != len(reference):
            raise ValueError("point binding does not match the reference cloud")
        order = np.argsort(labels, kind="stable")
        P = np.asarray(reference.positions, dtype=float)[order]
        super().__init__(PointCloud(P), observation, gmm, residual_mode, process_group,
                         sort=False)
        nb = tree.n_bodies
        self.nb = nb
        lab = labels[order]
        counts = np.bincount(lab, minlength=nb)
        starts = np.concatenate([[0], np.cumsum(counts)])
        # per-body centres in the body frame (conditioning of the statistics)
        P32 = P.astype(np.float32).astype(float)
        self.c_body = np.zeros((nb, 3))
        chunk_body, chunk_beg, body_chunks = [], [], [0]
        for b in range(nb):
            s, e = int(starts[b]), int(starts[b + 1])
            if e > s:
                self.c_body[b] = P32[s:e].mean(axis=0)
            for a in range(s, e, self.CHUNK):
                chunk_body.append(b)
                chunk_beg.append(a)
            body_chunks.append(len(chunk_body))
        chunk_beg.append(int(starts[-1]))
        if not chunk_body:
            chunk_body, chunk_beg, body_chunks = [0], [0, 0], [0] + [1] * nb
        self.n_chunks = len(chunk_body)
        dev = self.dev
        self.chunk_body = torch.tensor(chunk_body, dtype=torch.int32, device=dev)
        self.chunk_beg = torch.tensor(chunk_beg, dtype=torch.int64, device=dev)
        self.body_chunks = torch.tensor(body_chunks, dtype=torch.int32, device=dev)
        f64 = dict(dtype=torch.float64, device=dev)
        w = self.width
        self.bsums = torch.empty((nb, w), **f64)
        self.bscratch = torch.empty(self.n_chunks * max(w, 16), **f64)
        self.params = torch.empty(self.lib.fr_body_params_doubles(max(nb * 16, nb)), **f64)
        self.bhost = torch.empty((nb, w), dtype=torch.float64, pin_memory=True)

    def _poses(self, tree, n_cand=1, trees=None):
        trees = trees if trees is not None else [tree]
        arr = (BodyPose * (len(trees) * self.nb))()
        for c, tr in enumerate(trees):
            for b in range(self.nb):
                T = tr.body_pose(b)
                p = arr[c * self.nb + b]
                p.R[:] = list(T.rotation.reshape(-1))
                p.c_ref[:] = list(self.c_body[b])
                p.c_world[:] = list(T.rotation @ self.c_body[b] + T.translation)
        return arr

    def centres(self, tree) -> np.ndarray:
        return np.stack([tree.body_pose(b).rotation @ self.c_body[b]
                         + tree.body_pose(b).translation for b in range(self.nb)])

    def run_body_pass(self, tree) -> np.ndarray:
        poses = self._poses(tree)
        flags = _lib.FR_PASS_FAST if FAST_QUERY else 0
        _lib.check(self.lib.fr_body_pass(
            self.lattice.handle, _lib.ptr(self.ref), self.M, poses, self.nb,
            _lib.ptr(self.chunk_body), _lib.ptr(self.chunk_beg), self.n_chunks,
            _lib.ptr(self.body_chunks), self.mode, self.c_prime, flags, _lib.ptr(self.params),
            _lib.ptr(self.bsums), _lib.ptr(self.wtn), _lib.ptr(self.bscratch),
            _lib.stream_handle()))
        self.reduce_device(self.bsums)
        self.bhost.copy_(self.bsums)
        return self.bhost.numpy().copy()

    def candidate_objectives_trees(self, trees) -> np.ndarray:
        out = []
        for a in range(0, len(trees), 16):
            chunk = trees[a:a + 16]
            poses = self._poses(None, trees=chunk)
            _lib.check(self.lib.fr_body_objective(
                _lib.ptr(self.ref), _lib.ptr(self.wtn), self.M, poses, self.nb, len(chunk),
                _lib.ptr(self.chunk_body), _lib.ptr(self.chunk_beg), self.n_chunks,
                _lib.ptr(self.params), _lib.ptr(self.sums), _lib.ptr(self.bscratch),
                _lib.stream_handle()))
            self.reduce_device(self.sums[:16])
            self.host[:16].copy_(self.sums[:16])
            out += list(0.5 * self.host[:len(chunk)].numpy())
        return np.asarray(out)


def articulated_m_step(path: ArticulatedDevicePath, sums, tree, s2, opts):
    """One M step of an articulated tree from per-body pass statistics
    (mstep.py:421-459 with assemble_articulated, mstep.py:213-229)."""
    from .mstep import MStepDiagnostics, NormalEquations, _accepts, gn_solve
    diag = MStepDiagnostics()
    p2p = path.mode == _lib.FR_POINT_TO_POINT
    nb = path.nb
    current = tree
    if p2p:
        moms = [RigidMoments.from_sums(sums[b]) for b in range(nb)]
        cents = path.centres(tree)
        value = float(sum(m.energy(s2) for m in moms))
    else:
        value = 0.5 * float(sums[:, 28].sum())
        Hb = np.stack([unpack_upper6(sums[b, 1:22]) for b in range(nb)])
        gb = np.asarray(sums[:, 22:28], dtype=float)
        if opts.max_gn_iters > 1:
            raise NotImplementedError("point_to_plane with max_gn_iters > 1 is not in this build")
    diag.objectives.append(value)

    def system(tr):
        S = tr.spatial_velocity_jacobians()
        if p2p:
            HG = [m.normal_equations(c, s2) for m, c in zip(moms, cents)]
            H = np.stack([h for h, _ in HG])
            g = np.stack([gg for _, gg in HG])
        else:
            H, g = Hb, gb
        live = np.flatnonzero(H.any(axis=(1, 2)) | g.any(axis=1))
        A = np.einsum("bip,bij,bjq->pq", S[live], H[live], S[live], optimize=True)
        b = np.einsum("bip,bi->p", S[live], g[live])
        return NormalEquations(tr.n_params, b=b, A=A)

    eq = system(current)
    for _ in range(opts.max_gn_iters):
        if not np.any(eq.b):
            break
        stats: dict = {}
        step = gn_solve(eq, opts.damping, opts.solve_method, _stats=stats)
        diag.dampings.append(stats.get("damping", 0.0))
        cands, scale = [], 1.0
        for _h in range(opts.max_halvings + 1):
            cands.append((current.updated(scale * step), scale))
            scale *= 0.5
        accepted = None
        if p2p:
            for h, (cand, sc) in enumerate(cands):
                dE = 0.0
                motions = []
                for b in range(nb):
                    Tb, Tc = current.body_pose(b), cand.body_pose(b)
                    D = Tc.rotation @ Tb.rotation.T
                    delta = Tc.translation - D @ Tb.translation
                    motions.append((D, delta))
                    dE += moms[b].delta_energy(D, delta, cents[b], s2)
                cv = value + dE
                if _accepts(cv, value):
                    accepted = (cand, cv, h, sc, motions)
                    break
        else:
            vals = list(path.candidate_objectives_trees([cands[0][0]]))
            if not _accepts(vals[0], value) and len(cands) > 1:
                vals += list(path.candidate_objectives_trees([c for c, _ in cands[1:]]))
            for h, cv in enumerate(vals):
                if _accepts(cv, value):
                    accepted = (cands[h][0], cv, h, cands[h][1], None)
                    break
        if accepted is None:
            break
        cand, value, h, sc, motions = accepted
        diag.objectives.append(value)
        diag.halvings.append(h)
        sn = float(np.linalg.norm(sc * step))
        diag.step_norms.append(sn)
        current = cand
        if sn <= opts.step_tolerance:
            break
        if p2p:
            moms = [m.moved(D, delta, c) for m, (D, delta), c in zip(moms, motions, cents)]
            eq = system(current)
    return current, diag
