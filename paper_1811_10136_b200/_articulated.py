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
from ._rigid import FAST_QUERY, RigidDevicePath, unpack_upper6


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
        # per-body centres in the body frame (conditioning of the statistics);
        # under a process group every rank must take its statistics about the
        # same centres, so the coordinate sums and counts are all-reduced
        P32 = P.astype(np.float32).astype(float)
        sums = np.zeros((nb, 4))
        for b in range(nb):
            s, e = int(starts[b]), int(starts[b + 1])
            sums[b, :3] = P32[s:e].sum(axis=0)
            sums[b, 3] = e - s
        sums = self._allreduce(sums.ravel(), "sum").reshape(nb, 4)
        self.c_body = np.zeros((nb, 3))
        has = sums[:, 3] > 0
        self.c_body[has] = sums[has, :3] / sums[has, 3:4]      # = mean (np.add.reduce / n)
        chunk_body, chunk_beg, body_chunks = [], [], [0]
        for b in range(nb):
            s, e = int(starts[b]), int(starts[b + 1])
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
        """BodyPose records (R, c_ref, c_world) of every body of every tree,
        filled through a float64 view of the ctypes array."""
        trees = trees if trees is not None else [tree]
        arr = (BodyPose * (len(trees) * self.nb))()
        view = np.ctypeslib.as_array(ctypes.cast(arr, ctypes.POINTER(ctypes.c_double)),
                                     shape=(len(trees), self.nb, 15))
        cb = np.asarray(self.c_body, dtype=float)
        for c, tr in enumerate(trees):
            R, t = tr.world_arrays()
            view[c, :, :9] = R.reshape(self.nb, 9)
            view[c, :, 9:12] = cb
            view[c, :, 12:15] = np.einsum("bij,bj->bi", R, cb) + t
        return arr

    def centres(self, tree) -> np.ndarray:
        R, t = tree.world_arrays()
        return np.einsum("bij,bj->bi", R, np.asarray(self.c_body, dtype=float)) + t

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


class BodyMoments:
    """RigidMoments (_rigid.py) of all nb bodies at once: the same closed forms
    (normal equations, energy change and moved statistics of x' = D x + delta)
    as batched array expressions, one per M-step quantity instead of one per
    body."""

    _E = np.stack([np.array([[0.0, 0.0, 0.0], [0.0, 0.0, -1.0], [0.0, 1.0, 0.0]]),
                   np.array([[0.0, 0.0, 1.0], [0.0, 0.0, 0.0], [-1.0, 0.0, 0.0]]),
                   np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 0.0]])])

    def __init__(self, S0, S1, S2, R1, RX, Q):
        self.S0, self.S1, self.S2, self.R1, self.RX, self.Q = S0, S1, S2, R1, RX, Q

    @classmethod
    def from_sums(cls, sums) -> "BodyMoments":
        s = np.asarray(sums, dtype=float)
        S2 = np.empty((len(s), 3, 3))
        iu = [(0, 0, 4), (0, 1, 5), (0, 2, 6), (1, 1, 7), (1, 2, 8), (2, 2, 9)]
        for i, j, c in iu:
            S2[:, i, j] = S2[:, j, i] = s[:, c]
        return cls(s[:, 0].copy(), s[:, 1:4].copy(), S2, s[:, 10:13].copy(),
                   s[:, 13:22].reshape(-1, 3, 3).copy(), s[:, 22:25].copy())

    def energy(self, s2) -> float:
        return float(0.5 * np.sum(self.Q @ s2))

    def normal_equations(self, c, s2):
        """(nb, 6, 6) H and (nb, 6) g about centres c (nb, 3)."""
        E = self._E
        S0 = self.S0[:, None]
        X1 = self.S1 + c * S0
        X2 = (self.S2 + c[:, :, None] * self.S1[:, None, :] + self.S1[:, :, None] * c[:, None, :]
              + S0[:, :, None] * c[:, :, None] * c[:, None, :])
        XR = self.RX + self.R1[:, :, None] * c[:, None, :]
        Ssq = np.diag(s2)
        T = np.einsum("kji,jm,lmn->klin", E, Ssq, E)          # E_k^T Ssq E_l
        nb = len(self.S0)
        H = np.zeros((nb, 6, 6))
        H[:, :3, :3] = np.einsum("bkl,klin->bin", X2, T)
        K1 = np.zeros((nb, 3, 3))
        K1[:, 0, 1], K1[:, 0, 2] = -X1[:, 2], X1[:, 1]
        K1[:, 1, 0], K1[:, 1, 2] = X1[:, 2], -X1[:, 0]
        K1[:, 2, 0], K1[:, 2, 1] = -X1[:, 1], X1[:, 0]
        H[:, :3, 3:] = K1 @ Ssq
        H[:, 3:, :3] = np.transpose(H[:, :3, 3:], (0, 2, 1))
        H[:, 3:, 3:] = self.S0[:, None, None] * Ssq
        g = np.zeros((nb, 6))
        g[:, :3] = np.einsum("kij,bjk->bi", E, s2[None, :, None] * XR)
        g[:, 3:] = self.R1 * s2
        return H, g

    def _motion(self, D, delta, c):
        A = D - np.eye(3)
        dt = np.einsum("bij,bj->bi", A, c) + delta
        su2 = (np.einsum("bji,bik,bjk->bj", A, self.S2, A)
               + 2.0 * dt * np.einsum("bji,bi->bj", A, self.S1) + dt ** 2 * self.S0[:, None])
        sur = np.einsum("bji,bji->bj", A, self.RX) + dt * self.R1
        return A, dt, su2, sur

    def delta_energy(self, D, delta, c, s2) -> float:
        _, _, su2, sur = self._motion(D, delta, c)
        return float(0.5 * np.sum((su2 + 2.0 * sur) @ s2))

    def moved(self, D, delta, c) -> "BodyMoments":
        A, dt, su2, sur = self._motion(D, delta, c)
        S0 = self.S0[:, None]
        DS1 = np.einsum("bij,bj->bi", D, self.S1)
        S1n = DS1 + dt * S0
        outer = np.einsum
        S2n = (D @ self.S2 @ np.transpose(D, (0, 2, 1)) + outer("bi,bj->bij", DS1, dt)
               + outer("bi,bj->bij", dt, DS1) + S0[:, :, None] * outer("bi,bj->bij", dt, dt))
        AS1 = np.einsum("bij,bj->bi", A, self.S1)
        R1n = self.R1 + AS1 + dt * S0
        U = (A @ self.S2 @ np.transpose(D, (0, 2, 1)) + outer("bi,bj->bij", AS1, dt)
             + outer("bi,bj->bij", dt, DS1) + S0[:, :, None] * outer("bi,bj->bij", dt, dt))
        RXn = self.RX @ np.transpose(D, (0, 2, 1)) + outer("bi,bj->bij", self.R1, dt) + U
        Qn = self.Q + 2.0 * sur + su2
        return BodyMoments(self.S0, S1n, S2n, R1n, RXn, Qn)


def _body_motion(cur, cand):
    """Per-body (D, delta) taking the current body poses to the candidate's."""
    Rb, tb = cur.world_arrays()
    Rc, tc = cand.world_arrays()
    D = Rc @ np.transpose(Rb, (0, 2, 1))
    return D, tc - np.einsum("bij,bj->bi", D, tb)


class ArtTreeDesc(ctypes.Structure):
    """fr_art_tree_desc (include/filterreg_b200.h)."""
    _fields_ = [("n_bodies", ctypes.c_int), ("n_params", ctypes.c_int),
                ("floating", ctypes.c_int), ("parent", ctypes.c_void_p),
                ("kind", ctypes.c_void_p), ("slot", ctypes.c_void_p),
                ("axis", ctypes.c_void_p), ("frame_R", ctypes.c_void_p),
                ("frame_t", ctypes.c_void_p), ("c_body", ctypes.c_void_p)]


MAX_DEVICE_BODIES, MAX_DEVICE_PARAMS = 32, 40


def device_loop_fits(tree) -> bool:
    return tree.n_bodies <= MAX_DEVICE_BODIES and tree.n_params <= MAX_DEVICE_PARAMS


class DeviceArtEM:
    """The device-resident articulated point-to-point EM loop (fr_art_em_*):
    per iteration the body pass, per-body sums and a one-CTA M step (forward
    kinematics, projection, damped Cholesky, closed-form halving) replayed
    from a CUDA graph; the host only reads the termination flag."""

    KINDS = {"fixed": 0, "revolute": 1, "prismatic": 2}

    def __init__(self, path: ArticulatedDevicePath, tree, config):
        from . import _rigid
        self.path, self.lib, self.tree = path, path.lib, tree
        self.max_iters = int(config.max_em_iters)
        tp = tree._topo
        nb = tree.n_bodies
        slot = np.full(nb, -1, dtype=np.int32)
        for s_, i in enumerate(tp.movable):
            slot[i] = s_
        self._arrays = dict(
            parent=np.asarray(tp.parent, dtype=np.int32),
            kind=np.asarray([self.KINDS[b.joint.kind] for b in tp.bodies], dtype=np.int32),
            slot=slot, axis=np.ascontiguousarray(tp.axis, dtype=float),
            frame_R=np.ascontiguousarray(tp.FR.reshape(nb, 9), dtype=float),
            frame_t=np.ascontiguousarray(tp.Ft, dtype=float),
            c_body=np.ascontiguousarray(path.c_body, dtype=float))
        a = self._arrays
        desc = ArtTreeDesc(nb, tree.n_params, int(tree.floating),
                           *[a[k].ctypes.data for k in ("parent", "kind", "slot", "axis",
                                                         "frame_R", "frame_t", "c_body")])
        c = _lib.RigidEmConfig()
        c.sigma_inv[:] = list(1.0 / np.asarray(path.sigma, dtype=float))
        c.c_prime = path.c_prime
        c.diameter = path.diameter
        c.twist_tolerance = float(config.twist_tolerance)
        ms = config.mstep
        c.damping = -1.0 if ms.damping is None else float(ms.damping)
        c.step_tolerance = float(ms.step_tolerance)
        c.degenerate_mass = 1e-9 * path.M_total
        c.max_em_iters = self.max_iters
        c.max_gn_iters = int(ms.max_gn_iters)
        c.max_halvings = int(ms.max_halvings)
        c.fast = _lib.FR_PASS_FAST if FAST_QUERY else 0
        q0 = np.ascontiguousarray(tree.joint_values, dtype=float)
        bR = np.ascontiguousarray(tree.base_pose.rotation, dtype=float)
        bt = np.ascontiguousarray(tree.base_pose.translation, dtype=float)
        WR, Wt = tree.world_arrays()
        WR = np.ascontiguousarray(WR, dtype=float)
        Wt = np.ascontiguousarray(Wt, dtype=float)
        dp = lambda v: v.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        h = ctypes.c_void_p()
        _lib.check(self.lib.fr_art_em_create(
            path.lattice.handle, _lib.ptr(path.ref), path.M, ctypes.byref(desc),
            dp(q0) if len(q0) else None, dp(bR), dp(bt), dp(WR), dp(Wt),
            _lib.ptr(path.chunk_body), _lib.ptr(path.chunk_beg), path.n_chunks,
            _lib.ptr(path.body_chunks), ctypes.byref(c), _lib.stream_handle(), ctypes.byref(h)))
        self.h = h
        del _rigid

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.fr_art_em_destroy(h)
            except Exception:
                pass
            self.h = None

    def run(self) -> None:
        _lib.check(self.lib.fr_art_em_run(self.h, _lib.stream_handle()))

    def result(self):
        from .geometry import RigidTransform
        n = self.max_iters
        q = np.zeros(40)
        bR, bt = np.zeros(9), np.zeros(3)
        obj, tn, ms = np.zeros(n), np.zeros(n), np.zeros(n)
        it, term = ctypes.c_int(), ctypes.c_int()
        dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        _lib.check(self.lib.fr_art_em_result(self.h, dp(q), dp(bR), dp(bt), dp(obj), dp(tn),
                                             dp(ms), ctypes.byref(it), ctypes.byref(term),
                                             _lib.stream_handle()))
        k = min(int(it.value), n)
        nq = len(self.tree.joint_values)
        tree = self.tree.with_joint_values(q[:nq].copy(),
                                           base_pose=RigidTransform(bR.reshape(3, 3), bt.copy()))
        return tree, list(obj[:k]), list(tn[:k]), list(ms[:k]), int(it.value), \
            _lib.FR_TERM[int(term.value)]


def articulated_m_step(path: ArticulatedDevicePath, sums, tree, s2, opts):
    """One M step of an articulated tree from per-body pass statistics
    (mstep.py:421-459 with assemble_articulated, mstep.py:213-229)."""
    from .mstep import MStepDiagnostics, NormalEquations, _accepts, gn_solve
    diag = MStepDiagnostics()
    p2p = path.mode == _lib.FR_POINT_TO_POINT
    nb = path.nb
    current = tree
    if p2p:
        moms = BodyMoments.from_sums(sums[:nb])
        cents = np.asarray(path.centres(tree), dtype=float)
        value = moms.energy(s2)
    else:
        value = 0.5 * float(sums[:, 28].sum())
        Hb = np.stack([unpack_upper6(sums[b, 1:22]) for b in range(nb)])
        gb = np.asarray(sums[:, 22:28], dtype=float)
        if opts.max_gn_iters > 1:
            raise ValueError("point_to_plane with max_gn_iters > 1 and a process_group: the "
                             "explicit-spec m_step path runs on one GPU")
    diag.objectives.append(value)

    def system(tr):
        S = tr.spatial_velocity_jacobians()
        if p2p:
            H, g = moms.normal_equations(cents, s2)
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
        accepted = None
        if p2p:
            # candidates built one halving at a time (each is a forward
            # kinematics pass); the first acceptable one stops the search
            scale = 1.0
            for h in range(opts.max_halvings + 1):
                cand = current.updated(scale * step)
                D, delta = _body_motion(current, cand)
                cv = value + moms.delta_energy(D, delta, cents, s2)
                if _accepts(cv, value):
                    accepted = (cand, cv, h, scale, (D, delta))
                    break
                scale *= 0.5
        else:
            cands, scale = [], 1.0
            for _h in range(opts.max_halvings + 1):
                cands.append((current.updated(scale * step), scale))
                scale *= 0.5
            vals = list(path.candidate_objectives_trees([cands[0][0]]))
            if not _accepts(vals[0], value) and len(cands) > 1:
                vals += list(path.candidate_objectives_trees([c for c, _ in cands[1:]]))
            for h, cv in enumerate(vals):
                if _accepts(cv, value):
                    accepted = (cands[h][0], cv, h, cands[h][1], None)
                    break
        if accepted is None:
            break
        cand, value, h, sc, motion = accepted
        diag.objectives.append(value)
        diag.halvings.append(h)
        sn = float(np.linalg.norm(sc * step))
        diag.step_norms.append(sn)
        current = cand
        if sn <= opts.step_tolerance:
            break
        if p2p:
            moms = moms.moved(motion[0], motion[1], cents)
            eq = system(current)
    return current, diag
