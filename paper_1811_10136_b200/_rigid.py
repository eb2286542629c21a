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
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .estep import outlier_constant
from .geometry import skew
from .permutohedral import PermutohedralLattice

_E = [skew(e) for e in np.eye(3)]   # K_k = [e_k]x

# Query-side arithmetic of the EM pass: float32 ranks / barycentrics / table
# rows after a float64 embedding (FR_PASS_FAST), or the all-float64 path.
# Model points are not a bit-exact contract (the reference forms them with a
# BLAS product), and the float32 path keeps the E-step sums to ~1e-7 relative.
FAST_QUERY = True
# Point-to-point pass with float32 centred coordinates over the lattice's dense
# float32 grid (hash slots when the grid would be too large), float32 moment
# partials folded into float64 accumulators every 64 points per thread (FR_PASS_F32).
F32_POINTS = True
# Sort the model points along a Morton curve once per registration.
SPATIAL_ORDER = True
# point-to-point setup: observation upload and splat in one pipelined call
# (fr_lattice_splat_upload); False: upload, then splat
PIPELINED_SPLAT = True
# sigma re-estimation rebuilds splat a Morton-ordered copy of the observation
# points (same sites; sums in that order)
SORTED_REBUILD = True


# Arithmetic of the point-to-point device EM loop: "f64" (default) -- the
# reference's float64 everywhere: float64 point planes (the caller's values bit
# for bit), float64 forward map / simplex / slice over the dense float64 grid /
# epilogue / statistics in one grid-resident kernel (fr_em64_*); "f32" -- the
# float32 point path above (FR_PASS_F32).  FR_PRECISION overrides.
PRECISION = os.environ.get("FR_PRECISION", "f64")


def pass_flags() -> int:
    flags = _lib.FR_PASS_FAST if FAST_QUERY else 0
    if FAST_QUERY and F32_POINTS:
        flags |= _lib.FR_PASS_F32
    return flags


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


def upload_soa(points, dev):
    """(n, 3) host coordinates -> (3, n) float32 device planes through the
    native staged upload (fr_upload_points: threaded float32 conversion into
    pinned slots, DMA on the current stream)."""
    import torch
    P = np.ascontiguousarray(points, dtype=np.float64)
    soa = torch.empty((3, P.shape[0]), dtype=torch.float32, device=dev)
    _lib.check(_lib.load().fr_upload_points(P.ctypes.data_as(ctypes.c_void_p), P.shape[0],
                                            _lib.ptr(soa), _lib.stream_handle()))
    return soa


def upload_soa64(points, dev):
    """(n, 3) host coordinates -> (3, n) float64 device planes (a transpose
    through the native staged upload, fr_upload_points64; no rounding)."""
    import torch
    P = np.ascontiguousarray(points, dtype=np.float64)
    soa = torch.empty((3, P.shape[0]), dtype=torch.float64, device=dev)
    # the rows land in a scratch buffer of the current stream and are
    # transposed there (freed back to that stream's pool, so reuse is ordered)
    rows = torch.empty((P.shape[0], 3), dtype=torch.float64, device=dev)
    _lib.check(_lib.load().fr_upload_rows64(P.ctypes.data_as(ctypes.c_void_p), P.shape[0],
                                            _lib.ptr(rows), _lib.ptr(soa), _lib.stream_handle()))
    return soa


_SIDE_STREAMS: dict = {}
_SETUP_POOL = None

# model + observation points below which the setup runs on the calling thread
# (measured with the persistent worker pool: 100k + 100k points 4.3 -> 3.5 ms
# per registration overlapped; at 10k neither way is faster)
SETUP_OVERLAP_MIN = 50_000

# float64 point-to-point observation through fr_lattice_splat_rows64 (upload
# and splat in one call; page-locked clouds of >= 256k points go out in ranges
# whose splat entries run under the remaining copies).  Off by default:
# measured in the bench at 1M the e2e call takes 3.75 ms with it vs 2.82 ms
# with the single DMA + separate splat (the per-call copy / kernel streams and
# the worker's buffer allocations land on the model side's critical path,
# which the single-DMA order overlaps); FR_CHUNKED_F64=1 turns it on
CHUNKED_F64_SPLAT = os.environ.get("FR_CHUNKED_F64", "0") != "0"


class _InlineExecutor:
    """ThreadPoolExecutor stand-in that runs the job on submit."""

    class _Done:
        def __init__(self, fn, args):
            self._exc, self._val = None, None
            try:
                self._val = fn(*args)
            except BaseException as e:      # re-raised by result(), as a Future would
                self._exc = e

        def result(self):
            if self._exc is not None:
                raise self._exc
            return self._val

    def submit(self, fn, *args):
        return self._Done(fn, args)


def _setup_pool():
    """The process's persistent observation-side workers (spawning a thread
    per registration cost ~0.1 ms on the setup's critical path).  A job only
    waits on its own stream, so concurrent registrations queue, not block."""
    global _SETUP_POOL
    if _SETUP_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _SETUP_POOL = ThreadPoolExecutor(max_workers=4, thread_name_prefix="fr-obs")
    return _SETUP_POOL


def _side_stream():
    """The observation-side setup stream of this thread / device, kept for the
    process (torch's caching allocator pools blocks per stream)."""
    import threading

    import torch
    key = (torch.cuda.current_device(), threading.get_ident())
    st = _SIDE_STREAMS.get(key)
    if st is None:
        st = _SIDE_STREAMS[key] = torch.cuda.Stream()
    return st


class _SetupClock:
    """Per-phase wall times of the device-path setup when FR_PROFILE_SETUP=1
    (synchronising between phases); a no-op otherwise."""

    def __init__(self):
        import os
        import time
        mode = os.environ.get("FR_PROFILE_SETUP")
        self.on = mode == "1"
        self.marks = mode == "2"      # host timestamps since construction, no syncs
        self.phases = {}
        self._t0 = time.perf_counter()
        if self.on:
            import torch
            torch.cuda.synchronize()
            self._t = time.perf_counter()

    def __call__(self, name: str) -> None:
        import time
        if self.marks:
            self.phases[name] = time.perf_counter() - self._t0
        if self.on:
            import torch
            torch.cuda.synchronize()
            now = time.perf_counter()
            self.phases[name] = now - self._t
            self._t = now


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

    def __init__(self, reference, observation, gmm, residual_mode: str, process_group=None,
                 sort: bool = True, precision: str = "f32"):
        import torch
        self.dev = _lib.device()
        self.lib = _lib.load()
        if precision not in ("f32", "f64"):
            raise ValueError(f"unknown precision {precision!r}")
        # float64 planes for the float64 device loop (point_to_point, fixed sigma)
        self.f64 = precision == "f64" and not gmm.update_sigma
        self.mode = _lib.FR_POINT_TO_PLANE if residual_mode == "point_to_plane" \
            else _lib.FR_POINT_TO_POINT
        self.gmm = gmm
        self.group = process_group
        lap = _SetupClock()
        if observation.normals is None and residual_mode == "point_to_plane":
            raise ValueError("observation cloud has no normals")
        # the observation side (upload, splat, blur: host round trips) runs in
        # a worker thread on its own stream while this thread uploads, reduces
        # and Morton-sorts the model cloud
        normals = residual_mode == "point_to_plane"
        self.with_sigma = bool(gmm.update_sigma)
        self.value_mode = (_lib.FR_VALUES_M2 if self.with_sigma else 0) | \
            (_lib.FR_VALUES_NORMALS if normals else 0)
        self.m2_col = 4 if self.with_sigma else -1
        self.normal_col = (5 if self.with_sigma else 4) if normals else -1
        self.lattice = None
        self.sigma = None
        self._obs_dma = None
        main_stream = torch.cuda.current_stream()
        self._main_stream = main_stream
        side = _side_stream()
        # small clouds: the worker thread's handoff costs more than the
        # overlap saves (and serialises on the GIL in register_batch)
        small = len(reference.positions) + len(observation.positions) < SETUP_OVERLAP_MIN
        pool = _InlineExecutor() if small else _setup_pool()
        import threading
        self._obs_uploaded = threading.Event()
        obs_job = pool.submit(self._build_observation, observation, gmm, residual_mode, side,
                              lap if lap.marks else None)
        # the observation upload (the critical path: its splat follows) takes
        # the host memory bandwidth first; the model upload overlaps the splat
        if (residual_mode == "point_to_point" and (PIPELINED_SPLAT or self.f64)
                and not small):
            self._obs_uploaded.wait(timeout=120.0)
            if self.f64 and getattr(self, "_obs_dma", None) is not None:
                main_stream.wait_event(self._obs_dma)
        self.ref = upload_soa64(reference.positions, self.dev) if self.f64 \
            else upload_soa(reference.positions, self.dev)
        self.M = self.ref.shape[1]
        lap("upload_ref")
        # global quantities a shard must not compute locally:
        # total model count (outlier constant, degenerate test), the centre of
        # the whole reference cloud and its bounding-box diameter
        stats_ready = None
        if self.ref.dtype == torch.float64 and self.M > 0:
            # one fused reduction into pinned memory, read once the observation
            # side is done (a pageable D2H here would stall the host -- and the
            # observation thread's launches -- behind the model's DMA)
            work = torch.empty(self.lib.fr_point_stats64_work_doubles() + 9,
                               dtype=torch.float64, device=self.dev)
            _lib.check(self.lib.fr_point_stats64(_lib.ptr(self.ref), self.M, _lib.ptr(work),
                                                 _lib.ptr(work[-9:]), _lib.stream_handle()))
            st_host = torch.empty(9, dtype=torch.float64, pin_memory=True)
            st_host.copy_(work[-9:], non_blocking=True)
            stats_ready = torch.cuda.Event()
            stats_ready.record(main_stream)
        else:
            self._global_stats(self.ref.sum(dim=1, dtype=torch.float64).cpu().numpy(),
                               self.ref.amin(dim=1).double().cpu().numpy(),
                               self.ref.amax(dim=1).double().cpu().numpy())
        lap("global_stats")
        if sort and SPATIAL_ORDER and self.M > 1:
            # Morton order of the model points: reduction sums are order-free up
            # to float64 round-off, and neighbouring threads share table lines
            fn = self.lib.fr_sort_points_morton64 if self.f64 else self.lib.fr_sort_points_morton
            _lib.check(fn(_lib.ptr(self.ref), self.M, 3, None, _lib.stream_handle()))
        lap("morton_sort")
        self.width = self.lib.fr_rigid_pass_width(self.mode, int(self.with_sigma))
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.sums = torch.empty(max(self.width, 16), **f64)
        self.scratch = torch.empty(
            self.lib.fr_rigid_scratch_doubles(self.mode, int(self.with_sigma), self.M), **f64)
        self.host = torch.empty(max(self.width, 16), dtype=torch.float64, pin_memory=True)
        self.wtn = torch.empty((7, self.M), dtype=torch.float32, device=self.dev) \
            if self.mode == _lib.FR_POINT_TO_PLANE and not self.f64 else None
        lap("buffers")
        obs_job.result()              # the side stream is synchronised inside
        if stats_ready is not None:
            stats_ready.synchronize()
            st = st_host.numpy()
            self._global_stats(st[:3].copy(), st[3:6].copy(), st[6:9].copy())
        # later work (passes, rebuilds, frees) is ordered on the caller's stream
        self.obs.record_stream(main_stream)
        if self.obs_n is not None:
            self.obs_n.record_stream(main_stream)
        self.lattice.bind_stream(main_stream)
        lap("observation_side")
        self.setup_s = lap.phases

    def _global_stats(self, local_sum, local_lo, local_hi) -> None:
        """Model count, centre and bounding-box diameter of the whole
        (possibly sharded) reference cloud."""
        tot = self._allreduce(np.concatenate([[float(self.M)], local_sum]), "sum")
        self.M_total = int(round(tot[0]))
        self.c_ref = tot[1:] / tot[0]
        lo = self._allreduce(local_lo, "min")
        hi = self._allreduce(local_hi, "max")
        self.diameter = float(np.linalg.norm(hi - lo))

    def demote_f32(self) -> None:
        """Float32 copies of the float64 planes (for the float32-plane pass
        kernels; the caller's values round to nearest)."""
        import torch
        if self.ref.dtype != torch.float32:
            self.ref = self.ref.float()
        if self.mode == _lib.FR_POINT_TO_PLANE and self.wtn is None:
            self.wtn = torch.empty((7, self.M), dtype=torch.float32, device=self.dev)
        self.f64 = False

    @property
    def c_prime(self) -> float:
        """Outlier constant over the global model count (estep.py:97-112,
        SURVEY.md 8(e)) at the current kernel width."""
        return outlier_constant(self.gmm.outlier_ratio, self.N, self.M_total, self.sigma)

    def _build_observation(self, observation, gmm, residual_mode, stream, lap=None) -> None:
        try:
            self._build_observation_on(observation, gmm, residual_mode, stream, lap)
        finally:
            self._obs_uploaded.set()      # never leave the model side waiting

    def _build_observation_on(self, observation, gmm, residual_mode, stream, lap) -> None:
        import torch
        with torch.cuda.stream(stream):
            if self.f64 and residual_mode == "point_to_point" and CHUNKED_F64_SPLAT:
                # float64 planes, splat from them (keys bit-exact for any input);
                # page-locked rows go out in ranges whose splat entries run
                # under the remaining copies (fr_lattice_splat_rows64)
                if lap is not None:
                    lap("obs_start")
                P = np.ascontiguousarray(observation.positions, dtype=np.float64)
                n = len(P)
                self.obs = torch.empty((3, n), dtype=torch.float64, device=self.dev)
                rows = torch.empty((n, 3), dtype=torch.float64, device=self.dev)
                if lap is not None:
                    lap("obs_buffers")
                self.N, self.obs_n = n, None
                s = np.atleast_1d(np.asarray(gmm.sigma, dtype=float))
                s = np.full(3, s[0]) if s.size == 1 else s
                lat = PermutohedralLattice(3, s)
                if lap is not None:
                    lap("obs_lattice")

                def copied():
                    # the caller's stream already waits for the observation
                    # copies: the model's DMA queues behind them
                    self._obs_uploaded.set()
                    if lap is not None:
                        lap("obs_copies")

                lat.splat_rows64(P, rows, self.obs, self.value_mode, uploaded=copied,
                                 follow_stream=self._main_stream)
                if lap is not None:
                    lap("obs_upload")
                lat.blur()
                del rows
                self.lattice, self.sigma = lat, s
            elif self.f64:
                # float64 planes, splat from them (keys bit-exact for any input)
                self.obs = upload_soa64(observation.positions, self.dev)
                self.N, self.obs_n = self.obs.shape[1], None
                if residual_mode == "point_to_plane":
                    self.obs_n = upload_soa64(observation.normals, self.dev)
                # the model's DMA queues behind this one on the device (the
                # observation splat is the critical path: it gets the link first)
                self._obs_dma = torch.cuda.Event()
                self._obs_dma.record(stream)
                self._obs_uploaded.set()
                if lap is not None:
                    lap("obs_upload")
                self.build(gmm.sigma)
            elif residual_mode == "point_to_point" and PIPELINED_SPLAT:
                # upload and splat in one call: the splat entries of each
                # staged chunk overlap the rest of the upload
                P = np.ascontiguousarray(observation.positions, dtype=np.float64)
                self.obs = torch.empty((3, len(P)), dtype=torch.float32, device=self.dev)
                self.N, self.obs_n = len(P), None
                s = np.atleast_1d(np.asarray(gmm.sigma, dtype=float))
                s = np.full(3, s[0]) if s.size == 1 else s
                lat = PermutohedralLattice(3, s)
                lat.splat_upload(P, self.obs, self.value_mode, uploaded=self._obs_uploaded.set)
                if lap is not None:
                    lap("obs_upload")
                lat.blur()
                self.lattice, self.sigma = lat, s
            else:
                self.obs = upload_soa(observation.positions, self.dev)
                if lap is not None:
                    lap("obs_upload")
                self.N = self.obs.shape[1]
                self.obs_n = None
                if residual_mode == "point_to_plane":
                    self.obs_n = upload_soa(observation.normals, self.dev)
                self.build(gmm.sigma)
            if lap is not None:
                lap("obs_built")
            stream.synchronize()
            if lap is not None:
                lap("obs_synced")

    def build(self, sigma) -> None:
        """(Re)build the observation lattice at kernel width sigma.  The first
        build splats the points in the caller's order (per-entry path, site
        sums in a fixed tree order); sigma re-estimation rebuilds
        (estep.py:232-259, point-to-point) splat a Morton-ordered copy made
        once, with the warp-folded pairs (FR_SPLAT_SPATIAL: ~1/20 of the sort
        items).  Keys and occupied sites are the reference's either way;
        sums differ from np.add.at's flat order by float64 round-off (the
        operator API, PermutohedralLattice.splat, keeps the flat order).
        Measured at 1M: the Morton sort + warp-folded splat on the first
        build cost more than the per-entry path saves (launch-bound small
        sorts), at 16.8M sigma re-estimation it saves ~2 ms per rebuild."""
        import torch
        s = np.atleast_1d(np.asarray(sigma, dtype=float))
        if s.size == 1:
            s = np.full(3, s[0])
        pos = self.obs
        mode = self.value_mode
        if self.lattice is not None and SORTED_REBUILD and self.obs_n is None:
            if getattr(self, "_obs_sorted", None) is None:
                self._obs_sorted = self.obs.clone()
                fn = self.lib.fr_sort_points_morton64 if self.obs.dtype == torch.float64 \
                    else self.lib.fr_sort_points_morton
                _lib.check(fn(_lib.ptr(self._obs_sorted), self.N, 3, None, _lib.stream_handle()))
            pos = self._obs_sorted
            mode |= _lib.FR_SPLAT_SPATIAL
        lat = PermutohedralLattice(3, s)
        lat.splat_points(pos, self.obs_n, mode)
        lat.blur()
        self.lattice, self.sigma = lat, s

    def pass_params(self, R, t) -> "_lib.RigidPassParams":
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
        p.flags = pass_flags()
        return p

    def run_pass(self, R, t) -> np.ndarray:
        """One fused E + assembly sweep at pose (R, t); returns the host sums."""
        p = self.pass_params(R, t)
        _lib.check(self.lib.fr_rigid_pass(self.lattice.handle, _lib.ptr(self.ref), self.M,
                                          ctypes.byref(p), _lib.ptr(self.sums),
                                          _lib.ptr(self.wtn), _lib.ptr(self.scratch),
                                          _lib.stream_handle()))
        self.reduce_device(self.sums[:self.width])
        self.host[:self.width].copy_(self.sums[:self.width])   # synchronising D2H
        return self.host[:self.width].numpy().copy()

    def _allreduce(self, v, op: str) -> np.ndarray:
        """Host-side all-reduce of a small float64 vector over the group."""
        v = np.asarray(v, dtype=float)
        if self.group is None:
            return v
        import torch
        import torch.distributed as dist
        backend = dist.get_backend(self.group)
        dev = _lib.device() if backend == "nccl" else torch.device("cpu")
        t = torch.from_numpy(v.copy()).to(dev)
        red = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}[op]
        dist.all_reduce(t, op=red, group=self.group)
        return t.cpu().numpy()

    def reduce_device(self, t) -> None:
        """Sum the per-shard normal-equation partials across ranks (one NCCL
        all-reduce of <= 31 doubles per EM iteration)."""
        if self.group is not None:
            import torch.distributed as dist
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def centre(self, R, t) -> np.ndarray:
        return np.asarray(R, dtype=float) @ self.c_ref + np.asarray(t, dtype=float)

    def assemble_stored(self, R, t) -> np.ndarray:
        """point_to_plane normal equations at pose (R, t) over the residual spec
        stored by the last pass (the weight / target / normal planes; extra
        Gauss-Newton iterations of mstep.py:425-459 keep the E step's spec):
        [H upper 21 | g 6 | sum r^2], all-reduced over the group."""
        import torch
        R = torch.as_tensor(np.asarray(R, dtype=float), device=self.dev)
        t = torch.as_tensor(np.asarray(t, dtype=float), device=self.dev)
        X = (R @ self.ref.double() + t[:, None]).t().contiguous()       # (m, 3) float64
        w = self.wtn[0].double().contiguous()
        T = self.wtn[1:4].double().t().contiguous()
        N = self.wtn[4:7].double().t().contiguous()
        valid = (N != 0).any(dim=1).to(torch.uint8).contiguous()
        sums = torch.empty(28, dtype=torch.float64, device=self.dev)
        scratch = torch.empty(self.lib.fr_rigid_scratch_doubles(0, 0, self.M),
                              dtype=torch.float64, device=self.dev)
        si, _keep = _lib.dptr(1.0 / np.asarray(self.sigma, dtype=float))
        _lib.check(self.lib.fr_assemble_rigid(_lib.ptr(X), _lib.ptr(w), _lib.ptr(T), self.M, si,
                                              1, _lib.ptr(N), _lib.ptr(valid), _lib.ptr(sums),
                                              _lib.ptr(scratch), _lib.stream_handle()))
        self.reduce_device(sums)
        return sums.cpu().numpy()

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
        self.reduce_device(self.sums[:16])
        self.host[:16].copy_(self.sums[:16])
        return 0.5 * self.host[:k].numpy().copy()


class _DeviceArray:
    """__cuda_array_interface__ view of a raw device buffer (for torch.as_tensor)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3}


class _DeviceInts:
    """__cuda_array_interface__ view of a raw device int32 buffer."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4",
                                         "data": (int(ptr), False), "version": 3}


# sharded float64 loop over NCCL: replay captured chunks (False: the per-
# iteration Python loop with a synchronising status poll per chunk)
GROUP_GRAPH = True
# sharded iteration as one fused launch (solve-first) + the all-reduce
FUSED_SHARDED = True


class DeviceEM:
    """The whole rigid point-to-point EM loop resident on the GPU
    (fr_rigid_em_*): pass, fixed-order reduction and the float64 solver kernel
    per iteration, replayed from a CUDA graph, no host round trip.  With a
    process group the per-iteration partials are all-reduced between the pass
    and the solve, in fixed chunks so every rank enqueues the same number of
    collectives."""

    CHUNK = 8

    def __init__(self, path: RigidDevicePath, R0, t0, config, fast: bool | None = None):
        import torch
        self.path = path
        self.lib = path.lib
        self.max_iters = int(config.max_em_iters)
        c = _lib.RigidEmConfig()
        c.R0[:] = list(np.asarray(R0, dtype=float).reshape(-1))
        c.t0[:] = list(np.asarray(t0, dtype=float).reshape(-1))
        c.c_ref[:] = list(path.c_ref)
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
        c.fast = pass_flags() if fast is None else int(fast)
        self._cfg = c
        h = ctypes.c_void_p()
        _lib.check(self.lib.fr_rigid_em_create_on(path.lattice.handle, _lib.ptr(path.ref), path.M,
                                                  ctypes.byref(c), _lib.stream_handle(),
                                                  ctypes.byref(h)))
        self.h = h
        sp = ctypes.c_void_p()
        w = ctypes.c_int()
        _lib.check(self.lib.fr_rigid_em_sums(h, ctypes.byref(sp), ctypes.byref(w)))
        self.sums = torch.as_tensor(_DeviceArray(sp.value, w.value), device=path.dev)

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.fr_rigid_em_destroy(h)
            except Exception:
                pass
            self.h = None

    def enqueue(self, n: int) -> None:
        """Enqueue n iterations without synchronising (single rank)."""
        if self.path.group is None:
            _lib.check(self.lib.fr_rigid_em_enqueue(self.h, int(n), _lib.stream_handle()))
            return
        for _ in range(int(n)):
            _lib.check(self.lib.fr_rigid_em_pass(self.h, _lib.stream_handle()))
            self.path.reduce_device(self.sums)
            _lib.check(self.lib.fr_rigid_em_solve(self.h, _lib.stream_handle()))

    def status(self):
        d, it, term = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.check(self.lib.fr_rigid_em_status(self.h, ctypes.byref(d), ctypes.byref(it),
                                               ctypes.byref(term), _lib.stream_handle()))
        return bool(d.value), int(it.value), _lib.FR_TERM[int(term.value)]

    def run(self) -> None:
        """Iterate until termination (converged / degenerate / max_iters)."""
        if self.path.group is None:
            _lib.check(self.lib.fr_rigid_em_run(self.h, _lib.stream_handle()))
            return
        while True:
            self.enqueue(self.CHUNK)
            if self.status()[0]:
                return

    def result(self):
        n = self.max_iters
        R = np.zeros(9)
        t = np.zeros(3)
        obj, tn, ms = np.zeros(n), np.zeros(n), np.zeros(n)
        it, term = ctypes.c_int(), ctypes.c_int()
        dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        _lib.check(self.lib.fr_rigid_em_result(self.h, dp(R), dp(t), dp(obj), dp(tn), dp(ms),
                                               ctypes.byref(it), ctypes.byref(term),
                                               _lib.stream_handle()))
        k = min(int(it.value), n)
        return (R.reshape(3, 3), t, list(obj[:k]), list(tn[:k]), list(ms[:k]), int(it.value),
                _lib.FR_TERM[int(term.value)])


class DeviceEM64:
    """The float64 rigid point-to-point EM loop (fr_em64_*): one cooperative
    grid-resident kernel runs pass, fixed-order reduction and the float64
    solve of every iteration to termination.  With a process group each
    iteration is pass -> all-reduce of the 25 sums -> solve, and the
    termination flag is polled in chunks of iterations (every rank issues the
    same number of collectives)."""

    CHUNK = 8

    def __init__(self, path: RigidDevicePath, R0, t0, config):
        import torch
        self.path = path
        self.lib = path.lib
        self.max_iters = int(config.max_em_iters)
        c = _lib.RigidEmConfig()
        c.R0[:] = list(np.asarray(R0, dtype=float).reshape(-1))
        c.t0[:] = list(np.asarray(t0, dtype=float).reshape(-1))
        c.c_ref[:] = list(path.c_ref)
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
        c.fast = 0
        self._cfg = c
        h = ctypes.c_void_p()
        _lib.check(self.lib.fr_em64_create(path.lattice.handle, _lib.ptr(path.ref), path.M,
                                           ctypes.byref(c), _lib.stream_handle(),
                                           ctypes.byref(h)))
        self.h = h
        self._graph = None
        sp = ctypes.c_void_p()
        w = ctypes.c_int()
        _lib.check(self.lib.fr_em64_sums(h, ctypes.byref(sp), ctypes.byref(w)))
        self._sums_ptr = (sp.value, w.value)
        self._sums = None
        # sharded: one fused launch per iteration (solve of the previous
        # sums, then the pass) + one all-reduce; FUSED_SHARDED = False: pass,
        # all-reduce, solve kernel
        self._fused = path.group is not None and FUSED_SHARDED
        if path.group is not None and type(self) is DeviceEM64 and self._nccl_group():
            self._capture()

    @property
    def sums(self):
        """The device sums as a tensor (made on first use: only the sharded
        loop all-reduces them, and the wrapper costs tens of microseconds)."""
        if self._sums is None:
            import torch
            self._sums = torch.as_tensor(_DeviceArray(*self._sums_ptr), device=self.path.dev)
        return self._sums

    def __del__(self):
        self._graph = None             # the captured chunk goes before its buffers
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.fr_em64_destroy(h)
            except Exception:
                pass
            self.h = None

    def launch_info(self):
        g, b = ctypes.c_int(), ctypes.c_int()
        _lib.check(self.lib.fr_em64_launch_info(self.h, ctypes.byref(g), ctypes.byref(b)))
        return int(g.value), int(b.value)

    def enqueue(self, n: int) -> None:
        """Enqueue up to n more iterations without synchronising (sharded over
        NCCL: whole chunks as replays of the captured graph)."""
        if self.path.group is None:
            _lib.check(self.lib.fr_em64_run(self.h, int(n), _lib.stream_handle()))
            return
        n = int(n)
        if self._graph is not None:
            q, n = divmod(n, self.CHUNK)
            for _ in range(q):
                self._graph.replay()
        self._enqueue_eager(n)
        if self._fused:
            # the last pass's all-reduced sums still await their solve
            _lib.check(self.lib.fr_em64_solve(self.h, _lib.stream_handle()))

    def _enqueue_eager(self, n: int) -> None:
        for _ in range(int(n)):
            if self._fused:
                # solve of the previous pass's sums + this pass: one launch
                _lib.check(self.lib.fr_em64_pass_solve(self.h, _lib.stream_handle()))
                self.path.reduce_device(self.sums)
            else:
                _lib.check(self.lib.fr_em64_pass(self.h, _lib.stream_handle()))
                self.path.reduce_device(self.sums)
                _lib.check(self.lib.fr_em64_solve(self.h, _lib.stream_handle()))

    def _capture(self) -> None:
        """CHUNK iterations of pass -> all-reduce -> solve as one CUDA graph
        (captured at construction: nothing runs; the replays do)."""
        import torch
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._enqueue_eager(self.CHUNK)
        self._graph = g
        dp = ctypes.c_void_p()
        _lib.check(self.lib.fr_em64_done_ptr(self.h, ctypes.byref(dp)))
        self._done = torch.as_tensor(_DeviceInts(dp.value, 1), device=self.path.dev)
        self._flags = torch.zeros(2, dtype=torch.int32, pin_memory=True)
        self._events = [torch.cuda.Event(), torch.cuda.Event()]

    def _nccl_group(self) -> bool:
        import torch.distributed as dist
        return GROUP_GRAPH and dist.get_backend(self.path.group) == "nccl"

    def _run_graph(self) -> None:
        """Sharded loop over NCCL: replays of the captured chunk (no Python
        call per iteration); the termination flag is copied into a pinned
        double buffer after every replay and the previous replay's flag is
        read while the current one runs.  Every rank replays the same number
        of chunks (identical reduced sums -> identical flags); passes after
        termination are no-ops inside the kernel."""
        import torch
        chunks = (self.max_iters + self.CHUNK - 1) // self.CHUNK
        for k in range(chunks + 1):
            self._graph.replay()
            self._flags[k % 2:k % 2 + 1].copy_(self._done, non_blocking=True)
            self._events[k % 2].record()
            if k >= 1:
                self._events[(k - 1) % 2].synchronize()
                if int(self._flags[(k - 1) % 2]):
                    return
        torch.cuda.current_stream().synchronize()

    def pass_only(self) -> None:
        """One pass + reduction at the current pose (no solve)."""
        _lib.check(self.lib.fr_em64_pass(self.h, _lib.stream_handle()))

    def status(self):
        d, it, term = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.check(self.lib.fr_em64_status(self.h, ctypes.byref(d), ctypes.byref(it),
                                           ctypes.byref(term), _lib.stream_handle()))
        return bool(d.value), int(it.value), _lib.FR_TERM[int(term.value)]

    def run(self) -> None:
        if self.path.group is None:
            _lib.check(self.lib.fr_em64_run(self.h, 0, _lib.stream_handle()))
            return
        if self._graph is not None:
            self._run_graph()
            return
        while True:
            self.enqueue(self.CHUNK)
            if self.status()[0]:
                return

    def result(self):
        n = self.max_iters
        R = np.zeros(9)
        t = np.zeros(3)
        obj, tn, ms = np.zeros(n), np.zeros(n), np.zeros(n)
        it, term = ctypes.c_int(), ctypes.c_int()
        dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        _lib.check(self.lib.fr_em64_result(self.h, dp(R), dp(t), dp(obj), dp(tn), dp(ms),
                                           ctypes.byref(it), ctypes.byref(term),
                                           _lib.stream_handle()))
        k = min(int(it.value), n)
        return (R.reshape(3, 3), t, list(obj[:k]), list(tn[:k]), list(ms[:k]), int(it.value),
                _lib.FR_TERM[int(term.value)])


class DeviceEM64PL(DeviceEM64):
    """The float64 rigid point-to-plane EM loop (fr_em64pl_*): E pass with the
    stored residual spec, device Cholesky, parallel halving candidates and
    extra Gauss-Newton iterations in one cooperative launch.  Single GPU."""

    def __init__(self, path: RigidDevicePath, R0, t0, config):
        import torch
        if path.group is not None:
            raise ValueError("the point-to-plane device loop runs on one GPU")
        self.path = path
        self.lib = path.lib
        self.max_iters = int(config.max_em_iters)
        c = _lib.RigidEmConfig()
        c.R0[:] = list(np.asarray(R0, dtype=float).reshape(-1))
        c.t0[:] = list(np.asarray(t0, dtype=float).reshape(-1))
        c.c_ref[:] = list(path.c_ref)
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
        c.fast = 0
        self._cfg = c
        h = ctypes.c_void_p()
        _lib.check(self.lib.fr_em64pl_create(path.lattice.handle, _lib.ptr(path.ref), path.M,
                                             ctypes.byref(c), _lib.stream_handle(),
                                             ctypes.byref(h)))
        self.h = h
        sp = ctypes.c_void_p()
        w = ctypes.c_int()
        _lib.check(self.lib.fr_em64pl_sums(h, ctypes.byref(sp), ctypes.byref(w)))
        self._sums_ptr = (sp.value, w.value)
        self._sums = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.fr_em64pl_destroy(h)
            except Exception:
                pass
            self.h = None

    def launch_info(self):
        g, b = ctypes.c_int(), ctypes.c_int()
        _lib.check(self.lib.fr_em64pl_launch_info(self.h, ctypes.byref(g), ctypes.byref(b)))
        return int(g.value), int(b.value)

    def enqueue(self, n: int) -> None:
        _lib.check(self.lib.fr_em64pl_run(self.h, int(n), _lib.stream_handle()))

    def status(self):
        d, it, term = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.check(self.lib.fr_em64pl_status(self.h, ctypes.byref(d), ctypes.byref(it),
                                             ctypes.byref(term), _lib.stream_handle()))
        return bool(d.value), int(it.value), _lib.FR_TERM[int(term.value)]

    def run(self) -> None:
        _lib.check(self.lib.fr_em64pl_run(self.h, 0, _lib.stream_handle()))

    def result(self):
        n = self.max_iters
        R = np.zeros(9)
        t = np.zeros(3)
        obj, tn, ms = np.zeros(n), np.zeros(n), np.zeros(n)
        it, term = ctypes.c_int(), ctypes.c_int()
        dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        _lib.check(self.lib.fr_em64pl_result(self.h, dp(R), dp(t), dp(obj), dp(tn), dp(ms),
                                             ctypes.byref(it), ctypes.byref(term),
                                             _lib.stream_handle()))
        k = min(int(it.value), n)
        return (R.reshape(3, 3), t, list(obj[:k]), list(tn[:k]), list(ms[:k]), int(it.value),
                _lib.FR_TERM[int(term.value)])


def device_em(path: RigidDevicePath, R0, t0, config):
    """The device EM loop of a path: float64 (DeviceEM64) on float64 planes
    with a dense float64 grid, else the float32-point loop (DeviceEM; a
    lattice whose site box exceeds the float64 grid budget runs DeviceEM's
    all-float64 hash-table pass over float32 copies of the planes)."""
    if path.mode == _lib.FR_POINT_TO_PLANE:
        if path.f64 and path.lattice.dense64:
            return DeviceEM64PL(path, R0, t0, config)
        raise ValueError("the point-to-plane device loop needs float64 planes and the dense "
                         "float64 grid")
    if path.f64:
        if path.lattice.dense64:
            return DeviceEM64(path, R0, t0, config)
        path.demote_f32()
        return DeviceEM(path, R0, t0, config, fast=0)
    return DeviceEM(path, R0, t0, config)
