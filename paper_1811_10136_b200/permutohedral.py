"""Permutohedral-lattice Gaussian filter, device-resident (drop-in for the
reference's permutohedral.py, pkg/src/twistreg/permutohedral.py:1-378).

Same objects and semantics: `PermutohedralLattice(dim, sigma)` with staged
`splat` / `blur` / `slice`, the `keys` / `values` / `num_sites` / `blurred`
views, `build_lattice`, `filter_augmented`, `gaussian_transform_bruteforce`
and `valid_lattice_key`.  Every operator runs on the GPU through
libfilterreg_b200.so; the table lives in HBM and is only copied back when
`keys` / `values` are read.  Site keys, pre- and post-blur values are
bit-identical to the reference ("Parity").
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

_MAX_DIM = 12
COMPILED_DIMS = tuple(range(1, 13))   # d <= 3: hashed 63-bit keys; 4..12: sorted 128-bit keys
MAX_VALUE_COLUMNS = 15


def _as_sigma(sigma, dim: int) -> np.ndarray:
    """permutohedral.py:53-61"""
    s = np.asarray(sigma, dtype=float).reshape(-1)
    if s.size == 1:
        s = np.full(dim, s[0])
    if s.shape != (dim,):
        raise ValueError(f"sigma must be scalar or length {dim}, got {s.shape}")
    if not np.all(np.isfinite(s)) or np.any(s <= 0):
        raise ValueError("kernel widths must be finite and positive")
    return s


def _to_device(a, dtype=np.float64):
    import torch
    arr = np.ascontiguousarray(a, dtype=dtype)
    return torch.from_numpy(arr).to(_lib.device())


def valid_lattice_key(key) -> bool:
    """Zero sum and all components congruent mod d+1 (permutohedral.py:89-93)."""
    key = np.asarray(key)
    d1 = key.shape[-1]
    return int(key.sum()) == 0 and np.unique(key % d1).size == 1


def gaussian_transform_bruteforce(query_features, input_features, input_values,
                                  sigma) -> np.ndarray:
    """Exact unnormalised Gaussian transform on the GPU (permutohedral.py:64-86)."""
    import torch
    Q = np.asarray(query_features, dtype=float)
    F = np.asarray(input_features, dtype=float)
    V = np.asarray(input_values, dtype=float)
    if Q.ndim != 2 or F.ndim != 2 or Q.shape[1] != F.shape[1]:
        raise ValueError("query and input features must be 2-D with equal width")
    if V.ndim != 2 or V.shape[0] != F.shape[0]:
        raise ValueError("one value row per input feature row required")
    sig = _as_sigma(sigma, F.shape[1])
    if Q.shape[1] > _MAX_DIM:
        raise ValueError(f"feature dimension above {_MAX_DIM}")
    lib = _lib.load()
    out = torch.empty((len(Q), V.shape[1]), dtype=torch.float64, device=_lib.device())
    if len(Q) == 0:
        return out.cpu().numpy()
    if len(F) == 0:
        return np.zeros((len(Q), V.shape[1]))
    dq, df = _to_device(Q), _to_device(F)
    sp, _keep = _lib.dptr(sig)
    # value columns in chunks of <= 16 per launch
    for c0 in range(0, V.shape[1], 16):
        c1 = min(c0 + 16, V.shape[1])
        dv = _to_device(V[:, c0:c1])
        part = torch.empty((len(Q), c1 - c0), dtype=torch.float64, device=dq.device)
        _lib.check(lib.fr_gauss_bruteforce(_lib.ptr(dq), len(Q), _lib.ptr(df), len(F), F.shape[1],
                                           _lib.ptr(dv), c1 - c0, sp, _lib.ptr(part),
                                           _lib.stream_handle()))
        out[:, c0:c1] = part
    return out.cpu().numpy()


def _reference_row_order(rows: np.ndarray) -> np.ndarray:
    """Row order of the reference's site table (_RowCodec + _index,
    permutohedral.py:96-131, 253-260): numeric lexicographic when the product of
    the column spans is below 2**62 (mixed-radix int64 codes), else the order of
    the rows' raw little-endian int64 bytes (the codec's void-view fallback)."""
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    spans = (rows.max(axis=0) - rows.min(axis=0) + 1).astype(object)
    total = 1
    for sp in spans:
        total *= int(sp)
    if total < 2 ** 62:
        return np.lexsort(rows.T[::-1])
    return np.argsort(rows.view(np.dtype((np.void, 8 * rows.shape[1]))).reshape(-1),
                      kind="stable")


_UPLOADED_CB = ctypes.CFUNCTYPE(None, ctypes.c_void_p)


class PermutohedralLattice:
    """Splat/blur/slice Gaussian filter over an A*_d lattice, table in HBM
    (permutohedral.py:140-345)."""

    def __init__(self, dim: int, sigma):
        if not 1 <= dim <= _MAX_DIM:
            raise ValueError(f"feature dimension must be in [1, {_MAX_DIM}], got {dim}")
        if dim not in COMPILED_DIMS:
            raise ValueError(f"feature dimension {dim} is not compiled into this build "
                             f"(supported: {COMPILED_DIMS})")
        self.dim = dim
        self.sigma = _as_sigma(sigma, dim)
        self._lib = _lib.load()
        _lib.device()
        handle = ctypes.c_void_p()
        sp, _keep = _lib.dptr(self.sigma)
        _lib.check(self._lib.fr_lattice_create(dim, sp, ctypes.byref(handle)))
        self._h = handle
        self.blurred = False
        self._splatted = False
        self._export = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                self._lib.fr_lattice_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self) -> ctypes.c_void_p:
        return self._h

    # --- staged filter ---

    def _check_features(self, features) -> np.ndarray:
        F = np.asarray(features, dtype=float)
        if F.ndim != 2 or F.shape[1] != self.dim:
            raise ValueError(f"features must be (n, {self.dim}), got {F.shape}")
        if not np.all(np.isfinite(F)):
            raise ValueError("non-finite features")
        return F

    def _simplex(self, features):
        """Enclosing-simplex keys (n, d+1, d+1) and barycentrics (n, d+1),
        bit-identical to permutohedral.py:181-215."""
        import torch
        F = self._check_features(features)
        n, d1 = len(F), self.dim + 1
        keys = torch.empty((n, d1, d1), dtype=torch.int32, device=_lib.device())
        bary = torch.empty((n, d1), dtype=torch.float64, device=keys.device)
        if n:
            dF = _to_device(F)
            sp, _keep = _lib.dptr(self.sigma)
            _lib.check(self._lib.fr_simplex(self.dim, sp, _lib.ptr(dF), n, _lib.ptr(keys),
                                            _lib.ptr(bary), _lib.stream_handle()))
        return keys.cpu().numpy().astype(np.int64), bary.cpu().numpy()

    def splat(self, features, values) -> None:
        """permutohedral.py:219-251"""
        V = np.asarray(values, dtype=float)
        F = np.asarray(features, dtype=float)
        if V.ndim != 2 or V.shape[0] != F.shape[0]:
            raise ValueError("one value row per feature row required")
        if not np.all(np.isfinite(V)):
            raise ValueError("non-finite values")
        F = self._check_features(F)
        if V.shape[1] > MAX_VALUE_COLUMNS or V.shape[1] < 1:
            raise ValueError(f"1..{MAX_VALUE_COLUMNS} value columns supported, got {V.shape[1]}")
        dF, dV = _to_device(F), _to_device(V)
        _lib.check(self._lib.fr_lattice_splat(self._h, _lib.ptr(dF), _lib.ptr(dV), len(F),
                                              V.shape[1], _lib.stream_handle()))
        self.blurred = False
        self._splatted = True
        self._export = None

    def splat_points(self, positions_soa, normals_soa=None, value_mode: int = 0) -> None:
        """Splat [1, y, (|y|^2), (n)] generated on device from float32 or
        float64 SoA planes (the MomentEngine value columns, estep.py:153-165)."""
        import torch
        n = positions_soa.shape[1]
        fn = self._lib.fr_lattice_splat_points64 if positions_soa.dtype == torch.float64 \
            else self._lib.fr_lattice_splat_points
        _lib.check(fn(self._h, _lib.ptr(positions_soa), _lib.ptr(normals_soa), n, value_mode,
                      _lib.stream_handle()))
        self.blurred = False
        self._splatted = True
        self._export = None

    def splat_upload(self, host_positions, out_soa, value_mode: int = 0, uploaded=None) -> None:
        """Upload (n, 3) float64 host positions into the float32 planes
        `out_soa` (3, n) and splat [1, y, (|y|^2)] from them, each staged
        chunk's splat entries overlapping the rest of the upload.  `uploaded()`
        runs once the host-side staging is done."""
        P = np.ascontiguousarray(host_positions, dtype=np.float64)
        cb = _UPLOADED_CB((lambda _ctx: uploaded()) if uploaded is not None else (lambda _ctx: None))
        _lib.check(self._lib.fr_lattice_splat_upload(
            self._h, P.ctypes.data_as(ctypes.c_void_p), len(P), value_mode, _lib.ptr(out_soa),
            _lib.stream_handle(), ctypes.cast(cb, ctypes.c_void_p), None))
        self.blurred = False
        self._splatted = True
        self._export = None

    def splat_rows64(self, host_positions, out_rows, out_soa, value_mode: int = 0,
                     uploaded=None, follow_stream=None) -> None:
        """Upload (n, 3) float64 host positions (rows into `out_rows`, planes
        into `out_soa` (3, n), no rounding) and splat [1, y, (|y|^2)] from the
        planes; page-locked rows are copied in ranges whose splat entries run
        under the remaining copies.  Once every copy is enqueued,
        `follow_stream` (a torch stream, optional) waits for them and
        `uploaded()` runs."""
        P = np.ascontiguousarray(host_positions, dtype=np.float64)
        cb = _UPLOADED_CB((lambda _ctx: uploaded()) if uploaded is not None else (lambda _ctx: None))
        fs = ctypes.c_void_p(follow_stream.cuda_stream) if follow_stream is not None else None
        _lib.check(self._lib.fr_lattice_splat_rows64(
            self._h, P.ctypes.data_as(ctypes.c_void_p), len(P), value_mode, _lib.ptr(out_rows),
            _lib.ptr(out_soa), _lib.stream_handle(), fs, ctypes.cast(cb, ctypes.c_void_p), None))
        self.blurred = False
        self._splatted = True
        self._export = None

    def bind_stream(self, stream) -> None:
        """Stream the lattice's stream-ordered frees go behind (after a side-
        stream build has completed)."""
        _lib.check(self._lib.fr_lattice_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)))

    def blur(self) -> None:
        """permutohedral.py:291-327"""
        if self.blurred:
            raise RuntimeError("lattice already blurred")
        if not self._splatted:
            # an empty lattice blurs to an empty lattice
            self.splat(np.zeros((0, self.dim)), np.zeros((0, 1)))
        _lib.check(self._lib.fr_lattice_blur(self._h, _lib.stream_handle()))
        self.blurred = True
        self._export = None

    def slice(self, query_features) -> np.ndarray:
        """permutohedral.py:329-341"""
        if not self.blurred:
            raise RuntimeError("slice requires a blurred lattice")
        return self.slice_device(_to_device(self._check_features(query_features))).cpu().numpy()

    def slice_device(self, dQ):
        """Slice float64 (m, dim) device queries; returns a device tensor."""
        import torch
        if not self.blurred:
            raise RuntimeError("slice requires a blurred lattice")
        nv = self.width
        out = torch.empty((dQ.shape[0], nv), dtype=torch.float64, device=dQ.device)
        if dQ.shape[0]:
            _lib.check(self._lib.fr_lattice_slice(self._h, _lib.ptr(dQ), dQ.shape[0],
                                                  _lib.ptr(out), _lib.stream_handle()))
        return out

    # --- views ---

    def _info(self):
        n = ctypes.c_int64()
        nv = ctypes.c_int()
        bl = ctypes.c_int()
        _lib.check(self._lib.fr_lattice_info(self._h, ctypes.byref(n), ctypes.byref(nv),
                                             ctypes.byref(bl)))
        return int(n.value), int(nv.value), bool(bl.value)

    @property
    def width(self) -> int:
        return max(self._info()[1], 1)

    @property
    def dense_cells(self) -> int:
        """Cells of the dense float32 slice grid (0: the EM pass hashes)."""
        c = ctypes.c_int64()
        _lib.check(self._lib.fr_lattice_dense_cells(self._h, ctypes.byref(c)))
        return int(c.value)

    @property
    def dense64(self) -> bool:
        """True when the lattice carries the dense float64 slice grid of the
        float64 EM loop (site box within FR_DENSE64_MAX_CELLS)."""
        c = ctypes.c_int64()
        _lib.check(self._lib.fr_lattice_dense_cells64(self._h, ctypes.byref(c)))
        return c.value > 0

    @property
    def num_sites(self) -> int:
        return self._info()[0]

    def _exported(self):
        import torch
        if self._export is None:
            S, nv, _ = self._info()
            nv = max(nv, 1)
            keys = torch.empty((S, self.dim + 1), dtype=torch.int32, device=_lib.device())
            vals = torch.empty((S, nv), dtype=torch.float64, device=keys.device)
            if S:
                _lib.check(self._lib.fr_lattice_export(self._h, _lib.ptr(keys), _lib.ptr(vals),
                                                       _lib.stream_handle()))
            k = keys.cpu().numpy().astype(np.int64)
            v = vals.cpu().numpy()
            order = _reference_row_order(k[:, :self.dim]) if S else np.zeros(0, dtype=np.int64)
            self._export = (k[order], v[order])
        return self._export

    @property
    def keys(self) -> np.ndarray:
        return self._exported()[0]

    @property
    def values(self) -> np.ndarray:
        return self._exported()[1]


def build_lattice(input_features, input_values, sigma) -> PermutohedralLattice:
    """Splat + blur (permutohedral.py:348-357)."""
    F = np.asarray(input_features, dtype=float)
    if F.ndim != 2:
        raise ValueError("input features must be 2-D")
    lat = PermutohedralLattice(F.shape[1], sigma)
    lat.splat(F, input_values)
    lat.blur()
    return lat


def filter_augmented(model_features, obs_features, obs_values, sigma) -> np.ndarray:
    """Filter [model; obs] with values [0; obs_values], read at the model rows
    (permutohedral.py:360-378)."""
    Fm = np.asarray(model_features, dtype=float)
    Fo = np.asarray(obs_features, dtype=float)
    Vo = np.asarray(obs_values, dtype=float)
    if Fm.ndim != 2 or Fo.ndim != 2 or Fm.shape[1] != Fo.shape[1]:
        raise ValueError("model and observation features must be 2-D with equal width")
    lat = PermutohedralLattice(Fm.shape[1], sigma)
    lat.splat(np.vstack([Fm, Fo]), np.vstack([np.zeros((len(Fm), Vo.shape[1])), Vo]))
    lat.blur()
    return lat.slice(Fm)
