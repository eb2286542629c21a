"""CPU oracle for the FilterReg hot path.

TEST INFRASTRUCTURE ONLY.  This module is a plain NumPy restatement of the
reference `twistreg` algorithm (arxiv 1811.10136, package under
/root/reference/pkg/src/twistreg) for the data-parallel path the B200 engine
accelerates: the permutohedral-lattice E step and the twist Gauss-Newton
M step of the rigid EM loop.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s CPU-baseline / `--impl reference` legs may import it, and only as
the checker or the timed CPU arm -- never as a code path of the product.

Parity pinning: `tests/golden/make_golden.py` runs the live reference in the
build container and commits its outputs as fixtures; `tests/test_oracle_golden.py`
checks this module against them bit-for-bit (keys, barycentric weights,
pre/post-blur site tables) and to round-off (slices, moments, EM traces).

Each function cites the reference file:line it follows (paths relative to
/root/reference/pkg/src/twistreg/).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

# ---------------------------------------------------------------------------
# lattice constants (permutohedral.py:28-50, 147-163)

MAX_DIM = 12
# embedding stretch per dimension (permutohedral.py:33-36)
SCALE = {1: 1.00, 2: 1.00, 3: 1.05, 4: 1.05, 5: 1.05, 6: 1.05,
         7: 1.05, 8: 1.10, 9: 1.10, 10: 1.05, 11: 1.05, 12: 1.05}
# output gain per dimension (permutohedral.py:37-50)
GAIN = {1: 2.8952044967493156, 2: 7.26440867477451, 3: 19.65543341118011,
        4: 46.8204989056386, 5: 109.10733236095797, 6: 253.69798361851673,
        7: 585.8878389979589, 8: 1551.3475661281732, 9: 3556.1187473560817,
        10: 7167.31894204168, 11: 16021.44046866235, 12: 36206.979459505295}

M0_FLOOR = 1e-12            # estep.py:31
SIGMA_FLOOR = 1e-5          # estep.py:32
NORMAL_LENGTH_FLOOR = 0.1   # estep.py:33
DEGENERATE_MASS_FRACTION = 1e-9   # pipeline.py:26
EPS_ANGLE = 1e-9            # geometry.py:15


def widths(sigma, dim):
    """Scalar-or-vector kernel widths, validated (permutohedral.py:53-61)."""
    s = np.asarray(sigma, dtype=float).reshape(-1)
    if s.size == 1:
        s = np.full(dim, s[0])
    if s.shape != (dim,):
        raise ValueError(f"sigma must be scalar or length {dim}")
    if not np.all(np.isfinite(s)) or np.any(s <= 0):
        raise ValueError("kernel widths must be finite and positive")
    return s


def lattice_constants(dim):
    """(scale factors, gain, canonical offset table) (permutohedral.py:156-163)."""
    if not 1 <= dim <= MAX_DIM:
        raise ValueError(f"feature dimension must be in [1, {MAX_DIM}]")
    stretch = np.sqrt(2.0 / 3.0) * (dim + 1) * SCALE[dim]
    j = np.arange(1, dim + 1)
    sf = stretch / np.sqrt(j * (j + 1))
    lvl = np.arange(dim + 1)[:, None]
    rnk = np.arange(dim + 1)[None, :]
    canon = np.where(rnk <= dim - lvl, lvl, lvl - (dim + 1)).astype(np.int64)
    return sf, GAIN[dim], canon


def elevate(features, sig, sf):
    """Embed into the zero-sum hyperplane (permutohedral.py:171-179).

    Row i of the embedding has 1 in columns >= i, -i in column i-1 and zeros
    before; the products are accumulated left to right, matching the BLAS
    product bit for bit (every non-unit coefficient sits alone in its row up
    to that column, so fused multiply-adds cannot change the rounding).
    """
    f = features / sig * sf
    n, d = f.shape
    el = np.empty((n, d + 1))
    for i in range(d + 1):
        acc = None
        for k in range(d):
            if k < i - 1:
                continue
            term = f[:, k] * (-float(i)) if k == i - 1 else f[:, k]
            acc = term if acc is None else acc + term
        el[:, i] = acc
    return el


def embed_simplex(features, sigma):
    """Enclosing-simplex keys (n, d+1, d+1) int64 and barycentrics (n, d+1).

    Follows PermutohedralLattice._simplex (permutohedral.py:181-215): nearest
    remainder-0 point by round-half-even, stable descending rank of the
    residuals, one +-(d+1) wrap, barycentrics from the rank-ordered residuals.
    """
    F = np.asarray(features, dtype=float)
    if F.ndim != 2:
        raise ValueError("features must be 2-D")
    if not np.all(np.isfinite(F)):
        raise ValueError("non-finite features")
    n, d = F.shape
    sig = widths(sigma, d)
    sf, _, canon = lattice_constants(d)
    el = elevate(F, sig, sf)
    d1 = d + 1
    rem0 = np.rint(el / d1).astype(np.int64) * d1
    diff = el - rem0
    # stable descending rank: strictly larger residuals, then equal ones that
    # come earlier (argsort(-diff, kind="stable") at permutohedral.py:194)
    rank = np.zeros((n, d1), dtype=np.int64)
    for i in range(d1):
        for j in range(d1):
            if j == i:
                continue
            before = diff[:, j] > diff[:, i]
            if j < i:
                before |= diff[:, j] == diff[:, i]
            rank[:, i] += before
    h = rem0.sum(axis=1) // d1
    rank += h[:, None]
    lo = rank < 0
    hi = rank > d
    rank = rank + d1 * lo - d1 * hi
    rem0 = rem0 + d1 * lo - d1 * hi
    res = (el - rem0) / d1
    by_rank = np.empty_like(res)
    np.put_along_axis(by_rank, rank, res, axis=1)
    bary = np.empty((n, d1))
    bary[:, 0] = 1.0 + by_rank[:, d] - by_rank[:, 0]
    for lv in range(1, d1):
        bary[:, lv] = by_rank[:, d - lv] - by_rank[:, d - lv + 1]
    keys = rem0[:, None, :] + canon[:, rank].transpose(1, 0, 2)
    return keys, bary


# ---------------------------------------------------------------------------
# sorted site table with mixed-radix codes (permutohedral.py:96-137, 253-270)

class _Codes:
    """Sortable codes of the first d key columns (_RowCodec,
    permutohedral.py:96-131): mixed-radix int64 over the rows' bounds when the
    span product is below 2**62, else the raw bytes of the little-endian int64
    rows (numpy void view: memcmp order, no range test)."""

    def __init__(self, rows):
        rows = np.asarray(rows, dtype=np.int64)
        self.cols = rows.shape[1]
        if len(rows):
            self.lo = rows.min(axis=0)
            self.hi = rows.max(axis=0)
        else:
            self.lo = np.zeros(rows.shape[1], dtype=np.int64)
            self.hi = np.zeros(rows.shape[1], dtype=np.int64)
        span = [int(s) for s in (self.hi - self.lo + 1)]
        total = 1
        for s in span:
            total *= s
        self.arithmetic = total < 2 ** 62
        self.mult = np.ones(len(span), dtype=np.int64)
        if self.arithmetic:
            for c in range(len(span) - 2, -1, -1):
                self.mult[c] = self.mult[c + 1] * span[c + 1]

    def __call__(self, rows):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        if not self.arithmetic:
            codes = rows.view(np.dtype((np.void, 8 * self.cols))).reshape(-1)
            return codes, np.ones(len(rows), dtype=bool)
        ok = np.all((rows >= self.lo) & (rows <= self.hi), axis=1)
        return (np.clip(rows, self.lo, self.hi) - self.lo) @ self.mult, ok


class OracleLattice:
    """Splat / blur / slice with the reference's exact site semantics."""

    def __init__(self, dim, sigma):
        if not 1 <= dim <= MAX_DIM:
            raise ValueError(f"feature dimension must be in [1, {MAX_DIM}]")
        self.dim = dim
        self.sigma = widths(sigma, dim)
        _, self.gain, _ = lattice_constants(dim)
        self.keys = np.empty((0, dim + 1), dtype=np.int64)
        self.values = np.empty((0, 1))
        self.blurred = False
        self._reindex()

    def _reindex(self):
        self._code = _Codes(self.keys[:, :self.dim])
        c, _ = self._code(self.keys[:, :self.dim])
        order = np.argsort(c, kind="stable")
        self.keys = self.keys[order]
        self.values = self.values[order]
        self._sorted = c[order]

    def _find(self, rows):
        """Site index of each key row, -1 when absent (permutohedral.py:262-270)."""
        if len(self._sorted) == 0:
            return np.full(len(rows), -1, dtype=np.int64)
        c, ok = self._code(rows[:, :self.dim])
        pos = np.minimum(np.searchsorted(self._sorted, c), len(self._sorted) - 1)
        return np.where(ok & (self._sorted[pos] == c), pos, -1)

    def splat(self, features, values):
        """Accumulate barycentric contributions (permutohedral.py:219-251).

        Sums run in flat (point, vertex) order per site -- np.bincount adds in
        index order exactly like the reference's np.add.at -- and sites whose
        summed row is exactly zero are dropped.
        """
        V = np.asarray(values, dtype=float)
        F = np.asarray(features, dtype=float)
        if V.ndim != 2 or V.shape[0] != F.shape[0]:
            raise ValueError("one value row per feature row required")
        if not np.all(np.isfinite(V)):
            raise ValueError("non-finite values")
        keys, bary = embed_simplex(F, self.sigma)
        d1 = self.dim + 1
        flat = keys.reshape(-1, d1)
        uniq, inverse = np.unique(flat[:, :self.dim], axis=0, return_inverse=True)
        inverse = inverse.reshape(-1)
        contrib = bary.reshape(-1)[:, None] * np.repeat(V, d1, axis=0)
        acc = np.stack([np.bincount(inverse, weights=contrib[:, c], minlength=len(uniq))
                        for c in range(V.shape[1])], axis=1) if len(uniq) else \
            np.zeros((0, V.shape[1]))
        full = np.concatenate([uniq, -uniq.sum(axis=1, keepdims=True)], axis=1)
        live = np.any(acc != 0.0, axis=1)
        self.keys = full[live].astype(np.int64)
        self.values = acc[live]
        self.blurred = False
        self._reindex()

    def blur(self):
        """d+1 Jacobi [1,2,1]/4 passes with frontier growth (permutohedral.py:291-327)."""
        if self.blurred:
            raise RuntimeError("lattice already blurred")
        d = self.dim
        cap = max(64 * len(self.keys), 200_000)
        for axis in range(d + 1):
            src = np.any(self.values != 0.0, axis=1)
            if len(self.keys) + 2 * int(src.sum()) > cap:
                src[:] = False
            up = self.keys[src] + 1
            up[:, axis] -= d + 1
            dn = self.keys[src] - 1
            dn[:, axis] += d + 1
            cand = np.concatenate([up, dn])
            if len(cand):
                fresh = cand[self._find(cand) < 0]
                if len(fresh):
                    fresh = np.unique(fresh, axis=0)
                    self.keys = np.concatenate([self.keys, fresh])
                    self.values = np.concatenate(
                        [self.values, np.zeros((len(fresh), self.values.shape[1]))])
                    self._reindex()
            nb_up = self.keys + 1
            nb_up[:, axis] = self.keys[:, axis] - d
            nb_dn = self.keys - 1
            nb_dn[:, axis] = self.keys[:, axis] + d
            iu = self._find(nb_up)
            idn = self._find(nb_dn)
            vu = np.where((iu >= 0)[:, None], self.values[np.maximum(iu, 0)], 0.0)
            vd = np.where((idn >= 0)[:, None], self.values[np.maximum(idn, 0)], 0.0)
            self.values = 0.5 * self.values + 0.25 * (vu + vd)
        live = np.any(self.values != 0.0, axis=1)
        self.keys = self.keys[live]
        self.values = self.values[live]
        self._reindex()
        self.blurred = True

    def slice(self, queries):
        """Barycentric gather of the blurred table (permutohedral.py:329-341)."""
        if not self.blurred:
            raise RuntimeError("slice requires a blurred lattice")
        keys, bary = embed_simplex(np.asarray(queries, dtype=float), self.sigma)
        m, d1 = bary.shape
        width = self.values.shape[1]
        if len(self.keys) == 0:
            return np.zeros((m, width))
        idx = self._find(keys.reshape(-1, d1)).reshape(m, d1)
        vals = np.where((idx >= 0)[:, :, None], self.values[np.maximum(idx, 0)], 0.0)
        return self.gain * np.einsum("mk,mkv->mv", bary, vals)

    @property
    def num_sites(self):
        return len(self.keys)


def build_lattice(features, values, sigma):
    """splat + blur (permutohedral.py:348-357)."""
    F = np.asarray(features, dtype=float)
    lat = OracleLattice(F.shape[1], sigma)
    lat.splat(F, values)
    lat.blur()
    return lat


def gauss_bruteforce(queries, inputs, values, sigma):
    """Exact unnormalised Gaussian transform (permutohedral.py:64-86)."""
    Q = np.asarray(queries, dtype=float)
    F = np.asarray(inputs, dtype=float)
    V = np.asarray(values, dtype=float)
    sig = widths(sigma, F.shape[1])
    Fs, Qs = F / sig, Q / sig
    out = np.empty((len(Q), V.shape[1]))
    step = max(1, int(8_000_000 // max(1, F.shape[0] * F.shape[1])))
    for a in range(0, len(Q), step):
        b = min(a + step, len(Q))
        dq = Qs[a:b, None, :] - Fs[None, :, :]
        out[a:b] = np.exp(-0.5 * np.einsum("qnd,qnd->qn", dq, dq)) @ V
    return out


# ---------------------------------------------------------------------------
# E step (estep.py:99-259)

def obs_value_columns(obs_pos, obs_normals=None, with_m2=False):
    """[1, y, (|y|^2), (n)] (estep.py:153-165).  np.einsum's |y|^2 on 3-vectors
    evaluates (y0^2 + y2^2) + y1^2 in numpy 2.3; restated in that order."""
    Y = np.asarray(obs_pos, dtype=float)
    cols = [np.ones((len(Y), 1)), Y]
    if with_m2:
        sq = Y * Y
        cols.append(((sq[:, 0] + sq[:, 2]) + sq[:, 1])[:, None])
    if obs_normals is not None:
        cols.append(np.asarray(obs_normals, dtype=float))
    return np.hstack(cols)


def outlier_constant(w, n_obs, n_model, kernel_sigma):
    """c' on the unnormalised-kernel scale (estep.py:99-112)."""
    if not 0.0 <= w < 1.0:
        raise ValueError("outlier_ratio must be in [0, 1)")
    if n_obs <= 0 or n_model <= 0:
        raise ValueError("cloud sizes must be positive")
    ks = np.asarray(kernel_sigma, dtype=float).reshape(-1)
    c = w / (1.0 - w) * (n_obs / n_model)
    return float(c * np.prod(np.sqrt(2.0 * np.pi) * ks))


def moment_epilogue(out, model_pos, c_prime, m2_col=None, normal_cols=None):
    """Weights, targets, normals from raw kernel sums (estep.py:195-217)."""
    x = np.asarray(model_pos, dtype=float)
    m0 = np.maximum(out[:, 0], 0.0)
    m1 = out[:, 1:4]
    sup = m0 >= M0_FLOOR
    if c_prime > 0.0:
        w = np.where(sup, m0 / (m0 + c_prime), 0.0)
    else:
        w = np.where(sup, 1.0, 0.0)
    safe = np.where(sup, m0, 1.0)
    target = np.where(sup[:, None], m1 / safe[:, None], x)
    res = {"m0": m0, "m1": m1, "weight": w, "target": target, "c_prime": c_prime,
           "m2": out[:, m2_col] if m2_col is not None else None,
           "normal": None, "normal_valid": None}
    if normal_cols is not None:
        avg = out[:, normal_cols] / safe[:, None]
        ln = np.linalg.norm(avg, axis=1)
        valid = sup & (ln >= NORMAL_LENGTH_FLOOR)
        res["normal"] = np.where(valid[:, None],
                                 avg / np.maximum(ln, NORMAL_LENGTH_FLOOR)[:, None], 0.0)
        res["normal_valid"] = valid
    return res


class OracleMoments:
    """Build-once / slice-many moment engine (estep.py:132-217), position mode."""

    def __init__(self, obs_pos, sigma, outlier_ratio, obs_normals=None,
                 with_m2=False, backend="lattice"):
        self.obs = np.asarray(obs_pos, dtype=float)
        self.sigma = widths(sigma, 3)
        self.w = outlier_ratio
        self.values = obs_value_columns(self.obs, obs_normals, with_m2)
        self.m2_col = 4 if with_m2 else None
        self.normal_cols = (slice(5, 8) if with_m2 else slice(4, 7)) \
            if obs_normals is not None else None
        self.backend = backend
        self.lattice = build_lattice(self.obs, self.values, self.sigma) \
            if backend == "lattice" else None

    def raw(self, x):
        if self.lattice is not None:
            return self.lattice.slice(x)
        return gauss_bruteforce(x, self.obs, self.values, self.sigma)

    def moments(self, x, n_model=None):
        """`n_model`: the whole model cloud's size when x is one shard of it
        (the outlier constant uses the global count, estep.py:197-198)."""
        x = np.asarray(x, dtype=float)
        out = self.raw(x)
        cp = outlier_constant(self.w, len(self.obs), len(x) if n_model is None else n_model,
                              self.sigma)
        return moment_epilogue(out, x, cp, self.m2_col, self.normal_cols)


def update_sigma(x, mom, floor=SIGMA_FLOOR):
    """Closed-form isotropic width (estep.py:232-259)."""
    x = np.asarray(x, dtype=float)
    sup = mom["m0"] >= M0_FLOOR
    den = np.where(sup, mom["m0"] + mom["c_prime"], 1.0)
    num = np.where(sup, (mom["m0"] * np.einsum("nd,nd->n", x, x)
                         - 2.0 * np.einsum("nd,nd->n", x, mom["m1"]) + mom["m2"]) / den, 0.0)
    mass = np.where(sup, mom["m0"] / den, 0.0).sum()
    if mass <= 0.0:
        raise RuntimeError("no correspondence mass left")
    return max(float(np.sqrt(max(float(num.sum() / (3.0 * mass)), 0.0))), floor)


# ---------------------------------------------------------------------------
# SE(3) host math (geometry.py:18-210)

def skew(v):
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def polar(M):
    """Nearest rotation via SVD (geometry.py:41-48)."""
    U, _, Vt = np.linalg.svd(M)
    R = U @ Vt
    if np.linalg.det(R) < 0:
        U[:, -1] = -U[:, -1]
        R = U @ Vt
    return R


def twist_exp(tw):
    """(R, t) = exp(omega, v) (geometry.py:154-175)."""
    tw = np.asarray(tw, dtype=float).reshape(6)
    om, v = tw[:3], tw[3:]
    th = np.linalg.norm(om)
    S = skew(om)
    S2 = S @ S
    if th < EPS_ANGLE:
        a, b, c = 1.0 - th ** 2 / 6.0, 0.5 - th ** 2 / 24.0, 1.0 / 6.0 - th ** 2 / 120.0
    else:
        a = np.sin(th) / th
        b = (1.0 - np.cos(th)) / th ** 2
        c = (th - np.sin(th)) / th ** 3
    R = np.eye(3) + a * S + b * S2
    V = np.eye(3) + b * S + c * S2
    return polar(R), V @ v


def apply_twist(tw, R, t):
    """exp(tw) o (R, t), re-orthonormalised; zero twist is a bitwise no-op
    (geometry.py:178-189)."""
    tw = np.asarray(tw, dtype=float).reshape(6)
    if not np.any(tw):
        return R, t
    ER, Et = twist_exp(tw)
    return polar(ER @ R), ER @ t + Et


def rotation_angle(R):
    return float(np.arccos(np.clip((np.trace(R) - 1.0) / 2.0, -1.0, 1.0)))


def rotation_about_axis(axis, angle):
    axis = np.asarray(axis, dtype=float)
    S = skew(axis / np.linalg.norm(axis))
    return np.eye(3) + np.sin(angle) * S + (1.0 - np.cos(angle)) * (S @ S)


# ---------------------------------------------------------------------------
# rigid M step (mstep.py:87-459)

def residual_rows(w, tgt, sinv, mode, normals, valid, x):
    """(index, projection (k, r, 3), residual (k, r)) groups (mstep.py:102-129)."""
    live = np.flatnonzero(w > 0)
    if len(live) == 0:
        return []
    sw = np.sqrt(w[live])
    dx = x[live] - tgt[live]
    if mode == "point_to_point":
        P = sw[:, None, None] * np.diag(sinv)[None]
        return [(live, P, np.einsum("krc,kc->kr", P, dx))]
    groups = []
    ok = valid[live]
    if ok.any():
        P = (sw[ok, None] * normals[live[ok]])[:, None, :]
        groups.append((live[ok], P, np.einsum("krc,kc->kr", P, dx[ok])))
    if (~ok).any():
        P = sw[~ok, None, None] * np.eye(3)[None]
        groups.append((live[~ok], P, np.einsum("krc,kc->kr", P, dx[~ok])))
    return groups


def rigid_objective(spec, x):
    """(mstep.py:132-138)"""
    tot = 0.0
    for _, _, r in residual_rows(*spec, x):
        tot += 0.5 * float(np.sum(r * r))
    return tot


def point_jacobian(x):
    """(n, 3, 6) = [-skew(x) | I] (geometry.py:192-204)."""
    n = len(x)
    J = np.zeros((n, 3, 6))
    J[:, 0, 1], J[:, 0, 2] = x[:, 2], -x[:, 1]
    J[:, 1, 0], J[:, 1, 2] = -x[:, 2], x[:, 0]
    J[:, 2, 0], J[:, 2, 1] = x[:, 1], -x[:, 0]
    J[:, 0, 3] = J[:, 1, 4] = J[:, 2, 5] = 1.0
    return J


def assemble_rigid(spec, x):
    """6x6 normal equations (mstep.py:179-210)."""
    H = np.zeros((6, 6))
    g = np.zeros(6)
    for idx, P, r in residual_rows(*spec, x):
        G = (P @ point_jacobian(x[idx])).reshape(-1, 6)
        H += G.T @ G
        g += G.T @ r.reshape(-1)
    return H, g


def gn_solve(H, g, damping=None):
    """Damped Cholesky with x10 escalation (mstep.py:317-369)."""
    n = len(g)
    if not np.any(g):
        return np.zeros(n)
    tr = float(np.trace(H))
    lam = damping if damping is not None else 1e-6 * tr / n
    for _ in range(6):
        try:
            fac = scipy.linalg.cho_factor(H + lam * np.eye(n))
            return -scipy.linalg.cho_solve(fac, g)
        except (scipy.linalg.LinAlgError, RuntimeError):
            lam = lam * 10.0 if lam > 0 else max(tr / n, 1.0) * 1e-10
    raise RuntimeError("normal equations not factorizable after damping escalation")


def rigid_m_step(spec, ref, R, t, max_halvings=10, damping=None):
    """One GN iteration with step halving (mstep.py:421-459, max_gn_iters=1)."""
    value = rigid_objective(spec, ref @ R.T + t)
    objs = [value]
    x = ref @ R.T + t
    H, g = assemble_rigid(spec, x)
    if not np.any(g):
        return R, t, objs
    step = gn_solve(H, g, damping)
    scale = 1.0
    for _ in range(max_halvings + 1):
        Rc, tc = apply_twist(scale * step, R, t)
        cv = rigid_objective(spec, ref @ Rc.T + tc)
        if cv <= value * (1.0 + 1e-12) + 1e-300:
            objs.append(cv)
            return Rc, tc, objs
        scale *= 0.5
    return R, t, objs


def update_magnitude(Rb, tb, Ra, ta, diameter):
    """angle + shift/diameter (pipeline.py:79-86), single body."""
    return rotation_angle(Ra @ Rb.T) + float(np.linalg.norm(ta - tb)) / diameter


def bbox_diameter(P):
    P = np.asarray(P, dtype=float)
    return float(np.linalg.norm(P.max(axis=0) - P.min(axis=0)))


def register_rigid(ref_pos, obs_pos, R0=None, t0=None, sigma=0.05, outlier_ratio=0.1,
                   mode="point_to_point", obs_normals=None, max_em_iters=50,
                   twist_tolerance=1e-4, backend="lattice", update_sigma_flag=False,
                   sigma_floor=SIGMA_FLOOR, timing=None):
    """Rigid EM loop (pipeline.py:125-181).  Returns a dict trace."""
    import time
    ref = np.asarray(ref_pos, dtype=float)
    R = np.eye(3) if R0 is None else np.asarray(R0, dtype=float)
    t = np.zeros(3) if t0 is None else np.asarray(t0, dtype=float)
    eng = OracleMoments(obs_pos, sigma, outlier_ratio,
                        obs_normals if mode == "point_to_plane" else None,
                        with_m2=update_sigma_flag, backend=backend)
    diam = bbox_diameter(ref)
    sig_cur = eng.sigma.copy()
    tr = {"objectives": [], "twist_norms": [], "inlier_masses": [], "sigmas": [],
          "termination": "max_iters", "iterations": 0}
    for _ in range(max_em_iters):
        tr["iterations"] += 1
        tick = time.perf_counter()
        x = ref @ R.T + t
        mom = eng.moments(x)
        if timing is not None:
            timing["e_step_s"] = timing.get("e_step_s", 0.0) + time.perf_counter() - tick
        mass = float(mom["weight"].sum())
        tr["inlier_masses"].append(mass)
        if mass < DEGENERATE_MASS_FRACTION * len(ref):
            tr["objectives"].append(float("nan"))
            tr["twist_norms"].append(float("nan"))
            tr["termination"] = "degenerate"
            break
        if update_sigma_flag:
            s_new = update_sigma(x, mom, sigma_floor)
            if s_new != sig_cur[0]:
                eng = OracleMoments(obs_pos, s_new, outlier_ratio,
                                    obs_normals if mode == "point_to_plane" else None,
                                    with_m2=True, backend=backend)
                sig_cur = eng.sigma.copy()
            tr["sigmas"].append(s_new)
        spec = (mom["weight"], mom["target"], 1.0 / sig_cur, mode,
                mom["normal"], mom["normal_valid"])
        tick = time.perf_counter()
        Rc, tc, objs = rigid_m_step(spec, ref, R, t)
        if timing is not None:
            timing["m_step_s"] = timing.get("m_step_s", 0.0) + time.perf_counter() - tick
        nrm = update_magnitude(R, t, Rc, tc, diam)
        tr["twist_norms"].append(nrm)
        if nrm < twist_tolerance:
            tr["objectives"].append(objs[0])
            tr["termination"] = "converged"
            break
        R, t = Rc, tc
        tr["objectives"].append(objs[-1])
    tr["R"], tr["t"] = R, t
    if timing is not None:
        timing["iterations"] = tr["iterations"]
    return tr


# ---------------------------------------------------------------------------
# seeded synthetic clouds (synth.py:66-89, 193-284), restated so the GPU box
# (which has no /root/reference) can regenerate the reference's inputs

_PEBBLE_SEED = 1405


def pebble(n, radius=0.0405):
    """Scattered asymmetric blob (synth.py:69-89)."""
    g = np.random.default_rng(_PEBBLE_SEED)
    u = g.uniform(np.cos(np.pi - 0.12), np.cos(0.12), n)
    th = np.arccos(u)
    ph = g.uniform(0.0, 2.0 * np.pi, n)
    bump = (0.22 * np.sin(th) * np.cos(ph) + 0.16 * np.cos(2.0 * th) * np.sin(ph)
            + 0.10 * np.sin(3.0 * th) * np.cos(2.0 * ph + 0.7))
    r = radius * (1.0 + bump)
    return np.stack([r * np.sin(th) * np.cos(ph), r * np.sin(th) * np.sin(ph),
                     r * np.cos(th)], axis=-1)


def pebble_resample(n, seed, outlier_ratio=0.0, expansion=1.2, radius=0.0405):
    """An independent scattered sampling of the pebble surface (same surface as
    synth.py:69-89, sampling seed `seed`), with uniform outliers in its 1.2x
    box -- the extra model shards of the weak-scaling benchmark."""
    g = np.random.default_rng([_PEBBLE_SEED, seed])
    u = g.uniform(np.cos(np.pi - 0.12), np.cos(0.12), n)
    th = np.arccos(u)
    ph = g.uniform(0.0, 2.0 * np.pi, n)
    bump = (0.22 * np.sin(th) * np.cos(ph) + 0.16 * np.cos(2.0 * th) * np.sin(ph)
            + 0.10 * np.sin(3.0 * th) * np.cos(2.0 * ph + 0.7))
    r = radius * (1.0 + bump)
    pts = np.stack([r * np.sin(th) * np.cos(ph), r * np.sin(th) * np.sin(ph),
                    r * np.cos(th)], axis=-1)
    if outlier_ratio > 0.0:
        k = int(round(outlier_ratio * n))
        lo, hi = pts.min(axis=0), pts.max(axis=0)
        c, h = (lo + hi) / 2.0, (hi - lo) / 2.0 * expansion
        pts = np.vstack([pts, c + g.uniform(-1.0, 1.0, (k, 3)) * h])
    return pts


def pebble_pair(n, rotation_degrees=50.0, translation_fraction=0.02,
                outlier_ratio=0.0, seed=0, trial=0, expansion=1.2):
    """synthesize_pair for the pebble source, noise-free (synth.py:252-284)."""
    base = pebble(n)
    diam = bbox_diameter(base)
    g = np.random.default_rng([seed, trial])
    axis = g.standard_normal(3)
    shift = translation_fraction * diam * g.standard_normal(3)
    Rgt = rotation_about_axis(axis, np.radians(rotation_degrees))
    model = base.copy()
    obs = base @ Rgt.T + shift
    if outlier_ratio > 0.0:
        k = int(round(outlier_ratio * n))
        for which in (0, 1):
            pts = model if which == 0 else obs
            lo, hi = pts.min(axis=0), pts.max(axis=0)
            c, h = (lo + hi) / 2.0, (hi - lo) / 2.0 * expansion
            extra = c + g.uniform(-1.0, 1.0, (k, 3)) * h
            if which == 0:
                model = np.vstack([model, extra])
            else:
                obs = np.vstack([obs, extra])
    return model, obs, (Rgt, shift)
