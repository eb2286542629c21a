"""Behavioural properties the reference's own suite checks on this path
(pkg/tests/test_permutohedral.py, test_estep.py, test_mstep.py,
test_pipeline.py), run against the GPU engine: lattice invariants and accuracy
vs the exact transform, unsupported points, zero-weight rows, convergence,
EM ascent and rotation equivariance."""

import numpy as np
import pytest

from oracle import filterreg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fr():
    import paper_1811_10136_b200 as fr
    return fr


def surface(n, seed):
    return O.pebble_resample(n, seed=seed)


def ring_sphere(n_rings=16, n_per_ring=36, radius=0.075, cap=0.4):
    """A capless sphere on a regular (theta, phi) grid: symmetric under the
    2 pi / n_per_ring spin and the z-mirror, so the cloud's kernel pulls on
    itself cancel (the shape of test_pipeline.py's self-registration test)."""
    th, ph = np.meshgrid(np.linspace(cap, np.pi - cap, n_rings),
                         np.arange(n_per_ring) * (2.0 * np.pi / n_per_ring), indexing="ij")
    return radius * np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)],
                             axis=-1).reshape(-1, 3)


# --- lattice (test_permutohedral.py) ---------------------------------------

def test_keys_valid_after_blur_and_mass_bounded(fr):
    """Every site is a lattice point after blur (:89-95); a homogeneous cloud's
    slice mass stays within [0, n] (:153-160)."""
    rng = np.random.default_rng(10)
    n = 400
    F = rng.uniform(0, 2, size=(n, 3))
    lat = fr.build_lattice(F, np.ones((n, 1)), 0.3)
    assert all(fr.valid_lattice_key(k) for k in lat.keys)
    out = lat.slice(rng.uniform(0, 2, size=(200, 3)))[:, 0]
    assert (out >= 0).all() and (out <= n).all()


def test_lattice_accuracy_vs_exact_transform(fr):
    """Registration operating point (:177-195): median mass error <= 5 %,
    95th-percentile target displacement <= 0.1 sigma against the exact
    Gaussian transform."""
    rng = np.random.default_rng(12)
    n = 3000
    Y = surface(n, 1)
    X = surface(n, 2) + rng.normal(scale=0.0005, size=(n, 3))
    sigma = 0.05 * float(np.linalg.norm(Y.max(0) - Y.min(0)))
    V = np.c_[np.ones(n), Y]
    brute = fr.gaussian_transform_bruteforce(X, Y, V, sigma)
    approx = fr.build_lattice(Y, V, sigma).slice(X)
    good = brute[:, 0] >= 1e-3
    rel = np.abs(approx[good, 0] - brute[good, 0]) / brute[good, 0]
    assert np.median(rel) <= 0.05
    terr = np.linalg.norm(approx[good, 1:] / approx[good, :1] - brute[good, 1:] / brute[good, :1],
                          axis=1)
    assert np.percentile(terr, 95) <= 0.1 * sigma


def test_anisotropic_sigma_equals_whitened(fr):
    """Per-axis widths == isotropic filtering of pre-whitened features (:197-207)."""
    rng = np.random.default_rng(13)
    F = rng.uniform(0, 1, size=(200, 3))
    Q = rng.uniform(0, 1, size=(50, 3))
    V = rng.normal(size=(200, 2))
    sigma = np.array([0.05, 0.1, 0.2])
    a = fr.build_lattice(F, V, sigma).slice(Q)
    b = fr.build_lattice(F / sigma, V, 1.0).slice(Q / sigma)
    np.testing.assert_allclose(a, b, atol=1e-9)


# --- E step (test_estep.py) ---------------------------------------------------

def test_unsupported_points_zero_weight_own_target(fr):
    """Model points far from every observation: weight 0 and target = own
    position (estep.py:197-217; test_estep.py:161-168)."""
    Y = surface(2000, 3)
    X = np.vstack([surface(500, 4), surface(50, 5) + 5.0])
    gmm = fr.GmmConfig(sigma=0.004, outlier_ratio=0.1)
    mf = fr.compute_moments(fr.PointCloud(X), fr.PointCloud(Y), gmm)
    far = slice(500, 550)
    assert np.all(mf.weight[far] == 0.0)
    assert np.array_equal(mf.target[far], X[far])
    assert np.all(mf.weight[:500] > 0.0)


# --- M step (test_mstep.py) -----------------------------------------------------

def test_zero_weight_rows_equal_removal(fr):
    """Rows with zero weight contribute nothing: bit-identical to removing
    those points (test_mstep.py:162-171)."""
    rng = np.random.default_rng(7)
    m = 3000
    x = rng.uniform(-0.1, 0.1, (m, 3))
    tgt = x + rng.normal(scale=0.002, size=(m, 3))
    w = rng.uniform(0.2, 1.0, m)
    w[rng.random(m) < 0.3] = 0.0
    sinv = np.full(3, 1.0 / 0.005)
    keep = w > 0
    a = fr.assemble_rigid(fr.ResidualSpec(w, tgt, sinv, "point_to_point", None, None), x)
    b = fr.assemble_rigid(fr.ResidualSpec(w[keep], tgt[keep], sinv, "point_to_point", None, None),
                          x[keep])
    np.testing.assert_allclose(a.A, b.A, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(a.b, b.b, rtol=1e-12, atol=1e-12)


# --- EM driver (test_pipeline.py) -------------------------------------------------

def test_identical_clouds_stay_put(fr):
    """Identical clouds with the exact transform: converged within 2
    iterations at the identity (test_pipeline.py:161-173, brute force as
    there; the lattice's approximation moves a self-registration slightly)."""
    P = ring_sphere()
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.0075, outlier_ratio=0.1),
                                backend="bruteforce")
    res = fr.register(fr.PointCloud(P), fr.PointCloud(P.copy()), fr.RigidModel(), cfg)
    assert res.termination == "converged" and res.iterations <= 2
    assert fr.alignment_error(res.kinematics.pose, fr.RigidTransform.identity(),
                              fr.PointCloud(P)) <= 1e-9


def test_recovers_moderate_rotation(fr):
    """20 deg rotation + shift recovered within 2 mm (test_pipeline.py:175-188)."""
    P = surface(5000, 7)
    gt = fr.RigidTransform(O.rotation_about_axis([0.3, 1.0, 0.2], np.radians(20.0)),
                           np.array([0.004, -0.002, 0.003]))
    obs = fr.PointCloud(gt.apply(P))
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=fr.default_sigma(obs), outlier_ratio=0.1),
                                max_em_iters=250)
    res = fr.register(fr.PointCloud(P), obs, fr.RigidModel(), cfg)
    assert res.termination == "converged"
    assert fr.alignment_error(res.kinematics.pose, gt, fr.PointCloud(P)) <= 0.002


def test_em_log_likelihood_ascent(fr):
    """The exact-transform EM never decreases the log-likelihood
    (test_pipeline.py:301-321)."""
    rng = np.random.default_rng(11)
    for _ in range(6):
        obs_pts = 0.1 * rng.standard_normal((40, 3))
        model_pts = obs_pts[rng.permutation(40)[:35]]
        gt = fr.RigidTransform(O.rotation_about_axis(rng.standard_normal(3), 0.3),
                               0.02 * rng.standard_normal(3))
        ref, obs = fr.PointCloud(model_pts), fr.PointCloud(gt.apply(obs_pts))
        cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.03, outlier_ratio=0.2),
                                    backend="bruteforce", max_em_iters=8, twist_tolerance=1e-12,
                                    record_states=True)
        res = fr.register(ref, obs, fr.RigidModel(), cfg)
        models = [fr.RigidModel()] + list(res.states)
        vals = [fr.log_likelihood(mm.pose.apply(model_pts), obs, cfg.gmm) for mm in models]
        for prev, cur in zip(vals, vals[1:]):
            assert cur - prev >= -1e-10 * max(1.0, abs(prev))


def test_rotation_equivariance(fr):
    """A globally rotated problem gives the conjugated pose within 1e-6 m
    (test_pipeline.py:342-362), on both the lattice and the exact backends."""
    P = surface(2000, 8)
    rng = np.random.default_rng(5)
    gt = fr.RigidTransform(O.rotation_about_axis(rng.standard_normal(3), 0.25),
                           0.005 * rng.standard_normal(3))
    obs = fr.PointCloud(gt.apply(P))
    spin = fr.RigidTransform(O.rotation_about_axis([1.0, -0.3, 0.8], 1.1), np.zeros(3))
    for backend, tol in (("bruteforce", 1e-6), ("lattice", 1e-3)):
        cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=fr.default_sigma(obs),
                                                     outlier_ratio=0.1),
                                    backend=backend, max_em_iters=15)
        base = fr.register(fr.PointCloud(P), obs, fr.RigidModel(), cfg)
        conj = fr.register(fr.PointCloud(spin.apply(P)), fr.PointCloud(spin.apply(obs.positions)),
                           fr.RigidModel(spin.compose(spin.inverse())), cfg)
        expected = spin.compose(base.kinematics.pose).compose(spin.inverse())
        # the lattice is not rotation-invariant (axis-aligned embedding): the
        # conjugated run agrees to the filter's accuracy, the exact one to round-off
        assert fr.alignment_error(conj.kinematics.pose, expected,
                                  fr.PointCloud(spin.apply(P))) <= tol
