"""Feature / concatenated correspondences on the GPU (lattice d = 4..12,
SURVEY.md 8(f) rank 2) against the live reference's golden fixtures
(tests/golden/make_golden_features.py): bit-exact simplices and site tables
(including the reference's raw-byte row order at d = 12), slices to float64
round-off, and whole registration traces."""

import json
import os

import numpy as np
import pytest

from oracle import filterreg_oracle as O

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

FEATURE_LATTICES = ["lattice_feat_d4", "lattice_feat_d5", "lattice_feat_d6", "lattice_feat_d12"]


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.fixture(scope="module")
def fr():
    import paper_1811_10136_b200 as fr
    return fr


@pytest.mark.parametrize("case", FEATURE_LATTICES)
def test_feature_simplex_bit_exact(fr, case):
    g = load(case)
    lat = fr.PermutohedralLattice(g["features"].shape[1], g["sigma"])
    keys, bary = lat._simplex(g["features"])
    assert np.array_equal(keys, g["simplex_keys"].astype(np.int64))
    assert np.array_equal(bary, g["simplex_bary"])


@pytest.mark.parametrize("case", FEATURE_LATTICES)
def test_feature_site_tables_bit_exact(fr, case):
    g = load(case)
    lat = fr.PermutohedralLattice(g["features"].shape[1], g["sigma"])
    lat.splat(g["features"], g["values"])
    assert lat.num_sites == len(g["pre_keys"])
    assert np.array_equal(lat.keys, g["pre_keys"].astype(np.int64))
    assert np.array_equal(lat.values, g["pre_values"])
    lat.blur()
    assert lat.num_sites == len(g["post_keys"])
    assert np.array_equal(lat.keys, g["post_keys"].astype(np.int64))
    assert np.array_equal(lat.values, g["post_values"])
    np.testing.assert_allclose(lat.slice(g["queries"]), g["slice"], rtol=1e-12, atol=1e-13)


def test_feature_lattice_far_queries_and_cap(fr):
    """Queries outside the observation's key range slice to zero; a d = 8
    lattice on scattered points hits the reference's site cap and still
    matches the oracle."""
    rng = np.random.default_rng(7)
    F = rng.uniform(0.0, 1.0, (400, 8))
    V = np.hstack([np.ones((400, 1)), rng.standard_normal((400, 2))])
    sigma = np.full(8, 0.05)
    lat = fr.PermutohedralLattice(8, sigma)
    lat.splat(F, V)
    lat.blur()
    ref = O.OracleLattice(8, sigma)
    ref.splat(F, V)
    ref.blur()
    assert np.array_equal(lat.keys, ref.keys) and np.array_equal(lat.values, ref.values)
    Q = np.vstack([F[:50], F[:20] + 50.0])
    np.testing.assert_allclose(lat.slice(Q), ref.slice(Q), rtol=1e-12, atol=1e-13)
    assert not np.any(lat.slice(F[:20] + 50.0))


@pytest.mark.parametrize("case", ["register_concat_d6", "register_feature_d3"])
def test_feature_registration_golden(fr, case):
    g = load(case)
    cfg = json.loads(str(g["config"]))
    gmm = fr.GmmConfig(sigma=cfg["sigma"], outlier_ratio=cfg["w"], mode=cfg["mode"],
                       feature_sigma=cfg["feature_sigma"])
    config = fr.RegistrationConfig(gmm=gmm, max_em_iters=cfg["max_iters"],
                                   twist_tolerance=cfg["tol"])
    res = fr.register(fr.PointCloud(g["X"], features=g["CX"]),
                      fr.PointCloud(g["Y"], features=g["CY"]), fr.RigidModel(), config)
    R, t = res.kinematics.pose.rotation, res.kinematics.pose.translation
    extent = O.bbox_diameter(g["X"])
    assert O.rotation_angle(R @ g["R"].T) <= 1e-4
    assert np.linalg.norm(t - g["t"]) <= 1e-5 * extent
    assert res.termination == str(g["termination"])
    assert abs(res.iterations - int(g["iterations"])) <= 1
    n = min(len(res.objectives), len(g["objectives"])) - 1
    np.testing.assert_allclose(res.objectives[:n], g["objectives"][:n], rtol=1e-5)
    np.testing.assert_allclose(res.inlier_masses[:n], g["inlier_masses"][:n], rtol=1e-5)


def test_bruteforce_backend_registration(fr):
    """backend="bruteforce" (exact Gaussian transform, permutohedral.py:64-86)
    through register(): same trace as the oracle's exact-transform loop."""
    model, obs, _ = O.pebble_pair(1200, outlier_ratio=0.05, seed=9)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    sigma = 0.05 * O.bbox_diameter(X[:1200])
    tr = O.register_rigid(X, Y, sigma=sigma, outlier_ratio=0.1, max_em_iters=60,
                          twist_tolerance=1e-4, backend="bruteforce")
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                                backend="bruteforce", max_em_iters=60, twist_tolerance=1e-4)
    res = fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg)
    assert O.rotation_angle(res.kinematics.pose.rotation @ tr["R"].T) <= 1e-4
    assert np.linalg.norm(res.kinematics.pose.translation - tr["t"]) <= 1e-5 * O.bbox_diameter(X)
    assert res.termination == tr["termination"]
    assert abs(res.iterations - tr["iterations"]) <= 1
