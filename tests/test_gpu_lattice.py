"""GPU parity of the E-step filter operator against the reference's golden
fixtures and the CPU oracle (mirrors pkg/tests/test_permutohedral.py and
test_estep.py).  Bar: bit-exact keys / barycentrics / site tables, slices and
moments to float64 round-off."""

import os

import numpy as np
import pytest

from oracle import filterreg_oracle as O

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu

LATTICE_CASES = ["lattice_pebble_s5", "lattice_pebble_s05", "lattice_aniso",
                 "lattice_cuboid_normals"]


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.fixture(scope="module")
def fr():
    import paper_1811_10136_b200 as fr
    return fr


@pytest.mark.parametrize("case", LATTICE_CASES)
def test_simplex_bit_exact(fr, case):
    g = load(case)
    lat = fr.PermutohedralLattice(3, g["sigma"])
    keys, bary = lat._simplex(g["features"])
    assert np.array_equal(keys, g["simplex_keys"].astype(np.int64))
    assert np.array_equal(bary, g["simplex_bary"])


@pytest.mark.parametrize("case", LATTICE_CASES)
def test_site_tables_bit_exact(fr, case):
    g = load(case)
    lat = fr.PermutohedralLattice(3, g["sigma"])
    lat.splat(g["features"], g["values"])
    assert lat.num_sites == len(g["pre_keys"])
    assert np.array_equal(lat.keys, g["pre_keys"].astype(np.int64))
    assert np.array_equal(lat.values, g["pre_values"])
    lat.blur()
    assert np.array_equal(lat.keys, g["post_keys"].astype(np.int64))
    assert np.array_equal(lat.values, g["post_values"])
    np.testing.assert_allclose(lat.slice(g["queries"]), g["slice"], rtol=1e-12, atol=1e-13)


def test_point_splat_equals_generic_splat(fr):
    import torch
    from paper_1811_10136_b200 import _lib
    g = load("lattice_pebble_s5")
    Y = g["features"]
    lat = fr.PermutohedralLattice(3, g["sigma"])
    soa = torch.from_numpy(np.ascontiguousarray(Y.T, dtype=np.float32)).cuda()
    lat.splat_points(soa, None, _lib.FR_VALUES_M2 | _lib.FR_SPLAT_FLAT_ORDER)
    lat.blur()
    assert np.array_equal(lat.keys, g["post_keys"].astype(np.int64))
    assert np.array_equal(lat.values, g["post_values"])


@pytest.mark.parametrize("f64", [False, True])
def test_point_splat_tree_order_within_roundoff(fr, f64):
    """The EM path's default point splat (fixed-tree site sums): keys and
    occupied sites bit-exact, values within float64 round-off of np.add.at's
    flat order, and bit-identical from run to run."""
    import torch
    from paper_1811_10136_b200 import _lib
    g = load("lattice_pebble_s5")
    Y = g["features"]
    dt = np.float64 if f64 else np.float32
    soa = torch.from_numpy(np.ascontiguousarray(Y.T, dtype=dt)).cuda()
    out = []
    for _ in range(2):
        lat = fr.PermutohedralLattice(3, g["sigma"])
        lat.splat_points(soa, None, _lib.FR_VALUES_M2)
        lat.blur()
        out.append((lat.keys, lat.values))
    assert np.array_equal(out[0][0], g["post_keys"].astype(np.int64))
    scale = np.abs(g["post_values"]).max(axis=0)
    assert np.all(np.abs(out[0][1] - g["post_values"]) <= 1e-13 * scale)
    assert np.array_equal(out[0][1], out[1][1])


def test_moments_match_reference(fr):
    g = load("moments_pebble")
    eng = fr.MomentEngine(fr.PointCloud(g["Y"]), fr.GmmConfig(sigma=float(g["sigma"]),
                                                              outlier_ratio=0.1,
                                                              update_sigma=True))
    mf = eng.moments(g["X"])
    for k in ("m0", "m1", "weight", "target", "m2"):
        np.testing.assert_allclose(getattr(mf, k), g[k], rtol=1e-12, atol=1e-14, err_msg=k)
    assert fr.update_sigma(g["X"], mf) == pytest.approx(float(g["sigma_new"]), rel=1e-12)
    c = load("moments_cuboid")
    eng = fr.MomentEngine(fr.PointCloud(c["Y"], normals=c["N"]),
                          fr.GmmConfig(sigma=float(c["sigma"]), outlier_ratio=0.1),
                          include_normals=True)
    mf = eng.moments(c["X"])
    for k in ("m0", "m1", "weight", "target", "normal"):
        np.testing.assert_allclose(getattr(mf, k), c[k], rtol=1e-12, atol=1e-14, err_msg=k)
    assert np.array_equal(mf.normal_valid, c["normal_valid"])


def test_bruteforce_matches_oracle(fr):
    rng = np.random.default_rng(0)
    F = rng.normal(size=(700, 3))
    Q = rng.normal(size=(300, 3))
    V = rng.normal(size=(700, 2))
    got = fr.gaussian_transform_bruteforce(Q, F, V, np.array([0.5, 0.7, 0.9]))
    np.testing.assert_allclose(got, O.gauss_bruteforce(Q, F, V, np.array([0.5, 0.7, 0.9])),
                               rtol=1e-12, atol=1e-12)


def test_bruteforce_moments_backend(fr):
    rng = np.random.default_rng(1)
    X = rng.uniform(-0.1, 0.1, (80, 3))
    Y = rng.uniform(-0.1, 0.1, (120, 3))
    mf = fr.compute_moments(X, fr.PointCloud(Y), fr.GmmConfig(sigma=0.05, outlier_ratio=0.2),
                            backend="bruteforce")
    ref = O.OracleMoments(Y, 0.05, 0.2, backend="bruteforce").moments(X)
    np.testing.assert_allclose(mf.m0, ref["m0"], rtol=1e-12)
    np.testing.assert_allclose(mf.target, ref["target"], rtol=1e-12)


# --- structural / known-answer properties (test_permutohedral.py) ----------

def test_single_point_sites(fr):
    rng = np.random.default_rng(3)
    for d in (1, 2, 3):
        lat = fr.PermutohedralLattice(d, 1.0)
        lat.splat(rng.normal(size=(1, d)), np.ones((1, 1)))
        assert lat.num_sites <= d + 2
        for key in lat.keys:
            assert fr.valid_lattice_key(key)


def test_barycentrics_sum_to_one(fr):
    rng = np.random.default_rng(4)
    for d in (1, 2, 3):
        lat = fr.PermutohedralLattice(d, 1.0)
        F = rng.normal(size=(200, d)) * 5
        keys, bary = lat._simplex(F)
        k2, b2 = O.embed_simplex(F, 1.0)
        assert np.array_equal(keys, k2) and np.array_equal(bary, b2)
        np.testing.assert_allclose(bary.sum(axis=1), 1.0, atol=1e-12)


def test_errors(fr):
    lat = fr.PermutohedralLattice(3, 1.0)
    bad = np.zeros((2, 3))
    bad[0, 0] = np.nan
    with pytest.raises(ValueError):
        lat.splat(bad, np.ones((2, 1)))
    with pytest.raises(ValueError):
        lat.splat(np.zeros((2, 3)), np.array([[np.inf], [0.0]]))
    lat.splat(np.zeros((1, 3)), np.ones((1, 1)))
    with pytest.raises(RuntimeError):
        lat.slice(np.zeros((1, 3)))
    lat.blur()
    with pytest.raises(RuntimeError):
        lat.blur()
    with pytest.raises(ValueError):
        fr.PermutohedralLattice(13, 1.0)


def test_linearity_and_permutation(fr):
    rng = np.random.default_rng(6)
    F = rng.uniform(0, 5, size=(120, 3))
    Q = rng.uniform(0, 5, size=(40, 3))
    Va, Vb = rng.normal(size=(120, 2)), rng.normal(size=(120, 2))
    comb = fr.build_lattice(F, 1.7 * Va - 0.6 * Vb, 0.8).slice(Q)
    parts = 1.7 * fr.build_lattice(F, Va, 0.8).slice(Q) - 0.6 * fr.build_lattice(F, Vb, 0.8).slice(Q)
    np.testing.assert_allclose(comb, parts, atol=1e-10)
    perm = rng.permutation(120)
    np.testing.assert_allclose(fr.build_lattice(F[perm], Va[perm], 0.6).slice(Q),
                               fr.build_lattice(F, Va, 0.6).slice(Q), atol=1e-9)


def test_far_query_and_zero_values(fr):
    rng = np.random.default_rng(8)
    F = rng.uniform(0, 1, size=(50, 3))
    out = fr.build_lattice(F, np.ones((50, 1)), 0.05).slice(np.array([[100.0, 100.0, 100.0]]))
    assert np.array_equal(out, np.zeros((1, 1)))
    lat = fr.build_lattice(F, np.zeros((50, 4)), 0.1)
    assert lat.num_sites == 0
    assert np.array_equal(lat.slice(F), np.zeros((50, 4)))


def test_augmented_equals_build_then_slice(fr):
    rng = np.random.default_rng(11)
    for _ in range(20):
        d = int(rng.integers(1, 4))
        n, m = int(rng.integers(5, 60)), int(rng.integers(5, 60))
        F = rng.uniform(0, 3, size=(n, d))
        Q = rng.uniform(0, 3, size=(m, d))
        V = rng.normal(size=(n, 2))
        s = float(rng.uniform(0.1, 1.0))
        a = fr.filter_augmented(Q, F, V, s)
        np.testing.assert_allclose(a, fr.build_lattice(F, V, s).slice(Q), atol=1e-10)
        np.testing.assert_allclose(a, O.build_lattice(F, V, s).slice(Q), rtol=1e-12, atol=1e-12)


def test_empty_inputs(fr):
    lat = fr.build_lattice(np.zeros((0, 3)), np.zeros((0, 2)), 0.5)
    assert lat.num_sites == 0
    assert lat.slice(np.ones((3, 3))).shape == (3, 2)


# --- larger clouds: bit-exact tables at C1/100k scale -----------------------

@pytest.mark.parametrize("n,frac", [(10000, 0.05), (100000, 0.05), (100000, 0.005)])
def test_large_cloud_tables_bit_exact(fr, n, frac):
    model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=2)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    sigma = frac * O.bbox_diameter(X[:n])
    V = O.obs_value_columns(Y)
    lat = fr.build_lattice(Y, V, sigma)
    ref = O.build_lattice(Y, V, sigma)
    assert np.array_equal(lat.keys, ref.keys)
    assert np.array_equal(lat.values, ref.values)
    np.testing.assert_allclose(lat.slice(X[:20000]), ref.slice(X[:20000]), rtol=1e-12,
                               atol=1e-12)


@pytest.mark.parametrize("order", ["morton", "shuffled"])
def test_point_splat_warp_folded(fr, order):
    """FR_SPLAT_SPATIAL (warp-folded pairs): on Morton-ordered points the
    pair path, on shuffled points the per-entry fallback -- keys and occupied
    sites bit-exact, values within float64 round-off of np.add.at's flat
    order, bit-identical reruns."""
    import torch
    from paper_1811_10136_b200 import _lib
    g = load("lattice_pebble_s5")
    Y = np.asarray(g["features"], dtype=np.float64)
    if order == "shuffled":
        Y = Y[np.random.default_rng(0).permutation(len(Y))]
    soa = torch.from_numpy(np.ascontiguousarray(Y.T)).cuda()
    if order == "morton":
        lib = _lib.load()
        _lib.check(lib.fr_sort_points_morton64(_lib.ptr(soa), soa.shape[1], 3, None,
                                               _lib.stream_handle()))
    out = []
    for _ in range(2):
        lat = fr.PermutohedralLattice(3, g["sigma"])
        lat.splat_points(soa, None, _lib.FR_VALUES_M2 | _lib.FR_SPLAT_SPATIAL)
        lat.blur()
        out.append((lat.keys, lat.values))
    assert np.array_equal(out[0][0], g["post_keys"].astype(np.int64))
    scale = np.abs(g["post_values"]).max(axis=0)
    assert np.all(np.abs(out[0][1] - g["post_values"]) <= 1e-13 * scale)
    assert np.array_equal(out[0][1], out[1][1])
