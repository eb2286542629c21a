"""GPU vs LIVE-reference parity at the BASELINE configs' full sizes (north-star
bars: final rotation within 1e-4 rad, translation within 1e-5 x cloud extent,
iteration count within 1).  The reference results come from
tests/golden/make_golden_configs.py (twistreg.register, pipeline.py:125-181,
on the same inputs); pebble inputs are rebuilt here by the oracle's generator
(bit-identical to synth.synthesize_pair, tests/test_oracle_golden.py).

Both query arithmetics of the rigid point-to-point device loop are checked:
"f64" (the default; the reference's float64 everywhere) and "f32" (the
float32 point path)."""

import os

import numpy as np
import pytest

from oracle import filterreg_oracle as O

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu


def load(name):
    path = os.path.join(GOLDEN, f"config_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing golden fixture {path}")
    return np.load(path, allow_pickle=False)


@pytest.fixture(scope="module")
def fr():
    import paper_1811_10136_b200 as fr
    return fr


@pytest.fixture
def precision(request):
    from paper_1811_10136_b200 import _rigid
    old = _rigid.PRECISION
    _rigid.PRECISION = request.param
    yield request.param
    _rigid.PRECISION = old


_PEBBLES: dict = {}


def pebble(n):
    if n not in _PEBBLES:
        model, obs, _ = O.pebble_pair(n, rotation_degrees=50.0, translation_fraction=0.02,
                                      outlier_ratio=0.05, seed=0)
        X = model.astype(np.float32).astype(np.float64)
        Y = obs.astype(np.float32).astype(np.float64)
        _PEBBLES[n] = (X, Y, 0.05 * O.bbox_diameter(X[:n]))
    return _PEBBLES[n]


def pose_errors(R, t, R_ref, t_ref):
    return O.rotation_angle(R @ R_ref.T), float(np.linalg.norm(t - t_ref))


def assert_pose(R, t, R_ref, t_ref, extent):
    dR, dt = pose_errors(R, t, R_ref, t_ref)
    assert dR <= 1e-4, f"rotation differs by {dR:.3e} rad"
    assert dt <= 1e-5 * extent, f"translation differs by {dt:.3e} m (extent {extent:.4f})"


@pytest.mark.parametrize("precision", ["f64", "f32"], indirect=True)
@pytest.mark.parametrize("case", ["c5_1m_fixed15", "c5_1m_conv", "p100k_fixed50", "p100k_conv"])
def test_rigid_pebble_config(fr, precision, case):
    g = load(case)
    n = int(g["n"])
    X, Y, sigma = pebble(n)
    assert sigma == float(g["sigma"])
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                                max_em_iters=int(g["max_iters"]),
                                twist_tolerance=float(g["tol"]))
    res = fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg)
    assert_pose(res.kinematics.pose.rotation, res.kinematics.pose.translation, g["R"], g["t"],
                O.bbox_diameter(X))
    assert abs(res.iterations - int(g["iterations"])) <= 1
    assert res.termination == str(g["termination"])
    k = min(len(res.objectives), len(g["objectives"])) - 1
    rtol = 1e-7 if precision == "f64" else 1e-5
    np.testing.assert_allclose(res.inlier_masses[:k], g["inlier_masses"][:k], rtol=rtol)
    np.testing.assert_allclose(res.objectives[:k], g["objectives"][:k], rtol=rtol)


@pytest.mark.parametrize("precision", ["f64", "f32"], indirect=True)
def test_c2_point_to_plane_100k(fr, precision):
    g = load("c2")
    ref = fr.PointCloud(g["X"].astype(np.float64), normals=g["N"].astype(np.float64))
    obs = fr.PointCloud(g["Y"].astype(np.float64), normals=g["YN"].astype(np.float64))
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=float(g["sigma"]), outlier_ratio=0.1),
                                residual_mode="point_to_plane", max_em_iters=int(g["max_iters"]),
                                twist_tolerance=1e-4,
                                mstep=fr.MStepOptions(max_gn_iters=int(g["max_gn_iters"])))
    res = fr.register(ref, obs, fr.RigidModel(), cfg)
    assert_pose(res.kinematics.pose.rotation, res.kinematics.pose.translation, g["R"], g["t"],
                O.bbox_diameter(ref.positions))
    assert abs(res.iterations - int(g["iterations"])) <= 1
    assert res.termination == str(g["termination"])


def test_c3_articulated_50k(fr):
    from .articulated_util import tree_from_arrays
    g = load("c3")
    tree = tree_from_arrays(fr, g)
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.006, outlier_ratio=0.1),
                                max_em_iters=15, twist_tolerance=1e-5)
    res = fr.register(fr.PointCloud(g["X"].astype(np.float64)),
                      fr.PointCloud(g["Y"].astype(np.float64)), tree, cfg)
    est = res.kinematics
    np.testing.assert_allclose(est.joint_values, g["joint_values"], atol=1e-4)
    extent = O.bbox_diameter(g["X"].astype(np.float64))
    assert_pose(est.base_pose.rotation, est.base_pose.translation, g["base_R"], g["base_t"],
                extent)
    assert abs(res.iterations - int(g["iterations"])) <= 1


def test_c4_nodegraph_100k(fr):
    from paper_1811_10136_b200.kinematics import NodeGraph, Skinning
    g = load("c4")
    graph = NodeGraph(g["nodes"], g["edges"], Skinning(g["skin_idx"], g["skin_w"]))
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.02, outlier_ratio=0.1),
                                max_em_iters=int(g["max_iters"]), twist_tolerance=1e-5,
                                mstep=fr.MStepOptions(lambda_reg=0.1))
    X = g["X"].astype(np.float64)
    res = fr.register(fr.PointCloud(X), fr.PointCloud(g["Y"].astype(np.float64)), graph, cfg)
    est = res.kinematics
    extent = O.bbox_diameter(X)
    worst_R = max(O.rotation_angle(a.rotation @ b.T)
                  for a, b in zip(est.node_transforms, g["node_R"]))
    worst_t = max(float(np.linalg.norm(a.translation - b))
                  for a, b in zip(est.node_transforms, g["node_t"]))
    assert worst_R <= 1e-4, worst_R
    assert worst_t <= 1e-5 * extent, worst_t
    assert abs(res.iterations - int(g["iterations"])) <= 1


def test_em64_matches_f32_statistics_at_scale(fr):
    """At the 16.8M-point bench workload (no CPU oracle at that size) the
    float32 fused pass's 25 statistics agree with the float64 pass's at the
    same pose to 1e-5 of each column's natural scale; the float64 pass is the
    one pinned to the reference above."""
    import torch
    from paper_1811_10136_b200 import _rigid
    model, obs, _ = O.pebble_pair(16_000_000, outlier_ratio=0.05, seed=0)
    X = model.astype(np.float32).astype(np.float64)
    Y = obs.astype(np.float32).astype(np.float64)
    sigma = 0.05 * O.bbox_diameter(X[:16_000_000])
    gmm = fr.GmmConfig(sigma=sigma, outlier_ratio=0.1)
    cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=4, twist_tolerance=1e-30)
    p64 = _rigid.RigidDevicePath(fr.PointCloud(X), fr.PointCloud(Y), gmm, "point_to_point",
                                 precision="f64")
    em = _rigid.DeviceEM64(p64, np.eye(3), np.zeros(3), cfg)
    em.pass_only()
    torch.cuda.synchronize()
    s64 = em.sums.cpu().numpy().copy()
    p32 = _rigid.RigidDevicePath(fr.PointCloud(X), fr.PointCloud(Y), gmm, "point_to_point",
                                 precision="f32")
    s32 = p32.run_pass(np.eye(3), np.zeros(3))[:25]
    mass = s64[0]
    rad = O.bbox_diameter(X) / 2
    scale = np.array([mass] + [mass * rad] * 3 + [mass * rad ** 2] * 6 + [mass * sigma] * 3
                     + [mass * rad * sigma] * 9 + [mass * sigma ** 2] * 3)
    assert np.all(np.abs(s32 - s64) <= 1e-5 * scale), np.max(np.abs(s32 - s64) / scale)


@pytest.mark.parametrize("precision", ["f64", "f32"], indirect=True)
def test_point_to_plane_extra_gauss_newton(fr, precision):
    """max_gn_iters = 3 point-to-plane (mstep.py:421-459: re-assembly at the
    accepted pose with the E step's spec): the float64 device loop and the
    host-driven float32 loop against the live reference."""
    g = load("gn3_pt2pl")
    ref = fr.PointCloud(g["X"].astype(np.float64), normals=g["N"].astype(np.float64))
    obs = fr.PointCloud(g["Y"].astype(np.float64), normals=g["YN"].astype(np.float64))
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=float(g["sigma"]), outlier_ratio=0.1),
                                residual_mode="point_to_plane", max_em_iters=int(g["max_iters"]),
                                twist_tolerance=1e-4,
                                mstep=fr.MStepOptions(max_gn_iters=int(g["max_gn_iters"])))
    res = fr.register(ref, obs, fr.RigidModel(), cfg)
    assert_pose(res.kinematics.pose.rotation, res.kinematics.pose.translation, g["R"], g["t"],
                O.bbox_diameter(ref.positions))
    assert abs(res.iterations - int(g["iterations"])) <= 1
    k = min(len(res.objectives), len(g["objectives"])) - 1
    np.testing.assert_allclose(res.objectives[:k], g["objectives"][:k],
                               rtol=1e-7 if precision == "f64" else 1e-4)


@pytest.mark.parametrize("precision", ["f64", "f32"], indirect=True)
def test_sigma_ladder_protocol(fr, precision):
    """The reference bench's coarse-to-fine width ladder (bench.py:66-110) on a
    corrupted pebble trial (10k + 20 % outliers), warm-started rungs with a
    lattice rebuild per rung, against the live reference's per-rung traces."""
    g = load("ladder_p10k")
    n, seed = int(g["n"]), int(g["seed"])
    model, obs, _ = O.pebble_pair(n, rotation_degrees=50.0, translation_fraction=0.02,
                                  outlier_ratio=float(g["outlier_ratio"]), seed=seed)
    X = model.astype(np.float32).astype(np.float64)
    Y = obs.astype(np.float32).astype(np.float64)
    diameter = float(g["diameter"])
    assert abs(O.bbox_diameter(X[:n]) - diameter) <= 1e-15 * diameter
    rungs = fr.filterreg_protocol(True, diameter, outliers=True)
    assert [c for _, c, _ in rungs] == list(g["caps"])
    out = fr.register_ladder(fr.PointCloud(X), fr.PointCloud(Y), rungs)
    extent = O.bbox_diameter(X)
    for k, res in enumerate(out):
        assert abs(res.iterations - int(g["rung_iterations"][k])) <= 1, k
        assert res.termination == str(g["rung_terminations"][k])
        assert_pose(res.kinematics.pose.rotation, res.kinematics.pose.translation,
                    g["rung_R"][k], g["rung_t"][k], extent)
    full = fr.ladder_result(out)
    k = min(len(full.objectives), len(g["objectives"]))
    np.testing.assert_allclose(full.objectives[:k][:60], g["objectives"][:k][:60],
                               rtol=1e-7 if precision == "f64" else 1e-4)
