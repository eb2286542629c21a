"""Articulated registration on the GPU vs the live reference's golden traces
(tests/golden/make_golden_articulated.py): joint values and base pose after the
same EM iterations, objectives, termination."""
import json
import os

import numpy as np
import pytest

from oracle import filterreg_oracle as O

from .articulated_util import tree_from_arrays
from .conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fr():
    import paper_1811_10136_b200 as fr
    return fr


@pytest.mark.parametrize("case", ["two_link", "chain20", "chain6_pt2pl"])
@pytest.mark.parametrize("fast", [True, False])
def test_golden_articulated(fr, case, fast):
    import paper_1811_10136_b200._articulated as art
    g = np.load(os.path.join(GOLDEN, f"articulated_{case}.npz"))
    cfg = json.loads(str(g["config"]))
    rest = tree_from_arrays(fr, g)
    pl = cfg["mode"] == "point_to_plane"
    ref = fr.PointCloud(g["X"], normals=g["N"] if pl else None)
    obs = fr.PointCloud(g["Y"], normals=g["YN"] if pl else None)
    config = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=cfg["sigma"], outlier_ratio=cfg["w"]),
                                   residual_mode=cfg["mode"], max_em_iters=cfg["max_iters"],
                                   twist_tolerance=cfg["tol"])
    old = art.FAST_QUERY
    art.FAST_QUERY = fast
    try:
        res = fr.register(ref, obs, rest, config)
    finally:
        art.FAST_QUERY = old
    est = res.kinematics
    assert res.iterations == int(g["iterations"]) and res.termination == str(g["termination"])
    assert np.abs(est.joint_values - g["joint_values"]).max() <= 1e-4
    dR = O.rotation_angle(est.base_pose.rotation @ g["base_R"].T)
    assert dR <= 1e-4
    assert np.linalg.norm(est.base_pose.translation - g["base_t"]) <= 1e-5 * O.bbox_diameter(g["X"])
    np.testing.assert_allclose(res.objectives, g["objectives"], rtol=1e-4)


def test_articulated_assembly_matches_reference_math(fr):
    """Per-body statistics -> projected normal equations equal the dense
    per-point assembly of mstep.py:213-229 (oracle restatement)."""
    import paper_1811_10136_b200._articulated as art
    from paper_1811_10136_b200.kinematics import forward_points
    g = np.load(os.path.join(GOLDEN, "articulated_chain20.npz"))
    rest = tree_from_arrays(fr, g, joint_values=0.02 * np.ones(20))
    ref, obs = fr.PointCloud(g["X"]), fr.PointCloud(g["Y"])
    gmm = fr.GmmConfig(sigma=0.006, outlier_ratio=0.1)
    path = art.ArticulatedDevicePath(ref, obs, gmm, "point_to_point", rest)
    sums = path.run_body_pass(rest)
    # oracle: moments at the same positions, dense per-body assembly
    x = forward_points(ref, rest).positions
    eng = O.OracleMoments(g["Y"], 0.006, 0.1)
    mf = eng.moments(x)
    s = np.full(3, 1.0 / 0.006)
    H = np.zeros((rest.n_params, rest.n_params))
    b = np.zeros(rest.n_params)
    S = rest.spatial_velocity_jacobians()
    for k in range(rest.n_bodies):
        sel = rest.point_bodies == k
        spec = (mf["weight"][sel], mf["target"][sel], s, "point_to_point", None, None)
        Hk, gk = O.assemble_rigid(spec, x[sel])
        H += S[k].T @ Hk @ S[k]
        b += S[k].T @ gk
    from paper_1811_10136_b200._rigid import RigidMoments
    cents = path.centres(rest)
    Hd = np.zeros_like(H)
    bd = np.zeros_like(b)
    for k in range(rest.n_bodies):
        hk, gk = RigidMoments.from_sums(sums[k]).normal_equations(cents[k], s ** 2)
        Hd += S[k].T @ hk @ S[k]
        bd += S[k].T @ gk
    np.testing.assert_allclose(Hd, H, rtol=1e-5, atol=1e-6 * np.abs(H).max())
    np.testing.assert_allclose(bd, b, rtol=1e-4, atol=1e-5 * np.abs(b).max())


@pytest.mark.parametrize("case", ["two_link", "chain20"])
def test_device_loop_matches_host_loop(fr, case, monkeypatch):
    """The device-resident articulated M step (fr_art_em: forward kinematics,
    projection, Cholesky, closed-form halving in one CTA) reproduces the host
    loop over the same body pass: iterations, termination, joint values and
    base pose to round-off (the two forward kinematics differ in last bits,
    which the float32 ranks of the body pass can turn into a float32 ulp)."""
    from paper_1811_10136_b200 import pipeline
    g = np.load(os.path.join(GOLDEN, f"articulated_{case}.npz"))
    cfg = json.loads(str(g["config"]))
    config = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=cfg["sigma"], outlier_ratio=cfg["w"]),
                                   max_em_iters=cfg["max_iters"], twist_tolerance=cfg["tol"])
    ref, obs = fr.PointCloud(g["X"]), fr.PointCloud(g["Y"])
    dev = fr.register(ref, obs, tree_from_arrays(fr, g), config)
    monkeypatch.setattr(pipeline, "ARTICULATED_DEVICE_LOOP", False)
    host = fr.register(ref, obs, tree_from_arrays(fr, g), config)
    assert dev.iterations == host.iterations and dev.termination == host.termination
    assert np.abs(dev.kinematics.joint_values - host.kinematics.joint_values).max() < 1e-6
    dR = O.rotation_angle(dev.kinematics.base_pose.rotation @ host.kinematics.base_pose.rotation.T)
    assert dR < 1e-6
    np.testing.assert_allclose(dev.objectives, host.objectives, rtol=1e-6)
    np.testing.assert_allclose(dev.twist_norms, host.twist_norms, rtol=1e-4, atol=1e-6)


def test_device_loop_extra_gauss_newton(fr, monkeypatch):
    """max_gn_iters = 3 through the device M step (moved per-body statistics,
    re-projected system) equals the host loop."""
    from paper_1811_10136_b200 import pipeline
    g = np.load(os.path.join(GOLDEN, "articulated_chain20.npz"))
    cfg = json.loads(str(g["config"]))
    config = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=cfg["sigma"], outlier_ratio=cfg["w"]),
                                   max_em_iters=8, twist_tolerance=cfg["tol"],
                                   mstep=fr.MStepOptions(max_gn_iters=3))
    ref, obs = fr.PointCloud(g["X"]), fr.PointCloud(g["Y"])
    dev = fr.register(ref, obs, tree_from_arrays(fr, g), config)
    monkeypatch.setattr(pipeline, "ARTICULATED_DEVICE_LOOP", False)
    host = fr.register(ref, obs, tree_from_arrays(fr, g), config)
    assert dev.iterations == host.iterations
    assert np.abs(dev.kinematics.joint_values - host.kinematics.joint_values).max() < 1e-6
    np.testing.assert_allclose(dev.objectives, host.objectives, rtol=1e-6)


def test_point_to_plane_extra_gauss_newton_against_reference(fr):
    """Articulated point_to_plane with max_gn_iters = 3 (the explicit-spec
    m_step path) against the live reference."""
    g = np.load(os.path.join(GOLDEN, "config_gn3_chain6_pt2pl.npz"))
    rest = tree_from_arrays(fr, g)
    ref = fr.PointCloud(g["X"].astype(float), normals=g["N"].astype(float))
    obs = fr.PointCloud(g["Y"].astype(float), normals=g["YN"].astype(float))
    config = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.006, outlier_ratio=0.1),
                                   residual_mode="point_to_plane", max_em_iters=15,
                                   twist_tolerance=1e-5, mstep=fr.MStepOptions(max_gn_iters=3))
    res = fr.register(ref, obs, rest, config)
    assert abs(res.iterations - int(g["iterations"])) <= 1
    assert np.abs(res.kinematics.joint_values - g["joint_values"]).max() <= 1e-4
    dR = O.rotation_angle(res.kinematics.base_pose.rotation @ g["base_R"].T)
    assert dR <= 1e-4
