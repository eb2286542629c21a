"""The tiled device EM loop (clouds above FR_PERSIST_MAX points: centred
1024-point tiles, pass constants in the constant bank, one kernel per
iteration whose last block reduces and solves -- fr_rigid.cu
k_rigid_pass_tiles) against the host-driven loop (pipeline.py:141-181 order,
k_rigid_pass_grid4 passes) and against the oracle's registration."""
import json

import numpy as np
import pytest

from oracle import filterreg_oracle as O
from tests.angles import angle_between

from .test_gpu_register import LOOP_TOL, assert_pose_parity, load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fr():
    import paper_1811_10136_b200 as fr
    return fr


def _loops(fr, X, Y, sigma, w, iters, tol):
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=w),
                                max_em_iters=iters, twist_tolerance=tol)
    ref, obs = fr.PointCloud(X), fr.PointCloud(Y)
    dev = fr.register(ref, obs, fr.RigidModel(), cfg)
    host = fr.register(ref, obs, fr.RigidModel(), fr.RegistrationConfig(
        gmm=cfg.gmm, max_em_iters=iters, twist_tolerance=tol, record_states=True))
    return dev, host


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("seed", [0, 1])
def test_tiled_loop_golden(fr, seed, fused, monkeypatch):
    """Golden traces through the tiled loop (persistent kernel disabled), with
    the fused tail and with the separate solver kernel: the host loop's
    decisions and the live reference's pose."""
    monkeypatch.setenv("FR_PERSIST_MAX", "0")
    monkeypatch.setenv("FR_EM_FUSED", fused)
    g = load(f"register_pt2pt_seed{seed}")
    cfg = json.loads(str(g["config"]))
    dev, host = _loops(fr, g["X"], g["Y"], cfg["sigma"], cfg["w"], cfg["max_iters"], cfg["tol"])
    tol = LOOP_TOL["f32"]
    assert dev.iterations == host.iterations and dev.termination == host.termination
    assert angle_between(dev.kinematics.pose.rotation, host.kinematics.pose.rotation) < tol
    # objectives: float32 statistics folded every 64 points on the device vs
    # the host loop's pass -- the point order (Morton cells) moves them by ~1e-6
    np.testing.assert_allclose(dev.objectives, host.objectives, rtol=5 * tol)
    assert_pose_parity(dev.kinematics.pose.rotation, dev.kinematics.pose.translation,
                       g["R"], g["t"], O.bbox_diameter(g["X"]))


@pytest.mark.parametrize("m", [100_003, 1_000_000])
def test_tiled_loop_partial_tiles(fr, m):
    """Cloud sizes with a partial last tile (m % 1024 != 0, m % 4 != 0) and a
    million points: the tiled loop against the host loop, and the oracle's
    registration on the same inputs to the pose tolerances."""
    model, obs, _ = O.pebble_pair(m, outlier_ratio=0.05, seed=9)
    X = model.astype(np.float32).astype(float)[:m]
    Y = obs.astype(np.float32).astype(float)
    sigma = 0.05 * O.bbox_diameter(X)
    dev, host = _loops(fr, X, Y, sigma, 0.1, 12, 1e-12)
    assert dev.iterations == host.iterations == 12
    tol = LOOP_TOL["f32"]
    assert angle_between(dev.kinematics.pose.rotation, host.kinematics.pose.rotation) < tol
    np.testing.assert_allclose(dev.objectives, host.objectives, rtol=1e-5)
    if m <= 100_003:
        tr = O.register_rigid(X, Y, sigma=sigma, outlier_ratio=0.1, max_em_iters=12,
                              twist_tolerance=1e-12)
        assert_pose_parity(dev.kinematics.pose.rotation, dev.kinematics.pose.translation,
                           tr["R"], tr["t"], O.bbox_diameter(X))


def test_tiled_loop_deterministic(fr):
    """Bit-identical reruns of the tiled loop (fixed-order reductions)."""
    model, obs, _ = O.pebble_pair(200_000, outlier_ratio=0.05, seed=3)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:200_000]),
                                                 outlier_ratio=0.1),
                                max_em_iters=20, twist_tolerance=1e-12)
    a = fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg)
    b = fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg)
    assert np.array_equal(a.kinematics.pose.matrix(), b.kinematics.pose.matrix())
    assert a.objectives == b.objectives
