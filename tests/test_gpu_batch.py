"""The batched multi-problem driver (register_batch):
every problem of one launch against the LIVE reference's golden traces, and
against running each problem alone (the float64 loop's reduction order depends
on the CTAs a problem gets, so the two agree to float64 round-off; the float32
cluster loop is bit-identical)."""

import json
import os

import numpy as np
import pytest

from oracle import filterreg_oracle as O

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_register_batch_against_reference_goldens():
    """The C1-scale live-reference traces (register_pt2pt_seed0..2) as one
    batch: north-star pose bars, iteration count, objectives."""
    import paper_1811_10136_b200 as fr
    probs, goldens = [], []
    for seed in range(3):
        g = np.load(os.path.join(GOLDEN, f"register_pt2pt_seed{seed}.npz"))
        cfg = json.loads(str(g["config"]))
        config = fr.RegistrationConfig(
            gmm=fr.GmmConfig(sigma=cfg["sigma"], outlier_ratio=cfg["w"]),
            max_em_iters=cfg["max_iters"], twist_tolerance=cfg["tol"])
        probs.append((fr.PointCloud(g["X"]), fr.PointCloud(g["Y"]), fr.RigidModel(), config))
        goldens.append(g)
    out = fr.register_batch(probs, max_concurrent=3)
    for res, g in zip(out, goldens):
        R, t = res.kinematics.pose.rotation, res.kinematics.pose.translation
        assert O.rotation_angle(R @ g["R"].T) <= 1e-4
        assert np.linalg.norm(t - g["t"]) <= 1e-5 * O.bbox_diameter(g["X"])
        assert abs(res.iterations - int(g["iterations"])) <= 1
        assert res.termination == str(g["termination"])
        n = min(len(res.objectives), len(g["objectives"])) - 1
        np.testing.assert_allclose(res.objectives[:n], g["objectives"][:n], rtol=1e-7)


def test_register_batch_equals_sequential():
    import paper_1811_10136_b200 as fr
    problems = []
    for seed in range(6):
        model, obs, _ = O.pebble_pair(3000 + 500 * seed, outlier_ratio=0.05, seed=seed)
        X = model.astype(np.float32).astype(float)
        Y = obs.astype(np.float32).astype(float)
        sigma = 0.05 * O.bbox_diameter(X[:3000])
        cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                                    max_em_iters=120, twist_tolerance=2e-4)
        problems.append((fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg))
    seq = [fr.register(*p) for p in problems]
    bat = fr.register_batch(problems, max_concurrent=4)
    assert len(bat) == len(seq)
    for a, b in zip(seq, bat):
        Ra, Rb = a.kinematics.pose.rotation, b.kinematics.pose.rotation
        # entrywise (acos resolves no angle below ~2e-8 near the identity)
        assert np.abs(Ra - Rb).max() < 1e-11
        assert np.linalg.norm(a.kinematics.pose.translation - b.kinematics.pose.translation) < 1e-12
        assert a.iterations == b.iterations and a.termination == b.termination
        np.testing.assert_allclose(a.objectives, b.objectives, rtol=1e-10)
    again = fr.register_batch(problems, max_concurrent=4)      # reruns: bit-identical
    for a, b in zip(bat, again):
        assert np.array_equal(a.kinematics.pose.matrix(), b.kinematics.pose.matrix())


def test_register_batch_mixed_models_and_empty():
    import paper_1811_10136_b200 as fr
    assert fr.register_batch([]) == []
    model, obs, _ = O.pebble_pair(2000, outlier_ratio=0.05, seed=3)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    sigma = 0.05 * O.bbox_diameter(X[:2000])
    base = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                                 max_em_iters=60, twist_tolerance=2e-4)
    sig = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=0.1,
                                                 update_sigma=True),
                                max_em_iters=30, twist_tolerance=2e-4)
    probs = [(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), base),
             (fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), sig)]
    out = fr.register_batch(probs, max_concurrent=2)
    ref = [fr.register(*p) for p in probs]
    for a, b in zip(out, ref):
        assert np.array_equal(a.kinematics.pose.matrix(), b.kinematics.pose.matrix())
        assert a.sigmas == b.sigmas
