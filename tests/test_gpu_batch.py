"""The batched multi-problem driver (register_batch):
concurrent registrations on separate streams give exactly the results of
running each problem alone."""

import numpy as np
import pytest

from oracle import filterreg_oracle as O

pytestmark = pytest.mark.gpu


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
        assert np.array_equal(a.kinematics.pose.matrix(), b.kinematics.pose.matrix())
        assert a.iterations == b.iterations and a.termination == b.termination
        assert a.objectives == b.objectives


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
