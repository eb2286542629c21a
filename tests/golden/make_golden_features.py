"""Golden fixtures for feature / concatenated correspondences (lattice
dimensions 4..12) from the LIVE reference package.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_features.py

Features are smooth colours of the model-frame position (outliers get random
colours), so an observation point carries the colour of the model point it was
transformed from.  All inputs are rounded to float32 first.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

import twistreg as T  # noqa: E402

from make_golden import f32, lattice_fixture  # noqa: E402


def colours(P, k, diam, rng, n_clean):
    """k smooth channels of the model-frame position; random for outliers."""
    w = np.array([[1.0, 0.3, -0.2], [-0.4, 1.0, 0.5], [0.2, -0.6, 1.0]] * ((k + 2) // 3))[:k]
    C = 0.5 + 0.5 * np.sin(2.0 * np.pi * (P @ w.T) / (0.6 * diam) + np.arange(k))
    C[n_clean:] = rng.uniform(0.0, 1.0, (len(P) - n_clean, k))
    return C


def pair(n, seed, k):
    m, o, gt = T.synthesize_pair(T.ExperimentSpec(source="pebble", n_points=n,
                                                  outlier_ratio=0.05, seed=seed))
    X, Y = f32(m.positions), f32(o.positions)
    diam = float(np.linalg.norm(X[:n].max(0) - X[:n].min(0)))
    rng = np.random.default_rng(seed + 100)
    CX = f32(colours(X, k, diam, rng, n))
    # observation point i (clean) is gt(model point i): same colour
    CY = CX.copy()
    CY[n:] = f32(rng.uniform(0.0, 1.0, (len(Y) - n, k)))
    return X, Y, CX, CY, diam, gt


def main():
    meta = {}
    # concatenated d = 4 (positions + 1 channel), values [1, y]
    X, Y, CX, CY, diam, _ = pair(3000, 1, 1)
    s = 0.05 * diam
    F = np.hstack([Y, CY])
    V = np.hstack([np.ones((len(Y), 1)), Y])
    lattice_fixture("lattice_feat_d4", F, V, np.array([s, s, s, 0.2]), np.hstack([X, CX]))
    meta["lattice_feat_d4"] = {"mode": "concatenated", "n_obs": len(Y)}
    # concatenated d = 6 (positions + rgb)
    X, Y, CX, CY, diam, _ = pair(1000, 2, 3)
    s = 0.05 * diam
    lattice_fixture("lattice_feat_d6", np.hstack([Y, CY]),
                    np.hstack([np.ones((len(Y), 1)), Y]),
                    np.array([s, s, s, 0.15, 0.15, 0.15]), np.hstack([X, CX]))
    meta["lattice_feat_d6"] = {"mode": "concatenated", "n_obs": len(Y)}
    # feature-only d = 5
    X, Y, CX, CY, diam, _ = pair(1500, 3, 5)
    lattice_fixture("lattice_feat_d5", CY, np.hstack([np.ones((len(Y), 1)), Y]),
                    np.full(5, 0.2), CX)
    meta["lattice_feat_d5"] = {"mode": "feature", "n_obs": len(Y)}
    # concatenated d = 12 (positions + 9 channels), small
    X, Y, CX, CY, diam, _ = pair(250, 4, 9)
    s = 0.08 * diam
    lattice_fixture("lattice_feat_d12", np.hstack([Y, CY]),
                    np.hstack([np.ones((len(Y), 1)), Y]),
                    np.array([s, s, s] + [0.3] * 9), np.hstack([X, CX]))
    meta["lattice_feat_d12"] = {"mode": "concatenated", "n_obs": len(Y)}

    # registrations
    for name, mode, k, seed, n in [("register_concat_d6", "concatenated", 3, 5, 2000),
                                   ("register_feature_d3", "feature", 3, 6, 2000)]:
        X, Y, CX, CY, diam, gt = pair(n, seed, k)
        sigma = 0.05 * diam
        gmm = T.GmmConfig(sigma=sigma, outlier_ratio=0.1, mode=mode, feature_sigma=0.15)
        cfg = T.RegistrationConfig(gmm=gmm, max_em_iters=40, twist_tolerance=1e-4)
        res = T.register(T.PointCloud(X, features=CX), T.PointCloud(Y, features=CY),
                         T.RigidModel(T.RigidTransform.identity()), cfg)
        pose = res.kinematics.pose
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"), X=X, Y=Y, CX=CX, CY=CY,
            config=json.dumps({"sigma": sigma, "w": 0.1, "mode": mode, "feature_sigma": 0.15,
                               "max_iters": 40, "tol": 1e-4}),
            R=pose.rotation, t=pose.translation, iterations=res.iterations,
            termination=res.termination, objectives=np.array(res.objectives),
            twist_norms=np.array(res.twist_norms), inlier_masses=np.array(res.inlier_masses),
            R_gt=gt.rotation, t_gt=gt.translation)
        meta[name] = {"mode": mode, "iterations": res.iterations,
                      "termination": res.termination,
                      "err_vs_gt_deg": float(np.degrees(np.arccos(np.clip(
                          (np.trace(pose.rotation.T @ gt.rotation) - 1) / 2, -1, 1))))}
    with open(os.path.join(HERE, "MANIFEST_features.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
