"""The bench's CPU reference arm (oracle EM iteration sharded over worker
processes) follows the single-process oracle iteration (oracle.rigid_m_step):
same poses up to the float64 re-association of the shard sums."""

import numpy as np

from oracle import filterreg_oracle as O


def test_cpu_arm_matches_single_process_oracle():
    import bench
    model, obs, _ = O.pebble_pair(6000, outlier_ratio=0.05, seed=3)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    sigma = 0.05 * O.bbox_diameter(X[:6000])
    arm = bench.CpuArm(X, Y, sigma, workers=3)
    try:
        eng = O.OracleMoments(Y, sigma, 0.1)
        R, t = np.eye(3), np.zeros(3)
        sinv = np.full(3, 1.0 / sigma)
        for _ in range(3):
            arm.iteration()
            mom = eng.moments(X @ R.T + t)
            spec = (mom["weight"], mom["target"], sinv, "point_to_point", None, None)
            R, t, _ = O.rigid_m_step(spec, X, R, t)
            # shard sums re-associate float64 round-off, amplified through the EM map
            assert np.abs(arm.R - R).max() < 1e-7
            assert np.linalg.norm(arm.t - t) < 1e-8      # extent ~0.15 m
    finally:
        arm.close()
