"""Diagnostic: per-column error of the float32 pass vs the exact pass."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import filterreg_oracle as O
import paper_1811_10136_b200 as fr
import paper_1811_10136_b200._rigid as rg
np.set_printoptions(linewidth=200, precision=3)
model, obs, _ = O.pebble_pair(30000, outlier_ratio=0.05, seed=11)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
far = np.random.default_rng(3).uniform(-5.0, 5.0, (2000, 3))
X = np.vstack([X, far]) if "far" in sys.argv else X
sigma = 0.05 * O.bbox_diameter(X[:30000])
path = rg.RigidDevicePath(fr.PointCloud(X), fr.PointCloud(Y), fr.GmmConfig(sigma=sigma, outlier_ratio=0.1), "point_to_point")
print("dense cells", path.lattice.dense_cells, "sites", path.lattice.num_sites)
L = float(np.sqrt(((X[:30000] - X[:30000].mean(axis=0)) ** 2).sum(axis=1).mean()))
k = np.array([0, 1, 1, 1, 2, 2, 2, 2, 2, 2, 1, 1, 1] + [2] * 9 + [2, 2, 2])
for R, t in [(np.eye(3), np.zeros(3)),
             (O.rotation_about_axis([0.3, -1.0, 0.5], 0.4), np.array([0.03, -0.05, 0.02])),
             (O.rotation_about_axis([1.0, 1.0, 0.0], 2.5), np.array([0.2, 0.1, -0.1]))]:
    rg.FAST_QUERY, rg.F32_POINTS = False, False
    ex = path.run_pass(R, t).copy()
    rg.FAST_QUERY, rg.F32_POINTS = True, False
    fa = path.run_pass(R, t).copy()
    rg.FAST_QUERY, rg.F32_POINTS = True, True
    f32 = path.run_pass(R, t).copy()
    print("exact", ex[:25])
    print("fast err", (np.abs(fa - ex) / (ex[0] * L ** k))[:25])
    print("f32 err ", (np.abs(f32 - ex) / (ex[0] * L ** k))[:25])
