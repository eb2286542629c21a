"""One float64 register() at C5 1M from pinned clouds (diagnostic: run under
ncu for the launch list / captures of the setup kernels)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
gmm = fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:n]), outlier_ratio=0.1)
cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=50, twist_tolerance=1e-30)
ref, ob = fr.pinned_cloud(fr.PointCloud(X)), fr.pinned_cloud(fr.PointCloud(Y))
for _ in range(reps):
    res = fr.register(ref, ob, fr.RigidModel(), cfg)
torch.cuda.synchronize()
print("iterations", res.iterations)
