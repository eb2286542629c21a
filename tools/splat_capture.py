"""A fixed launch sequence for ncu captures of the splat kernels at C5 1M
(diagnostic): the first build of register() (k_splat_entries, caller order)
and sigma-re-estimating rebuilds (k_splat_warp_pairs on the Morton copy).
FR_SPLAT_TIMING=1 prints the hash table's occupancy (sites / slots)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
s = 0.05 * O.bbox_diameter(X[:n])
ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
fr.register(ref, ob, fr.RigidModel(),
            fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=s, outlier_ratio=0.1), max_em_iters=3,
                                  twist_tolerance=1e-30))
fr.register(ref, ob, fr.RigidModel(),
            fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=s, outlier_ratio=0.1, update_sigma=True),
                                  max_em_iters=3, twist_tolerance=1e-30))
torch.cuda.synchronize()
print("done")
