"""cProfile of the sigma-re-estimating registration (host side of the per-
iteration lattice rebuild).   python tools/sigma_profile.py [points]"""
import cProfile
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import filterreg_oracle as O  # noqa: E402  (input generator)
import paper_1811_10136_b200 as fr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:n]), outlier_ratio=0.1,
                                             update_sigma=True),
                            max_em_iters=20, twist_tolerance=1e-30)
fr.register(ref, ob, fr.RigidModel(), cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
fr.register(ref, ob, fr.RigidModel(), cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
