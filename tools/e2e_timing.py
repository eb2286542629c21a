"""Wall-clock breakdown of the end-to-end register() call (the bench's e2e
number): repeated calls plus a cProfile of the host side.  Run on the GPU box:
    python tools/e2e_timing.py [points] [iters]"""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic tool, not the product)
import paper_1811_10136_b200 as fr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
sigma = 0.05 * O.bbox_diameter(X[:n])
gmm = fr.GmmConfig(sigma=sigma, outlier_ratio=0.1)
cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=iters, twist_tolerance=1e-30)
torch.cuda.init()
fr.register(fr.PointCloud(X[:2000]), fr.PointCloud(Y[:2000]), fr.RigidModel(), cfg)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg)
    torch.cuda.synchronize()
    print(f"register #{rep}: {time.perf_counter() - t0:.3f} s, {res.iterations} iters", flush=True)
pr = cProfile.Profile()
pr.enable()
res = fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
