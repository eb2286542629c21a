"""Median wall time of register() from pinned host clouds (the bench's e2e
call: 50 iterations, tolerance off) at the given sizes (diagnostic A/B)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [1_000_000]:
    model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    gmm = fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:n]), outlier_ratio=0.1)
    cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=50, twist_tolerance=1e-30)
    a, b = fr.pinned_cloud(fr.PointCloud(X)), fr.pinned_cloud(fr.PointCloud(Y))
    for _ in range(3):
        fr.register(a, b, fr.RigidModel(), cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        t0 = time.perf_counter()
        fr.register(a, b, fr.RigidModel(), cfg)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{len(X)} pinned e2e register (50 iterations): median {1e3 * np.median(ts):.3f} ms",
          flush=True)
