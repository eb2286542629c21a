"""Diagnostic: per-iteration cost of the sigma re-estimating EM (host loop,
lattice rebuilt whenever sigma changes).  python tools/sigma_timing.py [points]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
diam = O.bbox_diameter(X[:n])
ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
for rep in range(3):
    timing = {}
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.05 * diam, outlier_ratio=0.1,
                                                 update_sigma=True),
                                max_em_iters=30, twist_tolerance=1e-30)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = fr.register(ref, ob, fr.RigidModel(), cfg, timing=timing)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {res.iterations} its in {dt:.3f} s = {1e3 * dt / res.iterations:.2f} ms/it, "
          f"timing {({k: round(v, 3) for k, v in timing.items()})}, sigma {res.sigmas[-1]:.5f}",
          flush=True)
