"""Timeline of the rigid device-path setup at 16.8M + 16.8M points: host
timestamps (FR_PROFILE_SETUP=2, no device syncs) of the model side (main
thread) and the observation side (worker thread), plus the EM object."""
import os
import sys
import time

import numpy as np
import torch

os.environ["FR_PROFILE_SETUP"] = "2"
sys.path.insert(0, ".")
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402
from paper_1811_10136_b200._rigid import DeviceEM, RigidDevicePath  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
gmm = fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:n]), outlier_ratio=0.1)
cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=200, twist_tolerance=1e-30)
ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    path = RigidDevicePath(ref, ob, gmm, "point_to_point")
    t1 = time.perf_counter()
    em = DeviceEM(path, np.eye(3), np.zeros(3), cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    em.run()
    em.result()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    ph = sorted(path.setup_s.items(), key=lambda kv: kv[1])
    print(f"rep {rep}: path {1e3 * (t1 - t0):.1f} ms, em create {1e3 * (t2 - t1):.1f} ms, "
          f"run {1e3 * (t3 - t2):.1f} ms | " + ", ".join(f"{k} {1e3 * v:.1f}" for k, v in ph),
          flush=True)
    del em, path
