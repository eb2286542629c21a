"""Phase times of the float64 register() path at C5 sizes (FR_PROFILE_SETUP=1:
device-synchronised phases of RigidDevicePath; FR_SPLAT_TIMING=1: the splat's
own phases on stderr), then the EM object, the loop and the result read.

    python tools/setup64_profile.py [points] [--pinned]
"""
import os
import sys
import time

import numpy as np
import torch

os.environ.setdefault("FR_PROFILE_SETUP", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402
from paper_1811_10136_b200 import _rigid  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(args[0]) if args else 1_000_000
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
gmm = fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:n]), outlier_ratio=0.1)
cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=50, twist_tolerance=1e-30)
ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
if "--pinned" in sys.argv:
    ref, ob = fr.pinned_cloud(ref), fr.pinned_cloud(ob)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    path = _rigid.RigidDevicePath(ref, ob, gmm, "point_to_point", precision="f64")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    em = _rigid.device_em(path, np.eye(3), np.zeros(3), cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    em.run()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    em.result()
    t4 = time.perf_counter()
    ph = path.setup_s
    print(f"rep {rep}: path {1e3 * (t1 - t0):.2f} ms, em create {1e3 * (t2 - t1):.2f} ms, "
          f"run {1e3 * (t3 - t2):.2f} ms, result {1e3 * (t4 - t3):.2f} ms | "
          + ", ".join(f"{k} {1e3 * v:.2f}" for k, v in ph.items()), flush=True)
    del em, path
