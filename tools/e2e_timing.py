"""Wall-clock breakdown of the end-to-end register() call (the bench's e2e
number): repeated calls plus a cProfile of the host side.  Run on the GPU box:
    python tools/e2e_timing.py [points] [iters]"""
import cProfile
import gc
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
    t0 = time.perf_counter()
    ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    res = fr.register(ref, ob, fr.RigidModel(), cfg)
    torch.cuda.synchronize()
    print(f"PointCloud x2 {t1 - t0:.3f} s; register #{rep}: {time.perf_counter() - t1:.3f} s, "
          f"{res.iterations} iters", flush=True)
from paper_1811_10136_b200._rigid import DeviceEM, RigidDevicePath  # noqa: E402
for rep in range(8):
    ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    path = RigidDevicePath(ref, ob, gmm, "point_to_point")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print({k: round(v, 3) for k, v in path.setup_s.items()}, flush=True)
    em = DeviceEM(path, np.eye(3), np.zeros(3), cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    em.run()
    em.result()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    del em
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    del path
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    gc.collect()
    t6 = time.perf_counter()
    print(f"phases #{rep}: path {t1 - t0:.3f} s, em create {t2 - t1:.3f} s, em run {t3 - t2:.3f} s, "
          f"del em {t4 - t3:.3f} s, del path {t5 - t4:.3f} s, gc {t6 - t5:.3f} s", flush=True)
from paper_1811_10136_b200._rigid import upload_soa  # noqa: E402
from paper_1811_10136_b200.permutohedral import PermutohedralLattice  # noqa: E402
dev = torch.device("cuda", 0)


def lap(t):
    torch.cuda.synchronize()
    return time.perf_counter() - t


for rep in range(5):
    t = time.perf_counter()
    a = upload_soa(X, dev)
    b = upload_soa(Y, dev)
    up = lap(t)
    t = time.perf_counter()
    lat = PermutohedralLattice(3, sigma)
    lat.splat_points(b, None, 0)
    sp = lap(t)
    t = time.perf_counter()
    lat.blur()
    bl = lap(t)
    t = time.perf_counter()
    del lat
    de = lap(t)
    t = time.perf_counter()
    del a, b
    fr_ = lap(t)
    print(f"build #{rep}: upload {up:.3f} splat {sp:.3f} blur {bl:.3f} destroy {de:.3f} "
          f"free {fr_:.3f}", flush=True)
pr = cProfile.Profile()
pr.enable()
res = fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
