"""Diagnostic: phases of the sigma-re-estimating EM's per-iteration lattice
rebuild (splat / blur wall time with device syncs, site counts).
python tools/sigma_phases.py [points] [iters]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402
from paper_1811_10136_b200 import permutohedral as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
diam = O.bbox_diameter(X[:n])
ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
log = []


def timed(name, fn):
    def w(self, *a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(self, *a, **k)
        torch.cuda.synchronize()
        log.append((name, 1e3 * (time.perf_counter() - t0)))
        return r
    return w


P.PermutohedralLattice.splat_points = timed("splat", P.PermutohedralLattice.splat_points)
P.PermutohedralLattice.blur = timed("blur", P.PermutohedralLattice.blur)
for rep in range(3):
    log.clear()
    timing = {}
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.05 * diam, outlier_ratio=0.1,
                                                 update_sigma=True),
                                max_em_iters=iters, twist_tolerance=1e-30)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = fr.register(ref, ob, fr.RigidModel(), cfg, timing=timing)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    sp = [round(v, 1) for k, v in log if k == "splat"]
    bl = [round(v, 1) for k, v in log if k == "blur"]
    print(f"rep {rep}: {res.iterations} its {1e3 * dt / res.iterations:.1f} ms/it; "
          f"timing {({k: round(v, 3) for k, v in timing.items()})}", flush=True)
    print("  splat ms", sp, flush=True)
    print("  blur ms ", bl, flush=True)
    print("  sigmas  ", [round(s, 5) for s in res.sigmas], flush=True)
