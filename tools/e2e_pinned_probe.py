"""Median wall time of register() from pinned host clouds (the bench's e2e
call: 50 iterations, tolerance off) at the given sizes, interleaving the
chunked float64 observation splat (fr_lattice_splat_rows64) on and off
(diagnostic A/B)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402
from paper_1811_10136_b200 import _rigid  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [1_000_000]:
    model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    gmm = fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:n]), outlier_ratio=0.1)
    iters = int(os.environ.get("ITERS", "50"))
    cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=iters, twist_tolerance=1e-30)
    a, b = fr.pinned_cloud(fr.PointCloud(X)), fr.pinned_cloud(fr.PointCloud(Y))
    ts = {True: [], False: []}
    R = {}
    for rep in range(33):
        flag = rep % 2 == 0
        _rigid.CHUNKED_F64_SPLAT = flag
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = fr.register(a, b, fr.RigidModel(), cfg)
        torch.cuda.synchronize()
        if rep >= 3:
            ts[flag].append(time.perf_counter() - t0)
        R[flag] = res.kinematics.pose.matrix()
    print(f"{len(X)} pinned e2e register ({iters} iterations): chunked {1e3 * np.median(ts[True]):.3f} ms, "
          f"one copy {1e3 * np.median(ts[False]):.3f} ms; pose max diff "
          f"{np.abs(R[True] - R[False]).max():.2e}", flush=True)
