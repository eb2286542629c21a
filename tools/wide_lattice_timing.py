"""Diagnostic: build (splat + blur) and slice times of the d >= 4 lattice
(feature / concatenated kernels) at scale.   python tools/wide_lattice_timing.py"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1811_10136_b200 as fr  # noqa: E402
from oracle import filterreg_oracle as O  # noqa: E402  (input generator)

for n, d in ((200_000, 4), (1_000_000, 4), (1_000_000, 6), (200_000, 9), (100_000, 12)):
    P = O.pebble_resample(n, seed=1)
    rng = np.random.default_rng(0)
    C = 0.5 + 0.5 * np.sin(P @ rng.standard_normal((3, d - 3)) * 30.0)
    F = np.hstack([P, C])
    V = np.hstack([np.ones((n, 1)), P])
    diam = float(np.linalg.norm(P.max(0) - P.min(0)))
    sigma = np.array([0.05 * diam] * 3 + [0.15] * (d - 3))
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lat = fr.PermutohedralLattice(d, sigma)
        lat.splat(F, V)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        lat.blur()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        out = lat.slice(F[:100_000])
        torch.cuda.synchronize()
        t3 = time.perf_counter()
    print(f"n={n} d={d}: sites {lat.num_sites}, splat {1e3 * (t1 - t0):.1f} ms, "
          f"blur {1e3 * (t2 - t1):.1f} ms, slice(100k) {1e3 * (t3 - t2):.1f} ms, "
          f"mass>0 {np.mean(out[:, 0] > 0):.3f}", flush=True)
