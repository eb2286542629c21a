"""Phase timing of the registration setup (H2D, Morton sort, splat, blur) --
diagnostic for the e2e path; run on the GPU box."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import filterreg_oracle as O
import paper_1811_10136_b200 as fr
from paper_1811_10136_b200 import _lib
from paper_1811_10136_b200.permutohedral import PermutohedralLattice

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_000_000
t = time.perf_counter()
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float); Y = obs.astype(np.float32).astype(float)
print(f"generate {time.perf_counter()-t:.2f}s"); sigma = 0.05 * O.bbox_diameter(X[:n])
lib = _lib.load(); dev = _lib.device()
def tick(msg, t0):
    torch.cuda.synchronize(); print(f"{msg:28s} {1e3*(time.perf_counter()-t0):9.1f} ms", flush=True); return time.perf_counter()
for rep in range(2):
    t0 = time.perf_counter()
    a = np.ascontiguousarray(Y.T, dtype=np.float32); t0 = tick("numpy soa", t0)
    d = torch.from_numpy(a).to(dev); t0 = tick("h2d (pageable)", t0)
    pa = torch.from_numpy(a).pin_memory(); t0 = tick("pin", t0)
    d2 = pa.to(dev, non_blocking=True); t0 = tick("h2d (pinned)", t0)
    lat = PermutohedralLattice(3, sigma); t0 = tick("create", t0)
    lat.splat_points(d, None, 0); t0 = tick("splat", t0)
    lat.blur(); t0 = tick("blur", t0)
    lib.fr_sort_points_morton(_lib.ptr(d2), d2.shape[1], 3, None, _lib.stream_handle()); t0 = tick("morton", t0)
    P = X; tot = P.sum(axis=0); lo = P.min(axis=0); hi = P.max(axis=0); t0 = tick("host stats", t0)
