"""Device timeline of one float64 register() at C5 1M from pinned clouds
(diagnostic): torch.profiler (CUPTI) activity trace -> per-stream kernel and
memcpy intervals relative to the call's start, printed as a table."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
pinned = "--pageable" not in sys.argv
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
gmm = fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:n]), outlier_ratio=0.1)
cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=50, twist_tolerance=1e-30)
ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
if pinned:
    ref, ob = fr.pinned_cloud(ref), fr.pinned_cloud(ob)
for _ in range(3):
    fr.register(ref, ob, fr.RigidModel(), cfg)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    with torch.profiler.record_function("register"):
        fr.register(ref, ob, fr.RigidModel(), cfg)
    torch.cuda.synchronize()
path = os.path.join(ROOT, "gpurun_out", "timeline.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
t0 = min(e["ts"] for e in ev if e.get("name") == "register")
rows = []
for e in ev:
    cat = e.get("cat", "")
    if cat in ("kernel", "gpu_memcpy", "gpu_memset") or e.get("name") == "register":
        rows.append((e["ts"] - t0, e.get("dur", 0), e.get("args", {}).get("stream", "-"),
                     cat, e["name"][:70]))
rows.sort()
for r in rows:
    print(f"{r[0]:9.1f} {r[1]:8.1f}  s{r[2]!s:>4}  {r[3]:10s} {r[4]}")
