"""Registration wall time with and without the observation-side setup overlap
(SETUP_OVERLAP_MIN) at 2k / 10k / 100k points (diagnostic)."""
import sys, time, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from oracle import filterreg_oracle as O
import paper_1811_10136_b200 as fr
from paper_1811_10136_b200 import _rigid
for thr in (400_000, 0):
    _rigid.SETUP_OVERLAP_MIN = thr
    for n in (2000, 10000, 100000):
        model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
        X = model.astype(np.float32).astype(float); Y = obs.astype(np.float32).astype(float)
        s = 0.05 * O.bbox_diameter(X[:n])
        cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=s, outlier_ratio=0.1), max_em_iters=250, twist_tolerance=2e-4)
        a, b = fr.PointCloud(X), fr.PointCloud(Y)
        for _ in range(3): fr.register(a, b, fr.RigidModel(), cfg)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            t0 = time.perf_counter(); r = fr.register(a, b, fr.RigidModel(), cfg); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        print(thr, n, r.iterations, "median %.3f ms" % (1e3 * np.median(ts)))
