"""Fixed per-call cost of register(): one-iteration registrations at 2k / 20k /
1M points from pinned clouds, and a cProfile of 20 calls (diagnostic)."""
import sys, time, numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from oracle import filterreg_oracle as O
import paper_1811_10136_b200 as fr
for n in (2000, 20000, 1000000):
    model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
    X = model.astype(np.float32).astype(float); Y = obs.astype(np.float32).astype(float)
    s = 0.05 * O.bbox_diameter(X[:n])
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=s, outlier_ratio=0.1), max_em_iters=1, twist_tolerance=1e-30)
    a, b = fr.pinned_cloud(fr.PointCloud(X)), fr.pinned_cloud(fr.PointCloud(Y))
    for _ in range(3): fr.register(a, b, fr.RigidModel(), cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter(); r = fr.register(a, b, fr.RigidModel(), cfg); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(n, "1-iteration register: median %.3f ms" % (1e3 * np.median(ts)))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(20): fr.register(a, b, fr.RigidModel(), cfg)
torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
