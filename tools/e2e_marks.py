"""Timeline of one end-to-end register() at 16.8M + 16.8M points (the bench's
e2e call): host timestamps around the phases of pipeline._register_device_loop."""
import os
import sys
import time

import numpy as np
import torch

os.environ["FR_PROFILE_SETUP"] = "2"
sys.path.insert(0, ".")
from oracle import filterreg_oracle as O  # noqa: E402  (diagnostic input generator)
import paper_1811_10136_b200 as fr  # noqa: E402
import paper_1811_10136_b200.pipeline as pl  # noqa: E402
import paper_1811_10136_b200._rigid as rg  # noqa: E402

n = 16_000_000
model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
X = model.astype(np.float32).astype(float)
Y = obs.astype(np.float32).astype(float)
gmm = fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:n]), outlier_ratio=0.1)
cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=200, twist_tolerance=1e-30)
ref, ob = fr.PointCloud(X), fr.PointCloud(Y)
marks = {}
T0 = [0.0]


def mark(name):
    marks[name] = 1e3 * (time.perf_counter() - T0[0])


orig_path_init = rg.RigidDevicePath.__init__
orig_em_init = rg.DeviceEM.__init__
orig_run = rg.DeviceEM.run
orig_result = rg.DeviceEM.result


def path_init(self, *a, **k):
    mark("path_start")
    orig_path_init(self, *a, **k)
    mark("path_done")
    print("   setup", {k: round(1e3 * v, 1) for k, v in sorted(self.setup_s.items(), key=lambda kv: kv[1])}, flush=True)


def em_init(self, *a, **k):
    orig_em_init(self, *a, **k)
    mark("em_created")


def run(self):
    orig_run(self)
    mark("em_run_returned")


def result(self):
    r = orig_result(self)
    mark("result_read")
    return r


rg.RigidDevicePath.__init__ = path_init
rg.DeviceEM.__init__ = em_init
rg.DeviceEM.run = run
rg.DeviceEM.result = result
for rep in range(4):
    marks.clear()
    torch.cuda.synchronize()
    T0[0] = time.perf_counter()
    res = fr.register(ref, ob, fr.RigidModel(), cfg)
    _ = res.kinematics.pose.matrix()
    torch.cuda.synchronize()
    mark("end")
    print(f"rep {rep}: " + ", ".join(f"{k} {v:.1f}" for k, v in marks.items()), flush=True)
