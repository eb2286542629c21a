"""Probe: does a 16.8M-point fr_upload_points slow down while the GPU is busy
on another stream (pure device work) or while another thread runs a lattice
splat (device work + host syncs)?"""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import filterreg_oracle as O  # noqa: E402  (probe input generator)
import paper_1811_10136_b200 as fr  # noqa: E402
from paper_1811_10136_b200 import _lib  # noqa: E402
from paper_1811_10136_b200._rigid import upload_soa  # noqa: E402

lib = _lib.load()
n = 16_800_000
a = np.random.default_rng(0).random((n, 3))
d = torch.empty((3, n), dtype=torch.float32, device="cuda")
model, obs, _ = O.pebble_pair(16_000_000, outlier_ratio=0.05, seed=0)
Y = obs.astype(np.float32).astype(float)
sigma = 0.05 * O.bbox_diameter(model[:16_000_000])
side = torch.cuda.Stream()
with torch.cuda.stream(side):
    dobs = upload_soa(Y, torch.device("cuda"))
torch.cuda.synchronize()


def up():
    _lib.check(lib.fr_upload_points(a.ctypes.data, n, d.data_ptr(), _lib.stream_handle()))


def busy():
    x = torch.empty(1 << 29, device="cuda")
    with torch.cuda.stream(side):
        for _ in range(60):
            x.mul_(1.0001)


def splat():
    with torch.cuda.stream(side):
        lat = fr.PermutohedralLattice(3, np.full(3, sigma))
        lat.splat_points(dobs, None, 0)
        lat.blur()
        side.synchronize()


for name, job in [("idle", None), ("device-busy", busy), ("splat", splat)]:
    for rep in range(3):
        torch.cuda.synchronize()
        th = threading.Thread(target=job) if job else None
        if th:
            th.start()
            time.sleep(0.001)
        t = time.perf_counter()
        up()
        torch.cuda.synchronize() if not th else torch.cuda.current_stream().synchronize()
        dt = time.perf_counter() - t
        if th:
            th.join()
        torch.cuda.synchronize()
        print(f"{name}: upload {1e3 * dt:.1f} ms", flush=True)
