"""Probe: fr_upload_points throughput at 16.8M points (host float64 rows ->
device float32 planes), one upload and two concurrent uploads."""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1811_10136_b200 import _lib  # noqa: E402

lib = _lib.load()
n = 16_800_000
a = np.random.default_rng(0).random((n, 3))
b = np.random.default_rng(1).random((n, 3))
da = torch.empty((3, n), dtype=torch.float32, device="cuda")
db = torch.empty((3, n), dtype=torch.float32, device="cuda")


def up(x, d):
    _lib.check(lib.fr_upload_points(x.ctypes.data, n, d.data_ptr(), _lib.stream_handle()))


for rep in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    up(a, da)
    torch.cuda.synchronize()
    t1 = time.perf_counter() - t
    t = time.perf_counter()
    th = threading.Thread(target=up, args=(b, db))
    th.start()
    up(a, da)
    th.join()
    torch.cuda.synchronize()
    t2 = time.perf_counter() - t
    print(f"one upload {1e3 * t1:.1f} ms, two concurrent {1e3 * t2:.1f} ms", flush=True)
assert np.array_equal(da.cpu().numpy(), a.T.astype(np.float32))
print("bit-exact vs numpy astype")
