"""Diagnostic: host->device options for a (n, 3) float64 point cloud (the e2e
upload).  Run on the GPU box:  python tools/h2d_options.py [points]"""
import os
import sys
import time

import numpy as np
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16_800_000
X = np.random.default_rng(0).standard_normal((n, 3))
dev = torch.device("cuda", 0)
torch.ones(1, device=dev)
cud = torch.cuda.cudart()
print("cpu_count", os.cpu_count(), "sched", len(os.sched_getaffinity(0)), flush=True)


def t(label, fn, reps=3):
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        print(f"{label:34s} rep{r} {1e3 * (time.perf_counter() - t0):8.1f} ms", flush=True)


t("pageable f64 .to()", lambda: torch.from_numpy(X).to(dev))
t("host f32 astype + pageable", lambda: torch.from_numpy(X.astype(np.float32)).to(dev))


def registered():
    ptr, nbytes = X.ctypes.data, X.nbytes
    assert cud.cudaHostRegister(ptr, nbytes, 0) == 0
    d = torch.empty((n, 3), dtype=torch.float64, device=dev)
    d.copy_(torch.from_numpy(X), non_blocking=True)
    torch.cuda.synchronize()
    cud.cudaHostUnregister(ptr)


t("cudaHostRegister + DMA + unregister", registered)
pin = torch.empty((n, 3), dtype=torch.float64).pin_memory()


def staged():
    pin.numpy()[:] = X
    torch.empty((n, 3), dtype=torch.float64, device=dev).copy_(pin, non_blocking=True)


t("memcpy into pinned + DMA", staged)
t("DMA from pinned only", lambda: torch.empty((n, 3), dtype=torch.float64, device=dev).copy_(
    pin, non_blocking=True))
