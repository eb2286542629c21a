"""Timing probe of the float64 grid-resident EM loop (fr_em64) on the GPU box.

    python tools/em64_probe.py [points ...]

Per size: setup (upload, sort, lattice build), the pass alone (fr_em64_pass:
one cooperative launch, one iteration, no solve) and whole EM runs of 50
iterations (one launch), CUDA events on the launching stream."""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1811_10136_b200 as fr  # noqa: E402
from oracle import filterreg_oracle as O  # noqa: E402
from paper_1811_10136_b200 import _rigid  # noqa: E402


def ev_time(fn, reps):
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    sizes = [int(a) for a in sys.argv[1:]] or [100_000, 1_000_000]
    torch.cuda.set_device(0)
    for n in sizes:
        model, obs, _ = O.pebble_pair(n, outlier_ratio=0.05, seed=0)
        X = model.astype(np.float32).astype(np.float64)
        Y = obs.astype(np.float32).astype(np.float64)
        sigma = 0.05 * O.bbox_diameter(X[:n])
        gmm = fr.GmmConfig(sigma=sigma, outlier_ratio=0.1)
        _rigid.RigidDevicePath(fr.PointCloud(X), fr.PointCloud(Y), gmm, "point_to_point",
                               precision="f64")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        path = _rigid.RigidDevicePath(fr.PointCloud(X), fr.PointCloud(Y), gmm, "point_to_point",
                                      precision="f64")
        torch.cuda.synchronize()
        setup_ms = 1e3 * (time.perf_counter() - t0)
        iters = 50
        cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=10 ** 6, twist_tolerance=1e-30)
        em = _rigid.DeviceEM64(path, np.eye(3), np.zeros(3), cfg)
        pass_ms = ev_time(em.pass_only, 20)
        run_ms = ev_time(lambda: em.enqueue(iters), 5) / iters
        grid, block = em.launch_info()
        phases = None
        if os.environ.get("FR_EM64_PROFILE") == "1":
            import ctypes
            lib = path.lib
            fn = lib.fr_em64_profile
            fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
            em2 = _rigid.DeviceEM64(path, np.eye(3), np.zeros(3),
                                    fr.RegistrationConfig(gmm=gmm, max_em_iters=iters,
                                                          twist_tolerance=1e-30))
            em2.enqueue(iters)
            torch.cuda.synchronize()
            buf = np.zeros((iters, 8), dtype=np.uint64)
            from paper_1811_10136_b200 import _lib
            _lib.check(fn(em2.h, buf.ctypes.data, iters, _lib.stream_handle()))
            b = buf.astype(np.int64)[2:-1]
            phases = {"cta0_pass_us": float(np.median(b[:, 1] - b[:, 0])) / 1e3,
                      "barrier_wait_us": float(np.median(b[:, 2] - b[:, 1])) / 1e3,
                      "reduce_us": float(np.median(b[:, 3] - b[:, 2])) / 1e3,
                      "solve_us": float(np.median(b[:, 4] - b[:, 3])) / 1e3,
                      "solve_normal_eq_us": float(np.median(b[:, 5] - b[:, 3])) / 1e3,
                      "solve_chol_us": float(np.median(b[:, 6] - b[:, 5])) / 1e3,
                      "solve_halving_us": float(np.median(b[:, 7] - b[:, 6])) / 1e3,
                      "solve_update_us": float(np.median(b[:, 4] - b[:, 7])) / 1e3,
                      "next_start_us": float(np.median(buf.astype(np.int64)[3:, 0]
                                                       - buf.astype(np.int64)[2:-1, 4])) / 1e3}
        print(json.dumps({"points": len(X), "setup_ms": setup_ms, "pass_ms": pass_ms,
                          "iter_ms": run_ms, "pts_per_s": len(X) / (run_ms / 1e3),
                          "grid": grid, "block": block, "dense64": path.lattice.dense64,
                          "sites": path.lattice.num_sites, "phases": phases}), flush=True)


if __name__ == "__main__":
    main()
