"""FilterReg B200 benchmark: rigid point-to-point EM on the C5 workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--points P] [--impl b200|reference]

Workload (BASELINE.json configs[4], "large-scale rigid sweep", at the 1M point
of the metric "EM iters/sec & points/sec (100k/1M-pt rigid)"): the reference's
pebble pair (synth.py:252-284 restated in oracle/filterreg_oracle.py) with
P = 1,000,000 points per GPU plus 5% uniform outliers, 50 deg / 2% shift ground
truth, sigma = 5% of the clean bbox diagonal, w = 0.1.  Weak scaling: the job's
model cloud has N*P(1.05) points, sharded contiguously over the N ranks; every
rank builds the lattice of the whole observation cloud (once, outside the
timed region, reported as build_ms) and the per-iteration normal-equation
partials are NCCL all-reduced.

A step is ONE EM iteration over the whole job (fused E + assembly pass,
all-reduce, host GN solve + step halving).  The tolerance is 1e-30 so every
step does the full work.  Inputs are smaller than L2 at 1M points, so L2 is
flushed (256 MiB write) before every timed step, outside its events.

value = model points x timed EM iterations / device time (max over ranks).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "points/sec (model points x EM iterations / s, rigid point-to-point FilterReg)"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--points", type=int, default=1_000_000, help="clean points per GPU")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=262_144,
                    help="model points per CPU-baseline EM iteration")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_workload(points_per_gpu: int, world: int):
    """fp32-rounded pebble pair of world * points clean points (+5% outliers)."""
    from oracle import filterreg_oracle as O
    n = points_per_gpu * world
    model, obs, gt = O.pebble_pair(n, rotation_degrees=50.0, translation_fraction=0.02,
                                   outlier_ratio=0.05, seed=0)
    X = model.astype(np.float32).astype(np.float64)
    Y = obs.astype(np.float32).astype(np.float64)
    sigma = 0.05 * O.bbox_diameter(X[:n])
    return X, Y, sigma, gt


def shard(X, world, rank):
    bounds = np.linspace(0, len(X), world + 1).astype(np.int64)
    return X[bounds[rank]:bounds[rank + 1]]


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML every
    ~2 ms DURING the timed region (the same counters `nvidia-smi --query-gpu=
    clocks.sm,clocks_event_reasons.*` reads; the timed region is too short for
    nvidia-smi's 100 ms minimum period)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.rows.append((sm, rs))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self._thread = threading.Thread(target=poll, daemon=True)
            self._thread.start()
            self._ok = True
        except Exception:
            self._ok = False
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [r[0] for r in self.rows]
        reasons = sorted({n for _, rs in self.rows for n, bit in self.REASONS.items() if rs & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml"}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(points: int):
    """dram bytes per launch of the pass kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as fh:
            doc = json.load(fh)
        rec = doc.get("rigid_pass", {})
        if int(rec.get("points", -1)) == points:
            return float(rec["dram_bytes"])
    except Exception:
        pass
    return None


def cpu_baseline(X, Y, sigma, sample: int, iters: int):
    """The oracle port (oracle/filterreg_oracle.py) on host cores: lattice built
    on the full observation cloud (not timed), then `iters` EM iterations of the
    same registration over a `sample`-point subset of the model cloud."""
    from oracle import filterreg_oracle as O
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(len(X), min(sample, len(X)), replace=False))
    Xs = X[idx]
    eng = O.OracleMoments(Y, sigma, 0.1)
    R, t = np.eye(3), np.zeros(3)
    sinv = np.full(3, 1.0 / sigma)
    tick = time.perf_counter()
    for _ in range(iters):
        x = Xs @ R.T + t
        mom = eng.moments(x)
        spec = (mom["weight"], mom["target"], sinv, "point_to_point", None, None)
        R, t, _ = O.rigid_m_step(spec, Xs, R, t)
    dt = time.perf_counter() - tick
    return len(Xs) * iters / dt, dt, len(Xs)


def run_reference(args):
    """--impl reference: the reference algorithm's CPU path (oracle port; the
    Python reference itself cannot travel to the GPU box) on this box's cores."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    X, Y, sigma, _ = make_workload(args.points, world)
    from oracle import filterreg_oracle as O
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(len(X), min(args.cpu_sample, len(X)), replace=False))
    Xs = X[idx]
    tick = time.perf_counter()
    eng = O.OracleMoments(Y, sigma, 0.1)
    build_s = time.perf_counter() - tick
    R, t = np.eye(3), np.zeros(3)
    sinv = np.full(3, 1.0 / sigma)
    times = []
    for i in range(args.warmup + args.steps):
        tick = time.perf_counter()
        x = Xs @ R.T + t
        mom = eng.moments(x)
        spec = (mom["weight"], mom["target"], sinv, "point_to_point", None, None)
        R, t, _ = O.rigid_m_step(spec, Xs, R, t)
        if i >= args.warmup:
            times.append(time.perf_counter() - tick)
    total = sum(times)
    value = len(Xs) * args.steps / total
    cores = 1
    sample = (f"{len(Xs)}-point random subset of the {len(X)}-point model cloud per EM "
              f"iteration; lattice on all {len(Y)} observation points (build {build_s:.1f} s)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C5 rigid pt2pt pebble, {args.points} clean pts/GPU + 5% "
                               "outliers (CPU arm: bounded sample)",
                   "points_per_gpu": len(X) // world, "sigma_frac": 0.05,
                   "outlier_ratio": 0.1, "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def run_b200(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    group = None
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    import paper_1811_10136_b200 as fr
    from paper_1811_10136_b200._rigid import RigidDevicePath
    from paper_1811_10136_b200.pipeline import _rigid_m_step

    X, Y, sigma, _ = make_workload(args.points, world)
    Xl = shard(X, world, rank)
    M_local, M_total, N_obs = len(Xl), len(X), len(Y)
    gmm = fr.GmmConfig(sigma=sigma, outlier_ratio=0.1)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    path = RigidDevicePath(fr.PointCloud(Xl), fr.PointCloud(Y), gmm, "point_to_point", group)
    torch.cuda.synchronize()
    build_ms = 1e3 * (time.perf_counter() - t0)
    sites = path.lattice.num_sites

    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    need_flush = 12 * M_local < 2 * L2_BYTES
    s2 = np.full(3, 1.0 / sigma ** 2)
    opts = fr.MStepOptions()
    R, t = np.eye(3), np.zeros(3)
    stream = torch.cuda.current_stream()

    def step(times=None):
        nonlocal R, t
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        sums_pass = _timed_pass(path, R, t, ev[1])
        cand, _ = _rigid_m_step(path, sums_pass, R, t, s2, opts)
        R, t = cand.pose.rotation, cand.pose.translation
        ev[2].record(stream)
        if times is not None:
            times.append(ev)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if need_flush:
                flush.zero_()
            step(times)
        torch.cuda.synchronize()
    if group is not None:
        dist.barrier()
    step_ms = [a.elapsed_time(c) for a, _, c in times]
    pass_ms = [a.elapsed_time(b) for a, b, _ in times]
    total_ms = float(sum(step_ms))
    tot = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if group is not None:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    total_ms = float(tot.item())
    value = M_total * args.steps / (total_ms / 1e3)

    # roofline of the dominant kernel: the fused pass reads 12 B per model point
    # (float32 x, y, z); the lattice table (< L2) is not counted
    pass_avg_ms = float(np.mean(pass_ms))
    alg_bytes = 12 * M_local
    achieved = alg_bytes / (pass_avg_ms / 1e3) / 1e9
    peak, peak_kind = measured_peak()
    traffic = ncu_traffic(args.points)

    # end to end through the public API: register() from host arrays, H2D of
    # both clouds, lattice build, K EM iterations, D2H of the pose
    e2e = None
    if not args.no_e2e:
        cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=args.steps, twist_tolerance=1e-30)
        ref_host = fr.PointCloud(Xl)
        obs_host = fr.PointCloud(Y)
        fr.register(ref_host, obs_host, fr.RigidModel(), fr.RegistrationConfig(
            gmm=gmm, max_em_iters=2, twist_tolerance=1e-30), process_group=group)
        torch.cuda.synchronize()
        if group is not None:
            dist.barrier()
        t0 = time.perf_counter()
        res = fr.register(ref_host, obs_host, fr.RigidModel(), cfg, process_group=group)
        _ = res.kinematics.pose.matrix()
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        et = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if group is not None:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_s = float(et.item())
        h2d = (12 * M_local + 12 * N_obs) / args.steps
        e2e = {"value": M_total * res.iterations / e2e_s, "unit": "points/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * path.width,
               "em_iterations": res.iterations, "wall_s": e2e_s,
               "includes": "H2D of model shard + observation cloud, lattice build, "
                           "EM iterations, D2H of sums/pose"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, ns = cpu_baseline(X, Y, sigma, args.cpu_sample, 4)
        cpu = {"value": v, "unit": "points/s", "cores": 1, "kind": "port",
               "sample": f"4 EM iterations over a {ns}-point subset of the model cloud, "
                         f"lattice on all {N_obs} observation points ({dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"C5 rigid pt2pt pebble, {args.points} clean pts/GPU + 5% "
                                   "outliers (BASELINE configs[4])",
                       "points_per_gpu": M_local, "model_points_total": M_total,
                       "obs_points": N_obs, "sigma_frac": 0.05, "outlier_ratio": 0.1,
                       "lattice_sites": sites, "build_ms": build_ms,
                       "l2": "flushed before every timed step" if need_flush
                       else "inputs larger than L2",
                       "parallelism": f"dp{world} (model shards, replicated lattice)"},
            "em_iters_per_sec": args.steps / (total_ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_rigid_pass (+k_reduce_cols)",
                         "alg_bytes_per_launch": alg_bytes, "kernel_ms": pass_avg_ms,
                         "peak_source": peak_kind},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


def _timed_pass(path, R, t, ev_after):
    """run_pass with an event right after the pass kernels are enqueued (before
    the all-reduce / D2H), so the pass duration is [step start, ev_after]."""
    import ctypes
    from paper_1811_10136_b200 import _lib
    p = _lib.RigidPassParams()
    p.R[:] = list(np.asarray(R, dtype=float).reshape(-1))
    p.c_ref[:] = list(path.c_ref)
    p.c_world[:] = list(path.centre(R, t))
    p.sigma[:] = list(path.sigma)
    p.c_prime = path.c_prime
    p.mode = path.mode
    p.m2_col = path.m2_col
    p.normal_col = path.normal_col
    _lib.check(path.lib.fr_rigid_pass(path.lattice.handle, _lib.ptr(path.ref), path.M,
                                      ctypes.byref(p), _lib.ptr(path.sums), _lib.ptr(path.wtn),
                                      _lib.ptr(path.scratch), _lib.stream_handle()))
    import torch
    ev_after.record(torch.cuda.current_stream())
    path.reduce_device(path.sums[:path.width])
    path.host[:path.width].copy_(path.sums[:path.width])
    return path.host[:path.width].numpy().copy()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
