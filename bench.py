"""FilterReg B200 benchmark: rigid point-to-point EM, BASELINE metric
"EM iters/sec & points/sec (100k/1M-pt rigid)".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--points P]
                    [--precision f64|f32] [--impl b200|reference] [--mode fixed|sigma|batch]

Workload (BASELINE.json configs[4] at its 1M point; configs' 100k point as a
secondary line): the reference's pebble pair (synth.py:252-284, restated in
oracle/filterreg_oracle.py), P = 1,000,000 clean points + 5 % uniform
outliers (1.05M) for the model and the observation cloud, 50 deg / 2 % shift
ground truth, sigma = 5 % of the clean bbox diagonal, w = 0.1.  Inputs are
float64 (float32-rounded values, as every parity fixture).

A step is ONE registration of EM_PER_STEP = 50 EM iterations (the reference's
default max_em_iters; tolerance 1e-30 so every iteration runs) on the
resident lattice: the float64 grid-resident EM loop (fr_em64: pass,
fixed-order reduction and float64 solve of every iteration in one cooperative
launch).  The lattice build is once per run and reported as build_ms.  At 1M
the 25 MB of model points fit in L2, so L2 is flushed (a 256 MB write) before
every timed step, outside its CUDA-event bracket; within a step the
iterations re-read the points as a real registration does.

value = model points x EM iterations / device time (sum of the per-step event
times, max over ranks).  e2e = the same metric through the public register()
from host float64 arrays (H2D, Morton sort, lattice build, EM loop, D2H).
Weak scaling for N > 1: every rank holds its own model shard (1.05M points)
and the whole observation lattice; the 25 partial sums are NCCL all-reduced
per iteration.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "points/sec (model points x EM iterations / s, rigid point-to-point FilterReg)"
L2_BYTES = 126 * 1024 * 1024
EM_PER_STEP = 50


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--points", type=int, default=1_000_000, help="clean model points per GPU")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"],
                    help="query-side arithmetic of the headline line (the other is reported "
                         "beside it)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-iters", type=int, default=6,
                    help="EM iterations of the in-run CPU baseline (same clouds, all cores)")
    ap.add_argument("--ref-iters", type=int, default=4,
                    help="EM iterations per step of --impl reference")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="fixed", choices=["fixed", "sigma", "batch"],
                    help="fixed: the headline fixed-sigma EM (default); sigma: the "
                         "sigma-re-estimating EM, lattice rebuilt every iteration "
                         "(SURVEY.md 8(f) rank 1; single GPU); batch: the reference's "
                         "30-trial C1 protocol through register_batch (8(f) rank 4)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_shard(points: int, rank: int):
    """This rank's model shard and the (replicated) observation cloud.

    The observation cloud and rank 0's model shard are the reference's pebble
    pair (synth.py:252-284; 50 deg / 2% shift ground truth, 5% outliers);
    rank r > 0 holds an independent scattered re-sampling of the same surface
    (seeded by r) with its own 5% outliers, so the per-GPU work is fixed as
    the GPU count grows (weak scaling) and no rank materialises the job's
    whole model cloud.  Everything is rounded to float32 once."""
    from oracle import filterreg_oracle as O
    model, obs, (Rg, tg) = O.pebble_pair(points, rotation_degrees=50.0,
                                         translation_fraction=0.02, outlier_ratio=0.05, seed=0)
    sigma = 0.05 * O.bbox_diameter(model[:points])
    if rank > 0:
        model = O.pebble_resample(points, seed=1000 + rank, outlier_ratio=0.05)
    X = model.astype(np.float32).astype(np.float64)
    Y = obs.astype(np.float32).astype(np.float64)
    return X, Y, sigma


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


def _cpu_worker(conn, shard, eng, sinv, n_model):
    """One host core of the CPU arm: E step, assembly and candidate objectives
    of the oracle's rigid EM iteration over this worker's model shard (the
    outlier constant over the whole model count, estep.py:197-198)."""
    from threadpoolctl import threadpool_limits

    from oracle import filterreg_oracle as O
    with threadpool_limits(1):
        spec = None
        while True:
            msg = conn.recv()
            if msg[0] == "stop":
                return
            R, t = msg[1], msg[2]
            x = shard @ R.T + t
            if msg[0] == "estep":
                mom = eng.moments(x, n_model=n_model)
                spec = (mom["weight"], mom["target"], sinv, "point_to_point", None, None)
                H, g = O.assemble_rigid(spec, x)
                conn.send((O.rigid_objective(spec, x), H, g))
            else:
                conn.send(O.rigid_objective(spec, x))


class CpuArm:
    """The reference algorithm's CPU path (the oracle port of pipeline.py /
    mstep.py / estep.py, bit-identical to the reference on its fixtures) on all
    host cores, over the SAME clouds as the GPU arm (no subsampling): the
    lattice is built once on the whole observation cloud (not timed), the
    model cloud is split into one contiguous shard per core (forked worker
    processes sharing the lattice copy-on-write); per EM iteration the shards'
    objective / H / g are summed, the 6x6 solve and the step halving run as in
    oracle.rigid_m_step (mstep.py:421-459), candidate objectives are again
    summed over shards."""

    def __init__(self, X, Y, sigma, workers=None):
        import multiprocessing as mp

        from oracle import filterreg_oracle as O
        self.O = O
        tick = time.perf_counter()
        eng = O.OracleMoments(Y, sigma, 0.1)
        self.build_s = time.perf_counter() - tick
        self.workers = workers or max(1, len(os.sched_getaffinity(0)))
        ctx = mp.get_context("fork")
        sinv = np.full(3, 1.0 / sigma)
        self.conns, self.procs = [], []
        for shard in np.array_split(X, self.workers):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_cpu_worker,
                            args=(b, np.ascontiguousarray(shard), eng, sinv, len(X)), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)
        self.R, self.t = np.eye(3), np.zeros(3)

    def _all(self, msg):
        for c in self.conns:
            c.send(msg)
        return [c.recv() for c in self.conns]

    def iteration(self):
        O = self.O
        parts = self._all(("estep", self.R, self.t))
        value = sum(p[0] for p in parts)
        H = sum(p[1] for p in parts)
        g = sum(p[2] for p in parts)
        if not np.any(g):
            return
        step = O.gn_solve(H, g, None)
        scale = 1.0
        for _ in range(11):
            Rc, tc = O.apply_twist(scale * step, self.R, self.t)
            cv = sum(self._all(("obj", Rc, tc)))
            if cv <= value * (1.0 + 1e-12) + 1e-300:
                self.R, self.t = Rc, tc
                return
            scale *= 0.5

    def close(self):
        for c in self.conns:
            c.send(("stop",))
        for p in self.procs:
            p.join(timeout=10)


def cpu_baseline(X, Y, sigma, iters: int):
    """The CPU arm on the full clouds: `iters` EM iterations timed after one
    warm-up iteration (lattice build not timed)."""
    arm = CpuArm(X, Y, sigma)
    arm.iteration()                     # warm-up (worker start, first-touch)
    tick = time.perf_counter()
    for _ in range(iters):
        arm.iteration()
    dt = time.perf_counter() - tick
    arm.close()
    return len(X) * iters / dt, dt, arm.workers, arm.build_s


def workload_name(points: int) -> str:
    return (f"C5 rigid pt2pt pebble {points} clean pts + 5% outliers (model and observation), "
            f"{EM_PER_STEP}-iteration registrations (BASELINE configs[4] at 1M; metric "
            "'100k/1M-pt rigid')")


def run_reference(args):
    """--impl reference: the reference algorithm's CPU path (the oracle port;
    the Python reference itself cannot travel to the GPU box) on this box's
    cores, on the same clouds as the GPU arm.  Each step is a bounded sample of
    the workload: `--ref-iters` EM iterations of the full-size registration."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    X, Y, sigma = make_shard(args.points, 0)
    arm = CpuArm(X, Y, sigma)
    times = []
    for i in range(args.warmup + args.steps):
        tick = time.perf_counter()
        for _ in range(args.ref_iters):
            arm.iteration()
        if i >= args.warmup:
            times.append(time.perf_counter() - tick)
    arm.close()
    total = sum(times)
    value = len(X) * args.ref_iters * args.steps / total
    cores = arm.workers
    sample = (f"{args.ref_iters} EM iterations per step over the full {len(X)}-point model "
              f"cloud against the lattice of the full {len(Y)}-point observation cloud, "
              f"{cores} worker processes (lattice build {arm.build_s:.1f} s, not timed)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.points), "points_per_gpu": len(X),
                   "obs_points": len(Y), "sigma_frac": 0.05, "outlier_ratio": 0.1,
                   "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


class L2Flush:
    """A 256 MB device buffer written between timed steps (twice L2)."""

    def __init__(self, dev):
        import torch
        self.buf = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev)

    def __call__(self):
        self.buf.fill_(1.0)


def time_em_steps(em_factory, steps, warmup, flush, stream):
    """Per-step CUDA-event times of `steps` registrations (after `warmup`),
    each a fresh EM state at the identity run for EM_PER_STEP iterations in
    one launch, L2 flushed before each (outside the event bracket)."""
    import torch
    times = []
    for i in range(warmup + steps):
        em = em_factory()
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        em.enqueue(EM_PER_STEP)
        e1.record(stream)
        torch.cuda.synchronize()
        done, iters, term = em.status()
        assert iters == EM_PER_STEP, (iters, term)
        if i >= warmup:
            times.append(e0.elapsed_time(e1))
        del em
    return times


def run_b200(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    group = None
    # FR_BENCH_GROUP=1 drives the sharded (NCCL) path even at one rank: a
    # world-size-1 group exercises the captured pass -> all-reduce -> solve
    # chunks on the one GPU available to the builder
    if world > 1 or os.environ.get("FR_BENCH_GROUP") == "1":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    import paper_1811_10136_b200 as fr
    from paper_1811_10136_b200 import _lib, _rigid
    from paper_1811_10136_b200._rigid import RigidDevicePath

    X, Y, sigma = make_shard(args.points, rank)
    M_local, N_obs = len(X), len(Y)
    gmm = fr.GmmConfig(sigma=sigma, outlier_ratio=0.1)
    cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=EM_PER_STEP, twist_tolerance=1e-30)
    stream = torch.cuda.current_stream()
    flush = L2Flush(dev)
    l2_note = ("inputs smaller than L2: L2 flushed (256 MB write) before every timed step"
               if 24 * M_local < L2_BYTES else "inputs larger than L2 (and L2 flushed)")
    ref_pc, obs_pc = fr.PointCloud(X), fr.PointCloud(Y)          # host-side validation, untimed

    def measure(precision, points_tag):
        """Setup once (warm-up setup first), then the timed registrations."""
        first = RigidDevicePath(ref_pc, obs_pc, gmm, "point_to_point", group, precision=precision)
        del first
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        path = RigidDevicePath(ref_pc, obs_pc, gmm, "point_to_point", group, precision=precision)
        torch.cuda.synchronize()
        build_ms = 1e3 * (time.perf_counter() - t0)

        def factory():
            return _rigid.device_em(path, np.eye(3), np.zeros(3), cfg)
        if group is not None:
            dist.barrier()
        with ClockSampler(local) as clk:
            times = time_em_steps(factory, args.steps, args.warmup, flush, stream)
        tot = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
        if group is not None:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        total_ms = float(tot.item())
        out = {"path": path, "build_ms": build_ms, "total_ms": total_ms, "clocks": clk.summary(),
               "value": path.M_total * EM_PER_STEP * args.steps / (total_ms / 1e3),
               "ms_per_step": total_ms / args.steps}
        em = factory()
        out["em_kind"] = type(em).__name__
        if isinstance(em, _rigid.DeviceEM64):
            grid, block = em.launch_info()
            # unsharded: one launch per registration; sharded: one fused
            # (solve-first + pass) launch per iteration and a final solve
            # (+ NCCL's all-reduce kernel per iteration)
            kps = 1 if group is None else (EM_PER_STEP + 1 if em._fused else 2 * EM_PER_STEP)
            out["launch"] = {"grid": grid, "block": block, "kernels_per_step": kps}
            if group is not None:
                out["launch"]["nccl_allreduce_per_step"] = EM_PER_STEP
                out["launch"]["graph"] = em._graph is not None
            # the pass alone (one cooperative launch: pass + fixed-order
            # reduction, no solve), cold (L2 flushed) and warm
            cold = []
            for _ in range(10):
                flush()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                em.pass_only()
                e1.record(stream)
                torch.cuda.synchronize()
                cold.append(e0.elapsed_time(e1))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            em.pass_only()
            e0.record(stream)
            for _ in range(20):
                em.pass_only()
            e1.record(stream)
            torch.cuda.synchronize()
            out["pass_cold_ms"] = float(np.median(cold))
            out["pass_warm_ms"] = e0.elapsed_time(e1) / 20
        else:
            out["launch"] = {"kernels_per_step": EM_PER_STEP *
                             int(path.lib.fr_rigid_em_kernels_per_iter(em.h))}
        del em
        return out

    head = measure(args.precision, "head")
    other_precision = "f32" if args.precision == "f64" else "f64"
    other = measure(other_precision, "other")

    # the metric's 100k point (same protocol), rank 0 / N = 1 only
    p100k = None
    if world == 1 and args.points != 100_000:
        X1, Y1, s1 = make_shard(100_000, 0)
        g1 = fr.GmmConfig(sigma=s1, outlier_ratio=0.1)
        c1 = fr.RegistrationConfig(gmm=g1, max_em_iters=EM_PER_STEP, twist_tolerance=1e-30)
        path1 = RigidDevicePath(fr.PointCloud(X1), fr.PointCloud(Y1), g1, "point_to_point",
                                precision=args.precision)

        def f1():
            return _rigid.device_em(path1, np.eye(3), np.zeros(3), c1)
        t1 = time_em_steps(f1, args.steps, args.warmup, flush, stream)
        p100k = {"points": len(X1), "value": len(X1) * EM_PER_STEP * args.steps / (sum(t1) / 1e3),
                 "unit": "points/s", "ms_per_step": sum(t1) / args.steps,
                 "em_iters_per_sec": EM_PER_STEP * args.steps / (sum(t1) / 1e3),
                 "dtype": args.precision}
        del path1

    # roofline of the dominant kernel.  The timed region launches ONE kernel
    # per step (k_em64: the whole 50-iteration registration), so a launch's
    # algorithmic bytes are 24 B (float64 x, y, z) x model points x 50 passes
    # -- every pass reads every point; after the first they come from L2 --
    # and its duration is the step time measured by the CUDA events around
    # it (the L2 flush sits outside the bracket).  The dense slice grid
    # (~3 MB) is not counted.  The pass alone (one launch: pass + reduction,
    # cold and warm) is reported beside it.  The float64 pass is bound by the
    # FP64 pipe, not HBM: roofline_fp64 counts the pass's FP64 flops per point
    # from its SASS (61 DFMA x 2 + 26 DADD + 17 DMUL) against the measured
    # FP64 FMA peak (tools/gpu/fp64_peak.cu -> profiles/fp64_peak.json).
    peak, peak_kind = measured_peak()
    hp = head
    bpp = 24 if args.precision == "f64" else 12
    alg_bytes = bpp * M_local * EM_PER_STEP
    step_ms = hp["ms_per_step"]
    achieved = alg_bytes / (step_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": f"k_em64 (one launch = a {EM_PER_STEP}-iteration registration: "
                          "pass, fixed-order reduction, float64 solve per iteration)",
                "alg_bytes_per_launch": alg_bytes, "kernel_ms": step_ms,
                "alg_bytes_per_point_pass": bpp,
                "em_iteration_ms": step_ms / EM_PER_STEP,
                "pass_alone": {"cold_ms": hp.get("pass_cold_ms"), "warm_ms": hp.get("pass_warm_ms"),
                               "alg_bytes": bpp * M_local,
                               "note": "one launch: pass + grid reduction, no solve; cold = "
                                       "L2 flushed (points from HBM)"},
                "peak_source": peak_kind,
                "note": "traffic null: ncu DRAM bytes of the same launch are in profiles/ "
                        "(r02_ncu.json: 25.5 MB per registration launch at 1.05M -- the points "
                        "once, then L2; 403.8 MB per pass at 16.8M); the float64 pass is "
                        "FP64-bound (roofline_fp64)"}
    roofline_fp64 = None
    fp64_peak_path = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if args.precision == "f64" and os.path.exists(fp64_peak_path):
        fpk = json.load(open(fp64_peak_path))["fp64_tflops"]
        flops_pt = 165
        ach = flops_pt * M_local * EM_PER_STEP / (step_ms / 1e3) / 1e12
        roofline_fp64 = {"bound": "fp64", "achieved": ach, "peak": fpk, "unit": "TFLOP/s",
                         "frac": ach / fpk, "flops_per_point_pass": flops_pt,
                         "peak_source": "measured (profiles/fp64_peak.json)"}

    # end to end through the public API: register() from host float64
    # arrays, H2D of both clouds, sort, lattice build, the EM loop, D2H
    e2e = None
    build_ms = head["build_ms"]
    sites = head["path"].lattice.num_sites
    del head["path"], other["path"]
    torch.cuda.synchronize()
    if not args.no_e2e:
        old = _rigid.PRECISION
        _rigid.PRECISION = args.precision
        # the caller's inputs in page-locked host memory (as fr.load_cloud(...,
        # pinned=True) returns them), built before the timer; the same
        # registrations from pageable NumPy arrays are reported beside them
        pinned_ref, pinned_obs = fr.pinned_cloud(ref_pc), fr.pinned_cloud(obs_pc)

        def e2e_walls(a, b):
            for _ in range(3):          # warm-up registrations (pools, streams)
                fr.register(a, b, fr.RigidModel(), cfg, process_group=group)
            torch.cuda.synchronize()
            if group is not None:
                dist.barrier()
            walls = []
            for _ in range(max(3, min(args.steps, 10))):
                t0 = time.perf_counter()
                r = fr.register(a, b, fr.RigidModel(), cfg, process_group=group)
                _ = r.kinematics.pose.matrix()
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t0)
            et = torch.tensor([float(np.median(walls))], dtype=torch.float64, device=dev)
            if group is not None:
                dist.all_reduce(et, op=dist.ReduceOp.MAX)
            return float(et.item()), walls, r
        try:
            e2e_s, walls, res = e2e_walls(pinned_ref, pinned_obs)
            page_s, page_walls, _ = e2e_walls(ref_pc, obs_pc)
        finally:
            _rigid.PRECISION = old
        bpp = 24 if args.precision == "f64" else 12
        e2e = {"value": M_total_of(head, M_local, world) * res.iterations / e2e_s,
               "unit": "points/s", "h2d_bytes_per_step": bpp * (M_local + N_obs),
               "d2h_bytes_per_step": 8 * 12 + 24 * res.iterations,
               "em_iterations": res.iterations, "wall_s_median": e2e_s,
               "wall_s_reps": walls,
               "inputs": "float64 (n, 3) rows in pinned host memory (fr.pinned_cloud, built "
                         "before the timer): one DMA per cloud",
               "includes": "register() on host float64 PointClouds: H2D of the model shard "
                           "and observation cloud, Morton sort, lattice build (splat + blur + "
                           "dense grid), tile copy, the EM loop, D2H of pose and traces",
               "pageable": {"value": M_total_of(head, M_local, world) * res.iterations / page_s,
                            "wall_s_median": page_s, "wall_s_reps": page_walls,
                            "inputs": "the same clouds as pageable NumPy arrays (threaded "
                                      "staging copy into pinned slots, host-memory bound)"}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, nw, bs = cpu_baseline(X, Y, sigma, args.cpu_iters)
        cpu = {"value": v, "unit": "points/s", "cores": nw, "kind": "port",
               "sample": f"{args.cpu_iters} EM iterations over the full {len(X)}-point model "
                         f"cloud against the lattice of the full {len(Y)}-point observation "
                         f"cloud ({nw} worker processes, {dt:.1f} s timed; lattice build "
                         f"{bs:.1f} s not timed)",
               "same_config": True}

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": args.precision, "data": "synthetic",
            "config": {"workload": workload_name(args.points),
                       "points_per_gpu": M_local, "model_points_total": M_local * world,
                       "obs_points": N_obs, "sigma_frac": 0.05, "outlier_ratio": 0.1,
                       "em_iters_per_step": EM_PER_STEP, "lattice_sites": sites,
                       "build_ms": build_ms, "l2": l2_note,
                       "query_path": ("float64: forward map, simplex, dense float64 slice grid, "
                                      "epilogue and the 25 statistics all in float64; one "
                                      "cooperative grid-resident launch per registration")
                       if args.precision == "f64" else "float32 point path",
                       "parallelism": f"dp{world} (model shards, replicated lattice, NCCL "
                                      "all-reduce of 25 doubles per iteration)"},
            "em_iters_per_sec": EM_PER_STEP * args.steps / (head["total_ms"] / 1e3),
            "em_iteration_us": 1e3 * head["ms_per_step"] / EM_PER_STEP,
            "roofline": roofline, "roofline_fp64": roofline_fp64,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": head["launch"]["kernels_per_step"] * args.steps,
            "launch": head["launch"],
            "clocks": head["clocks"],
            "other_precision": {"dtype": other_precision, "value": other["value"],
                                "ms_per_step": other["ms_per_step"],
                                "em_iteration_us": 1e3 * other["ms_per_step"] / EM_PER_STEP,
                                "engine": other["em_kind"], "build_ms": other["build_ms"]},
            "p100k": p100k,
        }
        print(json.dumps(line), flush=True)
    if group is not None:
        dist.barrier()
        dist.destroy_process_group()


def M_total_of(head, M_local, world):
    return M_local * world


def run_sigma(args):
    """--mode sigma: register() with update_sigma=True (estep.py:232-259,
    pipeline.py:155-161): every EM iteration re-estimates sigma from the pass's
    fused sums and rebuilds the observation lattice (splat + blur) at the new
    width.  Host-timed through the public API (the loop syncs every
    iteration); inputs are host clouds uploaded by the call."""
    import torch

    import paper_1811_10136_b200 as fr
    torch.cuda.set_device(0)
    X, Y, sigma = make_shard(args.points, 0)
    ref, obs = fr.PointCloud(X), fr.PointCloud(Y)

    def cfg(n):
        return fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=0.1,
                                                      update_sigma=True),
                                     max_em_iters=n, twist_tolerance=1e-30)
    # warm-up: a full-length run, so the device pool has grown to the annealed
    # (small-sigma, many-site) lattice sizes before the timed run
    fr.register(ref, obs, fr.RigidModel(), cfg(max(args.warmup, args.steps)))
    torch.cuda.synchronize()
    # host-driven rebuild loop (allocation and sync patterns vary): median of 3
    walls = []
    for _ in range(3):
        timing = {}
        t0 = time.perf_counter()
        res = fr.register(ref, obs, fr.RigidModel(), cfg(args.steps), timing=timing)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    wall = float(np.median(walls))
    value = len(X) * res.iterations / wall
    print(json.dumps({
        "metric": "points/sec (model points x EM iterations / s, rigid point-to-point FilterReg, "
                  "sigma re-estimated every iteration)",
        "value": value, "unit": "points/s", "n_gpus": 1, "steps": res.iterations,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall / res.iterations,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "mode": "sigma",
        "config": {"workload": f"C5 pebble, {args.points} clean model pts + 5% outliers, "
                               "sigma re-estimated and the lattice rebuilt every iteration",
                   "points": len(X), "obs_points": len(Y), "sigma0": sigma,
                   "sigma_final": res.sigmas[-1] if res.sigmas else None},
        "wall_s_reps": walls,
        "e_step_ms_per_iter": 1e3 * timing.get("e_step_s", 0.0) / res.iterations,
        "m_step_ms_per_iter": 1e3 * timing.get("m_step_s", 0.0) / res.iterations,
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 24 * (len(X) + len(Y))
                / res.iterations, "d2h_bytes_per_step": 8 * 31},
    }), flush=True)


def run_batch(args):
    """--mode batch: the reference's C1 bench protocol (bench.py:92-130 there:
    30 seeded trials of a 10k-point pebble + 5 % outliers, sigma 5 % of the
    clean diagonal, <= 250 iterations, tolerance 2e-4) -- sequential register()
    calls vs one register_batch() call with concurrent streams."""
    import torch

    import paper_1811_10136_b200 as fr
    from oracle import filterreg_oracle as O
    torch.cuda.set_device(0)
    problems = []
    for trial in range(30):
        model, obs, _ = O.pebble_pair(10000, outlier_ratio=0.05, seed=trial)
        X = model.astype(np.float32).astype(float)
        Y = obs.astype(np.float32).astype(float)
        sigma = 0.05 * O.bbox_diameter(X[:10000])
        cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                                    max_em_iters=250, twist_tolerance=2e-4)
        problems.append((fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg))
    fr.register_batch(problems, max_concurrent=8)          # warm-up (pools, graphs, threads)
    torch.cuda.synchronize()
    # both arms are tens of milliseconds of host-threaded work: median of reps
    seqs, bats = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        seq = [fr.register(*p) for p in problems]
        torch.cuda.synchronize()
        seqs.append(time.perf_counter() - t0)
    for _ in range(7):
        t0 = time.perf_counter()
        bat = fr.register_batch(problems, max_concurrent=8)
        torch.cuda.synchronize()
        bats.append(time.perf_counter() - t0)
    t_seq, t_bat = float(np.median(seqs)), float(np.median(bats))
    same = all(np.array_equal(a.kinematics.pose.matrix(), b.kinematics.pose.matrix())
               for a, b in zip(seq, bat))
    dev = max(O.rotation_angle(a.kinematics.pose.rotation @ b.kinematics.pose.rotation.T)
              for a, b in zip(seq, bat))
    iters = sum(r.iterations for r in bat)
    print(json.dumps({
        "metric": "registrations/s (C1 bench protocol, 30 trials)", "value": 30 / t_bat,
        "unit": "registrations/s", "n_gpus": 1, "higher_is_better": True, "mode": "batch",
        "data": "synthetic", "dtype": fr._rigid.PRECISION,
        "config": {"workload": "C1 rigid pt2pt pebble 10k + 5% outliers, 30 seeded trials, "
                               "<= 250 iterations, tol 2e-4", "max_concurrent": 8},
        "batched_s": t_bat, "sequential_s": t_seq, "speedup_vs_sequential": t_seq / t_bat,
        "batched_s_reps": bats, "sequential_s_reps": seqs,
        "em_iterations_total": iters, "identical_to_sequential": bool(same),
        "max_rotation_deviation_vs_sequential_rad": dev,
    }), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "sigma":
        run_sigma(args)
    elif args.mode == "batch":
        run_batch(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
