"""BASELINE configs C1-C4 end to end on the GPU, next to the live reference's
timing on the same inputs (bench_data/, made by tools/make_config_inputs.py).

    python tools/configs_timing.py        # on the GPU box

Each config: one warm-up registration, then one timed registration through the
public register() from host float64 clouds (upload, lattice build, EM loop).
Prints one JSON object per config and writes bench_data/gpu_timing.json.
"""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1811_10136_b200 as fr  # noqa: E402
from paper_1811_10136_b200.kinematics import NodeGraph, Skinning  # noqa: E402
from tests.articulated_util import tree_from_arrays  # noqa: E402

DATA = os.path.join(ROOT, "bench_data")


def cases():
    g = np.load(os.path.join(DATA, "c1.npz"))
    yield "C1", fr.PointCloud(g["X"]), fr.PointCloud(g["Y"]), lambda: fr.RigidModel(), \
        fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=float(g["sigma"]), outlier_ratio=0.1),
                              max_em_iters=250, twist_tolerance=2e-4)
    g = np.load(os.path.join(DATA, "c2.npz"))
    yield "C2", fr.PointCloud(g["X"], normals=g["N"]), fr.PointCloud(g["Y"], normals=g["YN"]), \
        lambda: fr.RigidModel(), \
        fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=float(g["sigma"]), outlier_ratio=0.1),
                              residual_mode="point_to_plane", max_em_iters=50,
                              twist_tolerance=1e-4)
    g = np.load(os.path.join(DATA, "c3.npz"))
    yield "C3", fr.PointCloud(g["X"]), fr.PointCloud(g["Y"]), lambda: tree_from_arrays(fr, g), \
        fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.006, outlier_ratio=0.1),
                              max_em_iters=15, twist_tolerance=1e-5)
    g = np.load(os.path.join(DATA, "c4.npz"))
    yield "C4", fr.PointCloud(g["X"]), fr.PointCloud(g["Y"]), \
        lambda: NodeGraph(g["nodes"], g["edges"], Skinning(g["skin_idx"], g["skin_w"])), \
        fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.02, outlier_ratio=0.1),
                              max_em_iters=10, twist_tolerance=1e-5,
                              mstep=fr.MStepOptions(lambda_reg=0.1))


def main():
    ref_t = json.load(open(os.path.join(DATA, "reference_timing.json")))
    out = {}
    for name, ref, obs, model, config in cases():
        fr.register(ref, obs, model(), config)                    # warm-up
        torch.cuda.synchronize()
        timing = {}
        t0 = time.perf_counter()
        res = fr.register(ref, obs, model(), config, timing=timing)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        it = max(res.iterations, 1)
        r = ref_t[name]
        out[name] = {"iterations": res.iterations, "termination": res.termination,
                     "ref_iterations": r["iterations"], "wall_s": wall,
                     "em_it_per_s": it / wall, "e_ms_per_iter": 1e3 * timing["e_step_s"] / it,
                     "m_ms_per_iter": 1e3 * timing["m_step_s"] / it,
                     "ref_em_it_per_s": r["em_it_per_s"], "ref_wall_s": r["wall_s"],
                     "speedup_wall": r["wall_s"] / wall}
        print(name, json.dumps(out[name]), flush=True)
    with open(os.path.join(DATA, "gpu_timing.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
