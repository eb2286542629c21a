"""Inputs of BASELINE configs C1-C4 at their full sizes plus
the LIVE reference's own timing on them, for tools/configs_timing.py.

    PYTHONPATH=/root/reference/pkg/src python tools/make_config_inputs.py

Writes bench_data/c{1..4}.npz (git-ignored, travels to the GPU box) and
bench_data/reference_timing.json (reference register(..., timing=) on this
container's cores: E / M ms per iteration, iterations, wall time).
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import twistreg as T  # noqa: E402
from twistreg.synth import cuboid_shell, flat_strip  # noqa: E402

from make_golden_articulated import chain, tree_arrays  # noqa: E402

OUT = os.path.join(ROOT, "bench_data")


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def timed(name, ref, obs, model, config, meta):
    timing = {}
    t0 = time.perf_counter()
    res = T.register(ref, obs, model, config, timing=timing)
    wall = time.perf_counter() - t0
    it = max(res.iterations, 1)
    meta[name] = {"iterations": res.iterations, "termination": res.termination,
                  "e_ms_per_iter": 1e3 * timing["e_step_s"] / it,
                  "m_ms_per_iter": 1e3 * timing["m_step_s"] / it, "wall_s": wall,
                  "em_it_per_s": it / wall, "points": len(ref),
                  "cores": os.cpu_count()}
    print(name, json.dumps(meta[name]), flush=True)
    return res


def main():
    os.makedirs(OUT, exist_ok=True)
    meta = {}
    # C1: rigid pt2pt pebble 10k + 5 % outliers, sigma 5 % of the clean diagonal
    m, o, _ = T.synthesize_pair(T.ExperimentSpec(source="pebble", n_points=10000,
                                                 outlier_ratio=0.05, seed=0))
    X, Y = f32(m.positions), f32(o.positions)
    sigma = 0.05 * float(np.linalg.norm(X[:10000].max(0) - X[:10000].min(0)))
    np.savez(os.path.join(OUT, "c1.npz"), X=X, Y=Y, sigma=sigma)
    timed("C1", T.PointCloud(X), T.PointCloud(Y), T.RigidModel(),
          T.RegistrationConfig(gmm=T.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                               max_em_iters=250, twist_tolerance=2e-4), meta)
    # C2: rigid pt2pl, cuboid_shell(100000) with normals, 8 deg about (0, 1, 0.4)
    P, N = cuboid_shell(100000)
    P, N = f32(P), f32(N)
    R = T.rotation_about_axis(np.array([0.0, 1.0, 0.4]), np.radians(8.0))
    gt = T.RigidTransform(R, np.array([0.002, 0.001, -0.003]))
    Yc, Nc = f32(gt.apply(P)), f32(N @ R.T)
    sigma = 0.05 * float(np.linalg.norm(P.max(0) - P.min(0)))
    np.savez(os.path.join(OUT, "c2.npz"), X=P, N=N, Y=Yc, YN=Nc, sigma=sigma)
    timed("C2", T.PointCloud(P, normals=N), T.PointCloud(Yc, normals=Nc), T.RigidModel(),
          T.RegistrationConfig(gmm=T.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                               residual_mode="point_to_plane", max_em_iters=50,
                               twist_tolerance=1e-4), meta)
    # C3: articulated chain, 20 revolute links, ~2,500 points per link
    Pa, _, lab, rest, gta = chain(20, 2500, seed=0)
    obs = T.forward_points(T.PointCloud(Pa), gta)
    Ya = f32(obs.positions)
    np.savez(os.path.join(OUT, "c3.npz"), X=Pa, Y=Ya, labels=lab, **tree_arrays(rest))
    timed("C3", T.PointCloud(Pa), T.PointCloud(Ya), rest,
          T.RegistrationConfig(gmm=T.GmmConfig(sigma=0.006, outlier_ratio=0.1),
                               max_em_iters=15, twist_tolerance=1e-5), meta)
    # C4: node graph on a 100k-point strip (spacing 0.0135), warped target
    pts = f32(flat_strip(n_points=100000))
    nodes, edges = T.build_node_graph(pts, spacing=0.0135)
    skin = T.bind_points_to_nodes(pts, nodes, radius=2.0 * 0.0135)
    graph = T.NodeGraph(nodes, edges, skin)
    q = pts.copy()
    q[:, 2] += 0.04 * np.sin(np.pi * (q[:, 0] + 0.15) / 0.3)
    Yn = f32(q)
    np.savez(os.path.join(OUT, "c4.npz"), X=pts, Y=Yn, nodes=nodes, edges=edges,
             skin_idx=skin.indices, skin_w=skin.weights)
    timed("C4", T.PointCloud(pts), T.PointCloud(Yn), graph,
          T.RegistrationConfig(gmm=T.GmmConfig(sigma=0.02, outlier_ratio=0.1),
                               max_em_iters=10, twist_tolerance=1e-5,
                               mstep=T.MStepOptions(lambda_reg=0.1)), meta)
    with open(os.path.join(OUT, "reference_timing.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
