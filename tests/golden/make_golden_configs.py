"""Golden results of the LIVE reference at the BASELINE configs' full sizes.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_configs.py [case ...]

Each case runs `twistreg.register` (pipeline.py:125-181) on the exact inputs
the GPU parity tests rebuild, and stores the small result arrays (final pose /
joint values / node transforms, per-iteration objectives, twist norms, inlier
masses, iteration count, termination) in tests/golden/config_<case>.npz.

Inputs:
  * pebble cases: oracle.pebble_pair (bit-identical to synth.synthesize_pair,
    pinned by tests/test_oracle_golden.py), rounded to float32; not stored;
  * C2 / C3 / C4: float32 inputs stored in the fixture (the rotated clouds are
    BLAS products in the reference, so they are kept rather than regenerated).

Cases:
  c5_1m_fixed15   C5 rigid pt2pt pebble 1M + 5 % outliers, 15 iterations (tol 1e-30)
  c5_1m_conv      the same, tolerance 2e-4, <= 250 iterations (converging run)
  p100k_conv      rigid pt2pt pebble 100k + 5 % outliers, tolerance 2e-4
  p100k_fixed50   the same, 50 iterations at tol 1e-30 (the bench step)
  c2              rigid pt2pl cuboid_shell(100000), 8 deg about (0, 1, 0.4)
  c3              articulated chain, 20 links x 2,500 points (50k), sigma 6 mm
  c4              node graph, strip 100k, spacing 0.0135, lambda_reg 0.1
  gn3_pt2pl       rigid pt2pl cuboid_shell(20000), max_gn_iters = 3
  gn3_chain6_pt2pl articulated pt2pl chain(6, 480), max_gn_iters = 3
  gn2_strip2k     node graph pt2pt strip 2k, max_gn_iters = 2
  ladder_p10k     the bench's coarse-to-fine sigma ladder (bench.py:34-38,
                  66-78, 87-110) on a corrupted pebble 10k + 20 % outliers
"""

import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def pebble_inputs(n, outlier_ratio=0.05, seed=0):
    from oracle import filterreg_oracle as O
    model, obs, _ = O.pebble_pair(n, rotation_degrees=50.0, translation_fraction=0.02,
                                  outlier_ratio=outlier_ratio, seed=seed)
    X, Y = f32(model), f32(obs)
    sigma = 0.05 * O.bbox_diameter(X[:n])
    return X, Y, sigma


def result_arrays(r):
    return dict(objectives=np.asarray(r.objectives, dtype=float),
                twist_norms=np.asarray(r.twist_norms, dtype=float),
                inlier_masses=np.asarray(r.inlier_masses, dtype=float),
                iterations=r.iterations, termination=r.termination)


def rigid_case(name, n, tol, iters):
    import twistreg as T
    X, Y, sigma = pebble_inputs(n)
    cfg = T.RegistrationConfig(gmm=T.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                               max_em_iters=iters, twist_tolerance=tol)
    t0 = time.perf_counter()
    r = T.register(T.PointCloud(X), T.PointCloud(Y), T.RigidModel(), cfg)
    wall = time.perf_counter() - t0
    pose = r.kinematics.pose
    np.savez_compressed(os.path.join(HERE, f"config_{name}.npz"), R=pose.rotation,
                        t=pose.translation, n=n, sigma=sigma, tol=tol, max_iters=iters,
                        **result_arrays(r))
    return name, {"iterations": r.iterations, "termination": r.termination, "wall_s": wall,
                  "points": len(X)}


def c2_case(name="c2", n=100000, gn=1, iters=50):
    import twistreg as T
    from twistreg.synth import cuboid_shell
    P, N = cuboid_shell(n)
    P, N = f32(P), f32(N)
    R = T.rotation_about_axis(np.array([0.0, 1.0, 0.4]), np.radians(8.0))
    gt = T.RigidTransform(R, np.array([0.002, 0.001, -0.003]))
    Y, YN = f32(gt.apply(P)), f32(N @ R.T)
    sigma = 0.05 * float(np.linalg.norm(P.max(0) - P.min(0)))
    cfg = T.RegistrationConfig(gmm=T.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                               residual_mode="point_to_plane", max_em_iters=iters,
                               twist_tolerance=1e-4, mstep=T.MStepOptions(max_gn_iters=gn))
    t0 = time.perf_counter()
    r = T.register(T.PointCloud(P, normals=N), T.PointCloud(Y, normals=YN), T.RigidModel(), cfg)
    wall = time.perf_counter() - t0
    pose = r.kinematics.pose
    np.savez_compressed(os.path.join(HERE, f"config_{name}.npz"),
                        X=P.astype(np.float32), N=N.astype(np.float32),
                        Y=Y.astype(np.float32), YN=YN.astype(np.float32), sigma=sigma,
                        max_gn_iters=gn, max_iters=iters, R=pose.rotation, t=pose.translation,
                        R_gt=R, t_gt=gt.translation, **result_arrays(r))
    return name, {"iterations": r.iterations, "termination": r.termination, "wall_s": wall,
                  "points": len(P)}


def c3_case(name="c3", links=20, per_link=2500, seed=0, normals=False, gn=1):
    import twistreg as T
    from make_golden_articulated import chain, tree_arrays
    P, N, lab, rest, gt = chain(links, per_link, seed=seed, normals=normals)
    obs = T.forward_points(T.PointCloud(P, normals=N), gt)
    Y = f32(obs.positions)
    YN = f32(obs.normals) if N is not None else None
    mode = "point_to_plane" if normals else "point_to_point"
    cfg = T.RegistrationConfig(gmm=T.GmmConfig(sigma=0.006, outlier_ratio=0.1),
                               residual_mode=mode, max_em_iters=15, twist_tolerance=1e-5,
                               mstep=T.MStepOptions(max_gn_iters=gn))
    t0 = time.perf_counter()
    r = T.register(T.PointCloud(P, normals=N), T.PointCloud(Y, normals=YN), rest, cfg)
    wall = time.perf_counter() - t0
    est = r.kinematics
    extra = {"N": N.astype(np.float32), "YN": YN.astype(np.float32)} if N is not None else {}
    np.savez_compressed(os.path.join(HERE, f"config_{name}.npz"),
                        X=P.astype(np.float32), Y=Y.astype(np.float32), labels=lab,
                        joint_values=est.joint_values, base_R=est.base_pose.rotation,
                        base_t=est.base_pose.translation, gt_joints=gt.joint_values,
                        mode=mode, max_gn_iters=gn, **tree_arrays(rest), **extra,
                        **result_arrays(r))
    return name, {"iterations": r.iterations, "termination": r.termination, "wall_s": wall,
                  "points": len(P)}


def warp(p):
    q = p.copy()
    q[:, 2] += 0.04 * np.sin(np.pi * (q[:, 0] + 0.15) / 0.3)
    return q


def c4_case(name="c4", n=100000, spacing=0.0135, iters=10, gn=1):
    import twistreg as T
    from twistreg.synth import flat_strip
    pts = f32(flat_strip(n_points=n))
    nodes, edges = T.build_node_graph(pts, spacing=spacing)
    skin = T.bind_points_to_nodes(pts, nodes, radius=2.0 * spacing)
    graph = T.NodeGraph(nodes, edges, skin)
    Y = f32(warp(pts))
    cfg = T.RegistrationConfig(gmm=T.GmmConfig(sigma=0.02, outlier_ratio=0.1),
                               max_em_iters=iters, twist_tolerance=1e-5,
                               mstep=T.MStepOptions(lambda_reg=0.1, max_gn_iters=gn))
    t0 = time.perf_counter()
    r = T.register(T.PointCloud(pts), T.PointCloud(Y), graph, cfg)
    wall = time.perf_counter() - t0
    est = r.kinematics
    moved = T.forward_points(T.PointCloud(pts), est).positions
    np.savez_compressed(os.path.join(HERE, f"config_{name}.npz"),
                        X=pts.astype(np.float32), Y=Y.astype(np.float32), nodes=nodes,
                        edges=edges, skin_idx=skin.indices.astype(np.int32),
                        skin_w=skin.weights, spacing=spacing, max_iters=iters, max_gn_iters=gn,
                        node_R=np.stack([t.rotation for t in est.node_transforms]),
                        node_t=np.stack([t.translation for t in est.node_transforms]),
                        **result_arrays(r))
    return name, {"iterations": r.iterations, "termination": r.termination, "wall_s": wall,
                  "points": len(pts), "nodes": len(nodes)}


def ladder_case(name="ladder_p10k", n=10000, outlier_ratio=0.2, seed=3):
    """bench.run_trial's filterreg protocol (bench.py:66-110): warm-started
    rungs at sigma fractions LADDER_FRACS of the clean diameter, w = 0.3."""
    import twistreg as T
    from twistreg.bench import LADDER_CAPS, LADDER_FRACS
    X, Y, _ = pebble_inputs(n, outlier_ratio=outlier_ratio, seed=seed)
    diameter = T.PointCloud(X[:n]).diameter()
    state = T.RigidModel(T.RigidTransform.identity())
    rungs = []
    t0 = time.perf_counter()
    for frac, cap in zip(LADDER_FRACS, LADDER_CAPS):
        cfg = T.RegistrationConfig(gmm=T.GmmConfig(sigma=frac * diameter, outlier_ratio=0.3),
                                   max_em_iters=cap, twist_tolerance=1e-4)
        r = T.register(T.PointCloud(X), T.PointCloud(Y), state, cfg)
        state = r.kinematics
        rungs.append(r)
    wall = time.perf_counter() - t0
    pose = state.pose
    np.savez_compressed(
        os.path.join(HERE, f"config_{name}.npz"), R=pose.rotation, t=pose.translation, n=n,
        outlier_ratio=outlier_ratio, seed=seed, diameter=diameter,
        fracs=np.asarray(LADDER_FRACS), caps=np.asarray(LADDER_CAPS),
        rung_iterations=np.array([r.iterations for r in rungs]),
        rung_terminations=np.array([r.termination for r in rungs]),
        rung_R=np.stack([r.kinematics.pose.rotation for r in rungs]),
        rung_t=np.stack([r.kinematics.pose.translation for r in rungs]),
        objectives=np.concatenate([np.asarray(r.objectives, dtype=float) for r in rungs]))
    return name, {"iterations": [r.iterations for r in rungs],
                  "termination": [r.termination for r in rungs], "wall_s": wall}


CASES = {
    "c5_1m_fixed15": lambda: rigid_case("c5_1m_fixed15", 1_000_000, 1e-30, 15),
    "c5_1m_conv": lambda: rigid_case("c5_1m_conv", 1_000_000, 2e-4, 250),
    "p100k_conv": lambda: rigid_case("p100k_conv", 100_000, 2e-4, 250),
    "p100k_fixed50": lambda: rigid_case("p100k_fixed50", 100_000, 1e-30, 50),
    "c2": lambda: c2_case(),
    "c3": lambda: c3_case(),
    "c4": lambda: c4_case(),
    "gn3_pt2pl": lambda: c2_case("gn3_pt2pl", n=20000, gn=3, iters=30),
    "gn3_chain6_pt2pl": lambda: c3_case("gn3_chain6_pt2pl", links=6, per_link=480, seed=1,
                                        normals=True, gn=3),
    "gn2_strip2k": lambda: c4_case("gn2_strip2k", n=2000, spacing=0.03, iters=12, gn=2),
    "ladder_p10k": lambda: ladder_case(),
}


def _run(name):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    res = CASES[name]()
    print(json.dumps({res[0]: res[1]}), flush=True)
    return res


def main():
    names = sys.argv[1:] or list(CASES)
    with Pool(min(len(names), 6)) as pool:
        out = pool.map(_run, names, chunksize=1)
    path = os.path.join(HERE, "MANIFEST_configs.json")
    meta = json.load(open(path)) if os.path.exists(path) else {}
    meta.update(dict(out))
    with open(path, "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    main()
