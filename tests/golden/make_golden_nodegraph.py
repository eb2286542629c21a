"""Golden node-graph (deformable) fixtures from the LIVE reference (C4 family).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_nodegraph.py

The warped-strip setup of test_acceptance.py:414-440 at reduced size: a flat
strip registered onto its sine-warped copy with a node graph (greedy spacing
sampler, 4-NN Gaussian skinning, ARAP weight lambda_reg)."""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import twistreg as T  # noqa: E402
from twistreg.synth import flat_strip  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def warp(p):
    q = p.copy()
    q[:, 2] += 0.04 * np.sin(np.pi * (q[:, 0] + 0.15) / 0.3)
    return q


def main():
    meta = {}
    for name, n_pts, spacing, mode, iters in (("strip2k", 2000, 0.03, "point_to_point", 12),
                                              ("strip6k_pt2pl", 6000, 0.018, "point_to_plane", 8)):
        pts = f32(flat_strip(n_points=n_pts))
        nodes, edges = T.build_node_graph(pts, spacing=spacing)
        skin = T.bind_points_to_nodes(pts, nodes, radius=2.0 * spacing)
        graph = T.NodeGraph(nodes, edges, skin)
        obs = f32(warp(pts))
        normals = None
        obs_n = None
        if mode == "point_to_plane":
            # analytic unit normals of the warped strip z = f(x)
            slope = 0.04 * np.pi / 0.3 * np.cos(np.pi * (pts[:, 0] + 0.15) / 0.3)
            nn = np.stack([-slope, np.zeros_like(slope), np.ones_like(slope)], axis=1)
            obs_n = f32(nn / np.linalg.norm(nn, axis=1, keepdims=True))
            normals = np.tile([0.0, 0.0, 1.0], (len(pts), 1))
        cfg = dict(sigma=0.02, w=0.1, lambda_reg=0.1, max_iters=iters, tol=1e-5, mode=mode)
        config = T.RegistrationConfig(
            gmm=T.GmmConfig(sigma=cfg["sigma"], outlier_ratio=cfg["w"]), residual_mode=mode,
            max_em_iters=iters, twist_tolerance=cfg["tol"],
            mstep=T.MStepOptions(lambda_reg=cfg["lambda_reg"]))
        r = T.register(T.PointCloud(pts, normals=normals), T.PointCloud(obs, normals=obs_n),
                       graph, config)
        est = r.kinematics
        moved = T.forward_points(T.PointCloud(pts), est).positions
        extra = {"N": normals, "YN": obs_n} if normals is not None else {}
        np.savez_compressed(
            os.path.join(HERE, f"nodegraph_{name}.npz"), X=pts, Y=obs, nodes=nodes, edges=edges,
            skin_idx=skin.indices, skin_w=skin.weights,
            node_R=np.stack([t.rotation for t in est.node_transforms]),
            node_t=np.stack([t.translation for t in est.node_transforms]), moved=moved,
            objectives=np.asarray(r.objectives), twist_norms=np.asarray(r.twist_norms),
            iterations=r.iterations, termination=r.termination, config=json.dumps(cfg), **extra)
        err0 = float(np.linalg.norm(pts - warp(pts), axis=1).mean())
        err1 = float(np.linalg.norm(moved - warp(pts), axis=1).mean())
        meta[name] = {"nodes": len(nodes), "iterations": r.iterations,
                      "termination": r.termination, "error_before": err0, "error_after": err1}
    with open(os.path.join(HERE, "MANIFEST_nodegraph.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
