"""Node-graph registration on the GPU vs the live reference's golden traces
(tests/golden/make_golden_nodegraph.py), and the device block-sparse assembly
vs a dense per-point chain-rule restatement (test_mstep.py:89-116 style)."""
import json
import os

import numpy as np
import pytest

from oracle import filterreg_oracle as O

from .conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fr():
    import paper_1811_10136_b200 as fr
    return fr


def graph_from(fr, g):
    from paper_1811_10136_b200.kinematics import NodeGraph, Skinning
    return NodeGraph(g["nodes"], g["edges"], Skinning(g["skin_idx"], g["skin_w"]))


@pytest.mark.parametrize("case", ["strip2k", "strip6k_pt2pl"])
def test_golden_nodegraph(fr, case):
    g = np.load(os.path.join(GOLDEN, f"nodegraph_{case}.npz"))
    cfg = json.loads(str(g["config"]))
    pl = cfg["mode"] == "point_to_plane"
    ref = fr.PointCloud(g["X"], normals=g["N"] if pl else None)
    obs = fr.PointCloud(g["Y"], normals=g["YN"] if pl else None)
    config = fr.RegistrationConfig(
        gmm=fr.GmmConfig(sigma=cfg["sigma"], outlier_ratio=cfg["w"]), residual_mode=cfg["mode"],
        max_em_iters=cfg["max_iters"], twist_tolerance=cfg["tol"],
        mstep=fr.MStepOptions(lambda_reg=cfg["lambda_reg"]))
    res = fr.register(ref, obs, graph_from(fr, g), config)
    assert res.iterations == int(g["iterations"]) and res.termination == str(g["termination"])
    ext = O.bbox_diameter(g["X"])
    for T, Rg, tg in zip(res.kinematics.node_transforms, g["node_R"], g["node_t"]):
        assert O.rotation_angle(T.rotation @ Rg.T) <= 1e-4
        assert np.linalg.norm(T.translation - tg) <= 1e-5 * ext
    np.testing.assert_allclose(res.objectives, g["objectives"], rtol=1e-5)


def test_nodegraph_assembly_matches_dense_oracle(fr):
    """Device data blocks + host ARAP == dense J^T J over all parameters."""
    from paper_1811_10136_b200._nodegraph import NodeGraphDevicePath, normal_equations
    from paper_1811_10136_b200.geometry import skew
    from paper_1811_10136_b200.kinematics import forward_points
    g = np.load(os.path.join(GOLDEN, "nodegraph_strip2k.npz"))
    graph = graph_from(fr, g)
    rng = np.random.default_rng(0)
    graph = graph.updated(0.01 * rng.standard_normal(graph.n_params))
    ref, obs = fr.PointCloud(g["X"]), fr.PointCloud(g["Y"])
    gmm = fr.GmmConfig(sigma=0.02, outlier_ratio=0.1)
    path = NodeGraphDevicePath(ref, obs, gmm, "point_to_point", graph)
    s2 = np.full(3, 1.0 / 0.02 ** 2)
    g4, diag, off = path.run(graph, s2)
    eq = normal_equations(graph, diag, off, path, 0.1)
    A = eq.to_dense()
    b = eq.b
    # dense oracle over the device-computed spec (w, t) at the same positions
    x = forward_points(ref, graph).positions
    rec = path.rec.cpu().numpy()
    w, tg = rec[0], rec[1:4].T
    n = graph.n_nodes
    Ad = np.zeros((6 * n, 6 * n))
    bd = np.zeros(6 * n)
    sk = graph.skinning
    for i in np.flatnonzero(w > 0):
        P = np.sqrt(w[i]) * np.diag(np.sqrt(s2))
        base = P @ np.hstack([-skew(x[i]), np.eye(3)])
        J = np.zeros((3, 6 * n))
        for slot in range(sk.indices.shape[1]):
            k, wk = sk.indices[i, slot], sk.weights[i, slot]
            if k >= 0 and wk > 0:
                J[:, 6 * k:6 * k + 6] += wk * base
        r = P @ (x[i] - tg[i])
        Ad += J.T @ J
        bd += J.T @ r
    root = np.sqrt(0.1)
    for k, l in graph.edges:
        for p in (graph.node_positions[l], graph.node_positions[k]):
            xk = graph.node_transforms[k].apply(p[None])[0]
            xl = graph.node_transforms[l].apply(p[None])[0]
            J = np.zeros((3, 6 * n))
            J[:, 6 * k:6 * k + 6] = root * np.hstack([-skew(xk), np.eye(3)])
            J[:, 6 * l:6 * l + 6] = -root * np.hstack([-skew(xl), np.eye(3)])
            Ad += J.T @ J
            bd += J.T @ (root * (xk - xl))
    np.testing.assert_allclose(A, Ad, rtol=1e-9, atol=1e-9 * np.abs(Ad).max())
    np.testing.assert_allclose(b, bd, rtol=1e-9, atol=1e-9 * np.abs(bd).max())
    # the device forward map (DQB) reproduces the host blend
    ob = 0.5 * float(np.sum(w * ((x - tg) ** 2 @ s2)))
    assert float(g4[0]) == pytest.approx(ob, rel=1e-9)


def test_gather_lists_device_equals_host():
    """The device-built gather lists equal the host builder's, entry for entry."""
    import torch
    from paper_1811_10136_b200._nodegraph import gather_lists, gather_lists_device
    g = np.load(os.path.join(GOLDEN, "nodegraph_strip6k_pt2pl.npz"))
    idx = np.asarray(g["skin_idx"], dtype=np.int64)
    wts = np.where(idx >= 0, np.asarray(g["skin_w"], dtype=float), 0.0)
    n = len(g["nodes"])
    host = gather_lists(idx, wts, n)
    dev = gather_lists_device(torch.from_numpy(idx.astype(np.int32)).cuda(),
                              torch.from_numpy(wts).cuda(), n)
    for k in ("dptr", "dent", "pptr", "pent"):
        assert np.array_equal(dev[k].cpu().numpy(), host[k]), k
    for k in ("pair_lo", "pair_hi", "codes"):
        assert np.array_equal(dev[k], host[k]), k
    assert dev["n_pairs"] == host["n_pairs"]


@pytest.mark.parametrize("case", ["strip2k", "strip6k_pt2pl"])
def test_device_loop_matches_host_loop(fr, case, monkeypatch):
    """The device-resident node-graph loop (fr_ng_em: banded system with the
    ARAP term, block-banded damped Cholesky, all halvings in one pass) equals
    the host loop (SuperLU / dense GPU factorisation, host ARAP) to round-off."""
    from paper_1811_10136_b200 import _nodegraph
    g = np.load(os.path.join(GOLDEN, f"nodegraph_{case}.npz"))
    cfg = json.loads(str(g["config"]))
    pl = cfg["mode"] == "point_to_plane"
    ref = fr.PointCloud(g["X"], normals=g["N"] if pl else None)
    obs = fr.PointCloud(g["Y"], normals=g["YN"] if pl else None)
    config = fr.RegistrationConfig(
        gmm=fr.GmmConfig(sigma=cfg["sigma"], outlier_ratio=cfg["w"]), residual_mode=cfg["mode"],
        max_em_iters=cfg["max_iters"], twist_tolerance=cfg["tol"],
        mstep=fr.MStepOptions(lambda_reg=cfg["lambda_reg"]))
    dev = fr.register(ref, obs, graph_from(fr, g), config)
    monkeypatch.setattr(_nodegraph, "DEVICE_LOOP", False)
    host = fr.register(ref, obs, graph_from(fr, g), config)
    assert dev.iterations == host.iterations and dev.termination == host.termination
    # (entrywise: acos near 1 cannot resolve round-off-level angles)
    worst = max(float(np.abs(a.rotation - b.rotation).max())
                for a, b in zip(dev.kinematics.node_transforms, host.kinematics.node_transforms))
    assert worst < 1e-9
    np.testing.assert_allclose(dev.objectives, host.objectives, rtol=1e-8)


def test_extra_gauss_newton_against_reference(fr):
    """max_gn_iters = 2 node graph (respec passes between GN iterations)
    against the live reference."""
    g = np.load(os.path.join(GOLDEN, "config_gn2_strip2k.npz"))
    config = fr.RegistrationConfig(
        gmm=fr.GmmConfig(sigma=0.02, outlier_ratio=0.1), max_em_iters=int(g["max_iters"]),
        twist_tolerance=1e-5, mstep=fr.MStepOptions(lambda_reg=0.1, max_gn_iters=2))
    res = fr.register(fr.PointCloud(g["X"].astype(float)), fr.PointCloud(g["Y"].astype(float)),
                      graph_from(fr, g), config)
    assert abs(res.iterations - int(g["iterations"])) <= 1
    ext = O.bbox_diameter(g["X"].astype(float))
    for T, Rg, tg in zip(res.kinematics.node_transforms, g["node_R"], g["node_t"]):
        assert O.rotation_angle(T.rotation @ Rg.T) <= 1e-4
        assert np.linalg.norm(T.translation - tg) <= 1e-5 * ext
