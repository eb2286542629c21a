"""Standalone M-step API on the device (mirrors pkg/tests/test_mstep.py):
every assembler against dense per-point chain-rule oracles, SPD / sparse
solves, objective never increases across accepted steps."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fr():
    import paper_1811_10136_b200 as fr
    return fr


def random_spec(fr, rng, m, mode="point_to_point"):
    w = rng.uniform(0.2, 1.0, m)
    w[rng.random(m) < 0.1] = 0.0
    tg = rng.uniform(-0.2, 0.2, (m, 3))
    sinv = 1.0 / rng.uniform(0.02, 0.1, 3)
    n = valid = None
    if mode == "point_to_plane":
        n = rng.standard_normal((m, 3))
        n /= np.linalg.norm(n, axis=1, keepdims=True)
        valid = rng.random(m) > 0.2
        n[~valid] = 0.0
    return fr.ResidualSpec(w, tg, sinv, mode, n, valid)


def rows(spec, x, i):
    from paper_1811_10136_b200.geometry import skew
    w = spec.weights[i]
    d = x[i] - spec.targets[i]
    if spec.mode == "point_to_point":
        P = np.sqrt(w) * np.diag(spec.sigma_inv)
    elif spec.normal_valid[i]:
        P = np.sqrt(w) * spec.normals[i][None, :]
    else:
        P = np.sqrt(w) * np.eye(3)
    return P @ np.hstack([-skew(x[i]), np.eye(3)]), P @ d


def random_tree(fr, rng, n_moving=3, m=300):
    from paper_1811_10136_b200.kinematics import ArticulatedTree, Body, Joint
    bodies = [Body("root", -1, fr.RigidTransform(), Joint())]
    for i in range(n_moving):
        bodies.append(Body(f"b{i}", int(rng.integers(0, i + 1)),
                           fr.RigidTransform(fr.rotation_about_axis(rng.standard_normal(3), 0.3),
                                             0.05 * rng.standard_normal(3)),
                           Joint("revolute" if i % 2 == 0 else "prismatic",
                                 rng.standard_normal(3))))
    return ArticulatedTree(bodies, floating=True, joint_values=0.2 * rng.standard_normal(n_moving),
                           point_bodies=rng.integers(0, n_moving + 1, m))


@pytest.mark.parametrize("mode", ["point_to_point", "point_to_plane"])
def test_articulated_matches_dense(fr, mode):
    rng = np.random.default_rng(1)
    m = 300
    tree = random_tree(fr, rng, m=m)
    spec = random_spec(fr, rng, m, mode)
    x = rng.uniform(-0.2, 0.2, (m, 3))
    eq = fr.assemble_articulated(spec, x, tree)
    A = np.zeros((tree.n_params,) * 2)
    b = np.zeros(tree.n_params)
    for i in range(m):
        if spec.weights[i] == 0:
            continue
        G, r = rows(spec, x, i)
        G = G @ tree.spatial_velocity_jacobian(int(tree.point_bodies[i]))
        A += G.T @ G
        b += G.T @ r
    np.testing.assert_allclose(eq.A, A, rtol=1e-9, atol=1e-10 * np.abs(A).max())
    np.testing.assert_allclose(eq.b, b, rtol=1e-9, atol=1e-10 * np.abs(b).max())


def small_graph(fr, rng, n_pts=400, n_nodes=6):
    from paper_1811_10136_b200.kinematics import NodeGraph, bind_points_to_nodes
    pts = rng.uniform(-0.1, 0.1, (n_pts, 3))
    nodes = pts[rng.choice(n_pts, n_nodes, replace=False)]
    edges = np.array([(i, j) for i in range(n_nodes) for j in range(i + 1, n_nodes)])
    sk = bind_points_to_nodes(pts, nodes, radius=0.25)
    g = NodeGraph(nodes, edges, sk)
    return pts, g.updated(0.05 * rng.standard_normal(g.n_params))


def test_nodegraph_matches_dense(fr):
    from paper_1811_10136_b200.kinematics import forward_points
    rng = np.random.default_rng(2)
    pts, graph = small_graph(fr, rng)
    spec = random_spec(fr, rng, len(pts))
    x = forward_points(fr.PointCloud(pts), graph).positions
    eq = fr.assemble_nodegraph(spec, x, graph, lambda_reg=0.3)
    n = graph.n_nodes
    A = np.zeros((6 * n, 6 * n))
    b = np.zeros(6 * n)
    for i in range(len(pts)):
        if spec.weights[i] == 0:
            continue
        G, r = rows(spec, x, i)
        J = np.zeros((G.shape[0], 6 * n))
        for s in range(graph.skinning.indices.shape[1]):
            k, wk = graph.skinning.indices[i, s], graph.skinning.weights[i, s]
            if k >= 0 and wk > 0:
                J[:, 6 * k:6 * k + 6] += wk * G
        A += J.T @ J
        b += J.T @ r
    from paper_1811_10136_b200.geometry import skew
    root = np.sqrt(0.3)
    for k, l in graph.edges:
        for p in (graph.node_positions[l], graph.node_positions[k]):
            xk = graph.node_transforms[k].apply(p[None])[0]
            xl = graph.node_transforms[l].apply(p[None])[0]
            J = np.zeros((3, 6 * n))
            J[:, 6 * k:6 * k + 6] = root * np.hstack([-skew(xk), np.eye(3)])
            J[:, 6 * l:6 * l + 6] = -root * np.hstack([-skew(xl), np.eye(3)])
            A += J.T @ J
            b += J.T @ (root * (xk - xl))
    np.testing.assert_allclose(eq.to_dense(), A, rtol=1e-9, atol=1e-10 * np.abs(A).max())
    np.testing.assert_allclose(eq.b, b, rtol=1e-9, atol=1e-10 * np.abs(b).max())
    # sparse (SuperLU) solve equals the dense Cholesky solve
    s1 = fr.gn_solve(eq, method="sparse")
    s2 = fr.gn_solve(eq, method="dense")
    np.testing.assert_allclose(s1, s2, rtol=1e-8, atol=1e-12)


def test_objective_never_increases(fr):
    rng = np.random.default_rng(46)
    opts = fr.MStepOptions(max_gn_iters=6, lambda_reg=0.2)
    for _ in range(3):
        m = int(rng.integers(40, 120))
        spec = random_spec(fr, rng, m)
        ref = fr.PointCloud(rng.uniform(-0.3, 0.3, (m, 3)))
        models = [fr.RigidModel(fr.RigidTransform(
            fr.rotation_about_axis(rng.standard_normal(3), rng.uniform(0, 0.4)),
            rng.uniform(-0.05, 0.05, 3))), random_tree(fr, rng, n_moving=2, m=m)]
        for model in models:
            _, diag = fr.m_step(spec, ref, model, opts)
            obj = np.asarray(diag.objectives)
            assert np.all(np.diff(obj) / np.maximum(1.0, np.abs(obj[:-1])) <= 1e-12)
        pts, graph = small_graph(fr, rng, n_pts=m, n_nodes=3)
        _, diag = fr.m_step(random_spec(fr, rng, m), fr.PointCloud(pts), graph, opts)
        obj = np.asarray(diag.objectives)
        assert np.all(np.diff(obj) / np.maximum(1.0, np.abs(obj[:-1])) <= 1e-12)
