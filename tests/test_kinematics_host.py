"""Host kinematics of the drop-in API (CPU): spatial velocity Jacobians against
central finite differences of the forward kinematics (the reference's own
oracle, test_kinematics.py:109-197), update semantics, DQ blend."""
import numpy as np

import paper_1811_10136_b200 as fr
from paper_1811_10136_b200.geometry import nearest_rotation
from paper_1811_10136_b200.kinematics import (ArticulatedTree, Body, Joint, NodeGraph, Skinning,
                                              bind_points_to_nodes, build_node_graph)


def random_tree(rng, n=5):
    bodies = [Body("base", -1, fr.RigidTransform())]
    for i in range(1, n):
        kind = "prismatic" if i % 3 == 0 else "revolute"
        bodies.append(Body(f"l{i}", int(rng.integers(0, i)),
                           fr.RigidTransform(fr.rotation_about_axis(rng.standard_normal(3), 0.3),
                                             0.05 * rng.standard_normal(3)),
                           Joint(kind, rng.standard_normal(3))))
    return bodies


def test_spatial_jacobians_match_finite_differences():
    rng = np.random.default_rng(0)
    bodies = random_tree(rng, 6)
    tree = ArticulatedTree(bodies, floating=True, joint_values=0.3 * rng.standard_normal(5),
                           base_pose=fr.RigidTransform(fr.rotation_about_axis([1, 2, 3], 0.4),
                                                       [0.1, -0.2, 0.05]))
    J = tree.spatial_velocity_jacobians()
    eps = 1e-6
    for p in range(tree.n_params):
        d = np.zeros(tree.n_params)
        d[p] = eps
        tp, tm = tree.updated(d), tree.updated(-d)
        for b in range(tree.n_bodies):
            Rp, Rm = tp.body_pose(b).rotation, tm.body_pose(b).rotation
            W = (Rp - Rm) / (2 * eps) @ tree.body_pose(b).rotation.T
            omega = np.array([W[2, 1], W[0, 2], W[1, 0]])
            x = tree.body_pose(b).translation
            v = (tp.body_pose(b).translation - tm.body_pose(b).translation) / (2 * eps)
            # point velocity at the body origin: omega x x + v_lin
            np.testing.assert_allclose(omega, J[b, :3, p], atol=1e-6)
            np.testing.assert_allclose(v, np.cross(J[b, :3, p], x) + J[b, 3:, p], atol=1e-6)


def test_updates_and_rigid_single_body():
    bodies = [Body("base", -1, fr.RigidTransform())]
    tree = ArticulatedTree(bodies, floating=True)
    tw = np.array([0.01, -0.02, 0.03, 0.001, 0.002, -0.003])
    a = tree.updated(tw).body_pose(0)
    b = fr.RigidModel().updated(tw).pose
    assert a.almost_equal(b, 1e-15)
    assert np.allclose(nearest_rotation(a.rotation), a.rotation)


def test_node_graph_identity_blend_and_binding():
    pts = np.stack(np.meshgrid(np.linspace(0, 0.1, 20), np.linspace(0, 0.05, 10)), -1)
    pts = np.concatenate([pts.reshape(-1, 2), np.zeros((200, 1))], axis=1)
    nodes, edges = build_node_graph(pts, 0.02)
    sk = bind_points_to_nodes(pts, nodes, 0.04)
    g = NodeGraph(nodes, edges, sk)
    R, t = g.point_transforms()
    np.testing.assert_allclose(R, np.tile(np.eye(3), (len(pts), 1, 1)), atol=1e-12)
    np.testing.assert_allclose(t, 0.0, atol=1e-12)
    assert isinstance(sk, Skinning) and len(edges) > 0
