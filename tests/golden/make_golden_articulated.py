"""Golden articulated-registration fixtures from the LIVE reference (C3 family).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_articulated.py

Trees are stored as plain arrays (parent, joint frame R/t, joint kind/axis) so
both the reference and the B200 package can rebuild them; inputs are float32-
rounded like every other fixture.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import twistreg as T  # noqa: E402
from twistreg.synth import _cylinder, two_link_chain  # noqa: E402

KINDS = {"fixed": 0, "revolute": 1, "prismatic": 2}


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def tree_arrays(tree):
    bodies = tree.bodies
    return dict(parent=np.array([b.parent for b in bodies]),
                frame_R=np.stack([b.transform.rotation for b in bodies]),
                frame_t=np.stack([b.transform.translation for b in bodies]),
                kind=np.array([KINDS[b.joint.kind] for b in bodies]),
                axis=np.stack([b.joint.axis if b.joint.axis is not None else np.zeros(3)
                               for b in bodies]),
                floating=np.array(tree.floating))


def chain(n_links, per_link, seed, normals=False):
    rng = np.random.default_rng(seed)
    bodies = [T.Body("base", -1, T.RigidTransform.identity(), T.Joint("fixed"))]
    for i in range(n_links):
        axis = np.array([0.0, 0.0, 1.0]) if i % 2 == 0 else np.array([0.0, 1.0, 0.0])
        bodies.append(T.Body(f"link{i}", i, T.RigidTransform(np.eye(3), np.array([0.05, 0, 0])),
                             T.Joint("revolute", axis)))
    n_around = 24
    n_axial = max(2, per_link // n_around)
    cyl = _cylinder(n_axial, n_around, 0.012, 0.05)
    nrm = np.stack([np.zeros(len(cyl)), cyl[:, 1], cyl[:, 2]], axis=-1) / 0.012
    pts = np.concatenate([cyl] * (n_links + 1))
    nr = np.concatenate([nrm] * (n_links + 1))
    labels = np.repeat(np.arange(n_links + 1), len(cyl))
    rest = T.ArticulatedTree(bodies, floating=True, point_bodies=labels)
    base = T.RigidTransform(T.rotation_about_axis(rng.standard_normal(3), 0.05),
                            0.003 * rng.standard_normal(3))
    gt = rest.with_joint_values(0.05 * rng.standard_normal(n_links), base_pose=base)
    return f32(pts), (f32(nr) if normals else None), labels, rest, gt


def main():
    meta = {}
    cases = []
    ref, rest = two_link_chain()
    gt = rest.with_joint_values([0.2, -0.15], base_pose=T.RigidTransform(
        T.rotation_about_axis([0.3, 1.0, 0.2], 0.05), np.array([0.003, -0.002, 0.001])))
    cases.append(("two_link", f32(ref.positions), None, rest.point_bodies, rest, gt,
                  dict(sigma=0.006, w=0.1, max_iters=15, tol=1e-5, mode="point_to_point")))
    P, _, lab, rest, gt = chain(20, 240, seed=0)
    cases.append(("chain20", P, None, lab, rest, gt,
                  dict(sigma=0.006, w=0.1, max_iters=15, tol=1e-5, mode="point_to_point")))
    P, N, lab, rest, gt = chain(6, 480, seed=1, normals=True)
    cases.append(("chain6_pt2pl", P, N, lab, rest, gt,
                  dict(sigma=0.006, w=0.1, max_iters=15, tol=1e-5, mode="point_to_plane")))
    for name, P, N, lab, rest, gt, cfg in cases:
        reference = T.PointCloud(P, normals=N)
        obs = T.forward_points(reference, gt)
        Y = f32(obs.positions)
        YN = f32(obs.normals) if N is not None else None
        config = T.RegistrationConfig(gmm=T.GmmConfig(sigma=cfg["sigma"], outlier_ratio=cfg["w"]),
                                      residual_mode=cfg["mode"], max_em_iters=cfg["max_iters"],
                                      twist_tolerance=cfg["tol"])
        r = T.register(reference, T.PointCloud(Y, normals=YN), rest, config)
        est = r.kinematics
        extra = {"N": N, "YN": YN} if N is not None else {}
        np.savez_compressed(
            os.path.join(HERE, f"articulated_{name}.npz"), X=P, Y=Y, labels=lab,
            joint_values=est.joint_values, base_R=est.base_pose.rotation,
            base_t=est.base_pose.translation, gt_joints=gt.joint_values,
            objectives=np.asarray(r.objectives), twist_norms=np.asarray(r.twist_norms),
            iterations=r.iterations, termination=r.termination, config=json.dumps(cfg),
            **tree_arrays(rest), **extra)
        meta[name] = {"iterations": r.iterations, "termination": r.termination,
                      "joint_err_vs_gt": float(np.abs(est.joint_values - gt.joint_values).max())}
    with open(os.path.join(HERE, "MANIFEST_articulated.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
