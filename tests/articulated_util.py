"""Rebuild golden articulated trees with the B200 package's classes."""
import numpy as np

KINDS = {0: "fixed", 1: "revolute", 2: "prismatic"}


def tree_from_arrays(fr_pkg, g, joint_values=None, base_pose=None):
    from paper_1811_10136_b200.kinematics import ArticulatedTree, Body, Joint
    bodies = []
    for i in range(len(g["parent"])):
        kind = KINDS[int(g["kind"][i])]
        joint = Joint(kind, g["axis"][i] if kind != "fixed" else None)
        bodies.append(Body(f"b{i}", int(g["parent"][i]),
                           fr_pkg.RigidTransform(g["frame_R"][i], g["frame_t"][i]), joint))
    return ArticulatedTree(bodies, floating=bool(g["floating"]), joint_values=joint_values,
                           base_pose=base_pose, point_bodies=np.asarray(g["labels"]))
