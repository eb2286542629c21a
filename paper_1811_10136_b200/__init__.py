"""B200-native FilterReg engine (arxiv 1811.10136) -- drop-in for the
reference `twistreg` package's hot path.

Same API names as twistreg (`register`, `RegistrationConfig`, `GmmConfig`,
`MomentEngine`, `compute_moments`, `PermutohedralLattice`, `build_lattice`,
...); the point work runs in hand-written sm_100a kernels
(libfilterreg_b200.so, C ABI in include/filterreg_b200.h) on HBM-resident
float32 SoA point planes and an HBM hash-table lattice.

Typical use::

    from paper_1811_10136_b200 import GmmConfig, RegistrationConfig, RigidModel, register
    config = RegistrationConfig(gmm=GmmConfig(sigma=0.01, outlier_ratio=0.1))
    result = register(model, observation, RigidModel(), config)
"""

from .errors import (BindingError, DegenerateBlendError, DegenerateCorrespondenceError,
                     ParseError, SolverError)
from .estep import GmmConfig, MomentEngine, MomentField, compute_moments, outlier_constant, \
    update_sigma
from .geometry import PointCloud, RigidTransform, apply_twist, rotation_about_axis, twist_exp
from .kinematics import (ArticulatedTree, Body, Joint, NodeGraph, RigidModel, Skinning,
                         articulated_from_dict, bind_points_to_nodes, build_node_graph,
                         forward_points, load_articulated_model)
from .mstep import (MStepOptions, NormalEquations, ResidualSpec, assemble_articulated,
                    assemble_nodegraph, assemble_rigid, gn_solve, m_step, objective,
                    residuals_from_moments)
from .permutohedral import (PermutohedralLattice, build_lattice, filter_augmented,
                            gaussian_transform_bruteforce, valid_lattice_key)
from .hostmem import pinned_cloud, pinned_copy, pinned_empty
from .io import load_cloud, save_cloud
from .pipeline import (RegistrationConfig, RegistrationResult, alignment_error, default_sigma,
                       log_likelihood, register, register_batch, update_magnitude)
from .protocol import filterreg_protocol, ladder_result, register_ladder

__version__ = "0.1.0"

__all__ = [
    "ArticulatedTree", "BindingError", "Body", "DegenerateBlendError",
    "DegenerateCorrespondenceError", "GmmConfig", "Joint", "MStepOptions", "MomentEngine",
    "MomentField", "NodeGraph", "NormalEquations", "ParseError", "PermutohedralLattice",
    "PointCloud", "RegistrationConfig", "RegistrationResult", "ResidualSpec", "RigidModel",
    "RigidTransform", "Skinning", "SolverError", "alignment_error", "apply_twist",
    "articulated_from_dict", "assemble_articulated", "assemble_nodegraph", "assemble_rigid",
    "bind_points_to_nodes", "build_lattice", "build_node_graph", "compute_moments",
    "default_sigma", "filter_augmented", "filterreg_protocol", "forward_points",
    "gaussian_transform_bruteforce", "ladder_result", "register_ladder",
    "gn_solve", "load_articulated_model", "log_likelihood", "m_step", "objective",
    "outlier_constant", "load_cloud", "save_cloud", "pinned_cloud", "pinned_copy",
    "pinned_empty", "register", "register_batch", "residuals_from_moments", "rotation_about_axis",
    "twist_exp", "update_magnitude", "update_sigma", "valid_lattice_key",
]
