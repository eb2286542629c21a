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
from .kinematics import RigidModel, forward_points
from .mstep import MStepOptions, ResidualSpec, assemble_rigid, gn_solve, m_step, objective
from .permutohedral import (PermutohedralLattice, build_lattice, filter_augmented,
                            gaussian_transform_bruteforce, valid_lattice_key)
from .pipeline import (RegistrationConfig, RegistrationResult, alignment_error, default_sigma,
                       log_likelihood, register, update_magnitude)

__version__ = "0.1.0"

__all__ = [
    "BindingError", "DegenerateBlendError", "DegenerateCorrespondenceError", "GmmConfig",
    "MStepOptions", "MomentEngine", "MomentField", "ParseError", "PermutohedralLattice",
    "PointCloud", "RegistrationConfig", "RegistrationResult", "ResidualSpec", "RigidModel",
    "RigidTransform", "SolverError", "alignment_error", "apply_twist", "assemble_rigid",
    "build_lattice", "compute_moments", "default_sigma", "filter_augmented", "forward_points",
    "gaussian_transform_bruteforce", "gn_solve", "log_likelihood", "m_step", "objective",
    "outlier_constant", "register", "rotation_about_axis", "twist_exp", "update_magnitude",
    "update_sigma", "valid_lattice_key",
]
