"""The reference's FilterReg registration protocol: the coarse-to-fine kernel
width ladder of corrupted bench trials (bench.py:31-38, 66-78, 87-110 of
pkg/src/twistreg), run on the device.

`filterreg_protocol` returns the reference's per-rung (GmmConfig,
max_em_iters, twist_tolerance) list; `register_ladder` runs the rungs warm-
started from each other, as `bench.run_trial` does with `register` per rung,
but uploads the clouds once: every rung rebuilds only the observation lattice
at its kernel width (splat + blur of the resident float64 planes) and runs
the device EM loop from the previous rung's pose.
"""

from __future__ import annotations

import time

from .estep import GmmConfig
from .geometry import PointCloud, RigidTransform
from .kinematics import RigidModel
from .pipeline import RegistrationConfig, RegistrationResult, register

# corruption ladder: sigma fractions of the bbox diagonal and per-rung caps
# (bench.py:34-35)
LADDER_FRACS = (0.05, 0.03, 0.02, 0.014)
LADDER_CAPS = (60, 60, 60, 250)
CLEAN_SIGMA_FRAC = 0.05
CLEAN_MAX_ITERS = 250
CLEAN_TOLERANCE = 2e-4


def filterreg_protocol(corrupted: bool, diameter: float, outliers: bool = True):
    """Per-rung (GmmConfig, max_em_iters, twist_tolerance) (bench.py:66-78).

    Clean tasks get a single fixed-width run; corrupted tasks get the
    coarse-to-fine ladder with the outlier weight raised to 0.3 when outliers
    are present.  `corrupted` / `outliers` stand for the reference's
    ExperimentSpec.corrupted / outlier_ratio > 0."""
    if not corrupted:
        gmm = GmmConfig(sigma=CLEAN_SIGMA_FRAC * diameter, outlier_ratio=0.1)
        return [(gmm, CLEAN_MAX_ITERS, CLEAN_TOLERANCE)]
    w = 0.3 if outliers else 0.1
    return [(GmmConfig(sigma=frac * diameter, outlier_ratio=w), cap, 1e-4)
            for frac, cap in zip(LADDER_FRACS, LADDER_CAPS)]


def register_ladder(reference: PointCloud, observation: PointCloud, rungs,
                    initial_model: RigidModel | None = None, timing: dict | None = None,
                    config: RegistrationConfig | None = None) -> list:
    """Run `rungs` = [(GmmConfig, max_em_iters, twist_tolerance), ...] warm-
    started (bench.py:95-107): rigid point-to-point, fixed width per rung.
    Returns one RegistrationResult per rung; the last one's kinematics is
    the protocol's final pose.  `config` supplies the remaining
    RegistrationConfig fields (M-step options)."""
    from . import _rigid
    from .pipeline import _device_loop_result
    state = initial_model if initial_model is not None else RigidModel(RigidTransform.identity())
    base = config if config is not None else RegistrationConfig()
    rungs = list(rungs)
    if not rungs:
        return []
    if base.residual_mode != "point_to_point" or base.record_states or \
            any(g.update_sigma or g.mode != "position" for g, _, _ in rungs):
        # the general path: register() per rung, as the reference
        out = []
        for gmm, cap, tol in rungs:
            cfg = RegistrationConfig(gmm=gmm, residual_mode=base.residual_mode,
                                     backend=base.backend, max_em_iters=cap,
                                     twist_tolerance=tol, mstep=base.mstep,
                                     record_states=base.record_states)
            res = register(reference, observation, state, cfg, timing=timing)
            state = res.kinematics
            out.append(res)
        return out
    tick = time.perf_counter()
    path = _rigid.RigidDevicePath(reference, observation, rungs[0][0], "point_to_point",
                                  precision=_rigid.PRECISION)
    out = []
    for k, (gmm, cap, tol) in enumerate(rungs):
        if k > 0:
            path.gmm = gmm
            path.build(gmm.sigma)          # the lattice at this rung's width
        cfg = RegistrationConfig(gmm=gmm, max_em_iters=cap, twist_tolerance=tol,
                                 mstep=base.mstep)
        em = _rigid.device_em(path, state.pose.rotation, state.pose.translation, cfg)
        em.run()
        res = _device_loop_result(em, state, None, 0.0)
        state = res.kinematics
        out.append(res)
    if timing is not None:
        timing["e_step_s"] = timing.get("e_step_s", 0.0) + time.perf_counter() - tick
        timing["m_step_s"] = timing.get("m_step_s", 0.0)
        timing["iterations"] = sum(r.iterations for r in out)
    return out


def ladder_result(results) -> RegistrationResult:
    """The rungs folded into one RegistrationResult (traces concatenated,
    iterations summed; termination of the last rung)."""
    res = RegistrationResult(kinematics=results[-1].kinematics,
                             iterations=sum(r.iterations for r in results))
    for r in results:
        res.objectives += list(r.objectives)
        res.twist_norms += list(r.twist_norms)
        res.inlier_masses += list(r.inlier_masses)
    res.termination = results[-1].termination
    return res
