"""Closed-form rigid M-step math (paper_1811_10136_b200/_rigid.py) against the
oracle's per-point assembly and objective (oracle/filterreg_oracle.py, which
restates mstep.py:102-210).  CPU only: the statistics are formed here in NumPy
exactly as the device pass defines them."""

import numpy as np
import pytest

from oracle import filterreg_oracle as O
from paper_1811_10136_b200._rigid import RigidMoments
from paper_1811_10136_b200.geometry import RigidTransform, apply_twist


def stats(x, c, w, t):
    y = x - c
    r = x - t
    s = [w.sum()]
    s += list((w[:, None] * y).sum(0))
    S2 = np.einsum("n,ni,nj->ij", w, y, y)
    s += [S2[0, 0], S2[0, 1], S2[0, 2], S2[1, 1], S2[1, 2], S2[2, 2]]
    s += list((w[:, None] * r).sum(0))
    s += list(np.einsum("n,nj,nk->jk", w, r, y).reshape(-1))
    s += list((w[:, None] * r * r).sum(0))
    return np.array(s)


@pytest.fixture
def problem():
    rng = np.random.default_rng(3)
    m = 400
    ref = rng.uniform(-0.1, 0.1, (m, 3)) + np.array([0.3, -0.2, 0.5])
    R = O.rotation_about_axis([0.3, 1.0, -0.2], 0.4)
    t = np.array([0.01, 0.02, -0.03])
    x = ref @ R.T + t
    w = rng.uniform(0.0, 1.0, m)
    w[rng.random(m) < 0.1] = 0.0
    tg = x + rng.normal(scale=0.004, size=(m, 3))
    sinv = 1.0 / np.array([0.007, 0.009, 0.011])
    return ref, R, t, x, w, tg, sinv


def test_normal_equations_match_oracle(problem):
    ref, R, t, x, w, tg, sinv = problem
    c = x.mean(0) + 0.01
    mom = RigidMoments.from_sums(stats(x, c, w, tg))
    H, g = mom.normal_equations(c, sinv ** 2)
    spec = (w, tg, sinv, "point_to_point", None, None)
    Ho, go = O.assemble_rigid(spec, x)
    np.testing.assert_allclose(H, Ho, rtol=1e-10, atol=1e-9 * np.abs(Ho).max())
    np.testing.assert_allclose(g, go, rtol=1e-10, atol=1e-9 * np.abs(go).max())
    assert mom.energy(sinv ** 2) == pytest.approx(O.rigid_objective(spec, x), rel=1e-12)


def test_candidate_energy_change_matches_direct(problem):
    ref, R, t, x, w, tg, sinv = problem
    c = x.mean(0)
    mom = RigidMoments.from_sums(stats(x, c, w, tg))
    spec = (w, tg, sinv, "point_to_point", None, None)
    E0 = O.rigid_objective(spec, x)
    T = RigidTransform(R, t)
    for tw in ([1e-3, -2e-3, 5e-4, 1e-4, -2e-4, 3e-4], [0.2, 0.1, -0.3, 0.01, 0.0, -0.02],
               [1e-7, 0, 0, 0, 1e-8, 0]):
        C = apply_twist(np.array(tw), T)
        D = C.rotation @ R.T
        delta = C.translation - D @ t
        dE = mom.delta_energy(D, delta, c, sinv ** 2)
        direct = O.rigid_objective(spec, ref @ C.rotation.T + C.translation) - E0
        assert abs(dE - direct) <= 1e-13 * E0 + 1e-9 * abs(direct)


def test_moved_statistics_equal_recomputed(problem):
    ref, R, t, x, w, tg, sinv = problem
    c = x.mean(0)
    mom = RigidMoments.from_sums(stats(x, c, w, tg))
    C = apply_twist(np.array([0.05, -0.02, 0.03, 0.004, 0.0, -0.002]), RigidTransform(R, t))
    D = C.rotation @ R.T
    delta = C.translation - D @ t
    moved = mom.moved(D, delta, c)
    x2 = ref @ C.rotation.T + C.translation
    direct = RigidMoments.from_sums(stats(x2, c, w, tg))
    for name in ("S1", "S2", "R1", "RX", "Q"):
        np.testing.assert_allclose(getattr(moved, name), getattr(direct, name),
                                   rtol=1e-9, atol=1e-15)


def test_block_system_dict_and_arrays_agree():
    """NormalEquations block systems: the dict form and the block-array form
    (repeated keys add up) give the same dense A, trace and sparse solution."""
    import paper_1811_10136_b200.mstep as M
    rng = np.random.default_rng(3)
    nb = 9
    blocks = {}
    keys, vals = [], []
    for k in range(nb):
        G = rng.standard_normal((6, 6))
        blk = G @ G.T + 6 * np.eye(6)
        blocks[(k, k)] = blk
        half = 0.5 * blk
        keys += [(k, k), (k, k)]
        vals += [half, blk - half]
    for _ in range(12):
        k, l = sorted(rng.choice(nb, 2, replace=False))
        blk = 0.1 * rng.standard_normal((6, 6))
        blocks[(k, l)] = blocks.get((k, l), 0) + blk
        keys.append((k, l))
        vals.append(blk)
    b = rng.standard_normal(6 * nb)
    eq_d = M.NormalEquations(6 * nb, b=b, blocks=blocks)
    eq_a = M.NormalEquations(6 * nb, b=b, block_arrays=(np.array(keys), np.array(vals)))
    np.testing.assert_allclose(eq_d.to_dense(), eq_a.to_dense(), rtol=0, atol=1e-12)
    assert eq_d.trace() == pytest.approx(eq_a.trace(), rel=1e-14)
    x_d = M.gn_solve(eq_d, damping=1e-3, method="sparse")
    x_a = M.gn_solve(eq_a, damping=1e-3, method="sparse")
    x_dense = M.gn_solve(eq_a, damping=1e-3, method="dense")
    np.testing.assert_allclose(x_d, x_a, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(x_a, x_dense, rtol=1e-9, atol=1e-12)
