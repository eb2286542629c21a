"""Sharded registration host logic on CPU: world size 2 over gloo.

The device pass is replaced by an oracle-backed stand-in (test infrastructure)
that returns the same 25 point-to-point statistics the CUDA pass produces for
its shard; everything else -- global centre / diameter / model count, the
all-reduce of the partials, the M step and termination on every rank -- is the
product's `register(..., process_group=...)` path.  Two ranks holding half the
model points each must reproduce the single-process result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import filterreg_oracle as O


class OraclePath:
    """Implements the RigidDevicePath interface on CPU with the oracle."""

    mode = 0

    def __init__(self, reference, observation, gmm, residual_mode, process_group=None):
        assert residual_mode == "point_to_point" and not gmm.update_sigma
        self.group = process_group
        P = np.asarray(reference.positions, dtype=float)
        self.P, self.M = P, len(P)
        tot = self._allreduce(np.concatenate([[float(self.M)], P.sum(axis=0)]), "sum")
        self.M_total = int(round(tot[0]))
        self.c_ref = tot[1:] / tot[0]
        lo = self._allreduce(P.min(axis=0), "min")
        hi = self._allreduce(P.max(axis=0), "max")
        self.diameter = float(np.linalg.norm(hi - lo))
        self.Y = np.asarray(observation.positions, dtype=float)
        self.N = len(self.Y)
        self.gmm = gmm
        self.width = 25
        self.build(gmm.sigma)

    def _allreduce(self, v, op):
        v = np.asarray(v, dtype=float)
        if self.group is None:
            return v
        t = torch.from_numpy(v.copy())
        dist.all_reduce(t, op={"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN,
                               "max": dist.ReduceOp.MAX}[op], group=self.group)
        return t.numpy()

    def build(self, sigma):
        s = np.atleast_1d(np.asarray(sigma, dtype=float))
        self.sigma = np.full(3, s[0]) if s.size == 1 else s
        self.lat = O.build_lattice(self.Y, O.obs_value_columns(self.Y), self.sigma)
        self.c_prime = O.outlier_constant(self.gmm.outlier_ratio, self.N, self.M_total, self.sigma)

    def centre(self, R, t):
        return np.asarray(R) @ self.c_ref + np.asarray(t)

    def run_pass(self, R, t):
        x = self.P @ np.asarray(R).T + np.asarray(t)
        mom = O.moment_epilogue(self.lat.slice(x), x, self.c_prime)
        w, tg = mom["weight"], mom["target"]
        y = x - self.centre(R, t)
        r = x - tg
        S2 = np.einsum("n,ni,nj->ij", w, y, y)
        s = np.concatenate([[w.sum()], (w[:, None] * y).sum(0),
                            [S2[0, 0], S2[0, 1], S2[0, 2], S2[1, 1], S2[1, 2], S2[2, 2]],
                            (w[:, None] * r).sum(0), np.einsum("n,nj,nk->jk", w, r, y).ravel(),
                            (w[:, None] * r * r).sum(0)])
        return self._allreduce(s, "sum")


def _problem():
    model, obs, _ = O.pebble_pair(1200, outlier_ratio=0.05, seed=3)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    return X, Y, 0.05 * O.bbox_diameter(X[:1200])


def _run(X, Y, sigma, group):
    import paper_1811_10136_b200 as fr
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                                max_em_iters=40, twist_tolerance=2e-4)
    return fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg,
                       process_group=group, _path_factory=OraclePath)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, Y, sigma = _problem()
    bounds = np.linspace(0, len(X), world + 1).astype(int)
    res = _run(X[bounds[rank]:bounds[rank + 1]], Y, sigma, dist.group.WORLD)
    out[rank] = (res.kinematics.pose.matrix(), res.iterations, res.termination,
                 list(res.objectives))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_sharded_register_matches_single_process():
    X, Y, sigma = _problem()
    single = _run(X, Y, sigma, None)
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
        results = dict(out)
    for rank in (0, 1):
        T, iters, term, objs = results[rank]
        assert iters == single.iterations and term == single.termination
        np.testing.assert_allclose(T, single.kinematics.pose.matrix(), atol=1e-10)
        np.testing.assert_allclose(objs, single.objectives, rtol=1e-9)
    # identical decisions on every rank
    assert np.array_equal(results[0][0], results[1][0])
