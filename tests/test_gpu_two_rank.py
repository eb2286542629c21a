"""Two ranks through the product's sharded device path on one GPU: each rank
(a separate process on cuda:0) holds half of the model cloud and the whole
observation cloud, runs RigidDevicePath / DeviceEM with process_group=...,
and all-reduces its partial sums every iteration.  The group
is gloo: its all-reduce of the CUDA sums is host-mediated, so no kernel of
one rank waits on the other (the GPU only hosts both processes).  Every rank
must take the single-process decisions and reach its pose to round-off."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import filterreg_oracle as O

pytestmark = pytest.mark.gpu


def _problem(m):
    model, obs, _ = O.pebble_pair(m, outlier_ratio=0.05, seed=17)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    return X, Y, 0.05 * O.bbox_diameter(X[:m])


def _run(X, Y, sigma, group):
    import paper_1811_10136_b200 as fr
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=sigma, outlier_ratio=0.1),
                                max_em_iters=25, twist_tolerance=1e-5)
    return fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg,
                       process_group=group)


def _worker(rank, world, port, m, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, Y, sigma = _problem(m)
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


@pytest.mark.parametrize("m", [20_000, 200_000])
def test_two_rank_device_path_matches_single_process(m):
    X, Y, sigma = _problem(m)
    single = _run(X, Y, sigma, None)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_worker, args=(2, _free_port(), m, out), nprocs=2, join=True,
                           start_method="spawn")
        results = dict(out)
    T1 = single.kinematics.pose.matrix()
    for rank in (0, 1):
        T, iters, term, objs = results[rank]
        assert iters == single.iterations and term == single.termination
        assert O.rotation_angle(T[:3, :3] @ T1[:3, :3].T) < 1e-7
        assert np.linalg.norm(T[:3, 3] - T1[:3, 3]) < 1e-7 * O.bbox_diameter(X[:m])
        np.testing.assert_allclose(objs, single.objectives, rtol=1e-6)
    # identical decisions and poses on every rank (identical reduced sums)
    assert np.array_equal(results[0][0], results[1][0])


# -- articulated: per-body statistics about centres every rank agrees on ------

def _art_problem():
    import os as _os
    g = dict(np.load(_os.path.join(_os.path.dirname(__file__), "golden", "config_c3.npz")))
    return g


def _art_run(g, lo, hi, group):
    import paper_1811_10136_b200 as fr
    from tests.articulated_util import tree_from_arrays
    gs = dict(g)
    gs["labels"] = g["labels"][lo:hi]
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.006, outlier_ratio=0.1),
                                max_em_iters=15, twist_tolerance=1e-5)
    X = g["X"].astype(float)[lo:hi]
    return fr.register(fr.PointCloud(X), fr.PointCloud(g["Y"].astype(float)),
                       tree_from_arrays(fr, gs), cfg, process_group=group)


def _art_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _art_problem()
    b = np.linspace(0, len(g["X"]), world + 1).astype(int)
    res = _art_run(g, b[rank], b[rank + 1], dist.group.WORLD)
    out[rank] = (np.asarray(res.kinematics.joint_values), res.kinematics.base_pose.matrix(),
                 res.iterations, res.termination)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_articulated_matches_single_process():
    """C3 (50k points, 20 links) split in two contiguous halves: the shards
    hold different subsets of each body's points, so each rank's own body
    centres differ -- the statistics must still be taken about the global
    ones (_articulated.py)."""
    g = _art_problem()
    single = _art_run(g, 0, len(g["X"]), None)
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_art_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                           start_method="spawn")
        results = dict(out)
    for rank in (0, 1):
        q, T, iters, term = results[rank]
        assert iters == single.iterations and term == single.termination
        assert np.abs(q - np.asarray(single.kinematics.joint_values)).max() < 1e-6
        np.testing.assert_allclose(T, single.kinematics.base_pose.matrix(), atol=1e-6)
    assert np.array_equal(results[0][0], results[1][0])
