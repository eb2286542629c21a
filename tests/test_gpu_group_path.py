"""The sharded code path (process_group=...) on one GPU: an NCCL group of
world size 1 drives the split iteration (tiled pass with its fused
reduction, NCCL all-reduce of the 25 partial sums, separate solver kernel)
-- SURVEY.md 8(e).  With one rank the all-reduce is the identity, so the
decisions must be those of the ungrouped one-kernel iteration and the poses
and objectives equal to round-off (the separate solver kernel and the fused
tail compile the same float64 solve with their own FMA contractions)."""
import os
import socket

import numpy as np
import pytest

from oracle import filterreg_oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [40_000, 300_000])
def test_group_path_equals_single(nccl_group, m):
    import paper_1811_10136_b200 as fr
    model, obs, _ = O.pebble_pair(m, outlier_ratio=0.05, seed=13)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:m]),
                                                 outlier_ratio=0.1),
                                max_em_iters=30, twist_tolerance=1e-5)
    a = fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg)
    b = fr.register(fr.PointCloud(X), fr.PointCloud(Y), fr.RigidModel(), cfg,
                    process_group=nccl_group)
    assert a.iterations == b.iterations and a.termination == b.termination
    Ra, Rb = a.kinematics.pose.rotation, b.kinematics.pose.rotation
    assert np.abs(Ra - Rb).max() < 1e-10       # entrywise: acos resolves ~2e-8 at best
    assert np.linalg.norm(a.kinematics.pose.translation - b.kinematics.pose.translation) < \
        1e-9 * O.bbox_diameter(X[:m])
    np.testing.assert_allclose(a.objectives, b.objectives, rtol=1e-10)
    np.testing.assert_allclose(a.twist_norms, b.twist_norms, rtol=1e-8, atol=1e-12)
