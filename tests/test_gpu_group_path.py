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


@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("m", [40_000, 300_000])
def test_group_path_equals_single(nccl_group, m, graph, monkeypatch):
    """The sharded float64 loop over NCCL (world size 1): replayed captured
    chunks of pass -> ncclAllReduce -> solve (graph) or the per-iteration
    Python loop, against the single-process grid-resident loop."""
    import paper_1811_10136_b200 as fr
    from paper_1811_10136_b200 import _rigid
    monkeypatch.setattr(_rigid, "GROUP_GRAPH", graph)
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


def test_group_graph_issues_no_python_per_iteration(nccl_group):
    """With NCCL the sharded loop's all-reduce sits inside the captured
    chunk: after construction (capture) no Python-level all-reduce call is
    made while the loop runs."""
    import paper_1811_10136_b200 as fr
    from paper_1811_10136_b200 import _rigid
    model, obs, _ = O.pebble_pair(30_000, outlier_ratio=0.05, seed=2)
    X = model.astype(np.float32).astype(float)
    Y = obs.astype(np.float32).astype(float)
    gmm = fr.GmmConfig(sigma=0.05 * O.bbox_diameter(X[:30_000]), outlier_ratio=0.1)
    cfg = fr.RegistrationConfig(gmm=gmm, max_em_iters=40, twist_tolerance=1e-30)
    path = _rigid.RigidDevicePath(fr.PointCloud(X), fr.PointCloud(Y), gmm, "point_to_point",
                                  nccl_group, precision="f64")
    em = _rigid.DeviceEM64(path, np.eye(3), np.zeros(3), cfg)
    assert em._graph is not None
    calls = []
    orig = path.reduce_device
    path.reduce_device = lambda t: (calls.append(1), orig(t))
    em.run()
    assert calls == []
    _, _, _, _, _, iters, term = em.result()
    assert iters == 40 and term == "max_iters"
