"""The native staged upload (fr_upload_points) equals numpy's float32
rounding of the float64 rows, transposed to planes -- bit for bit, at sizes
around the staging sub-chunk and worker split boundaries."""

import numpy as np
import pytest

from oracle import filterreg_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 7, 131071, 131072, 131073, 1_000_003])
def test_upload_matches_numpy_rounding(n):
    import torch
    from paper_1811_10136_b200._lib import device
    from paper_1811_10136_b200._rigid import upload_soa
    rng = np.random.default_rng(n)
    P = rng.standard_normal((n, 3)) * 10.0 ** rng.integers(-3, 4, (n, 1))
    soa = upload_soa(P, device())
    torch.cuda.synchronize()
    ref = np.ascontiguousarray(P.astype(np.float32).T)
    assert soa.shape == (3, n)
    assert np.array_equal(soa.cpu().numpy(), ref)


def test_upload_reuses_slots_across_calls():
    """Back-to-back uploads reuse the pinned slots: each result stays intact."""
    import torch
    from paper_1811_10136_b200._lib import device
    from paper_1811_10136_b200._rigid import upload_soa
    rng = np.random.default_rng(0)
    clouds = [rng.uniform(-1, 1, (400_000 + 1000 * i, 3)) for i in range(4)]
    outs = [upload_soa(c, device()) for c in clouds]
    torch.cuda.synchronize()
    for c, o in zip(clouds, outs):
        assert np.array_equal(o.cpu().numpy(), c.astype(np.float32).T)


@pytest.mark.parametrize("value_mode", [0, 1])
def test_pipelined_upload_splat_matches_two_step(value_mode):
    """fr_lattice_splat_upload (entries of each staged chunk overlapping the
    upload) == fr_upload_points + fr_lattice_splat_points: planes bit-exact to
    numpy astype(float32), pre- and post-blur site tables bit-exact."""
    import torch
    import paper_1811_10136_b200 as fr
    from paper_1811_10136_b200.permutohedral import PermutohedralLattice
    from paper_1811_10136_b200._rigid import upload_soa
    model, obs, _ = O.pebble_pair(700_000, outlier_ratio=0.05, seed=2)
    Y = obs.astype(np.float32).astype(float)
    sigma = np.full(3, 0.03 * O.bbox_diameter(Y))
    dev = torch.device("cuda", 0)
    planes = torch.empty((3, len(Y)), dtype=torch.float32, device=dev)
    a = PermutohedralLattice(3, sigma)
    a.splat_upload(Y, planes, value_mode)
    assert np.array_equal(planes.cpu().numpy(), Y.T.astype(np.float32))
    b = PermutohedralLattice(3, sigma)
    b.splat_points(upload_soa(Y, dev), None, value_mode)
    for stage in ("splat", "blur"):
        if stage == "blur":
            a.blur()
            b.blur()
        assert a.num_sites == b.num_sites
        assert np.array_equal(a.keys, b.keys)
        assert np.array_equal(a.values, b.values)


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("n", [1, 65535, 65536, 65537, 262145, 1_000_003])
def test_upload64_rows_transpose_exact(n, pinned):
    """fr_upload_rows64 (threaded staging copy for pageable rows, one direct
    DMA for pinned rows, then the device transpose) keeps every float64 bit."""
    import torch
    import paper_1811_10136_b200 as fr
    from paper_1811_10136_b200._lib import device
    from paper_1811_10136_b200._rigid import upload_soa64
    rng = np.random.default_rng(n)
    P = rng.standard_normal((n, 3)) * 10.0 ** rng.integers(-3, 4, (n, 1))
    src = fr.pinned_copy(P) if pinned else P
    soa = upload_soa64(src, device())
    torch.cuda.synchronize()
    assert soa.dtype == torch.float64 and soa.shape == (3, n)
    assert np.array_equal(soa.cpu().numpy(), np.ascontiguousarray(P.T))


def test_pinned_load_cloud_registers_identically(tmp_path):
    """load_cloud(..., pinned=True) rows live in page-locked memory and give
    the bit-identical registration of the pageable load."""
    import torch
    import paper_1811_10136_b200 as fr
    model, obs, _ = O.pebble_pair(20000, outlier_ratio=0.05, seed=5)
    fr.save_cloud(tmp_path / "m.ply", fr.PointCloud(model))
    fr.save_cloud(tmp_path / "o.ply", fr.PointCloud(obs))
    a = fr.load_cloud(tmp_path / "m.ply", pinned=True)
    b = fr.load_cloud(tmp_path / "o.ply", pinned=True)
    assert type(a.positions.base).__name__ == "Tensor" and a.positions.base.is_pinned()
    pa, pb = fr.load_cloud(tmp_path / "m.ply"), fr.load_cloud(tmp_path / "o.ply")
    assert np.array_equal(a.positions, pa.positions)
    cfg = fr.RegistrationConfig(gmm=fr.GmmConfig(sigma=0.05 * O.bbox_diameter(model),
                                                 outlier_ratio=0.1),
                                max_em_iters=20, twist_tolerance=1e-6)
    r1 = fr.register(a, b, fr.RigidModel(), cfg)
    r2 = fr.register(pa, pb, fr.RigidModel(), cfg)
    torch.cuda.synchronize()
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.kinematics.pose.matrix(), r2.kinematics.pose.matrix())


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("value_mode_name", ["tree", "flat_m2"])
def test_splat_rows64_matches_two_step(pinned, value_mode_name):
    """fr_lattice_splat_rows64 (float64 rows in ranges, each range's transpose
    and splat entries under the remaining copies when page-locked) ==
    fr_upload_rows64 + fr_lattice_splat_points on the float64 planes: planes
    bit-exact, pre- and post-blur site tables bit-exact."""
    import torch
    import paper_1811_10136_b200 as fr
    from paper_1811_10136_b200 import _lib
    from paper_1811_10136_b200.permutohedral import PermutohedralLattice
    from paper_1811_10136_b200._rigid import upload_soa64
    mode = 0 if value_mode_name == "tree" else _lib.FR_VALUES_M2 | _lib.FR_SPLAT_FLAT_ORDER
    model, obs, _ = O.pebble_pair(700_000, outlier_ratio=0.05, seed=3)
    Y = obs.astype(np.float32).astype(float) + 0.125 * obs.astype(float) * 1e-7
    P = fr.pinned_copy(Y) if pinned else np.ascontiguousarray(Y)
    sigma = np.full(3, 0.03 * O.bbox_diameter(Y))
    dev = torch.device("cuda", 0)
    planes = torch.empty((3, len(Y)), dtype=torch.float64, device=dev)
    rows = torch.empty((len(Y), 3), dtype=torch.float64, device=dev)
    seen = []
    a = PermutohedralLattice(3, sigma)
    follow = torch.cuda.Stream()
    a.splat_rows64(P, rows, planes, mode, uploaded=lambda: seen.append(1), follow_stream=follow)
    follow.synchronize()
    assert seen == [1]
    assert np.array_equal(planes.cpu().numpy(), Y.T)
    b = PermutohedralLattice(3, sigma)
    b.splat_points(upload_soa64(Y, dev), None, mode)
    for stage in ("splat", "blur"):
        if stage == "blur":
            a.blur()
            b.blur()
        assert a.num_sites == b.num_sites
        assert np.array_equal(a.keys, b.keys)
        assert np.array_equal(a.values, b.values)
