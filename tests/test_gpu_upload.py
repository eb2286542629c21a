"""The native staged upload (fr_upload_points) equals numpy's float32
rounding of the float64 rows, transposed to planes -- bit for bit, at sizes
around the staging sub-chunk and worker split boundaries."""

import numpy as np
import pytest

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
