"""PLY / XYZ ingestion (drop-in for io.py, pkg/src/twistreg/io.py): files
written by the live reference (tests/golden/make_golden_io.py) load to the same
arrays; binary PLY round-trips float64 exactly; malformed input raises
ParseError like the reference.  CPU only."""

import os
import warnings

import numpy as np
import pytest

from .conftest import GOLDEN

IO = os.path.join(GOLDEN, "io")


@pytest.fixture(scope="module")
def fr():
    import paper_1811_10136_b200 as fr
    return fr


def arrays():
    g = np.load(os.path.join(IO, "arrays.npz"))
    return g["P"], g["N"], g["F"]


@pytest.mark.parametrize("name", ["pos", "normals", "features", "all"])
@pytest.mark.parametrize("suffix", ["_bin.ply", "_ascii.ply", ".xyz"])
def test_reference_files_load(fr, name, suffix):
    P, N, F = arrays()
    c = fr.load_cloud(os.path.join(IO, name + suffix))
    assert np.array_equal(c.positions, P)
    if name == "all" and suffix == ".xyz":
        # XYZ is read by column count: 3 + 3 + 4 columns = positions + 7 features
        assert c.normals is None
        assert np.array_equal(c.features, np.hstack([N, F]))
        return
    if name in ("normals", "all"):
        assert np.allclose(c.normals, N, rtol=0, atol=1e-15)
        if suffix == "_bin.ply":
            assert np.array_equal(c.normals, N)
    else:
        assert c.normals is None
    if name in ("features", "all") and suffix != ".xyz":
        assert np.array_equal(c.features, F)
    if name == "features" and suffix == ".xyz":
        # XYZ is read by column count: 3 + 4 columns = positions + features
        assert np.array_equal(c.features, F)


def test_binary_round_trip_exact(fr, tmp_path):
    P, N, F = arrays()
    c = fr.PointCloud(P, normals=N, features=F)
    for fmt, path in (("ply", tmp_path / "a.ply"), ("xyz", tmp_path / "a.txt")):
        fr.save_cloud(path, c)
        d = fr.load_cloud(path)
        assert np.array_equal(d.positions, P)
        if fmt == "ply":
            assert np.array_equal(d.normals, N) and np.array_equal(d.features, F)
    with open(tmp_path / "a.ply", "rb") as fh:
        ours = fh.read()
    with open(os.path.join(IO, "all_bin.ply"), "rb") as fh:
        assert ours == fh.read()          # byte-identical to the reference's writer


def _write(tmp_path, name, text, binary_tail=b""):
    p = tmp_path / name
    p.write_bytes(text.encode("ascii") + binary_tail)
    return p


@pytest.mark.parametrize("header", [
    "ply\nformat binary_big_endian 1.0\nelement vertex 1\nproperty float x\nend_header\n",
    "ply\nformat ascii 1.0\nelement face 1\nelement vertex 1\nproperty float x\nend_header\n",
    "ply\nformat ascii 1.0\nelement vertex 1\nproperty list uchar int x\nend_header\n",
    "ply\nformat ascii 1.0\nelement vertex 1\nproperty half x\nend_header\n",
    "ply\nformat ascii 1.0\nelement vertex 1\nend_header\n",
    "ply\nelement vertex 1\nproperty float x\nend_header\n",
    "nope\n",
    "ply\nformat ascii 1.0\nelement vertex 2\nproperty float x\nproperty float y\n"
    "property float z\nend_header\n1 2 3\n",
])
def test_malformed_ply_raises(fr, tmp_path, header):
    with pytest.raises(fr.ParseError):
        fr.load_cloud(_write(tmp_path, "bad.ply", header))


def test_truncated_binary_and_nonfinite(fr, tmp_path):
    head = ("ply\nformat binary_little_endian 1.0\nelement vertex 3\nproperty double x\n"
            "property double y\nproperty double z\nend_header\n")
    with pytest.raises(fr.ParseError):
        fr.load_cloud(_write(tmp_path, "t.ply", head, np.zeros(8).tobytes()))
    vals = np.zeros((3, 3))
    vals[1, 2] = np.nan
    with pytest.raises(fr.ParseError, match="vertex 1"):
        fr.load_cloud(_write(tmp_path, "n.ply", head, vals.tobytes()))


def test_xyz_rules(fr, tmp_path):
    with pytest.raises(fr.ParseError):
        fr.load_cloud(_write(tmp_path, "a.xyz", "1 2\n"))
    with pytest.raises(fr.ParseError):
        fr.load_cloud(_write(tmp_path, "b.xyz", "1 2 3\n1 2 3 4\n"))
    with pytest.raises(fr.ParseError):
        fr.load_cloud(_write(tmp_path, "c.xyz", "# only a comment\n\n"))
    with pytest.raises(fr.ParseError):
        fr.load_cloud(_write(tmp_path, "d.xyz", "1 2 x\n"))
    with pytest.raises(fr.ParseError):
        fr.load_cloud(_write(tmp_path, "z.xyz", "0 0 0 0 0 0\n"))      # zero normal
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        c = fr.load_cloud(_write(tmp_path, "e.xyz", "# c\n1 2 3 0 0 2\n\n4 5 6 0 3 0\n"))
    assert any("re-normalized" in str(x.message) for x in w)
    assert np.array_equal(c.normals, [[0, 0, 1.0], [0, 1.0, 0]])
    with pytest.raises(ValueError):
        fr.load_cloud(tmp_path / "x.obj")
