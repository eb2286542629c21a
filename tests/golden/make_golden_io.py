"""Point-cloud files written by the LIVE reference (io.py) for the drop-in
reader's parity tests.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_io.py
"""

import os
import sys

import numpy as np

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")
sys.path.insert(0, "/root/reference/pkg/src")

import twistreg as T  # noqa: E402
from twistreg.io import save_cloud  # noqa: E402


def main():
    os.makedirs(HERE, exist_ok=True)
    rng = np.random.default_rng(0)
    P = rng.standard_normal((257, 3))
    N = rng.standard_normal((257, 3))
    N /= np.linalg.norm(N, axis=1, keepdims=True)
    F = rng.uniform(0.0, 1.0, (257, 4))
    clouds = {"pos": T.PointCloud(P), "normals": T.PointCloud(P, normals=N),
              "features": T.PointCloud(P, features=F),
              "all": T.PointCloud(P, normals=N, features=F)}
    for name, c in clouds.items():
        save_cloud(os.path.join(HERE, f"{name}_bin.ply"), c, binary=True)
        save_cloud(os.path.join(HERE, f"{name}_ascii.ply"), c, binary=False)
        save_cloud(os.path.join(HERE, f"{name}.xyz"), c)
    np.savez(os.path.join(HERE, "arrays.npz"), P=P, N=N, F=F)


if __name__ == "__main__":
    main()
