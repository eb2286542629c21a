"""Generate golden fixtures from the LIVE reference package.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every input is rounded to float32 first so the GPU path (float32 point
buffers) and the reference see identical bits.  Outputs are the reference's
own results; `tests/test_oracle_golden.py` pins the oracle to them and the GPU
parity tests compare against both.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import twistreg as T  # noqa: E402
from twistreg.estep import MomentEngine  # noqa: E402
from twistreg.permutohedral import PermutohedralLattice, build_lattice  # noqa: E402
from twistreg.synth import cuboid_shell  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def pebble_case(n, seed, outliers=0.05):
    m, o, gt = T.synthesize_pair(T.ExperimentSpec(source="pebble", n_points=n,
                                                  outlier_ratio=outliers, seed=seed))
    X, Y = f32(m.positions), f32(o.positions)
    diam = float(np.linalg.norm(X[:n].max(0) - X[:n].min(0)))
    return X, Y, diam, gt


def lattice_fixture(name, Y, V, sigma, Q):
    lat = PermutohedralLattice(Y.shape[1], sigma)
    keys, bary = lat._simplex(Y)
    lat.splat(Y, V)
    pre_k, pre_v = lat.keys.copy(), lat.values.copy()
    lat.blur()
    out = lat.slice(Q)
    qk, qb = lat._simplex(Q)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                        features=Y, values=V, sigma=np.atleast_1d(sigma), queries=Q,
                        simplex_keys=keys.astype(np.int32), simplex_bary=bary,
                        query_keys=qk.astype(np.int32), query_bary=qb,
                        pre_keys=pre_k.astype(np.int32), pre_values=pre_v,
                        post_keys=lat.keys.astype(np.int32), post_values=lat.values,
                        slice=out)
    return lat


def main():
    meta = {}
    # 1. C1-style pebble, 2000 + 5% outliers, sigma 5% of the clean diameter;
    #    value columns [1, y, |y|^2] (pt2pt + sigma update)
    X, Y, diam, _ = pebble_case(2000, seed=0)
    sig = 0.05 * diam
    V = np.hstack([np.ones((len(Y), 1)), Y, np.einsum("nd,nd->n", Y, Y)[:, None]])
    lattice_fixture("lattice_pebble_s5", Y, V, sig, X)
    meta["lattice_pebble_s5"] = {"sigma": sig, "n_obs": len(Y), "n_query": len(X)}

    # 2. fine sigma (0.5%): many more sites, exercises hash growth
    sig_f = 0.005 * diam
    lattice_fixture("lattice_pebble_s05", Y, V[:, :4], sig_f, X)
    meta["lattice_pebble_s05"] = {"sigma": sig_f}

    # 3. anisotropic widths + signed random values (generic operator)
    rng = np.random.default_rng(7)
    F = f32(rng.uniform(0, 1, (300, 3)))
    Q = f32(rng.uniform(0, 1, (120, 3)))
    Vr = f32(rng.normal(size=(300, 2)))
    lattice_fixture("lattice_aniso", F, Vr, np.array([0.05, 0.1, 0.2]), Q)

    # 4. grid-aligned cuboid with normals: exact-zero barycentrics, V = 7
    P, N = cuboid_shell(3500)
    P, N = f32(P), f32(N)
    Vn = np.hstack([np.ones((len(P), 1)), P, N])
    sig_c = 0.05 * float(np.linalg.norm(P.max(0) - P.min(0)))
    lattice_fixture("lattice_cuboid_normals", P, Vn, sig_c, f32(P * 0.98 + 0.001))

    # 5. moment fields (MomentEngine.moments), pt2pt+m2 and pt2pl
    eng = MomentEngine(T.PointCloud(Y), T.GmmConfig(sigma=sig, outlier_ratio=0.1,
                                                     update_sigma=True))
    mf = eng.moments(X)
    np.savez_compressed(os.path.join(HERE, "moments_pebble.npz"), X=X, Y=Y,
                        sigma=sig, m0=mf.m0, m1=mf.m1, weight=mf.weight,
                        target=mf.target, m2=mf.m2, c_prime=mf.c_prime,
                        sigma_new=T.update_sigma(X, mf))
    Xc = f32(P @ T.rotation_about_axis([0, 1, 0.4], np.radians(8.0)).T
             + np.array([0.002, 0.001, -0.003]))
    eng_n = MomentEngine(T.PointCloud(P, normals=N),
                         T.GmmConfig(sigma=sig_c, outlier_ratio=0.1), include_normals=True)
    mn = eng_n.moments(Xc)
    np.savez_compressed(os.path.join(HERE, "moments_cuboid.npz"), X=Xc, Y=P, N=N,
                        sigma=sig_c, m0=mn.m0, m1=mn.m1, weight=mn.weight,
                        target=mn.target, normal=mn.normal,
                        normal_valid=mn.normal_valid, c_prime=mn.c_prime)

    # 6. registration traces
    traces = {}
    for seed in (0, 1, 2):
        X, Y, diam, gt = pebble_case(3500, seed=seed)
        cfg = T.RegistrationConfig(gmm=T.GmmConfig(sigma=0.05 * diam, outlier_ratio=0.1),
                                   max_em_iters=250, twist_tolerance=2e-4)
        r = T.register(T.PointCloud(X), T.PointCloud(Y), T.RigidModel(), cfg)
        traces[f"pt2pt_seed{seed}"] = dict(X=X, Y=Y, sigma=0.05 * diam, w=0.1,
                                           max_iters=250, tol=2e-4, r=r)
    # point-to-plane on the cuboid shell (test_pipeline.py:190-205 setup)
    Rg = T.rotation_about_axis([0, 1, 0.4], np.radians(8.0))
    tg = np.array([0.002, 0.001, -0.003])
    Yc = f32(P @ Rg.T + tg)
    Nc = f32(N @ Rg.T)
    sig_pl = T.default_sigma(T.PointCloud(Yc))
    cfg = T.RegistrationConfig(gmm=T.GmmConfig(sigma=sig_pl, outlier_ratio=0.1),
                               residual_mode="point_to_plane")
    r = T.register(T.PointCloud(P, normals=N), T.PointCloud(Yc, normals=Nc),
                   T.RigidModel(), cfg)
    traces["pt2pl_cuboid"] = dict(X=P, Y=Yc, N=Nc, sigma=sig_pl, w=0.1, max_iters=50,
                                  tol=1e-4, r=r)
    # sigma annealing from an inflated start
    X, Y, diam, _ = pebble_case(2000, seed=4, outliers=0.0)
    cfg = T.RegistrationConfig(gmm=T.GmmConfig(sigma=0.15 * diam, outlier_ratio=0.1,
                                               update_sigma=True), max_em_iters=40)
    r = T.register(T.PointCloud(X), T.PointCloud(Y), T.RigidModel(), cfg)
    traces["pt2pt_update_sigma"] = dict(X=X, Y=Y, sigma=0.15 * diam, w=0.1, max_iters=40,
                                        tol=1e-4, r=r, update_sigma=True)
    for name, tr in traces.items():
        r = tr.pop("r")
        arrays = {k: v for k, v in tr.items() if isinstance(v, np.ndarray)}
        scalars = {k: v for k, v in tr.items() if not isinstance(v, np.ndarray)}
        np.savez_compressed(
            os.path.join(HERE, f"register_{name}.npz"),
            R=r.kinematics.pose.rotation, t=r.kinematics.pose.translation,
            objectives=np.asarray(r.objectives), twist_norms=np.asarray(r.twist_norms),
            inlier_masses=np.asarray(r.inlier_masses), sigmas=np.asarray(r.sigmas),
            iterations=r.iterations, termination=r.termination,
            config=json.dumps(scalars), **arrays)
        meta[f"register_{name}"] = {"iterations": r.iterations,
                                    "termination": r.termination}
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "twistreg 0.1.0 (/root/reference/pkg)",
                   "numpy": np.__version__, "cases": meta}, fh, indent=1)


if __name__ == "__main__":
    main()
