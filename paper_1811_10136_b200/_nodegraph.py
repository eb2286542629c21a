"""Node-graph (deformable) FilterReg EM on the GPU (mstep.py:232-345,
kinematics.py:254-346).

Per EM iteration: `fr_graph_pass` (DQB forward map + slice + moments + each
point's E^T E / E^T r) and `fr_graph_blocks` (block-sparse normal equations,
one warp per node / co-skinned node pair over precomputed (point, slot) lists,
fixed order).  The as-rigid-as-possible regulariser touches only node states
(~10^3 edges) and is added on the host exactly as the reference forms it; the
block-sparse system is factorised with the reference's damping / SuperLU rule
(mstep.py:317-369).  Halving candidates are scored by `fr_graph_objective`
under the stored residual spec.
"""

from __future__ import annotations

import time

import numpy as np

from . import _lib
from ._rigid import RigidDevicePath
from .errors import DegenerateBlendError, DegenerateCorrespondenceError
from .geometry import point_twist_jacobian


_IU6 = np.triu_indices(6)


def _sym6_stack(v21) -> np.ndarray:
    """(n, 21) upper-triangular rows -> (n, 6, 6) symmetric blocks."""
    v21 = np.asarray(v21, dtype=float).reshape(-1, 21)
    out = np.zeros((len(v21), 6, 6))
    out[:, _IU6[0], _IU6[1]] = v21
    out[:, _IU6[1], _IU6[0]] = v21
    return out


def gather_lists(indices, weights, n_nodes, extra_codes=None):
    """(point, slot) lists for fr_graph_blocks: node lists (code p*K + slot,
    grouped by node, point order) and co-skinned pair lists (point, slot_a |
    slot_c << 8) grouped by the canonical (lo, hi) pair, point order."""
    idx = np.asarray(indices, dtype=np.int64)
    K = idx.shape[1]
    wts = np.where(idx >= 0, np.asarray(weights, dtype=float), 0.0)
    live = (idx >= 0) & (wts > 0)
    p_i, s_i = np.nonzero(live)
    node = idx[p_i, s_i]
    npts = len(idx)
    # (node, point) order via one combined integer key (cheaper than lexsort)
    order = np.argsort(node * npts + p_i, kind="stable")
    dcount = np.bincount(node, minlength=n_nodes)
    pts, sa, sc, codes = [np.zeros(0, dtype=np.int64)], [np.zeros(0, dtype=np.int64)], \
        [np.zeros(0, dtype=np.int64)], [np.zeros(0, dtype=np.int64)]
    for a in range(K):
        for c in range(a + 1, K):
            pp = np.flatnonzero(live[:, a] & live[:, c])
            ia, ic = idx[pp, a], idx[pp, c]
            pts.append(pp)
            sa.append(np.full(len(pp), a))
            sc.append(np.full(len(pp), c))
            codes.append(np.minimum(ia, ic) * n_nodes + np.maximum(ia, ic))
    pts, sa, sc, codes = map(np.concatenate, (pts, sa, sc, codes))
    if extra_codes is None and n_nodes * n_nodes <= (1 << 24):
        # codes < n_nodes^2: unique codes and their ranks by counting
        present = np.bincount(codes, minlength=n_nodes * n_nodes) > 0
        ucodes = np.flatnonzero(present)
        pid = (np.cumsum(present) - 1)[codes]
    else:
        ucodes = np.unique(codes) if extra_codes is None else np.asarray(extra_codes)
        pid = np.searchsorted(ucodes, codes)
    porder = np.argsort(pid * npts + pts, kind="stable")
    pcount = np.bincount(pid, minlength=len(ucodes))
    pent = np.stack([pts[porder], sa[porder] | (sc[porder] << 8)], axis=1).astype(np.int32)
    return {"dptr": np.concatenate([[0], np.cumsum(dcount)]).astype(np.int32),
            "dent": np.ascontiguousarray((p_i * K + s_i)[order].astype(np.int32)),
            "pptr": np.concatenate([[0], np.cumsum(pcount)]).astype(np.int32),
            "pent": np.ascontiguousarray(pent), "n_pairs": len(ucodes),
            "pair_lo": ucodes // n_nodes, "pair_hi": ucodes % n_nodes, "codes": ucodes}


def gather_lists_device(sidx, swt, n_nodes):
    """gather_lists on the device (torch's stable GPU sorts), for one GPU:
    the same lists and order, built where they are used."""
    import torch
    npts, K = sidx.shape
    idx = sidx.long()
    live = (idx >= 0) & (swt > 0)
    p_i, s_i = torch.nonzero(live, as_tuple=True)
    node = idx[p_i, s_i]
    _, order = torch.sort(node * npts + p_i, stable=True)
    dcount = torch.bincount(node, minlength=n_nodes)
    pts, sa, sc, codes = [], [], [], []
    for a in range(K):
        for c in range(a + 1, K):
            pp = torch.nonzero(live[:, a] & live[:, c], as_tuple=True)[0]
            ia, ic = idx[pp, a], idx[pp, c]
            pts.append(pp)
            sa.append(torch.full_like(pp, a))
            sc.append(torch.full_like(pp, c))
            codes.append(torch.minimum(ia, ic) * n_nodes + torch.maximum(ia, ic))
    z = torch.zeros(0, dtype=torch.int64, device=sidx.device)
    pts, sa, sc, codes = (torch.cat(v) if v else z for v in (pts, sa, sc, codes))
    present = torch.bincount(codes, minlength=n_nodes * n_nodes) > 0
    ucodes = torch.nonzero(present, as_tuple=True)[0]
    pid = (torch.cumsum(present.long(), 0) - 1)[codes]
    _, porder = torch.sort(pid * npts + pts, stable=True)
    pcount = torch.bincount(pid, minlength=len(ucodes))
    zero = torch.zeros(1, dtype=torch.int64, device=sidx.device)
    uc = ucodes.cpu().numpy()
    return {"dptr": torch.cat([zero, torch.cumsum(dcount, 0)]).int(),
            "dent": (p_i * K + s_i)[order].int().contiguous(),
            "pptr": torch.cat([zero, torch.cumsum(pcount, 0)]).int(),
            "pent": torch.stack([pts[porder], sa[porder] | (sc[porder] << 8)], 1).int().contiguous(),
            "n_pairs": len(uc), "pair_lo": uc // n_nodes, "pair_hi": uc % n_nodes, "codes": uc}


class NodeGraphDevicePath(RigidDevicePath):
    """Model planes in input order + skinning + gather lists + lattice."""

    def __init__(self, reference, observation, gmm, residual_mode, graph, process_group=None):
        import torch
        super().__init__(reference, observation, gmm, residual_mode, process_group, sort=False)
        sk = graph.skinning
        if len(sk.indices) != self.M:
            raise ValueError("skinning does not match the reference cloud")
        K = sk.indices.shape[1]
        self.K = K
        self.n = graph.n_nodes
        idx = np.asarray(sk.indices, dtype=np.int64)
        wts = np.where(idx >= 0, np.asarray(sk.weights, dtype=float), 0.0)
        dev = self.dev
        self.sidx = torch.from_numpy(idx.astype(np.int32)).to(dev)
        self.swt = torch.from_numpy(np.ascontiguousarray(wts)).to(dev)
        if self.group is None and self.n * self.n <= (1 << 24):
            L = gather_lists_device(self.sidx, self.swt, self.n)
        else:
            L = gather_lists(idx, wts, self.n)
            if self.group is not None:
                # the pair set (and its order) must be the union over all shards
                import torch.distributed as dist
                allc = [None] * dist.get_world_size(self.group)
                dist.all_gather_object(allc, L["codes"], group=self.group)
                L = gather_lists(idx, wts, self.n, extra_codes=np.unique(np.concatenate(allc)))
            L = {k: (torch.from_numpy(v).to(dev) if k in ("dptr", "dent", "pptr", "pent") else v)
                 for k, v in L.items()}
        self.pair_lo, self.pair_hi, self.n_pairs = L["pair_lo"], L["pair_hi"], L["n_pairs"]
        self.dptr, self.dent, self.pptr, self.pent = (L[k] for k in ("dptr", "dent", "pptr", "pent"))
        f64 = dict(dtype=torch.float64, device=dev)
        self.rec = torch.empty((7, self.M), **f64)
        self.ete = torch.empty((self.M, 28), **f64)
        self.diag = torch.zeros((self.n, 27), **f64)
        self.off = torch.zeros((max(self.n_pairs, 1), 21), **f64)
        self.gsums = torch.empty(16, **f64)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.cand_dq = torch.empty((16, self.n, 8), **f64)

    def _sinv(self, s2):
        return np.sqrt(np.asarray(s2, dtype=float))

    def run(self, graph, s2, respec=False):
        """E step (or re-assembly under the stored spec) at `graph`'s nodes:
        returns (data objective, mass, sigma num, sigma mass), diag, off."""
        import torch
        dq = torch.from_numpy(np.ascontiguousarray(graph.dual_quaternions)).to(self.dev)
        si, _keep = _lib.dptr(self._sinv(s2))
        self.flag.zero_()
        _lib.check(self.lib.fr_graph_pass(
            self.lattice.handle, _lib.ptr(self.ref), self.M, _lib.ptr(self.sidx),
            _lib.ptr(self.swt), self.K, _lib.ptr(dq), self.mode, si, self.c_prime, int(respec),
            _lib.ptr(self.rec), _lib.ptr(self.ete), _lib.ptr(self.gsums), _lib.ptr(self.scratch),
            _lib.ptr(self.flag), _lib.stream_handle()))
        _lib.check(self.lib.fr_graph_blocks(
            _lib.ptr(self.ete), _lib.ptr(self.swt), self.K, _lib.ptr(self.dptr),
            _lib.ptr(self.dent), self.n, _lib.ptr(self.pptr), _lib.ptr(self.pent), self.n_pairs,
            _lib.ptr(self.diag), _lib.ptr(self.off), _lib.stream_handle()))
        self.reduce_device(self.gsums[:4])
        self.reduce_device(self.diag)
        if self.n_pairs:
            self.reduce_device(self.off)
        if self._degenerate():
            raise DegenerateBlendError("blended real part vanished for some points")
        return (self.gsums[:4].cpu().numpy().copy(), self.diag.cpu().numpy().copy(),
                self.off[:self.n_pairs].cpu().numpy().copy())

    def _degenerate(self) -> bool:
        """The degenerate-blend flag, MAX-reduced over the group so every rank
        raises together (a rank raising alone would leave the others blocked
        in the next all-reduce)."""
        if self.group is not None:
            import torch.distributed as dist
            dist.all_reduce(self.flag, op=dist.ReduceOp.MAX, group=self.group)
        return bool(int(self.flag.item()))

    def candidate_objectives(self, graphs, s2):
        import torch
        out = []
        si, _keep = _lib.dptr(self._sinv(s2))
        for a in range(0, len(graphs), 16):
            chunk = graphs[a:a + 16]
            self.cand_dq[:len(chunk)].copy_(torch.from_numpy(
                np.stack([g.dual_quaternions for g in chunk])))
            self.flag.zero_()
            _lib.check(self.lib.fr_graph_objective(
                _lib.ptr(self.ref), self.M, _lib.ptr(self.sidx), _lib.ptr(self.swt), self.K,
                _lib.ptr(self.cand_dq), self.n, len(chunk), _lib.ptr(self.rec), self.mode, si,
                _lib.ptr(self.gsums), _lib.ptr(self.scratch), _lib.ptr(self.flag),
                _lib.stream_handle()))
            self.reduce_device(self.gsums)
            if self._degenerate():
                raise DegenerateBlendError("blended real part vanished for some points")
            out += list(self.gsums[:len(chunk)].cpu().numpy())
        return np.asarray(out)


def regularizer_objective(graph, lambda_reg: float) -> float:
    """0.5 lambda sum ||T_k p - T_l p||^2 over edges, both endpoints
    (mstep.py:390-401)."""
    if lambda_reg <= 0 or not len(graph.edges):
        return 0.0
    R, t = graph.node_rotations, graph.node_translations
    k_ids, l_ids = graph.edges[:, 0], graph.edges[:, 1]
    total = 0.0
    for p in (graph.node_positions[l_ids], graph.node_positions[k_ids]):
        xk = np.einsum("eij,ej->ei", R[k_ids], p) + t[k_ids]
        xl = np.einsum("eij,ej->ei", R[l_ids], p) + t[l_ids]
        total += 0.5 * lambda_reg * float(np.sum((xk - xl) ** 2))
    return total


_INCIDENCE: dict = {}


def _grouped(values, ids, n):
    """Per-node sums of per-edge values (np.add.at semantics) as one sparse
    incidence product; the incidence matrix of an edge list is cached."""
    import scipy.sparse as sp
    key = (n, len(ids), hash(np.ascontiguousarray(ids).tobytes()))
    A = _INCIDENCE.get(key)
    if A is None:
        A = sp.csr_matrix((np.ones(len(ids)), (ids, np.arange(len(ids)))), shape=(n, len(ids)))
        if len(_INCIDENCE) > 64:
            _INCIDENCE.clear()
        _INCIDENCE[key] = A
    flat = values.reshape(len(ids), -1)
    return np.asarray(A @ flat).reshape((n,) + values.shape[1:])


def normal_equations(graph, diag, off, path, lambda_reg):
    """Block-sparse system: device data term + host ARAP term (mstep.py:290-314)."""
    return normal_equations_from(graph, diag, off, path.pair_lo, path.pair_hi, lambda_reg)


def normal_equations_from(graph, diag, off, pair_lo, pair_hi, lambda_reg):
    """6x6-block system as block arrays (keys (m, 2) with k <= l, values
    (m, 6, 6); repeated keys add up): device data term + host ARAP term."""
    from .mstep import NormalEquations
    n = graph.n_nodes
    D = _sym6_stack(diag[:, :21])
    b = diag[:, 21:27].copy()
    keys = [np.stack([np.asarray(pair_lo), np.asarray(pair_hi)], axis=1).reshape(-1, 2)]
    vals = [_sym6_stack(off[:len(pair_lo), :21]) if len(pair_lo) else np.zeros((0, 6, 6))]
    if lambda_reg > 0 and len(graph.edges):
        R, t = graph.node_rotations, graph.node_translations
        root = np.sqrt(lambda_reg)
        k_ids, l_ids = graph.edges[:, 0], graph.edges[:, 1]
        lo, hi = np.minimum(k_ids, l_ids), np.maximum(k_ids, l_ids)
        swap = k_ids > l_ids
        for p in (graph.node_positions[l_ids], graph.node_positions[k_ids]):
            xk = np.einsum("eij,ej->ei", R[k_ids], p) + t[k_ids]
            xl = np.einsum("eij,ej->ei", R[l_ids], p) + t[l_ids]
            r = root * (xk - xl)
            Jk = root * point_twist_jacobian(xk)
            Jl = -root * point_twist_jacobian(xl)
            D += _grouped(np.einsum("eri,erj->eij", Jk, Jk), k_ids, n)
            D += _grouped(np.einsum("eri,erj->eij", Jl, Jl), l_ids, n)
            b += _grouped(np.einsum("eri,er->ei", Jk, r), k_ids, n)
            b += _grouped(np.einsum("eri,er->ei", Jl, r), l_ids, n)
            cross = np.einsum("eri,erj->eij", Jk, Jl)
            cross[swap] = np.transpose(cross[swap], (0, 2, 1))
            keys.append(np.stack([lo, hi], axis=1))
            vals.append(cross)
    keys.append(np.stack([np.arange(n), np.arange(n)], axis=1))
    vals.append(D)
    return NormalEquations(6 * n, b=b.reshape(-1),
                           block_arrays=(np.concatenate(keys).astype(np.int64),
                                         np.concatenate(vals)))


def nodegraph_m_step(path, g4, diag, off, graph, s2, opts):
    """mstep.py:421-459 for a NodeGraph."""
    from .mstep import MStepDiagnostics, _accepts, gn_solve
    current = graph
    value = float(g4[0]) + regularizer_objective(current, opts.lambda_reg)
    diagn = MStepDiagnostics(objectives=[value])
    for it in range(opts.max_gn_iters):
        if it > 0:
            g4, diag, off = path.run(current, s2, respec=True)
        eq = normal_equations(current, diag, off, path, opts.lambda_reg)
        if not np.any(eq.b):
            break
        stats: dict = {}
        step = gn_solve(eq, opts.damping, opts.solve_method, _stats=stats)
        diagn.dampings.append(stats.get("damping", 0.0))
        # the full step first; the halvings (built only when it is rejected)
        # are evaluated together in one device pass
        first = current.updated(step)
        cv0 = float(path.candidate_objectives([first], s2)[0]) + \
            regularizer_objective(first, opts.lambda_reg)
        accepted = (first, cv0, 0, 1.0) if _accepts(cv0, value) else None
        if accepted is None and opts.max_halvings > 0:
            scales = [0.5 ** h for h in range(1, opts.max_halvings + 1)]
            cands = [current.updated(sc * step) for sc in scales]
            vals = path.candidate_objectives(cands, s2)
            for h, (cand, dv) in enumerate(zip(cands, vals), start=1):
                cv = float(dv) + regularizer_objective(cand, opts.lambda_reg)
                if _accepts(cv, value):
                    accepted = (cand, cv, h, scales[h - 1])
                    break
        if accepted is None:
            break
        current, value, h, sc = accepted
        diagn.objectives.append(value)
        diagn.halvings.append(h)
        sn = float(np.linalg.norm(sc * step))
        diagn.step_norms.append(sn)
        if sn <= opts.step_tolerance:
            break
    return current, diagn


# the device-resident loop (fr_ng_em) for single-GPU fixed-width runs whose
# node order keeps the block bandwidth within the factorisation's window
DEVICE_LOOP = True
MAX_DEVICE_BANDWIDTH = 24


def band_structure(n, pair_lo, pair_hi, edges):
    """Bandwidth-reducing node order (reverse Cuthill-McKee over the block
    graph of co-skinned pairs and ARAP edges), the block bandwidth, the
    per-band-slot contribution lists (pairs in pair order, then edges in
    edge order) and the per-node incident-edge lists of fr_ng_em_create."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import reverse_cuthill_mckee
    lo = np.concatenate([np.asarray(pair_lo, dtype=np.int64), edges[:, 0].astype(np.int64)])
    hi = np.concatenate([np.asarray(pair_hi, dtype=np.int64), edges[:, 1].astype(np.int64)])
    A = sp.csr_matrix((np.ones(2 * len(lo) + n),
                       (np.concatenate([lo, hi, np.arange(n)]),
                        np.concatenate([hi, lo, np.arange(n)]))), shape=(n, n))
    order = np.asarray(reverse_cuthill_mckee(A, symmetric_mode=True), dtype=np.int64)
    pos = np.empty(n, dtype=np.int64)
    pos[order] = np.arange(n)
    pa, pb = pos[lo], pos[hi]
    bw = int(np.abs(pa - pb).max(initial=0))
    W = bw + 1
    slot = np.maximum(pa, pb) * W + np.abs(pa - pb)
    kind = np.concatenate([np.zeros(len(pair_lo), dtype=np.int64),
                           np.ones(len(edges), dtype=np.int64)])
    index = np.concatenate([np.arange(len(pair_lo)), np.arange(len(edges))])
    o = np.lexsort((index, kind, slot))
    ent = ((kind[o] << 30) | index[o]).astype(np.int32)
    counts = np.bincount(slot[o], minlength=n * W)
    slot_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    ev = np.concatenate([edges[:, 0], edges[:, 1]]).astype(np.int64)
    ee = np.concatenate([np.arange(len(edges)), np.arange(len(edges))])
    role = np.concatenate([np.zeros(len(edges), dtype=np.int64),
                           np.ones(len(edges), dtype=np.int64)])
    o2 = np.lexsort((ee, ev))
    inc_ent = ((ee[o2] << 1) | role[o2]).astype(np.int32)
    inc_ptr = np.concatenate([[0], np.cumsum(np.bincount(ev, minlength=n))]).astype(np.int32)
    return pos.astype(np.int32), bw, slot_ptr, ent, inc_ptr, inc_ent


def register_nodegraph_device(path, graph, config, timing=None, band=None):
    """The device-resident node-graph EM loop (fr_ng_em_*): per iteration
    one CUDA graph of the E pass, the banded system with the ARAP term, the
    block-banded damped Cholesky, all halving candidates, the first accepted
    step, extra GN iterations, update magnitude and termination."""
    import ctypes

    from .pipeline import RegistrationResult
    from .kinematics import NodeGraph
    tick = time.perf_counter()
    n = graph.n_nodes
    edges = np.ascontiguousarray(np.asarray(graph.edges, dtype=np.int64).reshape(-1, 2))
    lo = np.asarray(path.pair_lo, dtype=np.int64)
    hi = np.asarray(path.pair_hi, dtype=np.int64)
    pos, bw, slot_ptr, slot_ent, inc_ptr, inc_ent = band if band is not None else \
        band_structure(n, lo, hi, edges)
    c = _lib.RigidEmConfig()
    c.sigma_inv[:] = list(1.0 / np.asarray(path.sigma, dtype=float))
    c.c_prime = path.c_prime
    c.diameter = path.diameter
    c.twist_tolerance = float(config.twist_tolerance)
    ms = config.mstep
    c.damping = -1.0 if ms.damping is None else float(ms.damping)
    c.step_tolerance = float(ms.step_tolerance)
    c.degenerate_mass = 1e-9 * path.M_total
    c.max_em_iters = int(config.max_em_iters)
    c.max_gn_iters = int(ms.max_gn_iters)
    c.max_halvings = int(ms.max_halvings)
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    keep = dict(P=f64(graph.node_positions), E=i32(edges), lo=i32(lo), hi=i32(hi), pos=pos,
                sp=slot_ptr, se=slot_ent, ip=inc_ptr, ie=inc_ent,
                R=f64(graph.node_rotations.reshape(n, 9)), t=f64(graph.node_translations),
                dq=f64(graph.dual_quaternions))
    ptr = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    h = ctypes.c_void_p()
    lib = path.lib
    _lib.check(lib.fr_ng_em_create(
        path.lattice.handle, _lib.ptr(path.ref), path.M, _lib.ptr(path.sidx), _lib.ptr(path.swt),
        path.K, n, ptr(keep["P"]), ptr(keep["E"]), len(edges), _lib.ptr(path.dptr),
        _lib.ptr(path.dent), _lib.ptr(path.pptr), _lib.ptr(path.pent), path.n_pairs,
        ptr(keep["lo"]), ptr(keep["hi"]), ptr(keep["pos"]), bw, ptr(keep["sp"]),
        ptr(keep["se"]), len(slot_ent), ptr(keep["ip"]), ptr(keep["ie"]), ptr(keep["R"]),
        ptr(keep["t"]), ptr(keep["dq"]), path.mode, float(ms.lambda_reg), ctypes.byref(c),
        _lib.stream_handle(), ctypes.byref(h)))
    try:
        _lib.check(lib.fr_ng_em_run(h, _lib.stream_handle()))
        k = int(config.max_em_iters)
        R, t = np.zeros((n, 9)), np.zeros((n, 3))
        obj, tn, mass = np.zeros(k), np.zeros(k), np.zeros(k)
        it, term = ctypes.c_int(), ctypes.c_int()
        dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))  # noqa: E731
        _lib.check(lib.fr_ng_em_result(h, dp(R), dp(t), dp(obj), dp(tn), dp(mass),
                                       ctypes.byref(it), ctypes.byref(term),
                                       _lib.stream_handle()))
    finally:
        lib.fr_ng_em_destroy(h)
    if int(term.value) == 4:
        raise DegenerateBlendError("blended real part vanished for some points")
    iters = int(it.value)
    kk = min(iters, k)
    model = NodeGraph._with_poses(graph, R.reshape(n, 3, 3), t)
    if timing is not None:
        timing["e_step_s"] = timing.get("e_step_s", 0.0) + time.perf_counter() - tick
        timing["m_step_s"] = timing.get("m_step_s", 0.0)
        timing["iterations"] = iters
    return RegistrationResult(kinematics=model, iterations=iters, objectives=list(obj[:kk]),
                              twist_norms=list(tn[:kk]), inlier_masses=list(mass[:kk]),
                              sigmas=[], termination=_lib.FR_TERM[int(term.value)], states=None)


def register_nodegraph(reference, observation, graph, config, timing=None, process_group=None):
    """pipeline.py:125-181 for a NodeGraph model."""
    from .pipeline import DEGENERATE_MASS_FRACTION, RegistrationResult, update_magnitude
    if config.backend != "lattice" or config.gmm.mode != "position":
        raise ValueError("the device EM path runs the lattice backend with position "
                         "correspondences")
    path = NodeGraphDevicePath(reference, observation, config.gmm, config.residual_mode, graph,
                               process_group)
    ms = config.mstep
    if (DEVICE_LOOP and process_group is None and not config.gmm.update_sigma
            and not config.record_states and ms.max_halvings <= 15 and ms.max_gn_iters <= 8
            and ms.solve_method in ("auto", "sparse")):
        edges = np.ascontiguousarray(np.asarray(graph.edges, dtype=np.int64).reshape(-1, 2))
        band = band_structure(graph.n_nodes, np.asarray(path.pair_lo, dtype=np.int64),
                              np.asarray(path.pair_hi, dtype=np.int64), edges)
        if band[1] <= MAX_DEVICE_BANDWIDTH:
            return register_nodegraph_device(path, graph, config, timing, band=band)
    model = graph
    sigma_current = path.sigma
    result = RegistrationResult(kinematics=model, iterations=0,
                                states=[] if config.record_states else None)
    for _ in range(config.max_em_iters):
        result.iterations += 1
        tick = time.perf_counter()
        s2 = (1.0 / np.asarray(sigma_current, dtype=float)) ** 2
        g4, diag, off = path.run(model, s2)
        if timing is not None:
            timing["e_step_s"] = timing.get("e_step_s", 0.0) + time.perf_counter() - tick
        mass = float(g4[1])
        result.inlier_masses.append(mass)
        if mass < DEGENERATE_MASS_FRACTION * path.M_total:
            result.objectives.append(float("nan"))
            result.twist_norms.append(float("nan"))
            result.termination = "degenerate"
            break
        if config.gmm.update_sigma:
            num, den = float(g4[2]), float(g4[3])
            if den <= 0.0:
                raise DegenerateCorrespondenceError("no correspondence mass left")
            sigma_new = max(float(np.sqrt(max(num / (3.0 * den), 0.0))), config.gmm.sigma_floor)
            if sigma_new != sigma_current[0]:
                path.build(sigma_new)
                sigma_current = path.sigma
                s_new = (1.0 / np.asarray(sigma_current, dtype=float)) ** 2
                if config.residual_mode == "point_to_point":
                    # residual scaling follows the new width (pipeline.py:155-162)
                    g4, diag, off = path.run(model, s_new, respec=True)
                s2 = s_new
            result.sigmas.append(sigma_new)
        tick = time.perf_counter()
        candidate, mdiag = nodegraph_m_step(path, g4, diag, off, model, s2, config.mstep)
        if timing is not None:
            timing["m_step_s"] = timing.get("m_step_s", 0.0) + time.perf_counter() - tick
        norm = update_magnitude(model, candidate, path.diameter)
        result.twist_norms.append(norm)
        if norm < config.twist_tolerance:
            result.objectives.append(mdiag.objectives[0])
            result.termination = "converged"
            break
        model = candidate
        result.objectives.append(mdiag.objectives[-1])
        if result.states is not None:
            result.states.append(model)
    result.kinematics = model
    if timing is not None:
        timing["iterations"] = result.iterations
    return result
