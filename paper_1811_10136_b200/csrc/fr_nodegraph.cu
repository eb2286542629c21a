// Node-graph (deformable) FilterReg on B200 (mstep.py:232-314, kinematics.py:254-346,
// geometry.py:342-368).
//
//   k_graph_pass       per model point: dual-quaternion blend of its K skinned
//                      node states (hemisphere-aligned to the first live node),
//                      forward map, lattice slice + moments epilogue, residual
//                      rows, and the point's E^T E (21) / E^T r (6) with
//                      E = P J(x) (mstep.py:266-270); data objective, mass and
//                      sigma sums block-reduced in a fixed order.
//   k_graph_blocks     one warp per block of the block-sparse normal equations:
//                      node diagonal blocks sum w_a^2 E^T E and w_a E^T r over
//                      the node's (point, slot) list, co-skinned pairs sum
//                      w_a w_c E^T E over the pair's list (mstep.py:274-288) --
//                      fixed list order, no atomics, deterministic.
//   k_graph_objective  data objective of up to 16 candidate node states under
//                      the stored residual spec (halving, mstep.py:443-449).
// The ARAP regulariser (node-only, ~10^3 edges) and the sparse factorisation
// stay on the host, exactly as the reference forms them.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "fr_reduce.cuh"
#include "fr_solve.cuh"

namespace fr {

constexpr int kMaxK = 8;
constexpr int kGraphEte = 28;   // E^T E upper 21 | E^T r 6 | pad

struct GraphK {
    double A[4][3];   // embedding E diag(sf / sigma): elevated = A x
    double sinv[3];   // residual scaling (point_to_point)
    double cp;
    double gain;
    int mode;
    int K;
    int m2_col;
    int ncol;
};

// DQB of a point's skinned nodes -> (R, t); false when the blend degenerates
__device__ __forceinline__ bool dq_blend(const int *idx, const double *w, int K,
                                         const double *__restrict__ dq, double *R, double *t,
                                         bool *bound) {
    double b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int first = -1;
    double wsum = 0.0;
    for (int k = 0; k < K; ++k) {
        wsum += w[k];
        if (first < 0 && idx[k] >= 0) first = idx[k];
    }
    *bound = wsum > 0.0;
    if (!*bound || first < 0) {
        for (int q = 0; q < 9; ++q) R[q] = (q % 4 == 0) ? 1.0 : 0.0;
        t[0] = t[1] = t[2] = 0.0;
        return true;
    }
    const double *r0 = dq + 8 * first;
    for (int k = 0; k < K; ++k) {
        if (idx[k] < 0) continue;
        const double *q = dq + 8 * idx[k];
        const double dot = ((q[0] * r0[0] + q[1] * r0[1]) + q[2] * r0[2]) + q[3] * r0[3];
        const double s = (dot < 0.0 ? -1.0 : 1.0) * w[k];
        for (int c = 0; c < 8; ++c) b[c] += s * q[c];
    }
    const double nr = sqrt(((b[0] * b[0] + b[1] * b[1]) + b[2] * b[2]) + b[3] * b[3]);
    if (nr < 1e-12) return false;
    const double qw = b[0] / nr, qx = b[1] / nr, qy = b[2] / nr, qz = b[3] / nr;
    const double dw = b[4] / nr, dx = b[5] / nr, dy = b[6] / nr, dz = b[7] / nr;
    R[0] = 1 - 2 * (qy * qy + qz * qz);
    R[1] = 2 * (qx * qy - qw * qz);
    R[2] = 2 * (qx * qz + qw * qy);
    R[3] = 2 * (qx * qy + qw * qz);
    R[4] = 1 - 2 * (qx * qx + qz * qz);
    R[5] = 2 * (qy * qz - qw * qx);
    R[6] = 2 * (qx * qz - qw * qy);
    R[7] = 2 * (qy * qz + qw * qx);
    R[8] = 1 - 2 * (qx * qx + qy * qy);
    // t = 2 (dual * conj(real)).xyz
    t[0] = 2 * (-dw * qx + dx * qw - dy * qz + dz * qy);
    t[1] = 2 * (-dw * qy + dx * qz + dy * qw - dz * qx);
    t[2] = 2 * (-dw * qz - dx * qy + dy * qx + dz * qw);
    return true;
}

__device__ __forceinline__ void point_forward(const float *__restrict__ ref, long long m,
                                              long long p, const int *__restrict__ sidx,
                                              const double *__restrict__ swt, int K,
                                              const double *__restrict__ dq, double *x,
                                              int *bad) {
    int idx[kMaxK];
    double w[kMaxK];
    for (int k = 0; k < K; ++k) {
        idx[k] = sidx[p * K + k];
        w[k] = idx[k] >= 0 ? swt[p * K + k] : 0.0;
    }
    double R[9], t[3];
    bool bound;
    if (!dq_blend(idx, w, K, dq, R, t, &bound)) atomicOr(bad, 1);
    const double xr[3] = {(double)__ldg(ref + p), (double)__ldg(ref + m + p),
                          (double)__ldg(ref + 2 * m + p)};
    for (int i = 0; i < 3; ++i)
        x[i] = ((R[3 * i] * xr[0] + R[3 * i + 1] * xr[1]) + R[3 * i + 2] * xr[2]) + t[i];
}

// residual rows of one point -> E^T E (upper 21), E^T r (6), 0.5 |r|^2
__device__ __forceinline__ double point_rows(int mode, const double *sinv, double w,
                                             const double *x, const double *tg,
                                             const double *n, double *ete) {
    for (int q = 0; q < kGraphEte; ++q) ete[q] = 0.0;
    if (!(w > 0.0)) return 0.0;
    const double sw = sqrt(w);
    const double d[3] = {x[0] - tg[0], x[1] - tg[1], x[2] - tg[2]};
    const double J[3][6] = {{0.0, x[2], -x[1], 1.0, 0.0, 0.0},
                            {-x[2], 0.0, x[0], 0.0, 1.0, 0.0},
                            {x[1], -x[0], 0.0, 0.0, 0.0, 1.0}};
    double P[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    int rows = 3;
    if (mode == FR_POINT_TO_POINT) {
        for (int j = 0; j < 3; ++j) P[j][j] = sw * sinv[j];
    } else if (n[0] != 0.0 || n[1] != 0.0 || n[2] != 0.0) {
        rows = 1;
        for (int j = 0; j < 3; ++j) P[0][j] = sw * n[j];
    } else {
        for (int j = 0; j < 3; ++j) P[j][j] = sw;
    }
    double e = 0.0;
    for (int r = 0; r < rows; ++r) {
        double G[6];
        for (int c = 0; c < 6; ++c) G[c] = (P[r][0] * J[0][c] + P[r][1] * J[1][c]) + P[r][2] * J[2][c];
        const double rr = (P[r][0] * d[0] + P[r][1] * d[1]) + P[r][2] * d[2];
        int o = 0;
        for (int i = 0; i < 6; ++i) {
            for (int j = i; j < 6; ++j) { ete[o] = fma(G[i], G[j], ete[o]); ++o; }
            ete[21 + i] = fma(G[i], rr, ete[21 + i]);
        }
        e = fma(rr, rr, e);
    }
    return 0.5 * e;
}

constexpr int kGraphAcc = 4;   // objective, mass, sigma numerator, sigma mass

// RESPEC = false: E step at the current nodes (moments -> w, t, n stored);
// RESPEC = true: reuse the stored spec, recompute x and E^T E at new nodes
template <int NV, bool RESPEC>
__global__ void __launch_bounds__(kPassThreads, 2)
k_graph_pass(const float *__restrict__ ref, long long m, const int *__restrict__ sidx,
             const double *__restrict__ swt, const double *__restrict__ dq, GraphK g,
             SliceTable tab, double *__restrict__ rec, double *__restrict__ ete,
             double *__restrict__ partials, int *bad, const int *skip = nullptr) {
    if (skip && *skip) return;      // device-resident loop: stage not active
    double acc[kGraphAcc] = {0.0, 0.0, 0.0, 0.0};
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        double x[3];
        point_forward(ref, m, p, sidx, swt, g.K, dq, x, bad);
        double w, tg[3], n[3] = {0.0, 0.0, 0.0};
        if (!RESPEC) {
            double el[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                el[i] = fma(g.A[i][2], x[2], fma(g.A[i][1], x[1], g.A[i][0] * x[0]));
            Simplex<3> s;
            simplex_from_elevated<3>(el, s);
            double out[NV];
#pragma unroll
            for (int q = 0; q < NV; ++q) out[q] = 0.0;
            if (!s.overflow) {
                unsigned long long key[4];
#pragma unroll
                for (int l = 0; l < 4; ++l) key[l] = s.packed(l);
                double v[4][NV];
                bool hit[4];
                gather_simplex<3, NV>(tab, key, v, hit);
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    const double b = hit[l] ? s.bary[l] : 0.0;
#pragma unroll
                    for (int q = 0; q < NV; ++q) out[q] = fma(b, v[l][q], out[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) out[q] *= g.gain;
            const double m0 = fmax(out[0], 0.0);
            const bool sup = m0 >= 1e-12;
            w = sup ? (g.cp > 0.0 ? m0 / (m0 + g.cp) : 1.0) : 0.0;
            for (int j = 0; j < 3; ++j) tg[j] = sup ? out[1 + j] / m0 : x[j];
            if (g.ncol >= 0 && sup) {
                double a[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    double vv = 0.0;
#pragma unroll
                    for (int q = 0; q < NV; ++q) vv = (q == g.ncol + j) ? out[q] : vv;
                    a[j] = vv / m0;
                }
                const double len = sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]);
                if (len >= 0.1)
                    for (int j = 0; j < 3; ++j) n[j] = a[j] / len;
            }
            if (g.m2_col >= 0 && sup) {
                double m2v = 0.0;
#pragma unroll
                for (int q = 0; q < NV; ++q) m2v = (q == g.m2_col) ? out[q] : m2v;
                const double den = m0 + g.cp;
                const double xx = (x[0] * x[0] + x[1] * x[1]) + x[2] * x[2];
                const double xm = (x[0] * out[1] + x[1] * out[2]) + x[2] * out[3];
                acc[2] += (m0 * xx - 2.0 * xm + m2v) / den;
                acc[3] += m0 / den;
            }
            rec[p] = w;
            for (int j = 0; j < 3; ++j) {
                rec[(1 + j) * m + p] = tg[j];
                rec[(4 + j) * m + p] = n[j];
            }
        } else {
            w = rec[p];
            for (int j = 0; j < 3; ++j) {
                tg[j] = rec[(1 + j) * m + p];
                n[j] = rec[(4 + j) * m + p];
            }
        }
        double e[kGraphEte];
        acc[0] += point_rows(g.mode, g.sinv, w, x, tg, n, e);
        acc[1] += w;
        for (int q = 0; q < kGraphEte; ++q) ete[p * kGraphEte + q] = e[q];
    }
    block_reduce_store<kGraphAcc>(acc, partials + (long long)blockIdx.x * kGraphAcc);
}

// one warp per block: rows [0, n_nodes) are node diagonals (27 values),
// rows [n_nodes, n_nodes + n_pairs) co-skinned pairs (21 values)
__global__ void k_graph_blocks(const double *__restrict__ ete, const double *__restrict__ swt,
                               int K, const int *__restrict__ dptr, const int *__restrict__ dent,
                               int n_nodes, const int *__restrict__ pptr,
                               const int *__restrict__ pent, int n_pairs,
                               double *__restrict__ diag, double *__restrict__ off,
                               const int *skip = nullptr) {
    if (skip && *skip) return;
    const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (wg >= n_nodes + n_pairs) return;
    const bool is_diag = wg < n_nodes;
    const int nv = is_diag ? 27 : 21;
    double acc[27];
    for (int q = 0; q < 27; ++q) acc[q] = 0.0;
    const int beg = is_diag ? dptr[wg] : pptr[wg - n_nodes];
    const int end = is_diag ? dptr[wg + 1] : pptr[wg - n_nodes + 1];
    for (int e = beg + lane; e < end; e += 32) {
        double f1, f2;
        long long p;
        if (is_diag) {
            const int code = dent[e];                // p * K + slot
            p = code / K;
            const double wa = swt[code];
            f1 = wa * wa;
            f2 = wa;
        } else {
            const long long code = (unsigned)pent[2 * e];   // point
            p = code;
            const int sa = pent[2 * e + 1] & 0xff, sc = (pent[2 * e + 1] >> 8) & 0xff;
            f1 = swt[p * K + sa] * swt[p * K + sc];
            f2 = 0.0;
        }
        const double *src = ete + p * kGraphEte;
        for (int q = 0; q < 21; ++q) acc[q] = fma(f1, src[q], acc[q]);
        if (is_diag)
            for (int q = 0; q < 6; ++q) acc[21 + q] = fma(f2, src[21 + q], acc[21 + q]);
    }
    for (int q = 0; q < nv; ++q) {
        double v = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        acc[q] = v;
    }
    if (lane == 0) {
        if (is_diag)
            for (int q = 0; q < 27; ++q) diag[(long long)wg * 27 + q] = acc[q];
        else
            for (int q = 0; q < 21; ++q) off[(long long)(wg - n_nodes) * 21 + q] = acc[q];
    }
}

// the device loop's block gather in fixed pieces of kGraphPiece entries (one
// warp per piece: the 195 node blocks of C4 hold ~2,000 entries each, one
// warp per block left the gather latency bound), each piece's 27 / 21 sums
// by a warp tree; k_graph_pieces_combine adds a block's pieces in order
constexpr int kGraphPiece = 256;

__global__ void k_graph_block_pieces(const double *__restrict__ ete, const double *__restrict__ swt,
                                     int K, const int *__restrict__ dent,
                                     const int *__restrict__ pent, int n_nodes,
                                     const int *__restrict__ piece_blk,
                                     const int *__restrict__ piece_beg,
                                     const int *__restrict__ piece_end, int n_pieces,
                                     double *__restrict__ piece_vals, const int *skip) {
    if (skip && *skip) return;
    const int pc = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (pc >= n_pieces) return;
    const int blk = piece_blk[pc];
    const bool is_diag = blk < n_nodes;
    const int beg = piece_beg[pc], end = piece_end[pc];
    double acc[27];
#pragma unroll
    for (int q = 0; q < 27; ++q) acc[q] = 0.0;
    for (int e = beg + lane; e < end; e += 32) {
        double f1, f2;
        long long p;
        if (is_diag) {
            const int code = dent[e];                // p * K + slot
            p = code / K;
            const double wa = swt[code];
            f1 = wa * wa;
            f2 = wa;
        } else {
            p = (unsigned)pent[2 * e];
            const int sa = pent[2 * e + 1] & 0xff, sc = (pent[2 * e + 1] >> 8) & 0xff;
            f1 = swt[p * K + sa] * swt[p * K + sc];
            f2 = 0.0;
        }
        const double *src = ete + p * kGraphEte;
#pragma unroll
        for (int q = 0; q < 21; ++q) acc[q] = fma(f1, src[q], acc[q]);
        if (is_diag)
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[21 + q] = fma(f2, src[21 + q], acc[21 + q]);
    }
#pragma unroll
    for (int q = 0; q < 27; ++q) {
        double v = acc[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        acc[q] = v;
    }
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 27; ++q) piece_vals[(long long)pc * 27 + q] = acc[q];
}

__global__ void k_graph_pieces_combine(const int *__restrict__ blk_piece0, int n_nodes,
                                       int n_pairs, const double *__restrict__ piece_vals,
                                       double *__restrict__ diag, double *__restrict__ off,
                                       const int *skip) {
    if (skip && *skip) return;
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)(n_nodes + n_pairs) * 27) return;
    const int blk = (int)(t / 27), q = (int)(t % 27);
    const bool is_diag = blk < n_nodes;
    if (!is_diag && q >= 21) return;
    double v = 0.0;
    for (int pc = blk_piece0[blk]; pc < blk_piece0[blk + 1]; ++pc) v += piece_vals[(long long)pc * 27 + q];
    if (is_diag) diag[(long long)blk * 27 + q] = v;
    else off[(long long)(blk - n_nodes) * 21 + q] = v;
}

constexpr int kGraphMaxCand = 16;

__global__ void __launch_bounds__(kPassThreads, 2)
k_graph_objective(const float *__restrict__ ref, long long m, const int *__restrict__ sidx,
                  const double *__restrict__ swt, int K, const double *__restrict__ cand_dq,
                  int n_nodes, int ncand, const double *__restrict__ rec, int mode, double s0,
                  double s1, double s2, double *__restrict__ partials, int *bad,
                  const int *skip = nullptr, int c0 = 0, const int *skip2 = nullptr) {
    if ((skip && *skip) || (skip2 && *skip2)) return;
    double acc[kGraphMaxCand];
#pragma unroll
    for (int a = 0; a < kGraphMaxCand; ++a) acc[a] = 0.0;
    const double sinv[3] = {s0, s1, s2};
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        const double w = rec[p];
        if (!(w > 0.0)) continue;
        const double tg[3] = {rec[m + p], rec[2 * m + p], rec[3 * m + p]};
        const double n[3] = {rec[4 * m + p], rec[5 * m + p], rec[6 * m + p]};
#pragma unroll
        for (int c = 0; c < kGraphMaxCand; ++c) {
            if (c >= c0 + ncand) break;
            if (c < c0) continue;                  // candidates [c0, c0 + ncand)
            double x[3];
            point_forward(ref, m, p, sidx, swt, K, cand_dq + (size_t)c * n_nodes * 8, x, bad);
            const double d[3] = {x[0] - tg[0], x[1] - tg[1], x[2] - tg[2]};
            double e;
            if (mode == FR_POINT_TO_POINT) {
                e = 0.0;
                for (int j = 0; j < 3; ++j) {
                    const double r = sqrt(w) * sinv[j] * d[j];
                    e = fma(r, r, e);
                }
            } else if (n[0] != 0.0 || n[1] != 0.0 || n[2] != 0.0) {
                const double r = sqrt(w) * ((n[0] * d[0] + n[1] * d[1]) + n[2] * d[2]);
                e = r * r;
            } else {
                e = 0.0;
                for (int j = 0; j < 3; ++j) {
                    const double r = sqrt(w) * d[j];
                    e = fma(r, r, e);
                }
            }
            acc[c] += 0.5 * e;
        }
    }
    block_reduce_store<kGraphMaxCand>(acc, partials + (long long)blockIdx.x * kGraphMaxCand);
}

// per-point E^T E / E^T r of an explicit ResidualSpec at explicit positions
// (assemble_articulated / assemble_nodegraph API, mstep.py:213-314)
__global__ void k_point_rows(const double *__restrict__ X, const double *__restrict__ W,
                             const double *__restrict__ T, const double *__restrict__ N,
                             const unsigned char *__restrict__ valid, long long m, int mode,
                             double s0, double s1, double s2, double *__restrict__ ete) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= m) return;
    const double sinv[3] = {s0, s1, s2};
    const double x[3] = {X[3 * p], X[3 * p + 1], X[3 * p + 2]};
    const double t[3] = {T[3 * p], T[3 * p + 1], T[3 * p + 2]};
    double n[3] = {0.0, 0.0, 0.0};
    if (mode == FR_POINT_TO_PLANE && valid[p])
        for (int j = 0; j < 3; ++j) n[j] = N[3 * p + j];
    double e[kGraphEte];
    point_rows(mode, sinv, W[p], x, t, n, e);
    for (int q = 0; q < kGraphEte; ++q) ete[p * kGraphEte + q] = e[q];
}


// ===========================================================================
// Device-resident node-graph EM (pipeline.py:125-181 with a NodeGraph;
// mstep.py:232-369, 421-459): per EM iteration a fixed kernel sequence,
// replayed from a CUDA graph with no host round trip --
//   k_graph_pass / k_graph_blocks    E step + per-node / per-pair data blocks
//   k_ng_assemble                    data blocks + the ARAP term (mstep.py:
//                                    290-314, node-only, fixed order per
//                                    block) into a block-banded matrix over a
//                                    bandwidth-reducing node order (RCM),
//                                    objective, degenerate check
//   k_ng_factor (one CTA)            (A + lam I) x = b by a block-banded
//                                    Cholesky with the reference's damping
//                                    and tenfold escalation (replaces SuperLU,
//                                    mstep.py:317-345: same solution to
//                                    round-off)
//   k_ng_cands                       the full step and every halving as
//                                    candidate node states (per-node
//                                    exp(twist) o T with polar factor) and
//                                    their dual quaternions
//   k_graph_objective                data objectives of all candidates (one
//                                    pass over the stored spec)
//   k_ng_select                      + ARAP objectives, first accepted step,
//                                    state update; extra GN iterations repeat
//                                    the stages under the stored spec
//   k_ng_finish                      update magnitude, termination, traces.
// Stages whose skip flag is set return at once (finished loop / finished
// Gauss-Newton iterations).

constexpr int kNgThreads = 1024;
constexpr int kNgMaxCand = 16;
enum { kNgTermBlend = 4 };

struct NgDev {
    double sinv[3], cp, diameter, tol, damping, step_tol, degenerate_mass, lambda;
    int n, n_edges, bw, max_em_iters, max_gn_iters, max_halvings, use_damping, mode;
    int done, iterations, termination, gn_skip;
    int gn, ncand, mstep_ran, accepted;
    double value, value0, arap0, sn;
};

struct NgBufs {
    NgDev *st;
    double *R, *T, *DQ;            // node state (n x 9, 3, 8)
    double *R0, *T0, *DQ0;         // at the start of the M step
    const double *P;               // node positions n x 3
    const int *edges;              // E x 2
    const int *pos;                // node -> band position
    const int *node_at;            // band position -> node
    const int *slot_ptr, *slot_ent;   // per band slot: (kind << 30) | index (kind 0 pair, 1 edge)
    const int *inc_ptr, *inc_ent;     // per node: incident edges (edge << 1 | role: 0 = k, 1 = l)
    const int *pair_lo, *pair_hi;
    const double *gsums;           // E pass sums (objective, mass, ...)
    const double *diag, *off;      // data blocks (n x 27, pairs x 21)
    double *band, *bvec;           // assembled system: band [n][bw+1][36], b [n][6] (positions)
    double *L, *x, *step;          // factor, solution (positions), step (node order, 6n)
    double *candR, *candT, *candDQ;   // [16][n][9 / 3 / 8]
    const double *cand_data;       // 16 data objectives
    double *traces;                // [3][max_iters]
    int *flag;                     // degenerate blend flag of the passes
};

__device__ __forceinline__ void ng_jac(const double *x, double J[3][6]) {
    // point_twist_jacobian: [-[x]x | I]
    J[0][0] = 0.0;   J[0][1] = x[2];  J[0][2] = -x[1]; J[0][3] = 1.0; J[0][4] = 0.0; J[0][5] = 0.0;
    J[1][0] = -x[2]; J[1][1] = 0.0;   J[1][2] = x[0];  J[1][3] = 0.0; J[1][4] = 1.0; J[1][5] = 0.0;
    J[2][0] = x[1];  J[2][1] = -x[0]; J[2][2] = 0.0;   J[2][3] = 0.0; J[2][4] = 0.0; J[2][5] = 1.0;
}

__device__ __forceinline__ void ng_apply(const double *R, const double *t, const double *p,
                                         double *x) {
    for (int i = 0; i < 3; ++i) x[i] = R[3 * i] * p[0] + R[3 * i + 1] * p[1] + R[3 * i + 2] * p[2] + t[i];
}

// the ARAP rows of edge e at endpoint position p: xk, xl, r = sqrt(lam) (xk - xl)
__device__ __forceinline__ void ng_arap_rows(const NgBufs &b, int e, int which, const double *R,
                                             const double *T, double *xk, double *xl,
                                             double *r) {
    const int k = b.edges[2 * e], l = b.edges[2 * e + 1];
    const double *p = b.P + 3 * (which == 0 ? l : k);   // (node_positions[l], then [k])
    ng_apply(R + 9 * k, T + 3 * k, p, xk);
    ng_apply(R + 9 * l, T + 3 * l, p, xl);
    const double root = sqrt(b.st->lambda);
    for (int i = 0; i < 3; ++i) r[i] = root * (xk[i] - xl[i]);
}

// rigid pose -> unit dual quaternion [real | dual] (Shepperd, w >= 0; geometry.py:243-283)
__device__ void ng_dq(const double *R, const double *t, double *dq) {
    const double tr = (R[0] + R[4]) + R[8];
    double q[4];
    if (tr > 0) {
        const double s = 2.0 * sqrt(tr + 1.0);
        q[0] = 0.25 * s;
        q[1] = (R[7] - R[5]) / s;
        q[2] = (R[2] - R[6]) / s;
        q[3] = (R[3] - R[1]) / s;
    } else {
        int i = 0;
        if (R[4] > R[0]) i = 1;
        if (R[8] > R[3 * i + i]) i = 2;
        const int j = (i + 1) % 3, k = (i + 2) % 3;
        const double s = 2.0 * sqrt(R[3 * i + i] - R[3 * j + j] - R[3 * k + k] + 1.0);
        q[0] = (R[3 * k + j] - R[3 * j + k]) / s;
        q[1 + i] = 0.25 * s;
        q[1 + j] = (R[3 * j + i] + R[3 * i + j]) / s;
        q[1 + k] = (R[3 * k + i] + R[3 * i + k]) / s;
    }
    if (q[0] < 0) for (int c = 0; c < 4; ++c) q[c] = -q[c];
    const double nq = sqrt(((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3]);
    for (int c = 0; c < 4; ++c) q[c] /= nq;
    // dual = 0.5 (0, t) q
    const double a1 = 0.0, b1 = t[0], c1 = t[1], d1 = t[2];
    const double a2 = q[0], b2 = q[1], c2 = q[2], d2 = q[3];
    const double qd[4] = {a1 * a2 - b1 * b2 - c1 * c2 - d1 * d2, a1 * b2 + b1 * a2 + c1 * d2 - d1 * c2,
                          a1 * c2 - b1 * d2 + c1 * a2 + d1 * b2, a1 * d2 + b1 * c2 - c1 * b2 + d1 * a2};
    for (int c = 0; c < 4; ++c) {
        dq[c] = q[c];
        dq[4 + c] = 0.5 * qd[c];
    }
}

// the assembled system at the current node state: data blocks + ARAP
// (mstep.py:290-314), banded over the node order `pos`; first = 1 also runs
// the E-step bookkeeping (mass, degenerate test, objective, M-step start)
constexpr int kNgAsmThreads = 128;

// E-step bookkeeping (first = 1: mass, degenerate test, the M step's start
// state) and the objective value0 = data + ARAP at the current node state
__global__ void __launch_bounds__(kNgThreads, 1) k_ng_begin(NgBufs b, int first) {
    NgDev *st = b.st;
    if (first ? st->done : st->gn_skip) return;
    __shared__ double red[kNgThreads / 32];
    __shared__ int bad;
    const bool reg = st->lambda > 0.0 && st->n_edges > 0;
    if (first) {
        if (threadIdx.x == 0) {
            bad = 0;
            const int it = st->iterations;
            const double mass = b.gsums[1];
            b.traces[2 * st->max_em_iters + it] = mass;
            st->mstep_ran = 0;
            if (*b.flag) {
                st->termination = kNgTermBlend;
                st->done = 1;
                bad = 1;
            } else if (mass < st->degenerate_mass) {       // pipeline.py:148-154
                b.traces[it] = CUDART_NAN;
                b.traces[st->max_em_iters + it] = CUDART_NAN;
                st->iterations = it + 1;
                st->termination = kTermDegenerate;
                st->done = 1;
                bad = 1;
            }
        }
        __syncthreads();
        if (bad) {
            if (threadIdx.x == 0) st->gn_skip = 1;
            return;
        }
        for (int q = threadIdx.x; q < st->n; q += blockDim.x) {
            for (int c = 0; c < 9; ++c) b.R0[9 * q + c] = b.R[9 * q + c];
            for (int c = 0; c < 3; ++c) b.T0[3 * q + c] = b.T[3 * q + c];
            for (int c = 0; c < 8; ++c) b.DQ0[8 * q + c] = b.DQ[8 * q + c];
        }
    }
    // the regulariser objective at the current state (mstep.py:386-401)
    double part = 0.0;
    if (reg)
        for (int e2 = threadIdx.x; e2 < 2 * st->n_edges; e2 += blockDim.x) {
            double xk[3], xl[3], rr[3];
            ng_arap_rows(b, e2 >> 1, e2 & 1, b.R, b.T, xk, xl, rr);
            part += 0.5 * ((rr[0] * rr[0] + rr[1] * rr[1]) + rr[2] * rr[2]);
        }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0 && first) {
        double arap = 0.0;
        for (int w = 0; w < (int)(blockDim.x / 32); ++w) arap += red[w];
        st->value0 = st->value = b.gsums[0] + arap;
        st->gn = 0;
        st->gn_skip = 0;
        st->mstep_ran = 1;
    }
}

// the assembled system at the current node state: data blocks + ARAP
// (mstep.py:290-314), banded over the node order `pos`, one thread per band
// slot, each slot's contributions in a fixed order
__global__ void __launch_bounds__(kNgAsmThreads) k_ng_assemble(NgBufs b) {
    NgDev *st = b.st;
    if (st->gn_skip) return;
    const int n = st->n, bw = st->bw, W = bw + 1;
    const bool reg = st->lambda > 0.0 && st->n_edges > 0;
    // per band slot (i, d): d = 0 -> node diagonal block + its incident ARAP
    // terms; d > 0 -> the listed pair / edge blocks, in list order
    for (int sidx = blockIdx.x * blockDim.x + threadIdx.x; sidx < n * W;
         sidx += gridDim.x * blockDim.x) {
        const int i = sidx / W, d = sidx % W;
        double blk[36];
        for (int q = 0; q < 36; ++q) blk[q] = 0.0;
        if (d == 0) {
            const int node = b.node_at[i];
            const double *dg = b.diag + 27 * node;
            int o = 0;
            for (int r = 0; r < 6; ++r)
                for (int c = r; c < 6; ++c) {
                    blk[6 * r + c] = dg[o];
                    blk[6 * c + r] = dg[o];
                    ++o;
                }
            double g6[6];
            for (int q = 0; q < 6; ++q) g6[q] = dg[21 + q];
            if (reg) {
                // reference order: for p in (P[l], P[k]): D += grouped(JkJk, k);
                // D += grouped(JlJl, l) -- per node in edge order per sweep
                for (int which = 0; which < 2; ++which)
                    for (int role = 0; role < 2; ++role)
                        for (int a = b.inc_ptr[node]; a < b.inc_ptr[node + 1]; ++a) {
                            const int ent = b.inc_ent[a];
                            if ((ent & 1) != role) continue;
                            const int e = ent >> 1;
                            double xk[3], xl[3], rr[3], J[3][6];
                            ng_arap_rows(b, e, which, b.R, b.T, xk, xl, rr);
                            const double root = sqrt(st->lambda);
                            ng_jac(role == 0 ? xk : xl, J);
                            const double sg = role == 0 ? root : -root;
                            for (int r = 0; r < 6; ++r) {
                                for (int c = 0; c < 6; ++c) {
                                    double v = 0.0;
                                    for (int q = 0; q < 3; ++q) v += (sg * J[q][r]) * (sg * J[q][c]);
                                    blk[6 * r + c] += v;
                                }
                                double v = 0.0;
                                for (int q = 0; q < 3; ++q) v += (sg * J[q][r]) * rr[q];
                                g6[r] += v;
                            }
                        }
            }
            for (int q = 0; q < 6; ++q) b.bvec[6 * i + q] = g6[q];
        } else if (i - d >= 0) {
            const int j = i - d;
            const int ni = b.node_at[i], nj = b.node_at[j];
            for (int a = b.slot_ptr[sidx]; a < b.slot_ptr[sidx + 1]; ++a) {
                const int ent = b.slot_ent[a];
                const int kind = ent >> 30, idx = ent & 0x3fffffff;
                double X[36];     // block A[row node][col node] of the contribution
                int rn;
                if (kind == 0) {
                    const double *ob = b.off + 21 * idx;
                    int o = 0;
                    for (int r = 0; r < 6; ++r)
                        for (int c = r; c < 6; ++c) {
                            X[6 * r + c] = ob[o];
                            X[6 * c + r] = ob[o];
                            ++o;
                        }
                    rn = b.pair_lo[idx];
                } else {
                    // A[k][l] += Jk^T Jl over both endpoint positions
                    for (int q = 0; q < 36; ++q) X[q] = 0.0;
                    for (int which = 0; which < 2; ++which) {
                        double xk[3], xl[3], rr[3], Jk[3][6], Jl[3][6];
                        ng_arap_rows(b, idx, which, b.R, b.T, xk, xl, rr);
                        const double root = sqrt(st->lambda);
                        ng_jac(xk, Jk);
                        ng_jac(xl, Jl);
                        for (int r = 0; r < 6; ++r)
                            for (int c = 0; c < 6; ++c) {
                                double v = 0.0;
                                for (int q = 0; q < 3; ++q) v += (root * Jk[q][r]) * (-root * Jl[q][c]);
                                X[6 * r + c] += v;
                            }
                    }
                    rn = b.edges[2 * idx];
                }
                // symmetric pair blocks are stored as the band's A[ni][nj]
                const bool tr = rn != ni;
                for (int r = 0; r < 6; ++r)
                    for (int c = 0; c < 6; ++c) blk[6 * r + c] += tr ? X[6 * c + r] : X[6 * r + c];
                (void)nj;
            }
        }
        double *dst = b.band + (size_t)sidx * 36;
        for (int q = 0; q < 36; ++q) dst[q] = blk[q];
    }
}

// 6x6 in-place Cholesky (lower) of a diagonal block; false when not SPD
// 6x6 Cholesky in registers (A row-major, lower triangle out, upper zeroed);
// rd[j] = 1 / L_jj.  One column per template step so every index is a
// compile-time constant and A stays in registers.
template <int J>
__device__ __forceinline__ bool chol6_col(double (&A)[36], double *rd) {
    double d = A[6 * J + J];
#pragma unroll
    for (int k = 0; k < J; ++k) d -= A[6 * J + k] * A[6 * J + k];
    const bool good = d > 0.0 && isfinite(d);
    const double dd = fmax(d, 1e-300);
    const double r = rsqrt64(dd);            // 1 / l, and l = d / l
    A[6 * J + J] = dd * r;
    rd[J] = r;
#pragma unroll
    for (int i = J + 1; i < 6; ++i) {
        double v = A[6 * i + J];
#pragma unroll
        for (int k = 0; k < J; ++k) v -= A[6 * i + k] * A[6 * J + k];
        A[6 * i + J] = v * r;
    }
#pragma unroll
    for (int c = J + 1; c < 6; ++c) A[6 * J + c] = 0.0;
    return good;
}

__device__ __forceinline__ bool chol6_reg(double (&A)[36], double *rd) {
    bool g = chol6_col<0>(A, rd);
    g &= chol6_col<1>(A, rd);
    g &= chol6_col<2>(A, rd);
    g &= chol6_col<3>(A, rd);
    g &= chol6_col<4>(A, rd);
    g &= chol6_col<5>(A, rd);
    return g;
}

// (A + lam I) x = b by a block-banded Cholesky with the damping escalation
// of mstep.py:348-369; the step is -x in node order.  One CTA; the active
// window -- block rows k .. k + bw -- is held in REGISTERS: thread t owns the
// block whose two ring slots are the t-th unordered slot pair, for as long as
// both of its rows stay in the window (a block leaving with row k is
// replaced by one of the entering row k + bw + 1 on the same slots).  Per
// step k: the (k, k) owner factors its 6x6 pivot in registers and
// forward-substitutes y_k (sync); each (i, k) owner forms L_ik = A_ik
// L_kk^-T, takes its row's share of the forward substitution and publishes
// L_ik^T in shared memory (sync); every other owner applies
// A_ij -= L_ik L_jk^T from the published panel (broadcast reads, no
// read-modify-write of shared memory).  Rows of L go to global memory for the
// backward substitution.
constexpr int kNgMaxBw = 24;
constexpr int kNgW = kNgMaxBw + 1;
constexpr int kNgFacThreads = 352;      // >= kNgW (kNgW + 1) / 2 block owners

__global__ void __launch_bounds__(kNgFacThreads, 1) k_ng_factor(NgBufs b) {
    NgDev *st = b.st;
    if (st->gn_skip) return;
    const int n = st->n, bw = st->bw, W = bw + 1, P = 6 * n;
    const int tid = threadIdx.x, NT = blockDim.x;
    __shared__ int ok, anyb;
    __shared__ double s_trace, s_lam;
    __shared__ double red[kNgFacThreads / 32];
    __shared__ __align__(16) double Akk_s[36];            // the next pivot block
    __shared__ __align__(16) double panel2[1][kNgW][37];   // L_{k+d,k}^T (column c at 6c); 37: rows on distinct banks
    __shared__ double yring[(kNgW + 1) * 6];
    __shared__ __align__(16) double brow[2][kNgW * 36];     // backward: rows of L (and the
                                                            // forward loop's entering row)
    int nz = 0;
    double tr = 0.0;
    for (int q = tid; q < P; q += NT) {
        nz |= b.bvec[q] != 0.0;
        const int i = q / 6, r = q % 6;
        tr += b.band[(size_t)i * W * 36 + 6 * r + r];
    }
    nz = __syncthreads_or(nz);
    for (int o = 16; o > 0; o >>= 1) tr += __shfl_down_sync(0xffffffffu, tr, o);
    if ((tid & 31) == 0) red[tid >> 5] = tr;
    __syncthreads();
    if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NT / 32; ++w) t += red[w];
        s_trace = t;
        s_lam = st->use_damping ? st->damping : 1e-6 * t / P;
        anyb = nz;
        if (!nz) st->gn_skip = 1;           // zero gradient: no step (mstep.py:429)
    }
    __syncthreads();
    if (!anyb) return;
    // this thread's slot pair (pa >= pb): tid = pa (pa + 1) / 2 + pb
    int pa = 0;
    while ((pa + 1) * (pa + 2) / 2 <= tid) ++pa;
    const int pb = tid - pa * (pa + 1) / 2;
    const bool owner = pa < W;
    bool solved = false;
#pragma unroll 1
    for (int attempt = 0; attempt < 6 && !solved; ++attempt) {
        const double lam = s_lam;
        double blk[36];
        // block (i, i - d) of the assembled band (+ lam on the diagonal)
        auto load = [&](int i, int d) {
            const double *src = b.band + ((size_t)i * W + d) * 36;
#pragma unroll
            for (int q = 0; q < 36; ++q) blk[q] = src[q] + ((d == 0 && q % 7 == 0) ? lam : 0.0);
        };
#pragma unroll
        for (int q = 0; q < 36; ++q) blk[q] = 0.0;
        if (owner && pa < n) load(pa, pa - pb);          // window of k = 0: slot = row
        if (owner && pa == 0 && n > 0)
#pragma unroll
            for (int q = 0; q < 36; ++q) Akk_s[q] = blk[q];   // the first pivot block
        for (int e = tid; e < min(W, n) * 6; e += NT) yring[e] = b.bvec[e];
        if (tid == 0) ok = 1;
        __syncthreads();
        // (dataflow through shared-memory counters instead of the two barriers
        // per step was measured slower: 1.04 vs 0.72 ms per factorisation --
        // the spinning warps take issue slots from the trailing updates)
        int kw = 0;                                     // k % W
        constexpr int kPreF = kNgW * 36 / kNgFacThreads + 1;   // entering-row doubles per thread
#pragma unroll 1
        for (int k = 0; k < n; ++k) {
            constexpr int par = 0;     // (single buffers: two barriers per step)
            // the row entering after this step (k + W), loaded now by every
            // thread (coalesced; latency hidden behind the pivot and panel)
            double pre[kPreF];
            const bool incoming = k + W < n;
            if (incoming) {
                const double *src = b.band + (size_t)(k + W) * W * 36;
#pragma unroll
                for (int u = 0; u < kPreF; ++u) {
                    const int e = tid + u * NT;
                    pre[u] = e < W * 36 ? src[e] : 0.0;
                }
            }
            int oa = pa - kw, ob = pb - kw;
            oa += oa < 0 ? W : 0;
            ob += ob < 0 ? W : 0;
            const int hi = max(oa, ob), lo = min(oa, ob);
            const int i = k + hi;
            const bool live = owner && i < n;
            const int si = kw + hi >= W ? kw + hi - W : kw + hi;     // slot of row i
            // (1) the column k: every owner of a block (i, k) -- the pivot's
            //     and the panel's -- factors the published pivot block A_kk
            //     itself (no barrier between pivot and panel), forms
            //     y_k = L_kk^-1 b_k, then its own block row of L
            __syncthreads();                            // A_kk (and b_k) published
            if (live && lo == 0) {
                double Lk[36], rdk[6], yk[6];
#pragma unroll
                for (int q = 0; q < 36; ++q) Lk[q] = Akk_s[q];
                const bool good = chol6_reg(Lk, rdk);
#pragma unroll
                for (int r = 0; r < 6; ++r) {
                    double v = yring[6 * kw + r];
#pragma unroll
                    for (int q = 0; q < r; ++q) v -= Lk[6 * r + q] * yk[q];
                    yk[r] = v * rdk[r];
                }
                if (hi == 0) {
                    if (!good) {
                        ok = 0;
                    } else {
                        double *Lg = b.L + (size_t)k * W * 36;
#pragma unroll
                        for (int r = 0; r < 6; ++r) b.x[6 * k + r] = yk[r];
#pragma unroll
                        for (int q = 0; q < 36; ++q) Lg[q] = Lk[q];
                        // the reciprocal pivots ride in the stored block's
                        // (zero) upper triangle: (0, 1..5) and (1, 2); the
                        // backward substitution multiplies by them
#pragma unroll
                        for (int c = 0; c < 5; ++c) Lg[1 + c] = rdk[c];
                        Lg[8] = rdk[5];
                    }
                } else if (good) {
                    // L_ik = A_ik L_kk^-T, b_i -= L_ik y_k
                    double acc[6];
#pragma unroll
                    for (int r = 0; r < 6; ++r) {
                        double dot = 0.0;
#pragma unroll
                        for (int c = 0; c < 6; ++c) {
                            double u = blk[6 * r + c];
#pragma unroll
                            for (int q = 0; q < c; ++q) u -= blk[6 * r + q] * Lk[6 * c + q];
                            u *= rdk[c];
                            blk[6 * r + c] = u;
                            dot += u * yk[c];
                        }
                        acc[r] = dot;
                    }
#pragma unroll
                    for (int r = 0; r < 6; ++r) yring[6 * si + r] -= acc[r];
                    double *Lg = b.L + ((size_t)i * W + hi) * 36;
#pragma unroll
                    for (int r = 0; r < 6; ++r)
#pragma unroll
                        for (int c = 0; c < 6; ++c) {
                            panel2[par][hi][6 * c + r] = blk[6 * r + c];
                            Lg[6 * r + c] = blk[6 * r + c];
                        }
                }
            }
            if (incoming) {
                double *stage = brow[0];
#pragma unroll
                for (int u = 0; u < kPreF; ++u) {
                    const int e = tid + u * NT;
                    if (e < W * 36) stage[e] = pre[u];
                }
            }
            __syncthreads();
            if (!ok) break;
            // (3) the trailing update A_ij -= L_ik L_jk^T (both rows below k);
            //     the owner of (k + 1, k + 1) publishes it as the next pivot
            if (live && lo > 0) {
                const double *Pi = panel2[par][hi], *Pj = panel2[par][lo];
#pragma unroll
                for (int q = 0; q < 6; ++q) {
                    double li[6], lj[6];
#pragma unroll
                    for (int r = 0; r < 6; ++r) {
                        li[r] = Pi[6 * q + r];
                        lj[r] = Pj[6 * q + r];
                    }
#pragma unroll
                    for (int r = 0; r < 6; ++r)
#pragma unroll
                        for (int c = 0; c < 6; ++c) blk[6 * r + c] = fma(-li[r], lj[c], blk[6 * r + c]);
                }
                if (hi == 1 && lo == 1)
#pragma unroll
                    for (int q = 0; q < 36; ++q) Akk_s[q] = blk[q];
            }
            // (4) row k's blocks leave: their owners take the entering row k + W
            //     (slot kw; its right-hand side replaces b_k, read in (1))
            if (owner && lo == 0 && incoming) {
                const int d = hi == 0 ? 0 : W - hi;
                const double *src = brow[0] + d * 36;
#pragma unroll
                for (int q = 0; q < 36; ++q) blk[q] = src[q] + ((d == 0 && q % 7 == 0) ? lam : 0.0);
                if (hi == 0)
                    for (int r = 0; r < 6; ++r) yring[6 * kw + r] = b.bvec[6 * (k + W) + r];
            }
            kw = kw + 1 == W ? 0 : kw + 1;
        }
        __syncthreads();
        if (ok) {
            // L^T x = y, right-looking: x_k = L_kk^-T y_k, then y_j -= L_kj^T x_k
            // for the band's j < k; yring slot j % (W + 1) holds y_j for j in
            // [k - W, k] (the rows the step updates plus the one entering next)
            const int W1 = W + 1;
            for (int e = tid; e < W * 6; e += NT) {
                const int j = n - 1 - e / 6;
                if (j >= 0) yring[(j % W1) * 6 + e % 6] = b.x[6 * j + e % 6];
            }
            for (int e = tid; e < W * 36; e += NT)
                brow[(n - 1) & 1][e] = b.L[(size_t)(n - 1) * W * 36 + e];
            __syncthreads();
            constexpr int kPre = kNgW * 36 / kNgFacThreads + 1;
            int kw1 = (n - 1) % W1;                                 // k % (W + 1)
            for (int k = n - 1; k >= 0; --k, kw1 = kw1 == 0 ? W : kw1 - 1) {
                const double *row = brow[k & 1];
                double pre[kPre], ypre = 0.0;
                if (k > 0) {
                    const double *src = b.L + (size_t)(k - 1) * W * 36;
#pragma unroll
                    for (int u = 0; u < kPre; ++u) {
                        const int e = tid + u * NT;
                        pre[u] = e < W * 36 ? src[e] : 0.0;
                    }
                }
                if (tid < 6 && k - W >= 0) ypre = b.x[6 * (k - W) + tid];
                double *xk = yring + kw1 * 6;
                if (tid == 0) {
                    double x[6];
#pragma unroll
                    for (int r = 5; r >= 0; --r) {
                        double v = xk[r];
#pragma unroll
                        for (int q = r + 1; q < 6; ++q) v -= row[6 * q + r] * x[q];
                        // 1 / L_rr from the block's upper triangle (forward pass)
                        x[r] = v * (r < 5 ? row[1 + r] : row[8]);
                    }
#pragma unroll
                    for (int r = 0; r < 6; ++r) {
                        xk[r] = x[r];
                        b.x[6 * k + r] = x[r];
                    }
                }
                __syncthreads();
                for (int t = tid; t < bw * 6; t += NT) {
                    const int d = 1 + t / 6, r = t % 6;
                    if (k - d < 0) continue;
                    const double *Lkj = row + d * 36;      // block (k, k - d)
                    double v = 0.0;
#pragma unroll
                    for (int q = 0; q < 6; ++q) v += Lkj[6 * q + r] * xk[q];
                    const int sj = kw1 - d;
                    yring[(sj < 0 ? sj + W1 : sj) * 6 + r] -= v;
                }
                if (tid < 6 && k - W >= 0) {
                    const int sj = kw1 - W;
                    yring[(sj < 0 ? sj + W1 : sj) * 6 + tid] = ypre;
                }
                if (k > 0) {
                    double *dst = brow[(k - 1) & 1];
#pragma unroll
                    for (int u = 0; u < kPre; ++u) {
                        const int e = tid + u * NT;
                        if (e < W * 36) dst[e] = pre[u];
                    }
                }
                __syncthreads();
            }
            int fin = 1;
            for (int q = tid; q < P; q += NT) fin &= isfinite(b.x[q]) ? 1 : 0;
            fin = __syncthreads_and(fin);
            solved = fin;
        }
        if (!solved && tid == 0)
            s_lam = s_lam > 0.0 ? s_lam * 10.0 : fmax(s_trace / P, 1.0) * 1e-10;
        __syncthreads();
    }
    if (!solved) {
        if (tid == 0) {
            st->termination = kTermSolver;
            st->done = 1;
            st->gn_skip = 1;
            st->iterations += 1;
        }
        return;
    }
    for (int q = tid; q < P; q += NT) {
        const int node = q / 6, r = q % 6;
        b.step[q] = -b.x[6 * b.pos[node] + r];
    }
}

// candidate node states exp(0.5^h step) o T for h < ncand (kinematics.py:307-311)
__global__ void k_ng_cands(NgBufs b) {
    NgDev *st = b.st;
    if (st->gn_skip) return;
    const int n = st->n;
    const int nc = min(st->max_halvings + 1, kNgMaxCand);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->ncand = nc;
        st->accepted = 0;                       // this GN step's candidate not yet decided
    }
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nc * n; t += gridDim.x * blockDim.x) {
        const int h = t / n, node = t % n;
        const double scale = ldexp(1.0, -h);
        double tw[6];
        for (int q = 0; q < 6; ++q) tw[q] = scale * b.step[6 * node + q];
        double R2[9], t2[3];
        apply_twist_dev(tw, b.R + 9 * node, b.T + 3 * node, R2, t2);
        double *cR = b.candR + ((size_t)h * n + node) * 9;
        double *cT = b.candT + ((size_t)h * n + node) * 3;
        for (int q = 0; q < 9; ++q) cR[q] = R2[q];
        for (int q = 0; q < 3; ++q) cT[q] = t2[q];
        ng_dq(R2, t2, b.candDQ + ((size_t)h * n + node) * 8);
    }
}

// + ARAP objectives of the candidates, first accepted (mstep.py:443-459),
// state update, Gauss-Newton continuation
__global__ void __launch_bounds__(kNgThreads, 1) k_ng_select(NgBufs b, int h0, int h1) {
    // candidates [h0, h1) in halving order; the first launch takes h = 0
    // alone (the usual outcome: the full step is accepted, and the other
    // candidates' passes are skipped), the second the rest
    NgDev *st = b.st;
    if (st->gn_skip || st->accepted) return;
    const int n = st->n, nc = st->ncand;
    h1 = min(h1, nc);
    __shared__ double red[kNgThreads / 32][kNgMaxCand];
    __shared__ int acc_h;
    __shared__ double s_sn;
    const bool reg = st->lambda > 0.0 && st->n_edges > 0;
    double part[kNgMaxCand];
    for (int h = 0; h < kNgMaxCand; ++h) part[h] = 0.0;
    if (reg)
        for (int e2 = threadIdx.x; e2 < 2 * st->n_edges; e2 += blockDim.x)
            for (int h = h0; h < h1; ++h) {
                double xk[3], xl[3], rr[3];
                ng_arap_rows(b, e2 >> 1, e2 & 1, b.candR + (size_t)h * n * 9,
                             b.candT + (size_t)h * n * 3, xk, xl, rr);
                part[h] += 0.5 * ((rr[0] * rr[0] + rr[1] * rr[1]) + rr[2] * rr[2]);
            }
    for (int h = 0; h < kNgMaxCand; ++h) {
        double v = part[h];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][h] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        acc_h = -1;
        if (*b.flag) {
            st->termination = kNgTermBlend;
            st->done = 1;
            st->gn_skip = 1;
        } else {
            for (int h = h0; h < h1 && acc_h < 0; ++h) {
                double arap = 0.0;
                for (int w = 0; w < (int)(blockDim.x / 32); ++w) arap += red[w][h];
                const double cv = b.cand_data[h] + arap;
                if (cv <= st->value * (1.0 + 1e-12) + 1e-300) {
                    acc_h = h;
                    st->value = cv;
                }
            }
            if (acc_h >= 0 || h1 >= nc) st->accepted = 1;     // decided
            if (acc_h < 0 && h1 >= nc) st->gn_skip = 1;      // no acceptable step (mstep.py:450-451)
        }
    }
    __syncthreads();
    if (acc_h < 0) return;
    // the accepted step's norm (block tree) and the node states
    const double scale = ldexp(1.0, -acc_h);
    double sn = 0.0;
    for (int q = threadIdx.x; q < 6 * n; q += blockDim.x) sn += (scale * b.step[q]) * (scale * b.step[q]);
    for (int o = 16; o > 0; o >>= 1) sn += __shfl_down_sync(0xffffffffu, sn, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][0] = sn;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += red[w][0];
        s_sn = t;
        st->gn += 1;
        st->gn_skip = (sqrt(t) <= st->step_tol || st->gn >= st->max_gn_iters) ? 1 : 0;
    }
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const size_t o = (size_t)acc_h * n + q;
        for (int c = 0; c < 9; ++c) b.R[9 * q + c] = b.candR[9 * o + c];
        for (int c = 0; c < 3; ++c) b.T[3 * q + c] = b.candT[3 * o + c];
        for (int c = 0; c < 8; ++c) b.DQ[8 * q + c] = b.candDQ[8 * o + c];
    }
}

// update magnitude (batched form of pipeline.py:79-86) and termination
// (pipeline.py:167-177)
__global__ void __launch_bounds__(kNgThreads, 1) k_ng_finish(NgBufs b) {
    NgDev *st = b.st;
    if (st->done || !st->mstep_ran) return;
    const int n = st->n;
    __shared__ double red[kNgThreads / 32];
    double worst = 0.0;
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        double Rd[9];
        m3_mul_t(b.R + 9 * q, b.R0 + 9 * q, Rd);
        const double dx = b.T[3 * q] - b.T0[3 * q], dy = b.T[3 * q + 1] - b.T0[3 * q + 1],
                     dz = b.T[3 * q + 2] - b.T0[3 * q + 2];
        worst = fmax(worst, rotation_angle_dev(Rd) + sqrt((dx * dx + dy * dy) + dz * dz) /
                                                         st->diameter);
    }
    for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_down_sync(0xffffffffu, worst, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = worst;
    __syncthreads();
    __shared__ int conv;
    if (threadIdx.x == 0) {
        double norm = 0.0;
        for (int w = 0; w < (int)(blockDim.x / 32); ++w) norm = fmax(norm, red[w]);
        const int it = st->iterations;
        b.traces[st->max_em_iters + it] = norm;
        st->iterations = it + 1;
        conv = norm < st->tol;
        if (conv) {                 // sub-tolerance motion: dropped (pipeline.py:169-173)
            b.traces[it] = st->value0;
            st->termination = kTermConverged;
            st->done = 1;
        } else {
            b.traces[it] = st->value;
            if (it + 1 >= st->max_em_iters) {
                st->termination = kTermMaxIters;
                st->done = 1;
            }
        }
        st->mstep_ran = 0;
    }
    __syncthreads();
    if (conv)
        for (int q = threadIdx.x; q < n; q += blockDim.x) {
            for (int c = 0; c < 9; ++c) b.R[9 * q + c] = b.R0[9 * q + c];
            for (int c = 0; c < 3; ++c) b.T[3 * q + c] = b.T0[3 * q + c];
            for (int c = 0; c < 8; ++c) b.DQ[8 * q + c] = b.DQ0[8 * q + c];
        }
}

}  // namespace fr

using namespace fr;

extern "C" {

int fr_point_rows(const double *X, const double *W, const double *T, const double *N,
                  const uint8_t *valid, int64_t m, int mode, const double *sigma_inv,
                  double *ete, void *stream) {
    if (!X || !W || !T || !ete || !sigma_inv || (mode == FR_POINT_TO_PLANE && (!N || !valid))) {
        set_error("invalid point-rows arguments");
        return FR_EINVAL;
    }
    if (m == 0) return FR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    k_point_rows<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(X, W, T, N, valid, m, mode,
                                                            sigma_inv[0], sigma_inv[1],
                                                            sigma_inv[2], ete);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

int fr_graph_pass(const fr_lattice *lat, const float *ref, int64_t m, const int32_t *sidx,
                  const double *swt, int K, const double *node_dq, int mode,
                  const double *sigma_inv, double c_prime, int respec, double *rec, double *ete,
                  double *sums, double *scratch, int32_t *d_flag, void *stream) {
    if (!lat || !lat->blurred || lat->dim != 3 || !ref || !sidx || !swt || !node_dq || !rec ||
        !ete || !sums || !scratch || !d_flag || K < 1 || K > kMaxK || !sigma_inv) {
        set_error("invalid node-graph pass arguments (1 <= K <= %d)", kMaxK);
        return FR_EINVAL;
    }
    GraphK g;
    memset(&g, 0, sizeof(g));
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 3; ++j) {
            double e = 0.0;
            if (i == 0) e = 1.0;
            else if (j == i - 1) e = -(double)i;
            else if (j >= i) e = 1.0;
            g.A[i][j] = e * lat->c.sf[j] / lat->c.sigma[j];
        }
    for (int j = 0; j < 3; ++j) g.sinv[j] = sigma_inv[j];
    g.cp = c_prime;
    g.gain = lat->c.gain;
    g.mode = mode;
    g.K = K;
    const int nv = lat->nv;
    const bool pl = mode == FR_POINT_TO_PLANE;
    g.m2_col = (nv == 5 || nv == 8) ? 4 : -1;
    g.ncol = pl ? (nv == 8 ? 5 : 4) : -1;
    if ((pl && nv != 7 && nv != 8) || (!pl && nv != 4 && nv != 5)) {
        set_error("lattice value columns (%d) do not match the residual mode", nv);
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (m == 0) {
        FR_CUDA(cudaMemsetAsync(sums, 0, kGraphAcc * sizeof(double), s));
        return FR_OK;
    }
    const int grid = pass_grid();
    const SliceTable t = lat->table();
#define FR_G(NV, RS) \
    k_graph_pass<NV, RS><<<grid, kPassThreads, 0, s>>>(ref, m, sidx, swt, node_dq, g, t, rec, ete, scratch, d_flag)
    if (respec) {
        FR_G(4, true);
    } else {
        switch (nv) {
            case 4: FR_G(4, false); break;
            case 5: FR_G(5, false); break;
            case 7: FR_G(7, false); break;
            default: FR_G(8, false); break;
        }
    }
#undef FR_G
    FR_CHECK_LAUNCH();
    k_reduce_cols<<<1, 32 * kGraphAcc, 0, s>>>(scratch, grid, kGraphAcc, sums, nullptr);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

int fr_graph_blocks(const double *ete, const double *swt, int K, const int32_t *dptr,
                    const int32_t *dent, int n_nodes, const int32_t *pptr, const int32_t *pent,
                    int n_pairs, double *diag, double *off, void *stream) {
    if (!ete || !swt || !dptr || !diag || (n_pairs > 0 && (!pptr || !pent || !off))) {
        set_error("invalid node-graph block arguments");
        return FR_EINVAL;
    }
    const long long warps = (long long)n_nodes + n_pairs;
    if (warps == 0) return FR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int threads = 128;
    const unsigned blocks = (unsigned)((warps * 32 + threads - 1) / threads);
    k_graph_blocks<<<blocks, threads, 0, s>>>(ete, swt, K, dptr, dent, n_nodes, pptr, pent, n_pairs,
                                              diag, off);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

int fr_graph_objective(const float *ref, int64_t m, const int32_t *sidx, const double *swt, int K,
                       const double *d_cand_dq, int n_nodes, int ncand, const double *rec,
                       int mode, const double *sigma_inv, double *out, double *scratch,
                       int32_t *d_flag, void *stream) {
    if (!ref || !sidx || !swt || !d_cand_dq || ncand < 1 || ncand > kGraphMaxCand || !rec ||
        !out || !scratch || !d_flag || !sigma_inv || K < 1 || K > kMaxK) {
        set_error("invalid node-graph objective arguments (1 <= k <= %d)", kGraphMaxCand);
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = pass_grid();
    k_graph_objective<<<grid, kPassThreads, 0, s>>>(ref, m, sidx, swt, K, d_cand_dq, n_nodes, ncand,
                                                    rec, mode, sigma_inv[0], sigma_inv[1],
                                                    sigma_inv[2], scratch, d_flag);
    FR_CHECK_LAUNCH();
    k_reduce_cols<<<1, 32 * kGraphMaxCand, 0, s>>>(scratch, grid, kGraphMaxCand, out, nullptr);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

}  // extern "C"

// ---- device-resident node-graph EM object ---------------------------------
struct fr_ng_em {
    const fr_lattice *lat = nullptr;
    const float *ref = nullptr;
    long long m = 0;
    int K = 0, n = 0, n_pairs = 0, mode = 0, max_iters = 0, max_gn = 1, ncand = 1, bw = 0;
    const int32_t *sidx = nullptr, *dptr = nullptr, *dent = nullptr, *pptr = nullptr,
                  *pent = nullptr;
    const double *swt = nullptr;
    fr::GraphK g{};
    fr::NgBufs b{};
    // owned buffers
    fr::NgDev *d_st = nullptr;
    double *d_rec = nullptr, *d_ete = nullptr, *d_scratch = nullptr, *d_gsums = nullptr,
           *d_diag = nullptr, *d_off = nullptr, *d_cdata = nullptr;
    std::vector<void *> owned;
    int *d_flag = nullptr;
    int *d_piece_blk = nullptr, *d_piece_beg = nullptr, *d_piece_end = nullptr,
        *d_blk_piece0 = nullptr;
    double *d_piece_vals = nullptr;
    int n_pieces = 0;
    cudaGraphExec_t graph = nullptr;
    cudaStream_t stream = nullptr;
};

using namespace fr;

static void ng_blocks(fr_ng_em *em, const int *skip, cudaStream_t s) {
    const unsigned g = (unsigned)(((long long)em->n_pieces * 32 + 127) / 128);
    k_graph_block_pieces<<<g, 128, 0, s>>>(em->d_ete, em->swt, em->K, em->dent, em->pent, em->n,
                                           em->d_piece_blk, em->d_piece_beg, em->d_piece_end,
                                           em->n_pieces,
                                           em->d_piece_vals, skip);
    const long long t = (long long)(em->n + em->n_pairs) * 27;
    k_graph_pieces_combine<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(
        em->d_blk_piece0, em->n, em->n_pairs, em->d_piece_vals, em->d_diag, em->d_off, skip);
}

static int ng_iteration(fr_ng_em *em, cudaStream_t s) {
    const int grid = pass_grid();
    const SliceTable t = em->lat->table();
    FR_CUDA(cudaMemsetAsync(em->d_flag, 0, sizeof(int), s));
    const int *done = &em->d_st->done, *gskip = &em->d_st->gn_skip;
    const int nv = em->lat->nv;
#define FR_G(NV, RS, SKIP)                                                                      \
    k_graph_pass<NV, RS><<<grid, kPassThreads, 0, s>>>(em->ref, em->m, em->sidx, em->swt,         \
                                                       em->b.DQ, em->g, t, em->d_rec, em->d_ete, \
                                                       em->d_scratch, em->d_flag, SKIP)
    switch (nv) {
        case 4: FR_G(4, false, done); break;
        case 7: FR_G(7, false, done); break;
        default: set_error("node-graph device loop: lattice columns %d", nv); return FR_EINVAL;
    }
    FR_CHECK_LAUNCH();
    k_reduce_cols<<<1, 32 * kGraphAcc, 0, s>>>(em->d_scratch, grid, kGraphAcc, em->d_gsums, done);
    const long long warps = (long long)em->n + em->n_pairs;
    const unsigned gb = (unsigned)((warps * 32 + 127) / 128);
    (void)gb;
    ng_blocks(em, done, s);
    FR_CHECK_LAUNCH();
    const unsigned ga = (unsigned)(((long long)em->n * (em->bw + 1) + kNgAsmThreads - 1) / kNgAsmThreads);
    k_ng_begin<<<1, kNgThreads, 0, s>>>(em->b, 1);
    k_ng_assemble<<<ga, kNgAsmThreads, 0, s>>>(em->b);
    FR_CHECK_LAUNCH();
    for (int gn = 0; gn < em->max_gn; ++gn) {
        if (gn > 0) {
            FR_G(4, true, gskip);
            FR_CHECK_LAUNCH();
            k_reduce_cols<<<1, 32 * kGraphAcc, 0, s>>>(em->d_scratch, grid, kGraphAcc,
                                                      em->d_gsums + 8, gskip);
            ng_blocks(em, gskip, s);
            k_ng_assemble<<<ga, kNgAsmThreads, 0, s>>>(em->b);
            FR_CHECK_LAUNCH();
        }
        k_ng_factor<<<1, kNgFacThreads, 0, s>>>(em->b);
        k_ng_cands<<<(unsigned)((kNgMaxCand * em->n + 255) / 256), 256, 0, s>>>(em->b);
        // the full step first; the halved candidates only if it is rejected
        const int *decided = &em->d_st->accepted;
        k_graph_objective<<<grid, kPassThreads, 0, s>>>(
            em->ref, em->m, em->sidx, em->swt, em->K, em->b.candDQ, em->n, 1, em->d_rec,
            em->mode, em->g.sinv[0], em->g.sinv[1], em->g.sinv[2], em->d_scratch, em->d_flag,
            gskip, 0, decided);
        k_reduce_cols<<<1, 32 * kGraphMaxCand, 0, s>>>(em->d_scratch, grid, kGraphMaxCand,
                                                        em->d_cdata, gskip, decided);
        k_ng_select<<<1, kNgThreads, 0, s>>>(em->b, 0, 1);
        if (em->ncand > 1) {
            k_graph_objective<<<grid, kPassThreads, 0, s>>>(
                em->ref, em->m, em->sidx, em->swt, em->K, em->b.candDQ, em->n, em->ncand - 1,
                em->d_rec, em->mode, em->g.sinv[0], em->g.sinv[1], em->g.sinv[2], em->d_scratch,
                em->d_flag, gskip, 1, decided);
            k_reduce_cols<<<1, 32 * kGraphMaxCand, 0, s>>>(em->d_scratch, grid, kGraphMaxCand,
                                                            em->d_cdata, gskip, decided);
            k_ng_select<<<1, kNgThreads, 0, s>>>(em->b, 1, em->ncand);
        }
        FR_CHECK_LAUNCH();
    }
#undef FR_G
    k_ng_finish<<<1, kNgThreads, 0, s>>>(em->b);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

extern "C" {

int fr_ng_em_create(const fr_lattice *lat, const float *ref, int64_t m, const int32_t *sidx,
                    const double *swt, int K, int n_nodes, const double *node_pos,
                    const int32_t *edges, int n_edges, const int32_t *dptr, const int32_t *dent,
                    const int32_t *pptr, const int32_t *pent, int n_pairs, const int32_t *pair_lo,
                    const int32_t *pair_hi, const int32_t *pos, int bw, const int32_t *slot_ptr,
                    const int32_t *slot_ent, int n_slot_ent, const int32_t *inc_ptr,
                    const int32_t *inc_ent, const double *node_R, const double *node_t,
                    const double *node_dq, int mode, double lambda_reg,
                    const fr_rigid_em_config *cfg, void *stream, fr_ng_em **out) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!lat || !lat->blurred || lat->dim != 3 || !ref || !sidx || !swt || K < 1 || K > kMaxK ||
        n_nodes < 1 || !node_pos || (n_edges > 0 && !edges) || !dptr || !dent || !pos || bw < 0 ||
        !slot_ptr || !inc_ptr || !node_R || !node_t || !node_dq || !cfg || !out || m <= 0 ||
        (n_pairs > 0 && (!pptr || !pent || !pair_lo || !pair_hi))) {
        set_error("invalid node-graph device EM arguments");
        return FR_EINVAL;
    }
    const bool pl = mode == FR_POINT_TO_PLANE;
    if ((pl && lat->nv != 7) || (!pl && lat->nv != 4)) {
        set_error("node-graph device loop: lattice value columns (%d) do not match the mode", lat->nv);
        return FR_EINVAL;
    }
    if (bw > kNgMaxBw) {
        set_error("node-graph device loop: block bandwidth %d above %d", bw, kNgMaxBw);
        return FR_ECAPACITY;
    }
    if (cfg->max_halvings + 1 > kNgMaxCand || cfg->max_gn_iters < 0 || cfg->max_gn_iters > 8 ||
        cfg->max_em_iters < 1) {
        set_error("node-graph device loop: max_halvings <= %d, max_gn_iters <= 8", kNgMaxCand - 1);
        return FR_EINVAL;
    }
    fr_ng_em *em = new fr_ng_em();
    em->lat = lat;
    em->ref = ref;
    em->m = m;
    em->K = K;
    em->n = n_nodes;
    em->n_pairs = n_pairs;
    em->mode = mode;
    em->max_iters = cfg->max_em_iters;
    em->max_gn = std::max(cfg->max_gn_iters, 1);
    em->ncand = cfg->max_halvings + 1;
    em->bw = bw;
    em->sidx = sidx;
    em->swt = swt;
    em->dptr = dptr;
    em->dent = dent;
    em->pptr = pptr;
    em->pent = pent;
    em->stream = s;
    GraphK &g = em->g;
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 3; ++j) {
            double e = 0.0;
            if (i == 0) e = 1.0;
            else if (j == i - 1) e = -(double)i;
            else if (j >= i) e = 1.0;
            g.A[i][j] = e * lat->c.sf[j] / lat->c.sigma[j];
        }
    for (int j = 0; j < 3; ++j) g.sinv[j] = cfg->sigma_inv[j];
    g.cp = cfg->c_prime;
    g.gain = lat->c.gain;
    g.mode = mode;
    g.K = K;
    g.m2_col = -1;
    g.ncol = pl ? 4 : -1;
    NgDev h;
    memset(&h, 0, sizeof(h));
    for (int j = 0; j < 3; ++j) h.sinv[j] = cfg->sigma_inv[j];
    h.cp = cfg->c_prime;
    h.diameter = cfg->diameter;
    h.tol = cfg->twist_tolerance;
    h.use_damping = cfg->damping >= 0.0;
    h.damping = cfg->damping;
    h.step_tol = cfg->step_tolerance;
    h.degenerate_mass = cfg->degenerate_mass;
    h.lambda = lambda_reg;
    h.n = n_nodes;
    h.n_edges = n_edges;
    h.bw = bw;
    h.max_em_iters = cfg->max_em_iters;
    h.max_gn_iters = std::max(cfg->max_gn_iters, 0);
    h.max_halvings = cfg->max_halvings;
    h.mode = mode;
    h.gn_skip = 1;
    const int W = bw + 1, n = n_nodes;
    auto dalloc = [&](void **p, size_t bytes) -> bool {
        if (cudaMallocAsync(p, std::max<size_t>(bytes, 8), s) != cudaSuccess) return false;
        em->owned.push_back(*p);
        return true;
    };
    auto up = [&](void **p, const void *src, size_t bytes) -> bool {
        return dalloc(p, bytes) && (bytes == 0 ||
                                    cudaMemcpyAsync(*p, src, bytes, cudaMemcpyHostToDevice, s) ==
                                        cudaSuccess);
    };
    // band-position inverse
    std::vector<int32_t> node_at((size_t)n);
    for (int q = 0; q < n; ++q) node_at[pos[q]] = q;
    NgBufs &B = em->b;
    void *p = nullptr;
    bool ok = true;
    ok = ok && dalloc((void **)&em->d_st, sizeof(NgDev)) &&
         cudaMemcpyAsync(em->d_st, &h, sizeof(NgDev), cudaMemcpyHostToDevice, s) == cudaSuccess;
    B.st = em->d_st;
    ok = ok && up(&p, node_R, (size_t)n * 9 * 8); B.R = (double *)p;
    ok = ok && up(&p, node_t, (size_t)n * 3 * 8); B.T = (double *)p;
    ok = ok && up(&p, node_dq, (size_t)n * 8 * 8); B.DQ = (double *)p;
    ok = ok && dalloc(&p, (size_t)n * 9 * 8); B.R0 = (double *)p;
    ok = ok && dalloc(&p, (size_t)n * 3 * 8); B.T0 = (double *)p;
    ok = ok && dalloc(&p, (size_t)n * 8 * 8); B.DQ0 = (double *)p;
    ok = ok && up(&p, node_pos, (size_t)n * 3 * 8); B.P = (const double *)p;
    ok = ok && up(&p, edges, (size_t)n_edges * 2 * 4); B.edges = (const int *)p;
    ok = ok && up(&p, pos, (size_t)n * 4); B.pos = (const int *)p;
    ok = ok && up(&p, node_at.data(), (size_t)n * 4); B.node_at = (const int *)p;
    ok = ok && up(&p, slot_ptr, ((size_t)n * W + 1) * 4); B.slot_ptr = (const int *)p;
    ok = ok && up(&p, slot_ent, (size_t)n_slot_ent * 4); B.slot_ent = (const int *)p;
    ok = ok && up(&p, inc_ptr, ((size_t)n + 1) * 4); B.inc_ptr = (const int *)p;
    ok = ok && up(&p, inc_ent, (size_t)2 * n_edges * 4); B.inc_ent = (const int *)p;
    ok = ok && up(&p, pair_lo, (size_t)n_pairs * 4); B.pair_lo = (const int *)p;
    ok = ok && up(&p, pair_hi, (size_t)n_pairs * 4); B.pair_hi = (const int *)p;
    {
        // the block gather's pieces (fixed: the entry lists are set at create)
        std::vector<int32_t> hd((size_t)n + 1), hp((size_t)n_pairs + 1);
        ok = ok && cudaMemcpyAsync(hd.data(), dptr, hd.size() * 4, cudaMemcpyDeviceToHost, s) ==
                       cudaSuccess &&
             (n_pairs == 0 || cudaMemcpyAsync(hp.data(), pptr, hp.size() * 4,
                                              cudaMemcpyDeviceToHost, s) == cudaSuccess) &&
             cudaStreamSynchronize(s) == cudaSuccess;
        std::vector<int32_t> pblk, pbeg, pend, bp0((size_t)n + n_pairs + 1);
        if (ok)
            for (int blk = 0; blk < n + n_pairs; ++blk) {
                const int b0 = blk < n ? hd[blk] : hp[blk - n];
                const int b1 = blk < n ? hd[blk + 1] : hp[blk - n + 1];
                bp0[blk] = (int32_t)pblk.size();
                for (int e = b0; e < b1; e += kGraphPiece) {
                    pblk.push_back(blk);
                    pbeg.push_back(e);
                    pend.push_back(std::min(e + kGraphPiece, b1));
                }
            }
        bp0[(size_t)n + n_pairs] = (int32_t)pblk.size();
        em->n_pieces = (int)pblk.size();
        ok = ok && up((void **)&em->d_piece_blk, pblk.data(), pblk.size() * 4) &&
             up((void **)&em->d_piece_beg, pbeg.data(), pbeg.size() * 4) &&
             up((void **)&em->d_piece_end, pend.data(), pend.size() * 4) &&
             up((void **)&em->d_blk_piece0, bp0.data(), bp0.size() * 4) &&
             dalloc((void **)&em->d_piece_vals, (size_t)std::max(em->n_pieces, 1) * 27 * 8);
    }
    ok = ok && dalloc((void **)&em->d_gsums, 16 * 8); B.gsums = em->d_gsums;
    ok = ok && dalloc((void **)&em->d_diag, (size_t)n * 27 * 8); B.diag = em->d_diag;
    ok = ok && dalloc((void **)&em->d_off, (size_t)std::max(n_pairs, 1) * 21 * 8); B.off = em->d_off;
    ok = ok && dalloc(&p, (size_t)n * W * 36 * 8); B.band = (double *)p;
    ok = ok && dalloc(&p, (size_t)n * 6 * 8); B.bvec = (double *)p;
    ok = ok && dalloc(&p, (size_t)n * W * 36 * 8); B.L = (double *)p;
    ok = ok && dalloc(&p, (size_t)n * 6 * 8); B.x = (double *)p;
    ok = ok && dalloc(&p, (size_t)n * 6 * 8); B.step = (double *)p;
    ok = ok && dalloc(&p, (size_t)kNgMaxCand * n * 9 * 8); B.candR = (double *)p;
    ok = ok && dalloc(&p, (size_t)kNgMaxCand * n * 3 * 8); B.candT = (double *)p;
    ok = ok && dalloc(&p, (size_t)kNgMaxCand * n * 8 * 8); B.candDQ = (double *)p;
    ok = ok && dalloc((void **)&em->d_cdata, kNgMaxCand * 8); B.cand_data = em->d_cdata;
    ok = ok && dalloc(&p, (size_t)3 * cfg->max_em_iters * 8); B.traces = (double *)p;
    ok = ok && dalloc((void **)&em->d_flag, sizeof(int)); B.flag = em->d_flag;
    ok = ok && dalloc((void **)&em->d_rec, (size_t)7 * m * 8);
    ok = ok && dalloc((void **)&em->d_ete, (size_t)m * kGraphEte * 8);
    ok = ok && dalloc((void **)&em->d_scratch, (size_t)pass_grid_max() * 32 * 8);
    ok = ok && cudaMemsetAsync(B.traces, 0, (size_t)3 * cfg->max_em_iters * 8, s) == cudaSuccess;
    ok = ok && cudaStreamSynchronize(s) == cudaSuccess;
    if (!ok) {
        fr_ng_em_destroy(em);
        set_error("node-graph device EM allocation failed");
        return FR_ECUDA;
    }
    *out = em;
    return FR_OK;
}

int fr_ng_em_destroy(fr_ng_em *em) {
    if (!em) return FR_OK;
    cudaStreamSynchronize(em->stream);
    if (em->graph) cudaGraphExecDestroy(em->graph);
    for (void *p : em->owned) cudaFreeAsync(p, em->stream);
    delete em;
    return FR_OK;
}

int fr_ng_em_run(fr_ng_em *em, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    em->stream = s;
    if (!em->graph) {
        cudaStream_t cs;
        FR_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t g;
        FR_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        const int st = ng_iteration(em, cs);
        cudaStreamEndCapture(cs, &g);
        cudaStreamDestroy(cs);
        FR_TRY(st);
        FR_CUDA(cudaGraphInstantiate(&em->graph, g, 0));
        cudaGraphDestroy(g);
    }
    static thread_local int *flags = nullptr;       // [2][4] pinned
    static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
    if (!flags) {
        FR_CUDA(cudaHostAlloc((void **)&flags, 8 * sizeof(int), cudaHostAllocDefault));
        for (int i = 0; i < 2; ++i) FR_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    constexpr int kChunk = 2;
    int issued = 0, k = 0;
    auto chunk = [&]() -> int {
        for (int i = 0; i < kChunk; ++i) FR_CUDA(cudaGraphLaunch(em->graph, s));
        FR_CUDA(cudaMemcpyAsync(flags + 4 * (k & 1), &em->d_st->done, 3 * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
        FR_CUDA(cudaEventRecord(ev[k & 1], s));
        issued += kChunk;
        ++k;
        return FR_OK;
    };
    FR_TRY(chunk());
    while (true) {
        const bool more = issued < em->max_iters + kChunk;
        if (more) FR_TRY(chunk());
        const int prev = (k - (more ? 2 : 1)) & 1;
        FR_CUDA(cudaEventSynchronize(ev[prev]));
        if (flags[4 * prev] || !more) break;
    }
    FR_CUDA(cudaStreamSynchronize(s));
    return FR_OK;
}

// node poses (n x 9 / n x 3), traces, iterations, termination (4: a dual
// quaternion blend degenerated -> DegenerateBlendError)
int fr_ng_em_result(fr_ng_em *em, double *node_R, double *node_t, double *objectives,
                    double *twist_norms, double *inlier_masses, int *iterations,
                    int *termination, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    NgDev h;
    FR_CUDA(cudaMemcpyAsync(&h, em->d_st, sizeof(NgDev), cudaMemcpyDeviceToHost, s));
    std::vector<double> tr((size_t)3 * em->max_iters);
    FR_CUDA(cudaMemcpyAsync(tr.data(), em->b.traces, tr.size() * 8, cudaMemcpyDeviceToHost, s));
    if (node_R) FR_CUDA(cudaMemcpyAsync(node_R, em->b.R, (size_t)em->n * 9 * 8, cudaMemcpyDeviceToHost, s));
    if (node_t) FR_CUDA(cudaMemcpyAsync(node_t, em->b.T, (size_t)em->n * 3 * 8, cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaStreamSynchronize(s));
    const int n = std::min(h.iterations, em->max_iters);
    if (objectives) memcpy(objectives, tr.data(), n * 8);
    if (twist_norms) memcpy(twist_norms, tr.data() + em->max_iters, n * 8);
    if (inlier_masses) memcpy(inlier_masses, tr.data() + 2 * em->max_iters, n * 8);
    if (iterations) *iterations = h.iterations;
    if (termination) *termination = h.termination;
    if (h.termination == kTermSolver && h.done) {
        set_error("normal equations not factorizable after damping escalation");
        return FR_ESOLVER;
    }
    return FR_OK;
}

}  // extern "C"
