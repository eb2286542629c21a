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

#include "fr_reduce.cuh"

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
             double *__restrict__ partials, int *bad) {
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
                               double *__restrict__ diag, double *__restrict__ off) {
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

constexpr int kGraphMaxCand = 16;

__global__ void __launch_bounds__(kPassThreads, 2)
k_graph_objective(const float *__restrict__ ref, long long m, const int *__restrict__ sidx,
                  const double *__restrict__ swt, int K, const double *__restrict__ cand_dq,
                  int n_nodes, int ncand, const double *__restrict__ rec, int mode, double s0,
                  double s1, double s2, double *__restrict__ partials, int *bad) {
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
            if (c >= ncand) break;
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
