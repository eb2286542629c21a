// E step and fused rigid EM pass on B200.
//
//   fr_moments          MomentEngine.moments (estep.py:186-217): exact fp64
//                       slice + epilogue per model point (generic API).
//   fr_rigid_pass       one sweep over the model points per EM iteration:
//                       forward transform (kinematics.py:317-320), slice,
//                       moments epilogue, residual rows and the normal-equation
//                       sums (mstep.py:102-210), block-reduced in fp64 with a
//                       fixed-order tree (deterministic, no float atomics).
//   fr_rigid_objective  candidate objectives for step halving (mstep.py:443-449)
//                       in point_to_plane mode, from the stored weight/target/
//                       normal planes.
#include <algorithm>
#include <cmath>

#include "fr_common.cuh"

namespace fr {

// ---------------------------------------------------------------------------
// deterministic block / grid reductions

constexpr int kPassThreads = 256;

template <int NA>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NA], double *dst) {
    __shared__ double red[kPassThreads / 32][NA];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < NA; ++a) {
        double v = acc[a];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp][a] = v;
    }
    __syncthreads();
    if (threadIdx.x < NA) {
        double v = 0.0;
        for (int w = 0; w < kPassThreads / 32; ++w) v += red[w][threadIdx.x];
        dst[threadIdx.x] = v;
    }
}

// column c of partials[nblk][na] reduced by warp c, fixed order
__global__ void k_reduce_cols(const double *partials, int nblk, int na, double *out) {
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (c >= na) return;
    double v = 0.0;
    for (int b = lane; b < nblk; b += 32) v += partials[(long long)b * na + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) out[c] = v;
}

// ---------------------------------------------------------------------------
// generic moments (fp64 positions, exact query embedding)

template <int VP>
__global__ void k_moments(const double *X, long long m, LatticeConsts c, const SliceSlot<VP> *tab,
                          unsigned mask, double cp, int m2_col, int ncol, double *m0o,
                          double *m1o, double *wo, double *to, double *m2o, double *no,
                          unsigned char *nvo) {
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        double x[3] = {X[p * 3], X[p * 3 + 1], X[p * 3 + 2]};
        Simplex<3> s;
        simplex_exact<3>(x, c, s);
        double acc[VP];
#pragma unroll
        for (int q = 0; q < VP; ++q) acc[q] = 0.0;
        if (!s.overflow) {
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const SliceSlot<VP> *hit = probe<VP>(tab, mask, s.packed(l));
                if (hit) {
#pragma unroll
                    for (int q = 0; q < VP; ++q)
                        acc[q] = __dadd_rn(acc[q], __dmul_rn(s.bary[l], hit->v[q]));
                }
            }
        }
#pragma unroll
        for (int q = 0; q < VP; ++q) acc[q] = __dmul_rn(c.gain, acc[q]);
        // epilogue (estep.py:195-217)
        const double m0 = fmax(acc[0], 0.0);
        const bool sup = m0 >= 1e-12;
        const double w = sup ? (cp > 0.0 ? m0 / (m0 + cp) : 1.0) : 0.0;
        const double safe = sup ? m0 : 1.0;
        m0o[p] = m0;
        wo[p] = w;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            m1o[p * 3 + j] = acc[1 + j];
            to[p * 3 + j] = sup ? acc[1 + j] / safe : x[j];
        }
        if (m2o && m2_col >= 0) {
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < VP; ++q) v = (q == m2_col) ? acc[q] : v;
            m2o[p] = v;
        }
        if (ncol >= 0 && (no || nvo)) {
            double a[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                double v = 0.0;
#pragma unroll
                for (int q = 0; q < VP; ++q) v = (q == ncol + j) ? acc[q] : v;
                a[j] = v / safe;
            }
            const double len = sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]);
            const bool valid = sup && len >= 0.1;
            const double dn = fmax(len, 0.1);
            if (no)
                for (int j = 0; j < 3; ++j) no[p * 3 + j] = valid ? a[j] / dn : 0.0;
            if (nvo) nvo[p] = valid;
        }
    }
}

// ---------------------------------------------------------------------------
// fused rigid pass

struct RigidK {
    double M[4][3];      // elevated = M xh + e0 (embedding folded with the pose)
    double e0[4];
    double R[9];
    double c_ref[3];
    double c_world[3];
    double cp;
    double gain;
    int m2_col;
    int ncol;
};

// accumulator widths (layout documented in paper_1811_10136_b200/_rigid.py)
constexpr int kP2PtBase = 25;
constexpr int kP2PlBase = 29;

__device__ __forceinline__ double pt2pl_cost(double w, const double *t, const double *n,
                                             const double *x) {
    const double d0 = x[0] - t[0], d1 = x[1] - t[1], d2 = x[2] - t[2];
    if (n[0] != 0.0 || n[1] != 0.0 || n[2] != 0.0) {
        const double r = (n[0] * d0 + n[1] * d1) + n[2] * d2;
        return w * (r * r);
    }
    return w * ((d0 * d0 + d1 * d1) + d2 * d2);
}

template <int MODE, int VP, bool SIG>
__global__ void __launch_bounds__(kPassThreads, 2)
k_rigid_pass(const float *__restrict__ ref, long long m, RigidK k,
             const SliceSlot<VP> *__restrict__ tab, unsigned mask,
             float *__restrict__ wtn, double *__restrict__ partials) {
    constexpr int NA = (MODE == FR_POINT_TO_POINT ? kP2PtBase : kP2PlBase) + (SIG ? 2 : 0);
    double acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        const double xh[3] = {(double)__ldg(ref + p) - k.c_ref[0],
                              (double)__ldg(ref + m + p) - k.c_ref[1],
                              (double)__ldg(ref + 2 * m + p) - k.c_ref[2]};
        double xt[3], x[3];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            xt[i] = fma(k.R[3 * i + 2], xh[2], fma(k.R[3 * i + 1], xh[1], k.R[3 * i] * xh[0]));
            x[i] = xt[i] + k.c_world[i];
        }
        double el[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            el[i] = fma(k.M[i][2], xh[2], fma(k.M[i][1], xh[1], fma(k.M[i][0], xh[0], k.e0[i])));
        Simplex<3> s;
        simplex_from_elevated<3>(el, s);
        double out[VP];
#pragma unroll
        for (int q = 0; q < VP; ++q) out[q] = 0.0;
        if (!s.overflow) {
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const SliceSlot<VP> *hit = probe<VP>(tab, mask, s.packed(l));
                if (hit) {
                    const double b = s.bary[l];
#pragma unroll
                    for (int q = 0; q < VP; ++q) out[q] = fma(b, hit->v[q], out[q]);
                }
            }
        }
        const double m0 = fmax(k.gain * out[0], 0.0);
        const bool sup = m0 >= 1e-12;
        double w = sup ? (k.cp > 0.0 ? m0 / (m0 + k.cp) : 1.0) : 0.0;
        const double inv = sup ? 1.0 / m0 : 0.0;
        double t[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) t[j] = sup ? (k.gain * out[1 + j]) * inv : x[j];
        if (MODE == FR_POINT_TO_POINT) {
            if (w > 0.0) {
                double r[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) r[j] = x[j] - t[j];
                acc[0] += w;
                double wx[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    wx[j] = w * xt[j];
                    acc[1 + j] += wx[j];
                }
                acc[4] = fma(wx[0], xt[0], acc[4]);
                acc[5] = fma(wx[0], xt[1], acc[5]);
                acc[6] = fma(wx[0], xt[2], acc[6]);
                acc[7] = fma(wx[1], xt[1], acc[7]);
                acc[8] = fma(wx[1], xt[2], acc[8]);
                acc[9] = fma(wx[2], xt[2], acc[9]);
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const double wr = w * r[j];
                    acc[10 + j] += wr;
#pragma unroll
                    for (int q = 0; q < 3; ++q) acc[13 + 3 * j + q] = fma(wr, xt[q], acc[13 + 3 * j + q]);
                    acc[22 + j] = fma(wr, r[j], acc[22 + j]);
                }
            }
        } else {
            // point_to_plane: averaged normal, validity (estep.py:209-215)
            double n[3] = {0.0, 0.0, 0.0};
            if (sup) {
                double a[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) a[j] = (k.gain * out[k.ncol + j]) * inv;
                const double len = sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]);
                if (len >= 0.1) {
#pragma unroll
                    for (int j = 0; j < 3; ++j) n[j] = a[j] / len;
                }
            }
            // round to the stored float32 values so the candidate pass sees
            // exactly the residual definition assembled here
            const float wf = (float)w;
            const float tf[3] = {(float)t[0], (float)t[1], (float)t[2]};
            const float nf[3] = {(float)n[0], (float)n[1], (float)n[2]};
            wtn[p] = wf;
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                wtn[(1 + j) * m + p] = tf[j];
                wtn[(4 + j) * m + p] = nf[j];
            }
            acc[0] += w;
            const double wr = (double)wf;
            if (wr > 0.0) {
                const double tr[3] = {tf[0], tf[1], tf[2]};
                const double nr[3] = {nf[0], nf[1], nf[2]};
                const double d[3] = {x[0] - tr[0], x[1] - tr[1], x[2] - tr[2]};
                acc[28] += pt2pl_cost(wr, tr, nr, x);
                if (nr[0] != 0.0 || nr[1] != 0.0 || nr[2] != 0.0) {
                    // row [x x n, n], residual n.(x - t)
                    const double a6[6] = {x[1] * nr[2] - x[2] * nr[1], x[2] * nr[0] - x[0] * nr[2],
                                          x[0] * nr[1] - x[1] * nr[0], nr[0], nr[1], nr[2]};
                    const double rr = (nr[0] * d[0] + nr[1] * d[1]) + nr[2] * d[2];
                    int o = 1;
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
                        const double wa = wr * a6[i];
#pragma unroll
                        for (int j = i; j < 6; ++j) { acc[o] = fma(wa, a6[j], acc[o]); ++o; }
                        acc[22 + i] = fma(wa, rr, acc[22 + i]);
                    }
                } else {
                    // no usable plane: point rows J = [-[x]x | I] in meters
                    double J[3][6] = {{0.0, x[2], -x[1], 1.0, 0.0, 0.0},
                                      {-x[2], 0.0, x[0], 0.0, 1.0, 0.0},
                                      {x[1], -x[0], 0.0, 0.0, 0.0, 1.0}};
                    int o = 1;
#pragma unroll
                    for (int i = 0; i < 6; ++i) {
#pragma unroll
                        for (int j = i; j < 6; ++j) {
                            const double h = (J[0][i] * J[0][j] + J[1][i] * J[1][j]) + J[2][i] * J[2][j];
                            acc[o] = fma(wr, h, acc[o]);
                            ++o;
                        }
                        const double gi = (J[0][i] * d[0] + J[1][i] * d[1]) + J[2][i] * d[2];
                        acc[22 + i] = fma(wr, gi, acc[22 + i]);
                    }
                }
            }
        }
        if (SIG && sup) {
            // sigma update sums (estep.py:248-255)
            constexpr int B = (MODE == FR_POINT_TO_POINT ? kP2PtBase : kP2PlBase);
            const double den = m0 + k.cp;
            const double xx = (x[0] * x[0] + x[1] * x[1]) + x[2] * x[2];
            const double xm = (x[0] * (k.gain * out[1]) + x[1] * (k.gain * out[2])) + x[2] * (k.gain * out[3]);
            double m2v = 0.0;
#pragma unroll
            for (int q = 0; q < VP; ++q) m2v = (q == k.m2_col) ? k.gain * out[q] : m2v;
            acc[B] += (m0 * xx - 2.0 * xm + m2v) / den;
            acc[B + 1] += m0 / den;
        }
    }
    block_reduce_store<NA>(acc, partials + (long long)blockIdx.x * NA);
}

// candidate objectives for point_to_plane halving
constexpr int kMaxCand = 16;
struct CandK {
    double R[kMaxCand][9];
    double c[kMaxCand][3];
    double c_ref[3];
    int k;
};

__global__ void __launch_bounds__(kPassThreads, 2)
k_rigid_objective(const float *__restrict__ ref, const float *__restrict__ wtn, long long m,
                  CandK ck, double *__restrict__ partials) {
    double acc[kMaxCand];
#pragma unroll
    for (int a = 0; a < kMaxCand; ++a) acc[a] = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        const double w = (double)__ldg(wtn + p);
        if (!(w > 0.0)) continue;
        const double xh[3] = {(double)__ldg(ref + p) - ck.c_ref[0],
                              (double)__ldg(ref + m + p) - ck.c_ref[1],
                              (double)__ldg(ref + 2 * m + p) - ck.c_ref[2]};
        const double t[3] = {(double)__ldg(wtn + m + p), (double)__ldg(wtn + 2 * m + p),
                             (double)__ldg(wtn + 3 * m + p)};
        const double n[3] = {(double)__ldg(wtn + 4 * m + p), (double)__ldg(wtn + 5 * m + p),
                             (double)__ldg(wtn + 6 * m + p)};
#pragma unroll
        for (int c = 0; c < kMaxCand; ++c) {
            if (c >= ck.k) break;
            double x[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const double xt = fma(ck.R[c][3 * i + 2], xh[2],
                                      fma(ck.R[c][3 * i + 1], xh[1], ck.R[c][3 * i] * xh[0]));
                x[i] = xt + ck.c[c][i];
            }
            acc[c] += pt2pl_cost(w, t, n, x);
        }
    }
    block_reduce_store<kMaxCand>(acc, partials + (long long)blockIdx.x * kMaxCand);
}


// ---------------------------------------------------------------------------
// moments epilogue over raw kernel sums (estep.py:195-217), for the slice /
// brute-force paths that do not fuse it (feature modes, other dims)

__global__ void k_epilogue(const double *raw, long long m, int nv, const double *X, double cp,
                           int m2_col, int ncol, double *m0o, double *m1o, double *wo, double *to,
                           double *m2o, double *no, unsigned char *nvo) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= m) return;
    const double *o = raw + p * nv;
    const double m0 = fmax(o[0], 0.0);
    const bool sup = m0 >= 1e-12;
    const double safe = sup ? m0 : 1.0;
    m0o[p] = m0;
    wo[p] = sup ? (cp > 0.0 ? m0 / (m0 + cp) : 1.0) : 0.0;
    for (int j = 0; j < 3; ++j) {
        m1o[p * 3 + j] = o[1 + j];
        to[p * 3 + j] = sup ? o[1 + j] / safe : X[p * 3 + j];
    }
    if (m2o && m2_col >= 0) m2o[p] = o[m2_col];
    if (ncol >= 0 && (no || nvo)) {
        double a[3];
        for (int j = 0; j < 3; ++j) a[j] = o[ncol + j] / safe;
        const double len = sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]);
        const bool valid = sup && len >= 0.1;
        const double dn = fmax(len, 0.1);
        if (no)
            for (int j = 0; j < 3; ++j) no[p * 3 + j] = valid ? a[j] / dn : 0.0;
        if (nvo) nvo[p] = valid;
    }
}

// ---------------------------------------------------------------------------
// explicit rigid assembly over caller-provided residual specs
// (mstep.py:102-138, 179-210): sums [H upper 21 | g 6 | sum r^2]

constexpr int kExplicitWidth = 28;

__global__ void __launch_bounds__(kPassThreads, 2)
k_assemble_explicit(const double *__restrict__ X, const double *__restrict__ W,
                    const double *__restrict__ T, long long m, double s0, double s1, double s2,
                    int mode, const double *__restrict__ N, const unsigned char *__restrict__ valid,
                    double *__restrict__ partials) {
    double acc[kExplicitWidth];
#pragma unroll
    for (int a = 0; a < kExplicitWidth; ++a) acc[a] = 0.0;
    const double sinv[3] = {s0, s1, s2};
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        const double w = W[p];
        if (!(w > 0.0)) continue;
        const double sw = sqrt(w);
        const double x[3] = {X[p * 3], X[p * 3 + 1], X[p * 3 + 2]};
        const double d[3] = {x[0] - T[p * 3], x[1] - T[p * 3 + 1], x[2] - T[p * 3 + 2]};
        const double J[3][6] = {{0.0, x[2], -x[1], 1.0, 0.0, 0.0},
                                {-x[2], 0.0, x[0], 0.0, 1.0, 0.0},
                                {x[1], -x[0], 0.0, 0.0, 0.0, 1.0}};
        double P[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        int rows = 3;
        if (mode == FR_POINT_TO_POINT) {
            for (int j = 0; j < 3; ++j) P[j][j] = sw * sinv[j];
        } else if (valid[p]) {
            rows = 1;
            for (int j = 0; j < 3; ++j) P[0][j] = sw * N[p * 3 + j];
        } else {
            for (int j = 0; j < 3; ++j) P[j][j] = sw;
        }
        for (int r = 0; r < rows; ++r) {
            double G[6];
            for (int c = 0; c < 6; ++c) G[c] = (P[r][0] * J[0][c] + P[r][1] * J[1][c]) + P[r][2] * J[2][c];
            const double rr = (P[r][0] * d[0] + P[r][1] * d[1]) + P[r][2] * d[2];
            int o = 0;
            for (int i = 0; i < 6; ++i) {
                for (int j = i; j < 6; ++j) { acc[o] = fma(G[i], G[j], acc[o]); ++o; }
                acc[21 + i] = fma(G[i], rr, acc[21 + i]);
            }
            acc[27] = fma(rr, rr, acc[27]);
        }
    }
    block_reduce_store<kExplicitWidth>(acc, partials + (long long)blockIdx.x * kExplicitWidth);
}

// ---------------------------------------------------------------------------
// host

static int g_pass_grid = 0;

static int pass_grid() {
    if (g_pass_grid) return g_pass_grid;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_pass_grid = sms * 2;   // __launch_bounds__(256, 2): one full wave, fixed
    return g_pass_grid;
}

static int width(int mode, int sig) {
    return (mode == FR_POINT_TO_POINT ? kP2PtBase : kP2PlBase) + (sig ? 2 : 0);
}

template <int MODE, int VP, bool SIG>
static int launch_pass(const fr_lattice *lat, const float *ref, long long m, const RigidK &k,
                       float *wtn, double *scratch, double *sums, cudaStream_t s) {
    const int grid = pass_grid();
    k_rigid_pass<MODE, VP, SIG><<<grid, kPassThreads, 0, s>>>(
        ref, m, k, (const SliceSlot<VP> *)lat->slots, lat->smask, wtn, scratch);
    FR_CHECK_LAUNCH();
    const int na = width(MODE, SIG);
    k_reduce_cols<<<1, 32 * na, 0, s>>>(scratch, grid, na, sums);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

}  // namespace fr

using namespace fr;

extern "C" {

int fr_moments(const fr_lattice *lat, const double *X, int64_t m, double cp, int m2_col,
               int ncol, double *m0, double *m1, double *w, double *t, double *m2, double *nrm,
               uint8_t *nvalid, void *stream) {
    if (!lat || !lat->blurred) {
        set_error("moments require a built (blurred) lattice");
        return FR_ESTATE;
    }
    if (lat->dim != 3) {
        set_error("position moments need a 3-D lattice");
        return FR_EINVAL;
    }
    if (!m0 || !m1 || !w || !t) {
        set_error("null output");
        return FR_EINVAL;
    }
    if (m2_col >= lat->nv || ncol + 3 > lat->nv) {
        set_error("value column out of range");
        return FR_EINVAL;
    }
    if (m == 0) return FR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned grid = (unsigned)std::min<long long>((m + 255) / 256, 148LL * 16);
    switch (lat->vp) {
        case 3:
            k_moments<3><<<grid, 256, 0, s>>>(X, m, lat->c, (const SliceSlot<3> *)lat->slots,
                                              lat->smask, cp, m2_col, ncol, m0, m1, w, t, m2,
                                              nrm, nvalid);
            break;
        case 7:
            k_moments<7><<<grid, 256, 0, s>>>(X, m, lat->c, (const SliceSlot<7> *)lat->slots,
                                              lat->smask, cp, m2_col, ncol, m0, m1, w, t, m2,
                                              nrm, nvalid);
            break;
        default:
            k_moments<15><<<grid, 256, 0, s>>>(X, m, lat->c, (const SliceSlot<15> *)lat->slots,
                                               lat->smask, cp, m2_col, ncol, m0, m1, w, t, m2,
                                               nrm, nvalid);
            break;
    }
    FR_CHECK_LAUNCH();
    return FR_OK;
}


int fr_moments_epilogue(const double *raw, int64_t m, int nv, const double *X, double cp,
                        int m2_col, int ncol, double *m0, double *m1, double *w, double *t,
                        double *m2, double *nrm, uint8_t *nvalid, void *stream) {
    if (!raw || !X || !m0 || !m1 || !w || !t || nv < 4 || m2_col >= nv || ncol + 3 > nv) {
        set_error("invalid moments epilogue arguments");
        return FR_EINVAL;
    }
    if (m == 0) return FR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    k_epilogue<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(raw, m, nv, X, cp, m2_col, ncol, m0, m1,
                                                          w, t, m2, nrm, nvalid);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

int fr_assemble_rigid(const double *X, const double *W, const double *T, int64_t m,
                      const double *sigma_inv, int mode, const double *N, const uint8_t *valid,
                      double *sums, double *scratch, void *stream) {
    if (!sums || !scratch || !sigma_inv || (m > 0 && (!X || !W || !T)) ||
        (mode == FR_POINT_TO_PLANE && m > 0 && (!N || !valid))) {
        set_error("invalid rigid assembly arguments");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (m == 0) {
        FR_CUDA(cudaMemsetAsync(sums, 0, kExplicitWidth * sizeof(double), s));
        return FR_OK;
    }
    const int grid = pass_grid();
    k_assemble_explicit<<<grid, kPassThreads, 0, s>>>(X, W, T, m, sigma_inv[0], sigma_inv[1],
                                                      sigma_inv[2], mode, N, valid, scratch);
    FR_CHECK_LAUNCH();
    k_reduce_cols<<<1, 32 * kExplicitWidth, 0, s>>>(scratch, grid, kExplicitWidth, sums);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

int fr_rigid_pass_width(int mode, int with_sigma) { return width(mode, with_sigma); }

int fr_rigid_scratch_doubles(int mode, int with_sigma, int64_t m) {
    (void)m;
    return pass_grid() * std::max(std::max(width(mode, with_sigma), kMaxCand), kExplicitWidth);
}

int fr_rigid_pass(const fr_lattice *lat, const float *ref, int64_t m,
                  const fr_rigid_pass_params *p, double *sums, float *wtn, double *scratch,
                  void *stream) {
    if (!lat || !lat->blurred) {
        set_error("the EM pass needs a built (blurred) lattice");
        return FR_ESTATE;
    }
    if (lat->dim != 3 || !p || !sums || !scratch || (m > 0 && !ref)) {
        set_error("invalid rigid pass arguments");
        return FR_EINVAL;
    }
    const int mode = p->mode;
    if (mode != FR_POINT_TO_POINT && mode != FR_POINT_TO_PLANE) {
        set_error("unknown residual mode %d", mode);
        return FR_EINVAL;
    }
    if (mode == FR_POINT_TO_PLANE && (!wtn || p->normal_col < 0 || p->normal_col + 3 > lat->nv)) {
        set_error("point_to_plane needs the normal channel and weight/target/normal planes");
        return FR_EINVAL;
    }
    const bool sig = p->m2_col >= 0;
    if (sig && p->m2_col >= lat->nv) {
        set_error("m2 column out of range");
        return FR_EINVAL;
    }
    // fold embedding and pose: el = E diag(sf/sigma) (R xh + c_world)
    RigidK k;
    memset(&k, 0, sizeof(k));
    double A[4][3];   // E diag(sf / sigma)
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 3; ++j) {
            double e = 0.0;
            if (i == 0) e = 1.0;
            else if (j == i - 1) e = -(double)i;
            else if (j >= i) e = 1.0;
            A[i][j] = e * lat->c.sf[j] / lat->c.sigma[j];
        }
    for (int i = 0; i < 4; ++i) {
        for (int j = 0; j < 3; ++j) {
            double v = 0.0;
            for (int q = 0; q < 3; ++q) v += A[i][q] * p->R[3 * q + j];
            k.M[i][j] = v;
        }
        double e = 0.0;
        for (int q = 0; q < 3; ++q) e += A[i][q] * p->c_world[q];
        k.e0[i] = e;
    }
    memcpy(k.R, p->R, sizeof(k.R));
    memcpy(k.c_ref, p->c_ref, sizeof(k.c_ref));
    memcpy(k.c_world, p->c_world, sizeof(k.c_world));
    k.cp = p->c_prime;
    k.gain = lat->c.gain;
    k.m2_col = p->m2_col;
    k.ncol = p->normal_col;
    cudaStream_t s = (cudaStream_t)stream;
    const int na = width(mode, sig);
    if (m == 0) {
        FR_CUDA(cudaMemsetAsync(sums, 0, na * sizeof(double), s));
        return FR_OK;
    }
#define FR_PASS(MODE, VP)                                                                   \
    (sig ? launch_pass<MODE, VP, true>(lat, ref, m, k, wtn, scratch, sums, s)              \
         : launch_pass<MODE, VP, false>(lat, ref, m, k, wtn, scratch, sums, s))
    if (mode == FR_POINT_TO_POINT) {
        if (lat->vp == 3) return FR_PASS(FR_POINT_TO_POINT, 3);
        if (lat->vp == 7) return FR_PASS(FR_POINT_TO_POINT, 7);
        return FR_PASS(FR_POINT_TO_POINT, 15);
    }
    if (lat->vp == 7) return FR_PASS(FR_POINT_TO_PLANE, 7);
    return FR_PASS(FR_POINT_TO_PLANE, 15);
#undef FR_PASS
}

int fr_rigid_objective(const float *ref, const float *wtn, int64_t m, const double *c_ref, int k,
                       const double *cand_R, const double *cand_c, double *out, double *scratch,
                       void *stream) {
    if (k < 1 || k > kMaxCand || !ref || !wtn || !out || !scratch) {
        set_error("invalid candidate objective arguments (1 <= k <= %d)", kMaxCand);
        return FR_EINVAL;
    }
    CandK ck;
    memset(&ck, 0, sizeof(ck));
    for (int c = 0; c < k; ++c) {
        memcpy(ck.R[c], cand_R + 9 * c, 9 * sizeof(double));
        memcpy(ck.c[c], cand_c + 3 * c, 3 * sizeof(double));
    }
    memcpy(ck.c_ref, c_ref, sizeof(ck.c_ref));
    ck.k = k;
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = pass_grid();
    k_rigid_objective<<<grid, kPassThreads, 0, s>>>(ref, wtn, m, ck, scratch);
    FR_CHECK_LAUNCH();
    k_reduce_cols<<<1, 32 * kMaxCand, 0, s>>>(scratch, grid, kMaxCand, out);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

}  // extern "C"
