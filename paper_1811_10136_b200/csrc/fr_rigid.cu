// Rigid FilterReg EM on B200: the fused per-iteration pass and the
// device-resident Gauss-Newton solver.
//
//   k_rigid_pass     one sweep over the model points per EM iteration: forward
//                    transform (kinematics.py:317-320), lattice slice
//                    (permutohedral.py:329-341), moments epilogue
//                    (estep.py:195-217) and the residual statistics of the M
//                    step (mstep.py:102-210), reduced in a fixed order.
//   k_rigid_solve    the rest of one EM iteration on one GPU thread, in float64:
//                    normal equations from the point-to-point statistics,
//                    damped Cholesky with tenfold escalation (mstep.py:348-369),
//                    step halving with closed-form candidate objectives
//                    (mstep.py:421-459), twist update with polar
//                    re-orthonormalisation (geometry.py:154-189), update
//                    magnitude and termination (pipeline.py:141-177).
//   k_rigid_objective  candidate objectives for point_to_plane halving.
//   k_rigid_pass_grid4 the point-to-point pass over the dense float32 slice
//                    grid (quarter-scale embedding, clamped cells, four
//                    consecutive points per thread).
//   k_rigid_pass_tiles the device loop's pass over centred 1024-point tiles,
//                    pass constants in the constant bank; its last block
//                    reduces the partials and (in the EM loop) runs the
//                    solve: one kernel per EM iteration.
// With the iterations in a CUDA graph an EM iteration needs no host round trip.
#include <cooperative_groups.h>
#include <math_constants.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <type_traits>
#include <vector>

#include "fr_reduce.cuh"
#include "fr_solve.cuh"

namespace fr {

// accumulator widths (layout documented in paper_1811_10136_b200/_rigid.py)
constexpr int kP2PtBase = 25;
constexpr int kP2PlBase = 29;
constexpr int kMaxCand = 16;

__device__ __forceinline__ double pt2pl_cost(double w, const double *t, const double *n,
                                             const double *x) {
    const double d0 = x[0] - t[0], d1 = x[1] - t[1], d2 = x[2] - t[2];
    if (n[0] != 0.0 || n[1] != 0.0 || n[2] != 0.0) {
        const double r = (n[0] * d0 + n[1] * d1) + n[2] * d2;
        return w * (r * r);
    }
    return w * ((d0 * d0 + d1 * d1) + d2 * d2);
}

// slice at one model point, float64 table (exact-path arithmetic)
template <int NV>
__device__ __forceinline__ void slice_point_exact(const double *el, const SliceTable &tab,
                                                  double *out) {
    Simplex<3> s;
    simplex_from_elevated<3>(el, s);
#pragma unroll
    for (int q = 0; q < NV; ++q) out[q] = 0.0;
    if (s.overflow) return;
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

// slice at one model point, float32 ranks / barycentrics / table rows; the
// table rows already carry the gain, so out[] is the finished kernel sum
template <int NV>
__device__ __forceinline__ void slice_point_fast(const double *el, const SliceTableF &tab,
                                                 float *out) {
    constexpr int NF4 = (NV + 3) / 4;
    QSimplex3 q;
    qsimplex3(el, q);
#pragma unroll
    for (int c = 0; c < 4 * NF4; ++c) out[c] = 0.0f;
    if (!q.overflow) {
        float4 v[4][NF4];
        gather_simplex_f<NF4>(tab, q.key, v);
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            const float b = q.bary[l];
#pragma unroll
            for (int f = 0; f < NF4; ++f) {
                out[4 * f] = fmaf(b, v[l][f].x, out[4 * f]);
                out[4 * f + 1] = fmaf(b, v[l][f].y, out[4 * f + 1]);
                out[4 * f + 2] = fmaf(b, v[l][f].z, out[4 * f + 2]);
                out[4 * f + 3] = fmaf(b, v[l][f].w, out[4 * f + 3]);
            }
        }
    }
}

// one model point of the EM pass: forward map, slice, epilogue, residual
// statistics into acc (and, for point_to_plane, the stored w / t / n planes)
template <int MODE, int NV, bool SIG, bool FAST, int NA>
__device__ __forceinline__ void point_step(const RigidK &k, const SliceTable &tab,
                                           const SliceTableF &tabf, const double *xh,
                                           long long p, long long m, float *__restrict__ wtn,
                                           double (&acc)[NA]) {
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
        double out[NV];
        double m0, w, t[3];
        bool sup;
        if (FAST) {
            // float32 epilogue (estep.py:195-205) on the float32 kernel sums
            float o[4 * ((NV + 3) / 4)];
            slice_point_fast<NV>(el, tabf, o);
            const float m0f = fmaxf(o[0], 0.0f);
            sup = m0f >= 1e-12f;
            const float cpf = (float)k.cp;
            const float wf = sup ? (cpf > 0.0f ? __fdividef(m0f, m0f + cpf) : 1.0f) : 0.0f;
            const float invf = sup ? __frcp_rn(m0f) : 0.0f;
            m0 = (double)m0f;
            w = (double)wf;
#pragma unroll
            for (int j = 0; j < 3; ++j) t[j] = sup ? (double)(o[1 + j] * invf) : x[j];
#pragma unroll
            for (int q = 0; q < NV; ++q) out[q] = (double)o[q];
        } else {
            slice_point_exact<NV>(el, tab, out);
#pragma unroll
            for (int q = 0; q < NV; ++q) out[q] *= k.gain;
            m0 = fmax(out[0], 0.0);
            sup = m0 >= 1e-12;
            w = sup ? (k.cp > 0.0 ? m0 / (m0 + k.cp) : 1.0) : 0.0;
            const double inv = sup ? 1.0 / m0 : 0.0;
#pragma unroll
            for (int j = 0; j < 3; ++j) t[j] = sup ? out[1 + j] * inv : x[j];
        }
        if (MODE == FR_POINT_TO_POINT) {
            // branch-free: unsupported points have w = 0 and t = x
            double r[3], wy[3];
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                r[j] = x[j] - t[j];
                wy[j] = w * xt[j];
            }
            acc[0] += w;
#pragma unroll
            for (int j = 0; j < 3; ++j) acc[1 + j] += wy[j];
            acc[4] = fma(wy[0], xt[0], acc[4]);
            acc[5] = fma(wy[0], xt[1], acc[5]);
            acc[6] = fma(wy[0], xt[2], acc[6]);
            acc[7] = fma(wy[1], xt[1], acc[7]);
            acc[8] = fma(wy[1], xt[2], acc[8]);
            acc[9] = fma(wy[2], xt[2], acc[9]);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const double wr = w * r[j];
                acc[10 + j] += wr;
#pragma unroll
                for (int q = 0; q < 3; ++q) acc[13 + 3 * j + q] = fma(wr, xt[q], acc[13 + 3 * j + q]);
                acc[22 + j] = fma(wr, r[j], acc[22 + j]);
            }
        } else {
            // point_to_plane: averaged normal and validity (estep.py:209-215)
            double n[3] = {0.0, 0.0, 0.0};
            if (sup) {
                const double inv = 1.0 / m0;
                double a[3];
#pragma unroll
                for (int j = 0; j < 3; ++j) a[j] = out[k.ncol + j] * inv;
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
                    const double J[3][6] = {{0.0, x[2], -x[1], 1.0, 0.0, 0.0},
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
            const double xm = (x[0] * out[1] + x[1] * out[2]) + x[2] * out[3];
            double m2v = 0.0;
#pragma unroll
            for (int q = 0; q < NV; ++q) m2v = (q == k.m2_col) ? out[q] : m2v;
            acc[B] += (m0 * xx - 2.0 * xm + m2v) / den;
            acc[B + 1] += m0 / den;
        }
}

template <int MODE, int NV, bool SIG, bool FAST, bool DEV>
__global__ void __launch_bounds__(kPassThreads, MODE == FR_POINT_TO_POINT ? 2 : 1)
k_rigid_pass(const float *__restrict__ ref, long long m, RigidK kv, const RigidK *kd,
             const int *done, SliceTable tab, SliceTableF tabf, float *__restrict__ wtn,
             double *__restrict__ partials) {
    constexpr int NA = (MODE == FR_POINT_TO_POINT ? kP2PtBase : kP2PlBase) + (SIG ? 2 : 0);
    __shared__ RigidK k;
    if (DEV && *done) return;
    if (threadIdx.x == 0) k = DEV ? *kd : kv;
    __syncthreads();
    double acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    // software prefetch of the next point's float32 position (hides the HBM
    // latency behind this point's work)
    float nx = 0.f, ny = 0.f, nz = 0.f;
    if (p < m) {
        nx = __ldg(ref + p);
        ny = __ldg(ref + m + p);
        nz = __ldg(ref + 2 * m + p);
    }
    for (; p < m; p += stride) {
        const double xh[3] = {(double)nx - k.c_ref[0], (double)ny - k.c_ref[1],
                              (double)nz - k.c_ref[2]};
        const long long pn = p + stride;
        if (pn < m) {
            nx = __ldg(ref + pn);
            ny = __ldg(ref + m + pn);
            nz = __ldg(ref + 2 * m + pn);
        }
        point_step<MODE, NV, SIG, FAST, NA>(k, tab, tabf, xh, p, m, wtn, acc);
    }
    block_reduce_store<NA>(acc, partials + (long long)blockIdx.x * NA);
}

// ---------------------------------------------------------------------------
// float32 point path of the point_to_point pass (FR_PASS_F32).  Centred world
// coordinates xt = R (x_ref - c_ref) are float32 (|xt| ~ cloud radius); the
// elevated coordinates are A xt + A c with the pose constant A c split into an
// exact multiple of 4 and a float32 fraction, so every rounding acts on
// O(cloud / sigma) lattice units; targets are formed relative to the centre.
// Moments are accumulated in float32 over 16 points per thread, then folded
// into float64 accumulators (relative error ~1e-6, far below what moves a
// halving decision or the pose).  Only float64 left per point:
// the fold every 16 points.
struct F32K {
    float R[9];
    float cref[3];
    float cw[3];
    float A[4][3];
    float f0[4];
    int base[4];
    float cp;
};

constexpr int kF32Fold = 16;

template <bool DEV>
__global__ void __launch_bounds__(kPassThreads, 2)
k_rigid_pass_f32(const float *__restrict__ ref, long long m, RigidK kv, const RigidK *kd,
                 const int *done, SliceTableF tabf, double *__restrict__ partials) {
    constexpr int NA = kP2PtBase;
    __shared__ F32K f;
    if (DEV && *done) return;
    if (threadIdx.x == 0) {
        const RigidK &k = DEV ? *kd : kv;
        for (int q = 0; q < 9; ++q) f.R[q] = (float)k.R[q];
        for (int q = 0; q < 3; ++q) {
            f.cref[q] = (float)k.c_ref[q];
            f.cw[q] = (float)k.c_world[q];
        }
        for (int i = 0; i < 4; ++i) {
            for (int j = 0; j < 3; ++j) f.A[i][j] = (float)k.A[i][j];
            const double e = k.e0[i];
            const double b = rint(e * 0.25);
            f.base[i] = (int)b;
            f.f0[i] = (float)(e - 4.0 * b);
        }
        f.cp = (float)k.cp;
    }
    // per-thread float64 accumulators live in shared memory (column per
    // thread, conflict-free); registers hold only the float32 partials
    extern __shared__ double sacc[];   // [NA][kPassThreads]
#pragma unroll
    for (int q = 0; q < NA; ++q) sacc[q * kPassThreads + threadIdx.x] = 0.0;
    __syncthreads();
    float a[NA];
#pragma unroll
    for (int q = 0; q < NA; ++q) a[q] = 0.0f;
    int fold = 0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    float nx = 0.f, ny = 0.f, nz = 0.f;
    if (p < m) {
        nx = __ldg(ref + p);
        ny = __ldg(ref + m + p);
        nz = __ldg(ref + 2 * m + p);
    }
    for (; p < m; p += stride) {
        const float xh[3] = {nx - f.cref[0], ny - f.cref[1], nz - f.cref[2]};
        const long long pn = p + stride;
        if (pn < m) {
            nx = __ldg(ref + pn);
            ny = __ldg(ref + m + pn);
            nz = __ldg(ref + 2 * m + pn);
        }
        float y[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
            y[i] = fmaf(f.R[3 * i + 2], xh[2], fmaf(f.R[3 * i + 1], xh[1], f.R[3 * i] * xh[0]));
        float el[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            el[i] = fmaf(f.A[i][2], y[2], fmaf(f.A[i][1], y[1], fmaf(f.A[i][0], y[0], f.f0[i])));
        float o[4] = {0.f, 0.f, 0.f, 0.f};
        QSimplex3 q;
        qsimplex3f(el, f.base, q);
        if (!q.overflow) {
            float4 v[4][1];
            gather_simplex_f<1>(tabf, q.key, v);
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const float b = q.bary[l];
                o[0] = fmaf(b, v[l][0].x, o[0]);
                o[1] = fmaf(b, v[l][0].y, o[1]);
                o[2] = fmaf(b, v[l][0].z, o[2]);
                o[3] = fmaf(b, v[l][0].w, o[3]);
            }
        }
        const float m0 = fmaxf(o[0], 0.0f);
        const bool sup = m0 >= 1e-12f;
        const float w = sup ? (f.cp > 0.0f ? m0 * rcp_approx(m0 + f.cp) : 1.0f) : 0.0f;
        const float inv = sup ? rcp_approx(m0) : 0.0f;
        // residual r = x - t in centred coordinates; unsupported: t = x, w = 0
        float r[3], wy[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            r[j] = sup ? y[j] - fmaf(o[1 + j], inv, -f.cw[j]) : 0.0f;
            wy[j] = w * y[j];
        }
        a[0] += w;
#pragma unroll
        for (int j = 0; j < 3; ++j) a[1 + j] += wy[j];
        a[4] = fmaf(wy[0], y[0], a[4]);
        a[5] = fmaf(wy[0], y[1], a[5]);
        a[6] = fmaf(wy[0], y[2], a[6]);
        a[7] = fmaf(wy[1], y[1], a[7]);
        a[8] = fmaf(wy[1], y[2], a[8]);
        a[9] = fmaf(wy[2], y[2], a[9]);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const float wr = w * r[j];
            a[10 + j] += wr;
#pragma unroll
            for (int c = 0; c < 3; ++c) a[13 + 3 * j + c] = fmaf(wr, y[c], a[13 + 3 * j + c]);
            a[22 + j] = fmaf(wr, r[j], a[22 + j]);
        }
        if (++fold == kF32Fold) {
#pragma unroll
            for (int c = 0; c < NA; ++c) {
                sacc[c * kPassThreads + threadIdx.x] += (double)a[c];
                a[c] = 0.0f;
            }
            fold = 0;
        }
    }
    double acc[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) acc[c] = sacc[c * kPassThreads + threadIdx.x] + (double)a[c];
    block_reduce_store<NA>(acc, partials + (long long)blockIdx.x * NA);
}

constexpr size_t kF32Smem = (size_t)kP2PtBase * kPassThreads * sizeof(double);

// ---------------------------------------------------------------------------
// dense-grid point path (FR_PASS_F32 when the lattice has a dense grid; the
// EM hot loop of SURVEY.md 8(a)).  Same float32 geometry as k_rigid_pass_f32,
// restructured for issue throughput (the kernel is instruction-bound, not
// HBM-bound, at 12 B per point):
//   * rounding by the 1.5 * 2^23 magic constant (FFMA + FADD, no XU ops);
//     the integer cell comes from the float's bits;
//   * no per-point rank wrap: the six pairwise comparison bits and h (the
//     sum of the rounded coordinates, |h| <= 2) index a 320-entry table of the
//     four vertex slot offsets with the wrap and the rotation of the
//     barycentrics by h folded in (the cyclic gaps of the sorted residuals
//     are wrap-invariant, permutohedral.py:198-212);
//   * barycentrics from a 5-comparator sorting network;
//   * float32 pairs (FFMA2) for the transform, the slice and the moments.
struct GridK {
    float2 Rc[3];           // (R0k, R1k): rows 0-1 of column k
    float2 R2[3];           // (R2k, 0)
    float2 cw01, cw2;       // (cw0, cw1), (cw2, 0)
    float cref[3];
    float cp;
    int s0, s1;             // cell strides of coordinates 0 and 1
    unsigned H;             // h = sum bits + H
    // quarter-scale embedding: el / 4 directly
    float2 Q01[3], Q23[3];  // (A0k, A1k) / 4, (A2k, A3k) / 4
    float2 q01, q23;        // (e0 - 4 base) / 4
    unsigned Cq[3];         // v = bits(t) + Cq = ri - (a - 2), clamped to limq
    unsigned limq[3];       // span + 4
    unsigned Kq;            // cell of ri = v0 * s0 + v1 * s1 + v2 + Kq
};

constexpr float kMagic = 12582912.0f;          // 1.5 * 2^23
constexpr int kMagicBits = 0x4B400000;
constexpr int kGridTab = 64 * 5;
// points per thread between warp folds of the float32 partials into the
// float64 accumulators: 64 measured 98.9 vs 100.8 us per pass (32) at 16.8M
// points, inside the parity tolerances of the float32 query path
constexpr int kGridFold = 64;

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// table entry e = code * 5 + (h + 2): pre-wrap ranks from the comparison bits
// (pair order (0,1) (0,2) (0,3) (1,2) (1,3) (2,3); bit set: d[j] > d[i]; the
// earlier index wins ties, as the stable argsort of permutohedral.py:193-197),
// the +-4 wrap (:198-203), vertex l's cell ri_final - [rank_final >= 4 - l]
// (:214), and pre-wrap barycentric k -> vertex (k - h) mod 4
__device__ __forceinline__ int4 grid_entry(int e, int s0, int s1) {
    const int code = e / 5, h = e % 5 - 2;
    int rank[4] = {0, 0, 0, 0};
    int p = 0;
    for (int i = 0; i < 4; ++i)
        for (int j = i + 1; j < 4; ++j, ++p) {
            if ((code >> p) & 1) ++rank[i];
            else ++rank[j];
        }
    int rf[4], dri[4];
    for (int i = 0; i < 4; ++i) {
        const int rk = rank[i] + h;
        const int adj = rk < 0 ? -1 : (rk > 3 ? 1 : 0);
        rf[i] = rk - 4 * adj;
        dri[i] = -adj;
    }
    const int st[3] = {s0, s1, 1};
    int off[4];
    for (int l = 0; l < 4; ++l) {
        int c = 0;
        for (int i = 0; i < 3; ++i) c += (dri[i] - (rf[i] >= 4 - l ? 1 : 0)) * st[i];
        off[l] = 4 * c + l;
    }
    int rot[4];
    for (int k = 0; k < 4; ++k) {
        const int l = (k - h + 8) & 3;
        rot[k] = l == 0 ? off[0] : (l == 1 ? off[1] : (l == 2 ? off[2] : off[3]));
    }
    return make_int4(rot[0], rot[1], rot[2], rot[3]);
}

// grid_entry for a comparison code whose six pair bits are stored reversed
// (pair (0,1) in bit 5), as grid_point_q forms it
__device__ __forceinline__ int4 grid_entry_q(int e, int s0, int s1) {
    const int code = e / 5, hi = e % 5;
    int rev = 0;
    for (int b = 0; b < 6; ++b) rev |= ((code >> b) & 1) << (5 - b);
    return grid_entry(rev * 5 + hi, s0, s1);
}

__device__ __forceinline__ float2 bc(float x) { return make_float2(x, x); }

// float32 pair accumulators -> the 25 float64 columns (layout of _rigid.py)
struct GridAcc {
    float2 s1_01, s1_2_s0, s2_00_01, s2_02_12, rx01[3], rx2_r1[3], q01;
    float s2_11, s2_22, q2;
    __device__ __forceinline__ void zero() {
        s1_01 = s1_2_s0 = s2_00_01 = s2_02_12 = q01 = make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 3; ++j) rx01[j] = rx2_r1[j] = make_float2(0.f, 0.f);
        s2_11 = s2_22 = q2 = 0.f;
    }
    __device__ __forceinline__ float col(int c) const {
        switch (c) {
            case 0: return s1_2_s0.y;
            case 1: return s1_01.x;
            case 2: return s1_01.y;
            case 3: return s1_2_s0.x;
            case 4: return s2_00_01.x;
            case 5: return s2_00_01.y;
            case 6: return s2_02_12.x;
            case 7: return s2_11;
            case 8: return s2_02_12.y;
            case 9: return s2_22;
            case 22: return q01.x;
            case 23: return q01.y;
            case 24: return q2;
            default: break;
        }
        if (c < 13) return rx2_r1[c - 10].y;
        const int j = (c - 13) / 3, k = (c - 13) % 3;
        return k == 0 ? rx01[j].x : (k == 1 ? rx01[j].y : rx2_r1[j].x);
    }
};

// float32 pass constants of pose k over the dense grid dg (one thread).  The
// embedding is pre-scaled by 1/4 (exact: t = el/4 + magic, d/4 and the
// barycentrics are bit-identical to the unscaled forms); the integer part of
// the float64 pose constant e0 is split off exactly, so every float32
// rounding acts on O(cloud / sigma) lattice units.
__device__ __forceinline__ void grid_params(const RigidK &k, const DenseSliceF &dg, GridK &g) {
    for (int c = 0; c < 3; ++c) {
        g.Rc[c] = make_float2((float)k.R[c], (float)k.R[3 + c]);
        g.R2[c] = make_float2((float)k.R[6 + c], 0.0f);
        g.Q01[c] = make_float2(0.25f * (float)k.A[0][c], 0.25f * (float)k.A[1][c]);
        g.Q23[c] = make_float2(0.25f * (float)k.A[2][c], 0.25f * (float)k.A[3][c]);
        g.cref[c] = (float)k.c_ref[c];
    }
    int base[4];
    float fr0[4];
    for (int i = 0; i < 4; ++i) {
        const double b = rint(k.e0[i] * 0.25);
        base[i] = (int)b;
        fr0[i] = (float)(k.e0[i] - 4.0 * b);
    }
    g.q01 = make_float2(0.25f * fr0[0], 0.25f * fr0[1]);
    g.q23 = make_float2(0.25f * fr0[2], 0.25f * fr0[3]);
    g.cw01 = make_float2((float)k.c_world[0], (float)k.c_world[1]);
    g.cw2 = make_float2((float)k.c_world[2], 0.0f);
    g.cp = (float)k.cp;
    unsigned H = 0;
    for (int i = 0; i < 4; ++i) H += (unsigned)(base[i] - kMagicBits);
    for (int c = 0; c < 3; ++c) {
        g.Cq[c] = (unsigned)(base[c] - kMagicBits - (dg.a[c] - 2));
        g.limq[c] = dg.span[c] + 4u;
    }
    g.s0 = dg.s0;
    g.s1 = dg.s1;
    g.H = H;
    g.Kq = (unsigned)(kDensePad - 2) * (unsigned)(dg.s0 + dg.s1 + 1);
}

// base + 16 i as one IMAD.WIDE (keeps ptxas from re-associating the cell and
// vertex offsets into a 32-bit add plus a sign-extending 64-bit add per gather)
__device__ __forceinline__ const float4 *wide_ptr16(const float4 *base, unsigned i) {
    const float4 *r;
    asm("mad.wide.u32 %0, %1, 16, %2;" : "=l"(r) : "r"(i), "l"(base));
    return r;
}
__device__ __forceinline__ const float4 *wide_ptr16s(const float4 *base, int i) {
    const float4 *r;
    asm("mad.wide.s32 %0, %1, 16, %2;" : "=l"(r) : "r"(i), "l"(base));
    return r;
}

// one model point of the quarter-scale dense-grid pass: as grid_point, with
// the embedding pre-scaled by 1/4 (t = el/4 + magic, d/4 = el/4 - round(el/4),
// barycentrics = gaps of the sorted d/4 -- bit-identical, three multiplies
// fewer), the remainder-0 cell clamped into the zero-padded box instead of a
// range branch (an outside point reads padding rows: no mass, as the
// reference's absent sites), and the four gathers addressed from one cell
// pointer
template <bool CENTRED = false>
__device__ __forceinline__ void grid_point_q(float nx, float ny, float nz, bool valid,
                                             const GridK &g, const int4 *tab,
                                             const float4 *__restrict__ cells, GridAcc &a) {
    // CENTRED: the caller's coordinates are already x - (float)c_ref
    const float x0 = CENTRED ? nx : nx - g.cref[0];
    const float x1 = CENTRED ? ny : ny - g.cref[1];
    const float x2 = CENTRED ? nz : nz - g.cref[2];
    float2 y01 = __fmul2_rn(g.Rc[0], bc(x0));
    y01 = __ffma2_rn(g.Rc[1], bc(x1), y01);
    y01 = __ffma2_rn(g.Rc[2], bc(x2), y01);
    float2 y2v = __ffma2_rn(g.R2[0], bc(x0), make_float2(0.0f, 1.0f));
    y2v = __ffma2_rn(g.R2[1], bc(x1), y2v);
    y2v = __ffma2_rn(g.R2[2], bc(x2), y2v);
    float2 e01 = __ffma2_rn(g.Q01[0], bc(y01.x), g.q01);
    e01 = __ffma2_rn(g.Q01[1], bc(y01.y), e01);
    e01 = __ffma2_rn(g.Q01[2], bc(y2v.x), e01);
    float2 e23 = __ffma2_rn(g.Q23[0], bc(y01.x), g.q23);
    e23 = __ffma2_rn(g.Q23[1], bc(y01.y), e23);
    e23 = __ffma2_rn(g.Q23[2], bc(y2v.x), e23);
    const float2 t01 = __fadd2_rn(e01, bc(kMagic)), t23 = __fadd2_rn(e23, bc(kMagic));
    // round(el / 4) = t - magic exactly; d / 4 = el / 4 - round(el / 4) exactly
    const float2 d01 = __ffma2_rn(__fadd2_rn(t01, bc(-kMagic)), bc(-1.0f), e01);
    const float2 d23 = __ffma2_rn(__fadd2_rn(t23, bc(-kMagic)), bc(-1.0f), e23);
    const float d[4] = {d01.x, d01.y, d23.x, d23.y};
    const int tb[4] = {__float_as_int(t01.x), __float_as_int(t01.y), __float_as_int(t23.x),
                       __float_as_int(t23.y)};
    // comparison code: the sign bit of d[i] - d[j] (set iff d[j] > d[i]; a
    // tie gives +0, unset) shifted in by one funnel shift per pair, pair
    // (0,1) ending in bit 5 (grid_entry_q reverses the bit order)
    const float2 dd = __fadd2_rn(d01, make_float2(-d23.x, -d23.y));   // (d0 - d2, d1 - d3)
    const float df[6] = {d[0] - d[1], dd.x, d[0] - d[3], d[1] - d[2], dd.y, d[2] - d[3]};
    unsigned code = __float_as_uint(df[0]) >> 31;
#pragma unroll
    for (int q = 1; q < 6; ++q) code = __funnelshift_l(__float_as_uint(df[q]), code, 1);
    float s0 = fmaxf(d[0], d[1]), s1 = fminf(d[0], d[1]);
    float s2 = fmaxf(d[2], d[3]), s3 = fminf(d[2], d[3]);
    {
        const float hi = fmaxf(s0, s2), lo = fminf(s0, s2);
        s0 = hi;
        s2 = lo;
        const float hi2 = fmaxf(s1, s3), lo2 = fminf(s1, s3);
        s1 = hi2;
        s3 = lo2;
        const float hi3 = fmaxf(s1, s2), lo3 = fminf(s1, s2);
        s1 = hi3;
        s2 = lo3;
    }
    const float b0 = 1.0f + (s3 - s0);
    const float b1 = s2 - s3, b2 = s1 - s2, b3 = s0 - s1;
    const int h = (int)((unsigned)tb[0] + (unsigned)tb[1] + (unsigned)tb[2] + (unsigned)tb[3] + g.H);
    const int hi = min(max(h + 2, 0), 4);
    const int4 T = tab[code * 5 + hi];
    const unsigned v0 = min((unsigned)tb[0] + g.Cq[0], g.limq[0]);
    const unsigned v1 = min((unsigned)tb[1] + g.Cq[1], g.limq[1]);
    const unsigned v2 = min((unsigned)tb[2] + g.Cq[2], g.limq[2]);
    const float4 *cb = wide_ptr16(cells, 4u * (v0 * (unsigned)g.s0 + v1 * (unsigned)g.s1 + v2 + g.Kq));
    const float4 q0 = __ldg(wide_ptr16s(cb, T.x)), q1 = __ldg(wide_ptr16s(cb, T.y));
    const float4 q2 = __ldg(wide_ptr16s(cb, T.z)), q3 = __ldg(wide_ptr16s(cb, T.w));
    float2 o01 = __fmul2_rn(bc(b0), make_float2(q0.x, q0.y));
    float2 o23 = __fmul2_rn(bc(b0), make_float2(q0.z, q0.w));
    o01 = __ffma2_rn(bc(b1), make_float2(q1.x, q1.y), o01);
    o23 = __ffma2_rn(bc(b1), make_float2(q1.z, q1.w), o23);
    o01 = __ffma2_rn(bc(b2), make_float2(q2.x, q2.y), o01);
    o23 = __ffma2_rn(bc(b2), make_float2(q2.z, q2.w), o23);
    o01 = __ffma2_rn(bc(b3), make_float2(q3.x, q3.y), o01);
    o23 = __ffma2_rn(bc(b3), make_float2(q3.z, q3.w), o23);
    const float m0 = fmaxf(o23.y, 0.0f);
    const bool sup = m0 >= 1e-12f;
    // branch-free: both reciprocals unconditionally, then selects (the
    // c' > 0 test is block-uniform)
    const float wc = g.cp > 0.0f ? m0 * rcp_approx(m0 + g.cp) : 1.0f;
    const float w = (sup && valid) ? wc : 0.0f;
    const float rm = rcp_approx(m0);
    const float ninv = sup ? -rm : 0.0f;
    const float2 r01 = __fadd2_rn(y01, __ffma2_rn(o01, bc(ninv), g.cw01));
    const float r2 = y2v.x + fmaf(o23.x, ninv, g.cw2.x);
    const float2 wy01 = __fmul2_rn(bc(w), y01);
    const float2 wy2v = __fmul2_rn(bc(w), y2v);
    const float2 wr01 = __fmul2_rn(bc(w), r01);
    const float wr2 = w * r2;
    a.s1_01 = __fadd2_rn(a.s1_01, wy01);
    a.s1_2_s0 = __fadd2_rn(a.s1_2_s0, wy2v);
    a.s2_00_01 = __ffma2_rn(bc(wy01.x), y01, a.s2_00_01);
    a.s2_02_12 = __ffma2_rn(bc(y2v.x), wy01, a.s2_02_12);
    a.s2_11 = fmaf(wy01.y, y01.y, a.s2_11);
    a.s2_22 = fmaf(wy2v.x, y2v.x, a.s2_22);
    a.rx01[0] = __ffma2_rn(bc(wr01.x), y01, a.rx01[0]);
    a.rx2_r1[0] = __ffma2_rn(bc(wr01.x), y2v, a.rx2_r1[0]);
    a.rx01[1] = __ffma2_rn(bc(wr01.y), y01, a.rx01[1]);
    a.rx2_r1[1] = __ffma2_rn(bc(wr01.y), y2v, a.rx2_r1[1]);
    a.rx01[2] = __ffma2_rn(bc(wr2), y01, a.rx01[2]);
    a.rx2_r1[2] = __ffma2_rn(bc(wr2), y2v, a.rx2_r1[2]);
    a.q01 = __ffma2_rn(wr01, r01, a.q01);
    a.q2 = fmaf(wr2, r2, a.q2);
}

// the warp's float32 partials folded into its float64 accumulators: a
// butterfly reduce-scatter (5 shuffle rounds, 31 adds per lane) leaves lane c
// holding the warp sum of statistic c, which it adds into wacc[c].  Fixed
// order, hence deterministic; shared memory is 25 doubles per warp instead of
// per thread, so it no longer caps the CTAs per SM.
__device__ __forceinline__ void grid_warp_fold(const GridAcc &a, double *wacc) {
    const int lane = threadIdx.x & 31;
    float v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) v[c] = c < kP2PtBase ? a.col(c) : 0.0f;
#pragma unroll
    for (int n = 32, off = 16; off >= 1; n >>= 1, off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const float send = upper ? v[i] : v[i + n / 2];
            const float keep = upper ? v[i + n / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    if (lane < kP2PtBase) wacc[lane] += (double)v[0];
}

// streaming 16-byte load that leaves L1 to the grid gathers
__device__ __forceinline__ float4 ld_stream4(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

// the four consecutive points j .. j + 3 of a chunk (zero past cnt); VEC: the
// three planes are 16-byte aligned (m % 4 == 0, chunk starts at multiples of 4)
template <bool VEC>
__device__ __forceinline__ void load_quad(const float *p0, const float *p1, const float *p2,
                                          int j, int cnt, float4 &x, float4 &y, float4 &z) {
    if (VEC && j + 3 < cnt) {
        x = ld_stream4(p0 + j);
        y = ld_stream4(p1 + j);
        z = ld_stream4(p2 + j);
        return;
    }
    float t[3][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const bool ok = j + k < cnt;
        t[0][k] = ok ? __ldcs(p0 + j + k) : 0.0f;
        t[1][k] = ok ? __ldcs(p1 + j + k) : 0.0f;
        t[2][k] = ok ? __ldcs(p2 + j + k) : 0.0f;
    }
    x = make_float4(t[0][0], t[0][1], t[0][2], t[0][3]);
    y = make_float4(t[1][0], t[1][1], t[1][2], t[1][3]);
    z = make_float4(t[2][0], t[2][1], t[2][2], t[2][3]);
}

// dense-grid pass, four consecutive points per thread per trip: 16-byte
// streaming loads of each plane (one trip ahead in registers, no shared-memory
// staging), the quarter-scale clamped point (grid_point_q), warp fold every
// kGridFold points per thread.  Per-block contiguous chunks (multiples of
// 1024 points) keep a block's gathers in a compact grid region (Morton order).
constexpr int kQuadPts = 4 * kPassThreads;
// pass constants of the device loop in the constant bank (CONSTP): operands
// straight from the bank, no registers held for them (written by a
// device-to-device copy node after k_grid_params each iteration)
__constant__ GridK c_grid;

__global__ void k_grid_params(const RigidK *kd, const int *done, DenseSliceF dg, GridK *out) {
    if (*done) return;
    grid_params(*kd, dg, *out);
}

// RING: the point stream staged through a kRing4-deep shared-memory ring by
// 16-byte cp.async (L1-bypassing) instead of the register double buffer
constexpr int kRing4 = 3;
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void ring_issue_quad(float4 (*slot)[kPassThreads], const float *p0,
                                                const float *p1, const float *p2, int j, int cnt) {
    if (j + 3 < cnt) {
        cp_async16(&slot[0][threadIdx.x], p0 + j);
        cp_async16(&slot[1][threadIdx.x], p1 + j);
        cp_async16(&slot[2][threadIdx.x], p2 + j);
    } else if (j < cnt) {
        float4 x, y, z;
        load_quad<false>(p0, p1, p2, j, cnt, x, y, z);
        slot[0][threadIdx.x] = x;
        slot[1][threadIdx.x] = y;
        slot[2][threadIdx.x] = z;
    }
    cp_async_commit();
}

template <bool DEV, bool VEC, int MINB, bool CONSTP, bool RING = false, int FOLD = kGridFold>
__global__ void __launch_bounds__(kPassThreads, MINB)
k_rigid_pass_grid4(const float *__restrict__ ref, long long m, RigidK kv, const RigidK *kd,
                   const int *done, DenseSliceF dg, double *__restrict__ partials) {
    constexpr int NA = kP2PtBase;
    __shared__ float4 ring[RING ? kRing4 : 1][3][kPassThreads];
    __shared__ GridK gs;
    __shared__ int4 tab[kGridTab];
    __shared__ double wacc[kPassThreads / 32][NA];
    if (DEV && *done) return;
    const GridK &g = CONSTP ? c_grid : gs;
    if (!CONSTP && threadIdx.x == 0) grid_params(DEV ? *kd : kv, dg, gs);
    for (int e = threadIdx.x; e < kGridTab; e += blockDim.x) tab[e] = grid_entry_q(e, dg.s0, dg.s1);
    if ((threadIdx.x & 31) < NA) wacc[threadIdx.x >> 5][threadIdx.x & 31] = 0.0;
    __syncthreads();
    double *my_wacc = wacc[threadIdx.x >> 5];
    GridAcc a;
    a.zero();
    const long long chunk = ((m + gridDim.x - 1) / gridDim.x + kQuadPts - 1) / kQuadPts * kQuadPts;
    const long long beg = (long long)blockIdx.x * chunk;
    const int cnt = (int)max(0ll, min(beg + chunk, m) - beg);
    const float *p0 = ref + min(beg, m), *p1 = p0 + m, *p2 = p1 + m;
    const int me = 4 * (int)threadIdx.x;
    int fold = 0;
    // a trip is full (every point valid) except possibly the block's last
    auto quad_t = [&](auto full, int j, const float4 &cx, const float4 &cy, const float4 &cz) {
        constexpr bool F = decltype(full)::value;
        const int q = j + me;
        grid_point_q(cx.x, cy.x, cz.x, F || q < cnt, g, tab, dg.cells, a);
        grid_point_q(cx.y, cy.y, cz.y, F || q + 1 < cnt, g, tab, dg.cells, a);
        grid_point_q(cx.z, cy.z, cz.z, F || q + 2 < cnt, g, tab, dg.cells, a);
        grid_point_q(cx.w, cy.w, cz.w, F || q + 3 < cnt, g, tab, dg.cells, a);
        fold += 4;
        if (fold >= FOLD) {       // warp-uniform trips
            grid_warp_fold(a, my_wacc);
            a.zero();
            fold = 0;
        }
    };
    auto quad = [&](int j, const float4 &cx, const float4 &cy, const float4 &cz) {
        if (j + kQuadPts <= cnt) quad_t(std::true_type{}, j, cx, cy, cz);
        else quad_t(std::false_type{}, j, cx, cy, cz);
    };
    if (RING) {
        // each thread reads back only the slots it filled: no block barrier
#pragma unroll
        for (int st = 0; st < kRing4 - 1; ++st)
            ring_issue_quad(ring[st], p0, p1, p2, st * kQuadPts + me, cnt);
        int stage = 0;
        for (int j = 0; j < cnt; j += kQuadPts) {
            ring_issue_quad(ring[stage == 0 ? kRing4 - 1 : stage - 1], p0, p1, p2,
                            j + (kRing4 - 1) * kQuadPts + me, cnt);
            cp_async_wait<kRing4 - 1>();
            const float4 cx = ring[stage][0][threadIdx.x], cy = ring[stage][1][threadIdx.x],
                         cz = ring[stage][2][threadIdx.x];
            stage = stage + 1 == kRing4 ? 0 : stage + 1;
            quad(j, cx, cy, cz);
        }
    } else {
        // two register buffers alternate (trip t computes one while the
        // other receives trip t + 1): no buffer moves
        float4 ax, ay, az, bx, by, bz;
        load_quad<VEC>(p0, p1, p2, me, cnt, ax, ay, az);
        for (int j = 0; j < cnt; j += 2 * kQuadPts) {
            if (j + kQuadPts < cnt) load_quad<VEC>(p0, p1, p2, j + kQuadPts + me, cnt, bx, by, bz);
            quad(j, ax, ay, az);
            if (j + kQuadPts >= cnt) break;
            if (j + 2 * kQuadPts < cnt) load_quad<VEC>(p0, p1, p2, j + 2 * kQuadPts + me, cnt, ax, ay, az);
            quad(j + kQuadPts, bx, by, bz);
        }
    }
    grid_warp_fold(a, my_wacc);
    __syncthreads();
    if (threadIdx.x < NA) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < kPassThreads / 32; ++w) v += wacc[w][threadIdx.x];
        partials[(long long)blockIdx.x * NA + threadIdx.x] = v;
    }
}

// ---------------------------------------------------------------------------
// tiled dense-grid pass of the device loop: the EM object's model points,
// centred once (x - (float)c_ref: the same float32 subtraction the point
// kernels make per pass) and laid out as tiles of 1024 points, each tile
// [3][256] float4 (thread t's four consecutive points per plane).  One tile is
// one trip of the block: three 16-byte cp.async at immediate offsets from a
// pointer that advances 12 KB per trip (no per-trip 64-bit plane arithmetic),
// no centring adds in the point chain.
constexpr int kTileF4 = 3 * kPassThreads;   // float4 per tile

__global__ void k_tile_points(const float *__restrict__ ref, long long m, float c0, float c1,
                              float c2, float4 *__restrict__ tiles, long long ntiles) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;   // quad index
    if (i >= ntiles * kPassThreads) return;
    const long long t = i / kPassThreads, lane = i % kPassThreads, p = 4 * i;
    const float c[3] = {c0, c1, c2};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = p + k < m ? ref[d * m + p + k] - c[d] : 0.0f;
        tiles[t * kTileF4 + d * kPassThreads + lane] = make_float4(v[0], v[1], v[2], v[3]);
    }
}

// the tiled pass's fused tail: the last block to finish reduces the block
// partials (the fixed order of k_reduce_cols) into sums and, with SOLVE, runs
// the iteration's float64 solve and writes the next pose's pass constants --
// one kernel per EM iteration instead of pass + reduction + solver
struct EmDev;
struct TailArgs {
    unsigned *counter;      // zero between launches (the last block resets it)
    double *sums;
    EmDev *em;              // SOLVE only
    double *objs, *tnorms, *masses;
    GridK *gk_out;          // next iteration's pass constants (SOLVE only)
};
template <bool SOLVE>
__device__ void pass_tail(const double *partials, DenseSliceF dg, const TailArgs &ta);

template <int FOLD = kGridFold, int MINB = 2, bool SOLVE = false>
__global__ void __launch_bounds__(kPassThreads, MINB)
k_rigid_pass_tiles(const float4 *__restrict__ tiles, long long m, const int *done, DenseSliceF dg,
                   double *__restrict__ partials, TailArgs ta) {
    constexpr int NA = kP2PtBase;
    __shared__ float4 ring[kRing4][3][kPassThreads];
    __shared__ int4 tab[kGridTab];
    __shared__ double wacc[kPassThreads / 32][NA];
    if (*done) return;
    const GridK &g = c_grid;
    const long long ntiles = (m + kQuadPts - 1) / kQuadPts;
    const long long tpb = (ntiles + gridDim.x - 1) / gridDim.x;
    const long long t0 = (long long)blockIdx.x * tpb;
    const int nt = (int)max(0ll, min(t0 + tpb, ntiles) - t0);
    // points of this block's tiles that exist: the last tile of the cloud may
    // be partial (its padding is zeros, which are real coordinates: masked)
    const long long first = t0 * kQuadPts;
    const int cnt = (int)max(0ll, min((long long)nt * kQuadPts, m - first));
    const float4 *src = tiles + t0 * kTileF4 + threadIdx.x;
    // the first tiles' copies go out before the table is built (their DRAM
    // latency overlaps it); each thread later reads only its own slots
#pragma unroll
    for (int st = 0; st < kRing4 - 1; ++st) {
        if (st < nt) {
            cp_async16(&ring[st][0][threadIdx.x], src + st * kTileF4);
            cp_async16(&ring[st][1][threadIdx.x], src + st * kTileF4 + kPassThreads);
            cp_async16(&ring[st][2][threadIdx.x], src + st * kTileF4 + 2 * kPassThreads);
        }
        cp_async_commit();
    }
    for (int e = threadIdx.x; e < kGridTab; e += blockDim.x) tab[e] = grid_entry_q(e, dg.s0, dg.s1);
    if ((threadIdx.x & 31) < NA) wacc[threadIdx.x >> 5][threadIdx.x & 31] = 0.0;
    __syncthreads();
    double *my_wacc = wacc[threadIdx.x >> 5];
    GridAcc a;
    a.zero();
    const int me = 4 * (int)threadIdx.x;
    int fold = 0;
    auto quad_t = [&](auto full, int j, const float4 &cx, const float4 &cy, const float4 &cz) {
        constexpr bool F = decltype(full)::value;
        const int q = j + me;
        grid_point_q<true>(cx.x, cy.x, cz.x, F || q < cnt, g, tab, dg.cells, a);
        grid_point_q<true>(cx.y, cy.y, cz.y, F || q + 1 < cnt, g, tab, dg.cells, a);
        grid_point_q<true>(cx.z, cy.z, cz.z, F || q + 2 < cnt, g, tab, dg.cells, a);
        grid_point_q<true>(cx.w, cy.w, cz.w, F || q + 3 < cnt, g, tab, dg.cells, a);
        fold += 4;
        if (fold >= FOLD) {       // warp-uniform trips
            grid_warp_fold(a, my_wacc);
            a.zero();
            fold = 0;
        }
    };
    const float4 *nxt = src + (kRing4 - 1) * kTileF4;
    int stage = 0;
    for (int t = 0; t < nt; ++t) {
        const int ws = stage == 0 ? kRing4 - 1 : stage - 1;
        if (t + kRing4 - 1 < nt) {
            cp_async16(&ring[ws][0][threadIdx.x], nxt);
            cp_async16(&ring[ws][1][threadIdx.x], nxt + kPassThreads);
            cp_async16(&ring[ws][2][threadIdx.x], nxt + 2 * kPassThreads);
        }
        cp_async_commit();
        nxt += kTileF4;
        cp_async_wait<kRing4 - 1>();
        const float4 cx = ring[stage][0][threadIdx.x], cy = ring[stage][1][threadIdx.x],
                     cz = ring[stage][2][threadIdx.x];
        stage = stage + 1 == kRing4 ? 0 : stage + 1;
        const int j = t * kQuadPts;
        if (j + kQuadPts <= cnt) quad_t(std::true_type{}, j, cx, cy, cz);
        else quad_t(std::false_type{}, j, cx, cy, cz);
    }
    grid_warp_fold(a, my_wacc);
    __syncthreads();
    if (threadIdx.x < NA) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < kPassThreads / 32; ++w) v += wacc[w][threadIdx.x];
        partials[(long long)blockIdx.x * NA + threadIdx.x] = v;
    }
    pass_tail<SOLVE>(partials, dg, ta);
}

// owner flag of c_grid: the first device EM object over a dense grid takes it
static std::atomic<bool> g_const_grid_busy{false};
// largest model cloud fr_rigid_em_run sends through the persistent one-CTA
// loop (FR_PERSIST_MAX points; larger clouds use the graph-replayed iteration)
static long long persist_max() {
    const char *e = getenv("FR_PERSIST_MAX");
    return e ? atoll(e) : 32768;
}

static int set_f32_smem() {
    static bool done = false;
    if (!done) {
        FR_CUDA(cudaFuncSetAttribute(k_rigid_pass_f32<true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF32Smem));
        FR_CUDA(cudaFuncSetAttribute(k_rigid_pass_f32<false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF32Smem));
        done = true;
    }
    return FR_OK;
}

// articulated pass (mstep.py:179-202, 213-229): model points sorted by body,
// block b sweeps chunk b (one body) with that body's pose; partials per chunk
template <int MODE, int NV, bool SIG, bool FAST>
__global__ void __launch_bounds__(kPassThreads, MODE == FR_POINT_TO_POINT ? 2 : 1)
k_body_pass(const float *__restrict__ ref, long long m, const RigidK *__restrict__ bodies,
            const int *__restrict__ chunk_body, const long long *__restrict__ chunk_beg,
            SliceTable tab, SliceTableF tabf, float *__restrict__ wtn,
            double *__restrict__ partials, const int *done = nullptr) {
    constexpr int NA = (MODE == FR_POINT_TO_POINT ? kP2PtBase : kP2PlBase) + (SIG ? 2 : 0);
    __shared__ RigidK k;
    if (done && *done) return;      // device-resident articulated loop finished
    const long long beg = chunk_beg[blockIdx.x], end = chunk_beg[blockIdx.x + 1];
    if (threadIdx.x == 0) k = bodies[chunk_body[blockIdx.x]];
    __syncthreads();
    double acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0.0;
    for (long long p = beg + threadIdx.x; p < end; p += blockDim.x) {
        const double xh[3] = {(double)__ldg(ref + p) - k.c_ref[0],
                              (double)__ldg(ref + m + p) - k.c_ref[1],
                              (double)__ldg(ref + 2 * m + p) - k.c_ref[2]};
        point_step<MODE, NV, SIG, FAST, NA>(k, tab, tabf, xh, p, m, wtn, acc);
    }
    block_reduce_store<NA>(acc, partials + (long long)blockIdx.x * NA);
}

// per-segment column sums: segment s = chunks [seg[s], seg[s+1]), fixed order
__global__ void k_reduce_segments(const double *partials, const int *seg, int na, double *out,
                                  const int *done = nullptr) {
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31, s = blockIdx.x;
    if (c >= na || (done && *done)) return;
    double v = 0.0;
    for (int b = seg[s] + lane; b < seg[s + 1]; b += 32) v += partials[(long long)b * na + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) out[(long long)s * na + c] = v;
}

// candidate objectives for point_to_plane halving
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

// point_to_plane halving candidates for articulated trees: candidate c moves
// body b with cand[c * n_bodies + b] (R, c_world); one objective per candidate
__global__ void __launch_bounds__(kPassThreads, 2)
k_body_objective(const float *__restrict__ ref, const float *__restrict__ wtn, long long m,
                 const RigidK *__restrict__ cand, int n_bodies, int ncand,
                 const int *__restrict__ chunk_body, const long long *__restrict__ chunk_beg,
                 double *__restrict__ partials) {
    double acc[kMaxCand];
#pragma unroll
    for (int a = 0; a < kMaxCand; ++a) acc[a] = 0.0;
    const int body = chunk_body[blockIdx.x];
    const long long beg = chunk_beg[blockIdx.x], end = chunk_beg[blockIdx.x + 1];
    for (long long p = beg + threadIdx.x; p < end; p += blockDim.x) {
        const double w = (double)__ldg(wtn + p);
        if (!(w > 0.0)) continue;
        const double t[3] = {(double)__ldg(wtn + m + p), (double)__ldg(wtn + 2 * m + p),
                             (double)__ldg(wtn + 3 * m + p)};
        const double n[3] = {(double)__ldg(wtn + 4 * m + p), (double)__ldg(wtn + 5 * m + p),
                             (double)__ldg(wtn + 6 * m + p)};
        const float px = __ldg(ref + p), py = __ldg(ref + m + p), pz = __ldg(ref + 2 * m + p);
#pragma unroll
        for (int c = 0; c < kMaxCand; ++c) {
            if (c >= ncand) break;
            const RigidK &k = cand[c * n_bodies + body];
            const double xh[3] = {(double)px - k.c_ref[0], (double)py - k.c_ref[1],
                                  (double)pz - k.c_ref[2]};
            double x[3];
#pragma unroll
            for (int i = 0; i < 3; ++i)
                x[i] = fma(k.R[3 * i + 2], xh[2], fma(k.R[3 * i + 1], xh[1], k.R[3 * i] * xh[0])) +
                       k.c_world[i];
            acc[c] += pt2pl_cost(w, t, n, x);
        }
    }
    block_reduce_store<kMaxCand>(acc, partials + (long long)blockIdx.x * kMaxCand);
}

// ---------------------------------------------------------------------------
// device-resident M step (point_to_point)


// EmDev staged through shared memory: the serial float64 solve touches the
// state hundreds of times, so it works on an on-chip copy
__device__ __forceinline__ void em_copy(EmDev *dst, const EmDev *src, int lane, int nlanes) {
    static_assert(sizeof(EmDev) % 8 == 0, "EmDev is copied as 8-byte words");
    const unsigned long long *a = reinterpret_cast<const unsigned long long *>(src);
    unsigned long long *b = reinterpret_cast<unsigned long long *>(dst);
    for (int w = lane; w < (int)(sizeof(EmDev) / 8); w += nlanes) b[w] = a[w];
}

__global__ void k_rigid_solve(const double *sums, EmDev *e, double *objs, double *tnorms,
                              double *masses, DenseSliceF dg = DenseSliceF{},
                              GridK *gk_out = nullptr) {
    __shared__ EmDev se;
    if (e->done) return;
    em_copy(&se, e, threadIdx.x, blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) {
        rigid_solve_body(sums, &se, objs, tnorms, masses);
        if (gk_out && !se.done) grid_params(se.k, dg, *gk_out);
    }
    __syncthreads();
    em_copy(e, &se, threadIdx.x, blockDim.x);
}

template <bool SOLVE>
__device__ void pass_tail(const double *partials, DenseSliceF dg, const TailArgs &ta) {
    constexpr int NA = kP2PtBase;
    __shared__ bool last;
    __shared__ double tsum[NA];
    __threadfence();            // this block's partials before its arrival
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ta.counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    // thread (c, k) of kSeg per column sums rows k, k + kSeg, ... with its
    // loads issued together (a latency chain of a few L2 trips, not one per
    // row), then the kSeg segment sums in order: fixed order, deterministic
    constexpr int kSeg = 10, kRows = 32;
    __shared__ double seg[NA][kSeg];
    const int nb = (int)gridDim.x;
    if (threadIdx.x < NA * kSeg) {
        const int c = threadIdx.x / kSeg, k = threadIdx.x % kSeg;
        double r[kRows];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const int b = k + i * kSeg;
            r[i] = b < nb ? __ldcg(partials + (long long)b * NA + c) : 0.0;
        }
        double v = 0.0;
        for (int b = k + kRows * kSeg; b < nb; b += kSeg) v += __ldcg(partials + (long long)b * NA + c);
#pragma unroll
        for (int i = 0; i < kRows; ++i) v += r[i];
        seg[c][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < NA) {
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < kSeg; ++k) v += seg[threadIdx.x][k];
        tsum[threadIdx.x] = v;
        ta.sums[threadIdx.x] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) *ta.counter = 0u;
    if (SOLVE) {
        __shared__ EmDev se;
        em_copy(&se, ta.em, threadIdx.x, blockDim.x);
        __syncthreads();
        if (threadIdx.x == 0) {
            rigid_solve_body(tsum, &se, ta.objs, ta.tnorms, ta.masses);
            if (!se.done) grid_params(se.k, dg, *ta.gk_out);
        }
        __syncthreads();
        em_copy(ta.em, &se, threadIdx.x, blockDim.x);
    }
}

// ---------------------------------------------------------------------------
// persistent EM for small problems: one CTA runs a whole registration -- the
// dense-grid pass over its points, the warp folds and a fixed-order block
// reduction, the float64 solve (thread 0) and the next pose's pass constants
// -- with no kernel launches or host polls between iterations.  A launch with
// P CTAs runs P independent problems (the batched driver, SURVEY.md 8(f)
// rank 4).  The per-CTA reduction order is fixed, so a problem's result does
// not depend on what else shares the launch.
struct PersistProblem {
    const float *ref;       // SoA planes of m points (Morton order)
    long long m;
    EmDev *em;
    double *sums;           // last iteration's 25 sums (fr_rigid_em_sums)
    double *objs, *tnorms, *masses;
    DenseSliceF dg;
};

constexpr int kPersistThreads = 256;

__global__ void __launch_bounds__(kPersistThreads, 1)
k_em_persistent(const PersistProblem *probs) {
    constexpr int NA = kP2PtBase;
    const PersistProblem P = probs[blockIdx.x];
    __shared__ EmDev se;
    __shared__ GridK g;
    __shared__ int4 tab[kGridTab];
    __shared__ double wacc[kPersistThreads / 32][NA];
    __shared__ double tsum[NA];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    em_copy(&se, P.em, threadIdx.x, blockDim.x);
    for (int e = threadIdx.x; e < kGridTab; e += blockDim.x) tab[e] = grid_entry_q(e, P.dg.s0, P.dg.s1);
    __syncthreads();
    if (threadIdx.x == 0 && !se.done) grid_params(se.k, P.dg, g);
    __syncthreads();
    while (!se.done) {                  // block-uniform: read after a barrier
        if (lane < NA) wacc[warp][lane] = 0.0;
        GridAcc a;
        a.zero();
        int fold = 0;
        // three independent points per thread per trip (warp-uniform trips)
        constexpr int PP = 3;
        for (long long base = 0; base < P.m; base += PP * kPersistThreads) {
            float x[PP], y[PP], z[PP];
            bool ok[PP];
#pragma unroll
            for (int k = 0; k < PP; ++k) {
                const long long p = base + k * kPersistThreads + threadIdx.x;
                ok[k] = p < P.m;
                x[k] = ok[k] ? __ldg(P.ref + p) : 0.0f;
                y[k] = ok[k] ? __ldg(P.ref + P.m + p) : 0.0f;
                z[k] = ok[k] ? __ldg(P.ref + 2 * P.m + p) : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < PP; ++k) grid_point_q(x[k], y[k], z[k], ok[k], g, tab, P.dg.cells, a);
            fold += PP;
            if (fold >= kGridFold) {
                grid_warp_fold(a, wacc[warp]);
                a.zero();
                fold = 0;
            }
        }
        grid_warp_fold(a, wacc[warp]);
        __syncthreads();
        if (threadIdx.x < NA) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < kPersistThreads / 32; ++w) v += wacc[w][threadIdx.x];
            tsum[threadIdx.x] = v;
            P.sums[threadIdx.x] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            rigid_solve_body(tsum, &se, P.objs, P.tnorms, P.masses);
            if (!se.done) grid_params(se.k, P.dg, g);
        }
        __syncthreads();
    }
    em_copy(P.em, &se, threadIdx.x, blockDim.x);
}

// ---------------------------------------------------------------------------
// cluster-cooperative EM for small problems: a thread-block cluster of
// kEmCluster CTAs (one per SM) runs one registration's whole EM loop.  Each
// CTA sweeps 1/kEmCluster of the points; the leader (rank 0) sums the CTAs'
// 25 partial sums over distributed shared memory in rank order, runs the
// float64 solve and publishes the next pass constants and the done flag in
// its shared memory, which the other CTAs read over DSMEM after the cluster
// barrier.  Two cluster barriers per iteration, no global memory round trip
// and no kernel launch between iterations.  A launch with P clusters runs P
// problems; the reduction order is fixed (warps, then ranks), so a problem's
// result does not depend on what else shares the launch.
constexpr int kEmCluster = 8;

__global__ void __cluster_dims__(kEmCluster, 1, 1) __launch_bounds__(kPersistThreads, 1)
k_em_cluster(const PersistProblem *probs) {
    namespace cg = cooperative_groups;
    constexpr int NA = kP2PtBase;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    const PersistProblem P = probs[blockIdx.x / kEmCluster];
    __shared__ EmDev se;               // leader only
    __shared__ GridK g;                // this CTA's copy of the pass constants
    __shared__ GridK g_next;           // leader: constants of the next iteration
    __shared__ int done_flag;          // leader: loop state
    __shared__ int4 tab[kGridTab];
    __shared__ double wacc[kPersistThreads / 32][NA];
    __shared__ double bsum[NA];        // this CTA's partial sums
    __shared__ double tsum[NA];        // leader: cluster sums
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long beg = P.m * rank / kEmCluster, end = P.m * (rank + 1) / kEmCluster;
    if (rank == 0) em_copy(&se, P.em, threadIdx.x, blockDim.x);
    for (int e = threadIdx.x; e < kGridTab; e += blockDim.x) tab[e] = grid_entry_q(e, P.dg.s0, P.dg.s1);
    __syncthreads();
    if (rank == 0 && threadIdx.x == 0) {
        done_flag = se.done;
        if (!se.done) grid_params(se.k, P.dg, g_next);
    }
    cl.sync();
    const volatile int *ldone = cl.map_shared_rank(&done_flag, 0);
    const unsigned *lg = reinterpret_cast<const unsigned *>(cl.map_shared_rank(&g_next, 0));
    while (!*ldone) {                  // cluster-uniform: read after a cluster barrier
        static_assert(sizeof(GridK) % 4 == 0, "GridK copied as words");
        for (int w = threadIdx.x; w < (int)(sizeof(GridK) / 4); w += blockDim.x)
            reinterpret_cast<unsigned *>(&g)[w] = lg[w];
        if (lane < NA) wacc[warp][lane] = 0.0;
        __syncthreads();
        GridAcc a;
        a.zero();
        int fold = 0;
        constexpr int PP = 3;
        for (long long base = beg; base < end; base += PP * kPersistThreads) {
            float x[PP], y[PP], z[PP];
            bool ok[PP];
#pragma unroll
            for (int k = 0; k < PP; ++k) {
                const long long p = base + k * kPersistThreads + threadIdx.x;
                ok[k] = p < end;
                x[k] = ok[k] ? __ldg(P.ref + p) : 0.0f;
                y[k] = ok[k] ? __ldg(P.ref + P.m + p) : 0.0f;
                z[k] = ok[k] ? __ldg(P.ref + 2 * P.m + p) : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < PP; ++k) grid_point_q(x[k], y[k], z[k], ok[k], g, tab, P.dg.cells, a);
            fold += PP;
            if (fold >= kGridFold) {
                grid_warp_fold(a, wacc[warp]);
                a.zero();
                fold = 0;
            }
        }
        grid_warp_fold(a, wacc[warp]);
        __syncthreads();
        if (threadIdx.x < NA) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < kPersistThreads / 32; ++w) v += wacc[w][threadIdx.x];
            bsum[threadIdx.x] = v;
        }
        cl.sync();                     // every CTA's partials are final
        if (rank == 0) {
            if (threadIdx.x < NA) {
                double v = 0.0;
                for (int r = 0; r < kEmCluster; ++r) v += cl.map_shared_rank(bsum, r)[threadIdx.x];
                tsum[threadIdx.x] = v;
                P.sums[threadIdx.x] = v;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                rigid_solve_body(tsum, &se, P.objs, P.tnorms, P.masses);
                if (!se.done) grid_params(se.k, P.dg, g_next);
                done_flag = se.done;
            }
        }
        cl.sync();                     // the leader's flag and constants are published
    }
    if (rank == 0) em_copy(P.em, &se, threadIdx.x, blockDim.x);
    cl.sync();                         // no CTA leaves while its DSMEM may still be read
}

// ---------------------------------------------------------------------------
// host

static int width(int mode, int sig) {
    return (mode == FR_POINT_TO_POINT ? kP2PtBase : kP2PlBase) + (sig ? 2 : 0);
}

template <int MODE, int NV, bool SIG, bool FAST, bool DEV>
static int launch_pass_t(const fr_lattice *lat, const float *ref, long long m, const RigidK &k,
                         const RigidK *kd, const int *done, float *wtn, double *scratch,
                         double *sums, cudaStream_t s) {
    const int grid = pass_grid();
    k_rigid_pass<MODE, NV, SIG, FAST, DEV><<<grid, kPassThreads, 0, s>>>(
        ref, m, k, kd, done, lat->table(), lat->table_f(), wtn, scratch);
    FR_CHECK_LAUNCH();
    const int na = width(MODE, SIG);
    k_reduce_cols<<<1, 32 * na, 0, s>>>(scratch, grid, na, sums, done);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

// dispatch on (mode, nv, sigma sums, fast, device params)
static int launch_pass(const fr_lattice *lat, int mode, bool sig, int qpath, bool dev,
                       const float *ref, long long m, const RigidK &k, const RigidK *kd,
                       const int *done, float *wtn, double *scratch, double *sums,
                       cudaStream_t s, GridK *gk_buf = nullptr) {
    const int nv = lat->nv;
    const bool fast = qpath != 0 && !sig && lat->fslots != nullptr;
    if (fast && qpath == 2 && mode == FR_POINT_TO_POINT && nv == 4) {
        const int grid = pass_grid();
        FR_TRY(set_f32_smem());
        const SliceTableF tf = lat->table_f();
        const DenseSliceF dg = lat->dense;
        if (lat->dcells != nullptr) {
            const bool vec = (m & 3) == 0;
            const int g4 = 2 * sm_count();
#define FR_GRID4(DEV, VEC, B, C) \
    k_rigid_pass_grid4<DEV, VEC, B, C><<<g4, kPassThreads, 0, s>>>(ref, m, k, kd, done, dg, scratch)
            if (dev && gk_buf) {
                // the owner of c_grid without the tiled copy (FR_GRID_TILES=0)
                k_grid_params<<<1, 1, 0, s>>>(kd, done, dg, gk_buf);
                FR_CHECK_LAUNCH();
                FR_CUDA(cudaMemcpyToSymbolAsync(c_grid, gk_buf, sizeof(GridK), 0,
                                                cudaMemcpyDeviceToDevice, s));
                if (vec)
                    k_rigid_pass_grid4<true, true, 2, true, true><<<g4, kPassThreads, 0, s>>>(
                        ref, m, k, kd, done, dg, scratch);
                else FR_GRID4(true, false, 2, true);
            }
            else if (vec) { if (dev) FR_GRID4(true, true, 2, false); else FR_GRID4(false, true, 2, false); }
            else { if (dev) FR_GRID4(true, false, 2, false); else FR_GRID4(false, false, 2, false); }
#undef FR_GRID4
            FR_CHECK_LAUNCH();
            k_reduce_cols<<<1, 32 * kP2PtBase, 0, s>>>(scratch, g4, kP2PtBase, sums, done);
            FR_CHECK_LAUNCH();
            return FR_OK;
        } else {
            if (dev) k_rigid_pass_f32<true><<<grid, kPassThreads, kF32Smem, s>>>(ref, m, k, kd, done, tf, scratch);
            else k_rigid_pass_f32<false><<<grid, kPassThreads, kF32Smem, s>>>(ref, m, k, kd, done, tf, scratch);
        }
        FR_CHECK_LAUNCH();
        k_reduce_cols<<<1, 32 * kP2PtBase, 0, s>>>(scratch, grid, kP2PtBase, sums, done);
        FR_CHECK_LAUNCH();
        return FR_OK;
    }
#define FR_L(MODE, NV, SIG, FAST, DEV) \
    return launch_pass_t<MODE, NV, SIG, FAST, DEV>(lat, ref, m, k, kd, done, wtn, scratch, sums, s)
    if (mode == FR_POINT_TO_POINT) {
        if (nv == 4 && !sig) {
            if (fast) { if (dev) FR_L(0, 4, false, true, true); FR_L(0, 4, false, true, false); }
            if (dev) FR_L(0, 4, false, false, true);
            FR_L(0, 4, false, false, false);
        }
        if (nv == 5 && sig) { if (dev) FR_L(0, 5, true, false, true); FR_L(0, 5, true, false, false); }
        if (nv == 5 && !sig) { if (dev) FR_L(0, 5, false, false, true); FR_L(0, 5, false, false, false); }
    } else if (!dev) {
        if (nv == 7 && !sig) {
            if (fast) FR_L(1, 7, false, true, false);
            FR_L(1, 7, false, false, false);
        }
        if (nv == 8 && sig) FR_L(1, 8, true, false, false);
        if (nv == 8 && !sig) FR_L(1, 8, false, false, false);
    }
#undef FR_L
    set_error("lattice value columns (%d) do not match the residual mode / options", nv);
    return FR_EINVAL;
}

}  // namespace fr

// the device-resident EM object behind fr_rigid_em*
struct fr_rigid_em {
    const fr_lattice *lat = nullptr;
    const float *ref = nullptr;
    long long m = 0;
    int fast = 1;
    int max_iters = 0;
    fr::EmDev *d_em = nullptr;
    double *d_sums = nullptr;
    double *d_scratch = nullptr;
    double *d_traces = nullptr;   // [3][max_iters]: objectives, twist norms, inlier masses
    cudaGraphExec_t graph = nullptr;
    int graph_iters = 0;
    cudaStream_t stream = nullptr;   // stream of the last call (destroy orders behind it)
    fr::GridK *d_gk = nullptr;       // staging of the c_grid constants (owner only)
    float4 *d_tiles = nullptr;       // centred tiled model points (owner only)
    unsigned *d_counter = nullptr;   // arrival counter of the tiled pass's fused tail
};

using namespace fr;

extern "C" {

int fr_rigid_pass_width(int mode, int with_sigma) { return width(mode, with_sigma); }

int fr_rigid_scratch_doubles(int mode, int with_sigma, int64_t m) {
    (void)m;
    return pass_grid_max() * std::max(std::max(width(mode, with_sigma), kMaxCand), 28);
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
    double A[4][3];
    embedding_matrix(lat->c, A);
    const double t[3] = {p->c_world[0] - (p->R[0] * p->c_ref[0] + p->R[1] * p->c_ref[1] + p->R[2] * p->c_ref[2]),
                         p->c_world[1] - (p->R[3] * p->c_ref[0] + p->R[4] * p->c_ref[1] + p->R[5] * p->c_ref[2]),
                         p->c_world[2] - (p->R[6] * p->c_ref[0] + p->R[7] * p->c_ref[1] + p->R[8] * p->c_ref[2])};
    RigidK k;
    memset(&k, 0, sizeof(k));
    make_rigid_k(A, p->R, t, p->c_ref, p->c_prime, lat->c.gain, p->m2_col, p->normal_col, &k);
    // the caller's centre is authoritative (the host-side moments use it)
    for (int i = 0; i < 3; ++i) k.c_world[i] = p->c_world[i];
    for (int i = 0; i < 4; ++i)
        k.e0[i] = A[i][0] * k.c_world[0] + A[i][1] * k.c_world[1] + A[i][2] * k.c_world[2];
    cudaStream_t s = (cudaStream_t)stream;
    const int na = width(mode, sig);
    if (m == 0) {
        FR_CUDA(cudaMemsetAsync(sums, 0, na * sizeof(double), s));
        return FR_OK;
    }
    const int qpath = (p->flags & FR_PASS_F32) ? 2 : ((p->flags & FR_PASS_FAST) ? 1 : 0);
    return launch_pass(lat, mode, sig, qpath, false, ref, m, k, nullptr, nullptr, wtn, scratch,
                       sums, s);
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
    k_reduce_cols<<<1, 32 * kMaxCand, 0, s>>>(scratch, grid, kMaxCand, out, nullptr);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

// ---- articulated trees (per-body statistics) --------------------------------

static int body_params(const fr_lattice *lat, const fr_body_pose *poses, int n, double cp,
                       int ncol, std::vector<RigidK> &out) {
    double A[4][3];
    embedding_matrix(lat->c, A);
    out.resize(n);
    for (int b = 0; b < n; ++b) {
        const fr_body_pose &p = poses[b];
        double t[3];
        for (int i = 0; i < 3; ++i)
            t[i] = p.c_world[i] -
                   (p.R[3 * i] * p.c_ref[0] + p.R[3 * i + 1] * p.c_ref[1] + p.R[3 * i + 2] * p.c_ref[2]);
        make_rigid_k(A, p.R, t, p.c_ref, cp, lat->c.gain, -1, ncol, &out[b]);
        for (int i = 0; i < 3; ++i) out[b].c_world[i] = p.c_world[i];
        for (int i = 0; i < 4; ++i)
            out[b].e0[i] = A[i][0] * p.c_world[0] + A[i][1] * p.c_world[1] + A[i][2] * p.c_world[2];
    }
    return FR_OK;
}

int fr_body_pass(const fr_lattice *lat, const float *ref, int64_t m, const fr_body_pose *poses,
                 int n_bodies, const int32_t *chunk_body, const int64_t *chunk_beg, int n_chunks,
                 const int32_t *body_chunks, int mode, double c_prime, int flags,
                 double *d_params, double *sums, float *wtn, double *scratch, void *stream) {
    if (!lat || !lat->blurred || !ref || !poses || n_bodies < 1 || n_chunks < 1 || !chunk_body ||
        !chunk_beg || !body_chunks || !sums || !scratch || !d_params) {
        set_error("invalid articulated pass arguments");
        return FR_EINVAL;
    }
    const bool pl = mode == FR_POINT_TO_PLANE;
    const bool sig = pl ? lat->nv == 8 : lat->nv == 5;   // |y|^2 column splatted
    if ((pl && (lat->nv < 7 || lat->nv > 8 || !wtn)) || (!pl && (lat->nv < 4 || lat->nv > 5))) {
        set_error("lattice value columns (%d) do not match the residual mode", lat->nv);
        return FR_EINVAL;
    }
    std::vector<RigidK> ks;
    FR_TRY(body_params(lat, poses, n_bodies, c_prime, pl ? (sig ? 5 : 4) : -1, ks));
    for (auto &k : ks) k.m2_col = sig ? 4 : -1;
    cudaStream_t s = (cudaStream_t)stream;
    FR_CUDA(cudaMemcpyAsync(d_params, ks.data(), ks.size() * sizeof(RigidK), cudaMemcpyHostToDevice, s));
    const RigidK *kd = reinterpret_cast<const RigidK *>(d_params);
    const long long *cb = reinterpret_cast<const long long *>(chunk_beg);
    const bool fast = (flags & FR_PASS_FAST) && lat->fslots && !sig;
    const int na = (pl ? kP2PlBase : kP2PtBase) + (sig ? 2 : 0);
    const SliceTable t = lat->table();
    const SliceTableF tf = lat->table_f();
#define FR_B(MODE, NV, SIG, FAST) \
    k_body_pass<MODE, NV, SIG, FAST><<<n_chunks, kPassThreads, 0, s>>>(ref, m, kd, chunk_body, cb, t, tf, wtn, scratch)
    if (!pl) {
        if (sig) FR_B(0, 5, true, false);
        else if (fast) FR_B(0, 4, false, true);
        else FR_B(0, 4, false, false);
    } else {
        if (sig) FR_B(1, 8, true, false);
        else if (fast) FR_B(1, 7, false, true);
        else FR_B(1, 7, false, false);
    }
#undef FR_B
    FR_CHECK_LAUNCH();
    k_reduce_segments<<<n_bodies, 32 * na, 0, s>>>(scratch, body_chunks, na, sums);
    FR_CHECK_LAUNCH();
    // the host copy of the params must outlive the async copy
    FR_CUDA(cudaStreamSynchronize(s));
    return FR_OK;
}

// the body pass over device-resident per-body pass constants (RigidK records
// maintained by the articulated device solve), no host copy or sync; a no-op
// once *d_done is set.  point_to_point, 4 value columns.
int fr_body_pass_dev(const fr_lattice *lat, const float *ref, int64_t m, const void *d_bodies,
                     int n_bodies, const int32_t *chunk_body, const int64_t *chunk_beg,
                     int n_chunks, const int32_t *body_chunks, int flags, double *sums,
                     double *scratch, const int32_t *d_done, void *stream) {
    if (!lat || !lat->blurred || !ref || !d_bodies || n_bodies < 1 || n_chunks < 1 ||
        !chunk_body || !chunk_beg || !body_chunks || !sums || !scratch || lat->nv != 4) {
        set_error("invalid device articulated pass arguments");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const RigidK *kd = reinterpret_cast<const RigidK *>(d_bodies);
    const long long *cb = reinterpret_cast<const long long *>(chunk_beg);
    const bool fast = (flags & FR_PASS_FAST) && lat->fslots;
    if (fast)
        k_body_pass<0, 4, false, true><<<n_chunks, kPassThreads, 0, s>>>(
            ref, m, kd, chunk_body, cb, lat->table(), lat->table_f(), nullptr, scratch, d_done);
    else
        k_body_pass<0, 4, false, false><<<n_chunks, kPassThreads, 0, s>>>(
            ref, m, kd, chunk_body, cb, lat->table(), lat->table_f(), nullptr, scratch, d_done);
    FR_CHECK_LAUNCH();
    k_reduce_segments<<<n_bodies, 32 * kP2PtBase, 0, s>>>(scratch, body_chunks, kP2PtBase, sums,
                                                          d_done);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

int fr_body_objective(const float *ref, const float *wtn, int64_t m, const fr_body_pose *cand,
                      int n_bodies, int ncand, const int32_t *chunk_body, const int64_t *chunk_beg,
                      int n_chunks, double *d_params, double *out, double *scratch, void *stream) {
    if (!ref || !wtn || !cand || ncand < 1 || ncand > kMaxCand || !out || !scratch || !d_params) {
        set_error("invalid articulated objective arguments (1 <= k <= %d)", kMaxCand);
        return FR_EINVAL;
    }
    std::vector<RigidK> ks((size_t)ncand * n_bodies);
    memset(ks.data(), 0, ks.size() * sizeof(RigidK));
    for (size_t i = 0; i < ks.size(); ++i) {
        memcpy(ks[i].R, cand[i].R, sizeof(ks[i].R));
        memcpy(ks[i].c_ref, cand[i].c_ref, sizeof(ks[i].c_ref));
        memcpy(ks[i].c_world, cand[i].c_world, sizeof(ks[i].c_world));
    }
    cudaStream_t s = (cudaStream_t)stream;
    FR_CUDA(cudaMemcpyAsync(d_params, ks.data(), ks.size() * sizeof(RigidK), cudaMemcpyHostToDevice, s));
    k_body_objective<<<n_chunks, kPassThreads, 0, s>>>(
        ref, wtn, m, reinterpret_cast<const RigidK *>(d_params), n_bodies, ncand, chunk_body,
        reinterpret_cast<const long long *>(chunk_beg), scratch);
    FR_CHECK_LAUNCH();
    k_reduce_cols<<<1, 32 * kMaxCand, 0, s>>>(scratch, n_chunks, kMaxCand, out, nullptr);
    FR_CHECK_LAUNCH();
    FR_CUDA(cudaStreamSynchronize(s));
    return FR_OK;
}

int fr_body_params_doubles(int n) { return (int)((n * sizeof(RigidK) + 7) / 8); }

// ---- device-resident EM loop -----------------------------------------------

int fr_rigid_em_create(const fr_lattice *lat, const float *ref, int64_t m,
                       const fr_rigid_em_config *cfg, fr_rigid_em **out) {
    return fr_rigid_em_create_on(lat, ref, m, cfg, nullptr, out);
}

// every allocation, copy and kernel of the setup is ordered on the caller's
// stream (which also orders it after the caller's upload / sort of ref)
int fr_rigid_em_create_on(const fr_lattice *lat, const float *ref, int64_t m,
                          const fr_rigid_em_config *cfg, void *stream, fr_rigid_em **out) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!lat || !lat->blurred || !ref || !cfg || !out || m <= 0) {
        set_error("invalid device EM arguments");
        return FR_EINVAL;
    }
    if (lat->dim != 3 || lat->nv != 4) {
        set_error("the device EM loop runs point_to_point with a fixed kernel (4 value columns)");
        return FR_EINVAL;
    }
    if (cfg->max_em_iters < 1 || cfg->max_gn_iters < 0 || cfg->max_halvings < 0) {
        set_error("invalid iteration limits");
        return FR_EINVAL;
    }
    fr_rigid_em *em = new fr_rigid_em();
    em->stream = s;
    em->lat = lat;
    em->ref = ref;
    em->m = m;
    em->fast = (cfg->fast & FR_PASS_F32) ? 2 : ((cfg->fast & FR_PASS_FAST) ? 1 : 0);
    em->max_iters = cfg->max_em_iters;
    EmDev h;
    memset(&h, 0, sizeof(h));
    embedding_matrix(lat->c, h.A);
    for (int i = 0; i < 3; ++i) {
        h.c_ref[i] = cfg->c_ref[i];
        h.s2[i] = cfg->sigma_inv[i] * cfg->sigma_inv[i];
        h.t[i] = cfg->t0[i];
    }
    for (int q = 0; q < 9; ++q) h.R[q] = cfg->R0[q];
    h.cp = cfg->c_prime;
    h.gain = lat->c.gain;
    h.diameter = cfg->diameter;
    h.tol = cfg->twist_tolerance;
    h.use_damping = cfg->damping >= 0.0;
    h.damping = cfg->damping;
    h.step_tol = cfg->step_tolerance;
    h.degenerate_mass = cfg->degenerate_mass;
    h.max_em_iters = cfg->max_em_iters;
    h.max_gn_iters = cfg->max_gn_iters;
    h.max_halvings = cfg->max_halvings;
    make_rigid_k(h.A, h.R, h.t, h.c_ref, h.cp, h.gain, -1, -1, &h.k);
    const int grid = pass_grid_max();
    // stream-ordered pool (see fr_lattice.cu pool_alloc): no cudaMalloc /
    // cudaFree mapping work per registration
    if (cudaMallocAsync((void **)&em->d_em, sizeof(EmDev), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_sums, 32 * sizeof(double), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_scratch, (size_t)grid * 32 * sizeof(double), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_traces, (size_t)3 * cfg->max_em_iters * sizeof(double), s) !=
            cudaSuccess ||
        cudaMemcpyAsync(em->d_em, &h, sizeof(EmDev), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        fr_rigid_em_destroy(em);
        set_error("device EM allocation failed");
        return FR_ECUDA;
    }
    // the constant-bank tiled loop for clouds fr_rigid_em_run does not send
    // through the persistent one-CTA kernel
    bool idle = false;
    if (lat->dcells != nullptr && em->fast == 2 && m > persist_max() &&
        g_const_grid_busy.compare_exchange_strong(idle, true)) {
        const long long ntiles = (m + kQuadPts - 1) / kQuadPts;
        const bool tiled = !(getenv("FR_GRID_TILES") && getenv("FR_GRID_TILES")[0] == '0');
        if (cudaMallocAsync((void **)&em->d_gk, sizeof(GridK), s) != cudaSuccess ||
            (tiled && (cudaMallocAsync((void **)&em->d_tiles,
                                       (size_t)ntiles * kTileF4 * sizeof(float4), s) != cudaSuccess ||
                       cudaMallocAsync((void **)&em->d_counter, sizeof(unsigned), s) != cudaSuccess))) {
            cudaStreamSynchronize(s);
            for (void *p : {(void *)em->d_gk, (void *)em->d_tiles, (void *)em->d_counter})
                if (p) cudaFreeAsync(p, s);
            em->d_gk = nullptr;
            em->d_tiles = nullptr;
            em->d_counter = nullptr;
            g_const_grid_busy.store(false);
            cudaGetLastError();
        } else if (tiled) {
            const long long quads = ntiles * kPassThreads;
            k_tile_points<<<(unsigned)((quads + 255) / 256), 256, 0, s>>>(
                ref, m, (float)cfg->c_ref[0], (float)cfg->c_ref[1], (float)cfg->c_ref[2],
                em->d_tiles, ntiles);
            cudaMemsetAsync(em->d_counter, 0, sizeof(unsigned), s);
            // the tiled pass reads d_gk (via c_grid) as maintained by the solver
            k_grid_params<<<1, 1, 0, s>>>(&em->d_em->k, &em->d_em->done, lat->dense, em->d_gk);
        }
        cudaStreamSynchronize(s);
    }
    *out = em;
    return FR_OK;
}

int fr_rigid_em_destroy(fr_rigid_em *em) {
    if (!em) return FR_OK;
    // the loop may still run on the caller's stream: wait for that stream only
    // (other streams' independent registrations keep running)
    cudaStreamSynchronize(em->stream);
    if (em->graph) cudaGraphExecDestroy(em->graph);
    for (void *p : {(void *)em->d_em, (void *)em->d_sums, (void *)em->d_scratch,
                    (void *)em->d_traces})
        if (p) cudaFreeAsync(p, em->stream);
    if (em->d_tiles) cudaFreeAsync(em->d_tiles, em->stream);
    if (em->d_counter) cudaFreeAsync(em->d_counter, em->stream);
    if (em->d_gk) {     // the stream is drained: no pass still reads c_grid
        cudaFreeAsync(em->d_gk, em->stream);
        g_const_grid_busy.store(false);
    }
    delete em;
    return FR_OK;
}

int fr_rigid_em_sums(fr_rigid_em *em, double **d_sums, int *width_out) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    if (d_sums) *d_sums = em->d_sums;
    if (width_out) *width_out = kP2PtBase;
    return FR_OK;
}

// the tiled pass of the device loop (EM objects holding c_grid): the pass
// constants of the current pose (d_gk, kept by the solver) copied into the
// constant bank, then one kernel; SOLVE fuses the iteration's solve
static int em_tiles_pass(fr_rigid_em *em, cudaStream_t s, bool solve, bool copy = true) {
    if (copy)
        FR_CUDA(cudaMemcpyToSymbolAsync(c_grid, em->d_gk, sizeof(GridK), 0,
                                        cudaMemcpyDeviceToDevice, s));
    const int n = em->max_iters;
    const TailArgs ta{em->d_counter, em->d_sums, solve ? em->d_em : nullptr, em->d_traces,
                      em->d_traces + n, em->d_traces + 2 * n, solve ? em->d_gk : nullptr};
    if (solve)
        k_rigid_pass_tiles<kGridFold, 2, true><<<2 * sm_count(), kPassThreads, 0, s>>>(
            em->d_tiles, em->m, &em->d_em->done, em->lat->dense, em->d_scratch, ta);
    else
        k_rigid_pass_tiles<kGridFold, 2, false><<<2 * sm_count(), kPassThreads, 0, s>>>(
            em->d_tiles, em->m, &em->d_em->done, em->lat->dense, em->d_scratch, ta);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

static int em_pass(fr_rigid_em *em, cudaStream_t s) {
    if (em->d_tiles) return em_tiles_pass(em, s, false);
    RigidK unused;
    memset(&unused, 0, sizeof(unused));
    return launch_pass(em->lat, FR_POINT_TO_POINT, false, em->fast, true, em->ref, em->m,
                       unused, &em->d_em->k, &em->d_em->done, nullptr, em->d_scratch, em->d_sums,
                       s, em->d_gk);
}

static int em_solve(fr_rigid_em *em, cudaStream_t s) {
    const int n = em->max_iters;
    k_rigid_solve<<<1, 32, 0, s>>>(em->d_sums, em->d_em, em->d_traces, em->d_traces + n,
                                   em->d_traces + 2 * n, em->lat->dense,
                                   em->d_tiles ? em->d_gk : nullptr);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

// FR_EM_FUSED=0: pass and solver as separate kernels in the tiled loop
static bool em_fused() {
    const char *e = getenv("FR_EM_FUSED");
    return !(e && e[0] == '0');
}

static int em_iteration(fr_rigid_em *em, cudaStream_t s) {
    if (em->d_tiles && em_fused()) return em_tiles_pass(em, s, true);
    FR_TRY(em_pass(em, s));
    return em_solve(em, s);
}

int fr_rigid_em_pass_kernel(fr_rigid_em *em, void *stream) {
    if (!em || !em->d_tiles) {
        set_error("fr_rigid_em_pass_kernel needs an EM object on the tiled loop");
        return FR_EINVAL;
    }
    em->stream = (cudaStream_t)stream;
    return em_tiles_pass(em, (cudaStream_t)stream, false, false);
}

int fr_rigid_em_kernels_per_iter(const fr_rigid_em *em) {
    if (!em) return 0;
    if (em->d_tiles) return em_fused() ? 1 : 2;    // tiled pass (+ solver kernel)
    if (em->d_gk) return 4;                          // params, grid pass, reduction, solver
    return 3;                                        // pass, reduction, solver
}

int fr_rigid_em_pass(fr_rigid_em *em, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    em->stream = (cudaStream_t)stream;
    return em_pass(em, (cudaStream_t)stream);
}

int fr_rigid_em_solve(fr_rigid_em *em, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    em->stream = (cudaStream_t)stream;
    return em_solve(em, (cudaStream_t)stream);
}

// enqueue n EM iterations (pass + solve each); iterations after termination
// are no-ops.  Groups of iterations replay one captured CUDA graph.
int fr_rigid_em_enqueue(fr_rigid_em *em, int n, void *stream) {
    if (!em || n < 0) {
        set_error("invalid enqueue arguments");
        return FR_EINVAL;
    }
    em->stream = (cudaStream_t)stream;
    cudaStream_t s = (cudaStream_t)stream;
    constexpr int kGraphIters = 8;
    if (!em->graph) {
        cudaStream_t cs;
        FR_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t g;
        FR_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < kGraphIters; ++i) {
            int st = em_iteration(em, cs);
            if (st != FR_OK) {
                cudaStreamEndCapture(cs, &g);
                cudaStreamDestroy(cs);
                return st;
            }
        }
        FR_CUDA(cudaStreamEndCapture(cs, &g));
        FR_CUDA(cudaGraphInstantiate(&em->graph, g, 0));
        cudaGraphDestroy(g);
        cudaStreamDestroy(cs);
        em->graph_iters = kGraphIters;
    }
    int left = n;
    while (left >= em->graph_iters) {
        FR_CUDA(cudaGraphLaunch(em->graph, s));
        left -= em->graph_iters;
    }
    for (; left > 0; --left) FR_TRY(em_iteration(em, s));
    return FR_OK;
}

int fr_rigid_em_status(fr_rigid_em *em, int *done, int *iterations, int *termination,
                       void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    int h[3];
    cudaStream_t s = (cudaStream_t)stream;
    FR_CUDA(cudaMemcpyAsync(h, &em->d_em->done, 3 * sizeof(int), cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaStreamSynchronize(s));
    if (done) *done = h[0];
    if (iterations) *iterations = h[1];
    if (termination) *termination = h[2];
    return FR_OK;
}

static bool em_persist_ok(const fr_rigid_em *em) {
    return em && em->fast == 2 && em->lat && em->lat->dcells != nullptr && em->lat->nv == 4 &&
           em->m > 0;
}


// FR_EM_CLUSTER=0: one CTA per small problem (k_em_persistent) instead of a
// cluster of kEmCluster CTAs (k_em_cluster)
static bool em_cluster() {
    const char *e = getenv("FR_EM_CLUSTER");
    return !(e && e[0] == '0');
}

int fr_rigid_em_run_batch(fr_rigid_em **ems, int n, void *stream) {
    if (n < 0 || (n > 0 && !ems)) {
        set_error("invalid batch arguments");
        return FR_EINVAL;
    }
    if (n == 0) return FR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    std::vector<PersistProblem> h((size_t)n);
    for (int i = 0; i < n; ++i) {
        fr_rigid_em *em = ems[i];
        if (!em_persist_ok(em)) {
            set_error("batch problem %d does not run the dense-grid float32 point path", i);
            return FR_EINVAL;
        }
        const int k = em->max_iters;
        h[i] = PersistProblem{em->ref, em->m, em->d_em, em->d_sums, em->d_traces,
                              em->d_traces + k, em->d_traces + 2 * k, em->lat->dense};
        em->stream = s;
    }
    PersistProblem *d = nullptr;
    FR_CUDA(cudaMallocAsync((void **)&d, h.size() * sizeof(PersistProblem), s));
    FR_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(PersistProblem), cudaMemcpyHostToDevice,
                            s));
    if (em_cluster()) k_em_cluster<<<n * kEmCluster, kPersistThreads, 0, s>>>(d);
    else k_em_persistent<<<n, kPersistThreads, 0, s>>>(d);
    FR_CHECK_LAUNCH();
    FR_CUDA(cudaFreeAsync(d, s));
    FR_CUDA(cudaStreamSynchronize(s));   // the host vector h backs the copy
    return FR_OK;
}

int fr_rigid_em_persistent(const fr_rigid_em *em) {
    return em_persist_ok(em) && em->m <= persist_max() ? 1 : 0;
}

int fr_rigid_em_run(fr_rigid_em *em, void *stream) {
    if (fr_rigid_em_persistent(em)) return fr_rigid_em_run_batch(&em, 1, stream);
    // one chunk of iterations always in flight: chunk k + 1 is enqueued before
    // the host waits for chunk k's done flag (copied into pinned memory behind
    // it), so the GPU never drains for a poll; iterations after termination
    // are no-op launches (8 first, then chunks of 32)
    cudaStream_t s = (cudaStream_t)stream;
    static thread_local int *flags = nullptr;      // [2][4] pinned
    static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
    if (!flags) {
        FR_CUDA(cudaHostAlloc((void **)&flags, 8 * sizeof(int), cudaHostAllocDefault));
        for (int i = 0; i < 2; ++i) FR_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    int issued = 0, k = 0;
    auto chunk = [&](int n) -> int {
        FR_TRY(fr_rigid_em_enqueue(em, n, stream));
        FR_CUDA(cudaMemcpyAsync(flags + 4 * (k & 1), &em->d_em->done, 3 * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
        FR_CUDA(cudaEventRecord(ev[k & 1], s));
        issued += n;
        ++k;
        return FR_OK;
    };
    FR_TRY(chunk(8));
    while (true) {
        const bool more = issued < em->max_iters + 40;
        if (more) FR_TRY(chunk(32));
        const int prev = (k - (more ? 2 : 1)) & 1;
        FR_CUDA(cudaEventSynchronize(ev[prev]));
        if (flags[4 * prev] || !more) break;
    }
    FR_CUDA(cudaStreamSynchronize(s));
    return FR_OK;
}

int fr_rigid_em_result(fr_rigid_em *em, double *R, double *t, double *objectives,
                       double *twist_norms, double *inlier_masses, int *iterations,
                       int *termination, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    EmDev h;
    FR_CUDA(cudaMemcpyAsync(&h, em->d_em, sizeof(EmDev), cudaMemcpyDeviceToHost, s));
    std::vector<double> tr((size_t)3 * em->max_iters);
    FR_CUDA(cudaMemcpyAsync(tr.data(), em->d_traces, tr.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaStreamSynchronize(s));
    if (R) memcpy(R, h.R, 9 * sizeof(double));
    if (t) memcpy(t, h.t, 3 * sizeof(double));
    const int n = std::min(h.iterations, em->max_iters);
    if (objectives) memcpy(objectives, tr.data(), n * sizeof(double));
    if (twist_norms) memcpy(twist_norms, tr.data() + em->max_iters, n * sizeof(double));
    if (inlier_masses) memcpy(inlier_masses, tr.data() + 2 * em->max_iters, n * sizeof(double));
    if (iterations) *iterations = h.iterations;
    if (termination) *termination = h.termination;
    if (h.termination == kTermSolver && h.done) {
        set_error("normal equations not factorizable after damping escalation");
        return FR_ESOLVER;
    }
    return FR_OK;
}

}  // extern "C"
