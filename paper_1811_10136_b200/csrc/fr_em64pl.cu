// The float64 rigid point-to-plane EM loop on B200: one cooperative,
// grid-resident kernel runs the whole registration (pipeline.py:125-181 with
// residual_mode = "point_to_plane"), in the reference's float64 arithmetic.
//
// Per EM iteration, in every CTA over its contiguous tiles of the centred,
// Morton-ordered model points:
//   E pass       forward map, simplex + slice of the dense float64 grid of
//                [1, y, n] (permutohedral.py:171-215, 329-341), moments
//                epilogue with the averaged normal and its validity
//                (estep.py:195-217), the residual spec of the M step
//                (mstep.py:39-98: plane row sqrt(w) n^T where the normal is
//                valid, point rows sqrt(w) I in meters where it is not) stored
//                per point in float64, and the normal equations H (21), g (6),
//                the objective and the inlier mass (mstep.py:179-210);
//   barrier      every CTA sums the partial rows in the same fixed order and
//                runs the same float64 logic on them (bit-identical decisions
//                in every CTA, no broadcast);
//   M step       (mstep.py:421-459) damped 6x6 Cholesky with tenfold
//                escalation, step halving: the candidate poses of a batch of
//                halvings are built in parallel by warp 0 (twist exponential
//                + polar factor, geometry.py:154-189), one pass evaluates
//                their objectives over the stored spec, the first accepted
//                one wins (the first batch is the full step alone); with
//                max_gn_iters > 1 an assembly pass re-forms H, g at the
//                accepted pose with the same spec; then update magnitude and
//                termination (pipeline.py:167-177).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fr_common.cuh"
#include "fr_reduce.cuh"
#include "fr_solve.cuh"
#include "fr_em64.cuh"

namespace fr {

constexpr int kPlStats = 29;     // mass | H upper 21 | g 6 | sum of squared rows
constexpr int kPlMaxCand = 16;   // candidates per objective pass
constexpr int kPlSpec = 7;       // w | t 3 | n 3 (n = 0: point rows)

struct EmPlDev {
    double R[9], t[3];
    double c_ref[3];
    double diameter, tol, damping, step_tol, degenerate_mass;
    int max_em_iters, max_gn_iters, max_halvings, use_damping;
    int done, iterations, termination, pad;
};

struct Em64PlArgs {
    const double *tiles;   // [n_tiles][3][T] centred model points
    long long m;
    long long m_pad;       // n_tiles * T (spec plane stride)
    int tiles_per_cta;
    DenseSliceD g;         // r2 = 4: [y0 y1 | y2 m | n0 n1 | n2 0]
    EmPlDev *em;
    double *spec;          // [kPlSpec][m_pad]
    double *partials;      // [2][grid][kE64Row]
    double *sums;          // [kE64Row] the last E pass's sums
    double *traces;        // [3][max_iters]
    unsigned *counter;
    int n_iters;
    double sc[3];
    double cp;
};

// 6-vector row a with residual r and weight w into (H upper 21, g 6)
__device__ __forceinline__ void pl_row(double w, const double *a, double r, double *acc) {
    int o = 1;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        const double wa = w * a[i];
#pragma unroll
        for (int j = i; j < 6; ++j) {
            acc[o] = fma(wa, a[j], acc[o]);
            ++o;
        }
        acc[22 + i] = fma(wa, r, acc[22 + i]);
    }
}

// normal equations of one point's spec at world position x (mstep.py:179-210):
// plane row [x x n, n] with residual n.(x - t), or the point rows
// J = [-[x]x | I] with residual x - t; acc[28] += the squared rows
__device__ __forceinline__ void pl_assemble(double w, const double *x, const double *t,
                                            const double *n, bool plane, double *acc) {
    const double d0 = x[0] - t[0], d1 = x[1] - t[1], d2 = x[2] - t[2];
    if (plane) {
        const double a6[6] = {x[1] * n[2] - x[2] * n[1], x[2] * n[0] - x[0] * n[2],
                              x[0] * n[1] - x[1] * n[0], n[0], n[1], n[2]};
        const double rr = (n[0] * d0 + n[1] * d1) + n[2] * d2;
        pl_row(w, a6, rr, acc);
        acc[28] = fma(w * rr, rr, acc[28]);
    } else if (w > 0.0) {
        // J^T J = [[|x|^2 I - x x^T, [x]x], [[x]x^T, I]], J^T d = [x x d, d]
        const double xx = (x[0] * x[0] + x[1] * x[1]) + x[2] * x[2];
        const double h6[21] = {xx - x[0] * x[0], -x[0] * x[1], -x[0] * x[2], 0.0, -x[2], x[1],
                               xx - x[1] * x[1], -x[1] * x[2], x[2], 0.0, -x[0],
                               xx - x[2] * x[2], -x[1], x[0], 0.0,
                               1.0, 0.0, 0.0, 1.0, 0.0, 1.0};
#pragma unroll
        for (int q = 0; q < 21; ++q) acc[1 + q] = fma(w, h6[q], acc[1 + q]);
        const double gv[6] = {x[1] * d2 - x[2] * d1, x[2] * d0 - x[0] * d2, x[0] * d1 - x[1] * d0,
                              d0, d1, d2};
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[22 + q] = fma(w, gv[q], acc[22 + q]);
        acc[28] = fma(w, (d0 * d0 + d1 * d1) + d2 * d2, acc[28]);
    }
}

// squared residual rows of one point's spec at x (mstep.py:132-138)
__device__ __forceinline__ double pl_cost(double w, const double *x, const double *t,
                                          const double *n, bool plane) {
    const double d0 = x[0] - t[0], d1 = x[1] - t[1], d2 = x[2] - t[2];
    const double rr = (n[0] * d0 + n[1] * d1) + n[2] * d2;
    return w * (plane ? rr * rr : (d0 * d0 + d1 * d1) + d2 * d2);
}

// the E pass of one point: moments, spec (stored), normal equations
__device__ __forceinline__ void pl_point(const Em64PlArgs &a, const Pose64 &k, double cp,
                                         double h0, double h1, double h2, bool valid,
                                         long long pidx, double *acc) {
    double x[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        x[i] = fma(k.R[3 * i + 2], h2, fma(k.R[3 * i + 1], h1, k.R[3 * i] * h0)) + k.cw[i];
    Simplex64 S;
    e64_simplex(a.g, a.sc, x, S);
    double o[8];
    e64_gather<4>(a.g, S, o);
    // epilogue (estep.py:195-217): m0 = max(out0, 0), supported iff m0 >= 1e-12,
    // w = m0 / (m0 + c'), target = m1 / m0, avg = n-sum / m0, the normal
    // avg / max(|avg|, 0.1) valid iff supported and |avg| >= 0.1
    const double m0 = o[3] > 0.0 ? o[3] : 0.0;
    const bool sup = m0 >= 1e-12 && S.in_range && valid;
    const double den = m0 + cp;
    const double q = rcp64(m0 * den);
    const double inv = den * q;
    const double w = sup ? (cp > 0.0 ? (m0 * m0) * q : 1.0) : 0.0;
    double t[3], n[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) t[j] = sup ? o[j] * inv : x[j];
    const double av0 = o[4] * inv, av1 = o[5] * inv, av2 = o[6] * inv;
    const double len2 = (av0 * av0 + av1 * av1) + av2 * av2;
    const bool plane = sup && len2 >= 0.01;
    const double il = plane ? 1.0 / sqrt(len2) : 0.0;
    n[0] = av0 * il;
    n[1] = av1 * il;
    n[2] = av2 * il;
    // the spec, kept for the halving / extra Gauss-Newton passes
    double *sp = a.spec + pidx;
    sp[0] = w;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        sp[(1 + j) * a.m_pad] = t[j];
        sp[(4 + j) * a.m_pad] = n[j];
    }
    acc[0] += w;
    if (sup) pl_assemble(w, x, t, n, plane, acc);
}

__device__ __forceinline__ void pl_load_spec(const Em64PlArgs &a, long long pidx, double &w,
                                             double *t, double *n) {
    const double *sp = a.spec + pidx;
    w = sp[0];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        t[j] = sp[(1 + j) * a.m_pad];
        n[j] = sp[(4 + j) * a.m_pad];
    }
}

// block reduction of NA columns into this CTA's row of `rows`
template <int THREADS, int NA>
__device__ __forceinline__ void pl_block_row(double (&acc)[NA], double (*red)[32], double *rows) {
    constexpr int W = THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    red[warp][lane] = warp_reduce_scatter(acc);
    __syncthreads();
    if (threadIdx.x < NA) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) s += red[w][threadIdx.x];
        rows[(long long)blockIdx.x * kE64Row + threadIdx.x] = s;
        __threadfence();
    }
    __syncthreads();
}

// grid barrier #k (monotone counter) + the fixed-order column sums of the
// first `na` columns into out[] (every CTA, same order)
template <int THREADS, int MINB>
__device__ __forceinline__ void pl_barrier_reduce(const Em64PlArgs &a, unsigned k,
                                                  const double *rows, int na, double (*red)[32],
                                                  double *out) {
    constexpr int W = THREADS / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nb = (int)gridDim.x;
    if (threadIdx.x == 0) {
        const unsigned target = (unsigned)nb * (k + 1);
        atomicAdd(a.counter, 1u);
        while (ld_acquire(a.counter) < target) __nanosleep(20);
    }
    __syncthreads();
    double s = 0.0;
    if (lane < na) {
        constexpr int kMaxRows = (kE64MaxSms * MINB + W - 1) / W;
        double r[kMaxRows];
#pragma unroll
        for (int u = 0; u < kMaxRows; ++u) {
            const int b = warp + W * u;
            r[u] = b < nb ? __ldcg(rows + (long long)b * kE64Row + lane) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kMaxRows; ++u) s += r[u];
    }
    __syncthreads();
    red[warp][lane] = s;
    __syncthreads();
    if (threadIdx.x < na) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < W; ++j) v += red[j][threadIdx.x];
        out[threadIdx.x] = v;
    }
    __syncthreads();
}

__device__ __forceinline__ void unpack_h21(const double *s21, double (*H)[6]) {
    int o = 0;
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = i; j < 6; ++j) {
            H[i][j] = s21[o];
            H[j][i] = s21[o];
            ++o;
        }
}

// shared control block of the M step (written by thread 0, read by all after
// a barrier; identical in every CTA)
struct PlCtl {
    double Rc[9], tc[3];            // current GN pose
    double step[6];
    double value, value0;
    double H21[21], g[6];
    double candR[kPlMaxCand][9], candT[kPlMaxCand][3], candW[kPlMaxCand][3];
    double cand_cost[kPlMaxCand];
    int phase;                      // 0 E pass, 1 candidates, 2 assembly, 3 finish
    int n_cand, h0, gn, accepted_h;
};

// the serial pieces run out of line (one thread / one lane each), so the
// point loops keep their registers
static __device__ __noinline__ int pl_solve(PlCtl &c, const EmPlDev &se) {
    double H[6][6];
    unpack_h21(c.H21, H);
    return gn_solve_dev(H, c.g, se.use_damping, se.damping, c.step) ? 1 : 0;
}

static __device__ __noinline__ void pl_candidate(PlCtl &c, const EmPlDev &se, int lane) {
    const int h = c.h0 + lane;
    double tw[6];
    const double scale = ldexp(1.0, -h);           // 0.5^h exactly
#pragma unroll
    for (int q = 0; q < 6; ++q) tw[q] = scale * c.step[q];
    double Rn[9], tn[3];
    apply_twist_dev(tw, c.Rc, c.tc, Rn, tn);
#pragma unroll
    for (int q = 0; q < 9; ++q) c.candR[lane][q] = Rn[q];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        c.candT[lane][i] = tn[i];
        c.candW[lane][i] = Rn[3 * i] * se.c_ref[0] + Rn[3 * i + 1] * se.c_ref[1] +
                           Rn[3 * i + 2] * se.c_ref[2] + tn[i];
    }
}

static __device__ __noinline__ void pl_finish(PlCtl &c, EmPlDev &se, double *traces,
                                              bool record) {
    const int k = se.iterations - 1;
    double Rd[9];
    m3_mul_t(c.Rc, se.R, Rd);
    const double dx = c.tc[0] - se.t[0], dy = c.tc[1] - se.t[1], dz = c.tc[2] - se.t[2];
    const double norm = rotation_angle_dev(Rd) + sqrt((dx * dx + dy * dy) + dz * dz) / se.diameter;
    if (record) traces[se.max_em_iters + k] = norm;
    if (norm < se.tol) {          // sub-tolerance motion: dropped (pipeline.py:169-173)
        if (record) traces[k] = c.value0;
        se.termination = kTermConverged;
        se.done = 1;
        return;
    }
    for (int q = 0; q < 9; ++q) se.R[q] = c.Rc[q];
    for (int q = 0; q < 3; ++q) se.t[q] = c.tc[q];
    if (record) traces[k] = c.value;
    if (k + 1 >= se.max_em_iters) {
        se.termination = kTermMaxIters;
        se.done = 1;
    }
}

template <int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) k_em64pl(Em64PlArgs a) {
    constexpr int W = THREADS / 32;
    __shared__ double red[W][32];
    __shared__ double tsum[kE64Row];
    __shared__ EmPlDev se;
    __shared__ PlCtl c;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = (int)gridDim.x;
    const long long t0 = (long long)blockIdx.x * a.tiles_per_cta;
    const long long n_tiles_all = (a.m + THREADS - 1) / THREADS;
    const int nt = (int)max(0LL, min((long long)a.tiles_per_cta, n_tiles_all - t0));
    const double cp = a.cp;
    copy_cg(&se, a.em, tid, THREADS);
    __syncthreads();
    unsigned bar = 0;                 // barriers passed (uniform)
    auto rows_of = [&](unsigned k) { return a.partials + (long long)(k & 1) * nb * kE64Row; };
    for (int it = 0; it < a.n_iters; ++it) {
        if (se.done) break;
        // ---- E pass at the current pose --------------------------------
        {
            Pose64 pose;
#pragma unroll
            for (int q = 0; q < 9; ++q) pose.R[q] = se.R[q];
#pragma unroll
            for (int i = 0; i < 3; ++i)
                pose.cw[i] = se.R[3 * i] * se.c_ref[0] + se.R[3 * i + 1] * se.c_ref[1] +
                             se.R[3 * i + 2] * se.c_ref[2] + se.t[i];
            double acc[kPlStats];
#pragma unroll
            for (int q = 0; q < kPlStats; ++q) acc[q] = 0.0;
            const double *src = a.tiles + t0 * 3 * THREADS + tid;
            long long pidx = t0 * THREADS + tid;
            for (int tt = 0; tt < nt; ++tt, src += 3 * THREADS, pidx += THREADS)
                pl_point(a, pose, cp, src[0], src[THREADS], src[2 * THREADS], pidx < a.m, pidx,
                         acc);
            pl_block_row<THREADS, kPlStats>(acc, red, rows_of(bar));
            pl_barrier_reduce<THREADS, MINB>(a, bar, rows_of(bar), kPlStats, red, tsum);
            ++bar;
        }
        if (blockIdx.x == 0 && tid < kPlStats) a.sums[tid] = tsum[tid];
        // ---- M step (mstep.py:421-459) ---------------------------------
        if (tid == 0) {
            const int k = se.iterations;
            se.iterations = k + 1;
            const double mass = tsum[0];
            if (blockIdx.x == 0) a.traces[2 * se.max_em_iters + k] = mass;
            c.phase = 3;
            c.accepted_h = -1;
            if (mass < se.degenerate_mass) {
                if (blockIdx.x == 0) {
                    a.traces[k] = CUDART_NAN;
                    a.traces[se.max_em_iters + k] = CUDART_NAN;
                }
                se.termination = kTermDegenerate;
                se.done = 1;
                c.phase = 4;            // no update magnitude
            } else {
                c.value0 = c.value = 0.5 * tsum[28];
#pragma unroll
                for (int q = 0; q < 21; ++q) c.H21[q] = tsum[1 + q];
#pragma unroll
                for (int q = 0; q < 6; ++q) c.g[q] = tsum[22 + q];
#pragma unroll
                for (int q = 0; q < 9; ++q) c.Rc[q] = se.R[q];
#pragma unroll
                for (int q = 0; q < 3; ++q) c.tc[q] = se.t[q];
                c.gn = 0;
                c.phase = 0;            // solve
            }
        }
        __syncthreads();
        // GN iterations (uniform control: every CTA makes the same decisions)
        while (c.phase == 0) {
            if (tid == 0) {
                bool any = false;
#pragma unroll
                for (int q = 0; q < 6; ++q) any |= c.g[q] != 0.0;
                if (!any || c.gn >= se.max_gn_iters) {
                    c.phase = 3;
                } else {
                    if (!pl_solve(c, se)) {
                        se.termination = kTermSolver;
                        se.done = 1;
                        c.phase = 4;
                    } else {
                        c.h0 = 0;
                        c.n_cand = 1;      // the full step first (the common case)
                        c.phase = 1;
                    }
                }
            }
            __syncthreads();
            // halving batches: candidate poses built in parallel, one pass
            while (c.phase == 1) {
                if (warp == 0 && lane < c.n_cand) pl_candidate(c, se, lane);
                __syncthreads();
                const int ncand = c.n_cand;
                double cost[kPlMaxCand];
#pragma unroll
                for (int h = 0; h < kPlMaxCand; ++h) cost[h] = 0.0;
                // candidate-major: one candidate pose in registers per sweep
                // (the full step alone in the common case)
#pragma unroll 1
                for (int h = 0; h < ncand; ++h) {
                    Pose64 cand;
#pragma unroll
                    for (int q = 0; q < 9; ++q) cand.R[q] = c.candR[h][q];
#pragma unroll
                    for (int q = 0; q < 3; ++q) cand.cw[q] = c.candW[h][q];
                    double sum = 0.0;
                    const double *src = a.tiles + t0 * 3 * THREADS + tid;
                    long long pidx = t0 * THREADS + tid;
                    for (int tt = 0; tt < nt; ++tt, src += 3 * THREADS, pidx += THREADS) {
                        const double h0 = src[0], h1 = src[THREADS], h2 = src[2 * THREADS];
                        double w, t[3], n[3], x[3];
                        pl_load_spec(a, pidx, w, t, n);
                        const bool plane = (n[0] != 0.0 || n[1] != 0.0) || n[2] != 0.0;
#pragma unroll
                        for (int i = 0; i < 3; ++i)
                            x[i] = fma(cand.R[3 * i + 2], h2,
                                       fma(cand.R[3 * i + 1], h1, cand.R[3 * i] * h0)) + cand.cw[i];
                        sum += pidx < a.m ? pl_cost(w, x, t, n, plane) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < kPlMaxCand; ++q) cost[q] = q == h ? sum : cost[q];
                }
                pl_block_row<THREADS, kPlMaxCand>(cost, red, rows_of(bar));
                pl_barrier_reduce<THREADS, MINB>(a, bar, rows_of(bar), kPlMaxCand, red,
                                                 c.cand_cost);
                ++bar;
                if (tid == 0) {
                    int acc_h = -1;
                    for (int h = 0; h < ncand && acc_h < 0; ++h) {
                        const double cv = 0.5 * c.cand_cost[h];
                        if (cv <= c.value * (1.0 + 1e-12) + 1e-300) acc_h = h;   // mstep.py:446
                    }
                    if (acc_h >= 0) {
                        const int h = c.h0 + acc_h;
                        const double scale = ldexp(1.0, -h);
#pragma unroll
                        for (int q = 0; q < 9; ++q) c.Rc[q] = c.candR[acc_h][q];
#pragma unroll
                        for (int q = 0; q < 3; ++q) c.tc[q] = c.candT[acc_h][q];
                        c.value = 0.5 * c.cand_cost[acc_h];
                        c.accepted_h = h;
                        double sn = 0.0;
#pragma unroll
                        for (int q = 0; q < 6; ++q) sn += (scale * c.step[q]) * (scale * c.step[q]);
                        c.gn += 1;
                        c.phase = (sqrt(sn) <= se.step_tol || c.gn >= se.max_gn_iters) ? 3 : 2;
                    } else if (c.h0 + ncand <= se.max_halvings) {
                        c.h0 += ncand;
                        c.n_cand = min(kPlMaxCand, se.max_halvings + 1 - c.h0);
                    } else {
                        c.phase = 3;       // no acceptable step: stop (mstep.py:450-451)
                    }
                }
                __syncthreads();
            }
            // another GN iteration: H, g at the accepted pose, same spec
            if (c.phase == 2) {
                double cw[3];
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    cw[i] = c.Rc[3 * i] * se.c_ref[0] + c.Rc[3 * i + 1] * se.c_ref[1] +
                            c.Rc[3 * i + 2] * se.c_ref[2] + c.tc[i];
                double acc[kPlStats];
#pragma unroll
                for (int q = 0; q < kPlStats; ++q) acc[q] = 0.0;
                const double *src = a.tiles + t0 * 3 * THREADS + tid;
                long long pidx = t0 * THREADS + tid;
                for (int tt = 0; tt < nt; ++tt, src += 3 * THREADS, pidx += THREADS) {
                    const double h0 = src[0], h1 = src[THREADS], h2 = src[2 * THREADS];
                    double w, t[3], n[3], x[3];
                    pl_load_spec(a, pidx, w, t, n);
                    if (pidx >= a.m) w = 0.0;
#pragma unroll
                    for (int i = 0; i < 3; ++i)
                        x[i] = fma(c.Rc[3 * i + 2], h2, fma(c.Rc[3 * i + 1], h1, c.Rc[3 * i] * h0)) +
                               cw[i];
                    const bool plane = (n[0] != 0.0 || n[1] != 0.0) || n[2] != 0.0;
                    if (w > 0.0) pl_assemble(w, x, t, n, plane, acc);
                }
                pl_block_row<THREADS, kPlStats>(acc, red, rows_of(bar));
                pl_barrier_reduce<THREADS, MINB>(a, bar, rows_of(bar), kPlStats, red, tsum);
                ++bar;
                if (tid == 0) {
#pragma unroll
                    for (int q = 0; q < 21; ++q) c.H21[q] = tsum[1 + q];
#pragma unroll
                    for (int q = 0; q < 6; ++q) c.g[q] = tsum[22 + q];
                    c.phase = 0;
                }
                __syncthreads();
            }
        }
        // ---- update magnitude and termination (pipeline.py:167-177) -------
        if (tid == 0 && c.phase == 3) pl_finish(c, se, a.traces, blockIdx.x == 0);
        __syncthreads();
    }
    if (blockIdx.x == 0) {
        const unsigned long long *s8 = reinterpret_cast<const unsigned long long *>(&se);
        for (int q = tid; q < (int)(sizeof(EmPlDev) / 8); q += THREADS)
            reinterpret_cast<unsigned long long *>(a.em)[q] = s8[q];
    }
}

constexpr int kPlThreads = 384;
constexpr int kPlMinB = 1;

static int pl_grid() {
    static int grid = 0;
    if (!grid) {
        int per = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_em64pl<kPlThreads, kPlMinB>,
                                                          kPlThreads, 0) != cudaSuccess ||
            per < 1)
            per = 1;
        grid = std::min(per, kPlMinB) * std::min(sm_count(), kE64MaxSms);
    }
    return grid;
}

__global__ void k_pl_tiles(const double *ref, long long m, double c0, double c1, double c2,
                           int T, long long n_tiles, double *tiles) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_tiles * T) return;
    const long long t = i / T;
    const int j = (int)(i % T);
    const double c[3] = {c0, c1, c2};
#pragma unroll
    for (int q = 0; q < 3; ++q) tiles[(t * 3 + q) * T + j] = i < m ? ref[q * m + i] - c[q] : 0.0;
}

}  // namespace fr

struct fr_em64pl {
    const fr_lattice *lat = nullptr;
    long long m = 0, n_tiles = 0;
    int max_iters = 0, grid = 0;
    double cp = 0.0;
    fr::EmPlDev *d_em = nullptr;
    double *d_tiles = nullptr, *d_spec = nullptr, *d_partials = nullptr, *d_sums = nullptr,
           *d_traces = nullptr;
    unsigned *d_sync = nullptr;
    cudaStream_t stream = nullptr;
};

using namespace fr;

extern "C" {

int fr_em64pl_create(const fr_lattice *lat, const double *ref, int64_t m,
                     const fr_rigid_em_config *cfg, void *stream, fr_em64pl **out) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!lat || !lat->blurred || !ref || !cfg || !out || m <= 0) {
        set_error("invalid float64 point-to-plane EM arguments");
        return FR_EINVAL;
    }
    if (lat->dim != 3 || lat->nv != 7) {
        set_error("the float64 point-to-plane loop needs the [1, y, n] lattice (7 value columns)");
        return FR_EINVAL;
    }
    if (!lat->dcells64) {
        set_error("lattice has no dense float64 slice grid (site box above FR_DENSE64_MAX_CELLS)");
        return FR_ECAPACITY;
    }
    if (cfg->max_em_iters < 1 || cfg->max_gn_iters < 0 || cfg->max_halvings < 0) {
        set_error("invalid iteration limits");
        return FR_EINVAL;
    }
    fr_em64pl *em = new fr_em64pl();
    em->stream = s;
    em->lat = lat;
    em->m = m;
    em->max_iters = cfg->max_em_iters;
    em->cp = cfg->c_prime;
    em->n_tiles = (m + kPlThreads - 1) / kPlThreads;
    em->grid = (int)std::min<long long>(pl_grid(), em->n_tiles);
    EmPlDev h;
    memset(&h, 0, sizeof(h));
    for (int q = 0; q < 9; ++q) h.R[q] = cfg->R0[q];
    for (int i = 0; i < 3; ++i) {
        h.t[i] = cfg->t0[i];
        h.c_ref[i] = cfg->c_ref[i];
    }
    h.diameter = cfg->diameter;
    h.tol = cfg->twist_tolerance;
    h.use_damping = cfg->damping >= 0.0;
    h.damping = cfg->damping;
    h.step_tol = cfg->step_tolerance;
    h.degenerate_mass = cfg->degenerate_mass;
    h.max_em_iters = cfg->max_em_iters;
    h.max_gn_iters = cfg->max_gn_iters;
    h.max_halvings = cfg->max_halvings;
    const long long m_pad = em->n_tiles * kPlThreads;
    if (cudaMallocAsync((void **)&em->d_em, sizeof(EmPlDev), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_sums, kE64Row * sizeof(double), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_partials,
                        (size_t)2 * kE64MaxSms * kPlMinB * kE64Row * sizeof(double), s) !=
            cudaSuccess ||
        cudaMallocAsync((void **)&em->d_traces, (size_t)3 * cfg->max_em_iters * sizeof(double), s) !=
            cudaSuccess ||
        cudaMallocAsync((void **)&em->d_sync, 2 * sizeof(unsigned), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_tiles, (size_t)m_pad * 3 * sizeof(double), s) !=
            cudaSuccess ||
        cudaMallocAsync((void **)&em->d_spec, (size_t)m_pad * kPlSpec * sizeof(double), s) !=
            cudaSuccess ||
        cudaMemcpyAsync(em->d_em, &h, sizeof(EmPlDev), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemsetAsync(em->d_sums, 0, kE64Row * sizeof(double), s) != cudaSuccess ||
        cudaMemsetAsync(em->d_traces, 0, (size_t)3 * cfg->max_em_iters * sizeof(double), s) !=
            cudaSuccess) {
        fr_em64pl_destroy(em);
        set_error("float64 point-to-plane EM allocation failed");
        return FR_ECUDA;
    }
    k_pl_tiles<<<(unsigned)((m_pad + 255) / 256), 256, 0, s>>>(
        ref, m, cfg->c_ref[0], cfg->c_ref[1], cfg->c_ref[2], kPlThreads, em->n_tiles, em->d_tiles);
    if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(s) != cudaSuccess) {
        fr_em64pl_destroy(em);
        set_error("float64 point-to-plane EM tile copy failed");
        return FR_ECUDA;
    }
    *out = em;
    return FR_OK;
}

int fr_em64pl_destroy(fr_em64pl *em) {
    if (!em) return FR_OK;
    cudaStreamSynchronize(em->stream);
    for (void *p : {(void *)em->d_em, (void *)em->d_sums, (void *)em->d_partials,
                    (void *)em->d_traces, (void *)em->d_sync, (void *)em->d_tiles,
                    (void *)em->d_spec})
        if (p) cudaFreeAsync(p, em->stream);
    delete em;
    return FR_OK;
}

int fr_em64pl_run(fr_em64pl *em, int n_iters, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    em->stream = s;
    Em64PlArgs a;
    a.tiles = em->d_tiles;
    a.m = em->m;
    a.m_pad = em->n_tiles * kPlThreads;
    a.tiles_per_cta = (int)((em->n_tiles + em->grid - 1) / em->grid);
    a.g = em->lat->dense64;
    a.em = em->d_em;
    a.spec = em->d_spec;
    a.partials = em->d_partials;
    a.sums = em->d_sums;
    a.traces = em->d_traces;
    a.counter = em->d_sync;
    a.n_iters = n_iters > 0 ? n_iters : em->max_iters;
    for (int j = 0; j < 3; ++j) a.sc[j] = em->lat->c.sf[j] / em->lat->c.sigma[j];
    a.cp = em->cp;
    FR_CUDA(cudaMemsetAsync(em->d_sync, 0, 2 * sizeof(unsigned), s));
    void *args[] = {&a};
    FR_CUDA(cudaLaunchCooperativeKernel((const void *)k_em64pl<kPlThreads, kPlMinB>,
                                        dim3(em->grid), dim3(kPlThreads), args, 0, s));
    return FR_OK;
}

int fr_em64pl_launch_info(const fr_em64pl *em, int *grid, int *block) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    if (grid) *grid = em->grid;
    if (block) *block = kPlThreads;
    return FR_OK;
}

int fr_em64pl_sums(fr_em64pl *em, double **d_sums, int *width) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    if (d_sums) *d_sums = em->d_sums;
    if (width) *width = kPlStats;
    return FR_OK;
}

int fr_em64pl_status(fr_em64pl *em, int *done, int *iterations, int *termination, void *stream) {
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

int fr_em64pl_result(fr_em64pl *em, double *R, double *t, double *objectives,
                     double *twist_norms, double *inlier_masses, int *iterations,
                     int *termination, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    EmPlDev h;
    FR_CUDA(cudaMemcpyAsync(&h, em->d_em, sizeof(EmPlDev), cudaMemcpyDeviceToHost, s));
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
