// The float64 rigid point-to-point EM loop on B200 (the reference's arithmetic:
// every operation on the query path is float64, as twistreg's NumPy code).
//
// One cooperative, grid-resident kernel runs a whole registration:
//
//   per EM iteration (pipeline.py:141-177)
//     every CTA   sweeps its contiguous slice of the Morton-ordered model
//                 points (float64 SoA planes, the caller's values bit for
//                 bit): forward map x = R (x_ref - c_ref) + c_world
//                 (kinematics.py:317-320), elevation and enclosing simplex
//                 (permutohedral.py:171-215: remainder-0 point, stable
//                 descending ranks, single wrap, barycentrics), slice over the
//                 dense float64 grid (permutohedral.py:329-341: four 32-byte
//                 rows, index arithmetic instead of hashing), the moments
//                 epilogue (estep.py:195-205: m0 clamp, w = m0 / (m0 + c'),
//                 target = m1 / m0) and the 25 point-to-point sufficient
//                 statistics of the M step (mstep.py:102-210), accumulated in
//                 float64 registers;
//     block       warp reduce-scatter (31 shuffles for 25 columns) + a fixed-
//                 order sum over the warps -> one row of partials;
//     grid        one arrival barrier (monotone counter, release / acquire);
//                 then EVERY CTA sums the rows in the same fixed order and
//                 runs the same float64 solve (fr_solve.cuh: normal
//                 equations, damped Cholesky with tenfold escalation, step
//                 halving with closed-form candidate objectives, twist update,
//                 update magnitude, termination) on its shared-memory copy of
//                 the state -- bit-identical in every CTA, so no broadcast.
//
// No launches, host polls or graph replays between iterations; all sums are
// formed in a fixed order, so reruns are bit-identical.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fr_common.cuh"
#include "fr_reduce.cuh"
#include "fr_solve.cuh"
#include "fr_em64.cuh"

namespace fr {

constexpr int kE64Stats = 25;        // point-to-point sufficient statistics (_rigid.py)

struct Em64Args {
    const double *tiles; // [n_tiles][3][T] centred model points (Morton order), T = threads
    long long m;
    int tiles_per_cta;   // contiguous tiles per CTA
    DenseSliceD g;
    EmDev *em;           // state; em->k holds the current pass constants
    double *partials;    // [gridDim.x][kE64Row]
    double *sums;        // [kE64Row] the last pass's reduced statistics
    double *traces;      // [4][max_iters]: objectives, update magnitudes, masses, cos(angle)
    unsigned *counter;   // arrivals of the current iteration
    unsigned *gen;       // release generation
    int n_iters;         // iterations of this launch (or fewer: termination)
    int solve;           // 0: pass + reduction only; 1: + the solve (unsharded loop);
                         // 2: solve the pending all-reduced sums first (sharded)
    unsigned long long *prof;   // optional phase timestamps [n_iters][8] (FR_EM64_PROFILE)
    // pose-independent constants (kernel parameters: constant-bank operands)
    double sc[3];        // sf_j / sigma_j: f = x * sc (permutohedral.py:172)
    double cp;           // outlier constant c' (estep.py:99-112)
};



// the record (w, r, x - c_world) of one model point: forward map, simplex,
// slice, epilogue.  (h0, h1, h2) = x_ref - c_ref (the centred tile); valid = 0
// for the padding of the last tile (computed, contributes nothing: no branch).
// Moments epilogue (estep.py:195-205): m0 = max(out0, 0), supported iff
// m0 >= 1e-12, w = m0 / (m0 + c'), target = m1 / m0; unsupported points get
// w = 0 and target = x (zero residual).  One reciprocal: q = 1 / (m0 (m0 + c')),
// 1 / m0 = (m0 + c') q, w = m0^2 q.
__device__ __forceinline__ void e64_record(const Em64Args &a, const Pose64 &k, double cp,
                                           double h0, double h1, double h2, bool valid,
                                           double &w, double (&r)[3], double (&xt)[3]) {
    const DenseSliceD &g = a.g;
    double X[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        xt[i] = fma(k.R[3 * i + 2], h2, fma(k.R[3 * i + 1], h1, k.R[3 * i] * h0));
        X[i] = xt[i] + k.cw[i];
    }
    Simplex64 S;
    e64_simplex(g, a.sc, X, S);
    double o[4];
    e64_gather<2>(g, S, o);
    const double m0 = o[3] > 0.0 ? o[3] : 0.0;
    const bool sup = m0 >= 1e-12 && S.in_range && valid;
    const double den = m0 + cp;
    const double q = rcp64(m0 * den);
    const double inv = den * q;
    w = sup ? (cp > 0.0 ? (m0 * m0) * q : 1.0) : 0.0;
    r[0] = sup ? fma(-o[0], inv, X[0]) : 0.0;
    r[1] = sup ? fma(-o[1], inv, X[1]) : 0.0;
    r[2] = sup ? fma(-o[2], inv, X[2]) : 0.0;
}

// the 25 point-to-point sufficient statistics of one record, about c_world
// (layout: _rigid.py)
__device__ __forceinline__ void e64_accumulate(double w, const double (&r)[3],
                                               const double (&xt)[3],
                                               double (&acc)[kE64Stats]) {
    double wy[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) wy[j] = w * xt[j];
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
        for (int q2 = 0; q2 < 3; ++q2) acc[13 + 3 * j + q2] = fma(wr, xt[q2], acc[13 + 3 * j + q2]);
        acc[22 + j] = fma(wr, r[j], acc[22 + j]);
    }
}

// one model point: its record, then its statistics
__device__ __forceinline__ void e64_point(const Em64Args &a, const Pose64 &k, double cp,
                                          double h0, double h1, double h2, bool valid,
                                          double (&acc)[kE64Stats]) {
    double w, r[3], xt[3];
    e64_record(a, k, cp, h0, h1, h2, valid, w, r, xt);
    e64_accumulate(w, r, xt, acc);
}

// One CTA of the grid-resident loop.  Every CTA keeps the EM state (EmDev)
// in shared memory and runs the SAME fixed-order reduction and float64 solve
// on the same partial rows, so all CTAs hold bit-identical poses without a
// broadcast: an iteration costs one arrival barrier (monotone counter,
// release/acquire) and one read of the partial rows -- no release hop, no
// state round trip through global memory.  Partial rows are double-buffered
// by iteration parity (a CTA can only reuse a buffer after every CTA passed
// the next barrier, i.e. finished reading it).  The CTA's tiles stream
// through an S-stage TMA ring that runs ahead across iteration boundaries
// (the points do not depend on the pose), so the next iteration's first
// tiles land during the barrier and the solve.
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#ifndef FR_EM64_PTS
#define FR_EM64_PTS 2
#endif
constexpr int kEmPts = FR_EM64_PTS;     // points per thread and step (256-thread variant)

template <int THREADS, int MINB, int S>
__device__ __forceinline__ void em64_cta(const Em64Args &a) {
    // S > 0: warp W produces tiles into an S-stage TMA ring; S == 0: every
    // thread prefetches its next point into registers (plain loads)
    constexpr int W = THREADS / 32;          // consumer warps
    constexpr int NT = THREADS + (S ? 32 : 0);
    constexpr int SS = S ? S : 1;
    constexpr unsigned kTileBytes = 3u * THREADS * sizeof(double);
    extern __shared__ __align__(128) double ring[];          // [S][3][THREADS]
    __shared__ double red[W][32];
    __shared__ double tsum[kE64Row];
    __shared__ EmDev se;
    __shared__ __align__(8) unsigned long long full[SS], empty[SS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = S && warp == W;
    const int nb = (int)gridDim.x;
    const long long t0 = (long long)blockIdx.x * a.tiles_per_cta;
    const long long n_tiles_all = (a.m + THREADS - 1) / THREADS;
    const int nt = (int)max(0LL, min((long long)a.tiles_per_cta, n_tiles_all - t0));
    const double cp = a.cp;
    copy_cg(&se, a.em, tid, NT);
    // the state's iteration count at entry (shared: a register live across
    // the whole loop would be spilled)
    __shared__ int it0;
    if (tid == 0) it0 = __ldcg(&a.em->iterations);
    if (S && tid == 0) {
        for (int q = 0; q < S; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], W);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // tile sequence k = 0, 1, ... walks this CTA's tiles cyclically (iteration
    // k / nt, tile k % nt) through stage k % S; the producer keeps S tiles in
    // flight, across iteration boundaries (the points do not depend on the pose)
    const unsigned n_total = (unsigned)nt * (unsigned)a.n_iters;
    unsigned issued = 0;                     // producer lane 0 only
    auto produce_until = [&](unsigned upto) {
        for (; issued < upto && issued < n_total; ++issued) {
            const unsigned st = issued % SS;
            if (issued >= (unsigned)SS) mbar_wait(&empty[st], ((issued / SS) + 1) & 1);
            bulk_load(ring + st * 3 * THREADS, a.tiles + (t0 + issued % nt) * 3 * THREADS,
                      kTileBytes, &full[st]);
        }
    };
    if (producer && lane == 0) produce_until(SS);
    unsigned n = 0;                          // consumed tiles (uniform)
    int it = 0;
    constexpr bool kInlineSolve = MINB == 1 && THREADS <= 256;
    // ONE solve site at the top of the loop (a second inlined copy of the
    // serial solve costs the pass its registers): solve == 1 solves the
    // previous iteration's reduced sums (tsum) there, one trip past the last
    // pass; solve == 2 (sharded, fused: one pass per launch) the previous
    // launch's sums, all-reduced across ranks between the launches, then runs
    // this launch's pass
    for (;; ++it) {
        const bool solve_now = a.solve == 1 ? it > 0 : (a.solve == 2 && it == 0 && se.pending);
        if (solve_now) {
            if (a.solve == 2 && tid < kE64Stats) tsum[tid] = __ldcg(a.sums + tid);
            __syncthreads();
            if (tid == 0) {
                const int n = se.max_em_iters;
                unsigned long long *st =
                    a.prof && blockIdx.x == 0 && a.solve == 1 ? a.prof + 8 * (it - 1) + 5 : nullptr;
                se.pending = 0;
                if (kInlineSolve)   // 255 registers: the lean solve inlined
                    rigid_solve_impl<true>(tsum, &se, a.traces, a.traces + n, a.traces + 2 * n,
                                           blockIdx.x == 0, st, a.traces + 3 * n);
                else
                    rigid_solve_body(tsum, &se, a.traces, a.traces + n, a.traces + 2 * n,
                                     blockIdx.x == 0, st);
                if (st) a.prof[8 * (it - 1) + 4] = gtime();
            }
            __syncthreads();
        }
        // identical in every CTA; a pass-only launch after termination is a
        // no-op too (the sharded loop's replayed chunks run past the end)
        if (it >= a.n_iters || se.done) break;
        if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[8 * it + 0] = gtime();
        double acc[kE64Stats];
#pragma unroll
        for (int q = 0; q < kE64Stats; ++q) acc[q] = 0.0;
        if (producer) {
            if (lane == 0) produce_until(n + nt + SS);
            n += nt;
        } else {
            Pose64 pose;
#pragma unroll
            for (int q = 0; q < 9; ++q) pose.R[q] = se.k.R[q];
#pragma unroll
            for (int q = 0; q < 3; ++q) pose.cw[q] = se.k.c_world[q];
            // contiguous tiles per CTA (Morton order: the CTA's grid rows stay
            // in L1), one point per consumer thread and tile
            const double *src = a.tiles + t0 * 3 * THREADS + tid;
            long long pidx = t0 * THREADS + tid;
            if (S) {
                // a warp frees a stage as soon as its 32 lanes read it
                for (int tt = 0; tt < nt; ++tt, ++n, pidx += THREADS) {
                    const unsigned st = n % SS;
                    mbar_wait(&full[st], (n / SS) & 1);
                    const double *tile = ring + st * 3 * THREADS;
                    const double h0 = tile[tid], h1 = tile[THREADS + tid], h2 = tile[2 * THREADS + tid];
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[st]);
                    e64_point(a, pose, cp, h0, h1, h2, pidx < a.m, acc);
                }
            } else if (THREADS <= 256) {
                // kEmPts tiles per step: independent point chains in one basic
                // block for the scheduler to interleave (the pass is FP64-
                // latency bound at 8 warps per SM); the next group is
                // prefetched into registers
                constexpr int P = kEmPts;
                double nx[P], ny[P], nz[P];
#pragma unroll
                for (int u = 0; u < P; ++u) {
                    nx[u] = ny[u] = nz[u] = 0.0;
                    if (u < nt) {
                        nx[u] = __ldg(src + u * 3 * THREADS);
                        ny[u] = __ldg(src + u * 3 * THREADS + THREADS);
                        nz[u] = __ldg(src + u * 3 * THREADS + 2 * THREADS);
                    }
                }
                int tt = 0;
                for (; tt + P - 1 < nt; tt += P, pidx += P * THREADS) {
                    double hx[P], hy[P], hz[P];
#pragma unroll
                    for (int u = 0; u < P; ++u) {
                        hx[u] = nx[u];
                        hy[u] = ny[u];
                        hz[u] = nz[u];
                    }
                    src += 3 * P * THREADS;
#pragma unroll
                    for (int u = 0; u < P; ++u)
                        if (tt + P + u < nt) {
                            nx[u] = __ldg(src + u * 3 * THREADS);
                            ny[u] = __ldg(src + u * 3 * THREADS + THREADS);
                            nz[u] = __ldg(src + u * 3 * THREADS + 2 * THREADS);
                        }
#pragma unroll
                    for (int u = 0; u < P; ++u)
                        e64_point(a, pose, cp, hx[u], hy[u], hz[u], pidx + u * THREADS < a.m, acc);
                }
#pragma unroll
                for (int u = 0; u < P - 1; ++u)
                    if (tt + u < nt)
                        e64_point(a, pose, cp, nx[u], ny[u], nz[u], pidx + u * THREADS < a.m, acc);
                n += nt;
            } else {
                double nx = 0.0, ny = 0.0, nz = 0.0;
                if (nt > 0) {
                    nx = __ldg(src);
                    ny = __ldg(src + THREADS);
                    nz = __ldg(src + 2 * THREADS);
                }
                for (int tt = 0; tt < nt; ++tt, pidx += THREADS) {
                    const double h0 = nx, h1 = ny, h2 = nz;
                    if (tt + 1 < nt) {
                        src += 3 * THREADS;
                        nx = __ldg(src);
                        ny = __ldg(src + THREADS);
                        nz = __ldg(src + 2 * THREADS);
                    }
                    e64_point(a, pose, cp, h0, h1, h2, pidx < a.m, acc);
                }
                n += nt;
            }
        }
        if (!producer) red[warp][lane] = warp_reduce_scatter(acc);
        __syncthreads();
        double *rows = a.partials + (long long)(it & 1) * nb * kE64Row;
        if (tid < kE64Stats) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < W; ++w) s += red[w][tid];
            rows[(long long)blockIdx.x * kE64Row + tid] = s;
            __threadfence();             // the row before this CTA's arrival
        }
        __syncthreads();
        if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[8 * it + 1] = gtime();
        if (tid == 0) {
            const unsigned target = (unsigned)nb * (unsigned)(it + 1);
            atomicAdd(a.counter, 1u);
            while (ld_acquire(a.counter) < target) __nanosleep(20);
        }
        __syncthreads();
        if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[8 * it + 2] = gtime();
        if (a.solve == 2 && tid == 0) se.pending = 1;     // solved by the next launch
        if (a.solve != 1 && blockIdx.x != 0) continue;
        // fixed-order column sums: thread (g, c) adds the rows g, g + W, ...
        // of column c with every load issued up front (one L2 round trip),
        // then the W group sums in order -- the same order in every CTA
        {
            const int c = lane, grp = warp;
            double s = 0.0;
            if (!producer && c < kE64Stats) {
                constexpr int kMaxRows = (kE64MaxSms * MINB + W - 1) / W;
                double r[kMaxRows];
#pragma unroll
                for (int u = 0; u < kMaxRows; ++u) {
                    const int b = grp + W * u;
                    r[u] = b < nb ? __ldcg(rows + (long long)b * kE64Row + c) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kMaxRows; ++u) s += r[u];
            }
            __syncthreads();             // red[] reuse
            if (!producer) red[grp][c] = s;
        }
        __syncthreads();
        if (tid < kE64Stats) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < W; ++j) s += red[j][tid];
            tsum[tid] = s;
            if (blockIdx.x == 0) a.sums[tid] = s;
        }
        __syncthreads();
        if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[8 * it + 3] = gtime();
    }
    // the deferred update magnitudes of this launch's iterations (lean solve)
    if (kInlineSolve && a.solve && blockIdx.x == 0)
        rigid_finish_tnorms(a.traces + se.max_em_iters, a.traces + 3 * se.max_em_iters, it0,
                            se.iterations, se.diameter);
    // no bulk copy may still target this CTA's shared memory when it exits
    if (producer && lane == 0)
        for (; n < issued; ++n) mbar_wait(&full[n % SS], (n / SS) & 1);
    // the state after the last iteration (status / result / a later launch)
    if (blockIdx.x == 0 && a.solve) {
        const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&se);
        for (int q = tid; q < (int)(sizeof(EmDev) / 8); q += NT)
            reinterpret_cast<unsigned long long *>(a.em)[q] = src[q];
    }
}

// ---------------------------------------------------------------------------
// Warp-specialised CTA (FR_EM64_VARIANT=4): 384 threads.  Warpgroups 0-1 (256
// "record" threads, setmaxnreg 208) run the forward map, simplex, gather and
// epilogue of P points per step and hand each point's record (w, r, x -
// c_world: 7 doubles) to warpgroup 2 (128 "statistics" threads, setmaxnreg
// 88) through a 2-stage shared-memory ring (named barriers: full = records
// written, empty = records consumed); the statistics threads hold the 25
// accumulators, so the record side keeps its registers for P independent
// point chains.  Reduction, grid barrier and solve as in em64_cta.
constexpr int kWsE = 256, kWsM = 128, kWsThreads = kWsE + kWsM;
constexpr int kWsRec = 7, kWsStages = 2;

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct WsShared {
    double red[kWsThreads / 32][32];
    double tsum[kE64Row];
    EmDev se;
    int it0;
};

// the whole loop of one role (kStat: the statistics warpgroup), so each
// role's code sits after its own setmaxnreg; both roles pass the same
// sequence of CTA barriers
template <int P, bool kStat>
__device__ __forceinline__ void em64_ws_loop(const Em64Args &a, WsShared &sh, double *ring) {
    constexpr int NT = kWsThreads, W = NT / 32, WM = kWsM / 32;
    EmDev &se = sh.se;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = (int)gridDim.x;
    const long long t0 = (long long)blockIdx.x * a.tiles_per_cta;
    const long long n_tiles_all = (a.m + kWsE - 1) / kWsE;
    const int nt = (int)max(0LL, min((long long)a.tiles_per_cta, n_tiles_all - t0));
    const int steps = (nt + P - 1) / P;
    const double cp = a.cp;
    int it = 0;
    for (;; ++it) {
        const bool solve_now = a.solve == 1 ? it > 0 : (a.solve == 2 && it == 0 && se.pending);
        if (solve_now) {
            if (a.solve == 2 && tid < kE64Stats) sh.tsum[tid] = __ldcg(a.sums + tid);
            __syncthreads();
            if (!kStat && tid == 0) {
                const int n = se.max_em_iters;
                unsigned long long *st =
                    a.prof && blockIdx.x == 0 && a.solve == 1 ? a.prof + 8 * (it - 1) + 5 : nullptr;
                se.pending = 0;
                rigid_solve_impl<true>(sh.tsum, &se, a.traces, a.traces + n, a.traces + 2 * n,
                                       blockIdx.x == 0, st, a.traces + 3 * n);
                if (st) a.prof[8 * (it - 1) + 4] = gtime();
            }
            __syncthreads();
        }
        if (it >= a.n_iters || se.done) break;
        if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[8 * it + 0] = gtime();
        if constexpr (!kStat) {
            Pose64 pose;
#pragma unroll
            for (int q = 0; q < 9; ++q) pose.R[q] = se.k.R[q];
#pragma unroll
            for (int q = 0; q < 3; ++q) pose.cw[q] = se.k.c_world[q];
            const double *src = a.tiles + t0 * 3 * kWsE + tid;
            long long pidx = t0 * kWsE + tid;
            double nx[P], ny[P], nz[P];
#pragma unroll
            for (int u = 0; u < P; ++u) {
                nx[u] = ny[u] = nz[u] = 0.0;
                if (u < nt) {
                    nx[u] = __ldg(src + u * 3 * kWsE);
                    ny[u] = __ldg(src + u * 3 * kWsE + kWsE);
                    nz[u] = __ldg(src + u * 3 * kWsE + 2 * kWsE);
                }
            }
            for (int st = 0; st < steps; ++st, pidx += P * kWsE) {
                double hx[P], hy[P], hz[P];
#pragma unroll
                for (int u = 0; u < P; ++u) {
                    hx[u] = nx[u];
                    hy[u] = ny[u];
                    hz[u] = nz[u];
                }
                src += 3 * P * kWsE;
#pragma unroll
                for (int u = 0; u < P; ++u)
                    if ((st + 1) * P + u < nt) {
                        nx[u] = __ldg(src + u * 3 * kWsE);
                        ny[u] = __ldg(src + u * 3 * kWsE + kWsE);
                        nz[u] = __ldg(src + u * 3 * kWsE + 2 * kWsE);
                    }
                const int stage = st & 1;
                if (st >= kWsStages) named_sync(3 + stage, NT);      // records consumed
                double *slot = ring + (size_t)stage * P * kWsRec * kWsE + tid;
#pragma unroll
                for (int u = 0; u < P; ++u) {
                    double w, r[3], xt[3];
                    const bool valid = st * P + u < nt && pidx + u * kWsE < a.m;
                    e64_record(a, pose, cp, hx[u], hy[u], hz[u], valid, w, r, xt);
                    double *rec = slot + u * kWsRec * kWsE;
                    rec[0] = w;
                    rec[kWsE] = r[0];
                    rec[2 * kWsE] = r[1];
                    rec[3 * kWsE] = r[2];
                    rec[4 * kWsE] = xt[0];
                    rec[5 * kWsE] = xt[1];
                    rec[6 * kWsE] = xt[2];
                }
                named_arrive(1 + stage, NT);                        // records written
            }
            // balance the empty barrier: one wait per consumed stage
            for (int st = max(steps - kWsStages, 0); st < steps; ++st) named_sync(3 + (st & 1), NT);
        } else {
            double acc[kE64Stats];
#pragma unroll
            for (int q = 0; q < kE64Stats; ++q) acc[q] = 0.0;
            const int mt = tid - kWsE;
            for (int st = 0; st < steps; ++st) {
                const int stage = st & 1;
                named_sync(1 + stage, NT);
                const double *slot = ring + (size_t)stage * P * kWsRec * kWsE + mt;
#pragma unroll
                for (int u = 0; u < P; ++u)
#pragma unroll
                    for (int hh = 0; hh < kWsE / kWsM; ++hh) {
                        const double *rec = slot + u * kWsRec * kWsE + hh * kWsM;
                        const double r[3] = {rec[kWsE], rec[2 * kWsE], rec[3 * kWsE]};
                        const double xt[3] = {rec[4 * kWsE], rec[5 * kWsE], rec[6 * kWsE]};
                        e64_accumulate(rec[0], r, xt, acc);
                    }
                named_arrive(3 + stage, NT);
            }
            sh.red[warp - kWsE / 32][lane] = warp_reduce_scatter(acc);
        }
        __syncthreads();
        double *rows = a.partials + (long long)(it & 1) * nb * kE64Row;
        if (tid < kE64Stats) {
            double s = 0.0;
#pragma unroll
            for (int w = 0; w < WM; ++w) s += sh.red[w][tid];
            rows[(long long)blockIdx.x * kE64Row + tid] = s;
            __threadfence();             // the row before this CTA's arrival
        }
        __syncthreads();
        if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[8 * it + 1] = gtime();
        if (tid == 0) {
            const unsigned target = (unsigned)nb * (unsigned)(it + 1);
            atomicAdd(a.counter, 1u);
            while (ld_acquire(a.counter) < target) __nanosleep(20);
        }
        __syncthreads();
        if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[8 * it + 2] = gtime();
        if (a.solve == 2 && tid == 0) se.pending = 1;     // solved by the next launch
        if (a.solve != 1 && blockIdx.x != 0) continue;
        {
            const int c = lane, grp = warp;
            double s = 0.0;
            if (c < kE64Stats) {
                constexpr int kMaxRows = (kE64MaxSms + W - 1) / W;
                double r[kMaxRows];
#pragma unroll
                for (int u = 0; u < kMaxRows; ++u) {
                    const int b = grp + W * u;
                    r[u] = b < nb ? __ldcg(rows + (long long)b * kE64Row + c) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < kMaxRows; ++u) s += r[u];
            }
            __syncthreads();             // red[] reuse
            sh.red[grp][c] = s;
        }
        __syncthreads();
        if (tid < kE64Stats) {
            double s = 0.0;
#pragma unroll
            for (int j = 0; j < W; ++j) s += sh.red[j][tid];
            sh.tsum[tid] = s;
            if (blockIdx.x == 0) a.sums[tid] = s;
        }
        __syncthreads();
        if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[8 * it + 3] = gtime();
    }
}

template <int P>
__device__ __forceinline__ void em64_cta_ws(const Em64Args &a) {
    extern __shared__ __align__(128) double ring[];     // [kWsStages][P][kWsRec][kWsE]
    __shared__ WsShared sh;
    const int tid = threadIdx.x;
    copy_cg(&sh.se, a.em, tid, kWsThreads);
    if (tid == 0) sh.it0 = __ldcg(&a.em->iterations);
    __syncthreads();
    if (tid >= kWsE) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;" ::: "memory");
        em64_ws_loop<P, true>(a, sh, ring);
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory");
        em64_ws_loop<P, false>(a, sh, ring);
    }
    __syncthreads();
    if (a.solve && blockIdx.x == 0)
        rigid_finish_tnorms(a.traces + sh.se.max_em_iters, a.traces + 3 * sh.se.max_em_iters,
                            sh.it0, sh.se.iterations, sh.se.diameter);
    if (blockIdx.x == 0 && a.solve) {
        const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&sh.se);
        for (int q = tid; q < (int)(sizeof(EmDev) / 8); q += kWsThreads)
            reinterpret_cast<unsigned long long *>(a.em)[q] = src[q];
    }
}

#ifndef FR_EM64_WS_PTS
#define FR_EM64_WS_PTS 2
#endif

template <bool BATCH>
__global__ void __launch_bounds__(kWsThreads, 1)
k_em64_ws(Em64Args a0, const Em64Args *__restrict__ batch) {
    if constexpr (BATCH) {
        const Em64Args &a = batch[blockIdx.y];
        em64_cta_ws<FR_EM64_WS_PTS>(a);
    } else {
        em64_cta_ws<FR_EM64_WS_PTS>(a0);
    }
}

// the kernel: one problem (parameters by value: constant-bank operands), or a
// batch of independent problems, blockIdx.y = problem (replicas, no
// collectives; every problem has its own state, partial rows and counter)
template <int THREADS, int MINB, int S, bool BATCH>
__global__ void __launch_bounds__(THREADS + (S ? 32 : 0), MINB)
k_em64(Em64Args a0, const Em64Args *__restrict__ batch) {
    if constexpr (BATCH) {
        // a reference (L1-cached loads), not a copy: a local struct copy
        // would live in local memory
        const Em64Args &a = batch[blockIdx.y];
        em64_cta<THREADS, MINB, S>(a);
    } else {
        em64_cta<THREADS, MINB, S>(a0);
    }
}

// the solve alone (sharded runs: after the all-reduce of the pass sums)
__global__ void k_em64_solve(const double *sums, EmDev *e, double *traces) {
    __shared__ EmDev se;
    __shared__ double ts[kE64Row];
    if (e->done) return;
    copy_cg(&se, e, threadIdx.x, blockDim.x);
    if (threadIdx.x < kE64Stats) ts[threadIdx.x] = sums[threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) {
        const int n = se.max_em_iters;
        se.pending = 0;
        rigid_solve_body(ts, &se, traces, traces + n, traces + 2 * n, true);
    }
    __syncthreads();
    const unsigned long long *src = reinterpret_cast<const unsigned long long *>(&se);
    for (int q = threadIdx.x; q < (int)(sizeof(EmDev) / 8); q += blockDim.x)
        reinterpret_cast<unsigned long long *>(e)[q] = src[q];
}

// launch variants (FR_EM64_VARIANT): 4 = warp-specialised (em64_cta_ws: 256
// record threads at 208 registers + 128 statistics threads at 88, setmaxnreg;
// measured at 1M: pass 17.7 / 18.6 / 17.8 us with 2 / 3 / 4 points per record
// thread vs 16.0-16.4 for variant 0 -- the ring's stores and barriers cost
// more than the freed registers buy); 0 (default) = 256 threads x 1 CTA/SM, 255
// registers (no spills, the solve inlined), two points per thread and step
// with the next pair prefetched into registers; 2 = 512 x 1 with one point
// per step (128 registers: 116 B of spills; 10-20% slower per iteration);
// 1 = 384 x 1 with an 8-stage TMA bulk-copy ring fed by a producer warp
// (slower still: the pass is issue / FP64-latency bound, not stream bound;
// DESIGN.md)
using E64Kernel = void (*)(Em64Args, const Em64Args *);
struct E64Variant {
    E64Kernel fn, batch;
    int threads, minb, stages;
    int ws = 0;              // warp-specialised (threads = record side; + kWsM statistics threads)
    int block() const { return threads + (stages ? 32 : 0) + (ws ? kWsM : 0); }
    size_t smem() const {
        return ws ? (size_t)kWsStages * FR_EM64_WS_PTS * kWsRec * kWsE * sizeof(double)
                  : (size_t)stages * 3 * threads * sizeof(double);
    }
};

static E64Variant e64_variant() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("FR_EM64_VARIANT");
        v = e ? atoi(e) : 0;
    }
    if (v == 1) return {k_em64<384, 1, 8, false>, k_em64<384, 1, 8, true>, 384, 1, 8};
    if (v == 2) return {k_em64<512, 1, 0, false>, k_em64<512, 1, 0, true>, 512, 1, 0};
    if (v == 4) return {k_em64_ws<false>, k_em64_ws<true>, kWsE, 1, 0, 1};
    return {k_em64<256, 1, 0, false>, k_em64<256, 1, 0, true>, 256, 1, 0};
}

static int e64_grid(const E64Variant &k) {
    // once per device (attribute + occupancy queries cost ~10 us a call)
    static int cached[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && cached[dev] > 0) return cached[dev];
    cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem());
    cudaFuncSetAttribute(k.batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem());
    int per = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k.fn, k.block(), k.smem()) !=
            cudaSuccess || per < 1)
        per = 1;
    const int g = std::min(per, k.minb) * std::min(sm_count(), kE64MaxSms);
    if (dev >= 0 && dev < 64) cached[dev] = g;
    return g;
}

// centred point tiles: tiles[t][c][j] = ref[c][t T + j] - c_ref[c] (zero past m)
__global__ void k_em64_tiles(const double *ref, long long m, double c0, double c1, double c2,
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

// the float64 device EM object behind fr_em64*
struct fr_em64 {
    const fr_lattice *lat = nullptr;
    long long m = 0;
    int max_iters = 0;
    int grid = 0;
    int threads = 0;
    int block = 0;
    size_t smem = 0;
    long long n_tiles = 0;
    double *d_tiles = nullptr;       // centred [n_tiles][3][threads] copy of the model points
    fr::E64Kernel fn = nullptr, batch_fn = nullptr;
    fr::EmDev *d_em = nullptr;
    double *d_sums = nullptr;
    double *d_partials = nullptr;
    double *d_traces = nullptr;
    unsigned *d_sync = nullptr;      // [0] counter, [1] generation
    cudaStream_t stream = nullptr;
    unsigned long long *d_prof = nullptr;   // FR_EM64_PROFILE=1: phase timestamps
    double cp = 0.0;
};

using namespace fr;

static Em64Args e64_args(fr_em64 *em, int n_iters, int solve, int grid) {
    Em64Args a;
    a.tiles = em->d_tiles;
    a.m = em->m;
    a.tiles_per_cta = (int)((em->n_tiles + grid - 1) / grid);
    a.g = em->lat->dense64;
    a.em = em->d_em;
    a.partials = em->d_partials;
    a.sums = em->d_sums;
    a.traces = em->d_traces;
    a.counter = em->d_sync;
    a.gen = em->d_sync + 1;
    a.n_iters = n_iters;
    a.solve = solve;
    a.prof = em->d_prof;
    for (int j = 0; j < 3; ++j) a.sc[j] = em->lat->c.sf[j] / em->lat->c.sigma[j];
    a.cp = em->cp;
    return a;
}

static int e64_launch(fr_em64 *em, int n_iters, int solve, cudaStream_t s) {
    Em64Args a = e64_args(em, n_iters, solve, em->grid);
    const Em64Args *none = nullptr;
    FR_CUDA(cudaMemsetAsync(em->d_sync, 0, 2 * sizeof(unsigned), s));
    void *args[] = {&a, &none};
    FR_CUDA(cudaLaunchCooperativeKernel((const void *)em->fn, dim3(em->grid), dim3(em->block),
                                        args, em->smem, s));
    return FR_OK;
}

extern "C" {

int fr_em64_create(const fr_lattice *lat, const double *ref, int64_t m,
                   const fr_rigid_em_config *cfg, void *stream, fr_em64 **out) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!lat || !lat->blurred || !ref || !cfg || !out || m <= 0) {
        set_error("invalid float64 EM arguments");
        return FR_EINVAL;
    }
    if (lat->dim != 3 || lat->nv != 4) {
        set_error("the float64 EM loop runs point_to_point with a fixed kernel (4 value columns)");
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
    fr_em64 *em = new fr_em64();
    em->stream = s;
    em->lat = lat;
    em->m = m;
    em->max_iters = cfg->max_em_iters;
    em->cp = cfg->c_prime;
    const E64Variant kv = e64_variant();
    em->fn = kv.fn;
    em->batch_fn = kv.batch;
    em->threads = kv.threads;
    em->block = kv.block();
    em->smem = kv.smem();
    em->n_tiles = (m + kv.threads - 1) / kv.threads;
    // small clouds: no more CTAs than tiles (fewer arrivals per barrier, and
    // the SMs stay free for other problems)
    em->grid = (int)std::min<long long>(e64_grid(kv), em->n_tiles);
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
    h.conv_q = cfg->twist_tolerance * cfg->diameter * (cfg->twist_tolerance * cfg->diameter) *
               (1.0 + 1e-9);
    h.use_damping = cfg->damping >= 0.0;
    h.damping = cfg->damping;
    h.step_tol = cfg->step_tolerance;
    h.degenerate_mass = cfg->degenerate_mass;
    h.max_em_iters = cfg->max_em_iters;
    h.max_gn_iters = cfg->max_gn_iters;
    h.max_halvings = cfg->max_halvings;
    make_rigid_k(h.A, h.R, h.t, h.c_ref, h.cp, h.gain, -1, -1, &h.k);
    if (cudaMallocAsync((void **)&em->d_em, sizeof(EmDev), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_sums, kE64Row * sizeof(double), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_partials,
                        (size_t)2 * kE64MaxSms * kv.minb * kE64Row * sizeof(double), s) !=
            cudaSuccess ||
        cudaMallocAsync((void **)&em->d_traces, (size_t)4 * cfg->max_em_iters * sizeof(double), s) !=
            cudaSuccess ||
        cudaMallocAsync((void **)&em->d_sync, 2 * sizeof(unsigned), s) != cudaSuccess ||
        cudaMemcpyAsync(em->d_em, &h, sizeof(EmDev), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemsetAsync(em->d_sync, 0, 2 * sizeof(unsigned), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_tiles, (size_t)em->n_tiles * 3 * em->threads * sizeof(double),
                        s) != cudaSuccess ||
        cudaMemsetAsync(em->d_sums, 0, kE64Row * sizeof(double), s) != cudaSuccess ||
        (getenv("FR_EM64_PROFILE") && getenv("FR_EM64_PROFILE")[0] == '1' &&
         (cudaMallocAsync((void **)&em->d_prof, (size_t)8 * cfg->max_em_iters * 8, s) != cudaSuccess ||
          cudaMemsetAsync(em->d_prof, 0, (size_t)8 * cfg->max_em_iters * 8, s) != cudaSuccess))) {
        fr_em64_destroy(em);
        set_error("float64 EM allocation failed");
        return FR_ECUDA;
    }
    {
        const long long tot = em->n_tiles * em->threads;
        k_em64_tiles<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(
            ref, m, cfg->c_ref[0], cfg->c_ref[1], cfg->c_ref[2], em->threads, em->n_tiles,
            em->d_tiles);
        if (cudaGetLastError() != cudaSuccess) {
            fr_em64_destroy(em);
            set_error("float64 EM tile copy failed");
            return FR_ECUDA;
        }
    }
    *out = em;
    return FR_OK;
}

int fr_em64_destroy(fr_em64 *em) {
    if (!em) return FR_OK;
    cudaStreamSynchronize(em->stream);
    for (void *p : {(void *)em->d_em, (void *)em->d_sums, (void *)em->d_partials,
                    (void *)em->d_traces, (void *)em->d_sync, (void *)em->d_prof,
                    (void *)em->d_tiles})
        if (p) cudaFreeAsync(p, em->stream);
    delete em;
    return FR_OK;
}

int fr_em64_launch_info(const fr_em64 *em, int *grid, int *block) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    if (grid) *grid = em->grid;
    if (block) *block = em->block;
    return FR_OK;
}

int fr_em64_run(fr_em64 *em, int n_iters, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    em->stream = (cudaStream_t)stream;
    const int n = n_iters > 0 ? n_iters : em->max_iters;
    return e64_launch(em, n, 1, (cudaStream_t)stream);
}

// independent float64 registrations in one cooperative launch: problem i
// runs on its own G CTAs (blockIdx.y = i), G = SMs / n (at least 1; waves of
// at most SMs problems).  Every problem's result equals fr_em64_run's on the
// same grid size.  Synchronises `stream`.
int fr_em64_run_batch(fr_em64 **ems, int n, void *stream) {
    if (n < 0 || (n > 0 && !ems)) {
        set_error("invalid batch arguments");
        return FR_EINVAL;
    }
    if (n == 0) return FR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    for (int i = 0; i < n; ++i)
        if (!ems[i] || ems[i]->fn != ems[0]->fn) {
            set_error("batch problem %d is null or was created under another launch variant", i);
            return FR_EINVAL;
        }
    const int sms = std::min(sm_count(), kE64MaxSms);
    for (int w0 = 0; w0 < n; w0 += sms) {
        const int nw = std::min(n - w0, sms);
        int g = std::max(1, sms / nw);
        long long max_tiles = 0;
        for (int i = w0; i < w0 + nw; ++i) max_tiles = std::max(max_tiles, ems[i]->n_tiles);
        g = (int)std::min<long long>(g, max_tiles);
        std::vector<Em64Args> h((size_t)nw);
        for (int i = 0; i < nw; ++i) {
            fr_em64 *em = ems[w0 + i];
            em->stream = s;
            h[i] = e64_args(em, em->max_iters, 1, g);
            FR_CUDA(cudaMemsetAsync(em->d_sync, 0, 2 * sizeof(unsigned), s));
        }
        Em64Args *d = nullptr;
        FR_CUDA(cudaMallocAsync((void **)&d, h.size() * sizeof(Em64Args), s));
        FR_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(Em64Args), cudaMemcpyHostToDevice, s));
        Em64Args unused = h[0];
        void *args[] = {&unused, &d};
        FR_CUDA(cudaLaunchCooperativeKernel((const void *)ems[0]->batch_fn, dim3(g, nw),
                                            dim3(ems[0]->block), args, ems[0]->smem, s));
        FR_CUDA(cudaFreeAsync(d, s));
        FR_CUDA(cudaStreamSynchronize(s));       // the host vector backs the copy
    }
    return FR_OK;
}

int fr_em64_pass(fr_em64 *em, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    em->stream = (cudaStream_t)stream;
    return e64_launch(em, 1, 0, (cudaStream_t)stream);
}

int fr_em64_pass_solve(fr_em64 *em, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    em->stream = (cudaStream_t)stream;
    return e64_launch(em, 1, 2, (cudaStream_t)stream);
}

int fr_em64_done_ptr(fr_em64 *em, int **d_done) {
    if (!em || !d_done) {
        set_error("null argument");
        return FR_EINVAL;
    }
    *d_done = &em->d_em->done;
    return FR_OK;
}

int fr_em64_solve(fr_em64 *em, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    em->stream = (cudaStream_t)stream;
    k_em64_solve<<<1, 32, 0, (cudaStream_t)stream>>>(em->d_sums, em->d_em, em->d_traces);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

// FR_EM64_PROFILE=1 diagnostics: the phase timestamps of the last launch's
// iterations ([n][8] ns: CTA 0 pass start / end, last CTA tail start / after
// the reduction / after the solve, CTA 0 release seen); not part of the C ABI
int fr_em64_profile(fr_em64 *em, unsigned long long *host, int n, void *stream) {
    if (!em || !em->d_prof) {
        set_error("profiling is off (FR_EM64_PROFILE=1 at create)");
        return FR_ESTATE;
    }
    n = std::min(n, em->max_iters);
    FR_CUDA(cudaMemcpyAsync(host, em->d_prof, (size_t)8 * n * 8, cudaMemcpyDeviceToHost,
                            (cudaStream_t)stream));
    FR_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return FR_OK;
}

int fr_em64_sums(fr_em64 *em, double **d_sums, int *width) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    if (d_sums) *d_sums = em->d_sums;
    if (width) *width = kE64Stats;
    return FR_OK;
}

int fr_em64_status(fr_em64 *em, int *done, int *iterations, int *termination, void *stream) {
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

int fr_em64_result(fr_em64 *em, double *R, double *t, double *objectives, double *twist_norms,
                   double *inlier_masses, int *iterations, int *termination, void *stream) {
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
