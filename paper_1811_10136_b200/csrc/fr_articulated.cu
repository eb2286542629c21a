// Device-resident articulated FilterReg EM (pipeline.py:125-181 with an
// ArticulatedTree; mstep.py:213-229, 348-369, 421-459; kinematics.py:76-229).
//
// Per EM iteration, replayed from a CUDA graph with no host round trip:
//   k_body_pass (fr_rigid.cu)  per-body point-to-point statistics of the
//                              body-sorted model points at the body poses the
//                              solve kernel left in device memory;
//   k_reduce_segments          per-body sums (fixed order);
//   k_art_solve (one CTA)      the whole M step: per-body normal equations
//                              about each body's centre, forward kinematics
//                              (joint motions in parallel over bodies, the
//                              parent chain in order), the spatial velocity
//                              Jacobian columns, the projection
//                              A = sum S_b^T H_b S_b, b = sum S_b^T g_b, the
//                              damped Cholesky of A with tenfold escalation
//                              (parallel right-looking factorisation in
//                              shared memory), step halving with closed-form
//                              candidate objectives from the per-body
//                              statistics (each candidate a forward
//                              kinematics pass), extra Gauss-Newton
//                              iterations on the moved statistics, update
//                              magnitude, termination, traces and the next
//                              pass constants of every body.
#include <algorithm>
#include <cstring>
#include <vector>

#include "fr_common.cuh"
#include "fr_reduce.cuh"
#include "fr_solve.cuh"

namespace fr {

constexpr int kArtMaxBodies = 32;
constexpr int kArtMaxParams = 40;
constexpr int kArtThreads = 256;
constexpr int kArtStats = 25;        // the rigid point-to-point pass layout

struct ArtTree {
    int nb, np, floating, n_mov;
    int parent[kArtMaxBodies], kind[kArtMaxBodies], slot[kArtMaxBodies];
    int mov[kArtMaxParams];                  // movable slot -> body
    unsigned anc[kArtMaxBodies];             // bit i: body i is an ancestor-or-self
    double axis[kArtMaxBodies][3], FR[kArtMaxBodies][9], Ft[kArtMaxBodies][3];
    double cb[kArtMaxBodies][3];             // body-frame centre of the body's points
};

struct ArtState {
    double A[4][3];                          // lattice embedding (pass constants)
    double s2[3];
    double cp, gain, diameter, tol, damping, step_tol, degenerate_mass;
    int max_em_iters, max_gn_iters, max_halvings, use_damping;
    double baseR[9], baset[3];
    double q[kArtMaxParams];
    int done, iterations, termination, pad;
};

struct ArtWork {
    Mom mo[kArtMaxBodies];
    double WR[kArtMaxBodies][9], Wt[kArtMaxBodies][3];      // current body poses
    double W0R[kArtMaxBodies][9], W0t[kArtMaxBodies][3];    // at the start of the M step
    double CR[kArtMaxBodies][9], Ct[kArtMaxBodies][3];      // candidate body poses
    double lR[kArtMaxBodies][9], lt[kArtMaxBodies][3];      // local (frame o motion)
    double cent[kArtMaxBodies][3];
    double Hb[kArtMaxBodies][36], gb[kArtMaxBodies][6];
    double D[kArtMaxBodies][9], delta[kArtMaxBodies][3], dE[kArtMaxBodies];
    double Z[6][kArtMaxParams];
    double bvec[kArtMaxParams], step[kArtMaxParams], x[kArtMaxParams], rdiag[kArtMaxParams];
    double cbaseR[9], cbaset[3], cq[kArtMaxParams];          // candidate state
    double value, value0, lam, trace, cv;
    int flag, accepted, gn;
};

__device__ __forceinline__ bool anc_of(const ArtTree &T, int b, int body) {
    return (T.anc[b] >> body) & 1u;
}

// local transform frame o motion(q) of body b (kinematics.py:59-65, 148-178)
__device__ void art_local(const ArtTree &T, const double *q, int b, double *lR, double *lt) {
    double mR[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, mt[3] = {0, 0, 0};
    const int s = T.slot[b];
    if (s >= 0) {
        const double v = q[s];
        if (T.kind[b] == 1) {
            const double tw[6] = {T.axis[b][0] * v, T.axis[b][1] * v, T.axis[b][2] * v, 0, 0, 0};
            const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1}, z[3] = {0, 0, 0};
            apply_twist_dev(tw, I, z, mR, mt);
        } else if (T.kind[b] == 2) {
            for (int i = 0; i < 3; ++i) mt[i] = T.axis[b][i] * v;
        }
    }
    m3_mul(T.FR[b], mR, lR);
    for (int i = 0; i < 3; ++i)
        lt[i] = T.FR[b][3 * i] * mt[0] + T.FR[b][3 * i + 1] * mt[1] + T.FR[b][3 * i + 2] * mt[2] +
                T.Ft[b][i];
}

// world poses: parent o local, in body order (one thread)
__device__ void art_chain(const ArtTree &T, const double *baseR, const double *baset,
                          const double (*lR)[9], const double (*lt)[3], double (*WR)[9],
                          double (*Wt)[3]) {
    for (int i = 0; i < T.nb; ++i) {
        const double *PR = i == 0 ? baseR : WR[T.parent[i]];
        const double *Pt = i == 0 ? baset : Wt[T.parent[i]];
        m3_mul(PR, lR[i], WR[i]);
        for (int r = 0; r < 3; ++r)
            Wt[i][r] = PR[3 * r] * lt[i][0] + PR[3 * r + 1] * lt[i][1] + PR[3 * r + 2] * lt[i][2] +
                       Pt[r];
    }
}

// forward kinematics of (base, q) into (WR, Wt): all threads call
__device__ void art_fk(const ArtTree &T, ArtWork &w, const double *baseR, const double *baset,
                       const double *q, double (*WR)[9], double (*Wt)[3]) {
    for (int b = threadIdx.x; b < T.nb; b += blockDim.x) art_local(T, q, b, w.lR[b], w.lt[b]);
    __syncthreads();
    if (threadIdx.x == 0) art_chain(T, baseR, baset, w.lR, w.lt, WR, Wt);
    __syncthreads();
}

// one EM iteration's M step (all threads of the CTA; S / T / w in shared memory)
__device__ void art_mstep(const double *__restrict__ bsums, const ArtState *st, const ArtTree &T,
                          ArtState &S, ArtWork &w, double *dyn, double *traces, RigidK *params) {
    const int tid = threadIdx.x;
    const int nb = T.nb, np = T.np, c0 = T.floating ? 6 : 0;
    double *HZ = dyn;                                   // [nb][6][np]
    double *Am = HZ + nb * 6 * np;                      // [np][np]
    double *L = Am + np * np;                           // [np][np]
    for (int b = tid; b < nb; b += blockDim.x) mom_from_sums(bsums + b * kArtStats, w.mo[b]);
    __syncthreads();
    const int it = S.iterations;
    if (tid == 0) {
        double mass = 0.0, val = 0.0;
        for (int b = 0; b < nb; ++b) mass += w.mo[b].S0;
        for (int b = 0; b < nb; ++b) val += mom_energy(w.mo[b], S.s2);
        traces[2 * S.max_em_iters + it] = mass;
        w.value0 = w.value = val;
        w.flag = mass < S.degenerate_mass;
        w.gn = 0;
        w.accepted = 0;
    }
    __syncthreads();
    if (w.flag) {           // no correspondence mass (pipeline.py:148-154)
        if (tid == 0) {
            traces[it] = CUDART_NAN;
            traces[S.max_em_iters + it] = CUDART_NAN;
            S.iterations = it + 1;
            S.termination = kTermDegenerate;
            S.done = 1;
        }
        __syncthreads();
        return;
    }
    // body poses of the current state, the body centres (fixed for the M step)
    art_fk(T, w, S.baseR, S.baset, S.q, w.WR, w.Wt);
    for (int b = tid; b < nb; b += blockDim.x) {
        for (int i = 0; i < 3; ++i)
            w.cent[b][i] = w.WR[b][3 * i] * T.cb[b][0] + w.WR[b][3 * i + 1] * T.cb[b][1] +
                           w.WR[b][3 * i + 2] * T.cb[b][2] + w.Wt[b][i];
        for (int q = 0; q < 9; ++q) w.W0R[b][q] = w.WR[b][q];
        for (int q = 0; q < 3; ++q) w.W0t[b][q] = w.Wt[b][q];
    }
    for (int q = tid; q < np; q += blockDim.x) w.cq[q] = S.q[q];
    if (tid == 0)
        for (int q = 0; q < 9; ++q) w.cbaseR[q] = S.baseR[q], w.cbaset[q % 3] = S.baset[q % 3];
    __syncthreads();
    for (int gn = 0; gn < S.max_gn_iters; ++gn) {
        // ---- the projected normal equations (mstep.py:213-229) ----------
        for (int b = tid; b < nb; b += blockDim.x) {
            double H[6][6], g[6];
            mom_normal_eq(w.mo[b], w.cent[b], S.s2, H, g);
            for (int i = 0; i < 6; ++i) {
                for (int j = 0; j < 6; ++j) w.Hb[b][6 * i + j] = H[i][j];
                w.gb[b][i] = g[i];
            }
        }
        for (int e = tid; e < 6 * np; e += blockDim.x) {
            const int k = e / np, c = e % np;
            double v = 0.0;
            if (c < c0) {
                v = k == c ? 1.0 : 0.0;
            } else {
                const int body = T.mov[c - c0];
                const double *R = w.WR[body];
                const double *ax = T.axis[body];
                const double aw[3] = {R[0] * ax[0] + R[1] * ax[1] + R[2] * ax[2],
                                      R[3] * ax[0] + R[4] * ax[1] + R[5] * ax[2],
                                      R[6] * ax[0] + R[7] * ax[1] + R[8] * ax[2]};
                if (T.kind[body] == 1) {
                    const double *o = w.Wt[body];
                    const double cr[3] = {o[1] * aw[2] - o[2] * aw[1], o[2] * aw[0] - o[0] * aw[2],
                                          o[0] * aw[1] - o[1] * aw[0]};
                    v = k < 3 ? aw[k] : cr[k - 3];
                } else {
                    v = k < 3 ? 0.0 : aw[k - 3];
                }
            }
            w.Z[k][c] = v;
        }
        __syncthreads();
        // HZ_b = H_b S_b (masked columns)
        for (int e = tid; e < nb * 6 * np; e += blockDim.x) {
            const int b = e / (6 * np), r = e % (6 * np), k = r / np, c = r % np;
            const bool on = c < c0 || anc_of(T, b, T.mov[c - c0]);
            double v = 0.0;
            if (on)
                for (int j = 0; j < 6; ++j) v += w.Hb[b][6 * k + j] * w.Z[j][c];
            HZ[e] = v;
        }
        __syncthreads();
        for (int e = tid; e < np * np; e += blockDim.x) {
            const int p = e / np, c = e % np;
            if (p > c) continue;
            double v = 0.0;
            for (int b = 0; b < nb; ++b) {
                if (!(p < c0 || anc_of(T, b, T.mov[p - c0]))) continue;
                const double *hz = HZ + b * 6 * np;
                for (int k = 0; k < 6; ++k) v += w.Z[k][p] * hz[k * np + c];
            }
            Am[p * np + c] = v;
            Am[c * np + p] = v;
        }
        for (int p = tid; p < np; p += blockDim.x) {
            double v = 0.0;
            for (int b = 0; b < nb; ++b) {
                if (!(p < c0 || anc_of(T, b, T.mov[p - c0]))) continue;
                for (int k = 0; k < 6; ++k) v += w.Z[k][p] * w.gb[b][k];
            }
            w.bvec[p] = v;
        }
        __syncthreads();
        if (tid == 0) {
            bool any = false;
            double tr = 0.0;
            for (int p = 0; p < np; ++p) {
                any |= w.bvec[p] != 0.0;
                tr += Am[p * np + p];
            }
            w.flag = any ? 1 : 0;
            w.trace = tr;
            w.lam = S.use_damping ? S.damping : 1e-6 * tr / np;
        }
        __syncthreads();
        if (!w.flag) break;                        // zero gradient: no step
        // ---- damped Cholesky with tenfold escalation (mstep.py:348-369) --
        bool solved = false;
        for (int attempt = 0; attempt < 6 && !solved; ++attempt) {
            for (int e = tid; e < np * np; e += blockDim.x)
                L[e] = Am[e] + ((e / np) == (e % np) ? w.lam : 0.0);
            if (tid == 0) w.flag = 1;
            __syncthreads();
            for (int k = 0; k < np; ++k) {
                if (tid == 0) {
                    const double d = L[k * np + k];
                    if (!(d > 0.0) || !isfinite(d)) {
                        w.flag = 0;
                    } else {
                        const double l = sqrt(d);
                        L[k * np + k] = l;
                        w.rdiag[k] = 1.0 / l;
                    }
                }
                __syncthreads();
                if (!w.flag) break;
                for (int i = k + 1 + tid; i < np; i += blockDim.x) L[i * np + k] *= w.rdiag[k];
                __syncthreads();
                const int rem = np - k - 1;
                for (int e = tid; e < rem * rem; e += blockDim.x) {
                    const int i = k + 1 + e / rem, j = k + 1 + e % rem;
                    if (j <= i) L[i * np + j] -= L[i * np + k] * L[j * np + k];
                }
                __syncthreads();
            }
            if (w.flag) {
                if (tid == 0) {
                    // L y = b, L^T x = y
                    for (int i = 0; i < np; ++i) {
                        double v = w.bvec[i];
                        for (int k = 0; k < i; ++k) v -= L[i * np + k] * w.x[k];
                        w.x[i] = v * w.rdiag[i];
                    }
                    for (int i = np - 1; i >= 0; --i) {
                        double v = w.x[i];
                        for (int k = i + 1; k < np; ++k) v -= L[k * np + i] * w.x[k];
                        w.x[i] = v * w.rdiag[i];
                    }
                    bool fin = true;
                    for (int i = 0; i < np; ++i) fin &= isfinite(w.x[i]);
                    w.flag = fin;
                    for (int i = 0; i < np; ++i) w.step[i] = -w.x[i];
                }
                __syncthreads();
                solved = w.flag;
            }
            if (!solved && tid == 0)
                w.lam = w.lam > 0.0 ? w.lam * 10.0 : fmax(w.trace / np, 1.0) * 1e-10;
            __syncthreads();
        }
        if (!solved) {
            if (tid == 0) {
                S.iterations = it + 1;
                S.termination = kTermSolver;
                S.done = 1;
            }
            __syncthreads();
            return;
        }
        // ---- step halving with closed-form candidate objectives ---------
        if (tid == 0) w.accepted = -1;
        __syncthreads();
        {
            double scale = 1.0;
            for (int h = 0; h <= S.max_halvings; ++h) {
                if (tid == 0) {
                    // base multiplicative, joints additive (kinematics.py:213-224)
                    if (T.floating) {
                        double tw[6];
                        for (int q = 0; q < 6; ++q) tw[q] = scale * w.step[q];
                        apply_twist_dev(tw, w.cbaseR, w.cbaset, S.baseR, S.baset);
                    } else {
                        for (int q = 0; q < 9; ++q) S.baseR[q] = w.cbaseR[q];
                        for (int q = 0; q < 3; ++q) S.baset[q] = w.cbaset[q];
                    }
                    for (int s = 0; s < np - c0; ++s) S.q[s] = w.cq[s] + scale * w.step[c0 + s];
                }
                __syncthreads();
                art_fk(T, w, S.baseR, S.baset, S.q, w.CR, w.Ct);
                for (int b = tid; b < nb; b += blockDim.x) {
                    m3_mul_t(w.CR[b], w.WR[b], w.D[b]);
                    for (int i = 0; i < 3; ++i)
                        w.delta[b][i] = w.Ct[b][i] - (w.D[b][3 * i] * w.Wt[b][0] +
                                                      w.D[b][3 * i + 1] * w.Wt[b][1] +
                                                      w.D[b][3 * i + 2] * w.Wt[b][2]);
                    w.dE[b] = mom_delta_energy(w.mo[b], w.D[b], w.delta[b], w.cent[b], S.s2);
                }
                __syncthreads();
                if (tid == 0) {
                    double e = 0.0;
                    for (int b = 0; b < nb; ++b) e += w.dE[b];
                    w.cv = w.value + e;
                    if (w.cv <= w.value * (1.0 + 1e-12) + 1e-300) w.accepted = h;   // mstep.py:446
                }
                __syncthreads();
                if (w.accepted >= 0) break;
                scale *= 0.5;
            }
            if (w.accepted < 0) {
                // no acceptable step: the M step keeps the state it had
                if (tid == 0) {
                    for (int q = 0; q < 9; ++q) S.baseR[q] = w.cbaseR[q];
                    for (int q = 0; q < 3; ++q) S.baset[q] = w.cbaset[q];
                    for (int s = 0; s < np - c0; ++s) S.q[s] = w.cq[s];
                }
                __syncthreads();
                break;
            }
            // accepted: the candidate becomes the current state
            for (int b = tid; b < nb; b += blockDim.x) {
                for (int q = 0; q < 9; ++q) w.WR[b][q] = w.CR[b][q];
                for (int q = 0; q < 3; ++q) w.Wt[b][q] = w.Ct[b][q];
            }
            if (tid == 0) {
                for (int q = 0; q < 9; ++q) w.cbaseR[q] = S.baseR[q];
                for (int q = 0; q < 3; ++q) w.cbaset[q] = S.baset[q];
                for (int s = 0; s < np - c0; ++s) w.cq[s] = S.q[s];
                w.value = w.cv;
                double sn = 0.0;
                for (int q = 0; q < np; ++q) sn += (scale * w.step[q]) * (scale * w.step[q]);
                w.flag = (sqrt(sn) <= S.step_tol || gn + 1 >= S.max_gn_iters) ? 0 : 1;
            }
            __syncthreads();
            if (!w.flag) break;
            // statistics at the accepted pose for the next Gauss-Newton iteration
            for (int b = tid; b < nb; b += blockDim.x)
                mom_moved(w.mo[b], w.D[b], w.delta[b], w.cent[b]);
            __syncthreads();
        }
    }
    // ---- update magnitude and termination (pipeline.py:79-86, 167-177) ----
    for (int b = tid; b < nb; b += blockDim.x) {
        double Rd[9];
        m3_mul_t(w.WR[b], w.W0R[b], Rd);
        const double dx = w.Wt[b][0] - w.W0t[b][0], dy = w.Wt[b][1] - w.W0t[b][1],
                     dz = w.Wt[b][2] - w.W0t[b][2];
        w.dE[b] = rotation_angle_dev(Rd) + sqrt((dx * dx + dy * dy) + dz * dz) / S.diameter;
    }
    __syncthreads();
    if (tid == 0) {
        double norm = 0.0;
        for (int b = 0; b < nb; ++b) norm = fmax(norm, w.dE[b]);
        traces[S.max_em_iters + it] = norm;
        S.iterations = it + 1;
        if (norm < S.tol) {         // sub-tolerance motion: dropped (pipeline.py:169-173)
            traces[it] = w.value0;
            S.termination = kTermConverged;
            S.done = 1;
            w.flag = 0;
        } else {
            traces[it] = w.value;
            // S.baseR / S.baset / S.q hold the accepted state (or the old one)
            if (it + 1 >= S.max_em_iters) {
                S.termination = kTermMaxIters;
                S.done = 1;
            }
            w.flag = 1;
        }
    }
    __syncthreads();
    if (S.termination == kTermConverged && S.done) {
        // reload the pre-M-step state from global memory (unchanged there)
        if (tid == 0) {
            for (int q = 0; q < 9; ++q) S.baseR[q] = st->baseR[q];
            for (int q = 0; q < 3; ++q) S.baset[q] = st->baset[q];
            for (int s = 0; s < np - c0; ++s) S.q[s] = st->q[s];
        }
        __syncthreads();
    } else {
        // next pass constants of every body at the new state
        for (int b = tid; b < nb; b += blockDim.x)
            make_rigid_k(S.A, w.WR[b], w.Wt[b], T.cb[b], S.cp, S.gain, -1, -1, &params[b]);
    }
}

__global__ void __launch_bounds__(kArtThreads, 1)
k_art_solve(const double *__restrict__ bsums, ArtState *st, const ArtTree *tree, double *traces,
            RigidK *params) {
    extern __shared__ double dyn[];          // HZ [nb][6][np] | Amat [np][np] | L [np][np]
    __shared__ ArtTree T;
    __shared__ ArtState S;
    __shared__ ArtWork w;
    const int tid = threadIdx.x;
    {
        const unsigned long long *a = reinterpret_cast<const unsigned long long *>(st);
        unsigned long long *b = reinterpret_cast<unsigned long long *>(&S);
        for (int q = tid; q < (int)(sizeof(ArtState) / 8); q += blockDim.x) b[q] = a[q];
        const int *ta = reinterpret_cast<const int *>(tree);
        int *tb = reinterpret_cast<int *>(&T);
        for (int q = tid; q < (int)(sizeof(ArtTree) / 4); q += blockDim.x) tb[q] = ta[q];
    }
    __syncthreads();
    if (S.done) return;
    art_mstep(bsums, st, T, S, w, dyn, traces, params);
    __syncthreads();
    const unsigned long long *a = reinterpret_cast<const unsigned long long *>(&S);
    unsigned long long *b = reinterpret_cast<unsigned long long *>(st);
    for (int q = tid; q < (int)(sizeof(ArtState) / 8); q += blockDim.x) b[q] = a[q];
}

static size_t art_smem(int nb, int np) {
    return ((size_t)nb * 6 * np + 2 * (size_t)np * np) * sizeof(double);
}

}  // namespace fr

extern "C" int fr_body_pass_dev(const fr_lattice *lat, const float *ref, int64_t m,
                                const void *d_bodies, int n_bodies, const int32_t *chunk_body,
                                const int64_t *chunk_beg, int n_chunks, const int32_t *body_chunks,
                                int flags, double *sums, double *scratch, const int32_t *d_done,
                                void *stream);

struct fr_art_em {
    const fr_lattice *lat = nullptr;
    const float *ref = nullptr;
    long long m = 0;
    int nb = 0, np = 0, n_chunks = 0, flags = 0, max_iters = 0;
    const int32_t *chunk_body = nullptr, *body_chunks = nullptr;
    const int64_t *chunk_beg = nullptr;
    fr::ArtTree *d_tree = nullptr;
    fr::ArtState *d_state = nullptr;
    fr::RigidK *d_params = nullptr;
    double *d_bsums = nullptr, *d_scratch = nullptr, *d_traces = nullptr;
    cudaGraphExec_t graph = nullptr;
    cudaStream_t stream = nullptr;
};

using namespace fr;

static int art_iteration(fr_art_em *em, cudaStream_t s) {
    FR_TRY(fr_body_pass_dev(em->lat, em->ref, em->m, em->d_params, em->nb, em->chunk_body,
                            em->chunk_beg, em->n_chunks, em->body_chunks, em->flags, em->d_bsums,
                            em->d_scratch, &em->d_state->done, s));
    k_art_solve<<<1, kArtThreads, art_smem(em->nb, em->np), s>>>(em->d_bsums, em->d_state,
                                                                 em->d_tree, em->d_traces,
                                                                 em->d_params);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

extern "C" {

int fr_art_em_create(const fr_lattice *lat, const float *ref, int64_t m,
                     const fr_art_tree_desc *tree, const double *q0, const double *base_R0,
                     const double *base_t0, const double *body_R0, const double *body_t0,
                     const int32_t *d_chunk_body,
                     const int64_t *d_chunk_beg, int n_chunks, const int32_t *d_body_chunks,
                     const fr_rigid_em_config *cfg, void *stream, fr_art_em **out) {
    cudaStream_t s = (cudaStream_t)stream;
    if (!lat || !lat->blurred || !ref || !tree || !cfg || !out || !base_R0 || !base_t0 ||
        !d_chunk_body || !d_chunk_beg || !d_body_chunks || n_chunks < 1 || m <= 0) {
        set_error("invalid device articulated EM arguments");
        return FR_EINVAL;
    }
    if (lat->dim != 3 || lat->nv != 4) {
        set_error("the device articulated loop runs point_to_point with a fixed kernel width");
        return FR_EINVAL;
    }
    const int nb = tree->n_bodies, np = tree->n_params;
    const int c0 = tree->floating ? 6 : 0;
    if (nb < 1 || nb > kArtMaxBodies || np < 1 || np > kArtMaxParams || np - c0 < 0) {
        set_error("device articulated loop: at most %d bodies and %d parameters", kArtMaxBodies,
                  kArtMaxParams);
        return FR_EINVAL;
    }
    if (cfg->max_em_iters < 1 || cfg->max_gn_iters < 0 || cfg->max_halvings < 0) {
        set_error("invalid iteration limits");
        return FR_EINVAL;
    }
    ArtTree T;
    memset(&T, 0, sizeof(T));
    T.nb = nb;
    T.np = np;
    T.floating = tree->floating ? 1 : 0;
    T.n_mov = np - c0;
    for (int b = 0; b < nb; ++b) {
        T.parent[b] = tree->parent[b];
        T.kind[b] = tree->kind[b];
        T.slot[b] = tree->slot[b];
        if (T.slot[b] >= 0) {
            if (T.slot[b] >= T.n_mov) {
                set_error("joint slot out of range");
                return FR_EINVAL;
            }
            T.mov[T.slot[b]] = b;
        }
        if (b > 0 && (T.parent[b] < 0 || T.parent[b] >= b)) {
            set_error("body %d must have a parent earlier in the list", b);
            return FR_EINVAL;
        }
        T.anc[b] = (1u << b) | (b > 0 ? T.anc[T.parent[b]] : 0u);
        for (int i = 0; i < 3; ++i) {
            T.axis[b][i] = tree->axis[3 * b + i];
            T.Ft[b][i] = tree->frame_t[3 * b + i];
            T.cb[b][i] = tree->c_body[3 * b + i];
        }
        for (int q = 0; q < 9; ++q) T.FR[b][q] = tree->frame_R[9 * b + q];
    }
    ArtState S;
    memset(&S, 0, sizeof(S));
    embedding_matrix(lat->c, S.A);
    for (int i = 0; i < 3; ++i) S.s2[i] = cfg->sigma_inv[i] * cfg->sigma_inv[i];
    S.cp = cfg->c_prime;
    S.gain = lat->c.gain;
    S.diameter = cfg->diameter;
    S.tol = cfg->twist_tolerance;
    S.use_damping = cfg->damping >= 0.0;
    S.damping = cfg->damping;
    S.step_tol = cfg->step_tolerance;
    S.degenerate_mass = cfg->degenerate_mass;
    S.max_em_iters = cfg->max_em_iters;
    S.max_gn_iters = cfg->max_gn_iters;
    S.max_halvings = cfg->max_halvings;
    for (int q = 0; q < 9; ++q) S.baseR[q] = base_R0[q];
    for (int q = 0; q < 3; ++q) S.baset[q] = base_t0[q];
    for (int q = 0; q < np - c0; ++q) S.q[q] = q0 ? q0[q] : 0.0;
    fr_art_em *em = new fr_art_em();
    em->lat = lat;
    em->ref = ref;
    em->m = m;
    em->nb = nb;
    em->np = np;
    em->n_chunks = n_chunks;
    em->flags = cfg->fast;
    em->max_iters = cfg->max_em_iters;
    em->chunk_body = d_chunk_body;
    em->chunk_beg = d_chunk_beg;
    em->body_chunks = d_body_chunks;
    em->stream = s;
    const size_t smem = art_smem(nb, np);
    if (cudaFuncSetAttribute(k_art_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaMallocAsync((void **)&em->d_tree, sizeof(ArtTree), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_state, sizeof(ArtState), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_params, (size_t)nb * sizeof(RigidK), s) != cudaSuccess ||
        cudaMallocAsync((void **)&em->d_bsums, (size_t)nb * kArtStats * sizeof(double), s) !=
            cudaSuccess ||
        cudaMallocAsync((void **)&em->d_scratch, (size_t)n_chunks * kArtStats * sizeof(double), s) !=
            cudaSuccess ||
        cudaMallocAsync((void **)&em->d_traces, (size_t)3 * cfg->max_em_iters * sizeof(double), s) !=
            cudaSuccess ||
        cudaMemcpyAsync(em->d_tree, &T, sizeof(ArtTree), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(em->d_state, &S, sizeof(ArtState), cudaMemcpyHostToDevice, s) !=
            cudaSuccess ||
        cudaMemsetAsync(em->d_traces, 0, (size_t)3 * cfg->max_em_iters * sizeof(double), s) !=
            cudaSuccess) {
        fr_art_em_destroy(em);
        set_error("device articulated EM allocation failed");
        return FR_ECUDA;
    }
    // the first pass constants from the caller's body poses of the initial state
    std::vector<RigidK> ks((size_t)nb);
    for (int b = 0; b < nb; ++b)
        make_rigid_k(S.A, body_R0 + 9 * b, body_t0 + 3 * b, T.cb[b], S.cp, S.gain, -1, -1, &ks[b]);
    if (cudaMemcpyAsync(em->d_params, ks.data(), ks.size() * sizeof(RigidK), cudaMemcpyHostToDevice,
                        s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess) {
        fr_art_em_destroy(em);
        set_error("device articulated EM setup failed");
        return FR_ECUDA;
    }
    *out = em;
    return FR_OK;
}

int fr_art_em_destroy(fr_art_em *em) {
    if (!em) return FR_OK;
    cudaStreamSynchronize(em->stream);
    if (em->graph) cudaGraphExecDestroy(em->graph);
    for (void *p : {(void *)em->d_tree, (void *)em->d_state, (void *)em->d_params,
                    (void *)em->d_bsums, (void *)em->d_scratch, (void *)em->d_traces})
        if (p) cudaFreeAsync(p, em->stream);
    delete em;
    return FR_OK;
}

// iterate to termination: graphs of 4 iterations (pass, per-body sums, solve),
// the done flag read through pinned memory one chunk behind
int fr_art_em_run(fr_art_em *em, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    em->stream = s;
    constexpr int kChunk = 4;
    if (!em->graph) {
        cudaStream_t cs;
        FR_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaGraph_t g;
        FR_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        int st = FR_OK;
        for (int i = 0; i < kChunk && st == FR_OK; ++i) st = art_iteration(em, cs);
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
    int issued = 0, k = 0;
    auto chunk = [&]() -> int {
        FR_CUDA(cudaGraphLaunch(em->graph, s));
        FR_CUDA(cudaMemcpyAsync(flags + 4 * (k & 1), &em->d_state->done, 3 * sizeof(int),
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

int fr_art_em_result(fr_art_em *em, double *q, double *base_R, double *base_t,
                     double *objectives, double *twist_norms, double *inlier_masses,
                     int *iterations, int *termination, void *stream) {
    if (!em) {
        set_error("null EM object");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    ArtState h;
    FR_CUDA(cudaMemcpyAsync(&h, em->d_state, sizeof(ArtState), cudaMemcpyDeviceToHost, s));
    std::vector<double> tr((size_t)3 * em->max_iters);
    FR_CUDA(cudaMemcpyAsync(tr.data(), em->d_traces, tr.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaStreamSynchronize(s));
    if (q) memcpy(q, h.q, sizeof(h.q));
    if (base_R) memcpy(base_R, h.baseR, 9 * sizeof(double));
    if (base_t) memcpy(base_t, h.baset, 3 * sizeof(double));
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
