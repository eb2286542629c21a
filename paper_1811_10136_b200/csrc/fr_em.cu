// E step on B200 (generic API) and the explicit rigid assembly.
//
//   fr_moments           MomentEngine.moments (estep.py:186-217): exact fp64
//                        slice fused with the moments epilogue per model point.
//   fr_moments_epilogue  the epilogue alone over raw kernel sums (feature modes,
//                        brute-force backend).
//   fr_assemble_rigid    assemble_rigid + objective (mstep.py:102-138, 179-210)
//                        over an explicit ResidualSpec.
// The fused per-iteration EM pass lives in fr_rigid.cu.
#include <algorithm>
#include <cmath>

#include "fr_reduce.cuh"

namespace fr {

template <int VP>
__global__ void k_moments(const double *X, long long m, LatticeConsts c, SliceTable tab,
                          double cp, int m2_col, int ncol, double *m0o, double *m1o, double *wo,
                          double *to, double *m2o, double *no, unsigned char *nvo) {
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        double x[3] = {X[p * 3], X[p * 3 + 1], X[p * 3 + 2]};
        Simplex<3> s;
        simplex_exact<3>(x, c, s);
        double acc[VP];
#pragma unroll
        for (int q = 0; q < VP; ++q) acc[q] = 0.0;
        if (!s.overflow) {
            unsigned long long key[4];
#pragma unroll
            for (int l = 0; l < 4; ++l) key[l] = s.packed(l);
            double v[4][VP];
            bool hit[4];
            gather_simplex<3, VP>(tab, key, v, hit);
#pragma unroll
            for (int l = 0; l < 4; ++l)
#pragma unroll
                for (int q = 0; q < VP; ++q)
                    acc[q] = hit[l] ? __dadd_rn(acc[q], __dmul_rn(s.bary[l], v[l][q])) : acc[q];
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

// sums [H upper 21 | g 6 | sum r^2] over explicit residual rows
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
            for (int c = 0; c < 6; ++c)
                G[c] = (P[r][0] * J[0][c] + P[r][1] * J[1][c]) + P[r][2] * J[2][c];
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
    const SliceTable tab = lat->table();
#define FR_MOM(NV)                                                                          \
    k_moments<NV><<<grid, 256, 0, s>>>(X, m, lat->c, tab, cp, m2_col, ncol, m0, m1, w, t, m2, \
                                       nrm, nvalid)
    switch (lat->nv) {
        case 4: FR_MOM(4); break;
        case 5: FR_MOM(5); break;
        case 6: FR_MOM(6); break;
        case 7: FR_MOM(7); break;
        case 8: FR_MOM(8); break;
        default:
            set_error("fused moments support 4..8 value columns, lattice has %d", lat->nv);
            return FR_EINVAL;
    }
#undef FR_MOM
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
    k_reduce_cols<<<1, 32 * kExplicitWidth, 0, s>>>(scratch, grid, kExplicitWidth, sums, nullptr);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

}  // extern "C"
