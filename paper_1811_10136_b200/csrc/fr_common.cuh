// Shared helpers of the B200 FilterReg engine: status/error plumbing, the
// bit-exact permutohedral embedding (permutohedral.py:171-215) and the
// packed lattice-key codec.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string.h>

#include "../../include/filterreg_b200.h"

namespace fr {

// ---------------------------------------------------------------------------
// errors

void set_error(const char *fmt, ...);

#define FR_CUDA(expr)                                                          \
    do {                                                                       \
        cudaError_t _e = (expr);                                               \
        if (_e != cudaSuccess) {                                               \
            ::fr::set_error("%s failed: %s (%s:%d)", #expr,                    \
                            cudaGetErrorString(_e), __FILE__, __LINE__);       \
            return FR_ECUDA;                                                   \
        }                                                                      \
    } while (0)

#define FR_CHECK_LAUNCH() FR_CUDA(cudaGetLastError())

#define FR_TRY(expr)                                                           \
    do {                                                                       \
        int _s = (expr);                                                       \
        if (_s != FR_OK) return _s;                                            \
    } while (0)

// ---------------------------------------------------------------------------
// lattice constants: passed by value into kernels, computed on the host with
// the reference's exact expressions (permutohedral.py:156-163)

constexpr int kMaxDim = 12;

struct LatticeConsts {
    int dim;
    double sigma[kMaxDim];
    double sf[kMaxDim];   // s_d / sqrt((j+1)(j+2))
    double gain;
};

int make_consts(int dim, const double *sigma, LatticeConsts *out);

// ---------------------------------------------------------------------------
// packed keys: the first D coordinates of a lattice key (the last is minus
// their sum), 21 bits each with a +2^20 offset for D <= 3, so unsigned order
// equals the reference's lexicographic site order (permutohedral.py:96-137).

constexpr int kKeyBits = 21;
constexpr long long kKeyOff = 1LL << (kKeyBits - 1);
constexpr long long kKeyLim = kKeyOff - 2;           // |coord| must stay below
constexpr unsigned long long kEmptyKey = ~0ull;       // never a valid packed key

template <int D>
__host__ __device__ __forceinline__ unsigned long long pack_key(const int *k) {
    unsigned long long p = 0;
#pragma unroll
    for (int i = 0; i < D; ++i)
        p = (p << kKeyBits) | (unsigned long long)(k[i] + kKeyOff);
    return p;
}

template <int D>
__host__ __device__ __forceinline__ void unpack_key(unsigned long long p, int *k) {
    int s = 0;
#pragma unroll
    for (int i = D - 1; i >= 0; --i) {
        k[i] = (int)((long long)(p & ((1ull << kKeyBits) - 1)) - kKeyOff);
        p >>= kKeyBits;
        s += k[i];
    }
    k[D] = -s;
}

__host__ __device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    // splitmix64 finaliser: spreads the structured lattice codes over slots
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

// ---------------------------------------------------------------------------
// bit-exact enclosing simplex (permutohedral.py:171-215)
//
// Every floating-point operation mirrors the NumPy expression it restates,
// with explicit round-to-nearest intrinsics so nvcc cannot contract into FMAs:
//   f = features / sigma * sf                     (:172)
//   el = f @ E.T, k-ascending                    (:174-179)
//   rem0 = rint(el / (d+1)) * (d+1)               (:191-192)
//   rank = stable descending order of el - rem0   (:193-197)
//   h, +-(d+1) wrap                               (:198-203)
//   res = (el - rem0) / (d+1), bary               (:206-212)
//   keys[l][i] = rem0[i] + canonical[l][rank[i]]  (:214)

template <int D>
struct Simplex {
    int rem0[D + 1];
    int rank[D + 1];
    double bary[D + 1];
    int overflow;   // 1 when a coordinate leaves the packable range

    __device__ __forceinline__ void vertex(int l, int *key) const {
#pragma unroll
        for (int i = 0; i <= D; ++i)
            key[i] = rem0[i] + ((rank[i] <= D - l) ? l : l - (D + 1));
    }
    __device__ __forceinline__ unsigned long long packed(int l) const {
        int k[D + 1];
        vertex(l, k);
        return pack_key<D>(k);
    }
};

template <int D>
__device__ __forceinline__ void simplex_from_elevated(const double *el, Simplex<D> &s) {
    const double d1 = (double)(D + 1);
    double diff[D + 1];
    long long hsum = 0;
    s.overflow = 0;
#pragma unroll
    for (int i = 0; i <= D; ++i) {
        double r = rint(__ddiv_rn(el[i], d1));
        if (!(fabs(r) < (double)(kKeyLim / (D + 1)))) { s.overflow = 1; r = 0.0; }
        int ri = (int)r;
        s.rem0[i] = ri * (D + 1);
        hsum += ri;
        diff[i] = __dsub_rn(el[i], (double)s.rem0[i]);
    }
#pragma unroll
    for (int i = 0; i <= D; ++i) {
        int rk = 0;
#pragma unroll
        for (int j = 0; j <= D; ++j) {
            if (j == i) continue;
            rk += (diff[j] > diff[i]) || (j < i && diff[j] == diff[i]);
        }
        s.rank[i] = rk;
    }
    const int h = (int)hsum;   // sum(rem0) // (d+1)
#pragma unroll
    for (int i = 0; i <= D; ++i) {
        int rk = s.rank[i] + h;
        if (rk < 0) { rk += D + 1; s.rem0[i] += D + 1; }
        else if (rk > D) { rk -= D + 1; s.rem0[i] -= D + 1; }
        s.rank[i] = rk;
    }
    double res[D + 1], sv[D + 1];
#pragma unroll
    for (int i = 0; i <= D; ++i) res[i] = __ddiv_rn(__dsub_rn(el[i], (double)s.rem0[i]), d1);
#pragma unroll
    for (int r = 0; r <= D; ++r) {
        double v = 0.0;
#pragma unroll
        for (int i = 0; i <= D; ++i) v = (s.rank[i] == r) ? res[i] : v;
        sv[r] = v;
    }
    s.bary[0] = __dsub_rn(__dadd_rn(1.0, sv[D]), sv[0]);
#pragma unroll
    for (int l = 1; l <= D; ++l) s.bary[l] = __dsub_rn(sv[D - l], sv[D - l + 1]);
}

template <int D>
__device__ __forceinline__ void elevate_exact(const double *feat, const LatticeConsts &c,
                                              double *el) {
    double f[D];
#pragma unroll
    for (int j = 0; j < D; ++j) f[j] = __dmul_rn(__ddiv_rn(feat[j], c.sigma[j]), c.sf[j]);
#pragma unroll
    for (int i = 0; i <= D; ++i) {
        // row i: coefficient -i at column i-1, 1 at columns >= i, 0 before
        double acc = (i == 0) ? f[0] : __dmul_rn(f[i - 1], -(double)i);
#pragma unroll
        for (int k = (i == 0 ? 1 : i); k < D; ++k) acc = __dadd_rn(acc, f[k]);
        el[i] = acc;
    }
}

template <int D>
__device__ __forceinline__ void simplex_exact(const double *feat, const LatticeConsts &c,
                                              Simplex<D> &s) {
    double el[D + 1];
    elevate_exact<D>(feat, c, el);
    simplex_from_elevated<D>(el, s);
}

// ---------------------------------------------------------------------------
// slice table: open addressing, linear probing, key and float64 values inline
// in one 32/64/128-byte slot so a hit costs one sector-aligned gather.

template <int VP>
struct alignas(8 * (VP + 1)) SliceSlot {
    unsigned long long key;
    double v[VP];
};

template <int VP>
__device__ __forceinline__ const SliceSlot<VP> *probe(const SliceSlot<VP> *tab, unsigned mask,
                                                      unsigned long long key) {
    unsigned h = (unsigned)mix64(key) & mask;
    for (unsigned it = 0; it <= mask; ++it) {
        unsigned long long k = __ldg(&tab[h].key);
        if (k == key) return tab + h;
        if (k == kEmptyKey) return nullptr;
        h = (h + 1) & mask;
    }
    return nullptr;
}

inline int vp_for(int nv) { return nv <= 3 ? 3 : (nv <= 7 ? 7 : (nv <= 15 ? 15 : -1)); }

inline unsigned next_pow2(unsigned long long x) {
    unsigned long long p = 64;
    while (p < x) p <<= 1;
    return (unsigned)p;
}

}  // namespace fr

// the opaque lattice object behind fr_lattice*
struct fr_lattice {
    fr::LatticeConsts c;
    int dim = 3;
    int nv = 0;
    int blurred = 0;
    int splatted = 0;
    // site table (build state): full int32 keys [cap][dim+1], values [2][cap][nv]
    long long n_sites = 0;
    long long site_cap = 0;
    int *site_keys = nullptr;
    double *vals = nullptr;
    double *vals_alt = nullptr;
    // build hash: packed key -> site id
    unsigned long long *hkeys = nullptr;
    int *hsite = nullptr;
    unsigned hmask = 0;
    // slice table
    void *slots = nullptr;
    unsigned smask = 0;
    int vp = 0;
    // device counters / flags
    unsigned long long *d_counters = nullptr;   // [0] sites, [1] src count, [2] overflow
};
