// Shared helpers of the B200 FilterReg engine: status/error plumbing, the
// bit-exact permutohedral embedding (permutohedral.py:171-215) and the
// packed lattice-key codec.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string.h>

#include <functional>

#include "../../include/filterreg_b200.h"

namespace fr {

// staged host -> device point upload (fr_upload.cu); the hook runs on the
// worker threads after each sub-chunk's copy is enqueued, with the event that
// marks the chunk [a, a + len) landed on the device
using ChunkHook = std::function<int(long long, long long, cudaEvent_t)>;
int upload_points_hooked(const double *host_xyz, long long n, float *d_soa, cudaStream_t s,
                         const ChunkHook &hook);
// page-locked host range (cudaPointerGetAttributes); rows [a, b) of (n, 3)
// float64 device rows -> the (3, n) planes, on `s` (fr_upload.cu)
bool host_is_pinned(const void *p, size_t bytes);
void rows_to_soa64_range(const double *rows, long long n, double *soa, long long a, long long b,
                         cudaStream_t s);

// ---------------------------------------------------------------------------
// errors

void set_error(const char *fmt, ...);
const char *last_error();

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

// x / (d+1): for d+1 a power of two the product with its reciprocal is the
// same correctly rounded real, so the cheaper multiply is bit-identical
template <int D>
__device__ __forceinline__ double div_d1(double x) {
    constexpr bool pow2 = ((D + 1) & D) == 0;
    return pow2 ? __dmul_rn(x, 1.0 / (double)(D + 1)) : __ddiv_rn(x, (double)(D + 1));
}

template <int D>
__device__ __forceinline__ void simplex_from_elevated(const double *el, Simplex<D> &s) {
    double diff[D + 1];
    long long hsum = 0;
    s.overflow = 0;
#pragma unroll
    for (int i = 0; i <= D; ++i) {
        double r = rint(div_d1<D>(el[i]));
        // d <= 3: the 21-bit packed key range; d >= 4: int32 keys
        constexpr double kLim = D <= 3 ? (double)(kKeyLim / (D + 1)) : (double)((1 << 28) / (D + 1));
        if (!(fabs(r) < kLim)) { s.overflow = 1; r = 0.0; }
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
    for (int i = 0; i <= D; ++i) res[i] = div_d1<D>(__dsub_rn(el[i], (double)s.rem0[i]));
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
// slice table: open addressing with linear probing, keys and values in two
// arrays indexed by the same slot.  A gather issues the key load and the
// (32/64/128-byte, sector-aligned) value-row load of all d+1 vertices at once;
// only a key mismatch that is not EMPTY (rare at load factor <= 1/2) probes on.

struct SliceTable {
    const unsigned long long *keys;
    const double *vals;     // [cap][nvp]
    unsigned mask;
    int shift;              // 64 - log2(cap)
    int nvp;                // padded row width: 4, 8 or 16
};

__host__ __device__ __forceinline__ unsigned slot_hash(unsigned long long key, int shift) {
    return (unsigned)((key * 0x9E3779B97F4A7C15ull) >> shift);
}

template <int NV>
__device__ __forceinline__ void load_row(const double *row, double *v) {
    if (NV % 2 == 0 || NV > 1) {
#pragma unroll
        for (int q = 0; q + 1 < NV; q += 2) {
            const double2 d = __ldg(reinterpret_cast<const double2 *>(row) + q / 2);
            v[q] = d.x;
            v[q + 1] = d.y;
        }
    }
    if (NV % 2 == 1) v[NV - 1] = __ldg(row + NV - 1);
}

// probe for `key`; returns the slot or -1 when absent
__device__ __forceinline__ int find_slot(const SliceTable &t, unsigned long long key, unsigned h) {
    for (unsigned it = 0; it <= t.mask; ++it) {
        const unsigned long long k = __ldg(t.keys + h);
        if (k == key) return (int)h;
        if (k == kEmptyKey) return -1;
        h = (h + 1) & t.mask;
    }
    return -1;
}

// gather the d+1 vertex rows of one simplex; hit[l] = 0 for absent vertices
template <int D, int NV>
__device__ __forceinline__ void gather_simplex(const SliceTable &t, const unsigned long long *key,
                                               double (*v)[NV], bool *hit) {
    unsigned h[D + 1];
    unsigned long long k[D + 1];
#pragma unroll
    for (int l = 0; l <= D; ++l) {
        h[l] = slot_hash(key[l], t.shift);
        k[l] = __ldg(t.keys + h[l]);
        load_row<NV>(t.vals + (size_t)h[l] * t.nvp, v[l]);
    }
#pragma unroll
    for (int l = 0; l <= D; ++l) {
        hit[l] = k[l] == key[l];
        if (!hit[l] && k[l] != kEmptyKey) {
            const int s = find_slot(t, key[l], (h[l] + 1) & t.mask);
            hit[l] = s >= 0;
            if (hit[l]) load_row<NV>(t.vals + (size_t)s * t.nvp, v[l]);
        }
    }
}

inline int nvp_for(int nv) { return nv <= 4 ? 4 : (nv <= 8 ? 8 : (nv <= 16 ? 16 : -1)); }

// ---------------------------------------------------------------------------
// fast query path of the EM pass (model points are not bit-exact contracts:
// they come out of a BLAS product in the reference, geometry.py:77).  The
// embedding and the nearest remainder-0 point stay float64 (lattice
// coordinates reach ~1e3-1e4); the residuals el - rem0 lie in [-2, 2], so
// ranks and barycentrics are float32 (abs. error ~1e-7), the packed keys are
// formed linearly from the packed remainder-0 point, and the value table
// holds float32 rows (16 or 32 bytes: one or two float4 per vertex).

// interleaved slot: packed key, then gain * value row as float32; 32 bytes
// (one sector) for nv <= 4, 64 bytes for nv <= 8.  The hash is a 32-bit fold.
// 128-bit key codec of the d >= 4 lattice (fr_lattice_wide.cuh): coordinate i
// of the first d occupies `bits[i]` bits at `shift[i]` (coordinate 0 highest),
// stored as k[i] - lo[i]
struct WideCodec {
    int d;
    int lo[kMaxDim];
    int bits[kMaxDim];
    int shift[kMaxDim];
    int total;
};

struct SliceTableF {
    const float4 *slots;    // [cap][1 + nf4] float4; slot word 0 holds the key
    unsigned mask;
    int shift32;            // 32 - log2(cap)
    int nf4;                // value float4 per slot: 1 (nv <= 4) or 2 (nv <= 8)
};

__host__ __device__ __forceinline__ unsigned slot_hash32(unsigned long long key, int shift32) {
    const unsigned k = (unsigned)key ^ (unsigned)(key >> 32) * 0x85EBCA6Bu;
    return (k * 0x9E3779B1u) >> shift32;
}

struct QSimplex3 {
    unsigned long long key[4];
    float bary[4];
    int overflow;
};

__device__ __forceinline__ void qsimplex3(const double *el, QSimplex3 &q) {
    constexpr long long kLim = kKeyLim / 4 - 2;
    double r[4];
    float d[4];
    int ri[4];
    q.overflow = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        r[i] = rint(el[i] * 0.25);
        q.overflow |= !(fabs(r[i]) < (double)kLim);
        ri[i] = (int)r[i];
        d[i] = (float)fma(-4.0, r[i], el[i]);     // el - rem0, exact product
    }
    int rank[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int rk = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (j == i) continue;
            rk += (d[j] > d[i]) || (j < i && d[j] == d[i]);
        }
        rank[i] = rk;
    }
    const int h = ri[0] + ri[1] + ri[2] + ri[3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int rk = rank[i] + h;
        if (rk < 0) { rk += 4; ri[i] += 1; d[i] -= 4.0f; }
        else if (rk > 3) { rk -= 4; ri[i] -= 1; d[i] += 4.0f; }
        rank[i] = rk;
    }
    float sv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float v = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) v = (rank[i] == k) ? d[i] : v;
        sv[k] = 0.25f * v;
    }
    q.bary[0] = 1.0f + sv[3] - sv[0];
#pragma unroll
    for (int l = 1; l < 4; ++l) q.bary[l] = sv[3 - l] - sv[4 - l];
    // packed(rem0 + canonical[l]) = packed(rem0) + l*U - 4*B_l, B_l = sum of the
    // field units of the coordinates whose rank exceeds 3 - l (fields never borrow)
    const unsigned long long unit[3] = {1ull << (2 * kKeyBits), 1ull << kKeyBits, 1ull};
    unsigned long long p0 = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) p0 += (unsigned long long)(4 * ri[i] + kKeyOff) * unit[i];
    const unsigned long long U = unit[0] + unit[1] + unit[2];
    unsigned long long B = 0;
    q.key[0] = p0;
#pragma unroll
    for (int l = 1; l < 4; ++l) {
#pragma unroll
        for (int i = 0; i < 3; ++i) B += (rank[i] == 4 - l) ? unit[i] : 0ull;
        q.key[l] = p0 + (unsigned long long)l * U - 4ull * B;
    }
}

// float32 simplex core: el = 4 * base + frac with `base` an exact integer offset
// per coordinate (from the float64 pose constant) and |frac| = O(cloud / sigma).
// Outputs the remainder-0 point / 4 (ri, wrapped), the stable descending ranks
// and the barycentric weights.  Vertex l has lattice coordinates
// 4 * (ri_i - [rank_i > 3 - l]) + l (the canonical simplex of
// permutohedral.py:140-160).
__device__ __forceinline__ void simplex3f_core(const float *frac, const int *base, int *ri,
                                               int *rank, float *bary) {
    float d[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float r = rintf(frac[i] * 0.25f);
        d[i] = fmaf(-4.0f, r, frac[i]);
        ri[i] = (int)r + base[i];
        rank[i] = 0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i + 1; j < 4; ++j) {
            if (d[j] > d[i]) ++rank[i];
            else ++rank[j];
        }
    const int h = ri[0] + ri[1] + ri[2] + ri[3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        // single wrap into [0, 3] (select form: no divergent branches)
        const int rk = rank[i] + h;
        const bool lo = rk < 0, hi = rk > 3;
        rank[i] = lo ? rk + 4 : (hi ? rk - 4 : rk);
        ri[i] += lo ? 1 : (hi ? -1 : 0);
        d[i] -= lo ? 4.0f : (hi ? -4.0f : 0.0f);
    }
    float sv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        float v = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) v = (rank[i] == k) ? d[i] : v;
        sv[k] = 0.25f * v;
    }
    bary[0] = 1.0f + sv[3] - sv[0];
#pragma unroll
    for (int l = 1; l < 4; ++l) bary[l] = sv[3 - l] - sv[4 - l];
}

// approximate float32 reciprocal (MUFU.RCP, ~1 ulp; no slow path)
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// dense float32 slice grid (d = 3, nv == 4): one float4 per (cell q =
// floor(k / 4) over the first three lattice coordinates, remainder class
// r = k mod 4); the fourth coordinate is implied by the zero sum.  A row holds
// gain * (sum y0, sum y1, sum y2, mass) -- the value columns [1, y] of
// estep.py:153-165 rotated so the pass forms float32 pairs without moves.
// The grid spans the sites' q box [a, b] padded by kDensePad cells per side:
// a query's pre-wrap remainder-0 cell ri and its final vertices differ by at
// most 2 per coordinate (vertex cells ri - 2 .. ri + 1), so every ri in
// [a - 1, b + 2] addresses inside the grid, and a point outside that range has
// no site among its vertices.  The fourth pad cell lets the pass clamp ri into
// [a - 2, b + 3] instead of branching: a clamped cell's vertices are all
// padding (zero rows), exactly as an out-of-range point has no site.
constexpr int kDensePad = 4;

struct DenseSliceF {
    const float4 *cells;    // [n0][n1][n2][4]
    int a[3];               // site q minimum per coordinate
    unsigned span[3];       // b - a + 1
    int s0, s1;             // cell strides of coordinates 0 and 1 (coordinate 2: 1)
};

// dense float64 slice grid, the float64 query path's table (same cells and
// padding as DenseSliceF): per (cell, remainder class) one 32-byte row
// gain * (sum y0, sum y1 | sum y2, mass) as two double2
struct DenseSliceD {
    const double2 *cells;   // [n0][n1][n2][4][2]
    int a[3];               // site q minimum per coordinate
    int n[3];               // padded extents (span + 2 * kDensePad)
    int s0, s1;             // cell strides of coordinates 0 and 1
    int r2;                 // double2 per row: 2 ([1, y]) or 4 ([1, y, n])
};

// float32 variant of qsimplex3 (packed keys for the hash-slot table)
__device__ __forceinline__ void qsimplex3f(const float *frac, const int *base, QSimplex3 &q) {
    constexpr int kLim = (int)(kKeyLim / 4 - 2);
    int ri[4], rank[4];
    simplex3f_core(frac, base, ri, rank, q.bary);
    q.overflow = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) q.overflow |= (ri[i] >= kLim) | (ri[i] <= -kLim);
    const unsigned long long unit[3] = {1ull << (2 * kKeyBits), 1ull << kKeyBits, 1ull};
    unsigned long long p0 = 0;
#pragma unroll
    for (int i = 0; i < 3; ++i) p0 += (unsigned long long)(4 * ri[i] + kKeyOff) * unit[i];
    const unsigned long long U = unit[0] + unit[1] + unit[2];
    unsigned long long B = 0;
    q.key[0] = p0;
#pragma unroll
    for (int l = 1; l < 4; ++l) {
#pragma unroll
        for (int i = 0; i < 3; ++i) B += (rank[i] == 4 - l) ? unit[i] : 0ull;
        q.key[l] = p0 + (unsigned long long)l * U - 4ull * B;
    }
}

template <int NF4>
__device__ __forceinline__ unsigned long long slot_key(const float4 *slot) {
    return __ldg(reinterpret_cast<const unsigned long long *>(slot));
}

// gather the 4 vertex rows of one simplex; absent vertices get zero rows
template <int NF4>
__device__ __forceinline__ void gather_simplex_f(const SliceTableF &t, const unsigned long long *key,
                                                 float4 (*v)[NF4]) {
    constexpr int W = 1 + NF4;   // float4 per slot (32 or 48 -> padded 64 bytes)
    constexpr int S = (W == 2) ? 2 : 4;
    unsigned h[4];
    unsigned long long k[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        h[l] = slot_hash32(key[l], t.shift32);
        const float4 *slot = t.slots + (size_t)h[l] * S;
        k[l] = slot_key<NF4>(slot);
#pragma unroll
        for (int f = 0; f < NF4; ++f) v[l][f] = __ldg(slot + 1 + f);
    }
#pragma unroll
    for (int l = 0; l < 4; ++l) {
        if (k[l] != key[l]) {
            bool hit = false;
            unsigned s = h[l];
            if (k[l] != kEmptyKey) {
                s = (s + 1) & t.mask;
                for (unsigned it = 0; it <= t.mask; ++it) {
                    const unsigned long long kk = slot_key<NF4>(t.slots + (size_t)s * S);
                    if (kk == key[l]) { hit = true; break; }
                    if (kk == kEmptyKey) break;
                    s = (s + 1) & t.mask;
                }
            }
#pragma unroll
            for (int f = 0; f < NF4; ++f)
                v[l][f] = hit ? __ldg(t.slots + (size_t)s * S + 1 + f) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
}

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
    unsigned long long *skeys = nullptr;
    double *svals = nullptr;
    unsigned smask = 0;
    int sshift = 0;
    int nvp = 0;
    fr::SliceTable table() const {
        return fr::SliceTable{skeys, svals, smask, sshift, nvp};
    }
    // interleaved float32 slice table (gain folded in) for the fast EM pass
    float4 *fslots = nullptr;
    unsigned fmask = 0;
    int fshift32 = 0;
    int nf4 = 0;
    fr::SliceTableF table_f() const {
        return fr::SliceTableF{fslots, fmask, fshift32, nf4};
    }
    // dense float32 slice grid (d = 3, nv <= 4, box small enough); null otherwise
    float4 *dcells = nullptr;
    fr::DenseSliceF dense{};
    long long dense_cells = 0;
    // dense float64 slice grid (same box; FR_DENSE64_MAX_CELLS) for the float64 EM loop
    double2 *dcells64 = nullptr;
    fr::DenseSliceD dense64{};
    long long dense64_cells = 0;
    // d >= 4: sorted 128-bit site keys (hi / lo words) and their codec
    unsigned long long *wkh = nullptr, *wkl = nullptr;
    fr::WideCodec wc{};
    // set by the device-resident blur (its one host read): the nonzero site
    // count after the last axis (-1: unknown) and, for d = 3, the q = k >> 2
    // box of those sites' first three coordinates (lo[3], hi[3])
    long long blur_keep = -1;
    int blur_box[6] = {0, 0, 0, 0, 0, 0};
    int box_valid = 0;
    // device counters / flags
    unsigned long long *d_counters = nullptr;   // [0] sites, [1] src count, [2] overflow
    cudaStream_t stream = nullptr;              // stream of the last build call (pool ordering)
};
