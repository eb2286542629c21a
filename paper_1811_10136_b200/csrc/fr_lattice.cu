// Permutohedral lattice on B200: deterministic splat, frontier-growing blur,
// slice table build, generic slice / simplex / brute-force kernels.
//
// Reference: permutohedral.py (pkg/src/twistreg).  The build reproduces the
// reference's site set and float64 values bit for bit:
//   * keys: fp64 embedding with the reference's operation order (fr_common.cuh)
//   * splat: entries are grouped per site by a stable radix sort of their hash
//     slot, then each site's contributions are summed sequentially in flat
//     (point, vertex) order -- exactly np.add.at's order (permutohedral.py:242)
//   * blur: Jacobi passes with the same fp64 expression (permutohedral.py:322)
//     and the same frontier materialisation + site cap (:304-313)
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <vector>

#include "fr_common.cuh"

namespace fr {

static thread_local char g_err[1024];

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

const char *last_error() { return g_err; }

static const double kScale[13] = {0, 1.00, 1.00, 1.05, 1.05, 1.05, 1.05,
                                  1.05, 1.10, 1.10, 1.05, 1.05, 1.05};
static const double kGain[13] = {0,
                                 2.8952044967493156, 7.26440867477451, 19.65543341118011,
                                 46.8204989056386,   109.10733236095797, 253.69798361851673,
                                 585.8878389979589,  1551.3475661281732, 3556.1187473560817,
                                 7167.31894204168,   16021.44046866235,  36206.979459505295};

int make_consts(int dim, const double *sigma, LatticeConsts *out) {
    if (dim < 1 || dim > kMaxDim) {
        set_error("lattice dimension %d outside 1..12", dim);   // permutohedral.py:148-149
        return FR_EINVAL;
    }
    memset(out, 0, sizeof(*out));
    out->dim = dim;
    for (int j = 0; j < dim; ++j) {
        if (!std::isfinite(sigma[j]) || !(sigma[j] > 0)) {
            set_error("kernel widths must be finite and positive");
            return FR_EINVAL;
        }
        out->sigma[j] = sigma[j];
    }
    // s_d = sqrt(2/3) * (d+1) * SCALE[d]; sf[j] = s_d / sqrt((j+1)(j+2))
    const double sd = std::sqrt(2.0 / 3.0) * (double)(dim + 1) * kScale[dim];
    for (int j = 0; j < dim; ++j) out->sf[j] = sd / std::sqrt((double)((j + 1) * (j + 2)));
    out->gain = kGain[dim];
    return FR_OK;
}

// ---------------------------------------------------------------------------
// device helpers

struct BuildHash {
    unsigned long long *keys;
    int *site;
    unsigned mask;
};

// returns slot, or -1 when the table is full; *created = 1 for the CAS winner
__device__ __forceinline__ int hash_insert(BuildHash h, unsigned long long key, int *created) {
    unsigned s = (unsigned)mix64(key) & h.mask;
    *created = 0;
    for (unsigned it = 0; it <= h.mask; ++it) {
        unsigned long long k = h.keys[s];
        if (k == key) return (int)s;
        if (k == kEmptyKey) {
            unsigned long long prev = atomicCAS(&h.keys[s], kEmptyKey, key);
            if (prev == kEmptyKey) { *created = 1; return (int)s; }
            if (prev == key) return (int)s;
        }
        s = (s + 1) & h.mask;
    }
    return -1;
}

__device__ __forceinline__ int hash_find(BuildHash h, unsigned long long key) {
    unsigned s = (unsigned)mix64(key) & h.mask;
    for (unsigned it = 0; it <= h.mask; ++it) {
        unsigned long long k = h.keys[s];
        if (k == key) return h.site[s];
        if (k == kEmptyKey) return -1;
        s = (s + 1) & h.mask;
    }
    return -1;
}

// value sources ------------------------------------------------------------

struct GenericSrc {
    const double *F;   // n x D
    const double *V;   // n x nv
    int nv;
    template <int D>
    __device__ __forceinline__ void feat(long long p, double *f) const {
#pragma unroll
        for (int j = 0; j < D; ++j) f[j] = F[p * D + j];
    }
    __device__ __forceinline__ double value(long long p, int c) const { return V[p * nv + c]; }
};

// [1, y, (|y|^2), (n)] from float32 or float64 SoA planes (estep.py:153-165)
template <class T>
struct PointSrcT {
    const T *pos;       // 3 planes of n
    const T *nrm;       // 3 planes of n or null
    long long n;
    int m2;             // 1 when the |y|^2 column is present
    int nv;
    template <int D>
    __device__ __forceinline__ void feat(long long p, double *f) const {
#pragma unroll
        for (int j = 0; j < D; ++j) f[j] = (double)pos[j * n + p];
    }
    __device__ __forceinline__ double value(long long p, int c) const {
        if (c == 0) return 1.0;
        if (c <= 3) return (double)pos[(c - 1) * n + p];
        if (m2 && c == 4) {
            double y0 = pos[p], y1 = pos[n + p], y2 = pos[2 * n + p];
            // np.einsum("nd,nd->n") on 3-vectors sums (y0^2 + y2^2) + y1^2
            return __dadd_rn(__dadd_rn(__dmul_rn(y0, y0), __dmul_rn(y2, y2)), __dmul_rn(y1, y1));
        }
        int k = c - 4 - m2;
        return (double)nrm[k * n + p];
    }
};
using PointSrc = PointSrcT<float>;
using PointSrc64 = PointSrcT<double>;

// splat phase 1: embed, insert keys, record (slot, bary) per (point, vertex)
template <int D, class Src>
__global__ void k_splat_entries(Src src, long long p0, long long p1, long long n_all,
                                LatticeConsts c, BuildHash h,
                                unsigned sentinel, unsigned *entry_slot, unsigned *entry_idx,
                                double *entry_bary, double *contrib, unsigned long long *counters,
                                unsigned *created_list) {
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long p = p0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; p < p1; p += stride) {
        double f[D];
        src.template feat<D>(p, f);
        Simplex<D> s;
        simplex_exact<D>(f, c, s);
        if (s.overflow) atomicOr(&counters[2], 1ull);
        bool any_value = false;
        for (int cc = 0; cc < src.nv; ++cc) any_value |= (src.value(p, cc) != 0.0);
        // the vertices' home slots probed together (their keys are mostly
        // present already: one L2 round trip for the four, not four in a
        // row); a miss takes the full insert
        unsigned long long key[D + 1], home[D + 1];
        unsigned hs[D + 1];
#pragma unroll
        for (int l = 0; l <= D; ++l) {
            key[l] = s.packed(l);
            hs[l] = (unsigned)mix64(key[l]) & h.mask;
        }
#pragma unroll
        for (int l = 0; l <= D; ++l) home[l] = __ldcg(h.keys + hs[l]);
#pragma unroll
        for (int l = 0; l <= D; ++l) {
            long long e = p * (D + 1) + l;
            unsigned slot = sentinel;
            if (s.bary[l] != 0.0 && any_value && !s.overflow) {
                if (home[l] == key[l]) {
                    slot = hs[l];
                } else {
                    int created;
                    int sl = hash_insert(h, key[l], &created);
                    if (sl < 0) atomicOr(&counters[2], 2ull);
                    else {
                        slot = (unsigned)sl;
                        if (created) {
                            // the occupied slots, listed (capacity h.mask / 2 + 1:
                            // beyond it the table is reported full anyway)
                            const unsigned long long q = atomicAdd(&counters[0], 1ull);
                            if (q <= (h.mask >> 1)) created_list[q] = (unsigned)sl;
                        }
                    }
                }
            }
            entry_slot[e] = slot;
            entry_idx[e] = (unsigned)e;
            if (!contrib) entry_bary[e] = s.bary[l];      // the product rows carry it
            // the entry's products bary * value (NumPy's single rounding), one
            // row per entry, vertex-major ([l][p] rows): a site's entries share
            // their vertex index l, so for spatially ordered points its rows
            // are near-contiguous for the site sums' gathers
            if (contrib && slot != sentinel)
                for (int cc = 0; cc < src.nv; ++cc)
                    contrib[((size_t)l * n_all + p) * src.nv + cc] =
                        __dmul_rn(s.bary[l], src.value(p, cc));
        }
    }
}

// splat phase 2: one block per site.  All threads form 256 contributions
// bary * value at a time (one rounding each, as NumPy's product) into a
// kSegStages-deep shared-memory ring; lane c of warp 0 adds column c in flat
// (point, vertex) order -- np.add.at's accumulation order
// (permutohedral.py:241-242), hence bit-identical sums -- while the other
// threads already gather the following chunks.  A heavy site (10^5-10^6
// entries at C5 sizes) is then bound by its one float64 add chain per column,
// not by the latency of its random gathers.
constexpr int kSegBlock = 256;

// the per-entry product rows take E * nv doubles of pool memory: formed in the
// entries kernel when that stays within 8 GiB, else in the site-sum kernel
static inline bool contrib_fits(long long E, int nv) {
    return (unsigned long long)E * (unsigned long long)nv * 8ull <= (8ull << 30);
}
constexpr int kSegStages = 3;

// contrib != null: the entries' products were formed by the entries kernel
// (point-coalesced) and are gathered as rows; else formed here from the
// point values (random gathers of bary and coordinates)
template <int D, class Src>
__global__ void __launch_bounds__(kSegBlock)
k_splat_segsum(Src src, const unsigned *run_slot, const int *run_off, const int *run_cnt,
               const unsigned *sorted_idx, const double *entry_bary, const double *contrib,
               unsigned sentinel, int nv, double *run_vals, long long lmajor_n = 0) {
    extern __shared__ double ring[];   // [kSegStages][kSegBlock][nv]
    const int r = blockIdx.x;
    if (run_slot && run_slot[r] == sentinel) return;   // (null: no sentinel runs)
    const int beg = run_off[r], cnt = run_cnt[r];
    const int chunks = (cnt + kSegBlock - 1) / kSegBlock;
    const int t = threadIdx.x;
    auto stage = [&](int ch) {
        const int j = ch * kSegBlock + t;
        if (j < cnt) {
            const unsigned e = sorted_idx[beg + j];
            double *row = ring + ((size_t)(ch % kSegStages) * kSegBlock + t) * nv;
            if (contrib) {
                // rows [l][p] (lmajor_n = point count) or [p][l] (0)
                const size_t rix = lmajor_n ? (size_t)(e % (D + 1)) * lmajor_n + e / (D + 1) : e;
                const double *cr = contrib + rix * nv;
                for (int c = 0; c < nv; ++c) row[c] = __ldg(cr + c);
            } else {
                const double b = entry_bary[e];
                const long long p = e / (D + 1);
                for (int c = 0; c < nv; ++c) row[c] = __dmul_rn(b, src.value(p, c));
            }
        }
    };
    for (int st = 0; st < kSegStages - 1 && st < chunks; ++st) stage(st);
    __syncthreads();
    double acc = 0.0;
    for (int ch = 0; ch < chunks; ++ch) {
        if (ch + kSegStages - 1 < chunks) stage(ch + kSegStages - 1);
        if (t < nv) {
            const double *col = ring + (size_t)(ch % kSegStages) * kSegBlock * nv + t;
            const int n = min(kSegBlock, cnt - ch * kSegBlock);
            int i = 0;
            for (; i + 8 <= n; i += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = col[(i + u) * nv];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
            }
            for (; i < n; ++i) acc = __dadd_rn(acc, col[i * nv]);
        }
        __syncthreads();
    }
    if (t < nv) run_vals[(long long)r * nv + t] = acc;
}

// splat phase 2, fixed-tree order (the point splats of the EM path).  Each
// site's sorted entries are cut into pieces of kSegPiece; one block per piece
// (a heavy site -- 2e4 entries at C5 1M -- spreads over many SMs): every
// thread gathers one entry row per 256-entry chunk (the next chunk's row
// prefetched into registers), each warp sums its 32 rows per column by a
// shuffle tree, the 8 warp sums add in warp order, the chunk sums in chunk
// order; k_seg_pieces_combine adds a site's piece sums in piece order.
// Deterministic (no atomics, no scheduling-dependent order) but not
// np.add.at's flat order: site sums differ from it by float64 round-off (the
// reference's own sums carry the same order of error).
constexpr int kSegPiece = 1024;

template <int NV>
__device__ __forceinline__ void seg_row(const unsigned *sorted_idx, const double *contrib,
                                        long long lmajor_n, int D1, int beg, int j, int cnt,
                                        double (&v)[NV]) {
    if (j < cnt) {
        const unsigned e = sorted_idx[beg + j];
        const size_t rix = lmajor_n ? (size_t)(e % D1) * lmajor_n + e / D1 : e;
        const double *cr = contrib + rix * NV;
#pragma unroll
        for (int c = 0; c < NV; ++c) v[c] = __ldg(cr + c);
    } else {
#pragma unroll
        for (int c = 0; c < NV; ++c) v[c] = 0.0;
    }
}

// pieces per run (0 for the sentinel run)
__global__ void k_seg_piece_counts(int n_runs, const unsigned *run_slot, unsigned sentinel,
                                   const int *run_cnt, int *pieces) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_runs) return;
    const bool skip = run_slot && run_slot[r] == sentinel;
    pieces[r] = skip ? 0 : (run_cnt[r] + kSegPiece - 1) / kSegPiece;
}

template <int D, int NV>
__global__ void __launch_bounds__(kSegBlock)
k_splat_segsum_tree(int n_runs, const int *piece_off, const int *run_off, const int *run_cnt,
                    const unsigned *sorted_idx, const double *contrib, double *piece_vals,
                    long long lmajor_n) {
    constexpr int W = kSegBlock / 32;
    __shared__ double wsum[W][NV];
    __shared__ int s_run;
    const int pc = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) {
        // the run owning piece pc: last r with piece_off[r] <= pc
        int lo = 0, hi = n_runs;          // piece_off has n_runs + 1 entries
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (piece_off[mid] <= pc) lo = mid;
            else hi = mid;
        }
        s_run = pc < piece_off[n_runs] ? lo : -1;
    }
    __syncthreads();
    const int r = s_run;
    if (r < 0) return;
    const int j0 = (pc - piece_off[r]) * kSegPiece;
    const int beg = run_off[r] + j0, cnt = min(kSegPiece, run_cnt[r] - j0);
    double cur[NV], nxt[NV];
    seg_row<NV>(sorted_idx, contrib, lmajor_n, D + 1, beg, t, cnt, cur);
    double acc = 0.0;
    for (int base = 0; base < cnt; base += kSegBlock) {
        seg_row<NV>(sorted_idx, contrib, lmajor_n, D + 1, beg, base + kSegBlock + t, cnt, nxt);
#pragma unroll
        for (int c = 0; c < NV; ++c) {
            double v = cur[c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) wsum[warp][c] = v;
        }
        __syncthreads();
        if (t < NV) {
            double sc = wsum[0][t];
#pragma unroll
            for (int w = 1; w < W; ++w) sc += wsum[w][t];
            acc += sc;
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < NV; ++c) cur[c] = nxt[c];
    }
    if (t < NV) piece_vals[(long long)pc * NV + t] = acc;
}

// run_vals[r] = its pieces' sums in piece order (zero for the sentinel run)
__global__ void k_seg_pieces_combine(int n_runs, const int *piece_off, const double *piece_vals,
                                     int nv, double *run_vals) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)n_runs * nv) return;
    const int r = (int)(q / nv), c = (int)(q % nv);
    double acc = 0.0;
    for (int p = piece_off[r]; p < piece_off[r + 1]; ++p) acc += piece_vals[(long long)p * nv + c];
    run_vals[q] = acc;
}

// dense site ids for the sort keys: the occupied hash slots (listed as they
// are created) sorted ascending, id = rank (sc_site_ids); entry keys are
// rewritten slot -> id (the sentinel -> K, after every id), so the radix sort
// runs over 1 + floor(log2 K) bits instead of the hash's log2(cap) + 1; the
// runs' ids are mapped back to slots afterwards
__global__ void k_entries_to_ids(long long E, unsigned sentinel, unsigned K, const int *ids,
                                 unsigned *entry_key) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E;
         e += (long long)gridDim.x * blockDim.x) {
        const unsigned sl = entry_key[e];
        entry_key[e] = sl == sentinel ? K : (unsigned)ids[sl];
    }
}

// row K of the run arrays as an empty sentinel run (overwritten by the RLE
// when the sentinel run exists)
__global__ void k_run_pad(unsigned K, unsigned sentinel, unsigned *run_slot, int *run_cnt) {
    if (threadIdx.x == 0) {
        run_slot[K] = sentinel;
        run_cnt[K] = 0;
    }
}

__global__ void k_runs_to_slots(const int *d_nruns, unsigned K, unsigned sentinel,
                                const int *slot_of_id, unsigned *run_slot) {
    const int nr = *d_nruns;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nr; r += gridDim.x * blockDim.x) {
        const unsigned id = run_slot[r];
        run_slot[r] = id >= K ? sentinel : (unsigned)slot_of_id[id];
    }
}

// ---------------------------------------------------------------------------
// warp-aggregated splat (spatially ordered points: the EM path's Morton-
// sorted observation copies).  A warp takes 32 consecutive points; per
// simplex vertex the lanes whose vertex hits the same site (match_any) fold
// their products bary * value in lane order into the group's lowest lane,
// which emits ONE (site slot, warp-vertex index, sums) pair.  For Morton-
// ordered points a warp's 32 points share one or two simplices, so the
// pairs are ~1/20 of the entries: the sort and the site sums run over pairs.
// Deterministic: the pairs are sorted by (site id, warp-vertex index) before
// the fixed-order tree sums, whatever order the warps appended them in.
template <int D, int NV, class Src>
__global__ void __launch_bounds__(256)
k_splat_warp_pairs(Src src, long long n, LatticeConsts c, BuildHash h, unsigned *pair_slot,
                   unsigned *pair_lo, double *pair_vals, long long max_pairs,
                   unsigned long long *counters, unsigned *created_list) {
    constexpr unsigned FULL = 0xffffffffu, kNone = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w * 32 < n;
         w += nwarps) {
        const long long p = w * 32 + lane;
        const bool inb = p < n;
        Simplex<D> sx;
        double v[NV];
        bool any_value = false, ovf = false;
        if (inb) {
            double f[D];
            src.template feat<D>(p, f);
            simplex_exact<D>(f, c, sx);
            ovf = sx.overflow;
            if (ovf) atomicOr(&counters[2], 1ull);
#pragma unroll
            for (int cc = 0; cc < NV; ++cc) {
                v[cc] = src.value(p, cc);
                any_value |= v[cc] != 0.0;
            }
        } else {
#pragma unroll
            for (int cc = 0; cc < NV; ++cc) v[cc] = 0.0;
        }
#pragma unroll
        for (int l = 0; l <= D; ++l) {
            unsigned slot = kNone;
            if (inb && !ovf && any_value && sx.bary[l] != 0.0) {
                const unsigned long long key = sx.packed(l);
                const unsigned hs = (unsigned)mix64(key) & h.mask;
                if (__ldcg(h.keys + hs) == key) {
                    slot = hs;
                } else {
                    int created;
                    const int sl = hash_insert(h, key, &created);
                    if (sl < 0) atomicOr(&counters[2], 2ull);
                    else {
                        slot = (unsigned)sl;
                        if (created) {
                            const unsigned long long q = atomicAdd(&counters[0], 1ull);
                            if (q <= (h.mask >> 1)) created_list[q] = (unsigned)sl;
                        }
                    }
                }
            }
            const unsigned mask = __match_any_sync(FULL, slot);
            double cv[NV], acc[NV];
#pragma unroll
            for (int cc = 0; cc < NV; ++cc) {
                cv[cc] = slot != kNone ? __dmul_rn(sx.bary[l], v[cc]) : 0.0;
                acc[cc] = 0.0;
            }
            // fold each group's rows: when every group is a contiguous run of
            // lanes (the rule for spatially ordered points) a segmented
            // shuffle tree (fixed shape given the runs); else the members in
            // lane order (all lanes shuffle in lockstep, each from its own
            // group's next member)
            const int lo = __ffs(mask) - 1;
            const unsigned run = mask >> lo;
            const bool contiguous = slot == kNone || (run & (run + 1u)) == 0u;
            if (__all_sync(FULL, contiguous)) {
                const int end = lo + __popc(mask);
#pragma unroll
                for (int cc = 0; cc < NV; ++cc) acc[cc] = cv[cc];
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                    for (int cc = 0; cc < NV; ++cc) {
                        const double x = __shfl_down_sync(FULL, acc[cc], o);
                        if (lane + o < end) acc[cc] = __dadd_rn(acc[cc], x);
                    }
                }
            } else {
                unsigned rem = slot != kNone ? mask : 0u;
                while (__any_sync(FULL, rem != 0u)) {
                    const int from = rem ? __ffs(rem) - 1 : lane;
#pragma unroll
                    for (int cc = 0; cc < NV; ++cc) {
                        const double x = __shfl_sync(FULL, cv[cc], from);
                        if (rem) acc[cc] = __dadd_rn(acc[cc], x);
                    }
                    rem &= rem - 1u;
                }
            }
            const bool leader = slot != kNone && __ffs(mask) - 1 == lane;
            const unsigned lead = __ballot_sync(FULL, leader);
            unsigned long long base = 0;
            if (lane == 0 && lead) base = atomicAdd(&counters[3], (unsigned long long)__popc(lead));
            base = __shfl_sync(FULL, base, 0);
            if (leader) {
                const unsigned long long pos = base + __popc(lead & ((1u << lane) - 1u));
                if ((long long)pos < max_pairs) {
                    pair_slot[pos] = slot;
                    pair_lo[pos] = (unsigned)(w * (D + 1) + l);
#pragma unroll
                    for (int cc = 0; cc < NV; ++cc) pair_vals[pos * NV + cc] = acc[cc];
                } else {
                    atomicOr(&counters[2], 4ull);     // pair buffer full: caller falls back
                }
            }
        }
    }
}

// site ids: the occupied slots sorted ascending, ids[slot] = rank (the same
// numbering as flags + scan over the table, without touching empty slots)
__global__ void k_scatter_ids(unsigned K, const unsigned *sorted_slots, int *ids) {
    for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < K; i += gridDim.x * blockDim.x)
        ids[sorted_slots[i]] = (int)i;
}

// sort keys (site id << lo_bits) | warp-vertex index, and the identity values
__global__ void k_pair_keys(long long np, const unsigned *pair_slot, const unsigned *pair_lo,
                            const int *ids, int lo_bits, unsigned long long *keys, unsigned *idx) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < np;
         i += (long long)gridDim.x * blockDim.x) {
        keys[i] = ((unsigned long long)ids[pair_slot[i]] << lo_bits) | pair_lo[i];
        idx[i] = (unsigned)i;
    }
}

__global__ void k_key_ids(long long np, const unsigned long long *keys, int lo_bits,
                          unsigned *out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < np;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = (unsigned)(keys[i] >> lo_bits);
}

__global__ void k_run_live(int n_runs, const unsigned *run_slot, unsigned sentinel,
                           const double *run_vals, int nv, unsigned char *run_live) {
    int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_runs) return;
    bool live = false;
    if (!run_slot || run_slot[r] != sentinel)
        for (int c = 0; c < nv; ++c) live |= run_vals[(long long)r * nv + c] != 0.0;
    run_live[r] = live;
}

template <int D>
__global__ void k_fill_sites(int S, const int *live_runs, const unsigned *run_slot,
                             const unsigned long long *hkeys, const double *run_vals, int nv,
                             int *site_keys, double *vals) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    int r = live_runs[i];
    int k[D + 1];
    unpack_key<D>(hkeys[run_slot[r]], k);
#pragma unroll
    for (int q = 0; q <= D; ++q) site_keys[(long long)i * (D + 1) + q] = k[q];
    for (int cc = 0; cc < nv; ++cc) vals[(long long)i * nv + cc] = run_vals[(long long)r * nv + cc];
}

template <int D>
__global__ void k_hash_sites(long long S, const int *site_keys, BuildHash h,
                             unsigned long long *counters) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    int created;
    int sl = hash_insert(h, pack_key<D>(site_keys + i * (D + 1)), &created);
    if (sl < 0) { atomicOr(&counters[2], 2ull); return; }
    h.site[sl] = (int)i;
}

__global__ void k_count_nonzero(long long S, const double *vals, int nv,
                                unsigned long long *counter) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool nz = false;
    if (i < S)
        for (int c = 0; c < nv; ++c) nz |= vals[i * nv + c] != 0.0;
    unsigned ballot = __ballot_sync(0xffffffffu, nz);
    if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(counter, (unsigned long long)__popc(ballot));
}

__global__ void k_nonzero_flags(long long S, const double *vals, int nv, unsigned char *flags) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    bool nz = false;
    for (int c = 0; c < nv; ++c) nz |= vals[i * nv + c] != 0.0;
    flags[i] = nz;
}

// blur: materialise the +-1 neighbours along `axis` of every non-zero site
template <int D>
__global__ void k_extend(long long S, int axis, const double *vals, int nv, BuildHash h,
                         int *site_keys, unsigned long long *counters) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    bool nz = false;
    for (int c = 0; c < nv; ++c) nz |= vals[i * nv + c] != 0.0;
    if (!nz) return;
    int k[D + 1];
#pragma unroll
    for (int q = 0; q <= D; ++q) k[q] = site_keys[i * (D + 1) + q];
#pragma unroll
    for (int sgn = -1; sgn <= 1; sgn += 2) {
        int nk[D + 1];
#pragma unroll
        for (int q = 0; q <= D; ++q) nk[q] = k[q] + sgn;
        nk[axis] -= sgn * (D + 1);
        bool ok = true;
#pragma unroll
        for (int q = 0; q < D; ++q) ok &= (nk[q] > -kKeyLim) && (nk[q] < kKeyLim);
        if (!ok) { atomicOr(&counters[2], 1ull); continue; }
        int created;
        int sl = hash_insert(h, pack_key<D>(nk), &created);
        if (sl < 0) { atomicOr(&counters[2], 2ull); continue; }
        if (created) {
            long long id = (long long)atomicAdd(&counters[0], 1ull);
            h.site[sl] = (int)id;
#pragma unroll
            for (int q = 0; q <= D; ++q) site_keys[id * (D + 1) + q] = nk[q];
        }
    }
}

// blur: one Jacobi [1,2,1]/4 pass, 0.5*v + 0.25*(v_up + v_dn) (permutohedral.py:314-322)
template <int D>
__global__ void k_jacobi(long long S, int axis, const int *site_keys, const double *vin,
                         double *vout, int nv, BuildHash h) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    int k[D + 1], up[D + 1], dn[D + 1];
#pragma unroll
    for (int q = 0; q <= D; ++q) k[q] = site_keys[i * (D + 1) + q];
#pragma unroll
    for (int q = 0; q <= D; ++q) { up[q] = k[q] + 1; dn[q] = k[q] - 1; }
    up[axis] = k[axis] - D;
    dn[axis] = k[axis] + D;
    int iu = hash_find(h, pack_key<D>(up));
    int id = hash_find(h, pack_key<D>(dn));
    for (int c = 0; c < nv; ++c) {
        double vu = iu >= 0 ? vin[(long long)iu * nv + c] : 0.0;
        double vd = id >= 0 ? vin[(long long)id * nv + c] : 0.0;
        vout[i * nv + c] = __dadd_rn(__dmul_rn(0.5, vin[i * nv + c]),
                                     __dmul_rn(0.25, __dadd_rn(vu, vd)));
    }
}

// the device-resident blur as ONE cooperative launch (no host round trip per
// axis): per axis the reference's extension decision (taken by every CTA
// from the same counts), the extension, and the Jacobi pass (which also
// counts the next axis's nonzero inputs), separated by 2 grid barriers (8 in
// all for d = 3) instead of launches.  The site count lives in counters[0],
// error flags in counters[2], nonzero counts per axis in nz[axis]; site rows
// past the count stay zero in both value buffers (zeroed once up front; the
// Jacobi pass writes rows < count).
__device__ __forceinline__ void blur_grid_sync(unsigned *bar, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            if (v < target) __nanosleep(20);
        } while (v < target);
    }
    __syncthreads();
}

// the cooperative blur's scratch: nz[0..n_nz), the barrier word, the box
__global__ void k_blur_scratch_init(unsigned long long *nz, int n_nz, int *box) {
    const int t = threadIdx.x;
    if (t < n_nz) nz[t] = 0ull;
    if (t < 6) box[t] = t < 3 ? INT_MAX : INT_MIN;
}

template <int D>
__global__ void __launch_bounds__(256)
k_blur_coop(double *vals, double *vals_alt, int nv, BuildHash h, int *site_keys,
            unsigned long long *ctr, unsigned long long *nz, long long cap, unsigned *bar,
            int *box) {
    const unsigned nb = gridDim.x;
    unsigned phase = 0;
    const long long tid0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    double *vin = vals, *vout = vals_alt;
    for (int axis = 0; axis <= D; ++axis) {
        // the axis's input site count: nothing changes ctr[0] until the
        // extension below, which every CTA reaches only after the barrier
        const long long S_in = (long long)*(volatile unsigned long long *)&ctr[0];
        // nonzero sites of this axis's input (axis > 0: counted by the
        // previous axis's Jacobi pass as it wrote them)
        if (axis == 0) {
            const long long S = S_in;
            unsigned long long mine = 0;
            for (long long i = tid0; i < S; i += stride) {
                bool z = false;
                for (int c = 0; c < nv; ++c) z |= vin[i * nv + c] != 0.0;
                mine += z;
            }
            for (int o = 16; o > 0; o >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, o);
            if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&nz[axis], mine);
        }
        if (axis == 0) blur_grid_sync(bar, nb * ++phase);
        {
            // permutohedral.py:304-306: extend only while S + 2 nsrc <= cap
            // (decided by every CTA from the same counts: no extra barrier)
            const unsigned long long nsrc = *(volatile unsigned long long *)&nz[axis];
            const long long S = ((unsigned long long)S_in + 2 * nsrc <= (unsigned long long)cap &&
                                 nsrc > 0) ? S_in : 0;
            for (long long i = tid0; i < S; i += stride) {
                bool z = false;
                for (int c = 0; c < nv; ++c) z |= vin[i * nv + c] != 0.0;
                if (!z) continue;
                int k[D + 1];
#pragma unroll
                for (int q = 0; q <= D; ++q) k[q] = site_keys[i * (D + 1) + q];
#pragma unroll
                for (int sgn = -1; sgn <= 1; sgn += 2) {
                    int nk[D + 1];
#pragma unroll
                    for (int q = 0; q <= D; ++q) nk[q] = k[q] + sgn;
                    nk[axis] -= sgn * (D + 1);
                    bool ok = true;
#pragma unroll
                    for (int q = 0; q < D; ++q) ok &= (nk[q] > -kKeyLim) && (nk[q] < kKeyLim);
                    if (!ok) { atomicOr(&ctr[2], 1ull); continue; }
                    int created;
                    const int sl = hash_insert(h, pack_key<D>(nk), &created);
                    if (sl < 0) { atomicOr(&ctr[2], 2ull); continue; }
                    if (created) {
                        const long long id = (long long)atomicAdd(&ctr[0], 1ull);
                        h.site[sl] = (int)id;
#pragma unroll
                        for (int q = 0; q <= D; ++q) site_keys[id * (D + 1) + q] = nk[q];
                    }
                }
            }
        }
        blur_grid_sync(bar, nb * ++phase);
        {
            const long long S = (long long)*(volatile unsigned long long *)&ctr[0];
            unsigned long long mine = 0;
            int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
            for (long long i = tid0; i < S; i += stride) {
                int k[D + 1], up[D + 1], dn[D + 1];
#pragma unroll
                for (int q = 0; q <= D; ++q) k[q] = site_keys[i * (D + 1) + q];
#pragma unroll
                for (int q = 0; q <= D; ++q) { up[q] = k[q] + 1; dn[q] = k[q] - 1; }
                up[axis] = k[axis] - D;
                dn[axis] = k[axis] + D;
                const int iu = hash_find(h, pack_key<D>(up));
                const int id = hash_find(h, pack_key<D>(dn));
                bool z = false;
                for (int c = 0; c < nv; ++c) {
                    const double vu = iu >= 0 ? vin[(long long)iu * nv + c] : 0.0;
                    const double vd = id >= 0 ? vin[(long long)id * nv + c] : 0.0;
                    const double o = __dadd_rn(__dmul_rn(0.5, vin[i * nv + c]),
                                               __dmul_rn(0.25, __dadd_rn(vu, vd)));
                    vout[i * nv + c] = o;
                    z |= o != 0.0;
                }
                mine += z;
                if (D == 3 && axis == D && z) {
#pragma unroll
                    for (int c = 0; c < 3 && c <= D; ++c) {
                        lo[c] = min(lo[c], k[c] >> 2);
                        hi[c] = max(hi[c], k[c] >> 2);
                    }
                }
            }
            // the next axis's nonzero input count; after the last axis the
            // nonzero rows that survive the final drop (nz[D + 1]) and their box
            for (int o = 16; o > 0; o >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, o);
            if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&nz[axis + 1], mine);
            if (D == 3 && axis == D) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        lo[c] = min(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
                        hi[c] = max(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
                    }
                    if ((threadIdx.x & 31) == 0 && lo[c] <= hi[c]) {
                        atomicMin(box + c, lo[c]);
                        atomicMax(box + 3 + c, hi[c]);
                    }
                }
            }
        }
        if (axis < D) blur_grid_sync(bar, nb * ++phase);   // the kernel's end orders the last
        double *t = vin;
        vin = vout;
        vout = t;
    }
}

template <int D>
__global__ void k_gather_sites(int S, const int *idx, const int *kin, const double *vin,
                               int nv, int *kout, double *vout) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    int j = idx[i];
#pragma unroll
    for (int q = 0; q <= D; ++q) kout[(long long)i * (D + 1) + q] = kin[(long long)j * (D + 1) + q];
    for (int c = 0; c < nv; ++c) vout[(long long)i * nv + c] = vin[(long long)j * nv + c];
}

template <int D>
__global__ void k_slice_insert(long long S, const int *site_keys, const double *vals, int nv,
                               unsigned long long *skeys, double *svals, int nvp, unsigned mask,
                               int shift, unsigned long long *counters) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    unsigned long long key = pack_key<D>(site_keys + i * (D + 1));
    unsigned s = slot_hash(key, shift);
    for (unsigned it = 0; it <= mask; ++it) {
        unsigned long long prev = atomicCAS(&skeys[s], kEmptyKey, key);
        if (prev == kEmptyKey) {
            for (int c = 0; c < nvp; ++c) svals[(size_t)s * nvp + c] = c < nv ? vals[i * nv + c] : 0.0;
            return;
        }
        s = (s + 1) & mask;
    }
    atomicOr(&counters[2], 2ull);
}

// generic slice (permutohedral.py:329-341): gain * sum_l bary_l * value(key_l),
// NV value columns handled per launch (columns [c0, c0 + NV) of the row)
template <int D, int NV>
__global__ void k_slice_generic(const double *Q, long long m, LatticeConsts c, SliceTable t,
                                int c0, int nv_out, double *out) {
    long long stride = (long long)gridDim.x * blockDim.x;
    SliceTable tc = t;
    tc.vals = t.vals + c0;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < m; p += stride) {
        double f[D];
#pragma unroll
        for (int j = 0; j < D; ++j) f[j] = Q[p * D + j];
        Simplex<D> s;
        simplex_exact<D>(f, c, s);
        double acc[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) acc[q] = 0.0;
        if (!s.overflow) {
            unsigned long long key[D + 1];
#pragma unroll
            for (int l = 0; l <= D; ++l) key[l] = s.packed(l);
            double v[D + 1][NV];
            bool hit[D + 1];
            gather_simplex<D, NV>(tc, key, v, hit);
#pragma unroll
            for (int l = 0; l <= D; ++l)
#pragma unroll
                for (int q = 0; q < NV; ++q)
                    acc[q] = hit[l] ? __dadd_rn(acc[q], __dmul_rn(s.bary[l], v[l][q])) : acc[q];
        }
#pragma unroll
        for (int q = 0; q < NV; ++q)
            if (c0 + q < nv_out) out[p * nv_out + c0 + q] = __dmul_rn(c.gain, acc[q]);
    }
}

template <int D>
__global__ void k_simplex(const double *F, long long n, LatticeConsts c, int *keys, double *bary,
                          unsigned long long *flag) {
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    double f[D];
#pragma unroll
    for (int j = 0; j < D; ++j) f[j] = F[p * D + j];
    Simplex<D> s;
    simplex_exact<D>(f, c, s);
    if (s.overflow) atomicOr(flag, 1ull);
#pragma unroll
    for (int l = 0; l <= D; ++l) {
        int k[D + 1];
        s.vertex(l, k);
#pragma unroll
        for (int q = 0; q <= D; ++q) keys[(p * (D + 1) + l) * (D + 1) + q] = k[q];
        bary[p * (D + 1) + l] = s.bary[l];
    }
}

// exact Gaussian transform (permutohedral.py:64-86), inputs staged in smem
constexpr int kBfTile = 128;
__global__ void k_bruteforce(const double *Q, long long m, const double *F, long long n, int d,
                             const double *V, int nv, LatticeConsts c, double *out) {
    extern __shared__ double sm[];
    double *sF = sm;                        // kBfTile x d
    double *sV = sm + kBfTile * d;          // kBfTile x nv
    long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double q[kMaxDim];
    for (int j = 0; j < d; ++j) q[j] = p < m ? __ddiv_rn(Q[p * d + j], c.sigma[j]) : 0.0;
    double acc[16];
    for (int k = 0; k < 16; ++k) acc[k] = 0.0;
    for (long long base = 0; base < n; base += kBfTile) {
        int cnt = (int)min((long long)kBfTile, n - base);
        __syncthreads();
        for (int t = threadIdx.x; t < cnt * d; t += blockDim.x) {
            int r = t / d, j = t % d;
            sF[t] = __ddiv_rn(F[(base + r) * d + j], c.sigma[j]);
        }
        for (int t = threadIdx.x; t < cnt * nv; t += blockDim.x) sV[t] = V[base * nv + t];
        __syncthreads();
        if (p < m) {
            for (int r = 0; r < cnt; ++r) {
                double d2 = 0.0;
                for (int j = 0; j < d; ++j) {
                    double df = q[j] - sF[r * d + j];
                    d2 += df * df;
                }
                double kv = exp(-0.5 * d2);
                for (int k = 0; k < nv; ++k) acc[k] += kv * sV[r * nv + k];
            }
        }
    }
    if (p < m)
        for (int k = 0; k < nv; ++k) out[p * nv + k] = acc[k];
}

// ---------------------------------------------------------------------------
// host side

static inline unsigned grid_for(long long n, int block = 256) {
    long long g = (n + block - 1) / block;
    return (unsigned)std::max<long long>(1, std::min<long long>(g, 1LL << 30));
}

// FR_SPLAT_TIMING=1: host wall-clock of the splat's phases (device-synchronised);
// FR_SPLAT_TIMING=2: host wall-clock only (no synchronisation: where the host
// thread waits)
struct PhaseClock {
    bool on, sync;
    cudaStream_t s;
    std::chrono::steady_clock::time_point t0;
    explicit PhaseClock(cudaStream_t st) : s(st) {
        const char *e = getenv("FR_SPLAT_TIMING");
        on = e != nullptr;
        sync = on && e[0] != '2';
        if (on) {
            if (sync) cudaStreamSynchronize(s);
            t0 = std::chrono::steady_clock::now();
        }
    }
    void lap(const char *what) {
        if (!on) return;
        if (sync) cudaStreamSynchronize(s);
        const auto t = std::chrono::steady_clock::now();
        fprintf(stderr, "[splat] %-14s %8.3f ms\n", what,
                std::chrono::duration<double, std::milli>(t - t0).count());
        t0 = t;
    }
};

struct Scratch {
    cudaStream_t s;
    std::vector<void *> bufs;
    explicit Scratch(cudaStream_t st) : s(st) {}
    ~Scratch() {
        for (void *p : bufs) cudaFreeAsync(p, s);
    }
    template <class T>
    int get(T **out, size_t count) {
        void *p = nullptr;
        cudaError_t e = cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), s);
        if (e != cudaSuccess) {
            set_error("device allocation of %zu bytes failed: %s", count * sizeof(T),
                      cudaGetErrorString(e));
            return FR_ECUDA;
        }
        bufs.push_back(p);
        *out = (T *)p;
        return FR_OK;
    }
};

// grow-only per-device workspace for a splat's entry-sized buffers (~64 B per
// entry: 4.3 GB at 16.8M points): a rebuild reuses one mapped block instead of
// asking the pool for GB-sized blocks that, fragmented, get freshly mapped
// (75-130 ms outliers in the sigma-re-estimating loop).  One lease at a time;
// a concurrent splat (register_batch threads) falls back to the pool.  The
// next lessee's stream waits on the previous lessee's release event.
struct Workspace {
    std::mutex mu;
    char *p = nullptr;
    size_t cap = 0;
    bool busy = false;
    cudaEvent_t ev = nullptr;
};
static Workspace g_ws[16];

struct WsLease {
    Workspace *w = nullptr;
    cudaStream_t s = nullptr;
    size_t off = 0;
    ~WsLease() { release(); }
    // 1: leased `need` bytes; 0: busy or unavailable (use the pool)
    int acquire(size_t need, cudaStream_t st) {
        int dev = 0;
        cudaGetDevice(&dev);
        Workspace &ws = g_ws[dev & 15];
        {
            std::lock_guard<std::mutex> g(ws.mu);
            if (ws.busy) return 0;
            ws.busy = true;
        }
        w = &ws;
        s = st;
        if (ws.ev) cudaStreamWaitEvent(s, ws.ev, 0);
        else cudaEventCreateWithFlags(&ws.ev, cudaEventDisableTiming);
        if (ws.cap < need) {
            if (ws.p) cudaFreeAsync(ws.p, s);
            ws.p = nullptr;
            ws.cap = 0;
            const size_t grow = need + need / 4;
            if (cudaMallocAsync((void **)&ws.p, grow, s) != cudaSuccess) {
                cudaGetLastError();
                ws.p = nullptr;
                release();
                return 0;
            }
            ws.cap = grow;
        }
        return 1;
    }
    template <class T>
    T *carve(size_t count) {
        const size_t bytes = (std::max<size_t>(count, 1) * sizeof(T) + 255) & ~(size_t)255;
        T *r = (T *)(w->p + off);
        off += bytes;
        return r;
    }
    void release() {
        if (!w) return;
        cudaEventRecord(w->ev, s);
        std::lock_guard<std::mutex> g(w->mu);
        w->busy = false;
        w = nullptr;
    }
};
static inline size_t ws_bytes(size_t count, size_t elem) {
    return (std::max<size_t>(count, 1) * elem + 255) & ~(size_t)255;
}

// small device -> host reads of the build (counters, run / site counts, the
// site box) through a per-thread pinned buffer: pageable transfers go through
// the driver's staging path and stalled a concurrent pinned upload on another
// thread (16.8M points: 7 -> 14 ms while a splat ran)
static void *pinned_scratch() {
    static thread_local void *p = nullptr;
    if (!p && cudaHostAlloc(&p, 4096, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
    }
    return p;
}
static int d2h_sync(void *host, const void *dev, size_t bytes, cudaStream_t s) {
    void *pin = bytes <= 4096 ? pinned_scratch() : nullptr;
    FR_CUDA(cudaMemcpyAsync(pin ? pin : host, dev, bytes, cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaStreamSynchronize(s));
    if (pin) memcpy(host, pin, bytes);
    return FR_OK;
}

__global__ void k_iota(int n, int *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

__global__ void k_fill_u64(unsigned long long *p, unsigned long long a, unsigned long long b,
                           unsigned long long c) {
    if (threadIdx.x == 0) {
        p[0] = a;
        p[1] = b;
        p[2] = c;
    }
}

static int read_counters(fr_lattice *lat, cudaStream_t s, unsigned long long *h) {
    FR_TRY(d2h_sync(h, lat->d_counters, 3 * sizeof(unsigned long long), s));
    if (h[2] & 1ull) {
        set_error("lattice coordinate outside the packable range (|key| >= %lld); "
                  "features / sigma too large", (long long)kKeyLim);
        return FR_ECAPACITY;
    }
    return FR_OK;
}

static void free_slice(fr_lattice *lat);

// every lattice buffer comes from the device's stream-ordered pool (release
// threshold: never), on the stream of the call that builds the lattice: a
// rebuild reuses mapped pages instead of cudaMalloc / cudaFree mapping and
// unmapping ~100 MB-GB per build (seconds-long outliers at C5 sizes)
static cudaError_t pool_alloc(fr_lattice *lat, void **p, size_t bytes) {
    return cudaMallocAsync(p, std::max<size_t>(bytes, 1), lat->stream);
}
static void pool_free(fr_lattice *lat, void *p) {
    if (p) cudaFreeAsync(p, lat->stream);
}

static void free_build(fr_lattice *lat) {
    pool_free(lat, lat->wkh);
    pool_free(lat, lat->wkl);
    lat->wkh = lat->wkl = nullptr;
    pool_free(lat, lat->site_keys);
    pool_free(lat, lat->vals);
    pool_free(lat, lat->vals_alt);
    pool_free(lat, lat->hkeys);
    pool_free(lat, lat->hsite);
    lat->site_keys = nullptr;
    lat->vals = lat->vals_alt = nullptr;
    lat->hkeys = nullptr;
    lat->hsite = nullptr;
    lat->hmask = 0;
}

static int alloc_hash(fr_lattice *lat, unsigned cap, cudaStream_t s) {
    pool_free(lat, lat->hkeys);
    pool_free(lat, lat->hsite);
    lat->hkeys = nullptr;
    lat->hsite = nullptr;
    FR_CUDA(pool_alloc(lat, (void **)&lat->hkeys, (size_t)cap * sizeof(unsigned long long)));
    FR_CUDA(pool_alloc(lat, (void **)&lat->hsite, (size_t)cap * sizeof(int)));
    FR_CUDA(cudaMemsetAsync(lat->hkeys, 0xff, (size_t)cap * sizeof(unsigned long long), s));
    FR_CUDA(cudaMemsetAsync(lat->hsite, 0xff, (size_t)cap * sizeof(int), s));
    lat->hmask = cap - 1;
    return FR_OK;
}

template <int D>
static int rehash_sites(fr_lattice *lat, unsigned cap, cudaStream_t s) {
    FR_TRY(alloc_hash(lat, cap, s));
    FR_CUDA(cudaMemsetAsync(lat->d_counters + 2, 0, sizeof(unsigned long long), s));
    if (lat->n_sites > 0) {
        k_hash_sites<D><<<grid_for(lat->n_sites), 256, 0, s>>>(
            lat->n_sites, lat->site_keys, BuildHash{lat->hkeys, lat->hsite, lat->hmask},
            lat->d_counters);
        FR_CHECK_LAUNCH();
    }
    return FR_OK;
}

// grow the site arrays to hold `need` sites, preserving the first n_sites rows
static int reserve_sites(fr_lattice *lat, long long need, cudaStream_t s) {
    if (need <= lat->site_cap) return FR_OK;
    long long cap = std::max<long long>(need, lat->site_cap * 2);
    const int D1 = lat->dim + 1, nv = lat->nv;
    int *nk = nullptr;
    double *nvals = nullptr, *nalt = nullptr;
    FR_CUDA(pool_alloc(lat, (void **)&nk, (size_t)cap * D1 * sizeof(int)));
    FR_CUDA(pool_alloc(lat, (void **)&nvals, (size_t)cap * nv * sizeof(double)));
    FR_CUDA(pool_alloc(lat, (void **)&nalt, (size_t)cap * nv * sizeof(double)));
    if (lat->n_sites > 0) {
        FR_CUDA(cudaMemcpyAsync(nk, lat->site_keys, (size_t)lat->n_sites * D1 * sizeof(int),
                                cudaMemcpyDeviceToDevice, s));
        FR_CUDA(cudaMemcpyAsync(nvals, lat->vals, (size_t)lat->n_sites * nv * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
    }
    // (no host sync: the pool's frees are stream-ordered behind the copies)
    pool_free(lat, lat->site_keys);
    pool_free(lat, lat->vals);
    pool_free(lat, lat->vals_alt);
    lat->site_keys = nk;
    lat->vals = nvals;
    lat->vals_alt = nalt;
    lat->site_cap = cap;
    return FR_OK;
}

// a caller-run entries pass: given launch(a, b, stream) for the point range
// [a, b), it enqueues every range and orders the splat's stream after them
using EntriesLaunch = std::function<int(long long, long long, cudaStream_t)>;
using EntriesHook = std::function<int(const EntriesLaunch &)>;

// flat: site sums in np.add.at's flat (point, vertex) order, bit-identical to
// the reference (the operator API, PermutohedralLattice.splat, and point
// splats with FR_SPLAT_FLAT_ORDER); else the fixed-tree order of
// k_splat_segsum_tree

// site ids from the list of created slots: sorted ascending (the table's
// slot order), ids[slot] = rank; slot_of_id = the sorted list
static int sc_site_ids(Scratch &sc, unsigned *created, unsigned K, unsigned cap, int *ids,
                       int **slot_of_id, cudaStream_t s) {
    unsigned *sorted;
    FR_TRY(sc.get(&sorted, (size_t)K + 1));
    if (K > 0) {
        int bits = 1;
        while ((1ull << bits) < cap) ++bits;
        size_t tb = 0;
        FR_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, created, sorted, (int)K, 0, bits, s));
        void *tmp;
        FR_TRY(sc.get((char **)&tmp, tb));
        FR_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, created, sorted, (int)K, 0, bits, s));
        k_scatter_ids<<<grid_for(K), 256, 0, s>>>(K, sorted, ids);
        FR_CHECK_LAUNCH();
    }
    *slot_of_id = reinterpret_cast<int *>(sorted);
    return FR_OK;
}

// initial splat hash size: FR_SPLAT_HASH_SHIFT (default 0) divides the
// entry-based bound (2E, at most 2^22 slots) by 2^shift, at least 2^15 slots;
// a table that fills grows x4 and the pass reruns
static unsigned long long splat_hash_cap(long long E) {
    static const int shift = getenv("FR_SPLAT_HASH_SHIFT") ? atoi(getenv("FR_SPLAT_HASH_SHIFT")) : 0;
    const unsigned long long full = next_pow2((unsigned long long)std::min<long long>(2 * E, 1LL << 22));
    return std::max<unsigned long long>(full >> std::max(0, std::min(shift, 20)), 1ull << 15);
}

constexpr int kAggFallback = 1000;

template <int D, class Src>
static int splat_agg(fr_lattice *lat, const Src &src, long long n, int nv, cudaStream_t s,
                     PhaseClock &pc) {
    const long long E = n * (D + 1);
    Scratch sc(s);
    const long long max_pairs = E / 4 + (1LL << 16);
    unsigned *pair_slot, *pair_lo;
    double *pair_vals;
    FR_TRY(sc.get(&pair_slot, (size_t)max_pairs));
    FR_TRY(sc.get(&pair_lo, (size_t)max_pairs));
    FR_TRY(sc.get(&pair_vals, (size_t)max_pairs * nv));
    pc.lap("alloc");
    unsigned long long cap = splat_hash_cap(E);
    unsigned long long hc[4];
    const unsigned g = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16);
    unsigned *created = nullptr;
    for (;;) {
        FR_TRY(alloc_hash(lat, (unsigned)cap, s));
        FR_TRY(sc.get(&created, (size_t)cap / 2 + 1));
        FR_CUDA(cudaMemsetAsync(lat->d_counters, 0, 4 * sizeof(unsigned long long), s));
        BuildHash h{lat->hkeys, lat->hsite, lat->hmask};
        switch (nv) {
#define FR_AGG(NVV)                                                                                \
    case NVV:                                                                                      \
        k_splat_warp_pairs<D, NVV, Src><<<g, 256, 0, s>>>(src, n, lat->c, h, pair_slot, pair_lo,  \
                                                         pair_vals, max_pairs, lat->d_counters,   \
                                                         created);                                \
        break;
            FR_AGG(1) FR_AGG(2) FR_AGG(3) FR_AGG(4) FR_AGG(5) FR_AGG(6) FR_AGG(7) FR_AGG(8)
#undef FR_AGG
        }
        FR_CHECK_LAUNCH();
        FR_TRY(d2h_sync(hc, lat->d_counters, 4 * sizeof(unsigned long long), s));
        if (hc[2] & 1ull) {
            set_error("lattice coordinate outside the packable range (|key| >= %lld); "
                      "features / sigma too large", (long long)kKeyLim);
            return FR_ECAPACITY;
        }
        if (hc[2] & 4ull) return kAggFallback;          // points not spatially ordered enough
        const bool full = (hc[2] & 2ull) || hc[0] * 2 > cap;
        if (!full) break;
        if (cap >= (1ull << 31)) {
            set_error("splat hash table exceeded 2^31 slots");
            return FR_ECAPACITY;
        }
        cap *= 4;
    }
    pc.lap("pairs");
    const unsigned K = (unsigned)hc[0];
    const long long np = (long long)hc[3];
    if (pc.on) fprintf(stderr, "[splat] %lld points, %lld pairs, %u sites in %llu slots (load %.4f)\n",
                       n, np, K, cap, (double)K / (double)cap);
    int *slot_of_id, *ids;
    FR_TRY(sc.get(&ids, (size_t)cap));
    FR_TRY(sc_site_ids(sc, created, K, (unsigned)cap, ids, &slot_of_id, s));
    const unsigned gg = 148 * 8;
    int lo_bits = 1;
    while ((1LL << lo_bits) < ((n + 31) / 32) * (D + 1)) ++lo_bits;
    int id_bits = 1;
    while ((1LL << id_bits) < (long long)K + 1) ++id_bits;
    unsigned long long *keys, *keys2;
    unsigned *idx, *idx2, *sid;
    FR_TRY(sc.get(&keys, (size_t)std::max(np, 1LL)));
    FR_TRY(sc.get(&keys2, (size_t)std::max(np, 1LL)));
    FR_TRY(sc.get(&idx, (size_t)std::max(np, 1LL)));
    FR_TRY(sc.get(&idx2, (size_t)std::max(np, 1LL)));
    FR_TRY(sc.get(&sid, (size_t)std::max(np, 1LL)));
    const long long max_runs = (long long)K + 1;
    unsigned *run_slot;
    int *run_cnt, *run_off, *d_nruns;
    FR_TRY(sc.get(&run_slot, (size_t)max_runs));
    FR_TRY(sc.get(&run_cnt, (size_t)max_runs));
    FR_TRY(sc.get(&run_off, (size_t)max_runs));
    FR_TRY(sc.get(&d_nruns, 1));
    int nruns = 0;
    if (np > 0) {
        k_pair_keys<<<gg, 256, 0, s>>>(np, pair_slot, pair_lo, ids, lo_bits, keys, idx);
        FR_CHECK_LAUNCH();
        size_t tb = 0, t2 = 0;
        FR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, idx, idx2, (int)np, 0,
                                                lo_bits + id_bits, s));
        FR_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, t2, sid, run_slot, run_cnt, d_nruns,
                                                   (int)np, s));
        tb = std::max(tb, t2);
        FR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, run_cnt, run_off, (int)max_runs, s));
        tb = std::max(tb, t2);
        void *tmp;
        FR_TRY(sc.get((char **)&tmp, tb));
        FR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, idx, idx2, (int)np, 0,
                                                lo_bits + id_bits, s));
        k_key_ids<<<gg, 256, 0, s>>>(np, keys2, lo_bits, sid);
        FR_CHECK_LAUNCH();
        FR_CUDA(cub::DeviceRunLengthEncode::Encode(tmp, tb, sid, run_slot, run_cnt, d_nruns,
                                                   (int)np, s));
        k_runs_to_slots<<<148, 256, 0, s>>>(d_nruns, K, (unsigned)cap, slot_of_id, run_slot);
        FR_CHECK_LAUNCH();
        FR_TRY(d2h_sync(&nruns, d_nruns, sizeof(int), s));
        FR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, run_cnt, run_off, nruns, s));
    }
    pc.lap("sort+runs");
    double *run_vals;
    unsigned char *run_live;
    int *live_runs, *iota, *d_nlive;
    FR_TRY(sc.get(&run_vals, (size_t)std::max(nruns, 1) * nv));
    FR_TRY(sc.get(&run_live, (size_t)std::max(nruns, 1)));
    FR_TRY(sc.get(&live_runs, (size_t)std::max(nruns, 1)));
    FR_TRY(sc.get(&iota, (size_t)std::max(nruns, 1)));
    FR_TRY(sc.get(&d_nlive, 1));
    if (nruns > 0) {
        // the runs' pairs in fixed-size pieces, tree sums, combined in order
        int *pieces, *piece_off;
        double *piece_vals;
        const long long max_pieces = (long long)nruns + np / kSegPiece + 1;
        FR_TRY(sc.get(&pieces, (size_t)nruns + 1));
        FR_TRY(sc.get(&piece_off, (size_t)nruns + 1));
        FR_TRY(sc.get(&piece_vals, (size_t)max_pieces * nv));
        FR_CUDA(cudaMemsetAsync(pieces + nruns, 0, sizeof(int), s));
        k_seg_piece_counts<<<grid_for(nruns), 256, 0, s>>>(nruns, nullptr, 0u, run_cnt, pieces);
        FR_CHECK_LAUNCH();
        size_t t4 = 0;
        FR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t4, pieces, piece_off, nruns + 1, s));
        void *tmp4;
        FR_TRY(sc.get((char **)&tmp4, t4));
        FR_CUDA(cub::DeviceScan::ExclusiveSum(tmp4, t4, pieces, piece_off, nruns + 1, s));
        switch (nv) {
#define FR_SEG_TREE(NVV)                                                                          \
    case NVV:                                                                                     \
        k_splat_segsum_tree<D, NVV><<<(unsigned)max_pieces, kSegBlock, 0, s>>>(                  \
            nruns, piece_off, run_off, run_cnt, idx2, pair_vals, piece_vals, 0);                  \
        break;
            FR_SEG_TREE(1) FR_SEG_TREE(2) FR_SEG_TREE(3) FR_SEG_TREE(4)
            FR_SEG_TREE(5) FR_SEG_TREE(6) FR_SEG_TREE(7) FR_SEG_TREE(8)
#undef FR_SEG_TREE
        }
        FR_CHECK_LAUNCH();
        k_seg_pieces_combine<<<grid_for((long long)nruns * nv), 256, 0, s>>>(
            nruns, piece_off, piece_vals, nv, run_vals);
        FR_CHECK_LAUNCH();
        k_run_live<<<grid_for(nruns), 256, 0, s>>>(nruns, run_slot, (unsigned)cap, run_vals, nv,
                                                   run_live);
        FR_CHECK_LAUNCH();
    }
    pc.lap("segsum");
    int S = 0;
    if (nruns > 0) {
        k_iota<<<grid_for(nruns), 256, 0, s>>>(nruns, iota);
        FR_CHECK_LAUNCH();
        size_t t3 = 0;
        FR_CUDA(cub::DeviceSelect::Flagged(nullptr, t3, iota, run_live, live_runs, d_nlive,
                                           nruns, s));
        void *tmp3;
        FR_TRY(sc.get((char **)&tmp3, t3));
        FR_CUDA(cub::DeviceSelect::Flagged(tmp3, t3, iota, run_live, live_runs, d_nlive, nruns,
                                           s));
        FR_TRY(d2h_sync(&S, d_nlive, sizeof(int), s));
    }
    unsigned long long *old_keys = lat->hkeys;
    lat->hkeys = nullptr;   // keep the splat hash alive for k_fill_sites
    FR_TRY(reserve_sites(lat, std::max(S, 1), s));
    if (S > 0) {
        k_fill_sites<D><<<grid_for(S), 256, 0, s>>>(S, live_runs, run_slot, old_keys, run_vals,
                                                    nv, lat->site_keys, lat->vals);
        FR_CHECK_LAUNCH();
    }
    pool_free(lat, old_keys);
    lat->n_sites = S;
    pc.lap("sites");
    // 2 S slots for S distinct keys: the inserts cannot fail, no flag read
    FR_TRY(rehash_sites<D>(lat, next_pow2(2ull * (unsigned long long)lat->n_sites), s));
    pc.lap("rehash");
    return FR_OK;
}

template <int D, class Src>
static int splat_impl(fr_lattice *lat, const Src &src, long long n, int nv, cudaStream_t s,
                      const EntriesHook *first = nullptr, bool flat = true, bool agg = false) {
    if (lat->blurred || lat->splatted) {
        // the reference allows re-splatting an unblurred lattice (it replaces the table)
    }
    if (nv < 1 || nv > 15) {
        set_error("value width %d unsupported (1..15 columns per lattice)", nv);
        return FR_EINVAL;
    }
    PhaseClock pc(s);
    free_build(lat);
    free_slice(lat);
    lat->nv = nv;
    lat->n_sites = 0;
    lat->site_cap = 0;
    lat->blurred = 0;
    lat->splatted = 1;
    if (n == 0) return reserve_sites(lat, 1, s);
    const long long E = n * (D + 1);
    if (E >= (1LL << 31) - 1) {
        set_error("too many points for one splat (%lld)", n);
        return FR_EINVAL;
    }
    if (agg && !flat && !first && nv <= 8) {
        const int st = splat_agg<D, Src>(lat, src, n, nv, s, pc);
        if (st != kAggFallback) return st;
        free_build(lat);                   // too many pairs: the per-entry path below
        lat->n_sites = 0;
        lat->site_cap = 0;
    }
    Scratch sc(s);
    unsigned *entry_slot, *entry_idx, *sorted_slot, *sorted_idx;
    double *entry_bary, *contrib = nullptr;
    const bool with_contrib = contrib_fits(E, nv);
    // the entry-sized buffers and an upper bound of the sort's temporary
    size_t sort_bound = 0;
    FR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bound, (unsigned *)nullptr,
                                            (unsigned *)nullptr, (unsigned *)nullptr,
                                            (unsigned *)nullptr, (int)E, 0, 32, s));
    const size_t need = 4 * ws_bytes(E, 4) + ws_bytes(E, 8) +
                        (with_contrib ? ws_bytes((size_t)E * nv, 8) : 0) + ws_bytes(sort_bound, 1);
    WsLease lease;
    char *sort_tmp = nullptr;
    if (lease.acquire(need, s)) {
        entry_slot = lease.carve<unsigned>(E);
        entry_idx = lease.carve<unsigned>(E);
        sorted_slot = lease.carve<unsigned>(E);
        sorted_idx = lease.carve<unsigned>(E);
        entry_bary = lease.carve<double>(E);
        if (with_contrib) contrib = lease.carve<double>((size_t)E * nv);
        sort_tmp = lease.carve<char>(sort_bound);
    } else {
        FR_TRY(sc.get(&entry_slot, E));
        FR_TRY(sc.get(&entry_idx, E));
        FR_TRY(sc.get(&sorted_slot, E));
        FR_TRY(sc.get(&sorted_idx, E));
        FR_TRY(sc.get(&entry_bary, E));
        if (with_contrib) FR_TRY(sc.get(&contrib, (size_t)E * nv));
    }
    pc.lap("alloc");
    // hash sized for the unique-key count; grown x4 on overflow
    unsigned long long cap = splat_hash_cap(E);
    unsigned long long hc[3];
    unsigned *created = nullptr;
    for (int attempt = 0;; ++attempt) {
        FR_TRY(alloc_hash(lat, (unsigned)cap, s));
        FR_TRY(sc.get(&created, (size_t)cap / 2 + 1));
        FR_CUDA(cudaMemsetAsync(lat->d_counters, 0, 3 * sizeof(unsigned long long), s));
        BuildHash h{lat->hkeys, lat->hsite, lat->hmask};
        if (attempt == 0 && first) {
            // the caller runs the entries pass itself (range by range as the
            // points land) and leaves s ordered after it
            const auto launch = [&](long long a, long long b, cudaStream_t st) -> int {
                k_splat_entries<D, Src><<<grid_for(b - a), 256, 0, st>>>(
                    src, a, b, n, lat->c, h, (unsigned)cap, entry_slot, entry_idx, entry_bary,
                    contrib, lat->d_counters, created);
                FR_CHECK_LAUNCH();     // on the launching (worker) thread
                return FR_OK;
            };
            FR_TRY((*first)(launch));
        } else {
            k_splat_entries<D, Src><<<grid_for(n), 256, 0, s>>>(src, 0, n, n, lat->c, h, (unsigned)cap,
                                                                entry_slot, entry_idx, entry_bary,
                                                                contrib, lat->d_counters, created);
        }
        FR_CHECK_LAUNCH();
        FR_TRY(read_counters(lat, s, hc));
        bool full = (hc[2] & 2ull) || hc[0] * 2 > cap;
        if (!full) break;
        if (cap >= (1ull << 31)) {
            set_error("splat hash table exceeded 2^31 slots");
            return FR_ECAPACITY;
        }
        cap *= 4;
    }
    pc.lap("entries");
    // dense site ids as sort keys (K = distinct keys, counted by the inserts)
    const unsigned K = (unsigned)hc[0];
    if (pc.on) fprintf(stderr, "[splat] %lld points, %lld entries, %u sites in %llu slots "
                       "(load %.4f)\n", n, E, K, cap, (double)K / (double)cap);
    int *slot_of_id = nullptr;
    {
        int *ids;
        FR_TRY(sc.get(&ids, (size_t)cap));
        FR_TRY(sc_site_ids(sc, created, K, (unsigned)cap, ids, &slot_of_id, s));
        k_entries_to_ids<<<148 * 8, 256, 0, s>>>(E, (unsigned)cap, K, ids, entry_slot);
        FR_CHECK_LAUNCH();
    }
    const int end_bit = 1 + (int)std::log2((double)std::max(K, 1u));
    // stable radix sort of entries by slot: per-site groups in flat order
    size_t tmp_bytes = 0, t2 = 0;
    FR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, entry_slot, sorted_slot,
                                            entry_idx, sorted_idx, (int)E, 0, end_bit, s));
    // runs = distinct slots (+ the sentinel run): hc[0] counted the CAS winners
    const long long max_runs = (long long)hc[0] + 2;
    unsigned *run_slot;
    int *run_cnt, *run_off, *d_nruns;
    FR_TRY(sc.get(&run_slot, max_runs));
    FR_TRY(sc.get(&run_cnt, max_runs));
    FR_TRY(sc.get(&run_off, max_runs));
    FR_TRY(sc.get(&d_nruns, 1));
    FR_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, t2, sorted_slot, run_slot, run_cnt,
                                               d_nruns, (int)E, s));
    tmp_bytes = std::max(tmp_bytes, t2);
    FR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, run_cnt, run_off, (int)E, s));
    tmp_bytes = std::max(tmp_bytes, t2);
    pc.lap("sort_setup");
    void *tmp = sort_tmp;
    if (!tmp || tmp_bytes > sort_bound) FR_TRY(sc.get((char **)&tmp, tmp_bytes));
    pc.lap("sort_tmp");
    k_run_pad<<<1, 32, 0, s>>>(K, (unsigned)cap, run_slot, run_cnt);
    FR_CHECK_LAUNCH();
    FR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, entry_slot, sorted_slot, entry_idx,
                                            sorted_idx, (int)E, 0, end_bit, s));
    pc.lap("sort_enqueue");
    FR_CUDA(cub::DeviceRunLengthEncode::Encode(tmp, tmp_bytes, sorted_slot, run_slot, run_cnt,
                                               d_nruns, (int)E, s));
    pc.lap("rle_enqueue");
    k_runs_to_slots<<<148, 256, 0, s>>>(d_nruns, K, (unsigned)cap, slot_of_id, run_slot);
    FR_CHECK_LAUNCH();
    // the runs are the K sites (every created slot holds its creator's entry)
    // plus the sentinel run when some entry has none: K + 1 rows with row K
    // padded as an empty sentinel run when the RLE wrote only K -- no host
    // read of the run count
    const int nruns = (int)K + 1;
    FR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, run_cnt, run_off, nruns, s));
    pc.lap("sort+runs");
    double *run_vals;
    unsigned char *run_live;
    int *live_runs, *iota, *d_nlive;
    FR_TRY(sc.get(&run_vals, (size_t)nruns * nv));
    FR_TRY(sc.get(&run_live, nruns));
    FR_TRY(sc.get(&live_runs, nruns));
    FR_TRY(sc.get(&iota, nruns));
    FR_TRY(sc.get(&d_nlive, 1));
    {
        const size_t smem = (size_t)kSegStages * kSegBlock * nv * sizeof(double);
        FR_CUDA(cudaFuncSetAttribute(k_splat_segsum<D, Src>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const bool tree = !flat && contrib && nv >= 1 && nv <= 8;
        if (nruns > 0 && tree) {
            // pieces per run -> exclusive offsets (n_runs + 1; the last is the
            // total); the launch takes the upper bound runs + E / piece
            int *pieces, *piece_off;
            double *piece_vals;
            const long long max_pieces = (long long)nruns + E / kSegPiece + 1;
            FR_TRY(sc.get(&pieces, (size_t)nruns + 1));
            FR_TRY(sc.get(&piece_off, (size_t)nruns + 1));
            FR_TRY(sc.get(&piece_vals, (size_t)max_pieces * nv));
            FR_CUDA(cudaMemsetAsync(pieces + nruns, 0, sizeof(int), s));
            k_seg_piece_counts<<<grid_for(nruns), 256, 0, s>>>(nruns, run_slot, (unsigned)cap,
                                                               run_cnt, pieces);
            FR_CHECK_LAUNCH();
            size_t t4 = 0;
            FR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t4, pieces, piece_off, nruns + 1, s));
            void *tmp4;
            FR_TRY(sc.get((char **)&tmp4, t4));
            FR_CUDA(cub::DeviceScan::ExclusiveSum(tmp4, t4, pieces, piece_off, nruns + 1, s));
            switch (nv) {
#define FR_SEG_TREE(NVV)                                                                          \
    case NVV:                                                                                     \
        k_splat_segsum_tree<D, NVV><<<(unsigned)max_pieces, kSegBlock, 0, s>>>(                  \
            nruns, piece_off, run_off, run_cnt, sorted_idx, contrib, piece_vals, n);              \
        break;
                FR_SEG_TREE(1) FR_SEG_TREE(2) FR_SEG_TREE(3) FR_SEG_TREE(4)
                FR_SEG_TREE(5) FR_SEG_TREE(6) FR_SEG_TREE(7) FR_SEG_TREE(8)
#undef FR_SEG_TREE
            }
            FR_CHECK_LAUNCH();
            k_seg_pieces_combine<<<grid_for((long long)nruns * nv), 256, 0, s>>>(
                nruns, piece_off, piece_vals, nv, run_vals);
            FR_CHECK_LAUNCH();
        } else if (nruns > 0) {
            k_splat_segsum<D, Src><<<nruns, kSegBlock, smem, s>>>(
                src, run_slot, run_off, run_cnt, sorted_idx, entry_bary, contrib, (unsigned)cap,
                nv, run_vals, n);
            FR_CHECK_LAUNCH();
        }
        k_run_live<<<grid_for(nruns), 256, 0, s>>>(nruns, run_slot, (unsigned)cap, run_vals, nv,
                                                   run_live);
        FR_CHECK_LAUNCH();
    }
    pc.lap("segsum");
    // live runs -> dense site rows
    {
        k_iota<<<grid_for(nruns), 256, 0, s>>>(nruns, iota);
        FR_CHECK_LAUNCH();
        size_t t3 = 0;
        FR_CUDA(cub::DeviceSelect::Flagged(nullptr, t3, iota, run_live, live_runs, d_nlive,
                                           nruns, s));
        void *tmp3;
        FR_TRY(sc.get((char **)&tmp3, t3));
        FR_CUDA(cub::DeviceSelect::Flagged(tmp3, t3, iota, run_live, live_runs, d_nlive, nruns,
                                           s));
        int S = 0;
        FR_TRY(d2h_sync(&S, d_nlive, sizeof(int), s));
        unsigned long long *old_keys = lat->hkeys;
        lat->hkeys = nullptr;   // keep the splat hash alive for k_fill_sites
        FR_TRY(reserve_sites(lat, std::max(S, 1), s));
        if (S > 0) {
            k_fill_sites<D><<<grid_for(S), 256, 0, s>>>(S, live_runs, run_slot, old_keys,
                                                        run_vals, nv, lat->site_keys, lat->vals);
            FR_CHECK_LAUNCH();
        }
        pool_free(lat, old_keys);           // stream-ordered behind k_fill_sites
        lat->n_sites = S;
    }
    pc.lap("sites");
    // 2 S slots for S distinct keys: the inserts cannot fail, no flag read
    FR_TRY(rehash_sites<D>(lat, next_pow2(2ull * (unsigned long long)lat->n_sites), s));
    pc.lap("rehash");
    return FR_OK;
}

template <int D>
static int compact_nonzero(fr_lattice *lat, cudaStream_t s) {
    long long S = lat->n_sites;
    if (S == 0) return FR_OK;
    // the device-resident blur counted the surviving rows: nothing to drop
    // (the usual case), or the count without a host read
    const long long known = lat->blur_keep;
    if (known == S) return FR_OK;
    Scratch sc(s);
    unsigned char *flags;
    int *iota, *sel, *d_n;
    FR_TRY(sc.get(&flags, S));
    FR_TRY(sc.get(&iota, S));
    FR_TRY(sc.get(&sel, S));
    FR_TRY(sc.get(&d_n, 1));
    k_nonzero_flags<<<grid_for(S), 256, 0, s>>>(S, lat->vals, lat->nv, flags);
    FR_CHECK_LAUNCH();
    k_iota<<<grid_for(S), 256, 0, s>>>((int)S, iota);
    FR_CHECK_LAUNCH();
    size_t t = 0;
    FR_CUDA(cub::DeviceSelect::Flagged(nullptr, t, iota, flags, sel, d_n, (int)S, s));
    void *tmp;
    FR_TRY(sc.get((char **)&tmp, t));
    FR_CUDA(cub::DeviceSelect::Flagged(tmp, t, iota, flags, sel, d_n, (int)S, s));
    int keep = (int)known;
    if (known < 0) FR_TRY(d2h_sync(&keep, d_n, sizeof(int), s));
    if (keep == S) return FR_OK;
    int *nk;
    double *nvls;
    FR_TRY(sc.get(&nk, (size_t)std::max(keep, 1) * (D + 1)));
    FR_TRY(sc.get(&nvls, (size_t)std::max(keep, 1) * lat->nv));
    if (keep > 0) {
        k_gather_sites<D><<<grid_for(keep), 256, 0, s>>>(keep, sel, lat->site_keys, lat->vals,
                                                         lat->nv, nk, nvls);
        FR_CHECK_LAUNCH();
        FR_CUDA(cudaMemcpyAsync(lat->site_keys, nk, (size_t)keep * (D + 1) * sizeof(int),
                                cudaMemcpyDeviceToDevice, s));
        FR_CUDA(cudaMemcpyAsync(lat->vals, nvls, (size_t)keep * lat->nv * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
    }
    lat->n_sites = keep;                    // scratch frees are stream-ordered
    return FR_OK;
}

static void free_slice(fr_lattice *lat) {
    pool_free(lat, lat->skeys);
    pool_free(lat, lat->svals);
    pool_free(lat, lat->fslots);
    pool_free(lat, lat->dcells);
    pool_free(lat, lat->dcells64);
    lat->skeys = nullptr;
    lat->svals = nullptr;
    lat->fslots = nullptr;
    lat->dcells = nullptr;
    lat->dcells64 = nullptr;
    lat->dense = fr::DenseSliceF{};
    lat->dense64 = fr::DenseSliceD{};
    lat->dense64_cells = 0;
    lat->dense_cells = 0;
    lat->nvp = 0;
    lat->nf4 = 0;
}

// dense grid budget: the grid replaces hashing in the EM pass when the padded
// site box needs at most this many cells (64 B each)
static long long dense_cell_limit() {
    const char *e = getenv("FR_DENSE_MAX_CELLS");
    return e ? atoll(e) : (16ll << 20);    // 1 GiB
}

// q = floor(k / 4) box of the sites' first three coordinates
__global__ void k_site_qbox(long long S, const int *site_keys, int *box) {
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < S;
         i += (long long)gridDim.x * blockDim.x) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int q = site_keys[i * 4 + c] >> 2;
            lo[c] = min(lo[c], q);
            hi[c] = max(hi[c], q);
        }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo[c] = min(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
            hi[c] = max(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(box + c, lo[c]);
            atomicMax(box + 3 + c, hi[c]);
        }
    }
}

__global__ void k_dense_fill(long long S, const int *site_keys, const double *vals, int nv,
                             double gain, fr::DenseSliceF t, float4 *cells) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const int *k = site_keys + i * 4;
    constexpr int P = fr::kDensePad;
    const int c = ((k[0] >> 2) - t.a[0] + P) * t.s0 + ((k[1] >> 2) - t.a[1] + P) * t.s1 +
                  ((k[2] >> 2) - t.a[2] + P);
    const double *v = vals + i * nv;
    // [1, y0, y1, y2] -> (y0, y1, y2, 1) rows, times the gain
    cells[4 * (long long)c + (k[0] & 3)] =
        make_float4((float)(gain * v[1]), (float)(gain * v[2]), (float)(gain * v[3]),
                    (float)(gain * v[0]));
}

// float64 rows: gain * (y0, y1 | y2, 1 [| n0, n1 | n2, 0]) sums of the value
// columns [1, y] or [1, y, n]
__global__ void k_dense_fill64(long long S, const int *site_keys, const double *vals, int nv,
                               double gain, fr::DenseSliceD t, double2 *cells) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const int *k = site_keys + i * 4;
    constexpr int P = fr::kDensePad;
    const long long c = ((long long)((k[0] >> 2) - t.a[0] + P) * t.s0 +
                         (long long)((k[1] >> 2) - t.a[1] + P) * t.s1 + ((k[2] >> 2) - t.a[2] + P));
    const double *v = vals + i * nv;
    double2 *row = cells + t.r2 * (4 * c + (k[0] & 3));
    row[0] = make_double2(gain * v[1], gain * v[2]);
    row[1] = make_double2(gain * v[3], gain * v[0]);
    if (t.r2 == 4) {          // [1, y, n] (estep.py:153-165): the normal sums
        row[2] = make_double2(gain * v[4], gain * v[5]);
        row[3] = make_double2(gain * v[6], 0.0);
    }
}

static long long dense64_cell_limit() {
    const char *e = getenv("FR_DENSE64_MAX_CELLS");
    return e ? atoll(e) : (8ll << 20);     // 1 GiB
}

__global__ void k_init_box(int *box) {
    if (threadIdx.x < 6) box[threadIdx.x] = threadIdx.x < 3 ? INT_MAX : INT_MIN;
}

static int build_dense_grid(fr_lattice *lat, cudaStream_t s) {
    // nv = 4 ([1, y]: both grids); nv = 7 ([1, y, n], point-to-plane: the
    // float64 grid only, 64-byte rows)
    if (lat->dim != 3 || (lat->nv != 4 && lat->nv != 7) || lat->n_sites == 0) return FR_OK;
    int box[6];
    if (lat->box_valid) {
        // from the device-resident blur's read (the same sites: the final
        // drop keeps exactly the rows the box was taken over)
        memcpy(box, lat->blur_box, sizeof(box));
    } else {
        int *dbox = nullptr;
        FR_CUDA(cudaMallocAsync(&dbox, 6 * sizeof(int), s));
        k_init_box<<<1, 32, 0, s>>>(dbox);
        k_site_qbox<<<std::min<long long>(grid_for(lat->n_sites), 1184), 256, 0, s>>>(
            lat->n_sites, lat->site_keys, dbox);
        FR_CHECK_LAUNCH();
        FR_TRY(d2h_sync(box, dbox, sizeof(box), s));
        FR_CUDA(cudaFreeAsync(dbox, s));
    }
    long long n[3], cells = 1;
    for (int c = 0; c < 3; ++c) {
        n[c] = (long long)box[3 + c] - box[c] + 1 + 2 * fr::kDensePad;
        cells *= n[c];
        if (cells > dense_cell_limit()) return FR_OK;     // hash slots only
    }
    if (lat->nv == 4) {
        fr::DenseSliceF t{};
        for (int c = 0; c < 3; ++c) {
            t.a[c] = box[c];
            t.span[c] = (unsigned)(box[3 + c] - box[c] + 1);
        }
        t.s1 = (int)n[2];
        t.s0 = (int)(n[1] * n[2]);
        FR_CUDA(pool_alloc(lat, (void **)&lat->dcells, (size_t)cells * 4 * sizeof(float4)));
        FR_CUDA(cudaMemsetAsync(lat->dcells, 0, (size_t)cells * 4 * sizeof(float4), s));
        k_dense_fill<<<grid_for(lat->n_sites), 256, 0, s>>>(lat->n_sites, lat->site_keys,
                                                            lat->vals, lat->nv, lat->c.gain, t,
                                                            lat->dcells);
        FR_CHECK_LAUNCH();
        t.cells = lat->dcells;
        lat->dense = t;
        lat->dense_cells = cells;
    }
    const int r2 = lat->nv == 4 ? 2 : 4;      // double2 per row
    if (cells * r2 / 2 <= dense64_cell_limit()) {
        fr::DenseSliceD d{};
        for (int c = 0; c < 3; ++c) {
            d.a[c] = box[c];
            d.n[c] = (int)n[c];
        }
        d.s1 = (int)n[2];
        d.s0 = (int)(n[1] * n[2]);
        d.r2 = r2;
        const size_t bytes = (size_t)cells * 4 * r2 * sizeof(double2);
        FR_CUDA(pool_alloc(lat, (void **)&lat->dcells64, bytes));
        FR_CUDA(cudaMemsetAsync(lat->dcells64, 0, bytes, s));
        k_dense_fill64<<<grid_for(lat->n_sites), 256, 0, s>>>(lat->n_sites, lat->site_keys,
                                                              lat->vals, lat->nv, lat->c.gain, d,
                                                              lat->dcells64);
        FR_CHECK_LAUNCH();
        d.cells = lat->dcells64;
        lat->dense64 = d;
        lat->dense64_cells = cells;
    }
    return FR_OK;
}

// interleaved float32 slice table for the fast EM pass (nv <= 8): slot =
// [packed key | pad][gain * values as float4 x nf4], 32 or 64 bytes
template <int D>
__global__ void k_fslice_insert(long long S, const int *site_keys, const double *vals, int nv,
                                double gain, float4 *slots, int stride4, int nf4, unsigned mask,
                                int shift32, unsigned long long *counters) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const unsigned long long key = pack_key<D>(site_keys + i * (D + 1));
    unsigned s = slot_hash32(key, shift32);
    for (unsigned it = 0; it <= mask; ++it) {
        unsigned long long *kw = reinterpret_cast<unsigned long long *>(slots + (size_t)s * stride4);
        if (atomicCAS(kw, kEmptyKey, key) == kEmptyKey) {
            float v[8];
            for (int c = 0; c < 8; ++c) v[c] = c < nv ? (float)(gain * vals[i * nv + c]) : 0.0f;
            for (int f = 0; f < nf4; ++f)
                slots[(size_t)s * stride4 + 1 + f] =
                    make_float4(v[4 * f], v[4 * f + 1], v[4 * f + 2], v[4 * f + 3]);
            return;
        }
        s = (s + 1) & mask;
    }
    atomicOr(&counters[2], 2ull);
}

template <int D>
static int build_slice_table(fr_lattice *lat, cudaStream_t s) {
    free_slice(lat);
    // load factor <= 1/4: a first-probe hit for almost every vertex
    unsigned cap = next_pow2(4ull * (unsigned long long)std::max<long long>(lat->n_sites, 1));
    int bits = 0;
    while ((1u << bits) < cap) ++bits;
    lat->nvp = nvp_for(lat->nv);
    FR_CUDA(pool_alloc(lat, (void **)&lat->skeys, (size_t)cap * sizeof(unsigned long long)));
    FR_CUDA(pool_alloc(lat, (void **)&lat->svals, (size_t)cap * lat->nvp * sizeof(double)));
    FR_CUDA(cudaMemsetAsync(lat->skeys, 0xff, (size_t)cap * sizeof(unsigned long long), s));
    FR_CUDA(cudaMemsetAsync(lat->svals, 0, (size_t)cap * lat->nvp * sizeof(double), s));
    lat->smask = cap - 1;
    lat->sshift = 64 - bits;
    FR_CUDA(cudaMemsetAsync(lat->d_counters + 2, 0, sizeof(unsigned long long), s));
    if (lat->n_sites > 0) {
        k_slice_insert<D><<<grid_for(lat->n_sites), 256, 0, s>>>(
            lat->n_sites, lat->site_keys, lat->vals, lat->nv, lat->skeys, lat->svals, lat->nvp,
            lat->smask, lat->sshift, lat->d_counters);
        FR_CHECK_LAUNCH();
    }
    if (lat->nv <= 8) {
        lat->nf4 = lat->nv <= 4 ? 1 : 2;
        const int stride4 = lat->nf4 == 1 ? 2 : 4;
        FR_CUDA(pool_alloc(lat, (void **)&lat->fslots, (size_t)cap * stride4 * sizeof(float4)));
        FR_CUDA(cudaMemsetAsync(lat->fslots, 0xff, (size_t)cap * stride4 * sizeof(float4), s));
        lat->fmask = cap - 1;
        lat->fshift32 = 32 - bits;
        if (lat->n_sites > 0) {
            k_fslice_insert<D><<<grid_for(lat->n_sites), 256, 0, s>>>(
                lat->n_sites, lat->site_keys, lat->vals, lat->nv, lat->c.gain, lat->fslots,
                stride4, lat->nf4, lat->fmask, lat->fshift32, lat->d_counters);
            FR_CHECK_LAUNCH();
        }
    }
    if (D == 3) FR_TRY(build_dense_grid(lat, s));
    unsigned long long hc[3];
    FR_TRY(read_counters(lat, s, hc));
    if (hc[2] & 2ull) {
        set_error("slice table overflow");
        return FR_ECAPACITY;
    }
    return FR_OK;
}

// site capacity up to which the blur runs device-resident (its whole capacity
// and hash allocated up front: <= 4M sites, ~0.5 GB)
constexpr long long kDeviceBlurMaxSites = 1LL << 22;

template <int D>
static int blur_impl(fr_lattice *lat, cudaStream_t s) {
    if (!lat->splatted) {
        set_error("blur requires a splatted lattice");
        return FR_ESTATE;
    }
    if (lat->blurred) {
        set_error("lattice already blurred");
        return FR_ESTATE;
    }
    PhaseClock pc(s);
    lat->blur_keep = -1;
    lat->box_valid = 0;
    const int nv = lat->nv;
    const long long cap = std::max<long long>(64 * lat->n_sites, 200000);   // permutohedral.py:304
    unsigned long long hc[3];
    if (cap <= kDeviceBlurMaxSites) {
        // every site the blur can create fits up front: no host round trip
        // until the end (one read of the final count and flags)
        FR_TRY(reserve_sites(lat, cap, s));
        const long long S0 = lat->n_sites;
        FR_CUDA(cudaMemsetAsync(lat->vals + S0 * nv, 0, (size_t)(cap - S0) * nv * sizeof(double), s));
        FR_CUDA(cudaMemsetAsync(lat->vals_alt + S0 * nv, 0,
                                (size_t)(cap - S0) * nv * sizeof(double), s));
        const unsigned long long hslots = next_pow2(4ull * (unsigned long long)cap);
        if (hslots > (unsigned long long)lat->hmask + 1)
            FR_TRY(rehash_sites<D>(lat, (unsigned)hslots, s));
        k_fill_u64<<<1, 32, 0, s>>>(lat->d_counters, (unsigned long long)S0, 0ull, 0ull);
        FR_CHECK_LAUNCH();
        const BuildHash h{lat->hkeys, lat->hsite, lat->hmask};
        Scratch bsc(s);
        unsigned long long *nzc;
        {
            // one cooperative launch: scratch = [nz[D + 2] | barrier | box[6]]
            FR_TRY(bsc.get(&nzc, (size_t)D + 6));
            unsigned *bar = reinterpret_cast<unsigned *>(nzc + D + 2);
            int *box = reinterpret_cast<int *>(nzc + D + 3);
            k_blur_scratch_init<<<1, 32, 0, s>>>(nzc, D + 3, box);
            FR_CHECK_LAUNCH();
            static int coop_max = 0;
            if (!coop_max) {
                int per = 0, sms = 148, dev = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_blur_coop<D>, 256, 0) !=
                        cudaSuccess || per < 1)
                    per = 1;
                coop_max = sms * std::min(per, 4);
            }
            // grid sized by the work (the sites grow ~3x over the axes): each
            // grid barrier costs about one arrival per CTA, so a few thousand
            // sites take a few dozen CTAs, not the whole co-resident grid
            const int coop_blocks = (int)std::min<long long>(
                coop_max, std::max<long long>(16, (3 * S0 + 255) / 256));
            double *v0 = lat->vals, *v1 = lat->vals_alt;
            int *keys = lat->site_keys;
            unsigned long long *ctr = lat->d_counters;
            long long capl = cap;
            int nvv = nv;
            BuildHash hh = h;
            void *args[] = {&v0, &v1, &nvv, &hh, &keys, &ctr, &nzc, &capl, &bar, &box};
            FR_CUDA(cudaLaunchCooperativeKernel((const void *)k_blur_coop<D>, dim3(coop_blocks),
                                                dim3(256), args, 0, s));
            // d + 1 swaps: the result is in vals after an even count
            if ((D + 1) & 1) std::swap(lat->vals, lat->vals_alt);
        }
        // ONE host read: counters, the final nonzero count and the box
        unsigned long long hx[4 + 1 + 3];
        {
            unsigned long long *pin = static_cast<unsigned long long *>(pinned_scratch());
            unsigned long long *dst = pin ? pin : hx;
            FR_CUDA(cudaMemcpyAsync(dst, lat->d_counters, 3 * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, s));
            FR_CUDA(cudaMemcpyAsync(dst + 4, nzc + D + 1, sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, s));
            FR_CUDA(cudaMemcpyAsync(dst + 5, nzc + D + 3, 3 * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, s));
            FR_CUDA(cudaStreamSynchronize(s));
            if (pin) memcpy(hx, pin, sizeof(hx));
        }
        if (hx[2] & 1ull) {
            set_error("lattice coordinate outside the packable range (|key| >= %lld); "
                      "features / sigma too large", (long long)kKeyLim);
            return FR_ECAPACITY;
        }
        if (hx[2] & 2ull) {
            set_error("blur hash table overflow");
            return FR_ECAPACITY;
        }
        lat->n_sites = (long long)hx[0];
        lat->blur_keep = (long long)hx[4];
        if (D == 3) {
            memcpy(lat->blur_box, hx + 5, sizeof(lat->blur_box));
            lat->box_valid = lat->blur_keep > 0;
        }
        pc.lap("blur_axes");
    }
    for (int axis = 0; axis <= D && cap > kDeviceBlurMaxSites; ++axis) {
        long long S = lat->n_sites;
        FR_CUDA(cudaMemsetAsync(lat->d_counters, 0, 3 * sizeof(unsigned long long), s));
        if (S > 0) {
            k_count_nonzero<<<grid_for(S), 256, 0, s>>>(S, lat->vals, nv, lat->d_counters + 1);
            FR_CHECK_LAUNCH();
        }
        FR_TRY(read_counters(lat, s, hc));
        long long nsrc = (long long)hc[1];
        if (S + 2 * nsrc <= cap && nsrc > 0) {
            long long need = S + 2 * nsrc;
            FR_TRY(reserve_sites(lat, need, s));
            if ((unsigned long long)need * 2 > (unsigned long long)lat->hmask + 1)
                FR_TRY(rehash_sites<D>(lat, next_pow2(4ull * (unsigned long long)need), s));
            FR_CUDA(cudaMemsetAsync(lat->vals + S * nv, 0, (size_t)2 * nsrc * nv * sizeof(double), s));
            k_fill_u64<<<1, 32, 0, s>>>(lat->d_counters, (unsigned long long)S, 0ull, 0ull);
            k_extend<D><<<grid_for(S), 256, 0, s>>>(S, axis, lat->vals, nv,
                                                    BuildHash{lat->hkeys, lat->hsite, lat->hmask},
                                                    lat->site_keys, lat->d_counters);
            FR_CHECK_LAUNCH();
            FR_TRY(read_counters(lat, s, hc));
            if (hc[2] & 2ull) {
                set_error("blur hash table overflow");
                return FR_ECAPACITY;
            }
            lat->n_sites = (long long)hc[0];
        }
        S = lat->n_sites;
        if (S > 0) {
            k_jacobi<D><<<grid_for(S), 256, 0, s>>>(S, axis, lat->site_keys, lat->vals,
                                                    lat->vals_alt, nv,
                                                    BuildHash{lat->hkeys, lat->hsite, lat->hmask});
            FR_CHECK_LAUNCH();
            std::swap(lat->vals, lat->vals_alt);
        }
        pc.lap("blur_axis");
    }
    FR_TRY(compact_nonzero<D>(lat, s));
    pc.lap("compact");
    pool_free(lat, lat->hkeys);
    pool_free(lat, lat->hsite);
    lat->hkeys = nullptr;
    lat->hsite = nullptr;
    lat->hmask = 0;
    FR_TRY(build_slice_table<D>(lat, s));
    pc.lap("slice_table");
    lat->blurred = 1;
    return FR_OK;
}

template <int D>
static int slice_impl(const fr_lattice *lat, const double *Q, long long m, double *out,
                      cudaStream_t s) {
    if (m == 0) return FR_OK;
    unsigned grid = (unsigned)std::min<long long>((m + 255) / 256, 148LL * 16);
    const SliceTable t = lat->table();
    for (int c0 = 0; c0 < lat->nv; c0 += 4) {
        const int w = std::min(4, lat->nv - c0);
        if (w == 4) k_slice_generic<D, 4><<<grid, 256, 0, s>>>(Q, m, lat->c, t, c0, lat->nv, out);
        else if (w == 3) k_slice_generic<D, 3><<<grid, 256, 0, s>>>(Q, m, lat->c, t, c0, lat->nv, out);
        else if (w == 2) k_slice_generic<D, 2><<<grid, 256, 0, s>>>(Q, m, lat->c, t, c0, lat->nv, out);
        else k_slice_generic<D, 1><<<grid, 256, 0, s>>>(Q, m, lat->c, t, c0, lat->nv, out);
        FR_CHECK_LAUNCH();
    }
    return FR_OK;
}

}  // namespace fr

// ---------------------------------------------------------------------------
// spatial (Morton) ordering of a point cloud: neighbouring threads then query
// neighbouring simplices, so slice-table gathers hit L1 and coalesce

__device__ __forceinline__ unsigned spread10(unsigned v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

// 8 bits per axis (a 24-bit code: three radix passes); within a cell the
// stable sort keeps the input order -- the cells (1/256 of the box per axis)
// are far below the kernel width for the EM path's lattices
constexpr int kMortonBits = 8;

template <class T>
__global__ void k_morton(const T *pos, long long n, const T *lohi, unsigned *codes,
                         unsigned *idx) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    constexpr float kQ = (float)((1 << kMortonBits) - 1);
    unsigned c = 0;
    for (int a = 0; a < 3; ++a) {
        const float span = fmaxf((float)(lohi[3 + a] - lohi[a]), 1e-30f);
        const float u = (float)(pos[a * n + i] - lohi[a]) / span;
        const unsigned q = (unsigned)fminf(fmaxf(u * kQ, 0.0f), kQ);
        c |= spread10(q) << (2 - a);
    }
    codes[i] = c;
    idx[i] = (unsigned)i;
}

// per-axis min / max of 3 planes: block partials, then one block combines
template <class T>
__global__ void k_bbox_part(const T *pos, long long n, T *part) {
    __shared__ T sh[6][256];
    T v[6];
    for (int a = 0; a < 3; ++a) {
        v[a] = (T)INFINITY;
        v[3 + a] = (T)-INFINITY;
    }
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256)
        for (int a = 0; a < 3; ++a) {
            const T x = pos[a * n + i];
            v[a] = x < v[a] ? x : v[a];
            v[3 + a] = x > v[3 + a] ? x : v[3 + a];
        }
    for (int q = 0; q < 6; ++q) sh[q][threadIdx.x] = v[q];
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (threadIdx.x < h)
            for (int q = 0; q < 6; ++q) {
                const T o = sh[q][threadIdx.x + h], m = sh[q][threadIdx.x];
                sh[q][threadIdx.x] = q < 3 ? (o < m ? o : m) : (o > m ? o : m);
            }
        __syncthreads();
    }
    if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

template <class T>
__global__ void k_bbox_final(const T *part, int nb, T *lohi) {
    // warp q combines column q (6 warps): lanes stride over the block rows,
    // then a shuffle tree (min / max are exact, any order gives the same value)
    const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (q >= 6) return;
    T v = q < 3 ? (T)INFINITY : (T)-INFINITY;
    for (int b = lane; b < nb; b += 32) {
        const T o = part[b * 6 + q];
        v = q < 3 ? (o < v ? o : v) : (o > v ? o : v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        const T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = q < 3 ? (w < v ? w : v) : (w > v ? w : v);
    }
    if (lane == 0) lohi[q] = v;
}

template <class T>
__global__ void k_gather_planes(const T *src, long long n, int planes, const unsigned *perm,
                                T *dst) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned j = perm[i];
    for (int a = 0; a < planes; ++a) dst[a * n + i] = src[a * n + j];
}

#include "fr_lattice_wide.cuh"

// ===========================================================================
// C ABI

using namespace fr;

#define FR_DISPATCH_D(dim, CALL)                                               \
    switch (dim) {                                                             \
        case 1: { constexpr int D = 1; CALL; } break;                          \
        case 2: { constexpr int D = 2; CALL; } break;                          \
        case 3: { constexpr int D = 3; CALL; } break;                          \
        default: set_error("dimension %d not compiled", dim); return FR_EINVAL; \
    }

// d = 4..12: the sorted 128-bit-key lattice (fr_lattice_wide.cuh)
#define FR_DISPATCH_WIDE(dim, CALL)                                            \
    switch (dim) {                                                             \
        case 4: { constexpr int D = 4; CALL; } break;                          \
        case 5: { constexpr int D = 5; CALL; } break;                          \
        case 6: { constexpr int D = 6; CALL; } break;                          \
        case 7: { constexpr int D = 7; CALL; } break;                          \
        case 8: { constexpr int D = 8; CALL; } break;                          \
        case 9: { constexpr int D = 9; CALL; } break;                          \
        case 10: { constexpr int D = 10; CALL; } break;                        \
        case 11: { constexpr int D = 11; CALL; } break;                        \
        case 12: { constexpr int D = 12; CALL; } break;                        \
        default: set_error("dimension %d not compiled", dim); return FR_EINVAL; \
    }

extern "C" {

int fr_abi_version(void) { return 1; }

}  // extern "C"

template <class T>
static int sort_morton_impl(T *pos, int64_t n, int planes, int32_t *perm_out, void *stream) {
    if (!pos || n < 0 || planes < 3) {
        set_error("invalid Morton sort arguments");
        return FR_EINVAL;
    }
    if (n < 2) return FR_OK;
    if (n >= (1LL << 31)) {
        set_error("too many points to sort");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    Scratch sc(s);
    T *lohi, *tmp;
    unsigned *codes, *codes2, *idx, *perm;
    FR_TRY(sc.get(&lohi, 6));
    FR_TRY(sc.get(&codes, n));
    FR_TRY(sc.get(&codes2, n));
    FR_TRY(sc.get(&idx, n));
    FR_TRY(sc.get(&perm, n));
    FR_TRY(sc.get(&tmp, (size_t)n * planes));
    constexpr int kBoxBlocks = 148 * 2;
    T *part;
    FR_TRY(sc.get(&part, (size_t)kBoxBlocks * 6));
    size_t t2 = 0;
    FR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t2, codes, codes2, idx, perm, (int)n, 0,
                                            3 * kMortonBits, s));
    void *tmpb;
    FR_TRY(sc.get((char **)&tmpb, t2));
    k_bbox_part<T><<<kBoxBlocks, 256, 0, s>>>(pos, n, part);
    k_bbox_final<T><<<1, 192, 0, s>>>(part, kBoxBlocks, lohi);
    k_morton<<<grid_for(n), 256, 0, s>>>(pos, n, lohi, codes, idx);
    FR_CHECK_LAUNCH();
    FR_CUDA(cub::DeviceRadixSort::SortPairs(tmpb, t2, codes, codes2, idx, perm, (int)n, 0,
                                            3 * kMortonBits, s));
    k_gather_planes<<<grid_for(n), 256, 0, s>>>(pos, n, planes, perm, tmp);
    FR_CHECK_LAUNCH();
    FR_CUDA(cudaMemcpyAsync(pos, tmp, (size_t)n * planes * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (perm_out)
        FR_CUDA(cudaMemcpyAsync(perm_out, perm, (size_t)n * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    return FR_OK;                           // stream-ordered; scratch frees likewise
}

extern "C" {

int fr_sort_points_morton(float *pos, int64_t n, int planes, int32_t *perm_out, void *stream) {
    return sort_morton_impl<float>(pos, n, planes, perm_out, stream);
}

int fr_sort_points_morton64(double *pos, int64_t n, int planes, int32_t *perm_out, void *stream) {
    return sort_morton_impl<double>(pos, n, planes, perm_out, stream);
}

const char *fr_last_error(void) { return fr::last_error(); }

// lattice counter blocks (4 u64): recycled behind an event recorded on the
// destroyed lattice's stream, so creating a lattice neither allocates
// stream-ordered memory on the legacy stream nor synchronises it (that
// synchronisation waited for every kernel already queued there)
namespace {
struct CounterRecycle {
    std::mutex mu;
    std::vector<std::pair<unsigned long long *, cudaEvent_t>> q;
};
CounterRecycle g_counter_recycle[16];

unsigned long long *counters_get() {
    int dev = 0;
    cudaGetDevice(&dev);
    CounterRecycle &r = g_counter_recycle[dev & 15];
    {
        std::lock_guard<std::mutex> g(r.mu);
        for (size_t i = 0; i < r.q.size(); ++i) {
            const cudaError_t e = cudaEventQuery(r.q[i].second);
            if (e == cudaSuccess) {
                unsigned long long *p = r.q[i].first;
                cudaEventDestroy(r.q[i].second);
                r.q.erase(r.q.begin() + (long)i);
                return p;
            }
            if (e == cudaErrorNotReady) cudaGetLastError();   // not an error: clear it
        }
    }
    unsigned long long *p = nullptr;
    if (cudaMalloc((void **)&p, 4 * sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void counters_put(unsigned long long *p, cudaStream_t s) {
    if (!p) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev, s) != cudaSuccess) {
        cudaGetLastError();
        return;                       // leaked (32 bytes) rather than reused unsafely
    }
    CounterRecycle &r = g_counter_recycle[dev & 15];
    std::lock_guard<std::mutex> g(r.mu);
    r.q.emplace_back(p, ev);
}
}  // namespace

int fr_lattice_create(int dim, const double *sigma, fr_lattice **out) {
    if (!out || !sigma) {
        set_error("null argument");
        return FR_EINVAL;
    }
    LatticeConsts c;
    FR_TRY(make_consts(dim, sigma, &c));
    {
        // keep the stream-ordered pool's pages mapped between builds (a splat
        // at 16.8M points stages ~2 GB of sort scratch)
        static bool pool_set = false;
        if (!pool_set) {
            int dev = 0;
            cudaMemPool_t pool;
            if (cudaGetDevice(&dev) == cudaSuccess &&
                cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                unsigned long long keep = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            pool_set = true;
        }
    }
    fr_lattice *lat = new fr_lattice();
    lat->c = c;
    lat->dim = dim;
    lat->d_counters = counters_get();
    if (!lat->d_counters) {
        delete lat;
        set_error("device allocation failed for lattice counters");
        return FR_ECUDA;
    }
    *out = lat;
    return FR_OK;
}

int fr_lattice_destroy(fr_lattice *lat) {
    if (!lat) return FR_OK;
    // stream-ordered: the buffers return to the pool behind the work already
    // enqueued on the lattice's build stream (callers that read the lattice
    // from other streams synchronise those first -- include/filterreg_b200.h)
    free_build(lat);
    free_slice(lat);
    counters_put(lat->d_counters, lat->stream);
    delete lat;
    return FR_OK;
}

int fr_lattice_splat(fr_lattice *lat, const double *F, const double *V, int64_t n, int nv,
                     void *stream) {
    if (!lat || (n > 0 && (!F || !V))) {
        set_error("null argument");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    lat->stream = s;
    GenericSrc src{F, V, nv};
    if (lat->dim >= 4) {
        FR_DISPATCH_WIDE(lat->dim, FR_TRY((wide_splat<D, GenericSrc>(lat, src, n, nv, s))));
        return FR_OK;
    }
    FR_DISPATCH_D(lat->dim, FR_TRY((splat_impl<D, GenericSrc>(lat, src, n, nv, s))));
    return FR_OK;
}

int fr_lattice_splat_points(fr_lattice *lat, const float *pos, const float *nrm, int64_t n,
                            int value_mode, void *stream) {
    if (!lat || (n > 0 && !pos)) {
        set_error("null argument");
        return FR_EINVAL;
    }
    if (lat->dim != 3) {
        set_error("point splat needs a 3-D lattice");
        return FR_EINVAL;
    }
    if ((value_mode & FR_VALUES_NORMALS) && !nrm) {
        set_error("observation cloud has no normals");
        return FR_EINVAL;
    }
    lat->stream = (cudaStream_t)stream;
    int m2 = (value_mode & FR_VALUES_M2) ? 1 : 0;
    int nv = 4 + m2 + ((value_mode & FR_VALUES_NORMALS) ? 3 : 0);
    PointSrc src{pos, nrm, n, m2, nv};
    return splat_impl<3, PointSrc>(lat, src, n, nv, (cudaStream_t)stream, nullptr,
                                   (value_mode & FR_SPLAT_FLAT_ORDER) != 0,
                                   (value_mode & FR_SPLAT_SPATIAL) != 0);
}

int fr_lattice_splat_points64(fr_lattice *lat, const double *pos, const double *nrm, int64_t n,
                              int value_mode, void *stream) {
    if (!lat || (n > 0 && !pos)) {
        set_error("null argument");
        return FR_EINVAL;
    }
    if (lat->dim != 3) {
        set_error("point splat needs a 3-D lattice");
        return FR_EINVAL;
    }
    if ((value_mode & FR_VALUES_NORMALS) && !nrm) {
        set_error("observation cloud has no normals");
        return FR_EINVAL;
    }
    lat->stream = (cudaStream_t)stream;
    int m2 = (value_mode & FR_VALUES_M2) ? 1 : 0;
    int nv = 4 + m2 + ((value_mode & FR_VALUES_NORMALS) ? 3 : 0);
    PointSrc64 src{pos, nrm, n, m2, nv};
    return splat_impl<3, PointSrc64>(lat, src, n, nv, (cudaStream_t)stream, nullptr,
                                     (value_mode & FR_SPLAT_FLAT_ORDER) != 0,
                                     (value_mode & FR_SPLAT_SPATIAL) != 0);
}

int fr_lattice_splat_upload(fr_lattice *lat, const double *host_xyz, int64_t n, int value_mode,
                            float *d_soa, void *stream, void (*uploaded)(void *), void *ctx) {
    if (!lat || (n > 0 && (!host_xyz || !d_soa))) {
        set_error("null argument");
        return FR_EINVAL;
    }
    if (lat->dim != 3) {
        set_error("point splat needs a 3-D lattice");
        return FR_EINVAL;
    }
    if (value_mode & FR_VALUES_NORMALS) {
        set_error("fr_lattice_splat_upload takes positions only (normals: fr_lattice_splat_points)");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    lat->stream = s;
    const int m2 = (value_mode & FR_VALUES_M2) ? 1 : 0;
    const int nv = 4 + m2;
    PointSrc src{d_soa, nullptr, n, m2, nv};
    // the entries of each staged chunk run on a side stream as soon as the
    // chunk's copy has landed, overlapping the rest of the upload
    const EntriesHook hook = [&](const EntriesLaunch &launch) -> int {
        cudaStream_t side;
        FR_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        std::mutex mu;
        const int st = upload_points_hooked(host_xyz, n, d_soa, s,
                                            [&](long long a, long long len, cudaEvent_t landed) -> int {
            std::lock_guard<std::mutex> g(mu);
            FR_CUDA(cudaStreamWaitEvent(side, landed, 0));
            return launch(a, a + len, side);
        });
        if (uploaded) uploaded(ctx);     // host staging done: the pinned slots are free
        cudaEvent_t done;
        cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
        cudaEventRecord(done, side);
        cudaStreamWaitEvent(s, done, 0);
        cudaEventDestroy(done);
        cudaStreamDestroy(side);
        return st;
    };
    return splat_impl<3, PointSrc>(lat, src, n, nv, s, &hook, (value_mode & FR_SPLAT_FLAT_ORDER) != 0);
}

int fr_lattice_splat_rows64(fr_lattice *lat, const double *host_xyz, int64_t n, int value_mode,
                            double *d_rows, double *d_soa, void *stream, void *follow_stream,
                            void (*uploaded)(void *), void *ctx) {
    if (!lat || (n > 0 && (!host_xyz || !d_rows || !d_soa))) {
        set_error("null argument");
        return FR_EINVAL;
    }
    if (lat->dim != 3) {
        set_error("point splat needs a 3-D lattice");
        return FR_EINVAL;
    }
    if (value_mode & (FR_VALUES_NORMALS | FR_SPLAT_SPATIAL)) {
        set_error("fr_lattice_splat_rows64 takes positions in the caller's order only");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    lat->stream = s;
    const int m2 = (value_mode & FR_VALUES_M2) ? 1 : 0;
    const int nv = 4 + m2;
    const bool flat = (value_mode & FR_SPLAT_FLAT_ORDER) != 0;
    PointSrc64 src{d_soa, nullptr, n, m2, nv};
    const auto follow = [&](cudaStream_t after) -> int {
        // `follow_stream` queues behind the copies (the caller's next
        // transfer does not share the link with them)
        if (follow_stream && (cudaStream_t)follow_stream != after) {
            cudaEvent_t ev;
            FR_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            FR_CUDA(cudaEventRecord(ev, after));
            FR_CUDA(cudaStreamWaitEvent((cudaStream_t)follow_stream, ev, 0));
            cudaEventDestroy(ev);
        }
        if (uploaded) uploaded(ctx);
        return FR_OK;
    };
    // chunks of >= 128k points: below that the DMA is too short to hide anything
    constexpr long long kChunkMin = 1LL << 17;
    const int chunks = (int)std::min<long long>(8, n / kChunkMin);
    if (chunks < 2 || !host_is_pinned(host_xyz, (size_t)n * 3 * sizeof(double))) {
        FR_TRY(fr_upload_rows64(host_xyz, n, d_rows, d_soa, stream));
        FR_TRY(follow(s));
        return splat_impl<3, PointSrc64>(lat, src, n, nv, s, nullptr, flat, false);
    }
    // page-locked rows: the copies of `chunks` ranges go out back to back on
    // a copy stream, enqueued FIRST (the link starts at once; the splat's
    // set-up on `s` does not queue behind them); each range's transpose and
    // splat entries run on a side stream as soon as its copy lands, under
    // the next copies
    cudaStream_t cs = nullptr, side = nullptr;
    std::vector<cudaEvent_t> landed(chunks, nullptr);
    std::vector<long long> lo(chunks + 1);
    for (int k = 0; k <= chunks; ++k) lo[k] = n * k / chunks;
    const auto cleanup = [&]() {
        for (int k = 0; k < chunks; ++k)
            if (landed[k]) cudaEventDestroy(landed[k]);
        if (cs) cudaStreamDestroy(cs);
        if (side) cudaStreamDestroy(side);
    };
    if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess) {
        set_error("CUDA error: %s", cudaGetErrorString(cudaGetLastError()));
        cleanup();
        return FR_ECUDA;
    }
    {
        // the copies overwrite d_rows: after the caller's earlier work on `s`
        cudaEvent_t before;
        cudaEventCreateWithFlags(&before, cudaEventDisableTiming);
        cudaEventRecord(before, s);
        cudaStreamWaitEvent(cs, before, 0);
        cudaEventDestroy(before);
    }
    for (int k = 0; k < chunks; ++k) {
        if (cudaEventCreateWithFlags(&landed[k], cudaEventDisableTiming) != cudaSuccess ||
            cudaMemcpyAsync(d_rows + 3 * lo[k], host_xyz + 3 * lo[k],
                            (size_t)(lo[k + 1] - lo[k]) * 3 * sizeof(double),
                            cudaMemcpyHostToDevice, cs) != cudaSuccess ||
            cudaEventRecord(landed[k], cs) != cudaSuccess) {
            set_error("CUDA error: %s", cudaGetErrorString(cudaGetLastError()));
            cleanup();
            return FR_ECUDA;
        }
    }
    if (const int st = follow(cs)) {
        cleanup();
        return st;
    }
    const EntriesHook hook = [&](const EntriesLaunch &launch) -> int {
        // the splat's set-up on `s` (hash table and counter fills) first
        cudaEvent_t ready;
        FR_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
        cudaEventRecord(ready, s);
        cudaStreamWaitEvent(side, ready, 0);
        cudaEventDestroy(ready);
        int st = FR_OK;
        for (int k = 0; k < chunks && st == FR_OK; ++k) {
            cudaStreamWaitEvent(side, landed[k], 0);
            rows_to_soa64_range(d_rows, n, d_soa, lo[k], lo[k + 1], side);
            st = launch(lo[k], lo[k + 1], side);
        }
        cudaEvent_t done;
        cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
        cudaEventRecord(done, side);
        cudaStreamWaitEvent(s, done, 0);
        cudaEventDestroy(done);
        return st;
    };
    const int st = splat_impl<3, PointSrc64>(lat, src, n, nv, s, &hook, flat, false);
    if (st != FR_OK) {
        // the copies may not have been waited for (an early failure)
        cudaEvent_t done;
        cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
        cudaEventRecord(done, cs);
        cudaStreamWaitEvent(s, done, 0);
        cudaEventDestroy(done);
    }
    cleanup();
    return st;
}

int fr_lattice_blur(fr_lattice *lat, void *stream) {
    if (!lat) {
        set_error("null lattice");
        return FR_EINVAL;
    }
    lat->stream = (cudaStream_t)stream;
    if (lat->dim >= 4) {
        FR_DISPATCH_WIDE(lat->dim, FR_TRY(wide_blur<D>(lat, (cudaStream_t)stream)));
        return FR_OK;
    }
    FR_DISPATCH_D(lat->dim, FR_TRY(blur_impl<D>(lat, (cudaStream_t)stream)));
    return FR_OK;
}

int fr_lattice_info(const fr_lattice *lat, int64_t *num_sites, int *nv, int *blurred) {
    if (!lat) {
        set_error("null lattice");
        return FR_EINVAL;
    }
    if (num_sites) *num_sites = lat->n_sites;
    if (nv) *nv = lat->nv;
    if (blurred) *blurred = lat->blurred;
    return FR_OK;
}

int fr_lattice_set_stream(fr_lattice *lat, void *stream) {
    if (!lat) {
        set_error("null lattice");
        return FR_EINVAL;
    }
    lat->stream = (cudaStream_t)stream;
    return FR_OK;
}

int fr_lattice_dense_cells(const fr_lattice *lat, int64_t *cells) {
    if (!lat || !cells) {
        set_error("null argument");
        return FR_EINVAL;
    }
    *cells = lat->dense_cells;
    return FR_OK;
}

int fr_lattice_dense_cells64(const fr_lattice *lat, int64_t *cells) {
    if (!lat || !cells) {
        set_error("null argument");
        return FR_EINVAL;
    }
    *cells = lat->dcells64 ? lat->dense64_cells : 0;
    return FR_OK;
}

int fr_lattice_export(const fr_lattice *lat, int32_t *keys, double *values, void *stream) {
    if (!lat) {
        set_error("null lattice");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (lat->n_sites == 0) return FR_OK;
    if (keys)
        FR_CUDA(cudaMemcpyAsync(keys, lat->site_keys,
                                (size_t)lat->n_sites * (lat->dim + 1) * sizeof(int),
                                cudaMemcpyDeviceToDevice, s));
    if (values)
        FR_CUDA(cudaMemcpyAsync(values, lat->vals, (size_t)lat->n_sites * lat->nv * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
    return FR_OK;
}

int fr_lattice_slice(const fr_lattice *lat, const double *Q, int64_t m, double *out,
                     void *stream) {
    if (!lat) {
        set_error("null lattice");
        return FR_EINVAL;
    }
    if (!lat->blurred) {
        set_error("slice requires a blurred lattice");
        return FR_ESTATE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (lat->dim >= 4) {
        FR_DISPATCH_WIDE(lat->dim, FR_TRY(wide_slice<D>(lat, Q, m, out, s)));
        return FR_OK;
    }
    FR_DISPATCH_D(lat->dim, FR_TRY(slice_impl<D>(lat, Q, m, out, s)));
    return FR_OK;
}

int fr_simplex(int dim, const double *sigma, const double *F, int64_t n, int32_t *keys,
               double *bary, void *stream) {
    LatticeConsts c;
    FR_TRY(make_consts(dim, sigma, &c));
    if (n == 0) return FR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long *flag = nullptr;
    FR_CUDA(cudaMallocAsync(&flag, sizeof(unsigned long long), s));
    FR_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned long long), s));
    if (dim >= 4) {
        FR_DISPATCH_WIDE(dim, (k_simplex<D><<<grid_for(n), 256, 0, s>>>(F, n, c, keys, bary, flag)));
    } else {
        FR_DISPATCH_D(dim, (k_simplex<D><<<grid_for(n), 256, 0, s>>>(F, n, c, keys, bary, flag)));
    }
    unsigned long long h = 0;
    FR_CUDA(cudaMemcpyAsync(&h, flag, sizeof(h), cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaFreeAsync(flag, s));
    FR_CUDA(cudaStreamSynchronize(s));
    FR_CHECK_LAUNCH();
    if (h) {
        set_error("lattice coordinate outside the packable range");
        return FR_ECAPACITY;
    }
    return FR_OK;
}

int fr_gauss_bruteforce(const double *Q, int64_t m, const double *F, int64_t n, int dim,
                        const double *V, int nv, const double *sigma, double *out,
                        void *stream) {
    if (dim < 1 || dim > kMaxDim || nv < 1 || nv > 16) {
        set_error("bruteforce supports dim 1..12 and 1..16 value columns");
        return FR_EINVAL;
    }
    LatticeConsts c;
    memset(&c, 0, sizeof(c));
    for (int j = 0; j < dim; ++j) {
        if (!std::isfinite(sigma[j]) || !(sigma[j] > 0)) {
            set_error("kernel widths must be finite and positive");
            return FR_EINVAL;
        }
        c.sigma[j] = sigma[j];
    }
    if (m == 0) return FR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    size_t smem = (size_t)kBfTile * (dim + nv) * sizeof(double);
    k_bruteforce<<<grid_for(m, 128), 128, smem, s>>>(Q, m, F, n, dim, V, nv, c, out);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

}  // extern "C"
