// Permutohedral lattice for feature dimensions d = 4..12 (GmmConfig.mode
// "feature" / "concatenated", estep.py:82-96, 171-179).
// Included by fr_lattice.cu: it reuses the bit-exact simplex (fr_common.cuh),
// the value sources and the flat-order site sums of the d <= 3 lattice.
//
// The d <= 3 lattice packs a key's first three coordinates into 63 bits and
// hashes them.  From d = 4 on the keys are packed into 128 bits with per-
// coordinate field widths taken from the data (the rounded remainder-0 range
// plus the simplex and blur margin), most significant field first, so the
// unsigned 128-bit order IS the reference's lexicographic site order
// (_RowCodec, permutohedral.py:96-137).  The site table is kept sorted, as the
// reference keeps it (_index :253-260), and every lookup is a binary search
// (_lookup :262-270):
//   splat  -- per (point, vertex) entry: packed key; a stable two-word LSD
//             radix sort groups the entries of a site in flat (point, vertex)
//             order, so the shared block-per-site kernel sums them in
//             np.add.at's order (:241-242) -- bit-identical values;
//   blur   -- per axis the +-(d+1) neighbours of the non-zero sites are
//             materialised (with the reference's site cap, :304-313), merged
//             into the sorted table, then one Jacobi pass with the reference's
//             float64 expression (:322); all-zero rows dropped at the end;
//   slice  -- bary-weighted gather of the d+1 vertices (:329-341).
#pragma once

namespace fr {

constexpr unsigned long long kWideSentinel = ~0ull;

__device__ __forceinline__ bool wide_lt(unsigned long long ah, unsigned long long al,
                                        unsigned long long bh, unsigned long long bl) {
    return ah < bh || (ah == bh && al < bl);
}

// the field of coordinate i lives at bits [shift[i], shift[i] + bits[i])
__device__ __forceinline__ bool wide_pack(const WideCodec &w, const int *k, unsigned long long &hi,
                                          unsigned long long &lo) {
    hi = 0ull;
    lo = 0ull;
    for (int i = 0; i < w.d; ++i) {
        const unsigned v = (unsigned)(k[i] - w.lo[i]);
        if (v >> w.bits[i]) return false;    // outside the codec range: no such site
        const int sh = w.shift[i];
        if (sh >= 64) {
            hi |= (unsigned long long)v << (sh - 64);
        } else {
            lo |= (unsigned long long)v << sh;
            if (sh + w.bits[i] > 64) hi |= (unsigned long long)v >> (64 - sh);
        }
    }
    return true;
}

__device__ __forceinline__ void wide_unpack(const WideCodec &w, unsigned long long hi,
                                            unsigned long long lo, int *k) {
    int sum = 0;
    for (int i = 0; i < w.d; ++i) {
        const int sh = w.shift[i], b = w.bits[i];
        unsigned long long v;
        if (sh >= 64) v = hi >> (sh - 64);
        else if (sh + b > 64) v = (lo >> sh) | (hi << (64 - sh));
        else v = lo >> sh;
        v &= (1ull << b) - 1ull;
        k[i] = (int)v + w.lo[i];
        sum += k[i];
    }
    k[w.d] = -sum;
}

// first index with key >= (hh, hl) in the sorted table, -1 when not equal
__device__ __forceinline__ long long wide_find(const unsigned long long *kh,
                                               const unsigned long long *kl, long long S,
                                               unsigned long long hh, unsigned long long hl) {
    long long a = 0, b = S;
    while (a < b) {
        const long long mid = (a + b) >> 1;
        if (wide_lt(kh[mid], kl[mid], hh, hl)) a = mid + 1;
        else b = mid;
    }
    return (a < S && kh[a] == hh && kl[a] == hl) ? a : -1;
}

// ---------------------------------------------------------------------------
// splat

template <int D, class Src>
__global__ void k_wide_range(Src src, long long n, LatticeConsts c, int *mn, int *mx,
                             unsigned long long *flag) {
    int lo[D], hi[D];
#pragma unroll
    for (int i = 0; i < D; ++i) { lo[i] = INT_MAX; hi[i] = INT_MIN; }
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        double f[D];
        src.template feat<D>(p, f);
        Simplex<D> s;
        simplex_exact<D>(f, c, s);
        if (s.overflow) { atomicOr(flag, 1ull); continue; }
#pragma unroll
        for (int i = 0; i < D; ++i) {
            lo[i] = min(lo[i], s.rem0[i]);
            hi[i] = max(hi[i], s.rem0[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
        atomicMin(mn + i, lo[i]);
        atomicMax(mx + i, hi[i]);
    }
}

template <int D, class Src>
__global__ void k_wide_entries(Src src, long long n, LatticeConsts c, WideCodec w,
                               unsigned long long *kh, unsigned long long *kl, unsigned *idx,
                               double *bary, double *contrib, unsigned long long *flag) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    double f[D];
    src.template feat<D>(p, f);
    Simplex<D> s;
    simplex_exact<D>(f, c, s);
    bool any_value = false;
    for (int cc = 0; cc < src.nv; ++cc) any_value |= (src.value(p, cc) != 0.0);
#pragma unroll
    for (int l = 0; l <= D; ++l) {
        const long long e = p * (D + 1) + l;
        unsigned long long h = kWideSentinel, lw = kWideSentinel;
        if (s.bary[l] != 0.0 && any_value && !s.overflow) {
            int k[D + 1];
            s.vertex(l, k);
            if (!wide_pack(w, k, h, lw)) {
                atomicOr(flag, 2ull);
                h = lw = kWideSentinel;
            }
        }
        kh[e] = h;
        kl[e] = lw;
        idx[e] = (unsigned)e;
        bary[e] = s.bary[l];
        if (contrib && h != kWideSentinel)
            for (int cc = 0; cc < src.nv; ++cc)
                contrib[e * src.nv + cc] = __dmul_rn(s.bary[l], src.value(p, cc));
    }
}

__global__ void k_gather_u64(long long n, const unsigned *idx, const unsigned long long *src,
                             unsigned long long *dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

// run heads of a sorted key array (the trailing sentinel run excluded)
__global__ void k_wide_heads(long long n, const unsigned long long *kh,
                             const unsigned long long *kl, unsigned char *head) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool sent = kh[i] == kWideSentinel && kl[i] == kWideSentinel;
    head[i] = !sent && (i == 0 || kh[i] != kh[i - 1] || kl[i] != kl[i - 1]);
}

__global__ void k_iota(long long n, int *a) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int)i;
}

__global__ void k_run_counts(int R, const int *off, const int *end_pos, int *cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < R) cnt[r] = (r + 1 < R ? off[r + 1] : *end_pos) - off[r];
}

__global__ void k_count_valid(long long n, const unsigned long long *kh,
                              const unsigned long long *kl, int *end_pos) {
    // entries are sorted with the sentinels last: the first sentinel position
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool sent = kh[i] == kWideSentinel && kl[i] == kWideSentinel;
    const bool prev = i == 0 || !(kh[i - 1] == kWideSentinel && kl[i - 1] == kWideSentinel);
    if (sent && prev) *end_pos = (int)i;
}

template <int D>
__global__ void k_wide_fill(int S, const int *live, const int *run_off,
                            const unsigned long long *kh, const unsigned long long *kl,
                            const double *run_vals, int nv, WideCodec w,
                            unsigned long long *skh, unsigned long long *skl, int *site_keys,
                            double *vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const int r = live[i];
    const unsigned long long h = kh[run_off[r]], l = kl[run_off[r]];
    skh[i] = h;
    skl[i] = l;
    int k[D + 1];
    wide_unpack(w, h, l, k);
#pragma unroll
    for (int q = 0; q <= D; ++q) site_keys[(long long)i * (D + 1) + q] = k[q];
    for (int c = 0; c < nv; ++c) vals[(long long)i * nv + c] = run_vals[(long long)r * nv + c];
}

// stable sort of positions 0..n-1 by the 128-bit key (hi, lo): two LSD passes
static int wide_sort(Scratch &sc, const unsigned long long *kh, const unsigned long long *kl,
                     long long n, int lo_bits, bool use_hi, unsigned long long **kh_out,
                     unsigned long long **kl_out, unsigned **perm_out, cudaStream_t s) {
    unsigned *iota, *p1, *p2;
    unsigned long long *lo1, *hi1, *hi2, *lo2;
    FR_TRY(sc.get(&iota, n));
    FR_TRY(sc.get(&p1, n));
    FR_TRY(sc.get(&p2, n));
    FR_TRY(sc.get(&lo1, n));
    FR_TRY(sc.get(&hi1, n));
    FR_TRY(sc.get(&hi2, n));
    FR_TRY(sc.get(&lo2, n));
    k_iota<<<grid_for(n), 256, 0, s>>>(n, (int *)iota);
    FR_CHECK_LAUNCH();
    size_t tb = 0, tb2 = 0;
    FR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kl, lo1, iota, p1, (int)n, 0, lo_bits, s));
    FR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb2, hi1, hi2, p1, p2, (int)n, 0, 64, s));
    void *tmp;
    FR_TRY(sc.get((char **)&tmp, std::max(tb, tb2)));
    tb = std::max(tb, tb2);
    // the sentinel (all ones) must sort last in the low pass too: sort all 64 bits then
    FR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, kl, lo1, iota, p1, (int)n, 0, 64, s));
    if (use_hi) {
        k_gather_u64<<<grid_for(n), 256, 0, s>>>(n, p1, kh, hi1);
        FR_CHECK_LAUNCH();
        FR_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, hi1, hi2, p1, p2, (int)n, 0, 64, s));
        k_gather_u64<<<grid_for(n), 256, 0, s>>>(n, p2, kl, lo2);
        FR_CHECK_LAUNCH();
        *kh_out = hi2;
        *kl_out = lo2;
        *perm_out = p2;
    } else {
        k_gather_u64<<<grid_for(n), 256, 0, s>>>(n, p1, kh, hi2);
        FR_CHECK_LAUNCH();
        *kh_out = hi2;
        *kl_out = lo1;
        *perm_out = p1;
    }
    (void)lo_bits;
    return FR_OK;
}

static int wide_alloc_sites(fr_lattice *lat, long long S) {
    pool_free(lat, lat->site_keys);
    pool_free(lat, lat->vals);
    pool_free(lat, lat->vals_alt);
    pool_free(lat, lat->wkh);
    pool_free(lat, lat->wkl);
    lat->site_keys = nullptr;
    lat->vals = lat->vals_alt = nullptr;
    lat->wkh = lat->wkl = nullptr;
    const long long c = std::max<long long>(S, 1);
    FR_CUDA(pool_alloc(lat, (void **)&lat->site_keys, (size_t)c * (lat->dim + 1) * sizeof(int)));
    FR_CUDA(pool_alloc(lat, (void **)&lat->vals, (size_t)c * lat->nv * sizeof(double)));
    FR_CUDA(pool_alloc(lat, (void **)&lat->vals_alt, (size_t)c * lat->nv * sizeof(double)));
    FR_CUDA(pool_alloc(lat, (void **)&lat->wkh, (size_t)c * sizeof(unsigned long long)));
    FR_CUDA(pool_alloc(lat, (void **)&lat->wkl, (size_t)c * sizeof(unsigned long long)));
    lat->n_sites = S;
    lat->site_cap = c;
    return FR_OK;
}

template <int D, class Src>
static int wide_splat(fr_lattice *lat, const Src &src, long long n, int nv, cudaStream_t s) {
    if (nv < 1 || nv > 15) {
        set_error("value width %d unsupported (1..15 columns per lattice)", nv);
        return FR_EINVAL;
    }
    free_build(lat);
    free_slice(lat);
    lat->nv = nv;
    lat->blurred = 0;
    lat->splatted = 1;
    if (n == 0) return wide_alloc_sites(lat, 0);
    const long long E = n * (D + 1);
    if (E >= (1LL << 31) - 1) {
        set_error("too many points for one splat (%lld)", n);
        return FR_EINVAL;
    }
    Scratch sc(s);
    // codec: remainder-0 range + the vertex offsets (<= d) + d+1 blur passes
    // of one lattice step (<= d each) per coordinate
    int *mm;
    unsigned long long *flag;
    FR_TRY(sc.get(&mm, 2 * D));
    FR_TRY(sc.get(&flag, 1));
    std::vector<int> init(2 * D);
    for (int i = 0; i < D; ++i) { init[i] = INT_MAX; init[D + i] = INT_MIN; }
    FR_CUDA(cudaMemcpyAsync(mm, init.data(), 2 * D * sizeof(int), cudaMemcpyHostToDevice, s));
    FR_CUDA(cudaMemsetAsync(flag, 0, sizeof(unsigned long long), s));
    k_wide_range<D, Src><<<std::min<long long>(grid_for(n), 1184), 256, 0, s>>>(
        src, n, lat->c, mm, mm + D, flag);
    FR_CHECK_LAUNCH();
    std::vector<int> h(2 * D);
    unsigned long long hflag = 0;
    FR_CUDA(cudaMemcpyAsync(h.data(), mm, 2 * D * sizeof(int), cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(hflag), cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaStreamSynchronize(s));
    if (hflag) {
        set_error("lattice coordinate outside the int32 range");
        return FR_ECAPACITY;
    }
    WideCodec w{};
    w.d = D;
    const long long margin = (long long)D + (long long)(D + 1) * D + 2;
    int total = 0;
    bool any = h[0] <= h[D];
    for (int i = 0; i < D; ++i) {
        const long long lo = any ? (long long)h[i] - margin : 0;
        const long long hi = any ? (long long)h[D + i] + margin : 0;
        int b = 1;
        while (b < 31 && (1LL << b) <= hi - lo) ++b;
        if ((1LL << b) <= hi - lo) {
            set_error("lattice coordinate range too wide for the packed key");
            return FR_ECAPACITY;
        }
        w.lo[i] = (int)lo;
        w.bits[i] = b;
        total += b;
    }
    if (total > 127) {
        set_error("packed lattice keys need %d bits (> 127) at d=%d", total, D);
        return FR_ECAPACITY;
    }
    int sh = total;
    for (int i = 0; i < D; ++i) {
        sh -= w.bits[i];
        w.shift[i] = sh;
    }
    w.total = total;
    lat->wc = w;
    // entries
    unsigned long long *kh, *kl;
    unsigned *eidx;
    double *ebary;
    FR_TRY(sc.get(&kh, E));
    FR_TRY(sc.get(&kl, E));
    FR_TRY(sc.get(&eidx, E));
    FR_TRY(sc.get(&ebary, E));
    double *contrib = nullptr;
    if (contrib_fits(E, nv)) FR_TRY(sc.get(&contrib, (size_t)E * nv));
    k_wide_entries<D, Src><<<grid_for(n), 256, 0, s>>>(src, n, lat->c, w, kh, kl, eidx, ebary,
                                                        contrib, flag);
    FR_CHECK_LAUNCH();
    unsigned long long *skh, *skl;
    unsigned *perm;
    FR_TRY(wide_sort(sc, kh, kl, E, std::min(total, 64), total > 64, &skh, &skl, &perm, s));
    // runs = distinct keys, sentinel run excluded
    unsigned char *head;
    int *iota, *run_off, *d_nruns, *end_pos;
    FR_TRY(sc.get(&head, E));
    FR_TRY(sc.get(&iota, E));
    FR_TRY(sc.get(&run_off, E));
    FR_TRY(sc.get(&d_nruns, 1));
    FR_TRY(sc.get(&end_pos, 1));
    const int Ei = (int)E;
    FR_CUDA(cudaMemcpyAsync(end_pos, &Ei, sizeof(int), cudaMemcpyHostToDevice, s));
    k_wide_heads<<<grid_for(E), 256, 0, s>>>(E, skh, skl, head);
    k_iota<<<grid_for(E), 256, 0, s>>>(E, iota);
    k_count_valid<<<grid_for(E), 256, 0, s>>>(E, skh, skl, end_pos);
    FR_CHECK_LAUNCH();
    size_t tb = 0;
    FR_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, head, run_off, d_nruns, Ei, s));
    void *tmp;
    FR_TRY(sc.get((char **)&tmp, tb));
    FR_CUDA(cub::DeviceSelect::Flagged(tmp, tb, iota, head, run_off, d_nruns, Ei, s));
    int R = 0;
    FR_CUDA(cudaMemcpyAsync(&R, d_nruns, sizeof(int), cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(hflag), cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaStreamSynchronize(s));
    if (hflag & 2ull) {
        set_error("splat key outside the packed range");
        return FR_ECAPACITY;
    }
    if (R == 0) return wide_alloc_sites(lat, 0);
    int *run_cnt;
    double *run_vals;
    FR_TRY(sc.get(&run_cnt, R));
    FR_TRY(sc.get(&run_vals, (size_t)R * nv));
    k_run_counts<<<grid_for(R), 256, 0, s>>>(R, run_off, end_pos, run_cnt);
    FR_CHECK_LAUNCH();
    const size_t smem = (size_t)kSegStages * kSegBlock * nv * sizeof(double);
    FR_CUDA(cudaFuncSetAttribute(k_splat_segsum<D, Src>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_splat_segsum<D, Src><<<R, kSegBlock, smem, s>>>(src, nullptr, run_off, run_cnt, perm, ebary,
                                                      contrib, 0u, nv, run_vals);
    FR_CHECK_LAUNCH();
    // live runs (any non-zero value) -> the sorted site table
    unsigned char *live;
    int *live_runs, *d_nlive;
    FR_TRY(sc.get(&live, R));
    FR_TRY(sc.get(&live_runs, R));
    FR_TRY(sc.get(&d_nlive, 1));
    k_run_live<<<grid_for(R), 256, 0, s>>>(R, nullptr, 0u, run_vals, nv, live);
    FR_CHECK_LAUNCH();
    size_t tb3 = 0;
    FR_CUDA(cub::DeviceSelect::Flagged(nullptr, tb3, iota, live, live_runs, d_nlive, R, s));
    void *tmp3;
    FR_TRY(sc.get((char **)&tmp3, tb3));
    FR_CUDA(cub::DeviceSelect::Flagged(tmp3, tb3, iota, live, live_runs, d_nlive, R, s));
    int S = 0;
    FR_CUDA(cudaMemcpyAsync(&S, d_nlive, sizeof(int), cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaStreamSynchronize(s));
    FR_TRY(wide_alloc_sites(lat, S));
    if (S > 0) {
        k_wide_fill<D><<<grid_for(S), 256, 0, s>>>(S, live_runs, run_off, skh, skl, run_vals, nv, w,
                                                    lat->wkh, lat->wkl, lat->site_keys, lat->vals);
        FR_CHECK_LAUNCH();
    }
    FR_CUDA(cudaStreamSynchronize(s));
    return FR_OK;
}

// ---------------------------------------------------------------------------
// blur

// neighbour keys of a site along `axis`: every coordinate +1 with the axis one
// moved by -d ("plus"), and the mirror ("minus") -- permutohedral.py:309-318
template <int D>
__device__ __forceinline__ void wide_neighbours(const int *k, int axis, int *up, int *dn) {
#pragma unroll
    for (int q = 0; q <= D; ++q) { up[q] = k[q] + 1; dn[q] = k[q] - 1; }
    up[axis] = k[axis] - D;
    dn[axis] = k[axis] + D;
}

template <int D>
__global__ void k_wide_candidates(long long S, int axis, const int *site_keys, const double *vals,
                                  int nv, WideCodec w, const unsigned long long *skh,
                                  const unsigned long long *skl, unsigned long long *ch,
                                  unsigned long long *cl, unsigned long long *counters) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    bool nz = false;
    for (int c = 0; c < nv; ++c) nz |= vals[i * nv + c] != 0.0;
    if (!nz) return;
    int k[D + 1], up[D + 1], dn[D + 1];
#pragma unroll
    for (int q = 0; q <= D; ++q) k[q] = site_keys[i * (D + 1) + q];
    wide_neighbours<D>(k, axis, up, dn);
    const int *nb[2] = {up, dn};
    for (int t = 0; t < 2; ++t) {
        unsigned long long h, l;
        if (!wide_pack(w, nb[t], h, l)) {
            atomicOr(&counters[1], 2ull);
            continue;
        }
        if (wide_find(skh, skl, S, h, l) >= 0) continue;
        const unsigned long long slot = atomicAdd(&counters[0], 1ull);
        ch[slot] = h;
        cl[slot] = l;
    }
}

// merged table: old sites (value rows kept) and fresh keys (zero rows), sorted
__global__ void k_wide_merge_src(long long n, const unsigned *perm, long long S_old,
                                 const unsigned long long *mh, const unsigned long long *ml,
                                 unsigned char *keep) {
    // drop duplicate fresh keys: a fresh key equal to its predecessor
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keep[i] = (i == 0 || mh[i] != mh[i - 1] || ml[i] != ml[i - 1]) ? 1 : 0;
    (void)perm;
    (void)S_old;
}

template <int D>
__global__ void k_wide_merge_fill(int S, const int *sel, const unsigned *perm, long long S_old,
                                  const unsigned long long *mh, const unsigned long long *ml,
                                  const double *old_vals, int nv, WideCodec w,
                                  unsigned long long *skh, unsigned long long *skl, int *site_keys,
                                  double *vals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const int j = sel[i];
    const unsigned src = perm[j];
    skh[i] = mh[j];
    skl[i] = ml[j];
    int k[D + 1];
    wide_unpack(w, mh[j], ml[j], k);
#pragma unroll
    for (int q = 0; q <= D; ++q) site_keys[(long long)i * (D + 1) + q] = k[q];
    for (int c = 0; c < nv; ++c)
        vals[(long long)i * nv + c] = src < S_old ? old_vals[(long long)src * nv + c] : 0.0;
}

template <int D>
__global__ void k_wide_jacobi(long long S, int axis, const int *site_keys, const double *vin,
                              double *vout, int nv, WideCodec w, const unsigned long long *skh,
                              const unsigned long long *skl) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    int k[D + 1], up[D + 1], dn[D + 1];
#pragma unroll
    for (int q = 0; q <= D; ++q) k[q] = site_keys[i * (D + 1) + q];
    wide_neighbours<D>(k, axis, up, dn);
    unsigned long long h, l;
    const long long iu = wide_pack(w, up, h, l) ? wide_find(skh, skl, S, h, l) : -1;
    const long long id = wide_pack(w, dn, h, l) ? wide_find(skh, skl, S, h, l) : -1;
    for (int c = 0; c < nv; ++c) {
        const double vu = iu >= 0 ? vin[iu * nv + c] : 0.0;
        const double vd = id >= 0 ? vin[id * nv + c] : 0.0;
        vout[i * nv + c] = __dadd_rn(__dmul_rn(0.5, vin[i * nv + c]),
                                     __dmul_rn(0.25, __dadd_rn(vu, vd)));
    }
}

template <int D>
__global__ void k_wide_keep_nonzero(long long S, const double *vals, int nv, unsigned char *keep) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    bool nz = false;
    for (int c = 0; c < nv; ++c) nz |= vals[i * nv + c] != 0.0;
    keep[i] = nz;
}

template <int D>
__global__ void k_wide_gather(int S, const int *sel, const unsigned long long *ih,
                              const unsigned long long *il, const int *ikeys, const double *ivals,
                              int nv, unsigned long long *oh, unsigned long long *ol, int *okeys,
                              double *ovals) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const int j = sel[i];
    oh[i] = ih[j];
    ol[i] = il[j];
#pragma unroll
    for (int q = 0; q <= D; ++q) okeys[(long long)i * (D + 1) + q] = ikeys[(long long)j * (D + 1) + q];
    for (int c = 0; c < nv; ++c) ovals[(long long)i * nv + c] = ivals[(long long)j * nv + c];
}

// keep the rows flagged in `keep` (order preserved) as the new site table
template <int D>
static int wide_compact(fr_lattice *lat, const unsigned char *keep, cudaStream_t s) {
    const long long S = lat->n_sites;
    if (S == 0) return FR_OK;
    Scratch sc(s);
    int *iota, *sel, *d_n;
    FR_TRY(sc.get(&iota, S));
    FR_TRY(sc.get(&sel, S));
    FR_TRY(sc.get(&d_n, 1));
    k_iota<<<grid_for(S), 256, 0, s>>>(S, iota);
    FR_CHECK_LAUNCH();
    size_t tb = 0;
    FR_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, keep, sel, d_n, (int)S, s));
    void *tmp;
    FR_TRY(sc.get((char **)&tmp, tb));
    FR_CUDA(cub::DeviceSelect::Flagged(tmp, tb, iota, keep, sel, d_n, (int)S, s));
    int K = 0;
    FR_CUDA(cudaMemcpyAsync(&K, d_n, sizeof(int), cudaMemcpyDeviceToHost, s));
    FR_CUDA(cudaStreamSynchronize(s));
    if (K == S) return FR_OK;
    // move the old table aside, allocate the compacted one
    unsigned long long *oh = lat->wkh, *ol = lat->wkl;
    int *okeys = lat->site_keys;
    double *ovals = lat->vals, *oalt = lat->vals_alt;
    lat->wkh = lat->wkl = nullptr;
    lat->site_keys = nullptr;
    lat->vals = lat->vals_alt = nullptr;
    FR_TRY(wide_alloc_sites(lat, K));
    if (K > 0) {
        k_wide_gather<D><<<grid_for(K), 256, 0, s>>>(K, sel, oh, ol, okeys, ovals, lat->nv,
                                                     lat->wkh, lat->wkl, lat->site_keys,
                                                     lat->vals);
        FR_CHECK_LAUNCH();
    }
    pool_free(lat, oh);
    pool_free(lat, ol);
    pool_free(lat, okeys);
    pool_free(lat, ovals);
    pool_free(lat, oalt);
    return FR_OK;
}

template <int D>
static int wide_blur(fr_lattice *lat, cudaStream_t s) {
    if (!lat->splatted) {
        set_error("blur requires a splatted lattice");
        return FR_ESTATE;
    }
    if (lat->blurred) {
        set_error("lattice already blurred");
        return FR_ESTATE;
    }
    const int nv = lat->nv;
    const WideCodec w = lat->wc;
    const long long cap = std::max<long long>(64 * lat->n_sites, 200000);   // permutohedral.py:304
    unsigned long long hc[3];
    for (int axis = 0; axis <= D; ++axis) {
        long long S = lat->n_sites;
        FR_CUDA(cudaMemsetAsync(lat->d_counters, 0, 3 * sizeof(unsigned long long), s));
        if (S > 0) {
            k_count_nonzero<<<grid_for(S), 256, 0, s>>>(S, lat->vals, nv, lat->d_counters + 1);
            FR_CHECK_LAUNCH();
        }
        FR_TRY(read_counters(lat, s, hc));
        const long long nsrc = (long long)hc[1];
        if (S + 2 * nsrc <= cap && nsrc > 0) {
            Scratch sc(s);
            unsigned long long *ch, *cl;
            FR_TRY(sc.get(&ch, 2 * nsrc + S));
            FR_TRY(sc.get(&cl, 2 * nsrc + S));
            // candidates first, then the old keys appended behind them
            FR_CUDA(cudaMemsetAsync(lat->d_counters, 0, 3 * sizeof(unsigned long long), s));
            k_wide_candidates<D><<<grid_for(S), 256, 0, s>>>(S, axis, lat->site_keys, lat->vals,
                                                             nv, w, lat->wkh, lat->wkl, ch, cl,
                                                             lat->d_counters);
            FR_CHECK_LAUNCH();
            FR_TRY(read_counters(lat, s, hc));
            if (hc[1] & 2ull) {
                set_error("blur neighbour outside the packed key range");
                return FR_ECAPACITY;
            }
            const long long F = (long long)hc[0];
            if (F > 0) {
                // merged key list: old sites at positions [0, S), fresh at [S, S+F)
                unsigned long long *mh, *ml;
                FR_TRY(sc.get(&mh, S + F));
                FR_TRY(sc.get(&ml, S + F));
                FR_CUDA(cudaMemcpyAsync(mh, lat->wkh, S * sizeof(unsigned long long),
                                        cudaMemcpyDeviceToDevice, s));
                FR_CUDA(cudaMemcpyAsync(ml, lat->wkl, S * sizeof(unsigned long long),
                                        cudaMemcpyDeviceToDevice, s));
                FR_CUDA(cudaMemcpyAsync(mh + S, ch, F * sizeof(unsigned long long),
                                        cudaMemcpyDeviceToDevice, s));
                FR_CUDA(cudaMemcpyAsync(ml + S, cl, F * sizeof(unsigned long long),
                                        cudaMemcpyDeviceToDevice, s));
                unsigned long long *sh, *sl;
                unsigned *perm;
                FR_TRY(wide_sort(sc, mh, ml, S + F, std::min(w.total, 64), w.total > 64, &sh, &sl,
                                 &perm, s));
                // old keys precede equal fresh ones (stable: positions [0, S) first),
                // so the first of each run keeps the old row
                unsigned char *keep;
                int *iota, *sel, *d_n;
                FR_TRY(sc.get(&keep, S + F));
                FR_TRY(sc.get(&iota, S + F));
                FR_TRY(sc.get(&sel, S + F));
                FR_TRY(sc.get(&d_n, 1));
                k_wide_merge_src<<<grid_for(S + F), 256, 0, s>>>(S + F, perm, S, sh, sl, keep);
                k_iota<<<grid_for(S + F), 256, 0, s>>>(S + F, iota);
                FR_CHECK_LAUNCH();
                size_t tb = 0;
                FR_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota, keep, sel, d_n, (int)(S + F), s));
                void *tmp;
                FR_TRY(sc.get((char **)&tmp, tb));
                FR_CUDA(cub::DeviceSelect::Flagged(tmp, tb, iota, keep, sel, d_n, (int)(S + F), s));
                int S2 = 0;
                FR_CUDA(cudaMemcpyAsync(&S2, d_n, sizeof(int), cudaMemcpyDeviceToHost, s));
                FR_CUDA(cudaStreamSynchronize(s));
                double *old_vals = lat->vals;
                lat->vals = nullptr;
                FR_TRY(wide_alloc_sites(lat, S2));
                k_wide_merge_fill<D><<<grid_for(S2), 256, 0, s>>>(S2, sel, perm, S, sh, sl,
                                                                  old_vals, nv, w, lat->wkh,
                                                                  lat->wkl, lat->site_keys,
                                                                  lat->vals);
                FR_CHECK_LAUNCH();
                pool_free(lat, old_vals);
            }
        }
        S = lat->n_sites;
        if (S > 0) {
            k_wide_jacobi<D><<<grid_for(S), 256, 0, s>>>(S, axis, lat->site_keys, lat->vals,
                                                         lat->vals_alt, nv, w, lat->wkh, lat->wkl);
            FR_CHECK_LAUNCH();
            std::swap(lat->vals, lat->vals_alt);
        }
    }
    if (lat->n_sites > 0) {
        Scratch sc(s);
        unsigned char *keep;
        FR_TRY(sc.get(&keep, lat->n_sites));
        k_wide_keep_nonzero<D><<<grid_for(lat->n_sites), 256, 0, s>>>(lat->n_sites, lat->vals, nv,
                                                                       keep);
        FR_CHECK_LAUNCH();
        FR_TRY(wide_compact<D>(lat, keep, s));
    }
    FR_CUDA(cudaStreamSynchronize(s));
    lat->blurred = 1;
    return FR_OK;
}

// ---------------------------------------------------------------------------
// slice

template <int D>
__global__ void k_wide_slice(const double *Q, long long m, LatticeConsts c, WideCodec w,
                             const unsigned long long *skh, const unsigned long long *skl,
                             long long S, const double *vals, int nv, double *out) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= m) return;
    double f[D];
#pragma unroll
    for (int j = 0; j < D; ++j) f[j] = Q[p * D + j];
    Simplex<D> s;
    simplex_exact<D>(f, c, s);
    double acc[16];
    for (int q = 0; q < nv; ++q) acc[q] = 0.0;
    if (!s.overflow) {
        for (int l = 0; l <= D; ++l) {
            int k[D + 1];
            s.vertex(l, k);
            unsigned long long h, lw;
            const long long i = wide_pack(w, k, h, lw) ? wide_find(skh, skl, S, h, lw) : -1;
            if (i < 0) continue;
            for (int q = 0; q < nv; ++q)
                acc[q] = __dadd_rn(acc[q], __dmul_rn(s.bary[l], vals[i * nv + q]));
        }
    }
    for (int q = 0; q < nv; ++q) out[p * nv + q] = __dmul_rn(c.gain, acc[q]);
}

template <int D>
static int wide_slice(const fr_lattice *lat, const double *Q, long long m, double *out,
                      cudaStream_t s) {
    if (m == 0) return FR_OK;
    if (lat->n_sites == 0) {
        FR_CUDA(cudaMemsetAsync(out, 0, (size_t)m * lat->nv * sizeof(double), s));
        return FR_OK;
    }
    k_wide_slice<D><<<grid_for(m, 128), 128, 0, s>>>(Q, m, lat->c, lat->wc, lat->wkh, lat->wkl,
                                                     lat->n_sites, lat->vals, lat->nv, out);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

}  // namespace fr
