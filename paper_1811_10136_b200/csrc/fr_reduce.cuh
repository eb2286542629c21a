// Deterministic fixed-order reductions shared by the point-sweep kernels:
// per-thread float64 accumulators -> warp shuffle tree -> per-block row of
// partials -> one fixed-order column reduction.  No floating-point atomics, so
// a given grid reproduces its sums bit for bit (the reference pins
// bit-identical reruns, test_pipeline.py:324-339).
#pragma once

#include "fr_common.cuh"

namespace fr {

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

// column c of partials[nblk][na] reduced by warp c in a fixed order; skipped
// when *done is set (device-resident EM loop finished)
static __global__ void k_reduce_cols(const double *partials, int nblk, int na, double *out,
                                     const int *done, const int *done2 = nullptr) {
    if ((done && *done) || (done2 && *done2)) return;
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (c >= na) return;
    double v = 0.0;
    for (int b = lane; b < nblk; b += 32) v += partials[(long long)b * na + c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) out[c] = v;
}

// one full wave of the point-sweep kernels (2 CTAs of 256 per SM); fixed per
// device so the reduction order -- and the sums -- are reproducible
static inline int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

// persistent pass grids: 2 blocks per SM, 3 for the dense-grid pass
static inline int pass_grid() { return 2 * sm_count(); }
static inline int pass_grid_dense() { return 3 * sm_count(); }
// scratch rows every pass grid fits in
static inline int pass_grid_max() { return 4 * sm_count(); }

}  // namespace fr
