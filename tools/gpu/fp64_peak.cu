// FP64 FMA throughput of one B200 (the roofline denominator of the float64
// EM pass): every thread runs 8 independent DFMA chains; 148 x 4 CTAs of 256
// threads; CUDA events around the kernel; prints TFLOP/s (2 flops per DFMA).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = fma(x[c], a, b);
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;      // keep the chains alive
}

int main() {
    double *out;
    cudaMalloc(&out, sizeof(double));
    const int blocks = 148 * 4, threads = 256, iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
    printf("{\"fp64_tflops\": %.3f, \"kernel_ms\": %.4f, \"blocks\": %d, \"threads\": %d, "
           "\"how\": \"8 independent DFMA chains per thread, best of 5, CUDA events\"}\n",
           flops / (best * 1e-3) / 1e12, best, blocks, threads);
    return 0;
}
