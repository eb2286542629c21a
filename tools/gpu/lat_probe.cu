// Dependent-chain latencies on one thread (diagnostic for the serial
// float64 solve): DFMA, DADD, MUFU.RCP64H, shared load, warp shuffle.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double a, double b) {
    __shared__ double sh[64];
    if (threadIdx.x < 64) sh[threadIdx.x] = (double)threadIdx.x * 1e-3;
    __syncwarp();
    double x = a;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = fma(x, b, a);
    }
    long long t1 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) x = x + b;
    }
    long long t2 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            double r;
            asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
            x = r;
        }
    }
    long long t3 = clock64();
    int idx = (int)x & 63;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) idx = ((int)(sh[idx] * 1e3) + 1) & 63;
    }
    long long t4 = clock64();
    double y = x;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) y = __shfl_xor_sync(0xffffffffu, y, 1) + 1.0;
    }
    long long t5 = clock64();
    double z = a;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) z = sqrt(z + b);
    }
    long long t6 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j) { double s, c; sincos(z, &s, &c); z = s + c * 1e-3; }
    }
    long long t7 = clock64();
    if (threadIdx.x == 0) {
        out[0] = x + idx + y + z;
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
        cyc[5] = t6 - t5; cyc[6] = t7 - t6;
    }
}
int main() {
    double *o; long long *c, h[7];
    cudaMalloc(&o, 8); cudaMalloc(&c, 7 * 8);
    for (int r = 0; r < 3; ++r) {
        k<<<1, 32>>>(o, c, 0.5, 0.999);
        cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    }
    printf("cycles per dependent op: DFMA %.1f DADD %.1f RCP64 %.1f LDS(+cvt) %.1f SHFL+DADD %.1f "
           "sqrt+DADD %.1f sincos+DFMA %.1f\n",
           h[0] / 4096.0, h[1] / 4096.0, h[2] / 4096.0, h[3] / 4096.0, h[4] / 4096.0, h[5] / 4096.0,
           h[6] / 1024.0);
    return 0;
}
