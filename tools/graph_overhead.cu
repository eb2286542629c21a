// Probe: per-node cost of the device loop's graph shape on this GPU.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/graph_overhead.cu -o /tmp/go && /tmp/go
// (a) N tiny kernels per graph; (b) memcpy-to-symbol + tiny kernel per step;
// (c) a 296-block kernel of fixed work per step, with / without the memcpy.
#include <cstdio>
#include <cuda_runtime.h>

struct P { float v[80]; };
__constant__ P c_p;

__global__ void k_tiny(float *o) { if (threadIdx.x == 0 && blockIdx.x == 0) o[0] += c_p.v[3]; }
__global__ void k_work(float *o, int iters) {
    float a = threadIdx.x * 1e-3f, b = c_p.v[1];
    for (int i = 0; i < iters; ++i) a = fmaf(a, 0.999f, b);
    if (a == 12345.f) o[0] = a;
}

static float time_graph(void (*body)(cudaStream_t, float *, P *, int), float *o, P *d, int arg,
                        int steps) {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 8; ++i) body(s, o, d, arg);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int i = 0; i < steps / 8; ++i) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return 1e3f * ms / steps;
}

static void b_tiny(cudaStream_t s, float *o, P *, int) { k_tiny<<<1, 32, 0, s>>>(o); }
static void b_tiny2(cudaStream_t s, float *o, P *, int) { k_tiny<<<1, 32, 0, s>>>(o); k_tiny<<<1, 32, 0, s>>>(o); }
static void b_cpy_tiny(cudaStream_t s, float *o, P *d, int) {
    cudaMemcpyToSymbolAsync(c_p, d, sizeof(P), 0, cudaMemcpyDeviceToDevice, s);
    k_tiny<<<1, 32, 0, s>>>(o);
}
static void b_work(cudaStream_t s, float *o, P *, int n) { k_work<<<296, 256, 0, s>>>(o, n); }
static void b_cpy_work(cudaStream_t s, float *o, P *d, int n) {
    cudaMemcpyToSymbolAsync(c_p, d, sizeof(P), 0, cudaMemcpyDeviceToDevice, s);
    k_work<<<296, 256, 0, s>>>(o, n);
}
static void b_work_tiny(cudaStream_t s, float *o, P *, int n) {
    k_work<<<296, 256, 0, s>>>(o, n);
    k_tiny<<<1, 32, 0, s>>>(o);
}

int main() {
    float *o;
    P *d;
    cudaMalloc(&o, 4);
    cudaMalloc(&d, sizeof(P));
    cudaMemset(d, 0, sizeof(P));
    printf("tiny kernel per step          %.2f us\n", time_graph(b_tiny, o, d, 0, 8000));
    printf("2 tiny kernels per step       %.2f us\n", time_graph(b_tiny2, o, d, 0, 8000));
    printf("memcpy-to-symbol + tiny       %.2f us\n", time_graph(b_cpy_tiny, o, d, 0, 8000));
    for (int n : {20000, 60000}) {
        printf("work(%d)                   %.2f us\n", n, time_graph(b_work, o, d, n, 800));
        printf("memcpy + work(%d)          %.2f us\n", n, time_graph(b_cpy_work, o, d, n, 800));
        printf("work(%d) + tiny            %.2f us\n", n, time_graph(b_work_tiny, o, d, n, 800));
    }
    return 0;
}
