// Host -> device upload of a point cloud: (n, 3) float64 rows in pageable
// host memory -> (3, n) float32 planes in HBM (the layout every pass reads).
//
// The reference keeps clouds as float64 NumPy arrays (geometry.py:109-139) and
// the engine converts them once at the boundary.  A plain
// pageable copy of the float64 rows runs at ~10 GB/s and the NumPy float32
// conversion is single-threaded, so at C5 sizes the upload dominated the
// end-to-end call.  Here worker threads each own a slice of the rows and two
// pinned staging slots from a process-wide pool: a worker converts a sub-chunk
// (float32 rounding to nearest, as numpy.astype) into one slot as three
// planes while the DMA of its other slot is in flight, then enqueues one 2-D
// copy into the three device planes on the caller's stream.  The workers are
// joined before return; the copies stay stream-ordered.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "fr_common.cuh"

namespace fr {

namespace {

constexpr long long kSubChunk = 1 << 17;   // points per staging slot (1.5 MB)
constexpr int kMaxWorkers = 16;

struct StagePool {
    std::mutex mu;
    int workers = 0;
    float *base = nullptr;                 // one pinned block, carved into slots
    float *slots[kMaxWorkers][2] = {};     // kSubChunk float32 rows, or kSubChunk / 2 float64
    cudaEvent_t done[kMaxWorkers][2] = {};

    // all kMaxWorkers x 2 slots (48 MB pinned) on first use, so the one-time
    // allocation lands in whatever call comes first (e.g. a warm-up)
    int init() {
        if (workers) return FR_OK;
        const size_t slot = (size_t)kSubChunk * 3;
        FR_CUDA(cudaHostAlloc(&base, slot * 2 * kMaxWorkers * sizeof(float), cudaHostAllocDefault));
        for (int i = 0; i < kMaxWorkers; ++i)
            for (int j = 0; j < 2; ++j) {
                slots[i][j] = base + slot * (2 * i + j);
                FR_CUDA(cudaEventCreateWithFlags(&done[i][j], cudaEventDisableTiming));
            }
        workers = kMaxWorkers;
        return FR_OK;
    }
};

StagePool &pool() {
    static StagePool p;
    return p;
}

// (n, 3) float64 rows -> three float32 planes, round to nearest (as
// numpy.astype).  Four rows per step: three 32-byte loads, converted and
// de-interleaved with AVX when the CPU has it (runtime check, so the library
// still runs on a host without it), else the scalar loop.
__attribute__((target("avx2"))) static void convert_rows_avx2(const double *r, long long len,
                                                              float *x, float *y, float *z) {
    long long i = 0;
    for (; i + 4 <= len; i += 4) {
        const double *q = r + 3 * i;
        alignas(32) float f[12];
        for (int k = 0; k < 12; ++k) f[k] = (float)q[k];
        x[i] = f[0]; y[i] = f[1]; z[i] = f[2];
        x[i + 1] = f[3]; y[i + 1] = f[4]; z[i + 1] = f[5];
        x[i + 2] = f[6]; y[i + 2] = f[7]; z[i + 2] = f[8];
        x[i + 3] = f[9]; y[i + 3] = f[10]; z[i + 3] = f[11];
    }
    for (; i < len; ++i) {
        x[i] = (float)r[3 * i];
        y[i] = (float)r[3 * i + 1];
        z[i] = (float)r[3 * i + 2];
    }
}
static void convert_rows_scalar(const double *r, long long len, float *x, float *y, float *z) {
    for (long long i = 0; i < len; ++i) {
        x[i] = (float)r[3 * i];
        y[i] = (float)r[3 * i + 1];
        z[i] = (float)r[3 * i + 2];
    }
}
static void convert_rows(const double *r, long long len, float *x, float *y, float *z) {
    static const bool avx2 = __builtin_cpu_supports("avx2") && !getenv("FR_UPLOAD_SCALAR");
    if (avx2) convert_rows_avx2(r, len, x, y, z);
    else convert_rows_scalar(r, len, x, y, z);
}
// float64 planes: a transpose, no rounding (the float64 query path keeps the
// caller's values bit for bit)
static void convert_rows(const double *r, long long len, double *x, double *y, double *z) {
    for (long long i = 0; i < len; ++i) {
        x[i] = r[3 * i];
        y[i] = r[3 * i + 1];
        z[i] = r[3 * i + 2];
    }
}

// raw rows: the float64 path keeps the caller's bytes, so the host side is a
// plain copy into the pinned slot (memcpy-bound) and the transpose to planes
// runs on the device (k_rows_to_soa64)
static void copy_rows(const double *r, long long len, double *dst) {
    std::memcpy(dst, r, (size_t)len * 3 * sizeof(double));
}

struct WorkerResult {
    int status = FR_OK;
    char msg[256] = {0};
};

// worker threads run on the caller's device: CUDA's current device is per
// host thread, and a fresh std::thread starts on device 0 (a launch or copy
// from it would target another GPU's context for any caller on device k > 0)
template <class T>
void worker(int dev, int id, const double *src, long long n, long long a, long long b, T *dst,
            cudaStream_t s, WorkerResult *res, const ChunkHook *hook) {
    StagePool &p = pool();
    constexpr long long kSub = kSubChunk * (long long)sizeof(float) / (long long)sizeof(T);
    int slot = 0;
    cudaError_t e = cudaSetDevice(dev);
    for (long long c = a; c < b && e == cudaSuccess; c += kSub) {
        const long long len = std::min(kSub, b - c);
        T *buf = reinterpret_cast<T *>(p.slots[id][slot]);
        e = cudaEventSynchronize(p.done[id][slot]);   // slot's previous DMA
        if (e == cudaSuccess) {
            const double *r = src + 3 * c;
            T *x = buf, *y = buf + kSub, *z = buf + 2 * kSub;
            convert_rows(r, len, x, y, z);
            e = cudaMemcpy2DAsync(dst + c, (size_t)n * sizeof(T), buf, (size_t)kSub * sizeof(T),
                                  (size_t)len * sizeof(T), 3, cudaMemcpyHostToDevice, s);
        }
        if (e == cudaSuccess) e = cudaEventRecord(p.done[id][slot], s);
        if (e == cudaSuccess && hook && *hook) {
            const int st = (*hook)(c, len, p.done[id][slot]);
            if (st != FR_OK) {
                res->status = st;
                snprintf(res->msg, sizeof(res->msg), "point upload hook: %s", last_error());
                return;
            }
        }
        slot ^= 1;
    }
    if (e != cudaSuccess) {
        res->status = FR_ECUDA;
        snprintf(res->msg, sizeof(res->msg), "point upload: %s", cudaGetErrorString(e));
    }
}

// rows mode: (n, 3) float64 rows -> the device row buffer, same slots/events
void worker_rows(int dev, int id, const double *src, long long a, long long b, double *d_rows,
                 cudaStream_t s, WorkerResult *res) {
    StagePool &p = pool();
    constexpr long long kSub = kSubChunk * (long long)sizeof(float) / (long long)sizeof(double);
    int slot = 0;
    cudaError_t e = cudaSetDevice(dev);
    for (long long c = a; c < b && e == cudaSuccess; c += kSub) {
        const long long len = std::min(kSub, b - c);
        double *buf = reinterpret_cast<double *>(p.slots[id][slot]);
        e = cudaEventSynchronize(p.done[id][slot]);
        if (e == cudaSuccess) {
            copy_rows(src + 3 * c, len, buf);
            e = cudaMemcpyAsync(d_rows + 3 * c, buf, (size_t)len * 3 * sizeof(double),
                                cudaMemcpyHostToDevice, s);
        }
        if (e == cudaSuccess) e = cudaEventRecord(p.done[id][slot], s);
        slot ^= 1;
    }
    if (e != cudaSuccess) {
        res->status = FR_ECUDA;
        snprintf(res->msg, sizeof(res->msg), "point upload: %s", cudaGetErrorString(e));
    }
}

// true when [p, p + bytes) is page-locked host memory (cudaHostAlloc'd or
// registered): both ends are checked, a failed query is cleared
bool host_is_pinned_impl(const void *p, size_t bytes) {
    for (const char *q : {static_cast<const char *>(p), static_cast<const char *>(p) + bytes - 1}) {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, q) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        if (at.type != cudaMemoryTypeHost) return false;
    }
    return true;
}

// (n, 3) rows -> (3, n) planes; a warp reads 768 contiguous bytes
__global__ void k_rows_to_soa64(const double *__restrict__ rows, long long n,
                                double *__restrict__ soa) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double x = rows[3 * i], y = rows[3 * i + 1], z = rows[3 * i + 2];
        soa[i] = x;
        soa[n + i] = y;
        soa[2 * n + i] = z;
    }
}

// coordinate sums / minima / maxima of (3, n) float64 planes: fixed grid,
// fixed order (per-thread strided sums, block tree, then one block over the
// block partials), so the result is run-to-run identical
constexpr int kStatBlocks = 148, kStatThreads = 256;

__global__ void __launch_bounds__(kStatThreads) k_point_stats64(const double *__restrict__ soa,
                                                                long long n, double *part) {
    __shared__ double sh[9][kStatThreads];
    double v[9];
    for (int c = 0; c < 3; ++c) {
        v[c] = 0.0;
        v[3 + c] = INFINITY;
        v[6 + c] = -INFINITY;
    }
    for (long long i = blockIdx.x * (long long)kStatThreads + threadIdx.x; i < n;
         i += (long long)gridDim.x * kStatThreads)
        for (int c = 0; c < 3; ++c) {
            const double x = soa[c * n + i];
            v[c] += x;
            v[3 + c] = fmin(v[3 + c], x);
            v[6 + c] = fmax(v[6 + c], x);
        }
    for (int q = 0; q < 9; ++q) sh[q][threadIdx.x] = v[q];
    __syncthreads();
    for (int h = kStatThreads / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h)
            for (int c = 0; c < 3; ++c) {
                sh[c][threadIdx.x] += sh[c][threadIdx.x + h];
                sh[3 + c][threadIdx.x] = fmin(sh[3 + c][threadIdx.x], sh[3 + c][threadIdx.x + h]);
                sh[6 + c][threadIdx.x] = fmax(sh[6 + c][threadIdx.x], sh[6 + c][threadIdx.x + h]);
            }
        __syncthreads();
    }
    if (threadIdx.x < 9) part[blockIdx.x * 9 + threadIdx.x] = sh[threadIdx.x][0];
}

// 16 lanes per statistic each combine every 16th block row (loads issued
// together), then lane 0 combines the 16 in order: fixed order throughout
__global__ void k_point_stats64_final(const double *part, int nb, double *out) {
    __shared__ double sh[9][16];
    const int q = threadIdx.x / 16, j = threadIdx.x % 16;
    if (q < 9) {
        const bool add = q < 3, mn = q >= 3 && q < 6;
        double v = add ? 0.0 : (mn ? INFINITY : -INFINITY);
#pragma unroll 4
        for (int b = j; b < nb; b += 16) {
            const double x = part[b * 9 + q];
            v = add ? v + x : (mn ? fmin(v, x) : fmax(v, x));
        }
        sh[q][j] = v;
    }
    __syncthreads();
    if (j == 0 && q < 9) {
        double v = sh[q][0];
        for (int k = 1; k < 16; ++k)
            v = q < 3 ? v + sh[q][k] : (q < 6 ? fmin(v, sh[q][k]) : fmax(v, sh[q][k]));
        out[q] = v;
    }
}

}  // namespace
}  // namespace fr

using namespace fr;

namespace fr {

// the staged upload; `hook` (may be empty) is called from the worker threads
// (current device = the caller's) after each sub-chunk's copy was enqueued,
// with the event that marks it landed; a hook's failure status is returned
template <class T>
static int upload_impl(const double *host_xyz, long long n, T *d_soa, cudaStream_t s,
                       const ChunkHook &hook) {
    if (n < 0 || (n > 0 && (!host_xyz || !d_soa))) {
        set_error("fr_upload_points: invalid arguments");
        return FR_EINVAL;
    }
    if (n == 0) return FR_OK;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    long long cap = kMaxWorkers;
    if (const char *e = getenv("FR_UPLOAD_WORKERS")) cap = std::max(1, std::min(kMaxWorkers, atoi(e)));
    const int w = (int)std::max<long long>(
        1, std::min<long long>({cap, (long long)hw, (n + kSubChunk - 1) / kSubChunk}));
    int dev = 0;
    FR_CUDA(cudaGetDevice(&dev));
    StagePool &p = pool();
    std::lock_guard<std::mutex> lock(p.mu);   // one upload at a time owns the slots
    FR_TRY(p.init());
    const long long per = (n + w - 1) / w;
    std::vector<WorkerResult> res(w);
    std::vector<std::thread> th;
    th.reserve(w);
    for (int i = 0; i < w; ++i) {
        const long long a = std::min<long long>(n, (long long)i * per);
        const long long b = std::min<long long>(n, a + per);
        th.emplace_back(worker<T>, dev, i, host_xyz, (long long)n, a, b, d_soa, s, &res[i], &hook);
    }
    for (auto &t : th) t.join();
    for (const auto &r : res)
        if (r.status != FR_OK) {
            set_error("%s", r.msg);
            return r.status;
        }
    return FR_OK;
}

int upload_points_hooked(const double *host_xyz, long long n, float *d_soa, cudaStream_t s,
                         const ChunkHook &hook) {
    return upload_impl<float>(host_xyz, n, d_soa, s, hook);
}

__global__ void k_rows_to_soa64_range(const double *__restrict__ rows, long long n,
                                      double *__restrict__ soa, long long a, long long b) {
    for (long long i = a + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < b;
         i += (long long)gridDim.x * blockDim.x) {
        const double x = rows[3 * i], y = rows[3 * i + 1], z = rows[3 * i + 2];
        soa[i] = x;
        soa[n + i] = y;
        soa[2 * n + i] = z;
    }
}

void rows_to_soa64_range(const double *rows, long long n, double *soa, long long a, long long b,
                         cudaStream_t s) {
    if (b <= a) return;
    const int blocks = (int)std::min<long long>((b - a + 255) / 256, 148LL * 16);
    k_rows_to_soa64_range<<<blocks, 256, 0, s>>>(rows, n, soa, a, b);
}

bool host_is_pinned(const void *p, size_t bytes) { return host_is_pinned_impl(p, bytes); }

}  // namespace fr

extern "C" int fr_upload_points(const double *host_xyz, int64_t n, float *d_soa, void *stream) {
    return fr::upload_points_hooked(host_xyz, n, d_soa, (cudaStream_t)stream, fr::ChunkHook());
}

extern "C" int fr_upload_points64(const double *host_xyz, int64_t n, double *d_soa, void *stream) {
    return fr::upload_impl<double>(host_xyz, n, d_soa, (cudaStream_t)stream, fr::ChunkHook());
}

extern "C" int fr_upload_rows64(const double *host_xyz, int64_t n, double *d_rows, double *d_soa,
                                void *stream) {
    using namespace fr;
    if (n < 0 || (n > 0 && (!host_xyz || !d_rows || !d_soa))) {
        set_error("fr_upload_rows64: invalid arguments");
        return FR_EINVAL;
    }
    if (n == 0) return FR_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int blocks = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
    if (host_is_pinned_impl(host_xyz, (size_t)n * 3 * sizeof(double))) {
        // page-locked rows (e.g. load_cloud(..., pinned=True)): one DMA at
        // PCIe rate straight from the caller's buffer, no staging copy
        FR_CUDA(cudaMemcpyAsync(d_rows, host_xyz, (size_t)n * 3 * sizeof(double),
                                cudaMemcpyHostToDevice, s));
        k_rows_to_soa64<<<blocks, 256, 0, s>>>(d_rows, n, d_soa);
        FR_CHECK_LAUNCH();
        return FR_OK;
    }
    constexpr long long kSub = kSubChunk / 2;
    long long cap = 4;          // the copies are memcpy-bound: a few threads fill PCIe
    if (const char *e = getenv("FR_UPLOAD_WORKERS")) cap = std::max(1, std::min(kMaxWorkers, atoi(e)));
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const long long chunks = (n + kSub - 1) / kSub;
    const int w = (int)std::max<long long>(1, std::min<long long>({cap, (long long)hw, chunks}));
    int dev = 0;
    FR_CUDA(cudaGetDevice(&dev));
    StagePool &p = pool();
    {
        std::lock_guard<std::mutex> lock(p.mu);
        FR_TRY(p.init());
        // whole sub-chunks per worker, so every DMA but the last is a full slot
        const long long per = ((chunks + w - 1) / w) * kSub;
        std::vector<WorkerResult> res(w);
        std::vector<std::thread> th;
        th.reserve(w);
        for (int i = 0; i < w; ++i) {
            const long long a = std::min<long long>(n, (long long)i * per);
            const long long b = std::min<long long>(n, a + per);
            th.emplace_back(worker_rows, dev, i, host_xyz, a, b, d_rows, s, &res[i]);
        }
        for (auto &t : th) t.join();
        for (const auto &r : res)
            if (r.status != FR_OK) {
                set_error("%s", r.msg);
                return r.status;
            }
    }
    k_rows_to_soa64<<<blocks, 256, 0, s>>>(d_rows, n, d_soa);
    FR_CHECK_LAUNCH();
    return FR_OK;
}

// d_out[0:3] coordinate sums, [3:6] minima, [6:9] maxima of (3, n) float64
// planes; d_work holds fr_point_stats64_work_doubles() doubles
extern "C" int fr_point_stats64_work_doubles(void) { return fr::kStatBlocks * 9; }

extern "C" int fr_point_stats64(const double *d_soa, int64_t n, double *d_work, double *d_out,
                                void *stream) {
    using namespace fr;
    if (n < 0 || !d_work || !d_out || (n > 0 && !d_soa)) {
        set_error("fr_point_stats64: invalid arguments");
        return FR_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    k_point_stats64<<<kStatBlocks, kStatThreads, 0, s>>>(d_soa, n, d_work);
    FR_CHECK_LAUNCH();
    k_point_stats64_final<<<1, 144, 0, s>>>(d_work, kStatBlocks, d_out);
    FR_CHECK_LAUNCH();
    return FR_OK;
}
