// validate.cu -- input validation of the boundary.
//
// The kept-tile lists the attention consumes must be exactly k distinct key tiles per query
// tile in ascending order ("exactly k", reading R11 "ascending key-tile
// index"), each in [0, n_tiles).  These kernels check that contract and the finiteness of
// bf16 inputs / fp32 scores and OR bits into a device flag word:
//   VEDA_FLAG_INDEX_RANGE  an entry outside [0, n_tiles)
//   VEDA_FLAG_INDEX_ORDER  a row that is not strictly ascending (a duplicate or a descent)
//   VEDA_FLAG_NONFINITE    an Inf/NaN bf16 input, or a NaN score
// They run on request (veda_validate_*) and, in debug mode (veda_set_debug(1) or
// VEDA_DEBUG=1 in the environment at library load), inside the path's entry points, which
// then synchronise and return VEDA_ERR_INDEX / VEDA_ERR_NONFINITE.  The default path never
// runs them; the attention kernel clamps every list entry into [0, n_tiles) regardless, so a
// bad list can give wrong outputs but never reads outside the head's tiles or slot masks.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace veda {
namespace {

// one warp per row: entries t and t+1 compared for the order check
__global__ void validate_index_kernel(const int32_t *__restrict__ idx, int64_t rows, int n_tiles, int k,
                                      uint32_t *__restrict__ flags)
{
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int32_t *r = idx + row * k;
    uint32_t f = 0;
    for (int t = lane; t < k; t += 32) {
        const int32_t j = __ldg(r + t);
        if (j < 0 || j >= n_tiles) f |= VEDA_FLAG_INDEX_RANGE;
        if (t + 1 < k && !(j < __ldg(r + t + 1))) f |= VEDA_FLAG_INDEX_ORDER;
    }
    f = __reduce_or_sync(0xFFFFFFFFu, f);
    if (lane == 0 && f) atomicOr(flags, f);
}

// bf16 token tensor x[h][n][c] (strides in elements): exponent bits all ones = Inf or NaN
__global__ void validate_finite_bf16_kernel(const uint16_t *__restrict__ x, int64_t hs, int64_t ts, int Hh,
                                            int64_t n, int d, uint32_t *__restrict__ flags)
{
    const int64_t vecs = (int64_t)Hh * n * (d / 8);
    uint32_t bad = 0;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < vecs; v += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c8 = v % (d / 8), tok = (v / (d / 8)) % n, h = v / ((int64_t)(d / 8) * n);
        const uint4 w = __ldg(reinterpret_cast<const uint4 *>(x + h * hs + tok * ts) + c8);
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e)
            bad |= ((ws[e] & 0x7F80u) == 0x7F80u) | ((ws[e] & 0x7F800000u) == 0x7F800000u);
    }
    if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, VEDA_FLAG_NONFINITE);
}

__global__ void validate_scores_kernel(const float *__restrict__ s, int64_t n, uint32_t *__restrict__ flags)
{
    uint32_t bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad |= isnan(__ldg(s + i)) ? 1u : 0u;
    if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, VEDA_FLAG_NONFINITE);
}

// fp32 inputs (pooled descriptors): NaN or +-inf is flagged
__global__ void validate_finite_f32_kernel(const float *__restrict__ x, int64_t n, uint32_t *__restrict__ flags)
{
    uint32_t bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad |= isfinite(__ldg(x + i)) ? 0u : 1u;
    if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, VEDA_FLAG_NONFINITE);
}

std::atomic<int> g_debug{-1};

// per-device flag word of debug mode (allocated on first use, debug mode only)
uint32_t *debug_flags()
{
    static std::mutex mu;
    static uint32_t *buf[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> g(mu);
    if (!buf[dev] && cudaMalloc(&buf[dev], sizeof(uint32_t)) != cudaSuccess) return nullptr;
    return buf[dev];
}

}  // namespace

veda_status launch_validate_index(const int32_t *idx, int64_t rows, int n_tiles, int k, uint32_t *flags,
                                  cudaStream_t s)
{
    if (rows == 0) return VEDA_OK;
    const int wpb = 8;
    validate_index_kernel<<<(unsigned)((rows + wpb - 1) / wpb), 32 * wpb, 0, s>>>(idx, rows, n_tiles, k, flags);
    count_launch();
    return check_launch("validate_index");
}

veda_status launch_validate_finite(const uint16_t *x, int64_t hs, int64_t ts, int Hh, int64_t n, int d,
                                   uint32_t *flags, cudaStream_t s)
{
    if ((int64_t)Hh * n == 0) return VEDA_OK;
    validate_finite_bf16_kernel<<<4 * num_sms(), 256, 0, s>>>(x, hs, ts, Hh, n, d, flags);
    count_launch();
    return check_launch("validate_finite");
}

veda_status launch_validate_scores(const float *scores, int64_t n, uint32_t *flags, cudaStream_t s)
{
    if (n == 0) return VEDA_OK;
    validate_scores_kernel<<<4 * num_sms(), 256, 0, s>>>(scores, n, flags);
    count_launch();
    return check_launch("validate_scores");
}

veda_status launch_validate_finite_f32(const float *x, int64_t n, uint32_t *flags, cudaStream_t s)
{
    if (n == 0) return VEDA_OK;
    validate_finite_f32_kernel<<<4 * num_sms(), 256, 0, s>>>(x, n, flags);
    count_launch();
    return check_launch("validate_finite_f32");
}

bool debug_mode()
{
    int v = g_debug.load(std::memory_order_relaxed);
    if (v < 0) {
        const char *e = getenv("VEDA_DEBUG");
        v = (e && e[0] && strcmp(e, "0") != 0) ? 1 : 0;
        int expected = -1;
        g_debug.compare_exchange_strong(expected, v);
        v = g_debug.load();
    }
    return v == 1;
}

void set_debug_mode(bool on) { g_debug.store(on ? 1 : 0); }

veda_status debug_validate(cudaStream_t s, const std::function<veda_status(uint32_t *)> &enqueue)
{
    uint32_t *f = debug_flags();
    if (!f) return fail(VEDA_ERR_CUDA, "debug mode: cannot allocate the flag word");
    if (cudaMemsetAsync(f, 0, sizeof(uint32_t), s) != cudaSuccess) return fail(VEDA_ERR_CUDA, "debug mode: memset");
    veda_status st = enqueue(f);
    if (st != VEDA_OK) return st;
    uint32_t h = 0;
    if (cudaMemcpyAsync(&h, f, sizeof(uint32_t), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return fail(VEDA_ERR_CUDA, "debug mode: %s", cudaGetErrorString(cudaGetLastError()));
    if (h & (VEDA_FLAG_INDEX_RANGE | VEDA_FLAG_INDEX_ORDER))
        return fail(VEDA_ERR_INDEX, "index list: %s%s", (h & VEDA_FLAG_INDEX_RANGE) ? "entry outside [0, n_tiles) " : "",
                    (h & VEDA_FLAG_INDEX_ORDER) ? "row not strictly ascending (duplicate or descent)" : "");
    if (h & VEDA_FLAG_NONFINITE) return fail(VEDA_ERR_NONFINITE, "non-finite input (Inf/NaN)");
    return VEDA_OK;
}

}  // namespace veda
