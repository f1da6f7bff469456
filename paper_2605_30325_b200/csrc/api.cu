// api.cu -- the C ABI of libveda (include/veda.h): argument validation, shape helpers,
// workspace carving and kernel dispatch.  All device work is in permute.cu, score.cu,
// ozaki.cu, topk.cu, attn_fwd.cu (+ attn_fwd_1q.cu), target.cu and search.cu, and the
// host-buffer pipeline in pipeline.cu; nothing here touches data.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <algorithm>
#include <vector>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace veda {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

veda_status fail(veda_status st, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return st;
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

veda_status check_launch(const char *what)
{
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return VEDA_OK;
}

int num_sms()
{
    static std::atomic<int> cache[64];  // per device, zero until first queried
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n == 0) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

veda_status make_tmap_bf16(CUtensorMap *map, const void *base, uint64_t rows, uint64_t cols,
                           uint32_t box_rows)
{
    auto fn = encode_fn();
    if (!fn) return fail(VEDA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides, box,
                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(VEDA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return VEDA_OK;
}

veda_status make_tmap_tile_tokens(CUtensorMap *map, const void *base, int64_t head_stride, int64_t token_stride,
                                  int Hh, int T, int H, int W, int d, int pt, int ph, int pw, int *tok_major,
                                  int box_c, bool swizzle)
{
    auto fn = encode_fn();
    if (!fn) return fail(VEDA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const bool tm = head_stride < token_stride;  // [N][Hh][d]-like: heads inside a token
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], estr[5] = {1, 1, 1, 1, 1};
    const cuuint64_t ts = (cuuint64_t)token_stride * 2, hs = (cuuint64_t)head_stride * 2;
    if (!tm) {  // d, W, H, T, Hh
        dims[0] = d; dims[1] = W; dims[2] = H; dims[3] = T; dims[4] = Hh;
        strides[0] = ts; strides[1] = ts * W; strides[2] = ts * W * H; strides[3] = hs;
        box[0] = box_c; box[1] = pw; box[2] = ph; box[3] = pt; box[4] = 1;
    } else {    // d, Hh, W, H, T
        dims[0] = d; dims[1] = Hh; dims[2] = W; dims[3] = H; dims[4] = T;
        strides[0] = hs; strides[1] = ts; strides[2] = ts * W; strides[3] = ts * W * H;
        box[0] = box_c; box[1] = 1; box[2] = pw; box[3] = ph; box[4] = pt;
    }
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(VEDA_ERR_CUDA, "cuTensorMapEncodeTiled (5-D tile box) failed (%d)", (int)r);
    *tok_major = tm ? 1 : 0;
    return VEDA_OK;
}

veda_status check_arch()
{
    static std::atomic<unsigned long long> ok_devs{0};  // bit d: device d checked and sm_100
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(VEDA_ERR_CUDA, "no CUDA device");
    if (dev >= 0 && dev < 64 && ((ok_devs.load(std::memory_order_relaxed) >> dev) & 1ull)) return VEDA_OK;
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return fail(VEDA_ERR_ARCH, "device %d is sm_%d%d; libveda is built for sm_100a", dev, major, minor);
    if (dev >= 0 && dev < 64) ok_devs.fetch_or(1ull << dev, std::memory_order_relaxed);
    return VEDA_OK;
}

static int lcm_int(int a, int b)
{
    int x = a, y = b;
    while (y) { const int t = x % y; x = y; y = t; }
    return a / x * b;
}

static bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

veda_status shape_of(veda_latent lat, const veda_tile_cfg *cfg, int Hh, Shape *sh, HeadCfgs *hc)
{
    if (!cfg) return fail(VEDA_ERR_NULL, "cfg is NULL");
    if (Hh < 1 || Hh > kMaxHeads) return fail(VEDA_ERR_SHAPE, "Hh=%d outside [1, %d]", Hh, kMaxHeads);
    if (lat.t < 1 || lat.h < 1 || lat.w < 1) return fail(VEDA_ERR_SHAPE, "latent must be positive");
    const int B = cfg[0].pt * cfg[0].ph * cfg[0].pw;
    int Pt = 1, Ph = 1, Pw = 1;
    for (int h = 0; h < Hh; ++h) {
        const veda_tile_cfg c = cfg[h];
        if (!is_pow2(c.pt) || !is_pow2(c.ph) || !is_pow2(c.pw))
            return fail(VEDA_ERR_CONFIG, "head %d: tile extents must be powers of two", h);
        if (c.pt * c.ph * c.pw != B) return fail(VEDA_ERR_CONFIG, "head %d: p_t*p_h*p_w != B=%d", h, B);
        Pt = lcm_int(Pt, c.pt);
        Ph = lcm_int(Ph, c.ph);
        Pw = lcm_int(Pw, c.pw);
        if (hc) { hc->pt[h] = (uint8_t)c.pt; hc->ph[h] = (uint8_t)c.ph; hc->pw[h] = (uint8_t)c.pw; }
    }
    if (B != 64 && B != 128) return fail(VEDA_ERR_CONFIG, "B=%d unsupported (64 or 128)", B);
    sh->Tp = (lat.t + Pt - 1) / Pt * Pt;
    sh->Hp = (lat.h + Ph - 1) / Ph * Ph;
    sh->Wp = (lat.w + Pw - 1) / Pw * Pw;
    sh->B = B;
    const int64_t npad = (int64_t)sh->Tp * sh->Hp * sh->Wp;
    if (npad / B > (1 << 24)) return fail(VEDA_ERR_SHAPE, "too many tiles");
    sh->NT = (int)(npad / B);
    if ((int64_t)Hh * sh->NT * B > INT32_MAX) return fail(VEDA_ERR_SHAPE, "Hh*n_pad exceeds 2^31 rows");
    return VEDA_OK;
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }


namespace {

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace
}  // namespace veda

using namespace veda;

extern "C" {

veda_status veda_tiled_shape_of(veda_latent lat, const veda_tile_cfg *cfg, int32_t Hh, veda_tiled_shape *out)
{
    if (!out) return fail(VEDA_ERR_NULL, "out is NULL");
    Shape sh;
    veda_status st = shape_of(lat, cfg, Hh, &sh, nullptr);
    if (st != VEDA_OK) return st;
    out->tp = sh.Tp; out->hp = sh.Hp; out->wp = sh.Wp; out->B = sh.B; out->n_tiles = sh.NT;
    out->reserved = 0;
    out->n_pad = (int64_t)sh.Tp * sh.Hp * sh.Wp;
    return VEDA_OK;
}

int32_t veda_k_for_sparsity(int32_t n_tiles, double sparsity)
{
    double kk = std::floor((1.0 - sparsity) * (double)n_tiles + 0.5);
    if (kk < 1) kk = 1;
    if (kk > n_tiles) kk = n_tiles;
    return (int32_t)kk;
}

veda_status veda_tile_score_workspace(int32_t Hh, int32_t n_tiles, int32_t d, const veda_scorer *w, size_t *bytes)
{
    if (!w || !bytes) return fail(VEDA_ERR_NULL, "scorer or bytes is NULL");
    if (w->d_in != 3 * d) return fail(VEDA_ERR_SHAPE, "d_in=%d must equal 3*d=%d", w->d_in, 3 * d);
    if (Hh < 1 || n_tiles < 1 || w->d_hidden < 1 || w->d_lat < 1) return fail(VEDA_ERR_SHAPE, "bad sizes");
    // the INT8 Ozaki scorer holds a row of each operand in registers
    if (w->d_in > 1024 || w->d_hidden > 1024 || w->d_lat > 1024)
        return fail(VEDA_ERR_SHAPE, "scorer dimensions (%d, %d, %d): each must be <= 1024", w->d_in, w->d_hidden,
                    w->d_lat);
    const size_t rows = (size_t)Hh * n_tiles;
    size_t b = 0;
    b += 2 * align256(rows * w->d_in * sizeof(float));      // Zq, Zk
    b += align256(rows * w->d_hidden * sizeof(double));     // hidden (reused by q and k)
    b += 2 * align256(rows * w->d_lat * sizeof(double));    // Eq, Ek
    b += ozaki_workspace(Hh, n_tiles, w->d_in, w->d_hidden, w->d_lat);  // int8 slices + row exponents
    *bytes = b;
    return VEDA_OK;
}

static veda_status tile_permute_impl(const uint16_t *x, int64_t head_stride, int64_t token_stride, veda_latent lat,
                                     const veda_tile_cfg *cfg, int32_t Hh, int32_t d, uint16_t *x_tiled,
                                     int32_t *tile_count, uint32_t *slot_mask, float *z, void *stream)
{
    if (!x || !x_tiled) return fail(VEDA_ERR_NULL, "tile_permute: NULL tensor");
    if (d != 64 && d != 128) return fail(VEDA_ERR_SHAPE, "tile_permute: d=%d unsupported", d);
    if (!aligned16(x) || !aligned16(x_tiled) || (head_stride % 8) || (token_stride % 8))
        return fail(VEDA_ERR_ALIGN, "tile_permute: pointers/strides must be 16-byte aligned");
    Shape sh;
    HeadCfgs hc;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &hc);  // argument errors before any device call
    if (st != VEDA_OK) return st;
    if ((st = check_arch()) != VEDA_OK) return st;
    return launch_tile_permute(x, head_stride, token_stride, hc, Hh, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h, lat.w,
                               sh.B, sh.NT, d, x_tiled, tile_count, slot_mask, z, S(stream));
}

veda_status veda_tile_permute(const uint16_t *x, int64_t head_stride, int64_t token_stride, veda_latent lat,
                              const veda_tile_cfg *cfg, int32_t Hh, int32_t d, uint16_t *x_tiled,
                              int32_t *tile_count, uint32_t *slot_mask, void *stream)
{
    return tile_permute_impl(x, head_stride, token_stride, lat, cfg, Hh, d, x_tiled, tile_count, slot_mask, nullptr,
                             stream);
}

veda_status veda_tile_permute_pool(const uint16_t *x, int64_t head_stride, int64_t token_stride, veda_latent lat,
                                   const veda_tile_cfg *cfg, int32_t Hh, int32_t d, uint16_t *x_tiled,
                                   int32_t *tile_count, uint32_t *slot_mask, float *z, void *stream)
{
    if (!z) return fail(VEDA_ERR_NULL, "tile_permute_pool: z is NULL");
    return tile_permute_impl(x, head_stride, token_stride, lat, cfg, Hh, d, x_tiled, tile_count, slot_mask, z, stream);
}

veda_status veda_tile_unpermute(const uint16_t *o_tiled, veda_latent lat, const veda_tile_cfg *cfg, int32_t Hh,
                                int32_t d, uint16_t *o, int64_t head_stride, int64_t token_stride, void *stream)
{
    if (!o || !o_tiled) return fail(VEDA_ERR_NULL, "tile_unpermute: NULL tensor");
    if (d != 64 && d != 128) return fail(VEDA_ERR_SHAPE, "tile_unpermute: d=%d unsupported", d);
    if (!aligned16(o) || !aligned16(o_tiled) || (head_stride % 8) || (token_stride % 8))
        return fail(VEDA_ERR_ALIGN, "tile_unpermute: pointers/strides must be 16-byte aligned");
    Shape sh;
    HeadCfgs hc;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &hc);  // argument errors before any device call
    if (st != VEDA_OK) return st;
    if ((st = check_arch()) != VEDA_OK) return st;
    return launch_tile_unpermute(o_tiled, hc, Hh, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h, lat.w, sh.B, sh.NT, d, o,
                                 head_stride, token_stride, S(stream));
}

veda_status veda_trippool(const uint16_t *x_tiled, const uint32_t *slot_mask, int32_t Hh, int32_t n_tiles,
                          int32_t B, int32_t d, float *z, void *stream)
{
    if (!x_tiled || !slot_mask || !z) return fail(VEDA_ERR_NULL, "trippool: NULL pointer");
    if ((B != 64 && B != 128) || (d != 64 && d != 128) || Hh < 1 || n_tiles < 1)
        return fail(VEDA_ERR_SHAPE, "trippool: unsupported B=%d d=%d", B, d);
    if (!aligned16(x_tiled)) return fail(VEDA_ERR_ALIGN, "trippool: x_tiled not 16-byte aligned");
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    return launch_trippool(x_tiled, slot_mask, Hh, n_tiles, B, d, z, S(stream));
}

veda_status veda_project(const float *z, int32_t Hh, int32_t n_tiles, int32_t d_in, int32_t d_hidden,
                         int32_t d_lat, const float *w1, const float *b1, const float *w2, const float *b2,
                         double *hidden, double *e, void *stream)
{
    if (!z || !w1 || !b1 || !w2 || !b2 || !hidden || !e) return fail(VEDA_ERR_NULL, "project: NULL pointer");
    if (Hh < 1 || n_tiles < 1 || d_in < 1 || d_hidden < 1 || d_lat < 1) return fail(VEDA_ERR_SHAPE, "project: bad sizes");
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    return launch_project(z, Hh, n_tiles, d_in, d_hidden, d_lat, w1, b1, w2, b2, hidden, e, S(stream));
}

veda_status veda_pair_scores(const double *eq, const double *ek, const int32_t *tile_count, int32_t Hh,
                             int32_t n_tiles, int32_t d_lat, float *scores, void *stream)
{
    if (!eq || !ek || !tile_count || !scores) return fail(VEDA_ERR_NULL, "pair_scores: NULL pointer");
    if (Hh < 1 || n_tiles < 1 || d_lat < 1) return fail(VEDA_ERR_SHAPE, "pair_scores: bad sizes");
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    return launch_pair_scores(eq, ek, tile_count, Hh, n_tiles, d_lat, scores, S(stream));
}

veda_status veda_scorer_prepare_bytes(int32_t Hh, int32_t d, const veda_scorer *w, size_t *bytes)
{
    if (!w || !bytes) return fail(VEDA_ERR_NULL, "scorer_prepare_bytes: NULL pointer");
    size_t unused = 0;
    veda_status st = veda_tile_score_workspace(Hh, 1, d, w, &unused);  // the scorer's shape checks
    if (st != VEDA_OK) return st;
    *bytes = ozaki_prepared_bytes(Hh, w->d_in, w->d_hidden, w->d_lat);
    return VEDA_OK;
}

veda_status veda_scorer_prepare(int32_t Hh, int32_t d, const veda_scorer *w, void *prepared, size_t bytes,
                                void *stream)
{
    if (!w || !prepared) return fail(VEDA_ERR_NULL, "scorer_prepare: NULL pointer");
    if (!w->w1q || !w->b1q || !w->w2q || !w->b2q || !w->w1k || !w->b1k || !w->w2k || !w->b2k)
        return fail(VEDA_ERR_NULL, "scorer_prepare: NULL scorer weight");
    size_t need = 0;
    veda_status st = veda_scorer_prepare_bytes(Hh, d, w, &need);
    if (st != VEDA_OK) return st;
    if (bytes < need) return fail(VEDA_ERR_WORKSPACE, "scorer_prepare: buffer %zu < %zu", bytes, need);
    if (!aligned16(prepared)) return fail(VEDA_ERR_ALIGN, "scorer_prepare: buffer not aligned");
    if ((st = check_arch()) != VEDA_OK) return st;
    const float *wq[4] = {w->w1q, w->b1q, w->w2q, w->b2q}, *wk[4] = {w->w1k, w->b1k, w->w2k, w->b2k};
    return launch_ozaki_prepare(wq, wk, Hh, w->d_in, w->d_hidden, w->d_lat, prepared, S(stream));
}

veda_status veda_tile_score(const uint16_t *q_tiled, const uint16_t *k_tiled, const int32_t *tile_count,
                            const uint32_t *slot_mask, int32_t Hh, int32_t n_tiles, int32_t B, int32_t d,
                            const veda_scorer *w, float *scores, void *workspace, size_t workspace_bytes,
                            void *stream)
{
    if (!q_tiled || !k_tiled || !tile_count || !slot_mask || !w || !scores || !workspace)
        return fail(VEDA_ERR_NULL, "tile_score: NULL pointer");
    if (!w->w1q || !w->b1q || !w->w2q || !w->b2q || !w->w1k || !w->b1k || !w->w2k || !w->b2k)
        return fail(VEDA_ERR_NULL, "tile_score: NULL scorer weight");
    size_t need = 0;
    veda_status st = veda_tile_score_workspace(Hh, n_tiles, d, w, &need);
    if (st != VEDA_OK) return st;
    if (workspace_bytes < need) return fail(VEDA_ERR_WORKSPACE, "tile_score: workspace %zu < %zu", workspace_bytes, need);
    if (!aligned16(workspace)) return fail(VEDA_ERR_ALIGN, "tile_score: workspace not aligned");
    const size_t rows = (size_t)Hh * n_tiles;
    char *p = static_cast<char *>(workspace);
    float *zq = reinterpret_cast<float *>(p); p += align256(rows * w->d_in * sizeof(float));
    float *zk = reinterpret_cast<float *>(p); p += align256(rows * w->d_in * sizeof(float));
    double *hid = reinterpret_cast<double *>(p); p += align256(rows * w->d_hidden * sizeof(double));
    double *eq = reinterpret_cast<double *>(p); p += align256(rows * w->d_lat * sizeof(double));
    double *ek = reinterpret_cast<double *>(p);
    if ((st = veda_trippool(q_tiled, slot_mask, Hh, n_tiles, B, d, zq, stream)) != VEDA_OK) return st;
    if ((st = veda_trippool(k_tiled, slot_mask, Hh, n_tiles, B, d, zk, stream)) != VEDA_OK) return st;
    const float *wq[4] = {w->w1q, w->b1q, w->w2q, w->b2q}, *wk[4] = {w->w1k, w->b1k, w->w2k, w->b2k};
    return launch_ozaki_score(zq, zk, tile_count, Hh, n_tiles, w->d_in, w->d_hidden, w->d_lat, wq, wk, w->prepared, hid, eq, ek,
                              scores, reinterpret_cast<char *>(ek) + align256(rows * w->d_lat * sizeof(double)),
                              S(stream));
}

veda_status veda_tile_score_pooled(const float *zq, const float *zk, const int32_t *tile_count, int32_t Hh,
                                   int32_t n_tiles, int32_t d, const veda_scorer *w, float *scores, void *workspace,
                                   size_t workspace_bytes, void *stream)
{
    if (!zq || !zk || !tile_count || !w || !scores || !workspace)
        return fail(VEDA_ERR_NULL, "tile_score_pooled: NULL pointer");
    if (!w->w1q || !w->b1q || !w->w2q || !w->b2q || !w->w1k || !w->b1k || !w->w2k || !w->b2k)
        return fail(VEDA_ERR_NULL, "tile_score_pooled: NULL scorer weight");
    size_t need = 0;
    veda_status st = veda_tile_score_workspace(Hh, n_tiles, d, w, &need);
    if (st != VEDA_OK) return st;
    if (workspace_bytes < need) return fail(VEDA_ERR_WORKSPACE, "tile_score_pooled: workspace %zu < %zu", workspace_bytes, need);
    if (!aligned16(workspace)) return fail(VEDA_ERR_ALIGN, "tile_score_pooled: workspace not aligned");
    const size_t rows = (size_t)Hh * n_tiles;
    char *p = static_cast<char *>(workspace);
    p += 2 * align256(rows * w->d_in * sizeof(float));  // Zq/Zk region unused here
    double *hid = reinterpret_cast<double *>(p); p += align256(rows * w->d_hidden * sizeof(double));
    double *eq = reinterpret_cast<double *>(p); p += align256(rows * w->d_lat * sizeof(double));
    double *ek = reinterpret_cast<double *>(p);
    const float *wq[4] = {w->w1q, w->b1q, w->w2q, w->b2q}, *wk[4] = {w->w1k, w->b1k, w->w2k, w->b2k};
    return launch_ozaki_score(zq, zk, tile_count, Hh, n_tiles, w->d_in, w->d_hidden, w->d_lat, wq, wk, w->prepared, hid, eq, ek,
                              scores, reinterpret_cast<char *>(ek) + align256(rows * w->d_lat * sizeof(double)),
                              S(stream));
}

// Steps 2 (phi, S_pred) + 3 (top-k) without a [Hh][N_T][N_T] score tensor: phi_q / phi_k
// and the digit images of e_q / e_k for all heads, then per chunk of heads the score GEMM
// into a [chunk][N_T][N_T] scratch that the top-k reads back.  Default chunk: as many heads
// as fit 128 MB of fp32 scores (8 of Waver's 24), double-buffered (236 MB instead of 354 MB),
// the top-k of chunk c on a side stream beside the score GEMM of chunk c+1
// (tools/select_bench.py at Waver: 8-head chunks 1.41 ms, 3-head chunks 1.54-1.63, one chunk
// = the two-call form with the full S 1.34-1.43: fewer, larger chunks waste less in the
// persistent GEMM's last wave and in the chunk hand-offs).
static int select_chunk_heads(int Hh, int NT, int heads_per_chunk)
{
    if (heads_per_chunk > 0) return std::min(heads_per_chunk, Hh);
    const size_t per_head = (size_t)NT * NT * sizeof(float);
    const size_t budget = (size_t)128 << 20;
    return (int)std::max<size_t>(1, std::min<size_t>((size_t)Hh, budget / per_head));
}

// score scratch buffers: one chunk, or two (double-buffered between the score GEMM on the
// caller's stream and the top-k on a side stream) when the call has several chunks
static int select_buffers(int Hh, int hc) { return Hh > hc ? 2 : 1; }

veda_status veda_tile_select_workspace(int32_t Hh, int32_t n_tiles, int32_t d, const veda_scorer *w,
                                       int32_t heads_per_chunk, size_t *bytes)
{
    size_t b = 0;
    veda_status st = veda_tile_score_workspace(Hh, n_tiles, d, w, &b);
    if (st != VEDA_OK) return st;
    if (heads_per_chunk < 0) return fail(VEDA_ERR_SHAPE, "tile_select_workspace: heads_per_chunk=%d < 0", heads_per_chunk);
    const int hc = select_chunk_heads(Hh, n_tiles, heads_per_chunk);
    *bytes = b + select_buffers(Hh, hc) * align256((size_t)hc * n_tiles * n_tiles * sizeof(float));
    return VEDA_OK;
}

// per-device side stream of veda_tile_select_pooled (the top-k of chunk c runs on it while
// the score GEMM of chunk c+1 runs on the caller's stream)
static veda_status select_side_stream(cudaStream_t *out)
{
    static std::mutex mu;
    static cudaStream_t cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail(VEDA_ERR_CUDA, "no CUDA device");
    std::lock_guard<std::mutex> lock(mu);
    if (!cache[dev] && cudaStreamCreateWithFlags(&cache[dev], cudaStreamNonBlocking) != cudaSuccess)
        return fail(VEDA_ERR_CUDA, "tile_select_pooled: stream creation failed");
    *out = cache[dev];
    return VEDA_OK;
}

veda_status veda_tile_select_pooled(const float *zq, const float *zk, const int32_t *tile_count, int32_t Hh,
                                    int32_t n_tiles, int32_t d, const veda_scorer *w, int32_t k,
                                    int32_t heads_per_chunk, int32_t *idx, void *workspace, size_t workspace_bytes,
                                    void *stream)
{
    if (!zq || !zk || !tile_count || !w || !idx || !workspace)
        return fail(VEDA_ERR_NULL, "tile_select_pooled: NULL pointer");
    if (!w->w1q || !w->b1q || !w->w2q || !w->b2q || !w->w1k || !w->b1k || !w->w2k || !w->b2k)
        return fail(VEDA_ERR_NULL, "tile_select_pooled: NULL scorer weight");
    size_t need = 0, score_ws = 0;
    veda_status st = veda_tile_select_workspace(Hh, n_tiles, d, w, heads_per_chunk, &need);
    if (st != VEDA_OK) return st;
    if (k < 1 || k > n_tiles) return fail(VEDA_ERR_K_RANGE, "tile_select_pooled: k=%d outside [1, %d]", k, n_tiles);
    if (workspace_bytes < need)
        return fail(VEDA_ERR_WORKSPACE, "tile_select_pooled: workspace %zu < %zu", workspace_bytes, need);
    if (!aligned16(workspace)) return fail(VEDA_ERR_ALIGN, "tile_select_pooled: workspace not aligned");
    if ((st = check_arch()) != VEDA_OK) return st;
    if (debug_mode() && (st = debug_validate(S(stream), [&](uint32_t *f) {
                             veda_status e = launch_validate_finite_f32(zq, (int64_t)Hh * n_tiles * w->d_in, f, S(stream));
                             if (e == VEDA_OK) e = launch_validate_finite_f32(zk, (int64_t)Hh * n_tiles * w->d_in, f, S(stream));
                             return e;
                         })) != VEDA_OK)
        return st;
    veda_tile_score_workspace(Hh, n_tiles, d, w, &score_ws);
    const size_t rows = (size_t)Hh * n_tiles;
    char *p = static_cast<char *>(workspace);
    p += 2 * align256(rows * w->d_in * sizeof(float));  // Zq/Zk region unused here
    double *hid = reinterpret_cast<double *>(p); p += align256(rows * w->d_hidden * sizeof(double));
    double *eq = reinterpret_cast<double *>(p); p += align256(rows * w->d_lat * sizeof(double));
    double *ek = reinterpret_cast<double *>(p); p += align256(rows * w->d_lat * sizeof(double));
    void *oz_scratch = p;
    const float *wq[4] = {w->w1q, w->b1q, w->w2q, w->b2q}, *wk[4] = {w->w1k, w->b1k, w->w2k, w->b2k};
    if ((st = launch_ozaki_phi(zq, zk, Hh, n_tiles, w->d_in, w->d_hidden, w->d_lat, wq, wk, w->prepared, hid, eq, ek, oz_scratch,
                               S(stream))) != VEDA_OK)
        return st;
    if ((st = launch_ozaki_split_e(eq, ek, Hh, n_tiles, w->d_in, w->d_hidden, w->d_lat, oz_scratch, S(stream))) !=
        VEDA_OK)
        return st;
    const int hc = select_chunk_heads(Hh, n_tiles, heads_per_chunk);
    const int nbuf = select_buffers(Hh, hc);
    const size_t buf_bytes = align256((size_t)hc * n_tiles * n_tiles * sizeof(float));
    cudaStream_t ms = S(stream), side = ms;
    if (nbuf == 2 && (st = select_side_stream(&side)) != VEDA_OK) return st;
    std::vector<cudaEvent_t> ev;  // per chunk: scores written (main) / top-k done (side)
    auto event = [&]() -> cudaEvent_t {
        cudaEvent_t e = nullptr;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        ev.push_back(e);
        return e;
    };
    cudaEvent_t last_topk = nullptr;
    auto finish = [&](veda_status r) {
        // the caller's stream resumes only after the last top-k (the side stream is in order);
        // also on an error, so no side-stream work outlives the call unseen
        if (side != ms && last_topk) cudaStreamWaitEvent(ms, last_topk, 0);
        for (cudaEvent_t e : ev) cudaEventDestroy(e);  // released once the device passes them
        return r;
    };
    std::vector<cudaEvent_t> topk_done;
    int c = 0;
    for (int h0 = 0; h0 < Hh; h0 += hc, ++c) {
        const int hn = std::min(hc, Hh - h0);
        float *s_chunk = reinterpret_cast<float *>(static_cast<char *>(workspace) + score_ws + (c % nbuf) * buf_bytes);
        if (c >= nbuf && side != ms) cudaStreamWaitEvent(ms, topk_done[c - nbuf], 0);  // buffer read by top-k c-2
        if ((st = launch_ozaki_score_gemm(tile_count, Hh, h0, hn, n_tiles, w->d_in, w->d_hidden, w->d_lat, s_chunk,
                                          oz_scratch, ms)) != VEDA_OK)
            return finish(st);
        if (debug_mode() && (st = debug_validate(ms, [&](uint32_t *f) {
                                 return launch_validate_scores(s_chunk, (int64_t)hn * n_tiles * n_tiles, f, ms);
                             })) != VEDA_OK)
            return finish(st);
        if (side != ms) {
            cudaEvent_t g = event();
            if (!g || cudaEventRecord(g, ms) != cudaSuccess || cudaStreamWaitEvent(side, g, 0) != cudaSuccess)
                return finish(fail(VEDA_ERR_CUDA, "tile_select_pooled: event record/wait failed"));
        }
        if ((st = launch_topk(s_chunk, hn, n_tiles, k, idx + (size_t)h0 * n_tiles * k, side)) != VEDA_OK)
            return finish(st);
        if (side != ms) {
            cudaEvent_t t = event();
            if (!t || cudaEventRecord(t, side) != cudaSuccess)
                return finish(fail(VEDA_ERR_CUDA, "tile_select_pooled: event record failed"));
            topk_done.push_back(t);
            last_topk = t;
        }
    }
    return finish(VEDA_OK);
}

veda_status veda_select_topk(const float *scores, int32_t Hh, int32_t n_tiles, int32_t k, int32_t *idx, void *stream)
{
    if (!scores || !idx) return fail(VEDA_ERR_NULL, "select_topk: NULL pointer");
    if (Hh < 1 || n_tiles < 1) return fail(VEDA_ERR_SHAPE, "select_topk: bad sizes");
    if (k < 1 || k > n_tiles) return fail(VEDA_ERR_K_RANGE, "select_topk: k=%d outside [1, %d]", k, n_tiles);
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    if (debug_mode() && (st = debug_validate(S(stream), [&](uint32_t *f) {
                             return launch_validate_scores(scores, (int64_t)Hh * n_tiles * n_tiles, f, S(stream));
                         })) != VEDA_OK)
        return st;
    return launch_topk(scores, Hh, n_tiles, k, idx, S(stream));
}

veda_status veda_sparse_attn_fwd(const uint16_t *q_tiled, const uint16_t *k_tiled, const uint16_t *v_tiled,
                                 const int32_t *idx, const uint32_t *slot_mask, int32_t Hh, int32_t n_tiles,
                                 int32_t B, int32_t d, int32_t k, float softmax_scale, uint16_t *o_tiled,
                                 float *lse, void *stream)
{
    if (!q_tiled || !k_tiled || !v_tiled || !idx || !slot_mask || !o_tiled)
        return fail(VEDA_ERR_NULL, "sparse_attn_fwd: NULL pointer");
    if (Hh < 1 || n_tiles < 1 || (int64_t)Hh * n_tiles * B > INT32_MAX)
        return fail(VEDA_ERR_SHAPE, "sparse_attn_fwd: bad sizes");
    if (k < 1 || k > n_tiles) return fail(VEDA_ERR_K_RANGE, "sparse_attn_fwd: k=%d outside [1, %d]", k, n_tiles);
    if (!aligned16(q_tiled) || !aligned16(k_tiled) || !aligned16(v_tiled) || !aligned16(o_tiled))
        return fail(VEDA_ERR_ALIGN, "sparse_attn_fwd: tensors must be 16-byte aligned");
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    if (debug_mode()) {
        const int64_t n = (int64_t)n_tiles * B;
        st = debug_validate(S(stream), [&](uint32_t *f) {
            veda_status e = launch_validate_index(idx, (int64_t)Hh * n_tiles, n_tiles, k, f, S(stream));
            if (e == VEDA_OK) e = launch_validate_finite(q_tiled, n * d, d, Hh, n, d, f, S(stream));
            if (e == VEDA_OK) e = launch_validate_finite(k_tiled, n * d, d, Hh, n, d, f, S(stream));
            if (e == VEDA_OK) e = launch_validate_finite(v_tiled, n * d, d, Hh, n, d, f, S(stream));
            return e;
        });
        if (st != VEDA_OK) return st;
    }
    const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt((float)d);
    return launch_sparse_attn(q_tiled, k_tiled, v_tiled, idx, slot_mask, Hh, n_tiles, B, d, k, scale, o_tiled, lse,
                              S(stream));
}

veda_status veda_tile_pool(const uint16_t *x, int64_t head_stride, int64_t token_stride, veda_latent lat,
                           const veda_tile_cfg *cfg, int32_t Hh, int32_t d, float *z, int32_t *tile_count,
                           uint32_t *slot_mask, void *stream)
{
    if (!x || !z) return fail(VEDA_ERR_NULL, "tile_pool: NULL pointer");
    if (d != 64 && d != 128) return fail(VEDA_ERR_SHAPE, "tile_pool: d=%d unsupported", d);
    if (!aligned16(x) || (head_stride % 8) || (token_stride % 8))
        return fail(VEDA_ERR_ALIGN, "tile_pool: pointer/strides must be 16-byte aligned");
    Shape sh;
    HeadCfgs hc;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &hc);  // argument errors before any device call
    if (st != VEDA_OK) return st;
    if ((st = check_arch()) != VEDA_OK) return st;
    if (debug_mode() && (st = debug_validate(S(stream), [&](uint32_t *f) {
                             return launch_validate_finite(x, head_stride, token_stride, Hh,
                                                           (int64_t)lat.t * lat.h * lat.w, d, f, S(stream));
                         })) != VEDA_OK)
        return st;
    return launch_tile_pool_tokens(x, head_stride, token_stride, hc, Hh, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h, lat.w, sh.B,
                                   sh.NT, d, z, tile_count, slot_mask, S(stream));
}

veda_status veda_tile_pool_qk(const uint16_t *q, const uint16_t *k, int64_t head_stride, int64_t token_stride,
                              veda_latent lat, const veda_tile_cfg *cfg, int32_t Hh, int32_t d, float *zq, float *zk,
                              int32_t *tile_count, uint32_t *slot_mask, void *stream)
{
    if (!q || !k || !zq || !zk) return fail(VEDA_ERR_NULL, "tile_pool_qk: NULL pointer");
    if (d != 64 && d != 128) return fail(VEDA_ERR_SHAPE, "tile_pool_qk: d=%d unsupported", d);
    if (!aligned16(q) || !aligned16(k) || (head_stride % 8) || (token_stride % 8))
        return fail(VEDA_ERR_ALIGN, "tile_pool_qk: pointers/strides must be 16-byte aligned");
    Shape sh;
    HeadCfgs hc;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &hc);  // argument errors before any device call
    if (st != VEDA_OK) return st;
    if ((st = check_arch()) != VEDA_OK) return st;
    if (debug_mode() && (st = debug_validate(S(stream), [&](uint32_t *f) {
                             const int64_t n = (int64_t)lat.t * lat.h * lat.w;
                             veda_status e = launch_validate_finite(q, head_stride, token_stride, Hh, n, d, f, S(stream));
                             if (e == VEDA_OK) e = launch_validate_finite(k, head_stride, token_stride, Hh, n, d, f, S(stream));
                             return e;
                         })) != VEDA_OK)
        return st;
    return launch_tile_pool_tokens2(q, k, head_stride, token_stride, hc, Hh, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h, lat.w,
                                    sh.B, sh.NT, d, zq, zk, tile_count, slot_mask, S(stream));
}

static veda_status tile_pool_range_impl(const uint16_t *x, int64_t head_stride, int64_t token_stride, veda_latent lat,
                                        const veda_tile_cfg *cfg, int32_t Hh, int32_t d, int32_t head_begin,
                                        int32_t head_end, float *z, int32_t *tile_count, uint32_t *slot_mask,
                                        bool local, void *stream)
{
    const bool empty = head_begin == head_end && head_begin >= 0 && head_end <= Hh;
    if ((!x || !z) && !(local && empty)) return fail(VEDA_ERR_NULL, "tile_pool_heads: NULL pointer");
    if (d != 64 && d != 128) return fail(VEDA_ERR_SHAPE, "tile_pool_heads: d=%d unsupported", d);
    if (!aligned16(x) || (head_stride % 8) || (token_stride % 8))
        return fail(VEDA_ERR_ALIGN, "tile_pool_heads: pointer/strides must be 16-byte aligned");
    Shape sh;
    HeadCfgs hc;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &hc);  // the whole call's padded grid
    (void)empty;
    if (st != VEDA_OK) return st;
    if (head_begin < 0 || head_begin > head_end || head_end > Hh)
        return fail(VEDA_ERR_SHAPE, "tile_pool_heads: [%d, %d) outside [0, %d]", head_begin, head_end, Hh);
    if ((st = check_arch()) != VEDA_OK) return st;
    if (head_begin == head_end) return VEDA_OK;
    // local: x and the outputs hold the range's heads only; else they are the whole call's
    const size_t h0 = local ? 0 : (size_t)head_begin;
    const int hn = head_end - head_begin;
    if (debug_mode() && (st = debug_validate(S(stream), [&](uint32_t *f) {
                             return launch_validate_finite(x + h0 * head_stride, head_stride, token_stride, hn,
                                                           (int64_t)lat.t * lat.h * lat.w, d, f, S(stream));
                         })) != VEDA_OK)
        return st;
    HeadCfgs sub;
    for (int h = 0; h < hn; ++h) {
        sub.pt[h] = hc.pt[head_begin + h];
        sub.ph[h] = hc.ph[head_begin + h];
        sub.pw[h] = hc.pw[head_begin + h];
    }
    return launch_tile_pool_tokens(x + h0 * head_stride, head_stride, token_stride, sub, hn, sh.Tp, sh.Hp, sh.Wp, lat.t,
                                   lat.h, lat.w, sh.B, sh.NT, d, z + h0 * sh.NT * 3 * d,
                                   tile_count ? tile_count + h0 * sh.NT : nullptr,
                                   slot_mask ? slot_mask + h0 * sh.NT * (sh.B / 32) : nullptr, S(stream));
}

veda_status veda_tile_pool_heads(const uint16_t *x, int64_t head_stride, int64_t token_stride, veda_latent lat,
                                 const veda_tile_cfg *cfg, int32_t Hh, int32_t d, int32_t head_begin,
                                 int32_t head_end, float *z, int32_t *tile_count, uint32_t *slot_mask, void *stream)
{
    return tile_pool_range_impl(x, head_stride, token_stride, lat, cfg, Hh, d, head_begin, head_end, z, tile_count,
                                slot_mask, false, stream);
}

veda_status veda_tile_pool_local(const uint16_t *x, int64_t head_stride, int64_t token_stride, veda_latent lat,
                                 const veda_tile_cfg *cfg, int32_t Hh, int32_t d, int32_t head_begin,
                                 int32_t head_end, float *z, int32_t *tile_count, uint32_t *slot_mask, void *stream)
{
    return tile_pool_range_impl(x, head_stride, token_stride, lat, cfg, Hh, d, head_begin, head_end, z, tile_count,
                                slot_mask, true, stream);
}

static veda_status sparse_attn_fwd_tokens_impl(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                               int64_t head_stride, int64_t token_stride, veda_latent lat,
                                               const veda_tile_cfg *cfg, int32_t Hh, int32_t d, const int32_t *idx,
                                               const uint32_t *slot_mask, int32_t k_keep, float softmax_scale,
                                               uint16_t *o, int64_t o_head_stride, int64_t o_token_stride, float *lse,
                                               bool all_units, int32_t unit_begin, int32_t unit_end, void *stream)
{
    if (!q || !k || !v || !idx || !slot_mask || !o) return fail(VEDA_ERR_NULL, "sparse_attn_fwd_tokens: NULL pointer");
    if (d != 64 && d != 128) return fail(VEDA_ERR_SHAPE, "sparse_attn_fwd_tokens: d=%d unsupported", d);
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || (head_stride % 8) || (token_stride % 8) ||
        (o_head_stride % 8) || (o_token_stride % 8))
        return fail(VEDA_ERR_ALIGN, "sparse_attn_fwd_tokens: pointers/strides must be 16-byte aligned");
    Shape sh;
    HeadCfgs hc;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &hc);  // argument errors before any device call
    if (st != VEDA_OK) return st;
    if (k_keep < 1 || k_keep > sh.NT)
        return fail(VEDA_ERR_K_RANGE, "sparse_attn_fwd_tokens: k=%d outside [1, %d]", k_keep, sh.NT);
    const int32_t n_units = Hh * sh.NT;
    if (all_units) {
        unit_begin = 0;
        unit_end = n_units;
    } else if (unit_begin < 0 || unit_begin > unit_end || unit_end > n_units) {
        return fail(VEDA_ERR_SHAPE, "sparse_attn_fwd_tokens_units: [%d, %d) outside [0, %d]", unit_begin, unit_end,
                    n_units);
    }
    if ((st = check_arch()) != VEDA_OK) return st;
    if (unit_begin == unit_end) return VEDA_OK;  // an empty share (e.g. a rank without units)
    if (debug_mode()) {
        const int64_t n = (int64_t)lat.t * lat.h * lat.w;
        st = debug_validate(S(stream), [&](uint32_t *f) {
            veda_status e = launch_validate_index(idx, (int64_t)n_units, sh.NT, k_keep, f, S(stream));
            if (e == VEDA_OK) e = launch_validate_finite(q, head_stride, token_stride, Hh, n, d, f, S(stream));
            if (e == VEDA_OK) e = launch_validate_finite(k, head_stride, token_stride, Hh, n, d, f, S(stream));
            if (e == VEDA_OK) e = launch_validate_finite(v, head_stride, token_stride, Hh, n, d, f, S(stream));
            return e;
        });
        if (st != VEDA_OK) return st;
    }
    const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt((float)d);
    return launch_sparse_attn_tok(q, k, v, head_stride, token_stride, hc, Hh, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h, lat.w,
                                  sh.B, sh.NT, d, idx, slot_mask, k_keep, scale, o, o_head_stride, o_token_stride, lse,
                                  unit_begin, unit_end, S(stream));
}

veda_status veda_sparse_attn_fwd_tokens(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t head_stride,
                                        int64_t token_stride, veda_latent lat, const veda_tile_cfg *cfg, int32_t Hh,
                                        int32_t d, const int32_t *idx, const uint32_t *slot_mask, int32_t k_keep,
                                        float softmax_scale, uint16_t *o, int64_t o_head_stride,
                                        int64_t o_token_stride, float *lse, void *stream)
{
    return sparse_attn_fwd_tokens_impl(q, k, v, head_stride, token_stride, lat, cfg, Hh, d, idx, slot_mask, k_keep,
                                       softmax_scale, o, o_head_stride, o_token_stride, lse, true, 0, 0, stream);
}

veda_status veda_sparse_attn_fwd_tokens_units(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                              int64_t head_stride, int64_t token_stride, veda_latent lat,
                                              const veda_tile_cfg *cfg, int32_t Hh, int32_t d, const int32_t *idx,
                                              const uint32_t *slot_mask, int32_t k_keep, float softmax_scale,
                                              uint16_t *o, int64_t o_head_stride, int64_t o_token_stride, float *lse,
                                              int32_t unit_begin, int32_t unit_end, void *stream)
{
    return sparse_attn_fwd_tokens_impl(q, k, v, head_stride, token_stride, lat, cfg, Hh, d, idx, slot_mask, k_keep,
                                       softmax_scale, o, o_head_stride, o_token_stride, lse, false, unit_begin,
                                       unit_end, stream);
}

veda_status veda_sparse_attn_fwd_tokens_local(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                                              int64_t head_stride, int64_t token_stride, veda_latent lat,
                                              const veda_tile_cfg *cfg, int32_t Hh, int32_t d, int32_t head_begin,
                                              int32_t head_end, const int32_t *idx, const uint32_t *slot_mask,
                                              int32_t k_keep, float softmax_scale, uint16_t *o, int64_t o_head_stride,
                                              int64_t o_token_stride, float *lse, void *stream)
{
    const bool empty = head_begin == head_end && head_begin >= 0 && head_end <= Hh;
    if ((!q || !k || !v || !idx || !slot_mask || !o) && !empty)
        return fail(VEDA_ERR_NULL, "sparse_attn_fwd_tokens_local: NULL pointer");
    if (d != 64 && d != 128) return fail(VEDA_ERR_SHAPE, "sparse_attn_fwd_tokens_local: d=%d unsupported", d);
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || (head_stride % 8) || (token_stride % 8) ||
        (o_head_stride % 8) || (o_token_stride % 8))
        return fail(VEDA_ERR_ALIGN, "sparse_attn_fwd_tokens_local: pointers/strides must be 16-byte aligned");
    Shape sh;
    HeadCfgs hc;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &hc);  // the whole call's padded grid
    if (st != VEDA_OK) return st;
    if (head_begin < 0 || head_begin > head_end || head_end > Hh)
        return fail(VEDA_ERR_SHAPE, "sparse_attn_fwd_tokens_local: [%d, %d) outside [0, %d]", head_begin, head_end, Hh);
    if (k_keep < 1 || k_keep > sh.NT)
        return fail(VEDA_ERR_K_RANGE, "sparse_attn_fwd_tokens_local: k=%d outside [1, %d]", k_keep, sh.NT);
    if ((st = check_arch()) != VEDA_OK) return st;
    const int hn = head_end - head_begin;
    if (hn == 0) return VEDA_OK;
    if (debug_mode()) {
        const int64_t n = (int64_t)lat.t * lat.h * lat.w;
        st = debug_validate(S(stream), [&](uint32_t *f) {
            veda_status e = launch_validate_index(idx, (int64_t)hn * sh.NT, sh.NT, k_keep, f, S(stream));
            if (e == VEDA_OK) e = launch_validate_finite(q, head_stride, token_stride, hn, n, d, f, S(stream));
            if (e == VEDA_OK) e = launch_validate_finite(k, head_stride, token_stride, hn, n, d, f, S(stream));
            if (e == VEDA_OK) e = launch_validate_finite(v, head_stride, token_stride, hn, n, d, f, S(stream));
            return e;
        });
        if (st != VEDA_OK) return st;
    }
    HeadCfgs sub;
    for (int h = 0; h < hn; ++h) {
        sub.pt[h] = hc.pt[head_begin + h];
        sub.ph[h] = hc.ph[head_begin + h];
        sub.pw[h] = hc.pw[head_begin + h];
    }
    const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt((float)d);
    return launch_sparse_attn_tok(q, k, v, head_stride, token_stride, sub, hn, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h, lat.w,
                                  sh.B, sh.NT, d, idx, slot_mask, k_keep, scale, o, o_head_stride, o_token_stride, lse,
                                  0, hn * sh.NT, S(stream));
}

veda_status veda_target_scores(const uint16_t *q_tiled, const uint16_t *k_tiled, const uint32_t *slot_mask,
                               const float *lse, int32_t Hh, int32_t n_tiles, int32_t B, int32_t d,
                               float softmax_scale, float *s_tgt, void *stream)
{
    if (!q_tiled || !k_tiled || !slot_mask || !lse || !s_tgt) return fail(VEDA_ERR_NULL, "target_scores: NULL pointer");
    if (Hh < 1 || n_tiles < 1 || (int64_t)Hh * n_tiles * B > INT32_MAX)
        return fail(VEDA_ERR_SHAPE, "target_scores: bad sizes");
    if (!aligned16(q_tiled) || !aligned16(k_tiled))
        return fail(VEDA_ERR_ALIGN, "target_scores: tensors must be 16-byte aligned");
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    const float scale = softmax_scale > 0.f ? softmax_scale : 1.0f / std::sqrt((float)d);
    return launch_target_scores(q_tiled, k_tiled, slot_mask, lse, Hh, n_tiles, B, d, scale, s_tgt, S(stream));
}

veda_status veda_tile_recall(const int32_t *idx_sp, const int32_t *idx_fu, const int32_t *tile_count, int64_t rows,
                             int32_t n_tiles, int32_t k, double *recall, void *stream)
{
    if (!idx_sp || !idx_fu || !recall) return fail(VEDA_ERR_NULL, "tile_recall: NULL pointer");
    if (rows < 1 || n_tiles < 1) return fail(VEDA_ERR_SHAPE, "tile_recall: bad sizes");
    if (k < 1 || k > n_tiles) return fail(VEDA_ERR_K_RANGE, "tile_recall: k=%d outside [1, %d]", k, n_tiles);
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    return launch_recall(idx_sp, idx_fu, tile_count, rows, n_tiles, k, recall, S(stream));
}

veda_status veda_tile_permute_scalar(const float *x, int64_t head_stride, veda_latent lat, const veda_tile_cfg *cfg,
                                     int32_t Hh, float pad, float *x_tiled, void *stream)
{
    if (!x || !x_tiled) return fail(VEDA_ERR_NULL, "tile_permute_scalar: NULL tensor");
    Shape sh;
    HeadCfgs hc;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &hc);  // argument errors before any device call
    if (st != VEDA_OK) return st;
    if ((st = check_arch()) != VEDA_OK) return st;
    if (head_stride < (int64_t)lat.t * lat.h * lat.w)
        return fail(VEDA_ERR_SHAPE, "tile_permute_scalar: head_stride < N");
    return launch_permute_scalar(x, head_stride, hc, Hh, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h, lat.w, sh.B, sh.NT, pad,
                                 x_tiled, S(stream));
}

veda_status veda_tile_unpermute_scalar(const float *x_tiled, veda_latent lat, const veda_tile_cfg *cfg, int32_t Hh,
                                       float *x, int64_t head_stride, void *stream)
{
    if (!x || !x_tiled) return fail(VEDA_ERR_NULL, "tile_unpermute_scalar: NULL tensor");
    Shape sh;
    HeadCfgs hc;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &hc);  // argument errors before any device call
    if (st != VEDA_OK) return st;
    if ((st = check_arch()) != VEDA_OK) return st;
    if (head_stride < (int64_t)lat.t * lat.h * lat.w)
        return fail(VEDA_ERR_SHAPE, "tile_unpermute_scalar: head_stride < N");
    return launch_unpermute_scalar(x_tiled, hc, Hh, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h, lat.w, sh.B, sh.NT, x,
                                   head_stride, S(stream));
}

veda_status veda_sq_err(const uint16_t *a, const uint16_t *b, int64_t head_stride, int64_t n, int32_t Hh,
                        double *err, void *stream)
{
    if (!a || !b || !err) return fail(VEDA_ERR_NULL, "sq_err: NULL pointer");
    if (Hh < 1 || n < 0 || Hh > 65535 || head_stride < n) return fail(VEDA_ERR_SHAPE, "sq_err: bad sizes");
    if ((n % 8) || (head_stride % 8) || !aligned16(a) || !aligned16(b))
        return fail(VEDA_ERR_ALIGN, "sq_err: n, head_stride must be multiples of 8, pointers 16-byte aligned");
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    if (n == 0) return VEDA_OK;
    return launch_sq_err(a, b, head_stride, n, Hh, err, S(stream));
}

const char *veda_status_str(veda_status st)
{
    switch (st) {
    case VEDA_OK: return "VEDA_OK";
    case VEDA_ERR_NULL: return "VEDA_ERR_NULL";
    case VEDA_ERR_SHAPE: return "VEDA_ERR_SHAPE";
    case VEDA_ERR_CONFIG: return "VEDA_ERR_CONFIG";
    case VEDA_ERR_K_RANGE: return "VEDA_ERR_K_RANGE";
    case VEDA_ERR_ALIGN: return "VEDA_ERR_ALIGN";
    case VEDA_ERR_WORKSPACE: return "VEDA_ERR_WORKSPACE";
    case VEDA_ERR_INDEX: return "VEDA_ERR_INDEX";
    case VEDA_ERR_NONFINITE: return "VEDA_ERR_NONFINITE";
    case VEDA_ERR_CUDA: return "VEDA_ERR_CUDA";
    case VEDA_ERR_ARCH: return "VEDA_ERR_ARCH";
    }
    return "VEDA_ERR_UNKNOWN";
}

const char *veda_last_error(void) { return g_err; }

uint64_t veda_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

veda_status veda_check_device(void) { return check_arch(); }

veda_status veda_validate_index(const int32_t *idx, int64_t rows, int32_t n_tiles, int32_t k, uint32_t *flags,
                                void *stream)
{
    if (!idx || !flags) return fail(VEDA_ERR_NULL, "validate_index: NULL pointer");
    if (rows < 0 || n_tiles < 1) return fail(VEDA_ERR_SHAPE, "validate_index: bad sizes");
    if (k < 1 || k > n_tiles) return fail(VEDA_ERR_K_RANGE, "validate_index: k=%d outside [1, %d]", k, n_tiles);
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    return launch_validate_index(idx, rows, n_tiles, k, flags, S(stream));
}

veda_status veda_validate_finite(const uint16_t *x, int64_t head_stride, int64_t token_stride, int32_t Hh, int64_t n,
                                 int32_t d, uint32_t *flags, void *stream)
{
    if (!x || !flags) return fail(VEDA_ERR_NULL, "validate_finite: NULL pointer");
    if (Hh < 0 || n < 0 || d < 8 || (d % 8)) return fail(VEDA_ERR_SHAPE, "validate_finite: bad sizes");
    if (!aligned16(x) || (head_stride % 8) || (token_stride % 8))
        return fail(VEDA_ERR_ALIGN, "validate_finite: pointer/strides must be 16-byte aligned");
    veda_status st = check_arch();
    if (st != VEDA_OK) return st;
    return launch_validate_finite(x, head_stride, token_stride, Hh, n, d, flags, S(stream));
}

int32_t veda_set_debug(int32_t on)
{
    const bool prev = debug_mode();
    set_debug_mode(on != 0);
    return prev ? 1 : 0;
}

}  // extern "C"
