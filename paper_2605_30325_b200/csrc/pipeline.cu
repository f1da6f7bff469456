// pipeline.cu -- the whole path on HOST buffers (veda_sparse_attention_host): the
// end-to-end call of a DiT layer whose Q/K/V live in host memory.
//
// Heads are independent (distinct phi per head; per-head loop of Alg. 2,
// PAPER.md:693-698), so the call is cut into chunks of heads and software-pipelined over
// three streams and two device buffer sets ("slots"):
//
//   h2d stream     : copy Q/K/V of chunk c            (waits: attention of chunk c-2 done)
//   caller stream  : pool Q/K -> score -> top-k -> attention (token layout in and out)
//                                                     (waits: H2D of c, D2H of chunk c-2)
//   d2h stream     : copy O of chunk c back to host   (waits: compute of c)
//
// so the PCIe transfers in both directions overlap the kernels.  The chunk runs the
// token-layout form of the path (veda_tile_pool, veda_tile_score_pooled, veda_select_topk,
// veda_sparse_attn_fwd_tokens): no tiled copies.  Every chunk is tiled on the padded grid
// of the WHOLE call (reading R5), so results are bit-identical to one call over all heads.
// Pure host code: only the existing kernels run.
#include <cuda_runtime.h>

#include <cmath>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace veda {
namespace {

constexpr int kSlots = 2;

struct SideStreams {
    cudaStream_t h2d = nullptr, d2h = nullptr;
};

veda_status side_streams(SideStreams *out)
{
    static std::mutex mu;
    static SideStreams cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail(VEDA_ERR_CUDA, "no CUDA device");
    std::lock_guard<std::mutex> lock(mu);
    SideStreams &s = cache[dev];
    if (!s.h2d) {
        if (cudaStreamCreateWithFlags(&s.h2d, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&s.d2h, cudaStreamNonBlocking) != cudaSuccess)
            return fail(VEDA_ERR_CUDA, "sparse_attention_host: stream creation failed");
    }
    *out = s;
    return VEDA_OK;
}

int chunk_heads(int Hh, int heads_per_chunk)
{
    if (heads_per_chunk > 0) return heads_per_chunk < Hh ? heads_per_chunk : Hh;
    // default: up to 32 chunks -- the call is PCIe-bound, so the pipeline fill (first H2D)
    // and drain (last chunk's path + D2H) are what chunking can shrink; measured at Waver
    // (24 heads): 80.8 ms with 1-head chunks vs 84.4 ms with 3-head chunks
    const int hc = (Hh + 31) / 32;
    return hc > 0 ? hc : 1;
}

// byte offsets of one slot's buffers
struct SlotLayout {
    size_t in, out, z, cnt, mask, scores, idx, ws, ws_bytes, total;
};

veda_status slot_layout(int hc, int64_t N, const Shape &sh, int d, int k, const veda_scorer *w, SlotLayout *L)
{
    size_t ws = 0;
    veda_status st = veda_tile_score_workspace(hc, sh.NT, d, w, &ws);
    if (st != VEDA_OK) return st;
    const size_t tok = align256((size_t)hc * N * d * 2);
    size_t p = 0;
    L->in = p; p += 3 * tok;
    L->out = p; p += tok;
    L->z = p; p += 2 * align256((size_t)hc * sh.NT * 3 * d * 4);
    L->cnt = p; p += align256((size_t)hc * sh.NT * 4);
    L->mask = p; p += align256((size_t)hc * sh.NT * (sh.B / 32) * 4);
    L->scores = p; p += align256((size_t)hc * sh.NT * sh.NT * 4);
    L->idx = p; p += align256((size_t)hc * sh.NT * k * 4);
    L->ws = p; p += align256(ws);
    L->ws_bytes = ws;
    L->total = p;
    return VEDA_OK;
}

struct EventSet {
    std::vector<cudaEvent_t> ev;
    ~EventSet()
    {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);  // released once the device passes them
    }
    cudaEvent_t make()
    {
        cudaEvent_t e = nullptr;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
        ev.push_back(e);
        return e;
    }
};

#define VEDA_CU(x)                                                                                          \
    do {                                                                                                    \
        const cudaError_t e_ = (x);                                                                         \
        if (e_ != cudaSuccess) return fail(VEDA_ERR_CUDA, "sparse_attention_host: %s: %s", #x,               \
                                           cudaGetErrorString(e_));                                         \
    } while (0)

}  // namespace
}  // namespace veda

using namespace veda;

extern "C" {

veda_status veda_sparse_attention_host_workspace(veda_latent lat, const veda_tile_cfg *cfg, int32_t Hh, int32_t d,
                                                 int32_t k, const veda_scorer *w, int32_t heads_per_chunk,
                                                 size_t *bytes)
{
    if (!w || !bytes) return fail(VEDA_ERR_NULL, "sparse_attention_host_workspace: NULL pointer");
    Shape sh;
    veda_status st = shape_of(lat, cfg, Hh, &sh, nullptr);
    if (st != VEDA_OK) return st;
    if (k < 1 || k > sh.NT) return fail(VEDA_ERR_K_RANGE, "sparse_attention_host: k=%d outside [1, %d]", k, sh.NT);
    SlotLayout L;
    const int64_t N = (int64_t)lat.t * lat.h * lat.w;
    if ((st = slot_layout(chunk_heads(Hh, heads_per_chunk), N, sh, d, k, w, &L)) != VEDA_OK) return st;
    *bytes = kSlots * L.total;
    return VEDA_OK;
}

veda_status veda_sparse_attention_host(const uint16_t *q_host, const uint16_t *k_host, const uint16_t *v_host,
                                       int64_t head_stride, int64_t token_stride, veda_latent lat,
                                       const veda_tile_cfg *cfg, int32_t Hh, int32_t d, int32_t k,
                                       const veda_scorer *w, int32_t heads_per_chunk, uint16_t *o_host,
                                       void *workspace, size_t workspace_bytes, void *stream)
{
    if (!q_host || !k_host || !v_host || !o_host || !w || !workspace)
        return fail(VEDA_ERR_NULL, "sparse_attention_host: NULL pointer");
    if (d != 64 && d != 128) return fail(VEDA_ERR_SHAPE, "sparse_attention_host: d=%d unsupported", d);
    Shape sh;
    HeadCfgs all;
    veda_status st = shape_of(lat, cfg, Hh, &sh, &all);  // argument errors before any device call
    if (st != VEDA_OK) return st;
    if (k < 1 || k > sh.NT) return fail(VEDA_ERR_K_RANGE, "sparse_attention_host: k=%d outside [1, %d]", k, sh.NT);
    const int64_t N = (int64_t)lat.t * lat.h * lat.w;
    const bool head_major = head_stride == N * d && token_stride == d;
    const bool token_major = head_stride == d && token_stride == (int64_t)Hh * d;
    if (!head_major && !token_major)
        return fail(VEDA_ERR_SHAPE, "sparse_attention_host: host layout must be [Hh][N][d] or [N][Hh][d] (dense)");
    const int hc = chunk_heads(Hh, heads_per_chunk);
    SlotLayout L;
    if ((st = slot_layout(hc, N, sh, d, k, w, &L)) != VEDA_OK) return st;
    // the scorer's arrays are checked before anything is enqueued
    if (!w->w1q || !w->b1q || !w->w2q || !w->b2q || !w->w1k || !w->b1k || !w->w2k || !w->b2k)
        return fail(VEDA_ERR_NULL, "sparse_attention_host: scorer weight pointer is NULL");
    if (workspace_bytes < kSlots * L.total)
        return fail(VEDA_ERR_WORKSPACE, "sparse_attention_host: workspace %zu < %zu", workspace_bytes,
                    kSlots * L.total);
    if (!aligned16(workspace)) return fail(VEDA_ERR_ALIGN, "sparse_attention_host: workspace not aligned");
    if ((st = check_arch()) != VEDA_OK) return st;
    SideStreams side;
    if ((st = side_streams(&side)) != VEDA_OK) return st;
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);

    const int n_chunks = (Hh + hc - 1) / hc;
    EventSet E;
    std::vector<cudaEvent_t> ev_h2d(n_chunks), ev_infree(n_chunks), ev_comp(n_chunks), ev_d2h(n_chunks);
    cudaEvent_t ev_start = E.make();
    for (int c = 0; c < n_chunks; ++c) {
        ev_h2d[c] = E.make(); ev_infree[c] = E.make(); ev_comp[c] = E.make(); ev_d2h[c] = E.make();
        if (!ev_h2d[c] || !ev_infree[c] || !ev_comp[c] || !ev_d2h[c])
            return fail(VEDA_ERR_CUDA, "sparse_attention_host: event creation failed");
    }
    if (!ev_start) return fail(VEDA_ERR_CUDA, "sparse_attention_host: event creation failed");
    // earlier work on the caller's stream may still use the workspace
    VEDA_CU(cudaEventRecord(ev_start, cs));
    VEDA_CU(cudaStreamWaitEvent(side.h2d, ev_start, 0));
    VEDA_CU(cudaStreamWaitEvent(side.d2h, ev_start, 0));

    auto enqueue = [&]() -> veda_status {
        const size_t tok = align256((size_t)hc * N * d * 2);
        const size_t zb = align256((size_t)hc * sh.NT * 3 * d * 4);
        const uint16_t *src[3] = {q_host, k_host, v_host};
        for (int c = 0; c < n_chunks; ++c) {
            const int h0 = c * hc;
            const int hn = (h0 + hc <= Hh) ? hc : Hh - h0;
            char *slot = static_cast<char *>(workspace) + (size_t)(c % kSlots) * L.total;
            uint16_t *in[3];
            for (int j = 0; j < 3; ++j) in[j] = reinterpret_cast<uint16_t *>(slot + L.in + j * tok);
            uint16_t *out = reinterpret_cast<uint16_t *>(slot + L.out);
            float *zq = reinterpret_cast<float *>(slot + L.z), *zk = reinterpret_cast<float *>(slot + L.z + zb);
            int32_t *cnt = reinterpret_cast<int32_t *>(slot + L.cnt);
            uint32_t *mask = reinterpret_cast<uint32_t *>(slot + L.mask);
            float *scores = reinterpret_cast<float *>(slot + L.scores);
            int32_t *idx = reinterpret_cast<int32_t *>(slot + L.idx);
            void *ws = slot + L.ws;
            // device strides of the chunk buffers (same layout kind as the host tensors)
            const int64_t dhs = head_major ? N * d : d;
            const int64_t dts = head_major ? d : (int64_t)hn * d;

            // 1. H2D of chunk c into slot c % 2 once the attention of chunk c-2 has read it
            if (c >= kSlots) VEDA_CU(cudaStreamWaitEvent(side.h2d, ev_infree[c - kSlots], 0));
            for (int j = 0; j < 3; ++j) {
                if (head_major)
                    VEDA_CU(cudaMemcpyAsync(in[j], src[j] + (size_t)h0 * N * d, (size_t)hn * N * d * 2,
                                            cudaMemcpyHostToDevice, side.h2d));
                else
                    VEDA_CU(cudaMemcpy2DAsync(in[j], (size_t)hn * d * 2, src[j] + (size_t)h0 * d, (size_t)Hh * d * 2,
                                              (size_t)hn * d * 2, (size_t)N, cudaMemcpyHostToDevice, side.h2d));
            }
            VEDA_CU(cudaEventRecord(ev_h2d[c], side.h2d));

            // 2. the path on the caller's stream (token layout in and out)
            VEDA_CU(cudaStreamWaitEvent(cs, ev_h2d[c], 0));
            HeadCfgs hcf;
            for (int h = 0; h < hn; ++h) { hcf.pt[h] = all.pt[h0 + h]; hcf.ph[h] = all.ph[h0 + h]; hcf.pw[h] = all.pw[h0 + h]; }
            if ((st = launch_tile_pool_tokens2(in[0], in[1], dhs, dts, hcf, hn, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h, lat.w,
                                               sh.B, sh.NT, d, zq, zk, cnt, mask, cs)) != VEDA_OK)
                return st;
            veda_scorer wc = *w;
        wc.prepared = nullptr;  // prepared images are laid out for the whole head range
            const size_t o1 = (size_t)h0 * w->d_in * w->d_hidden, o2 = (size_t)h0 * w->d_hidden * w->d_lat;
            wc.w1q += o1; wc.w1k += o1; wc.b1q += (size_t)h0 * w->d_hidden; wc.b1k += (size_t)h0 * w->d_hidden;
            wc.w2q += o2; wc.w2k += o2; wc.b2q += (size_t)h0 * w->d_lat; wc.b2k += (size_t)h0 * w->d_lat;
            if ((st = veda_tile_score_pooled(zq, zk, cnt, hn, sh.NT, d, &wc, scores, ws, L.ws_bytes, cs)) != VEDA_OK)
                return st;
            if ((st = veda_select_topk(scores, hn, sh.NT, k, idx, cs)) != VEDA_OK) return st;
            if (c >= kSlots) VEDA_CU(cudaStreamWaitEvent(cs, ev_d2h[c - kSlots], 0));  // out slot drained
            const float scale = 1.0f / std::sqrt((float)d);
            if ((st = launch_sparse_attn_tok(in[0], in[1], in[2], dhs, dts, hcf, hn, sh.Tp, sh.Hp, sh.Wp, lat.t, lat.h,
                                             lat.w, sh.B, sh.NT, d, idx, mask, k, scale, out, dhs, dts, nullptr, 0,
                                             hn * sh.NT, cs)) !=
                VEDA_OK)
                return st;
            VEDA_CU(cudaEventRecord(ev_infree[c], cs));  // the attention was the last reader of Q/K/V
            VEDA_CU(cudaEventRecord(ev_comp[c], cs));

            // 3. D2H of chunk c
            VEDA_CU(cudaStreamWaitEvent(side.d2h, ev_comp[c], 0));
            if (head_major)
                VEDA_CU(cudaMemcpyAsync(o_host + (size_t)h0 * N * d, out, (size_t)hn * N * d * 2, cudaMemcpyDeviceToHost,
                                        side.d2h));
            else
                VEDA_CU(cudaMemcpy2DAsync(o_host + (size_t)h0 * d, (size_t)Hh * d * 2, out, (size_t)hn * d * 2,
                                          (size_t)hn * d * 2, (size_t)N, cudaMemcpyDeviceToHost, side.d2h));
            VEDA_CU(cudaEventRecord(ev_d2h[c], side.d2h));
        }
        return VEDA_OK;
    };
    if ((st = enqueue()) != VEDA_OK) {
        // a mid-loop failure may leave H2D/D2H copies of the caller's host buffers queued on
        // the side streams: let them finish before the caller can free or reuse the buffers
        cudaStreamSynchronize(side.h2d);
        cudaStreamSynchronize(side.d2h);
        return st;
    }
    // the caller's stream completes only after the last D2H (the d2h stream is in order)
    VEDA_CU(cudaStreamWaitEvent(cs, ev_d2h[n_chunks - 1], 0));
    return VEDA_OK;
}

}  // extern "C"
