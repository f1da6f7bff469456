// target.cu -- exact pooled target scores S_tgt (Eq. 4) and tile recall (Eq. 3).
//
// Eq. 4 (Alg. 3):  A* = softmax(Q K^T / sqrt(d)),
//     S_tgt[i][j] = max_{u in tile i, v in tile j} A*_uv
//                 = exp2( max_u ( max_v s_uv * scale*log2e  -  lse_u * log2e ) ),
// because exp is monotone and lse_u (the row log-sum-exp over ALL real keys) is constant
// along a row.  PAPER.md:412-416 computes this in two passes: running row statistics
// first, then the per-tile maxima normalised by them.  Here pass 1 is the dense
// veda_sparse_attn_fwd (k = N_T, lse output); this file is pass 2, which needs only
// QK^T: no exponentials per element, no PV.  Readings (R4/R5/R19): padded key
// slots are excluded, padded query rows are excluded, an empty key tile scores -inf and
// an empty query tile 0.
//
// B200 design: persistent, one CTA per SM, 384 threads.
//   warp 0      TMA producer: the pair's two Q tiles, then K tiles j = 0..N_T-1 (ring)
//   warp 1      MMA issuer: S(b, s) = Q_s K_j^T for both slots from ONE K stage
//   warps 4-11  two reducer warpgroups (one per slot), one TMEM lane (query row) per thread
// A work item is a PAIR of query tiles (i, i+1) of one head: every K tile is loaded once
// per pair and feeds two 128xBxD MMAs.  S is double-buffered in TMEM
// (2 buffers x 2 slots x 128 columns = 512), so the MMAs of key tile j+1 run while the
// reducers read tile j.  Per (i, j) the CTA writes one fp32.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "sm100.cuh"

namespace veda {
namespace tgt {
using namespace sm100;

constexpr int NTHREADS = 384;
constexpr uint32_t TMEM_COLS = 512;

struct Params {
    const uint32_t *slot_mask;
    const float *lse;
    float *out;
    int NT, pairs_per_head, total_pairs;
    float scale_log2;
};

template <int B, int D>
struct Geo {
    static constexpr int QCHUNK = 128 * 128;  // one 64-col chunk of a 128-row Q buffer
    static constexpr int Q_BYTES = QCHUNK * (D / 64);
    static constexpr int KCHUNK = B * 128;
    static constexpr int TILE_BYTES = KCHUNK * (D / 64);
    static constexpr int NST_FIT = (200 * 1024 - 2 * Q_BYTES) / TILE_BYTES;
    static constexpr int NST = NST_FIT > 8 ? 8 : NST_FIT;
    static constexpr int MW = B / 32;
    static constexpr int NBAR = 2 * NST + 2 + 4;
    static constexpr int SMEM = 2 * Q_BYTES + NST * TILE_BYTES + NBAR * 8 + 16 + 2 * 2 * 4 * 4 + 1024;
    static_assert(NST >= 2, "ring too shallow");
};

template <int B, int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    target_scores_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const Params p)
{
    using G = Geo<B, D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sRing = sQ + 2 * G::Q_BYTES;
    const uint32_t sBar = sRing + G::NST * G::TILE_BYTES;
    uint8_t *after_bar = smem + 2 * G::Q_BYTES + G::NST * G::TILE_BYTES + G::NBAR * 8;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(after_bar);
    float *part = reinterpret_cast<float *>(after_bar + 16);  // [slot][j&1][quarter]
#define RING_FULL(i) (sBar + 8u * (i))
#define RING_EMPTY(i) (sBar + 8u * (G::NST + (i)))
#define Q_FULL (sBar + 8u * (2 * G::NST))
#define Q_EMPTY (sBar + 8u * (2 * G::NST + 1))
#define S_FULL(b) (sBar + 8u * (2 * G::NST + 2 + (b)))
#define S_EMPTY(b) (sBar + 8u * (2 * G::NST + 4 + (b)))

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (B < 128) {  // Q rows B..127 of the M=128 operand are never loaded: keep them zero
        uint4 *q4 = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < 2 * G::Q_BYTES / 16; i += NTHREADS) q4[i] = make_uint4(0, 0, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G::NST; ++i) {
            mbar_init(RING_FULL(i), 1);
            mbar_init(RING_EMPTY(i), 1);
        }
        mbar_init(Q_FULL, 1);
        mbar_init(Q_EMPTY, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(S_FULL(b), 1);
            mbar_init(S_EMPTY(b), 8);  // lane 0 of each of the 8 reducer warps
        }
        fence_barrier_init();
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    const int NT = p.NT, PPH = p.pairs_per_head, total = p.total_pairs;

    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            uint32_t stage = 0, ph = 0, qe = 0;
            for (int w = blockIdx.x; w < total; w += gridDim.x) {
                const int h = w / PPH, i0 = 2 * (w % PPH);
                const int nq = (i0 + 1 < NT) ? 2 : 1;
                mbar_wait(Q_EMPTY, qe ^ 1);
                qe ^= 1;
                mbar_expect_tx(Q_FULL, nq * B * D * 2);
                for (int s = 0; s < nq; ++s)
#pragma unroll
                    for (int c = 0; c < D / 64; ++c)
                        tma_load_2d(sQ + s * G::Q_BYTES + c * G::QCHUNK, &tmQ, c * 64, (h * NT + i0 + s) * B, Q_FULL);
                for (int j = 0; j < NT; ++j) {
                    mbar_wait(RING_EMPTY(stage), ph ^ 1);
                    mbar_expect_tx(RING_FULL(stage), G::TILE_BYTES);
#pragma unroll
                    for (int c = 0; c < D / 64; ++c)
                        tma_load_2d(sRing + stage * G::TILE_BYTES + c * G::KCHUNK, &tmK, c * 64, (h * NT + j) * B,
                                    RING_FULL(stage));
                    if (++stage == G::NST) { stage = 0; ph ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ============================ MMA issuer ============================
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(128, B, 0, 0);
            uint32_t stage = 0, ph = 0, qf = 0, step = 0;
            for (int w = blockIdx.x; w < total; w += gridDim.x) {
                const int i0 = 2 * (w % PPH);
                const int nq = (i0 + 1 < NT) ? 2 : 1;
                mbar_wait(Q_FULL, qf);
                qf ^= 1;
                for (int j = 0; j < NT; ++j, ++step) {
                    const uint32_t b = step & 1u, eph = ((step >> 1) & 1u) ^ 1u;
                    mbar_wait(S_EMPTY(b), eph);
                    mbar_wait(RING_FULL(stage), ph);
                    tc_fence_after();
                    const uint32_t kb = sRing + stage * G::TILE_BYTES;
                    for (int s = 0; s < nq; ++s) {
                        const uint32_t qa = sQ + s * G::Q_BYTES, tS = tbase + b * 256 + s * 128;
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint64_t ad = sdesc_sw128(qa + (kk >> 2) * G::QCHUNK + (kk & 3) * 32, 16, 1024);
                            const uint64_t bd = sdesc_sw128(kb + (kk >> 2) * G::KCHUNK + (kk & 3) * 32, 16, 1024);
                            mma_ss(tS, ad, bd, idesc, kk > 0 ? 1u : 0u);
                        }
                    }
                    tc_commit(S_FULL(b));
                    tc_commit(RING_EMPTY(stage));
                    if (j == NT - 1) tc_commit(Q_EMPTY);
                    if (++stage == G::NST) { stage = 0; ph ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        // ============================ reducers ============================
        const int slot = (warp - 4) >> 2;
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const float sl2 = p.scale_log2;
        uint32_t step = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            const int h = w / PPH, i = 2 * (w % PPH) + slot;
            const bool act = i < NT;
            const size_t u = (size_t)h * NT + (act ? i : 0);
            bool qvalid = false;
            if (act && row < B) qvalid = (__ldg(p.slot_mask + u * G::MW + (row >> 5)) >> (row & 31)) & 1u;
            const float lse2 = qvalid ? __ldg(p.lse + u * B + row) * 1.4426950408889634f : 0.f;
            const uint32_t *mk_head = p.slot_mask + (size_t)h * NT * G::MW;
            float *orow = p.out + u * NT;
            for (int j = 0; j < NT; ++j, ++step) {
                const uint32_t b = step & 1u, fph = (step >> 1) & 1u;
                uint32_t mk[G::MW];
                bool any = false, full = true;
#pragma unroll
                for (int x = 0; x < G::MW; ++x) {
                    mk[x] = __ldg(mk_head + (size_t)j * G::MW + x);
                    any |= mk[x] != 0u;
                    full &= mk[x] == 0xFFFFFFFFu;
                }
                mbar_wait(S_FULL(b), fph);
                tc_fence_after();
                uint32_t sr[B / 32][32];
                const uint32_t tS = tbase + lane_off + b * 256 + slot * 128;
#pragma unroll
                for (int c = 0; c < B / 32; ++c) tmem_ld32(tS + c * 32, sr[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < B / 32; ++c) reg_fence(sr[c]);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(S_EMPTY(b));
                if (!act) continue;
                if (!full) {
#pragma unroll
                    for (int c = 0; c < B / 32; ++c)
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (!((mk[c] >> e) & 1u)) sr[c][e] = __float_as_uint(-INFINITY);
                }
                float pm[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pm[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < B / 32; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e) pm[e & 7] = fmaxf(pm[e & 7], __uint_as_float(sr[c][e]));
                const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
                float r = (qvalid && any) ? fmaf(mx, sl2, -lse2) : -INFINITY;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) r = fmaxf(r, __shfl_xor_sync(0xFFFFFFFFu, r, o));
                float *pj = part + (slot * 2 + (j & 1)) * 4;
                if (lane == 0) pj[quarter] = r;
                asm volatile("bar.sync %0, 128;" ::"r"(1 + slot) : "memory");
                if (quarter == 0 && lane == 0) {
                    const float v = fmaxf(fmaxf(pj[0], pj[1]), fmaxf(pj[2], pj[3]));
                    orow[j] = any ? exp2f(v) : -INFINITY;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, TMEM_COLS);
    }
#undef RING_FULL
#undef RING_EMPTY
#undef Q_FULL
#undef Q_EMPTY
#undef S_FULL
#undef S_EMPTY
}

template <int B, int D>
static veda_status launch(const uint16_t *q, const uint16_t *k, const uint32_t *mask, const float *lse, int Hh,
                          int NT, float scale, float *out, cudaStream_t stream)
{
    using G = Geo<B, D>;
    CUtensorMap mq, mk;
    const uint64_t rows = (uint64_t)Hh * NT * B;
    veda_status st;
    if ((st = make_tmap_bf16(&mq, q, rows, D, B)) != VEDA_OK) return st;
    if ((st = make_tmap_bf16(&mk, k, rows, D, B)) != VEDA_OK) return st;
    {  // set per launch: the attribute belongs to the current device's context
        cudaError_t e = cudaFuncSetAttribute(target_scores_kernel<B, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             G::SMEM);
        if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
    Params p;
    p.slot_mask = mask;
    p.lse = lse;
    p.out = out;
    p.NT = NT;
    p.pairs_per_head = (NT + 1) / 2;
    p.total_pairs = Hh * p.pairs_per_head;
    p.scale_log2 = scale * 1.4426950408889634f;
    int grid = p.total_pairs;
    const int nsm = num_sms();
    if (grid > nsm) grid = nsm;
    target_scores_kernel<B, D><<<grid, NTHREADS, G::SMEM, stream>>>(mq, mk, p);
    count_launch();
    return check_launch("target_scores");
}

// ---------------------------------------------------------------------------- recall
// One CTA, one warp per row: the warp marks S_fu,i in a private smem bitmap, counts the
// members of S_sp,i, then clears its marks.  Sums are exact integers; the mean is formed
// once at the end in fp64.
constexpr int RC_THREADS = 1024;
constexpr int RC_WARPS = RC_THREADS / 32;

__global__ void __launch_bounds__(RC_THREADS) recall_kernel(const int32_t *__restrict__ sp,
                                                            const int32_t *__restrict__ fu,
                                                            const int32_t *__restrict__ cnt, int64_t rows, int NT,
                                                            int k, double *__restrict__ recall)
{
    extern __shared__ uint32_t bm[];
    __shared__ unsigned long long s_inter[RC_WARPS], s_rows[RC_WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int words = (NT + 31) / 32;
    uint32_t *my = bm + (size_t)warp * words;
    for (int x = lane; x < words; x += 32) my[x] = 0u;
    __syncwarp();
    unsigned long long inter = 0, nrows = 0;
    for (int64_t r = warp; r < rows; r += RC_WARPS) {
        if (cnt != nullptr && __ldg(cnt + r) == 0) continue;
        const int32_t *f = fu + r * k, *s = sp + r * k;
        for (int a = lane; a < k; a += 32) {
            const int j = __ldg(f + a);
            if (j >= 0 && j < NT) atomicOr(my + (j >> 5), 1u << (j & 31));
        }
        __syncwarp();
        int c = 0;
        for (int a = lane; a < k; a += 32) {
            const int j = __ldg(s + a);
            if (j >= 0 && j < NT) c += (my[j >> 5] >> (j & 31)) & 1u;
        }
        __syncwarp();
        for (int a = lane; a < k; a += 32) {
            const int j = __ldg(f + a);
            if (j >= 0 && j < NT) my[j >> 5] = 0u;
        }
        __syncwarp();
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
        inter += (unsigned long long)c;
        nrows += 1;
    }
    if (lane == 0) { s_inter[warp] = inter; s_rows[warp] = nrows; }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long ti = 0, tr = 0;
        for (int x = 0; x < RC_WARPS; ++x) { ti += s_inter[x]; tr += s_rows[x]; }
        *recall = tr ? (double)ti / ((double)tr * (double)k) : 0.0;
    }
}

}  // namespace tgt

veda_status launch_target_scores(const uint16_t *q, const uint16_t *k, const uint32_t *mask, const float *lse,
                                 int Hh, int NT, int B, int d, float scale, float *out, cudaStream_t s)
{
    if (B == 128 && d == 128) return tgt::launch<128, 128>(q, k, mask, lse, Hh, NT, scale, out, s);
    if (B == 128 && d == 64) return tgt::launch<128, 64>(q, k, mask, lse, Hh, NT, scale, out, s);
    if (B == 64 && d == 128) return tgt::launch<64, 128>(q, k, mask, lse, Hh, NT, scale, out, s);
    if (B == 64 && d == 64) return tgt::launch<64, 64>(q, k, mask, lse, Hh, NT, scale, out, s);
    return fail(VEDA_ERR_CONFIG, "target_scores: unsupported (B=%d, d=%d)", B, d);
}

veda_status launch_recall(const int32_t *sp, const int32_t *fu, const int32_t *cnt, int64_t rows, int NT, int k,
                          double *recall, cudaStream_t s)
{
    const size_t smem = (size_t)tgt::RC_WARPS * ((NT + 31) / 32) * sizeof(uint32_t);
    if (smem > 200 * 1024) return fail(VEDA_ERR_SHAPE, "tile_recall: n_tiles=%d too large", NT);
    if (smem > 48 * 1024) {  // set per launch: the attribute belongs to the current device's context
        cudaError_t e =
            cudaFuncSetAttribute(tgt::recall_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
    tgt::recall_kernel<<<1, tgt::RC_THREADS, smem, s>>>(sp, fu, cnt, rows, NT, k, recall);
    count_launch();
    return check_launch("tile_recall");
}

}  // namespace veda
