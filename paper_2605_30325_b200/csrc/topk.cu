// topk.cu -- per-query-tile exact top-k selection (step a5 of the path).
//
// PAPER.md:146-149 (exactly k kept key tiles per query tile), PAPER.md:280 ("retain the
// k highest-scoring key tiles for each query tile"), Alg. 2 line 697.  Readings R10/R11/
// R16: exactly k; among equal scores the lower key-tile index wins; output ascending;
// -0.0 == +0.0.
//
// One CTA (256 threads) per row.  Scores become order-preserving uint32 keys in smem;
// a 4-pass 8-bit MSB radix select finds the k-th largest key T and how many keys equal
// to T must be taken; a final pass in index order emits {key > T} plus the first
// `need` keys == T, compacted with warp ballots -- so the output is ascending by
// construction and identical to "sort by (S desc, j asc), take k, sort by j".
#include "common.cuh"

#include <cstdlib>
#include <cstring>

namespace veda {
namespace {

__device__ __forceinline__ uint32_t order_key(float f)
{
    uint32_t u = __float_as_uint(f);
    if (u == 0x80000000u) u = 0u;  // -0 -> +0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

constexpr int TK_THREADS = 256;
constexpr int TK_WARPS = TK_THREADS / 32;

__global__ void __launch_bounds__(TK_THREADS) topk_kernel(const float *__restrict__ S, int NT, int k,
                                                          int32_t *__restrict__ idx)
{
    extern __shared__ uint32_t keys[];
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_prefix, s_kk;
    __shared__ uint32_t s_w_eq[TK_WARPS], s_w_sel[TK_WARPS];
    const int row = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float *s = S + (size_t)row * NT;
    for (int j = tid; j < NT; j += TK_THREADS) keys[j] = order_key(__ldg(s + j));

    uint32_t prefix = 0, pmask = 0, kk = (uint32_t)k;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        hist[tid] = 0;  // TK_THREADS == 256 bins
        __syncthreads();
        for (int j = tid; j < NT; j += TK_THREADS) {
            const uint32_t key = keys[j];
            if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (warp == 0) {
            // lane l owns bins 255-8l ... 248-8l (descending)
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) { c[q] = hist[255 - 8 * lane - q]; tot += c[q]; }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += v;
            }
            uint32_t run = incl - tot;  // keys with a larger digit than this lane's first bin
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (run < kk && kk <= run + c[q]) {
                    s_prefix = prefix | ((uint32_t)(255 - 8 * lane - q) << shift);
                    s_kk = kk - run;
                }
                run += c[q];
            }
        }
        __syncthreads();
        prefix = s_prefix;
        kk = s_kk;
        pmask |= 255u << shift;
    }
    const uint32_t T = prefix;  // the k-th largest key; kk keys equal to T are taken
    uint32_t out_base = 0, eq_base = 0;
    int32_t *out = idx + (size_t)row * k;
    for (int base = 0; base < NT; base += TK_THREADS) {
        const int j = base + tid;
        const uint32_t key = j < NT ? keys[j] : 0u;
        const bool gt = j < NT && key > T;
        const bool eq = j < NT && key == T;
        const uint32_t beq = __ballot_sync(0xFFFFFFFFu, eq);
        if (lane == 0) s_w_eq[warp] = __popc(beq);
        __syncthreads();
        uint32_t eq_before = eq_base, eq_tot = 0;
#pragma unroll
        for (int w = 0; w < TK_WARPS; ++w) {
            if (w < warp) eq_before += s_w_eq[w];
            eq_tot += s_w_eq[w];
        }
        eq_before += __popc(beq & ((1u << lane) - 1u));
        const bool sel = gt || (eq && eq_before < kk);
        const uint32_t bsel = __ballot_sync(0xFFFFFFFFu, sel);
        if (lane == 0) s_w_sel[warp] = __popc(bsel);
        __syncthreads();
        uint32_t pos = out_base, sel_tot = 0;
#pragma unroll
        for (int w = 0; w < TK_WARPS; ++w) {
            if (w < warp) pos += s_w_sel[w];
            sel_tot += s_w_sel[w];
        }
        pos += __popc(bsel & ((1u << lane) - 1u));
        if (sel) out[pos] = j;
        out_base += sel_tot;
        eq_base += eq_tot;
        __syncthreads();  // s_w_* reused next chunk
    }
}


// Warp-per-row variant for n_tiles <= 32*C: lane l holds keys j = 32*i + l (i < C) in
// registers.  The k-th largest key T is built bit by bit from the MSB: a candidate bit is
// kept while at least k keys are >= the candidate (one compare per key plus a redux.sync
// per bit); the search stops as soon as exactly k keys are >= the candidate.  The index-
// order pass then takes keys > T plus the first (k - #{> T}) keys == T, compacted by
// ballots over i -- the same contract as topk_kernel above, without smem or CTA syncs.
constexpr int TKW_WARPS = 8;

// #{i : key[i] >= c} for this lane (c >= 1, or c = 0 meaning "none": see the caller): key +
// (2^32 - c) carries out iff key >= c, so each key costs one add-with-carry-out and one
// add of the carry (two instructions) instead of compare + select + add, and four
// independent accumulators keep the adds off a single dependency chain.
template <int C>
__device__ __forceinline__ uint32_t count_ge(const uint32_t (&key)[C], uint32_t c)
{
    const uint32_t negc = 0u - c;
    uint32_t n[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < C; ++i)
        asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, 0;\n\t}"
            : "+r"(n[i & 3])
            : "r"(key[i]), "r"(negc));
    return (n[0] + n[1]) + (n[2] + n[3]);
}

template <int C>
__global__ void __launch_bounds__(TKW_WARPS * 32, 3) topk_warp_kernel(const float *__restrict__ S, int rows, int NT,
                                                                   int k, int32_t *__restrict__ idx)
{
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * TKW_WARPS + (threadIdx.x >> 5);
    if (row >= rows) return;
    const float *s = S + (size_t)row * NT;
    uint32_t key[C];
#pragma unroll
    for (int i = 0; i < C; ++i) {
        const int j = 32 * i + lane;
        key[i] = j < NT ? order_key(__ldg(s + j)) : 0u;  // 0 sorts below every finite or -inf key
    }
    const uint32_t kk = (uint32_t)k;
    uint32_t T = 0;
#pragma unroll 1
    for (int b = 31; b >= 0; --b) {
        const uint32_t c = T | (1u << b);
        const uint32_t n = __reduce_add_sync(0xFFFFFFFFu, count_ge<C>(key, c));
        if (n >= kk) {
            T = c;
            if (n == kk) break;  // {key >= T} is exactly the answer
        }
    }
    // keys > T = keys >= T + 1 (T + 1 wraps to 0 only for T = 2^32 - 1, where none is greater:
    // count_ge(0) adds 2^32 - 0 = 0 and never carries)
    const uint32_t ngt = __reduce_add_sync(0xFFFFFFFFu, count_ge<C>(key, T + 1u));
    const uint32_t need = kk - ngt;  // keys == T to take, lowest indices first
    const uint32_t lt = (1u << lane) - 1u;
    int32_t *out = idx + (size_t)row * k;
    uint32_t base = 0, eq_seen = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) {
        const int j = 32 * i + lane;
        const bool eq = j < NT && key[i] == T;
        const uint32_t beq = __ballot_sync(0xFFFFFFFFu, eq);
        const bool sel = (j < NT && key[i] > T) || (eq && eq_seen + __popc(beq & lt) < need);
        eq_seen += __popc(beq);
        const uint32_t bsel = __ballot_sync(0xFFFFFFFFu, sel);
        if (sel) out[base + __popc(bsel & lt)] = j;
        base += __popc(bsel);
    }
}

}  // namespace

template <int C>
static veda_status launch_topk_warp(const float *scores, int rows, int NT, int k, int32_t *idx, cudaStream_t s)
{
    topk_warp_kernel<C><<<(rows + TKW_WARPS - 1) / TKW_WARPS, TKW_WARPS * 32, 0, s>>>(scores, rows, NT, k, idx);
    count_launch();
    return check_launch("select_topk");
}

veda_status launch_topk(const float *scores, int Hh, int NT, int k, int32_t *idx, cudaStream_t s)
{
    const int rows = Hh * NT;
    static const bool force_cta = [] {
        const char *e = getenv("VEDA_TOPK");
        return e && !strcmp(e, "cta");
    }();
    if (!force_cta) {
        if (NT <= 32 * 4) return launch_topk_warp<4>(scores, rows, NT, k, idx, s);
        if (NT <= 32 * 16) return launch_topk_warp<16>(scores, rows, NT, k, idx, s);
        if (NT <= 32 * 32) return launch_topk_warp<32>(scores, rows, NT, k, idx, s);
        if (NT <= 32 * 64) return launch_topk_warp<64>(scores, rows, NT, k, idx, s);
    }
    const size_t smem = (size_t)NT * sizeof(uint32_t);
    if (smem > 200 * 1024) return fail(VEDA_ERR_SHAPE, "select_topk: n_tiles=%d too large", NT);
    static size_t attr = 0;
    if (smem > 48 * 1024 && smem > attr) {
        cudaError_t e = cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        attr = smem;
    }
    topk_kernel<<<rows, TK_THREADS, smem, s>>>(scores, NT, k, idx);
    count_launch();
    return check_launch("select_topk");
}

}  // namespace veda
