// attn_fwd.cu -- tile-skipping FlashAttention forward for sm_100a (B200).
//
// Computes Eq. 2 of the paper: for every (head h, query tile i)
//     O_i = softmax(Q~_i K^_i^T * scale) V^_i,   K^_i / V^_i = concat of the k kept tiles
// visiting ONLY the kept key tiles named by idx[h][i][:] (producer
// fetches "only the selected non-contiguous key/value tiles" into a circular buffer).
//
// B200 design:
//  * persistent, one CTA per SM, 384 threads = 3 warpgroups:
//      warp 0      TMA producer: Q tiles and the kept K/V tiles -> SMEM ring (SWIZZLE_128B)
//      warp 1      MMA issuer (warp-uniform, one elected lane): tcgen05.mma,
//                  S = Q K^T (SS) and O += P V (TS)
//      warps 2-3   ring-stage release for slot 0 / slot 1 (warpgroup 0 gives its spare
//                  registers to the softmax warpgroups with setmaxnreg)
//      warps 4-11  two softmax warpgroups ("slots"), one query tile each, one row per thread
//  * two addressing modes: tiled tensors [Hh][N_T][B][d] (2-D TMA boxes, tiled output), or
//    TOK: tiles gathered from token order by one 5-D TMA box each and output rows stored
//    straight to token order (no tiled copies; the path's mode)
//  * each slot owns 256 TMEM columns: S (fp32, 128 cols; P aliases its first B/2 columns
//    as packed bf16) and O (fp32, D cols).  The two slots work on different query
//    tiles with independent kept lists, so one slot's softmax overlaps the other's MMAs.
//  * online softmax in the log2 domain with lazy rescaling: O (in TMEM) is rescaled
//    only when a row max grows by more than 8 (2^8 head-room in fp32/bf16).
//  * padded key slots (slot_mask bit clear) get -inf; padded query rows are written 0.
//  * ordering: the commit after S_{t} = Q K_t^T also covers the previous O += P_{t-1} V,
//    so when softmax sees S_t, O is quiescent and may be rescaled in place.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "sm100.cuh"

namespace veda {
namespace attn {
using namespace sm100;

constexpr int NSLOT = 2;
constexpr int NTHREADS = 128 + 128 * NSLOT;
constexpr int REGS_CTRL = 72;      // setmaxnreg budget of warpgroup 0 (producer / MMA)
constexpr int REGS_SOFTMAX = 216;  // ... and of each softmax warpgroup (72 + 2*216 = 504 per SMSP; 512 deadlocks)
constexpr uint32_t TMEM_COLS = 512;

struct Params {
    const int32_t *idx;
    const uint32_t *slot_mask;
    uint16_t *out;
    float *lse;
    int NT, k, total_units;
    float scale_log2;
    unsigned long long *trace;  // VEDA_ATTN_TRACE builds only: per-step clock64 stamps of CTA 0
};

// Token-layout mode (TOK): Q/K/V tiles are TMA'd straight from the token tensors with one
// 5-D box per tile (make_tmap_tile_tokens: same smem image as the tiled copy, padded
// slots zero-filled) and O rows are stored straight to token order, so the path needs no
// tiled copies of Q, K, V or O.  Heads of one launch may use at
// most MAXC distinct tile shapes (the host splits larger head sets into several launches).
constexpr int MAXC = 8;
struct TokParams {
    CUtensorMap q[MAXC], k[MAXC], v[MAXC];
    int T, H, W, Hp, Wp;
    int tok_major;  // 1: coordinates (d, h, w, h', t); 0: (d, w, h', t, h)
    int64_t o_hs, o_ts;
    uint8_t pt[MAXC], ph[MAXC], pw[MAXC];
    // per shape: tiles per padded row (nbw = Wp/pw) and per padded frame (nbhw), with
    // ceil(2^32/n) multipliers: the single producer thread decodes a tile index per load,
    // so the decode must not cost integer divisions
    uint32_t nbw[MAXC], nbhw[MAXC], mbw[MAXC], mbhw[MAXC];
    uint8_t cid[kMaxHeads];
};

// q = i / n, r = i % n for 0 <= i < 2^24 by a multiply-high with m = ceil(2^32 / n) and one correction
__device__ __forceinline__ int div_magic(int i, uint32_t n, uint32_t m, int &r)
{
    int q = (int)__umulhi((uint32_t)i, m);
    r = i - q * (int)n;
    if (r < 0) { --q; r += (int)n; }
    if (r >= (int)n) { ++q; r -= (int)n; }
    return q;
}

struct TileOrigin {
    int c, t0, h0, w0;
};
__device__ __forceinline__ TileOrigin tile_origin(const TokParams &tp, int h, int i)
{
    TileOrigin o;
    o.c = tp.cid[h];
    int rem, iw;
    const int it = div_magic(i, tp.nbhw[o.c], tp.mbhw[o.c], rem);
    const int ih = div_magic(rem, tp.nbw[o.c], tp.mbw[o.c], iw);
    o.t0 = it * tp.pt[o.c];
    o.h0 = ih * tp.ph[o.c];
    o.w0 = iw * tp.pw[o.c];
    return o;
}
// TMA of the NCH 64-channel chunks of tile (h, i) in token layout (chunk c lands at dst + c*stride)
template <int NCH>
__device__ __forceinline__ void tma_tile_tok(uint32_t dst, uint32_t stride, const CUtensorMap *maps,
                                             const TokParams &tp, int h, int i, uint32_t bar)
{
    const TileOrigin o = tile_origin(tp, h, i);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        if (tp.tok_major)
            tma_load_5d(dst + c * stride, &maps[o.c], c * 64, h, o.w0, o.h0, o.t0, bar);
        else
            tma_load_5d(dst + c * stride, &maps[o.c], c * 64, o.w0, o.h0, o.t0, h, bar);
    }
}

#ifdef VEDA_ATTN_TRACE
#define TR(role, step, field)                                                                      \
    do {                                                                                           \
        if (blockIdx.x == 0 && (step) < 128 && p.trace)                                            \
            p.trace[((role) * 128 + (step)) * 8 + (field)] = clock64();                           \
    } while (0)
#else
#define TR(role, step, field) do { } while (0)
#endif

#ifndef VEDA_RING_BUDGET_KB
#define VEDA_RING_BUDGET_KB 224  // Q buffers + K/V ring; 227 KB is the per-CTA maximum
#endif

template <int B, int D>
struct Geo {
    static constexpr int QCHUNK = 128 * 128;         // one 64-col chunk of the 128-row Q buffer
    static constexpr int Q_BYTES = QCHUNK * (D / 64);
    static constexpr int KCHUNK = B * 128;           // one 64-col chunk of a B-row K/V tile
    static constexpr int TILE_BYTES = KCHUNK * (D / 64);
    static constexpr int NST_FIT = (VEDA_RING_BUDGET_KB * 1024 - NSLOT * Q_BYTES) / TILE_BYTES;
    static constexpr int NST = NST_FIT > 8 ? 8 : NST_FIT;
    static constexpr int MW = B / 32;
    static constexpr int NBAR = 2 * NST + 5 * NSLOT;
    static constexpr int SMEM = NSLOT * Q_BYTES + NST * TILE_BYTES + NBAR * 8 + 16 + 1024;
    static_assert(NST >= 2, "ring too shallow");
};

#ifdef VEDA_ATTN_DEBUG
#define DBG(...) do { if (blockIdx.x == 0) printf(__VA_ARGS__); } while (0)
#else
#define DBG(...) do { } while (0)
#endif

// Fraction of exp2 evaluated on the FMA pipe instead of MUFU: one pair in every
// EMU_EVERY (0 disables).  MUFU.EX2 runs at 16/clk/SM, the same rate at which the
// tensor core consumes a 128x128 score tile.  Measured (profiles/r01_attn_experiments.md):
// slower at the current balance (the MMA issue chain, not MUFU, is critical), so off.
#ifndef VEDA_EMU_EVERY
#define VEDA_EMU_EVERY 0
#endif
constexpr int EMU_EVERY = VEDA_EMU_EVERY;

// 2^x for a PAIR on the FMA/ALU pipes with packed fp32x2 arithmetic (10 issue slots for
// two results, no MUFU): clamp (FMNMX x2), n = rint(x) via the 1.5*2^23 trick and
// f = x - n (FADD2 x3), cubic 2^f (FFMA2 x3, max rel. error 7.5e-5 << bf16's 2^-9),
// exponent insertion (LEA x2).  x = -inf (masked keys) gives ~2^-125 ~ 0.
__device__ __forceinline__ void ex2_emu2(float &y0, float &y1, float x0, float x1)
{
    x0 = fmaxf(x0, -125.0f);  // 2^n * p must stay a normal number (p in [0.7, 1.42))
    x1 = fmaxf(x1, -125.0f);
    float j0, j1, p0, p1;
    asm("{\n\t.reg .b64 rx, rm, rj, rt, rf, rp, c3, c2, c1, c0;\n\t"
        "mov.b64 rx, {%4, %5};\n\t"
        "mov.b64 rm, {%6, %6};\n\t"
        "add.rn.f32x2 rj, rx, rm;\n\t"
        "sub.rn.f32x2 rt, rj, rm;\n\t"
        "sub.rn.f32x2 rf, rx, rt;\n\t"
        "mov.b64 c3, {%7, %7};\n\t"
        "mov.b64 c2, {%8, %8};\n\t"
        "mov.b64 c1, {%9, %9};\n\t"
        "mov.b64 c0, {%10, %10};\n\t"
        "fma.rn.f32x2 rp, rf, c3, c2;\n\t"
        "fma.rn.f32x2 rp, rp, rf, c1;\n\t"
        "fma.rn.f32x2 rp, rp, rf, c0;\n\t"
        "mov.b64 {%0, %1}, rj;\n\t"
        "mov.b64 {%2, %3}, rp;\n\t}"
        : "=f"(j0), "=f"(j1), "=f"(p0), "=f"(p1)
        : "f"(x0), "f"(x1), "f"(12582912.0f), "f"(0.05517162f), "f"(0.24261113f), "f"(0.69326097f),
          "f"(0.99992806f));
    y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(j0) << 23));
    y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(j1) << 23));
}

// packed fp32x2 (sm_100): (d0, d1) = (a0, a1) * b + c
__device__ __forceinline__ void ffma2_bc(float &d0, float &d1, float a0, float a1, float b, float c)
{
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rb, {%4, %4};\n\t"
        "mov.b64 rc, {%5, %5};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1)
        : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
// packed fp32x2: (s0, s1) += (a, b)
__device__ __forceinline__ void fadd2_acc(float &s0, float &s1, float a, float b)
{
    asm("{\n\t.reg .b64 ra, rs;\n\t"
        "mov.b64 ra, {%2, %3};\n\t"
        "mov.b64 rs, {%0, %1};\n\t"
        "add.rn.f32x2 rs, rs, ra;\n\t"
        "mov.b64 {%0, %1}, rs;\n\t}"
        : "+f"(s0), "+f"(s1)
        : "f"(a), "f"(b));
}

__device__ __forceinline__ float u2f(uint32_t u) { return __uint_as_float(u); }
__device__ __forceinline__ uint32_t f2u(float f) { return __float_as_uint(f); }

template <int B, int D, bool TOK>
__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, const Params p,
                           const __grid_constant__ TokParams tp)
{
    using G = Geo<B, D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sRing = sQ + NSLOT * G::Q_BYTES;
    const uint32_t sBar = sRing + G::NST * G::TILE_BYTES;
    uint32_t *tmem_slot =
        reinterpret_cast<uint32_t *>(smem + NSLOT * G::Q_BYTES + G::NST * G::TILE_BYTES + G::NBAR * 8);
    // barrier addresses
#define RING_FULL(i) (sBar + 8u * (i))
#define RING_EMPTY(i) (sBar + 8u * (G::NST + (i)))
#define Q_FULL(s) (sBar + 8u * (2 * G::NST + (s)))
#define Q_EMPTY(s) (sBar + 8u * (2 * G::NST + NSLOT + (s)))
#define S_FULL(s) (sBar + 8u * (2 * G::NST + 2 * NSLOT + (s)))
#define P_FULL(s) (sBar + 8u * (2 * G::NST + 3 * NSLOT + (s)))
#define O_FULL(s) (sBar + 8u * (2 * G::NST + 4 * NSLOT + (s)))

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (B < 128) {  // rows B..127 of the M=128 Q operand are never loaded: keep them zero
        uint4 *q4 = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < NSLOT * G::Q_BYTES / 16; i += NTHREADS) q4[i] = make_uint4(0, 0, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G::NST; ++i) {
            mbar_init(RING_FULL(i), 1);
            mbar_init(RING_EMPTY(i), 1);
        }
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(Q_FULL(s), 1);
            mbar_init(Q_EMPTY(s), 1);
            mbar_init(S_FULL(s), 1);
            mbar_init(P_FULL(s), 128);
            mbar_init(O_FULL(s), 1);
        }
        fence_barrier_init();
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    const int NT = p.NT, K = p.k, total = p.total_units;
    const int gslots = gridDim.x * NSLOT;
    const int rounds = (total + gslots - 1) / gslots;
    // unit u = h*NT + i; consecutive CTAs/slots take consecutive query tiles of one head (L2 reuse)
#define UNIT_OF(r, s) ((r) * gslots + blockIdx.x * NSLOT + (s))

    if (warp < 4) {
#ifndef VEDA_NO_SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS_CTRL));
#endif
    if (lane == 0) DBG("w%d ctrl start tbase=%x\n", warp, tbase);
    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            uint32_t stage = 0, ph = 0;
            uint32_t qe_bits = 0;  // per-slot phase bits of Q_EMPTY
            for (int r = 0; r < rounds; ++r) {
                int u[NSLOT], hh[NSLOT], jv[NSLOT];
                bool act[NSLOT];
                const int32_t *il[NSLOT];
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) {
                    u[s] = UNIT_OF(r, s);
                    act[s] = u[s] < total;
                    hh[s] = act[s] ? u[s] / NT : 0;
                    il[s] = p.idx + (size_t)(act[s] ? u[s] : 0) * K;
                }
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) {
                    if (!act[s]) continue;
                    mbar_wait(Q_EMPTY(s), ((qe_bits >> s) & 1u) ^ 1u);
                    qe_bits ^= 1u << s;
                    mbar_expect_tx(Q_FULL(s), B * D * 2);
#pragma unroll
                    if (TOK)
                        tma_tile_tok<D / 64>(sQ + s * G::Q_BYTES, G::QCHUNK, tp.q, tp, hh[s], u[s] - hh[s] * NT,
                                             Q_FULL(s));
                    else
                        for (int c = 0; c < D / 64; ++c)
                            tma_load_2d(sQ + s * G::Q_BYTES + c * G::QCHUNK, &tmQ, c * 64, u[s] * B, Q_FULL(s));
                }
                auto load_tile = [&](const CUtensorMap *tm, int h, int j) {
                    mbar_wait(RING_EMPTY(stage), ph ^ 1);
#ifdef VEDA_DBG_SKIP_V  // timing experiment only: V tiles are not loaded (wrong results)
                    if (tm == &tmV) {
                        mbar_expect_tx(RING_FULL(stage), 0);
                        if (++stage == G::NST) { stage = 0; ph ^= 1; }
                        return;
                    }
#endif
                    mbar_expect_tx(RING_FULL(stage), G::TILE_BYTES);
                    const int row = (h * NT + j) * B;
                    if (TOK)
                        tma_tile_tok<D / 64>(sRing + stage * G::TILE_BYTES, G::KCHUNK, tm == &tmK ? tp.k : tp.v, tp,
                                             h, j, RING_FULL(stage));
                    else
#pragma unroll
                        for (int c = 0; c < D / 64; ++c)
                            tma_load_2d(sRing + stage * G::TILE_BYTES + c * G::KCHUNK, tm, c * 64, row,
                                        RING_FULL(stage));
                    if (++stage == G::NST) { stage = 0; ph ^= 1; }
                };
#pragma unroll
                for (int s = 0; s < NSLOT; ++s)
                    if (act[s]) { jv[s] = __ldg(il[s]); load_tile(&tmK, hh[s], jv[s]); }
                for (int t = 0; t < K; ++t) {
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!act[s]) continue;
                        const int jn = (t + 1 < K) ? __ldg(il[s] + t + 1) : 0;
                        load_tile(&tmV, hh[s], jv[s]);
                        if (t + 1 < K) { jv[s] = jn; load_tile(&tmK, hh[s], jv[s]); }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 2 || warp == 3) {
        // ============================ ring-stage release ============================
        // Warp 2 (slot 0) / warp 3 (slot 1): S_FULL(s) of tile t lands only when QK(s,t)
        // and every earlier MMA of the issuing thread -- in particular PV(s,t-1) -- are
        // complete, so the stages of K(s,t) and V(s,t-1) can go back to the producer at
        // once (O_FULL releases the unit's last V).  Keeping this off the MMA thread and
        // off the softmax keeps stage hold times short with a 5-stage ring.
        if (lane == 0) {
            const int s = warp - 2;
            uint32_t sf_ph = 0, of_ph = 0;
            for (int r = 0; r < rounds; ++r) {
                if (UNIT_OF(r, s) >= total) break;
                const int A = (UNIT_OF(r, 1) < total) ? 2 : 1;
                const uint32_t base = (uint32_t)r * (2 * NSLOT) * (uint32_t)K;
                // global load index of K(s,t) / V(s,t) in the producer's order
                auto gk = [&](int t) -> uint32_t { return base + (t == 0 ? s : A + 2 * A * (t - 1) + 2 * s + 1); };
                auto gv = [&](int t) -> uint32_t { return base + A + 2 * A * t + ((t < K - 1) ? 2 * s : s); };
                for (int t = 0; t < K; ++t) {
                    mbar_wait(S_FULL(s), sf_ph);
                    sf_ph ^= 1;
                    mbar_arrive(RING_EMPTY(gk(t) % G::NST));
                    if (t > 0) mbar_arrive(RING_EMPTY(gv(t - 1) % G::NST));
                }
                mbar_wait(O_FULL(s), of_ph);
                of_ph ^= 1;
                mbar_arrive(RING_EMPTY(gv(K - 1) % G::NST));
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ============================ MMA issuer ============================
        // One thread issues, slot by slot, groups [PV(s,t) ; QK(s,t+1)] back to back (the
        // QK reuses the S/P columns, so it must follow the PV: same thread => in order).
        // Before a group, the three barriers it needs (P(s,t), the V stage, the next K
        // stage) are probed in ONE asm block so their latencies overlap; only a barrier
        // that is not yet complete is then waited on.  Ring stages are released by the
        // softmax warps; the MMA thread only commits S_FULL (+ Q_EMPTY / O_FULL).
        // The whole warp runs the loop (warp-uniform values, one lane issues via elect.sync:
        // see sm100.cuh mma_ss_w); descriptors are advanced by constant offsets.
        {
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, B, 0, 0);  // Q, K both K-major
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D, 0, 1);  // P K-major (TMEM), V MN-major
            uint32_t stage = 0, ph = 0;
            uint32_t qf_bits = 0, pf_bits = 0;  // per-slot phase bits of Q_FULL / P_FULL
            int nqk = 0, npv = 0;
            (void)nqk; (void)npv;
            auto next_stage = [&](uint32_t &st, uint32_t &sp) {
                st = stage;
                sp = ph;
                if (++stage == G::NST) { stage = 0; ph ^= 1; }
            };
            auto issue_qk = [&](int s, int t, uint32_t st) {
                const uint64_t ad0 = sdesc_sw128(sQ + s * G::Q_BYTES, 16, 1024);
                const uint64_t bd0 = sdesc_sw128(sRing + st * G::TILE_BYTES, 16, 1024);
                const uint32_t tS = tbase + s * 256;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint64_t ao = (uint64_t)(((kk >> 2) * G::QCHUNK + (kk & 3) * 32) >> 4);
                    const uint64_t bo = (uint64_t)(((kk >> 2) * G::KCHUNK + (kk & 3) * 32) >> 4);
                    mma_ss_w(tS, ad0 + ao, bd0 + bo, idesc_qk, kk > 0 ? 1u : 0u);
                }
                tc_commit_w(S_FULL(s));
                if (t == K - 1) tc_commit_w(Q_EMPTY(s));
            };
            auto issue_pv = [&](int s, int t, uint32_t st) {
                // V tile as the MN-major B operand: 16 keys = 16 rows of 128 B; the second
                // 64-wide chunk of d sits one KCHUNK further (LBO).
                const uint64_t vd0 = sdesc_sw128(sRing + st * G::TILE_BYTES, G::KCHUNK, 1024);
                const uint32_t tP = tbase + s * 256, tO = tbase + s * 256 + 128;
#pragma unroll
                for (int kk = 0; kk < B / 16; ++kk)
                    mma_ts_w(tO, tP + kk * 8, vd0 + (uint64_t)((kk * 2048) >> 4), idesc_pv, (t > 0 || kk > 0) ? 1u : 0u);
                if (t == K - 1) tc_commit_w(O_FULL(s));
            };
            for (int r = 0; r < rounds; ++r) {
                uint32_t act_bits = 0;
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) act_bits |= (UNIT_OF(r, s) < total ? 1u : 0u) << s;
                for (int s = 0; s < NSLOT; ++s) {
                    if (!((act_bits >> s) & 1u)) continue;
                    uint32_t st, sp;
                    next_stage(st, sp);
                    mbar_wait(Q_FULL(s), (qf_bits >> s) & 1u);
                    qf_bits ^= 1u << s;
                    mbar_wait(RING_FULL(st), sp);
                    TR(0, nqk, 0);
                    tc_fence_after();
                    issue_qk(s, 0, st);
                    TR(0, nqk, 2);
                    ++nqk;
                }
                for (int t = 0; t < K; ++t) {
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!((act_bits >> s) & 1u)) continue;
                        const bool more = t + 1 < K;
                        uint32_t sv, vp, sk = 0, kp = 0;
                        next_stage(sv, vp);
                        if (more) next_stage(sk, kp);
                        const uint32_t pp = (pf_bits >> s) & 1u;
                        pf_bits ^= 1u << s;
                        TR(0, npv, 3);
                        // non-blocking probe of the group's barriers (test_wait: an incomplete
                        // P_FULL must not put the thread to sleep), then wait for the rest
                        const uint32_t ok = mbar_try_wait4(P_FULL(s), pp, RING_FULL(sv), vp,
                                                           RING_FULL(more ? sk : sv), more ? kp : vp,
                                                           RING_FULL(sv), vp);
                        if (!(ok & 1u)) mbar_wait(P_FULL(s), pp);
                        if (!(ok & 2u)) mbar_wait(RING_FULL(sv), vp);
                        if (more && !(ok & 4u)) mbar_wait(RING_FULL(sk), kp);
                        TR(0, npv, 4);
                        tc_fence_after();
                        issue_pv(s, t, sv);
                        if (more) issue_qk(s, t + 1, sk);
                        TR(0, npv, 5);
                        ++npv;
                    }
                }
            }
        }
        __syncwarp();
    }
    } else {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_SOFTMAX));
#endif
        if (lane == 0) DBG("w%d softmax start\n", warp);
        // ============================ softmax warpgroups ============================
        const int slot = (warp - 4) >> 2;
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const uint32_t tS = tbase + lane_off + slot * 256;
        const uint32_t tO = tS + 128;
        const float sl2 = p.scale_log2;
        uint32_t sf_ph = 0, of_ph = 0;
        for (int r = 0; r < rounds; ++r) {
            const int u = UNIT_OF(r, slot);
            if (u >= total) break;
            const int h = u / NT;
            const int32_t *il = p.idx + (size_t)u * K;
            const uint32_t *mbase = p.slot_mask + (size_t)h * NT * G::MW;
            float m = -INFINITY, l = 0.f;
            int jn = __ldg(il);
            for (int t = 0; t < K; ++t) {
                uint32_t mk[G::MW];
#pragma unroll
                for (int w = 0; w < G::MW; ++w) mk[w] = __ldg(mbase + (size_t)jn * G::MW + w);
                if (t + 1 < K) jn = __ldg(il + t + 1);

                const int trs = r * K + t, trr = 1 + slot * 4 + quarter;  // trace role per softmax warp
                if (lane == 0) TR(trr, trs, 0);
                mbar_wait(S_FULL(slot), sf_ph);
                if (lane == 0) TR(trr, trs, 1);
                sf_ph ^= 1;
                if (lane == 0) DBG("w%d slot%d t%d S ok\n", warp, slot, t);
                tc_fence_after();
                uint32_t sr[B / 32][32];
#pragma unroll
                for (int c = 0; c < B / 32; ++c) tmem_ld32(tS + c * 32, sr[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < B / 32; ++c) reg_fence(sr[c]);
                if (lane == 0) TR(trr, trs, 2);

                bool full = true;
#pragma unroll
                for (int w = 0; w < G::MW; ++w) full &= (mk[w] == 0xFFFFFFFFu);
                if (!full) {
#pragma unroll
                    for (int c = 0; c < B / 32; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!((mk[c] >> i) & 1u)) sr[c][i] = f2u(-INFINITY);
                }
                // row max with 8 independent partial maxima (no 128-long dependency chain)
                float pm[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pm[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < B / 32; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) pm[i & 7] = fmaxf(pm[i & 7], u2f(sr[c][i]));
                const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
                const float mnew = fmaxf(m, mx * sl2);
                if (lane == 0) TR(trr, trs, 3);
                // lazy rescale: only when some row of this warp grew its max by > 8 (log2 units)
                float f = 1.f;
                bool rescale = false;
                if (t == 0) {
                    m = mnew;
                } else if (__any_sync(0xFFFFFFFFu, mnew > m + 8.0f)) {
                    f = (mnew == -INFINITY) ? 1.f : ex2(m - mnew);
                    rescale = true;
                    l *= f;
                    m = mnew;
                }
                const float mu = (m == -INFINITY) ? 0.f : m;
                float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c2 = 0; c2 < B / 64; ++c2) {
                    uint32_t pk[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int c = 2 * c2 + (i >> 4), e = (i & 15) * 2;
                        float x0, x1;
                        ffma2_bc(x0, x1, u2f(sr[c][e]), u2f(sr[c][e + 1]), sl2, -mu);
                        float a, b;
                        if (EMU_EVERY > 0 && (i % EMU_EVERY) == EMU_EVERY - 1) {
                            ex2_emu2(a, b, x0, x1);  // FMA-pipe polynomial: unloads the MUFU unit
                        } else {
                            a = ex2(x0);
                            b = ex2(x1);
                        }
                        fadd2_acc(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, b);
                        pk[i] = pack_bf16(a, b);
                    }
                    tmem_st32(tS + c2 * 32, pk);  // P (bf16 pairs) over S columns already read
                }
                const float ls = (ps[0] + ps[1]) + (ps[2] + ps[3]);
                if (rescale) {  // O is quiescent (see header); scale it before PV_t accumulates
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_wait_ld();
                        reg_fence(o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = f2u(u2f(o[i]) * f);
                        tmem_st32(tO + c * 32, o);
                    }
                }
                l += ls;
                if (lane == 0) TR(trr, trs, 4);
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(P_FULL(slot));
                if (lane == 0) TR(trr, trs, 5);
                if (lane == 0) DBG("w%d slot%d t%d P arrive l=%f m=%f\n", warp, slot, t, l, m);
            }
            // ---- epilogue: O / l -> bf16, padded query rows -> 0
            mbar_wait(O_FULL(slot), of_ph);
            of_ph ^= 1;
            tc_fence_after();
            bool qvalid = false;
            if (row < B) qvalid = (__ldg(p.slot_mask + (size_t)u * G::MW + (row >> 5)) >> (row & 31)) & 1u;
            const float inv = (qvalid && l > 0.f) ? 1.f / l : 0.f;
            uint16_t *orow = p.out + ((size_t)u * B + (row < B ? row : 0)) * D;
            bool store = row < B;
            if (TOK) {  // row -> its token (reading R3); padded query slots have none
                const TileOrigin o = tile_origin(tp, h, u - h * NT);
                const int lpw = __ffs(tp.pw[o.c]) - 1, lphw = lpw + __ffs(tp.ph[o.c]) - 1;
                const int t = o.t0 + (row >> lphw), hq = o.h0 + ((row >> lpw) & (tp.ph[o.c] - 1)),
                          w = o.w0 + (row & (tp.pw[o.c] - 1));
                store = store && qvalid;
                orow = p.out + (size_t)h * tp.o_hs + (((size_t)t * tp.H + hq) * tp.W + w) * tp.o_ts;
            }
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + c * 32, o);
                tmem_wait_ld();
                reg_fence(o);
                if (store) {
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(u2f(o[2 * i]) * inv, u2f(o[2 * i + 1]) * inv);
                    uint4 *dst = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                    for (int v = 0; v < 4; ++v) dst[v] = make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                }
            }
            if (p.lse != nullptr && row < B)
                p.lse[(size_t)u * B + row] = (qvalid && l > 0.f) ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
        }
    }
#undef UNIT_OF
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, TMEM_COLS);
    }
}

// ==========================================================================================
// Half-step schedule ("hs", VEDA_ATTN=hs): each kept key tile is processed as two halves of
// B/2 keys.  Per slot the TMEM holds S for ONE half (B/2 columns), P in two separate
// buffers (B/4 columns each) and O (D columns): 2 x (64 + 64 + 128) = 512 at B = D = 128.
// Because S is free as soon as the softmax has copied it to registers (S_FREE) and P lives
// in its own double buffer, QK of the next half never waits for P V of the current one:
// the MMA issues QK(g+1) during softmax(g), and softmax(g+1) starts as soon as softmax(g)
// ends.  Static MMA order per half-step g: QK(s, g+1) for both slots, then PV(s, g) for both
// slots; ring stages are committed free by the MMA thread (K after its 2nd half's QK, V
// after its 2nd half's PV).  Producer order: K(s,0); then per tile t: V(s,t), K(s,t+1).
// The half-step softmax holds 64 scores per thread (not 128), so registers move from the
// softmax warpgroups to the control warpgroup, whose MMA thread keeps per-slot state for
// both slots (104 + 2 x 200 = 504 per thread slot, as 72 + 2 x 216).
constexpr int REGS_CTRL_HS = 104, REGS_SOFTMAX_HS = 200;

template <int B, int D>
struct GeoHS {
    static constexpr int HB = B / 2;                  // keys per half
    static constexpr int QCHUNK = 128 * 128;
    static constexpr int Q_BYTES = QCHUNK * (D / 64);
    static constexpr int KCHUNK = B * 128;
    static constexpr int TILE_BYTES = KCHUNK * (D / 64);
    static constexpr int NST_FIT = (VEDA_RING_BUDGET_KB * 1024 - NSLOT * Q_BYTES) / TILE_BYTES;
    static constexpr int NST = NST_FIT > 8 ? 8 : NST_FIT;
    static constexpr int MW = B / 32;
    static constexpr int NBAR = 2 * NST + 9 * NSLOT;
    static constexpr int SMEM = NSLOT * Q_BYTES + NST * TILE_BYTES + NBAR * 8 + 16 + 1024;
    // TMEM columns inside a slot's 256
    static constexpr int T_S = 0, T_P0 = 64, T_P1 = 96, T_O = 128;
    static_assert(HB <= 64 && HB / 2 <= 32 && D <= 128, "half-step TMEM layout");
    static_assert(NST >= 3, "ring too shallow");
};

template <int B, int D, bool TOK>
__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_attn_fwd_hs_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                              const __grid_constant__ CUtensorMap tmV, const Params p,
                              const __grid_constant__ TokParams tp)
{
    using G = GeoHS<B, D>;
    constexpr int HB = G::HB;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sRing = sQ + NSLOT * G::Q_BYTES;
    const uint32_t sBar = sRing + G::NST * G::TILE_BYTES;
    uint32_t *tmem_slot =
        reinterpret_cast<uint32_t *>(smem + NSLOT * G::Q_BYTES + G::NST * G::TILE_BYTES + G::NBAR * 8);
#define H_RING_FULL(i) (sBar + 8u * (i))
#define H_RING_EMPTY(i) (sBar + 8u * (G::NST + (i)))
#define H_BAR(k, s) (sBar + 8u * (2 * G::NST + (k) * NSLOT + (s)))
#define H_Q_FULL(s) H_BAR(0, s)
#define H_Q_EMPTY(s) H_BAR(1, s)
#define H_S_FULL(s) H_BAR(2, s)
#define H_S_FREE(s) H_BAR(3, s)
#define H_P_FULL(s, b) H_BAR(4 + (b), s)
#define H_P_EMPTY(s, b) H_BAR(6 + (b), s)
#define H_O_FULL(s) H_BAR(8, s)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (B < 128) {
        uint4 *q4 = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < NSLOT * G::Q_BYTES / 16; i += NTHREADS) q4[i] = make_uint4(0, 0, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G::NST; ++i) {
            mbar_init(H_RING_FULL(i), 1);
            mbar_init(H_RING_EMPTY(i), 1);
        }
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(H_Q_FULL(s), 1);
            mbar_init(H_Q_EMPTY(s), 1);
            mbar_init(H_S_FULL(s), 1);
            mbar_init(H_S_FREE(s), 128);
            mbar_init(H_P_FULL(s, 0), 128);
            mbar_init(H_P_FULL(s, 1), 128);
            mbar_init(H_P_EMPTY(s, 0), 1);
            mbar_init(H_P_EMPTY(s, 1), 1);
            mbar_init(H_O_FULL(s), 1);
        }
        fence_barrier_init();
        if (!TOK) {
            tma_prefetch_desc(&tmQ);
            tma_prefetch_desc(&tmK);
            tma_prefetch_desc(&tmV);
        }
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    const int NT = p.NT, K = p.k, total = p.total_units;
    const int gslots = gridDim.x * NSLOT;
    const int rounds = (total + gslots - 1) / gslots;
#define H_UNIT(r, s) ((r) * gslots + blockIdx.x * NSLOT + (s))

    if (warp < 4) {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS_CTRL_HS));
#endif
        if (warp == 0) {
            // ============================ TMA producer ============================
            if (lane == 0) {
                uint32_t stage = 0, ph = 0, qe_bits = 0;
                auto load_tile = [&](const CUtensorMap *tm, int h, int j) {
                    mbar_wait(H_RING_EMPTY(stage), ph ^ 1);
                    mbar_expect_tx(H_RING_FULL(stage), G::TILE_BYTES);
                    if (TOK)
                        tma_tile_tok<D / 64>(sRing + stage * G::TILE_BYTES, G::KCHUNK, tm == &tmK ? tp.k : tp.v, tp,
                                             h, j, H_RING_FULL(stage));
                    else
#pragma unroll
                        for (int c = 0; c < D / 64; ++c)
                            tma_load_2d(sRing + stage * G::TILE_BYTES + c * G::KCHUNK, tm, c * 64, (h * NT + j) * B,
                                        H_RING_FULL(stage));
                    if (++stage == G::NST) { stage = 0; ph ^= 1; }
                };
                for (int r = 0; r < rounds; ++r) {
                    int u[NSLOT], hh[NSLOT];
                    bool act[NSLOT];
                    const int32_t *il[NSLOT];
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        u[s] = H_UNIT(r, s);
                        act[s] = u[s] < total;
                        hh[s] = act[s] ? u[s] / NT : 0;
                        il[s] = p.idx + (size_t)(act[s] ? u[s] : 0) * K;
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!act[s]) continue;
                        mbar_wait(H_Q_EMPTY(s), ((qe_bits >> s) & 1u) ^ 1u);
                        qe_bits ^= 1u << s;
                        mbar_expect_tx(H_Q_FULL(s), B * D * 2);
                        if (TOK)
                            tma_tile_tok<D / 64>(sQ + s * G::Q_BYTES, G::QCHUNK, tp.q, tp, hh[s], u[s] - hh[s] * NT,
                                                 H_Q_FULL(s));
                        else
                            for (int c = 0; c < D / 64; ++c)
                                tma_load_2d(sQ + s * G::Q_BYTES + c * G::QCHUNK, &tmQ, c * 64, u[s] * B, H_Q_FULL(s));
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s)
                        if (act[s]) load_tile(&tmK, hh[s], __ldg(il[s]));
                    for (int t = 0; t < K; ++t) {
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if (act[s]) load_tile(&tmV, hh[s], __ldg(il[s] + t));
                        if (t + 1 < K)
#pragma unroll
                            for (int s = 0; s < NSLOT; ++s)
                                if (act[s]) load_tile(&tmK, hh[s], __ldg(il[s] + t + 1));
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            // ============================ MMA issuer ============================
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, HB, 0, 0);
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D, 0, 1);
            uint32_t stage = 0, ph = 0, qf_bits = 0;
            uint32_t sfree_cnt[NSLOT] = {0, 0}, pfull_cnt[NSLOT] = {0, 0};
            bool have_prev[NSLOT] = {false, false};  // an un-waited S_FREE of the previous unit's last half
            auto next_stage = [&](uint32_t &st, uint32_t &sp) {
                st = stage;
                sp = ph;
                if (++stage == G::NST) { stage = 0; ph ^= 1; }
            };
            // S(half) = Q K_half^T: keys [half*HB, half*HB + HB) of the tile in stage st
            auto issue_qk = [&](int s, uint32_t st, int half) {
                // shfl from lane 0: lets ptxas treat the operands as warp-uniform (UR registers,
                // MMAs back to back) instead of converting them per MMA
                const uint64_t ad0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sQ + s * G::Q_BYTES, 16, 1024), 0);
                const uint64_t bd0 = __shfl_sync(
                    0xFFFFFFFFu, sdesc_sw128(sRing + st * G::TILE_BYTES + (uint32_t)(half * HB * 128), 16, 1024), 0);
                const uint32_t tS = __shfl_sync(0xFFFFFFFFu, tbase + s * 256 + G::T_S, 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint64_t ao = (uint64_t)(((kk >> 2) * G::QCHUNK + (kk & 3) * 32) >> 4);
                    const uint64_t bo = (uint64_t)(((kk >> 2) * G::KCHUNK + (kk & 3) * 32) >> 4);
                    mma_ss_w(tS, ad0 + ao, bd0 + bo, idesc_qk, kk > 0 ? 1u : 0u);
                }
            };
            // O += P(half) V_half: P from TMEM buffer half&1... (global half parity), V keys of the half
            auto issue_pv = [&](int s, uint32_t st, int half, int pbuf, bool first) {
                const uint64_t vd0 = __shfl_sync(
                    0xFFFFFFFFu,
                    sdesc_sw128(sRing + st * G::TILE_BYTES + (uint32_t)(half * HB * 128), G::KCHUNK, 1024), 0);
                const uint32_t tP = __shfl_sync(0xFFFFFFFFu, tbase + s * 256 + (pbuf ? G::T_P1 : G::T_P0), 0);
                const uint32_t tO = __shfl_sync(0xFFFFFFFFu, tbase + s * 256 + G::T_O, 0);
#pragma unroll
                for (int kk = 0; kk < HB / 16; ++kk)  // 16 keys = 16 rows of 128 B of the V half
                    mma_ts_w(tO, tP + kk * 8, vd0 + (uint64_t)((kk * 2048) >> 4), idesc_pv, (!first || kk > 0) ? 1u : 0u);
            };
            uint32_t kst[NSLOT] = {0, 0}, kph[NSLOT] = {0, 0}, vst[NSLOT] = {0, 0}, vph[NSLOT] = {0, 0};
            for (int r = 0; r < rounds; ++r) {
                uint32_t act = 0;
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) act |= (H_UNIT(r, s) < total ? 1u : 0u) << s;
                // prologue: half 0 of tile 0 (after the previous unit's last S is in registers)
#pragma unroll
                for (int s = 0; s < NSLOT; ++s)
                    if ((act >> s) & 1u) next_stage(kst[s], kph[s]);
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) {
                    if (!((act >> s) & 1u)) continue;
                    if (have_prev[s]) { mbar_wait(H_S_FREE(s), sfree_cnt[s] & 1u); ++sfree_cnt[s]; }
                    mbar_wait(H_Q_FULL(s), (qf_bits >> s) & 1u);
                    qf_bits ^= 1u << s;
                    mbar_wait(H_RING_FULL(kst[s]), kph[s]);
                    tc_fence_after();
                    issue_qk(s, kst[s], 0);
                    tc_commit_w(H_S_FULL(s));
                }
                const int NH = 2 * K;
                for (int g = 0; g < NH; ++g) {
                    const int trs = r * NH + g;
                    if (lane == 0) TR(0, trs, 0);
                    // QK of half g+1 for both slots, once each slot's S(g) is in registers
                    if (g + 1 < NH) {
                        const int hn = (g + 1) & 1, tn = (g + 1) >> 1;
                        (void)tn;
                        if (hn == 0) {
#pragma unroll
                            for (int s = 0; s < NSLOT; ++s)
                                if ((act >> s) & 1u) next_stage(kst[s], kph[s]);
                        }
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s) {
                            if (!((act >> s) & 1u)) continue;
                            mbar_wait(H_S_FREE(s), sfree_cnt[s] & 1u);
                            ++sfree_cnt[s];
                            if (hn == 0) mbar_wait(H_RING_FULL(kst[s]), kph[s]);
                            tc_fence_after();
                            issue_qk(s, kst[s], hn);
                            tc_commit_w(H_S_FULL(s));
                            if (hn == 1) tc_commit_w(H_RING_EMPTY(kst[s]));  // both halves of this K tile issued
                            if (g + 1 == NH - 1) tc_commit_w(H_Q_EMPTY(s));
                        }
                    }
                    if (lane == 0) TR(0, trs, 1);
                    // P V of half g for both slots
                    const int h = g & 1;
                    if (h == 0) {
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if ((act >> s) & 1u) next_stage(vst[s], vph[s]);
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!((act >> s) & 1u)) continue;
                        // one P_FULL per P buffer: a single barrier could complete twice (halves g
                        // and g+1) before this wait, as QK(g+1) is already issued
                        mbar_wait(H_P_FULL(s, pfull_cnt[s] & 1u), (pfull_cnt[s] >> 1) & 1u);
                        ++pfull_cnt[s];
                        if (lane == 0) TR(0, trs, 2 + s);
                        if (h == 0) mbar_wait(H_RING_FULL(vst[s]), vph[s]);
                        tc_fence_after();
                        issue_pv(s, vst[s], h, g & 1, g == 0);
                        tc_commit_w(H_P_EMPTY(s, g & 1));
                        if (h == 1) tc_commit_w(H_RING_EMPTY(vst[s]));  // both halves of this V tile issued
                        if (g == NH - 1) tc_commit_w(H_O_FULL(s));
                    }
                    if (lane == 0) TR(0, trs, 4);
                }
#pragma unroll
                for (int s = 0; s < NSLOT; ++s)
                    if ((act >> s) & 1u) have_prev[s] = true;
            }
            __syncwarp();
        }
    } else {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_SOFTMAX_HS));
#endif
        // ============================ softmax warpgroups ============================
        const int slot = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const uint32_t tSl = tbase + lane_off + slot * 256;
        const uint32_t tS = tSl + G::T_S, tO = tSl + G::T_O;
        const float sl2 = p.scale_log2;
        uint32_t sfull_cnt = 0, gh = 0, of_ph = 0;  // gh: global half counter of this slot
        for (int r = 0; r < rounds; ++r) {
            const int u = H_UNIT(r, slot);
            if (u >= total) break;
            const int h = u / NT;
            const int32_t *il = p.idx + (size_t)u * K;
            const uint32_t *mbase = p.slot_mask + (size_t)h * NT * G::MW;
            float m = -INFINITY, l = 0.f;
            uint32_t mk[G::MW];
            const int NH = 2 * K;
            for (int g = 0; g < NH; ++g, ++gh) {
                const int half = g & 1;
                if (half == 0) {
                    const int j = __ldg(il + (g >> 1));
#pragma unroll
                    for (int w = 0; w < G::MW; ++w) mk[w] = __ldg(mbase + (size_t)j * G::MW + w);
                }
                const int trs = r * NH + g, trr = 1 + slot * 4 + quarter;
                if (lane == 0) TR(trr, trs, 0);
                mbar_wait(H_S_FULL(slot), sfull_cnt & 1u);
                ++sfull_cnt;
                if (lane == 0) TR(trr, trs, 1);
                tc_fence_after();
                uint32_t sr[HB / 32][32];
#pragma unroll
                for (int c = 0; c < HB / 32; ++c) tmem_ld32(tS + c * 32, sr[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < HB / 32; ++c) reg_fence(sr[c]);
                tc_fence_before();
                mbar_arrive(H_S_FREE(slot));  // S may take the next half's QK
                if (lane == 0) TR(trr, trs, 2);
                // padded key slots of this half -> -inf
#pragma unroll
                for (int c = 0; c < HB / 32; ++c) {
                    const uint32_t word = mk[half * (HB / 32) + c];
                    if (word != 0xFFFFFFFFu) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!((word >> i) & 1u)) sr[c][i] = f2u(-INFINITY);
                    }
                }
                float pm[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pm[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < HB / 32; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) pm[i & 7] = fmaxf(pm[i & 7], u2f(sr[c][i]));
                const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
                const float mnew = fmaxf(m, mx * sl2);
                if (g == 0) {
                    m = mnew;
                } else if (__any_sync(0xFFFFFFFFu, mnew > m + 8.0f)) {
                    const float f = (mnew == -INFINITY) ? 1.f : ex2(m - mnew);
                    // O must be quiescent: P V of the previous half complete (its commit covers
                    // every earlier MMA of the issuing thread)
                    const uint32_t pb = (gh - 1) & 1u, n = (gh - 1 - pb) >> 1;
                    mbar_wait(H_P_EMPTY(slot, pb), n & 1u);
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_wait_ld();
                        reg_fence(o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = f2u(u2f(o[i]) * f);
                        tmem_st32(tO + c * 32, o);
                    }
                    l *= f;
                    m = mnew;
                }
                if (lane == 0) TR(trr, trs, 3);
                const float mu = (m == -INFINITY) ? 0.f : m;
                float ps[4] = {0.f, 0.f, 0.f, 0.f};
                uint32_t pk[HB / 2];
#pragma unroll
                for (int i = 0; i < HB / 2; ++i) {
                    const int c = i >> 4, e = (i & 15) * 2;
                    float x0, x1;
                    ffma2_bc(x0, x1, u2f(sr[c][e]), u2f(sr[c][e + 1]), sl2, -mu);
                    const float a = ex2(x0), b2 = ex2(x1);
                    fadd2_acc(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, b2);
                    pk[i] = pack_bf16(a, b2);
                }
                l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
                if (lane == 0) TR(trr, trs, 4);
                // P buffer gh&1 is free once P V of half gh-2 completed
                const uint32_t pbuf = gh & 1u;
                if (gh >= 2) {
                    const uint32_t n = (gh - 2 - pbuf) >> 1;
                    mbar_wait(H_P_EMPTY(slot, pbuf), n & 1u);
                }
                if (lane == 0) TR(trr, trs, 5);
                const uint32_t tP = tSl + (pbuf ? G::T_P1 : G::T_P0);
                if (HB / 2 == 32) {
                    uint32_t (&pk32)[32] = *reinterpret_cast<uint32_t (*)[32]>(pk);
                    tmem_st32(tP, pk32);
                } else {
                    uint32_t (&pk16)[16] = *reinterpret_cast<uint32_t (*)[16]>(pk);
                    tmem_st16(tP, pk16);
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(H_P_FULL(slot, pbuf));
                if (lane == 0) TR(trr, trs, 6);
            }
            // ---- epilogue: O / l -> bf16, padded query rows -> 0
            mbar_wait(H_O_FULL(slot), of_ph);
            of_ph ^= 1;
            tc_fence_after();
            bool qvalid = false;
            if (row < B) qvalid = (__ldg(p.slot_mask + (size_t)u * G::MW + (row >> 5)) >> (row & 31)) & 1u;
            const float inv = (qvalid && l > 0.f) ? 1.f / l : 0.f;
            uint16_t *orow = p.out + ((size_t)u * B + (row < B ? row : 0)) * D;
            bool store = row < B;
            if (TOK) {
                const TileOrigin o = tile_origin(tp, h, u - h * NT);
                const int lpw = __ffs(tp.pw[o.c]) - 1, lphw = lpw + __ffs(tp.ph[o.c]) - 1;
                const int t = o.t0 + (row >> lphw), hq = o.h0 + ((row >> lpw) & (tp.ph[o.c] - 1)),
                          w = o.w0 + (row & (tp.pw[o.c] - 1));
                store = store && qvalid;
                orow = p.out + (size_t)h * tp.o_hs + (((size_t)t * tp.H + hq) * tp.W + w) * tp.o_ts;
            }
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + c * 32, o);
                tmem_wait_ld();
                reg_fence(o);
                if (store) {
                    uint32_t pk2[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) pk2[i] = pack_bf16(u2f(o[2 * i]) * inv, u2f(o[2 * i + 1]) * inv);
                    uint4 *dst = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        dst[v] = make_uint4(pk2[4 * v], pk2[4 * v + 1], pk2[4 * v + 2], pk2[4 * v + 3]);
                }
            }
            if (p.lse != nullptr && row < B)
                p.lse[(size_t)u * B + row] = (qvalid && l > 0.f) ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
        }
    }
#undef H_UNIT
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, TMEM_COLS);
    }
#undef H_RING_FULL
#undef H_RING_EMPTY
#undef H_BAR
#undef H_Q_FULL
#undef H_Q_EMPTY
#undef H_S_FULL
#undef H_S_FREE
#undef H_P_FULL
#undef H_P_EMPTY
#undef H_O_FULL
}

// ==========================================================================================
// P-in-shared-memory schedule ("ps", VEDA_ATTN=ps; B = d = 128): the softmax writes P (bf16,
// the SW128 K-major image a TMA load of a 128x128 tile would produce) to a per-slot shared
// buffer and P V is an SS MMA, so S is free as soon as the softmax has copied it to
// registers: QK(t+1) is issued at S_FREE(t), during softmax(t), instead of after P V(t)
// (the chain of the two-slot kernel).  TMEM per slot: S 128 + O 128 columns.  Shared
// memory: Q 2 x 32 KB + P 2 x 32 KB + a 3-stage K/V ring.  Static MMA order per kept tile t:
// QK(s, t+1) for both slots, then PV(s, t) for both slots; ring stages are committed free by
// the MMA thread.  Producer order: Q, K(s,0); then per tile t: K(s,t+1), V(s,t).
template <int B, int D>
struct GeoPS {
    static constexpr int QCHUNK = 128 * 128;  // 64-column chunk of a 128-row bf16 tile
    static constexpr int Q_BYTES = QCHUNK * (D / 64);
    static constexpr int P_BYTES = QCHUNK * (B / 64);
    static constexpr int KCHUNK = B * 128;
    static constexpr int TILE_BYTES = KCHUNK * (D / 64);
    static constexpr int NST_FIT = (VEDA_RING_BUDGET_KB * 1024 - NSLOT * (Q_BYTES + P_BYTES)) / TILE_BYTES;
    static constexpr int NST = NST_FIT > 8 ? 8 : NST_FIT;
    static constexpr int MW = B / 32;
    static constexpr int NBAR = 2 * NST + 8 * NSLOT;
    static constexpr int SMEM = NSLOT * (Q_BYTES + P_BYTES) + NST * TILE_BYTES + NBAR * 8 + 16 + 1024;
    static_assert(NST >= 3, "ring too shallow");
};

template <int B, int D, bool TOK>
__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_attn_fwd_ps_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                              const __grid_constant__ CUtensorMap tmV, const Params p,
                              const __grid_constant__ TokParams tp)
{
    static_assert(B == 128 && D == 128, "ps schedule: B = d = 128 only");
    using G = GeoPS<B, D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sP = sQ + NSLOT * G::Q_BYTES;
    const uint32_t sRing = sP + NSLOT * G::P_BYTES;
    const uint32_t sBar = sRing + G::NST * G::TILE_BYTES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + NSLOT * (G::Q_BYTES + G::P_BYTES) +
                                                       G::NST * G::TILE_BYTES + G::NBAR * 8);
#define X_RING_FULL(i) (sBar + 8u * (i))
#define X_RING_EMPTY(i) (sBar + 8u * (G::NST + (i)))
#define X_BAR(k, s) (sBar + 8u * (2 * G::NST + (k) * NSLOT + (s)))
#define X_Q_FULL(s) X_BAR(0, s)
#define X_Q_EMPTY(s) X_BAR(1, s)
#define X_S_FULL(s) X_BAR(2, s)
#define X_S_FREE(s) X_BAR(3, s)
#define X_P_FULL(s) X_BAR(4, s)
#define X_P_EMPTY(s) X_BAR(5, s)
#define X_O_FULL(s) X_BAR(6, s)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G::NST; ++i) {
            mbar_init(X_RING_FULL(i), 1);
            mbar_init(X_RING_EMPTY(i), 1);
        }
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(X_Q_FULL(s), 1);
            mbar_init(X_Q_EMPTY(s), 1);
            mbar_init(X_S_FULL(s), 1);
            mbar_init(X_S_FREE(s), 128);
            mbar_init(X_P_FULL(s), 128);
            mbar_init(X_P_EMPTY(s), 1);
            mbar_init(X_O_FULL(s), 1);
        }
        fence_barrier_init();
        if (!TOK) {
            tma_prefetch_desc(&tmQ);
            tma_prefetch_desc(&tmK);
            tma_prefetch_desc(&tmV);
        }
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    const int NT = p.NT, K = p.k, total = p.total_units;
    const int gslots = gridDim.x * NSLOT;
    const int rounds = (total + gslots - 1) / gslots;
#define X_UNIT(r, s) ((r) * gslots + blockIdx.x * NSLOT + (s))

    if (warp < 4) {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS_CTRL));
#endif
        if (warp == 0) {
            // ============================ TMA producer ============================
            if (lane == 0) {
                uint32_t stage = 0, ph = 0, qe_bits = 0;
                auto load_tile = [&](const CUtensorMap *tm, int h, int j) {
                    mbar_wait(X_RING_EMPTY(stage), ph ^ 1);
                    mbar_expect_tx(X_RING_FULL(stage), G::TILE_BYTES);
                    if (TOK)
                        tma_tile_tok<D / 64>(sRing + stage * G::TILE_BYTES, G::KCHUNK, tm == &tmK ? tp.k : tp.v, tp,
                                             h, j, X_RING_FULL(stage));
                    else
#pragma unroll
                        for (int c = 0; c < D / 64; ++c)
                            tma_load_2d(sRing + stage * G::TILE_BYTES + c * G::KCHUNK, tm, c * 64, (h * NT + j) * B,
                                        X_RING_FULL(stage));
                    if (++stage == G::NST) { stage = 0; ph ^= 1; }
                };
                for (int r = 0; r < rounds; ++r) {
                    int u[NSLOT], hh[NSLOT];
                    bool act[NSLOT];
                    const int32_t *il[NSLOT];
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        u[s] = X_UNIT(r, s);
                        act[s] = u[s] < total;
                        hh[s] = act[s] ? u[s] / NT : 0;
                        il[s] = p.idx + (size_t)(act[s] ? u[s] : 0) * K;
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!act[s]) continue;
                        mbar_wait(X_Q_EMPTY(s), ((qe_bits >> s) & 1u) ^ 1u);
                        qe_bits ^= 1u << s;
                        mbar_expect_tx(X_Q_FULL(s), B * D * 2);
                        if (TOK)
                            tma_tile_tok<D / 64>(sQ + s * G::Q_BYTES, G::QCHUNK, tp.q, tp, hh[s], u[s] - hh[s] * NT,
                                                 X_Q_FULL(s));
                        else
                            for (int c = 0; c < D / 64; ++c)
                                tma_load_2d(sQ + s * G::Q_BYTES + c * G::QCHUNK, &tmQ, c * 64, u[s] * B, X_Q_FULL(s));
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s)
                        if (act[s]) load_tile(&tmK, hh[s], __ldg(il[s]));
                    for (int t = 0; t < K; ++t) {
                        if (t + 1 < K)
#pragma unroll
                            for (int s = 0; s < NSLOT; ++s)
                                if (act[s]) load_tile(&tmK, hh[s], __ldg(il[s] + t + 1));
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if (act[s]) load_tile(&tmV, hh[s], __ldg(il[s] + t));
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            // ============================ MMA issuer ============================
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, B, 0, 0);  // Q, K both K-major
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D, 0, 1);  // P K-major (smem), V MN-major
            uint32_t stage = 0, ph = 0, qf_bits = 0;
            uint32_t sfree_cnt[NSLOT] = {0, 0}, pfull_cnt[NSLOT] = {0, 0};
            bool have_prev[NSLOT] = {false, false};
            auto next_stage = [&](uint32_t &st, uint32_t &sp) {
                st = stage;
                sp = ph;
                if (++stage == G::NST) { stage = 0; ph ^= 1; }
            };
            auto issue_qk = [&](int s, uint32_t st) {
                // operands broadcast from lane 0: ptxas keeps them uniform (MMAs back to back)
                const uint64_t ad0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sQ + s * G::Q_BYTES, 16, 1024), 0);
                const uint64_t bd0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sRing + st * G::TILE_BYTES, 16, 1024), 0);
                const uint32_t tS = __shfl_sync(0xFFFFFFFFu, tbase + s * 256, 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint64_t ao = (uint64_t)(((kk >> 2) * G::QCHUNK + (kk & 3) * 32) >> 4);
                    const uint64_t bo = (uint64_t)(((kk >> 2) * G::KCHUNK + (kk & 3) * 32) >> 4);
                    mma_ss_w(tS, ad0 + ao, bd0 + bo, idesc_qk, kk > 0 ? 1u : 0u);
                }
            };
            auto issue_pv = [&](int s, uint32_t st, bool first) {
                const uint64_t pd0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sP + s * G::P_BYTES, 16, 1024), 0);
                const uint64_t vd0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sRing + st * G::TILE_BYTES, G::KCHUNK, 1024), 0);
                const uint32_t tO = __shfl_sync(0xFFFFFFFFu, tbase + s * 256 + 128, 0);
#pragma unroll
                for (int kk = 0; kk < B / 16; ++kk) {
                    const uint64_t ao = (uint64_t)(((kk >> 2) * G::QCHUNK + (kk & 3) * 32) >> 4);
                    mma_ss_w(tO, pd0 + ao, vd0 + (uint64_t)((kk * 2048) >> 4), idesc_pv, (!first || kk > 0) ? 1u : 0u);
                }
            };
            uint32_t kst[NSLOT] = {0, 0}, kph[NSLOT] = {0, 0}, vst[NSLOT] = {0, 0}, vph[NSLOT] = {0, 0};
            for (int r = 0; r < rounds; ++r) {
                uint32_t act = 0;
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) act |= (X_UNIT(r, s) < total ? 1u : 0u) << s;
#pragma unroll
                for (int s = 0; s < NSLOT; ++s)
                    if ((act >> s) & 1u) next_stage(kst[s], kph[s]);
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) {
                    if (!((act >> s) & 1u)) continue;
                    if (have_prev[s]) { mbar_wait(X_S_FREE(s), sfree_cnt[s] & 1u); ++sfree_cnt[s]; }
                    mbar_wait(X_Q_FULL(s), (qf_bits >> s) & 1u);
                    qf_bits ^= 1u << s;
                    mbar_wait(X_RING_FULL(kst[s]), kph[s]);
                    tc_fence_after();
                    issue_qk(s, kst[s]);
                    tc_commit_w(X_S_FULL(s));
                    tc_commit_w(X_RING_EMPTY(kst[s]));
                    if (K == 1) tc_commit_w(X_Q_EMPTY(s));
                }
                for (int t = 0; t < K; ++t) {
                    if (lane == 0) TR(0, r * K + t, 0);
                    if (t + 1 < K) {
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if ((act >> s) & 1u) next_stage(kst[s], kph[s]);
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s) {
                            if (!((act >> s) & 1u)) continue;
                            mbar_wait(X_S_FREE(s), sfree_cnt[s] & 1u);  // S(t) is in registers
                            ++sfree_cnt[s];
                            mbar_wait(X_RING_FULL(kst[s]), kph[s]);
                            tc_fence_after();
                            issue_qk(s, kst[s]);
                            tc_commit_w(X_S_FULL(s));
                            tc_commit_w(X_RING_EMPTY(kst[s]));
                            if (t + 1 == K - 1) tc_commit_w(X_Q_EMPTY(s));
                        }
                    }
                    if (lane == 0) TR(0, r * K + t, 1);
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s)
                        if ((act >> s) & 1u) next_stage(vst[s], vph[s]);
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!((act >> s) & 1u)) continue;
                        mbar_wait(X_P_FULL(s), pfull_cnt[s] & 1u);
                        ++pfull_cnt[s];
                        if (lane == 0) TR(0, r * K + t, 2 + s);
                        mbar_wait(X_RING_FULL(vst[s]), vph[s]);
                        if (lane == 0) TR(0, r * K + t, 4 + s);
                        tc_fence_after();
                        issue_pv(s, vst[s], t == 0);
                        tc_commit_w(X_P_EMPTY(s));
                        tc_commit_w(X_RING_EMPTY(vst[s]));
                        if (t == K - 1) tc_commit_w(X_O_FULL(s));
                    }
                }
#pragma unroll
                for (int s = 0; s < NSLOT; ++s)
                    if ((act >> s) & 1u) have_prev[s] = true;
            }
            __syncwarp();
        }
    } else {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_SOFTMAX));
#endif
        // ============================ softmax warpgroups ============================
        const int slot = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const uint32_t tS = tbase + lane_off + slot * 256, tO = tS + 128;
        // this row's 128-byte lines in the two 64-key chunks of the P buffer (SW128: 16-byte
        // unit c of row r sits at unit c ^ (r & 7))
        const uint32_t pRow = sP + slot * G::P_BYTES + row * 128;
        const float sl2 = p.scale_log2;
        uint32_t sfull_cnt = 0, g = 0, of_ph = 0;  // g: this slot's global kept-tile counter
        for (int r = 0; r < rounds; ++r) {
            const int u = X_UNIT(r, slot);
            if (u >= total) break;
            const int h = u / NT;
            const int32_t *il = p.idx + (size_t)u * K;
            const uint32_t *mbase = p.slot_mask + (size_t)h * NT * G::MW;
            float m = -INFINITY, l = 0.f;
            for (int t = 0; t < K; ++t, ++g) {
                const int j = __ldg(il + t);
                uint32_t mk[G::MW];
#pragma unroll
                for (int w = 0; w < G::MW; ++w) mk[w] = __ldg(mbase + (size_t)j * G::MW + w);
                const int trs = r * K + t, trr = 1 + slot * 4 + quarter;
                if (lane == 0) TR(trr, trs, 0);
                mbar_wait(X_S_FULL(slot), sfull_cnt & 1u);
                ++sfull_cnt;
                if (lane == 0) TR(trr, trs, 1);
                tc_fence_after();
                uint32_t sr[B / 32][32];
#pragma unroll
                for (int c = 0; c < B / 32; ++c) tmem_ld32(tS + c * 32, sr[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < B / 32; ++c) reg_fence(sr[c]);
                tc_fence_before();
                mbar_arrive(X_S_FREE(slot));  // S may take QK(t+1)
                if (lane == 0) TR(trr, trs, 2);
                bool full = true;
#pragma unroll
                for (int w = 0; w < G::MW; ++w) full &= (mk[w] == 0xFFFFFFFFu);
                if (!full) {
#pragma unroll
                    for (int c = 0; c < B / 32; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!((mk[c] >> i) & 1u)) sr[c][i] = f2u(-INFINITY);
                }
                float pm[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pm[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < B / 32; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) pm[i & 7] = fmaxf(pm[i & 7], u2f(sr[c][i]));
                const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
                const float mnew = fmaxf(m, mx * sl2);
                // P buffer and O are both quiescent once P V(t-1) completed (P_EMPTY phase g-1)
                if (g > 0) {
                    mbar_wait(X_P_EMPTY(slot), (g - 1) & 1u);
                    tc_fence_after();
                }
                if (lane == 0) TR(trr, trs, 3);
                bool rescale = false;
                if (t == 0) {
                    m = mnew;
                } else if (__any_sync(0xFFFFFFFFu, mnew > m + 8.0f)) {
                    const float f = (mnew == -INFINITY) ? 1.f : ex2(m - mnew);
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_wait_ld();
                        reg_fence(o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = f2u(u2f(o[i]) * f);
                        tmem_st32(tO + c * 32, o);
                    }
                    rescale = true;
                    l *= f;
                    m = mnew;
                }
                const float mu = (m == -INFINITY) ? 0.f : m;
                float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c2 = 0; c2 < B / 64; ++c2) {
                    uint32_t pk[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int c = 2 * c2 + (i >> 4), e = (i & 15) * 2;
                        float x0, x1;
                        ffma2_bc(x0, x1, u2f(sr[c][e]), u2f(sr[c][e + 1]), sl2, -mu);
                        const float a = ex2(x0), b = ex2(x1);
                        fadd2_acc(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, b);
                        pk[i] = pack_bf16(a, b);
                    }
                    // keys 64*c2 .. 64*c2+63: eight 16-byte units of this row's line in chunk c2
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        const uint32_t addr = pRow + c2 * G::QCHUNK + (uint32_t)(((v ^ (row & 7)) & 7) << 4);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * v]),
                                     "r"(pk[4 * v + 1]), "r"(pk[4 * v + 2]), "r"(pk[4 * v + 3])
                                     : "memory");
                    }
                }
                l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
                if (lane == 0) TR(trr, trs, 4);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P visible to the MMA
                if (rescale) tmem_wait_st();
                tc_fence_before();
                mbar_arrive(X_P_FULL(slot));
                if (lane == 0) TR(trr, trs, 5);
            }
            // ---- epilogue: O / l -> bf16, padded query rows -> 0
            mbar_wait(X_O_FULL(slot), of_ph);
            of_ph ^= 1;
            tc_fence_after();
            bool qvalid = false;
            if (row < B) qvalid = (__ldg(p.slot_mask + (size_t)u * G::MW + (row >> 5)) >> (row & 31)) & 1u;
            const float inv = (qvalid && l > 0.f) ? 1.f / l : 0.f;
            uint16_t *orow = p.out + ((size_t)u * B + (row < B ? row : 0)) * D;
            bool store = row < B;
            if (TOK) {
                const TileOrigin o = tile_origin(tp, h, u - h * NT);
                const int lpw = __ffs(tp.pw[o.c]) - 1, lphw = lpw + __ffs(tp.ph[o.c]) - 1;
                const int t = o.t0 + (row >> lphw), hq = o.h0 + ((row >> lpw) & (tp.ph[o.c] - 1)),
                          w = o.w0 + (row & (tp.pw[o.c] - 1));
                store = store && qvalid;
                orow = p.out + (size_t)h * tp.o_hs + (((size_t)t * tp.H + hq) * tp.W + w) * tp.o_ts;
            }
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + c * 32, o);
                tmem_wait_ld();
                reg_fence(o);
                if (store) {
                    uint32_t pk2[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) pk2[i] = pack_bf16(u2f(o[2 * i]) * inv, u2f(o[2 * i + 1]) * inv);
                    uint4 *dst = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        dst[v] = make_uint4(pk2[4 * v], pk2[4 * v + 1], pk2[4 * v + 2], pk2[4 * v + 3]);
                }
            }
            if (p.lse != nullptr && row < B)
                p.lse[(size_t)u * B + row] = (qvalid && l > 0.f) ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
        }
    }
#undef X_UNIT
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, TMEM_COLS);
    }
#undef X_RING_FULL
#undef X_RING_EMPTY
#undef X_BAR
#undef X_Q_FULL
#undef X_Q_EMPTY
#undef X_S_FULL
#undef X_S_FREE
#undef X_P_FULL
#undef X_P_EMPTY
#undef X_O_FULL
}

static unsigned long long *g_attn_trace = nullptr;

template <int B, int D, bool TOK>
static veda_status launch_kernel(const CUtensorMap &mq, const CUtensorMap &mk, const CUtensorMap &mv, const Params &p,
                                 const TokParams &tp, int units, cudaStream_t stream)
{
    using G = Geo<B, D>;
    using GH = GeoHS<B, D>;
    static const bool hs = [] {
        const char *e = getenv("VEDA_ATTN");
        return e && e[0] == 'h' && e[1] == 's';
    }();
    static const bool ps = [] {
        const char *e = getenv("VEDA_ATTN");
        return e && e[0] == 'p' && e[1] == 's';
    }();
    if constexpr (B == 128 && D == 128) {
        if (ps) {
            using GP = GeoPS<B, D>;
            static bool attr_ps = false;
            if (!attr_ps) {
                cudaError_t e = cudaFuncSetAttribute(sparse_attn_fwd_ps_kernel<B, D, TOK>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, GP::SMEM);
                if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
                attr_ps = true;
            }
            int grid = (units + NSLOT - 1) / NSLOT;
            const int nsm = num_sms();
            if (grid > nsm) grid = nsm;
            sparse_attn_fwd_ps_kernel<B, D, TOK><<<grid, NTHREADS, GP::SMEM, stream>>>(mq, mk, mv, p, tp);
            count_launch();
            return check_launch("sparse_attn_fwd (ps)");
        }
    }
    static bool attr_set = false;  // per instantiation
    if (!attr_set) {
        cudaError_t e = hs ? cudaFuncSetAttribute(sparse_attn_fwd_hs_kernel<B, D, TOK>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, GH::SMEM)
                           : cudaFuncSetAttribute(sparse_attn_fwd_kernel<B, D, TOK>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        attr_set = true;
    }
    int grid = (units + NSLOT - 1) / NSLOT;
    const int nsm = num_sms();
    if (grid > nsm) grid = nsm;
    if (hs)
        sparse_attn_fwd_hs_kernel<B, D, TOK><<<grid, NTHREADS, GH::SMEM, stream>>>(mq, mk, mv, p, tp);
    else
        sparse_attn_fwd_kernel<B, D, TOK><<<grid, NTHREADS, G::SMEM, stream>>>(mq, mk, mv, p, tp);
    count_launch();
    return check_launch("sparse_attn_fwd");
}

static Params make_params(const int32_t *idx, const uint32_t *mask, uint16_t *o, float *lse, int Hh, int NT, int kk,
                          float scale)
{
    Params p;
    p.idx = idx;
    p.slot_mask = mask;
    p.out = o;
    p.lse = lse;
    p.NT = NT;
    p.k = kk;
    p.total_units = Hh * NT;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.trace = g_attn_trace;
    return p;
}

template <int B, int D>
static veda_status launch(const uint16_t *q, const uint16_t *k, const uint16_t *v, const int32_t *idx,
                          const uint32_t *mask, int Hh, int NT, int kk, float scale, uint16_t *o,
                          float *lse, cudaStream_t stream)
{
    CUtensorMap mq, mk, mv;
    const uint64_t rows = (uint64_t)Hh * NT * B;
    veda_status st;
    if ((st = make_tmap_bf16(&mq, q, rows, D, B)) != VEDA_OK) return st;
    if ((st = make_tmap_bf16(&mk, k, rows, D, B)) != VEDA_OK) return st;
    if ((st = make_tmap_bf16(&mv, v, rows, D, B)) != VEDA_OK) return st;
    static TokParams tp_unused;  // zero-initialised; the tiled instantiation never reads it
    return launch_kernel<B, D, false>(mq, mk, mv, make_params(idx, mask, o, lse, Hh, NT, kk, scale), tp_unused,
                                      Hh * NT, stream);
}

// Token-layout launch: heads are split into consecutive groups with at most MAXC distinct
// tile shapes; each group is one launch on pointers offset to its first head.
template <int B, int D>
static veda_status launch_tok(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t hs, int64_t ts,
                              const HeadCfgs &cf, int Hh, int Hp, int Wp, int T, int H, int W, int NT,
                              const int32_t *idx, const uint32_t *mask, int kk, float scale, uint16_t *o,
                              int64_t o_hs, int64_t o_ts, float *lse, cudaStream_t stream)
{
    static TokParams tp;  // host staging (3-4 KB): filled per launch, passed by value
    CUtensorMap dummy;
    memset(&dummy, 0, sizeof dummy);
    const int MW = B / 32;
    for (int h0 = 0; h0 < Hh;) {
        int nc = 0, h1 = h0;
        for (; h1 < Hh; ++h1) {
            int c = 0;
            while (c < nc && !(tp.pt[c] == cf.pt[h1] && tp.ph[c] == cf.ph[h1] && tp.pw[c] == cf.pw[h1])) ++c;
            if (c == nc) {
                if (nc == MAXC) break;
                tp.pt[c] = cf.pt[h1]; tp.ph[c] = cf.ph[h1]; tp.pw[c] = cf.pw[h1];
                ++nc;
            }
            tp.cid[h1 - h0] = (uint8_t)c;
        }
        const int hn = h1 - h0;
        veda_status st;
        int tm = 0;
        for (int c = 0; c < nc; ++c) {
            if ((st = make_tmap_tile_tokens(&tp.q[c], q + (size_t)h0 * hs, hs, ts, hn, T, H, W, D, tp.pt[c], tp.ph[c],
                                            tp.pw[c], &tm)) != VEDA_OK ||
                (st = make_tmap_tile_tokens(&tp.k[c], k + (size_t)h0 * hs, hs, ts, hn, T, H, W, D, tp.pt[c], tp.ph[c],
                                            tp.pw[c], &tm)) != VEDA_OK ||
                (st = make_tmap_tile_tokens(&tp.v[c], v + (size_t)h0 * hs, hs, ts, hn, T, H, W, D, tp.pt[c], tp.ph[c],
                                            tp.pw[c], &tm)) != VEDA_OK)
                return st;
        }
        for (int c = 0; c < nc; ++c) {
            tp.nbw[c] = (uint32_t)(Wp / tp.pw[c]);
            tp.nbhw[c] = (uint32_t)((Hp / tp.ph[c]) * (Wp / tp.pw[c]));
            auto magic = [](uint32_t n) {  // ceil(2^32 / n), saturated for n = 1 (div_magic corrects by one)
                const unsigned long long m = (0x100000000ull + n - 1) / n;
                return (uint32_t)(m > 0xFFFFFFFFull ? 0xFFFFFFFFull : m);
            };
            tp.mbw[c] = magic(tp.nbw[c]);
            tp.mbhw[c] = magic(tp.nbhw[c]);
        }
        tp.T = T; tp.H = H; tp.W = W; tp.Hp = Hp; tp.Wp = Wp;
        tp.tok_major = tm;
        tp.o_hs = o_hs;
        tp.o_ts = o_ts;
        const Params p = make_params(idx + (size_t)h0 * NT * kk, mask + (size_t)h0 * NT * MW, o + (size_t)h0 * o_hs,
                                     lse ? lse + (size_t)h0 * NT * B : nullptr, hn, NT, kk, scale);
        if ((st = launch_kernel<B, D, true>(dummy, dummy, dummy, p, tp, hn * NT, stream)) != VEDA_OK) return st;
        h0 = h1;
    }
    return VEDA_OK;
}

}  // namespace attn

#ifdef VEDA_ATTN_TRACE
extern "C" __attribute__((visibility("default"))) void veda_dbg_set_attn_trace(void *dev_buf)
{
    attn::g_attn_trace = static_cast<unsigned long long *>(dev_buf);
}
#endif

veda_status launch_sparse_attn(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                               const int32_t *idx, const uint32_t *mask, int Hh, int NT, int B, int d,
                               int kk, float scale, uint16_t *o, float *lse, cudaStream_t s)
{
    static const int sched = [] {
        const char *e = getenv("VEDA_ATTN");
        return (e && e[0] == '1' && e[1] == 'q') ? 1 : 0;
    }();
    if (sched == 1) return launch_sparse_attn_1q(q, k, v, idx, mask, Hh, NT, B, d, kk, scale, o, lse, s);
    if (B == 128 && d == 128) return attn::launch<128, 128>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    if (B == 128 && d == 64) return attn::launch<128, 64>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    if (B == 64 && d == 128) return attn::launch<64, 128>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    if (B == 64 && d == 64) return attn::launch<64, 64>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    return fail(VEDA_ERR_CONFIG, "sparse_attn_fwd: unsupported (B=%d, d=%d)", B, d);
}

veda_status launch_sparse_attn_tok(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t hs, int64_t ts,
                                   const HeadCfgs &cf, int Hh, int Tp, int Hp, int Wp, int T, int H, int W, int B,
                                   int NT, int d, const int32_t *idx, const uint32_t *mask, int kk, float scale,
                                   uint16_t *o, int64_t o_hs, int64_t o_ts, float *lse, cudaStream_t s)
{
    (void)Tp;
    // a stride that is never used (one token, or one head) may equal the other one; give it
    // a distinct value so the 5-D tensor maps get a well-ordered dimension set
    if (hs == ts) {
        if ((int64_t)T * H * W == 1)
            ts = hs * Hh;
        else if (Hh == 1)
            hs = ts * ((int64_t)T * H * W);
        else
            return fail(VEDA_ERR_ALIGN, "sparse_attn_fwd_tokens: head_stride == token_stride");
    }
#define VEDA_TOK_ARGS q, k, v, hs, ts, cf, Hh, Hp, Wp, T, H, W, NT, idx, mask, kk, scale, o, o_hs, o_ts, lse, s
    if (B == 128 && d == 128) return attn::launch_tok<128, 128>(VEDA_TOK_ARGS);
    if (B == 128 && d == 64) return attn::launch_tok<128, 64>(VEDA_TOK_ARGS);
    if (B == 64 && d == 128) return attn::launch_tok<64, 128>(VEDA_TOK_ARGS);
    if (B == 64 && d == 64) return attn::launch_tok<64, 64>(VEDA_TOK_ARGS);
#undef VEDA_TOK_ARGS
    return fail(VEDA_ERR_CONFIG, "sparse_attn_fwd_tokens: unsupported (B=%d, d=%d)", B, d);
}

}  // namespace veda
