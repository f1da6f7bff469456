// attn_fwd_1q.cu -- tile-skipping FlashAttention forward, one query tile per CTA with a
// double-buffered S (the "1q" schedule).  Same contract as attn_fwd.cu (Eq. 2,
// PAPER.md:150-157; producer fetches only the kept K/V tiles).
//
// Why a second schedule: in the two-slot kernel P aliases S in TMEM, so for each query tile
// the chain QK(t+1) -> softmax(t+1) cannot start before PV(t) has consumed P(t); the per-slot
// period is softmax + MMA, and two slots only partly hide it (profiles/r01_attn_experiments.md).
// Here TMEM (512 columns) holds, for ONE query tile,
//     S0 [0,128)  S1 [128,256)  P0 [256,320)  P1 [320,384)  O [384,512)
// so QK(t+1) runs while the softmax works on S(t), and the MMA pipe only waits for P(t).
// The per-tile period becomes max(MMA, softmax) instead of their sum.
//
//   warp 0      TMA producer (Q double-buffered, K/V ring in MMA consumption order)
//   warp 1      MMA issuer: flat over this CTA's tiles g: QK(g+1), then PV(g)
//   warps 4-11  softmax: warp (quarter q, half c) owns TMEM lanes 32q..32q+31 and key
//               columns [c*B/2, (c+1)*B/2) of S, P columns likewise, O columns [c*D/2, ...)
//               The two halves of a row exchange their row max through SMEM (named
//               barrier of the two warps of a quarter); row sums are combined at the end.
// Online softmax in the log2 domain with lazy rescale (threshold 8): rescaling O waits for
// the previous PV (O_DONE), which is rare.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "sm100.cuh"

namespace veda {
namespace attn1q {
using namespace sm100;

constexpr int NTHREADS = 384;
constexpr int REGS_CTRL = 72;
constexpr int REGS_SOFTMAX = 216;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t COL_S = 0, COL_P = 256, COL_O = 384;

struct Params {
    const int32_t *idx;
    const uint32_t *slot_mask;
    uint16_t *out;
    float *lse;
    int NT, k, total_units;
    float scale_log2;
    unsigned long long *trace;  // VEDA_ATTN_TRACE builds only: clock64 stamps of CTA 0
};

#ifdef VEDA_ATTN_TRACE
#define TR(role, step, field)                                                              \
    do {                                                                                   \
        if (blockIdx.x == 0 && (step) < 256 && p.trace)                                    \
            p.trace[((role) * 256 + (step)) * 8 + (field)] = clock64();                   \
    } while (0)
#else
#define TR(role, step, field) do { } while (0)
#endif

#ifndef VEDA_RING_BUDGET_KB
#define VEDA_RING_BUDGET_KB 224
#endif

template <int B, int D>
struct Geo {
    static constexpr int QCHUNK = 128 * 128;
    static constexpr int Q_BYTES = QCHUNK * (D / 64);
    static constexpr int KCHUNK = B * 128;
    static constexpr int TILE_BYTES = KCHUNK * (D / 64);
    static constexpr int NST_FIT = (VEDA_RING_BUDGET_KB * 1024 - 2 * Q_BYTES - 4096) / TILE_BYTES;
    static constexpr int NST = NST_FIT > 10 ? 10 : NST_FIT;
    static constexpr int MW = B / 32;
    static constexpr int CW = B / 2;   // S columns per half
    static constexpr int PW = B / 4;   // packed P columns per half
    static constexpr int OW = D / 2;   // O columns per half
    // barriers: ring full/empty, Q full/empty x2, S full/free x2, P full x2, O done, O free
    static constexpr int NBAR = 2 * NST + 4 + 4 + 2 + 2;
    static constexpr int XBYTES = (2 * 2 * 128 + 2 * 128) * 4;  // row-max exchange + row-sum exchange
    static constexpr int SMEM = 2 * Q_BYTES + NST * TILE_BYTES + NBAR * 8 + 16 + XBYTES + 1024;
    static_assert(NST >= 3, "ring too shallow");
};

__device__ __forceinline__ float u2f(uint32_t u) { return __uint_as_float(u); }
__device__ __forceinline__ uint32_t f2u(float f) { return __float_as_uint(f); }

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
__device__ __forceinline__ void named_bar(int id, int n)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Fraction of exp2 evaluated on the FMA pipe instead of MUFU: one pair in every EMU_EVERY
// (0 disables).  MUFU.EX2 (16/clk/SM) needs exactly the MMA time of a tile; moving some
// exponentials to the FMA pipe takes the softmax below that bound.
#ifndef VEDA_1Q_EMU_EVERY
#define VEDA_1Q_EMU_EVERY 0  // measured: 1/8 and 1/4 are slower (profiles/r01_attn_experiments.md)
#endif

// 2^x for x <= ~8 by 2^n * p(f), f in [-1/2, 1/2], cubic p (max rel. error 7.5e-5, far
// below the bf16 rounding of P, 2^-9)
__device__ __forceinline__ float ex2_emu(float x)
{
    x = fmaxf(x, -125.0f);
    const float j = x + 12582912.0f;
    const float f = x - (j - 12582912.0f);
    float p = fmaf(f, 0.05517162f, 0.24261113f);
    p = fmaf(p, f, 0.69326097f);
    p = fmaf(p, f, 0.99992806f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(j) << 23));
}

template <int CW>
__device__ __forceinline__ float row_max(const uint32_t (&sr)[CW / 32][32])
{
    float pm[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) pm[q] = -INFINITY;
#pragma unroll
    for (int c = 0; c < CW / 32; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) pm[i & 7] = fmaxf(pm[i & 7], u2f(sr[c][i]));
    return fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
}

// P = 2^(s*sl2 - mu) for this thread's CW scores -> bf16 pairs in TMEM at tP; returns the
// fp32 sum of the exponentials; with TRACK also the raw row max of s (in the same pass).
template <int CW, bool TRACK>
__device__ __forceinline__ float exp_store(const uint32_t (&sr)[CW / 32][32], float sl2, float mu, uint32_t tP,
                                           float &mx_out)
{
    float ps[4] = {0.f, 0.f, 0.f, 0.f};
    float pm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int c2 = 0; c2 < CW / 32; ++c2) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int e = c2 * 32 + 2 * i;
            const float s0 = u2f(sr[e >> 5][e & 31]), s1 = u2f(sr[e >> 5][(e & 31) + 1]);
            if (TRACK) pm[i & 3] = fmaxf(pm[i & 3], fmaxf(s0, s1));
            float x0, x1;
            ffma2_bc(x0, x1, s0, s1, sl2, -mu);
            float a, b;
            if (VEDA_1Q_EMU_EVERY > 0 && (i % VEDA_1Q_EMU_EVERY) == VEDA_1Q_EMU_EVERY - 1) {
                a = ex2_emu(x0);
                b = ex2_emu(x1);
            } else {
                a = ex2(x0);
                b = ex2(x1);
            }
            fadd2_acc(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, b);
            pk[i] = pack_bf16(a, b);
        }
        tmem_st16(tP + c2 * 16, pk);
    }
    if (TRACK) mx_out = fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3]));
    return (ps[0] + ps[1]) + (ps[2] + ps[3]);
}

template <int B, int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_1q_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const Params p)
{
    using G = Geo<B, D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sRing = sQ + 2 * G::Q_BYTES;
    const uint32_t sBar = sRing + G::NST * G::TILE_BYTES;
    uint8_t *tail = smem + 2 * G::Q_BYTES + G::NST * G::TILE_BYTES + G::NBAR * 8;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tail);
    float *xmax = reinterpret_cast<float *>(tail + 16);  // [2 parity][2 half][128 rows]
    float *xsum = xmax + 2 * 2 * 128;                    // [2 half][128 rows]
#define RING_FULL(i) (sBar + 8u * (i))
#define RING_EMPTY(i) (sBar + 8u * (G::NST + (i)))
#define Q_FULL(b) (sBar + 8u * (2 * G::NST + (b)))
#define Q_EMPTY(b) (sBar + 8u * (2 * G::NST + 2 + (b)))
#define S_FULL(b) (sBar + 8u * (2 * G::NST + 4 + (b)))
#define S_FREE(b) (sBar + 8u * (2 * G::NST + 6 + (b)))
#define P_FULL(b) (sBar + 8u * (2 * G::NST + 8 + (b)))
#define O_DONE (sBar + 8u * (2 * G::NST + 10))
#define O_FREE (sBar + 8u * (2 * G::NST + 11))

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (B < 128) {
        uint4 *q4 = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < 2 * G::Q_BYTES / 16; i += NTHREADS) q4[i] = make_uint4(0, 0, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G::NST; ++i) {
            mbar_init(RING_FULL(i), 1);
            mbar_init(RING_EMPTY(i), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(Q_FULL(b), 1);
            mbar_init(Q_EMPTY(b), 1);
            mbar_init(S_FULL(b), 1);
            mbar_init(S_FREE(b), 8);
            mbar_init(P_FULL(b), 8);
        }
        mbar_init(O_DONE, 1);
        mbar_init(O_FREE, 8);
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
    const int my_units = blockIdx.x < total ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    const int64_t G_tiles = (int64_t)my_units * K;
#define UNIT_OF(r) ((r) * (int)gridDim.x + (int)blockIdx.x)

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS_CTRL));
        if (warp == 0 && lane == 0) {
            // ============================ TMA producer ============================
            // ring order = MMA consumption order: K(0), then per g: K(g+1), V(g)
            uint32_t stage = 0, ph = 0;
            int nload = 0;
            auto load_tile = [&](const CUtensorMap *tm, int u, int j) {
                TR(3, nload, 0);
                mbar_wait(RING_EMPTY(stage), ph ^ 1);
                TR(3, nload, 1);
                ++nload;
                mbar_expect_tx(RING_FULL(stage), G::TILE_BYTES);
                const int row = ((u / NT) * NT + j) * B;
#pragma unroll
                for (int c = 0; c < D / 64; ++c)
                    tma_load_2d(sRing + stage * G::TILE_BYTES + c * G::KCHUNK, tm, c * 64, row, RING_FULL(stage));
                if (++stage == G::NST) { stage = 0; ph ^= 1; }
            };
            auto load_q = [&](int r) {
                const int qb = r & 1;
                mbar_wait(Q_EMPTY(qb), ((r >> 1) & 1) ^ 1);
                mbar_expect_tx(Q_FULL(qb), B * D * 2);
#pragma unroll
                for (int c = 0; c < D / 64; ++c)
                    tma_load_2d(sQ + qb * G::Q_BYTES + c * G::QCHUNK, &tmQ, c * 64, UNIT_OF(r) * B, Q_FULL(qb));
            };
            if (G_tiles > 0) {
                load_q(0);
                load_tile(&tmK, UNIT_OF(0), __ldg(p.idx + (size_t)UNIT_OF(0) * K));
                int r = 0, t = 0;
                for (int64_t g = 0; g < G_tiles; ++g) {
                    const int u = UNIT_OF(r);
                    const int r1 = (t + 1 < K) ? r : r + 1, t1 = (t + 1 < K) ? t + 1 : 0;
                    if (g + 1 < G_tiles) {
                        const int u1 = UNIT_OF(r1);
                        if (t1 == 0) load_q(r1);
                        load_tile(&tmK, u1, __ldg(p.idx + (size_t)u1 * K + t1));
                    }
                    load_tile(&tmV, u, __ldg(p.idx + (size_t)u * K + t));
                    r = r1;
                    t = t1;
                }
            }
        } else if (warp == 1) {
            // ============================ MMA issuer ============================
            // The whole warp runs this loop (warp-uniform values); one lane issues each
            // tcgen05 instruction via elect.sync.  Descriptors are built once per tile and
            // advanced by constant offsets (the 14-bit address field never carries).
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, B, 0, 0);
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D, 0, 1);
            uint32_t stage = 0, ph = 0;
            auto take = [&](uint32_t &st, uint32_t &sp) {
                st = stage;
                sp = ph;
                if (++stage == G::NST) { stage = 0; ph ^= 1; }
            };
            // QK(g) into S[g&1]: Q buffer r&1, K in ring stage st
            auto mma_qk = [&](int64_t g, int r, int t, uint32_t st) {
                tc_fence_after();
                const uint64_t ad0 = sdesc_sw128(sQ + (r & 1) * G::Q_BYTES, 16, 1024);
                const uint64_t bd0 = sdesc_sw128(sRing + st * G::TILE_BYTES, 16, 1024);
                const uint32_t dS = tbase + COL_S + (uint32_t)(g & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint64_t ao = (uint64_t)(((kk >> 2) * G::QCHUNK + (kk & 3) * 32) >> 4);
                    const uint64_t bo = (uint64_t)(((kk >> 2) * G::KCHUNK + (kk & 3) * 32) >> 4);
                    mma_ss_w(dS, ad0 + ao, bd0 + bo, idesc_qk, kk > 0 ? 1u : 0u);
                }
                tc_commit_w(S_FULL((uint32_t)(g & 1)));
                tc_commit_w(RING_EMPTY(st));
                if (t == K - 1) tc_commit_w(Q_EMPTY(r & 1));
            };
            // O += P[g&1] V with V in ring stage st
            auto mma_pv = [&](int64_t g, int t, uint32_t st) {
                tc_fence_after();
                const uint64_t vd0 = sdesc_sw128(sRing + st * G::TILE_BYTES, G::KCHUNK, 1024);
                const uint32_t aP = tbase + COL_P + (uint32_t)(g & 1) * 64;
#pragma unroll
                for (int kk = 0; kk < B / 16; ++kk)
                    mma_ts_w(tbase + COL_O, aP + kk * 8, vd0 + (uint64_t)((kk * 2048) >> 4), idesc_pv,
                             (t > 0 || kk > 0) ? 1u : 0u);
                tc_commit_w(O_DONE);
                tc_commit_w(RING_EMPTY(st));
            };
            if (G_tiles > 0) {
                // prologue: QK(0)
                {
                    uint32_t st, sp;
                    take(st, sp);
                    mbar_wait(Q_FULL(0), 0);
                    mbar_wait(RING_FULL(st), sp);
                    mma_qk(0, 0, 0, st);
                }
                // iteration g: [QK(g+1) ; PV(g)].  (r, t) of g and (r1, t1) of g+1 tracked
                // incrementally; the four barriers of an iteration are probed together.
                int r = 0, t = 0;
                for (int64_t g = 0; g < G_tiles; ++g) {
                    const bool more = g + 1 < G_tiles;
                    const int r1 = (t + 1 < K) ? r : r + 1, t1 = (t + 1 < K) ? t + 1 : 0;
                    const uint32_t b1 = (uint32_t)((g + 1) & 1), n1 = (uint32_t)((g + 1) >> 1);
                    const uint32_t b = (uint32_t)(g & 1), n = (uint32_t)(g >> 1);
                    uint32_t sk = 0, kp = 0, sv, vp;
                    if (more) take(sk, kp);
                    take(sv, vp);
                    TR(0, (int)g, 0);
                    const uint32_t ok = mbar_try_wait4(S_FREE(b1), (n1 & 1) ^ 1, RING_FULL(sk), kp,
                                                       P_FULL(b), n & 1, RING_FULL(sv), vp);
                    TR(0, (int)g, 1);
                    if (more) {
                        if (t1 == 0) mbar_wait(Q_FULL(r1 & 1), (r1 >> 1) & 1);
                        if (!(ok & 1u)) mbar_wait(S_FREE(b1), (n1 & 1) ^ 1);
                        if (!(ok & 2u)) mbar_wait(RING_FULL(sk), kp);
                        TR(0, (int)g, 2);
                        mma_qk(g + 1, r1, t1, sk);
                    }
                    TR(0, (int)g, 3);
                    if (t == 0 && r > 0) mbar_wait(O_FREE, (r - 1) & 1);
                    if (!(ok & 4u)) mbar_wait(P_FULL(b), n & 1);
                    TR(0, (int)g, 4);
                    if (!(ok & 8u)) mbar_wait(RING_FULL(sv), vp);
                    TR(0, (int)g, 5);
                    mma_pv(g, t, sv);
                    TR(0, (int)g, 6);
                    r = r1;
                    t = t1;
                }
            }
        }
        __syncwarp();
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_SOFTMAX));
        // ============================ softmax ============================
        const int sw = warp - 4;
        const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31
        const int half = sw >> 2;      // key/P/O column half
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const float sl2 = p.scale_log2;
        int64_t g = 0;
        for (int r = 0; r < my_units; ++r) {
            const int u = UNIT_OF(r);
            const int h = u / NT;
            const int32_t *il = p.idx + (size_t)u * K;
            const uint32_t *mbase = p.slot_mask + (size_t)h * NT * G::MW;
            float m = -INFINITY, l = 0.f;
            int jn = __ldg(il);
            for (int t = 0; t < K; ++t, ++g) {
                constexpr int HW = (G::CW + 31) / 32;  // mask words covering this half
                uint32_t mk[HW];
#pragma unroll
                for (int w = 0; w < HW; ++w) {
                    const uint32_t word = __ldg(mbase + (size_t)jn * G::MW + (half * G::CW) / 32 + w);
                    mk[w] = G::CW >= 32 ? word : (word >> ((half * G::CW) & 31));
                }
                if (t + 1 < K) jn = __ldg(il + t + 1);
                const uint32_t b = (uint32_t)(g & 1), n = (uint32_t)(g >> 1);
                const bool trw = lane == 0 && quarter == 0;
                if (trw) TR(1 + half, (int)g, 0);
                mbar_wait(S_FULL(b), n & 1);
                if (trw) TR(1 + half, (int)g, 1);
                tc_fence_after();
                uint32_t sr[G::CW / 32][32];
                const uint32_t tS = tbase + lane_off + COL_S + b * 128 + half * G::CW;
#pragma unroll
                for (int c = 0; c < G::CW / 32; ++c) tmem_ld32(tS + c * 32, sr[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < G::CW / 32; ++c) reg_fence(sr[c]);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(S_FREE(b));  // QK(g+2) may overwrite S(b) now
                if (trw) TR(1 + half, (int)g, 2);

                bool full = true;
#pragma unroll
                for (int w = 0; w < HW; ++w) full &= (mk[w] == 0xFFFFFFFFu);
                if (!full) {
#pragma unroll
                    for (int c = 0; c < G::CW / 32; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!((mk[c] >> i) & 1u)) sr[c][i] = f2u(-INFINITY);
                }
                float *xm = xmax + (b * 2) * 128;
                const uint32_t tP = tbase + lane_off + COL_P + b * 64 + half * G::PW;
                float f = 1.f;
                bool rescale = false;
                if (t == 0) {
                    // first tile of the unit: row max first (both halves), then exps
                    float mx = row_max<G::CW>(sr);
                    xm[half * 128 + row] = mx;
                    named_bar(1 + quarter, 64);
                    mx = fmaxf(mx, xm[(half ^ 1) * 128 + row]);
                    m = mx * sl2;
                    float dummy;
                    l += exp_store<G::CW, false>(sr, sl2, m == -INFINITY ? 0.f : m, tP, dummy);
                } else {
                    // speculative: exps against the running max m (stale by at most 2^8 under
                    // lazy rescaling), tracking this tile's row max in the same pass; the two
                    // halves then compare notes and the rare tile that outgrows m + 8 is redone
                    float mx;
                    const float ls = exp_store<G::CW, true>(sr, sl2, m == -INFINITY ? 0.f : m, tP, mx);
                    xm[half * 128 + row] = mx;
                    named_bar(1 + quarter, 64);
                    mx = fmaxf(mx, xm[(half ^ 1) * 128 + row]);
                    const float mnew = fmaxf(m, mx * sl2);
                    if (__any_sync(0xFFFFFFFFu, mnew > m + 8.0f)) {
                        f = (mnew == -INFINITY) ? 1.f : ex2(m - mnew);
                        rescale = true;
                        l *= f;
                        m = mnew;
                        float dummy;
                        l += exp_store<G::CW, false>(sr, sl2, m == -INFINITY ? 0.f : m, tP, dummy);
                    } else {
                        l += ls;
                    }
                }
                if (trw) TR(1 + half, (int)g, 3);
                if (trw) TR(1 + half, (int)g, 4);
                if (rescale) {
                    // O must be quiescent: wait for PV(g-1) (PV(g) needs our P_FULL)
                    mbar_wait(O_DONE, (uint32_t)((g - 1) & 1));
                    tc_fence_after();
                    const uint32_t tO = tbase + lane_off + COL_O + half * G::OW;
#pragma unroll
                    for (int c = 0; c < G::OW / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_wait_ld();
                        reg_fence(o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = f2u(u2f(o[i]) * f);
                        tmem_st32(tO + c * 32, o);
                    }
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(P_FULL(b));
                if (trw) TR(1 + half, (int)g, 5);
                if (trw && rescale) TR(1 + half, (int)g, 6);

                if (t == K - 1) {
                    // ---- epilogue: O / l -> bf16, padded query rows -> 0
                    xsum[half * 128 + row] = l;
                    // S_FULL(g) covered MMAs up to QK(g) only: PV(g-1) may still run, so O_DONE
                    // can be two phases short -- wait for PV(g-1) before the parity of PV(g)
                    if (g > 0) mbar_wait(O_DONE, (uint32_t)((g - 1) & 1));
                    mbar_wait(O_DONE, (uint32_t)(g & 1));
                    tc_fence_after();
                    named_bar(1 + quarter, 64);
                    const float lt = l + xsum[(half ^ 1) * 128 + row];
                    bool qvalid = false;
                    if (row < B) qvalid = (__ldg(p.slot_mask + (size_t)u * G::MW + (row >> 5)) >> (row & 31)) & 1u;
                    const float inv = (qvalid && lt > 0.f) ? 1.f / lt : 0.f;
                    uint16_t *orow = p.out + ((size_t)u * B + (row < B ? row : 0)) * D + half * G::OW;
                    const uint32_t tO = tbase + lane_off + COL_O + half * G::OW;
#pragma unroll
                    for (int c = 0; c < G::OW / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_wait_ld();
                        reg_fence(o);
                        if (row < B) {
                            uint32_t pk[16];
#pragma unroll
                            for (int i = 0; i < 16; ++i)
                                pk[i] = pack_bf16(u2f(o[2 * i]) * inv, u2f(o[2 * i + 1]) * inv);
                            uint4 *dst = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                            for (int v = 0; v < 4; ++v)
                                dst[v] = make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                        }
                    }
                    if (p.lse != nullptr && row < B && half == 0)
                        p.lse[(size_t)u * B + row] =
                            (qvalid && lt > 0.f) ? (m + __log2f(lt)) * 0.69314718055994531f : -INFINITY;
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(O_FREE);
                }
            }
        }
    }
#undef UNIT_OF
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
#undef S_FREE
#undef P_FULL
#undef O_DONE
#undef O_FREE
}

static unsigned long long *g_trace = nullptr;

template <int B, int D>
static veda_status launch(const uint16_t *q, const uint16_t *k, const uint16_t *v, const int32_t *idx,
                          const uint32_t *mask, int Hh, int NT, int kk, float scale, uint16_t *o, float *lse,
                          cudaStream_t stream)
{
    using G = Geo<B, D>;
    CUtensorMap mq, mk, mv;
    const uint64_t rows = (uint64_t)Hh * NT * B;
    veda_status st;
    if ((st = make_tmap_bf16(&mq, q, rows, D, B)) != VEDA_OK) return st;
    if ((st = make_tmap_bf16(&mk, k, rows, D, B)) != VEDA_OK) return st;
    if ((st = make_tmap_bf16(&mv, v, rows, D, B)) != VEDA_OK) return st;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(attn_1q_kernel<B, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
        attr_set = true;
    }
    Params p;
    p.idx = idx;
    p.slot_mask = mask;
    p.out = o;
    p.lse = lse;
    p.NT = NT;
    p.k = kk;
    p.total_units = Hh * NT;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.trace = g_trace;
    int grid = Hh * NT;
    const int nsm = num_sms();
    if (grid > nsm) grid = nsm;
    attn_1q_kernel<B, D><<<grid, NTHREADS, G::SMEM, stream>>>(mq, mk, mv, p);
    count_launch();
    return check_launch("sparse_attn_fwd(1q)");
}

}  // namespace attn1q

#ifdef VEDA_ATTN_TRACE
extern "C" __attribute__((visibility("default"))) void veda_dbg_set_attn1q_trace(void *dev_buf)
{
    attn1q::g_trace = static_cast<unsigned long long *>(dev_buf);
}
#endif

veda_status launch_sparse_attn_1q(const uint16_t *q, const uint16_t *k, const uint16_t *v, const int32_t *idx,
                                  const uint32_t *mask, int Hh, int NT, int B, int d, int kk, float scale,
                                  uint16_t *o, float *lse, cudaStream_t s)
{
    if (B == 128 && d == 128) return attn1q::launch<128, 128>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    if (B == 128 && d == 64) return attn1q::launch<128, 64>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    if (B == 64 && d == 128) return attn1q::launch<64, 128>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    if (B == 64 && d == 64) return attn1q::launch<64, 64>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    return fail(VEDA_ERR_CONFIG, "sparse_attn_fwd: unsupported (B=%d, d=%d)", B, d);
}

}  // namespace veda
