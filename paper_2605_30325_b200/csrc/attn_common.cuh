// attn_common.cuh -- pieces of the attention kernel (attn_fwd.cu): launch constants, kernel
// parameters, the token-layout tile decode and TMA gather, the trace macro and the
// packed-fp32 softmax helpers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

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
    int NT, k, total_units;  // units (head, query tile) of this launch: [unit0, unit0 + total_units)
    int unit0;
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


#ifdef VEDA_ATTN_DEBUG
#define DBG(...) do { if (blockIdx.x == 0) printf(__VA_ARGS__); } while (0)
#else
#define DBG(...) do { } while (0)
#endif

// Experiments only (tools/experimental/*.cu; the product kernel uses MUFU for every exp):
// fraction of exp2 evaluated on the FMA pipe instead of MUFU: one pair in every
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

}  // namespace attn
}  // namespace veda
