// pool.cu -- TripPool straight from the token tensor (steps a1 + a2 of the path; the
// path's veda_tile_pool / veda_tile_pool_heads / veda_tile_pool_local).
//
// Eq. 5 (Alg. 2): z = Avg (+) Max (+) Min per channel over
// the real tokens of each tile of the head-aware 3D tiling (Eq. 8;
// readings R1-R7), plus tile_count and slot_mask as veda_tile_permute writes them.
//
// B200 design: a persistent CTA per SM streams tiles through a shared-memory ring with TMA:
// one 5-D box per tile (channels x p_w x p_h x p_t x 1 head, rows of d*2 bytes in slot order,
// out-of-grid slots zero-filled, no swizzle) issued by one producer thread as soon as a ring
// stage frees, so several tiles' HBM reads are always in flight while the consumer warps
// reduce earlier tiles.  Consumer group = d/64 warps per tile, a thread owns a channel pair
// and walks the tile's rows in shared memory (conflict-free 4-byte reads): exact fp64 sums
// (bf16 -> fp32 by a shift, fp32 -> fp64 exact), fp32 Max/Min, one rounding of Avg -- the
// arithmetic of trippool_kernel (score.cu) row by row, so z is bit-identical to the tiled
// form.  Padded slots (rows outside the latent) are excluded by a per-tile slot mask the
// consumers compute from the tile's box origin.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "sm100.cuh"
#include <cuda_bf16.h>

namespace veda {
namespace {
using namespace sm100;

constexpr int PMAXC = 8;         // distinct tile shapes per launch
#ifndef VEDA_POOL_WARPS
#define VEDA_POOL_WARPS 16
#endif
constexpr int PWARPS = VEDA_POOL_WARPS;  // consumer warps
constexpr int PTHREADS = 32 + 32 * PWARPS;

struct PoolParams {
    CUtensorMap map[PMAXC];
    CUtensorMap map2[PMAXC];  // second tensor (K) of a two-tensor launch (ntensor == 2)
    int T, H, W, NT, units;  // units = heads_in_launch * NT (per tensor)
    int ntensor;             // 1, or 2: units [units, 2 units) are the second tensor's tiles
    int tok_major;
    uint8_t pt[PMAXC], ph[PMAXC], pw[PMAXC];
    uint32_t nbw[PMAXC], nbhw[PMAXC], mbw[PMAXC], mbhw[PMAXC];
    uint8_t cid[kMaxHeads];
};

__device__ __forceinline__ int pdiv(int i, uint32_t n, uint32_t m, int &r)
{
    int q = (int)__umulhi((uint32_t)i, m);
    r = i - q * (int)n;
    if (r < 0) { --q; r += (int)n; }
    if (r >= (int)n) { ++q; r -= (int)n; }
    return q;
}

struct Org {
    int c, t0, h0, w0;
};
__device__ __forceinline__ Org origin(const PoolParams &pp, int h, int i)
{
    Org o;
    o.c = pp.cid[h];
    int rem, iw;
    const int it = pdiv(i, pp.nbhw[o.c], pp.mbhw[o.c], rem);
    const int ih = pdiv(rem, pp.nbw[o.c], pp.mbw[o.c], iw);
    o.t0 = it * pp.pt[o.c];
    o.h0 = ih * pp.ph[o.c];
    o.w0 = iw * pp.pw[o.c];
    return o;
}

template <int D, int BT>
struct PGeo {
    static constexpr int TILE = BT * D * 2;
    static constexpr int CW = D / 64;            // warps across the channels of a tile
    static constexpr int RS = PWARPS >= 16 ? 2 : 1;  // row halves (partials combined in smem)
    static constexpr int GW = CW * RS;           // warps per tile
    static constexpr int NG = PWARPS / GW;       // tiles reduced concurrently
    static constexpr int NST_FIT = (200 * 1024) / TILE;
    static constexpr int NST = NST_FIT > 12 ? 12 : NST_FIT;
    static constexpr int XCH = NG * D * 16;     // row-half partials: fp64 sum + bf16x2 max/min per channel pair
    static constexpr int SMEM = NST * TILE + 2 * NST * 8 + XCH + 1024;
    static_assert(NST >= NG + 2, "ring too shallow");
};

template <int D, int BT>
__global__ void __launch_bounds__(PTHREADS, 1) pool_tma_kernel(const __grid_constant__ PoolParams pp,
                                                               float *__restrict__ z, float *__restrict__ z2,
                                                               int32_t *__restrict__ cnt,
                                                               uint32_t *__restrict__ mask)
{
    using G = PGeo<D, BT>;
    constexpr int MW = BT / 32;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sRing = smem_u32(smem);
    const uint32_t sBar = sRing + G::NST * G::TILE;
#define P_FULL(i) (sBar + 8u * (i))
#define P_EMPTY(i) (sBar + 8u * (G::NST + (i)))
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < G::NST; ++i) {
            mbar_init(P_FULL(i), 1);
            mbar_init(P_EMPTY(i), G::GW);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int grid = gridDim.x;
    const int all = pp.units * pp.ntensor;
    const int ntile = (all - (int)blockIdx.x + grid - 1) / grid;  // tiles of this CTA: n*grid + blockIdx.x
    if (warp == 0) {
        // ------------------------------------------------ producer: one TMA box per tile
        if (lane == 0) {
            for (int n = 0; n < ntile; ++n) {
                const int st = n % G::NST;
                const uint32_t ph = (uint32_t)(n / G::NST) & 1u;
                mbar_wait(P_EMPTY(st), ph ^ 1u);
                const int ua = n * grid + (int)blockIdx.x, second = ua >= pp.units;
                const int u = ua - (second ? pp.units : 0), h = u / pp.NT, i = u - h * pp.NT;
                const Org o = origin(pp, h, i);
                const CUtensorMap *mp = second ? &pp.map2[o.c] : &pp.map[o.c];
                mbar_expect_tx(P_FULL(st), G::TILE);
                if (pp.tok_major)
                    tma_load_5d(sRing + st * G::TILE, mp, 0, h, o.w0, o.h0, o.t0, P_FULL(st));
                else
                    tma_load_5d(sRing + st * G::TILE, mp, 0, o.w0, o.h0, o.t0, h, P_FULL(st));
            }
        }
        __syncwarp();
        return;
    }
    // ---------------------------------------------------- consumers
    const int cw = warp - 1;                     // 0 .. PWARPS-1
    const int grp = cw / G::GW, gw = cw % G::GW;  // tile group, warp within the group
    const int j = (gw % G::CW) * 32 + lane;      // channel pair 2j, 2j+1
    const int rh = gw / G::CW;                   // row half (RS = 2) or 0
    constexpr int RB = BT / G::RS;               // rows per warp
    uint8_t *xch = smem + G::NST * G::TILE + 2 * G::NST * 8 + (size_t)grp * D * 16;
    for (int n = grp; n < ntile; n += G::NG) {
        const int st = n % G::NST;
        const int ua = n * grid + (int)blockIdx.x, second = ua >= pp.units;
        const int u = ua - (second ? pp.units : 0), h = u / pp.NT, i = u - h * pp.NT;
        const Org o = origin(pp, h, i);
        const int pw = pp.pw[o.c], lpw = __ffs(pw) - 1, lphw = lpw + __ffs(pp.ph[o.c]) - 1;
        // slot mask of the tile: bit r set iff row r (dt, dh, dw raster) is a real token
        uint32_t mw[MW];
#pragma unroll
        for (int w = 0; w < MW; ++w) {
            const int r = 32 * w + lane;
            const bool ok = o.t0 + (r >> lphw) < pp.T && o.h0 + ((r >> lpw) & (pp.ph[o.c] - 1)) < pp.H &&
                            o.w0 + (r & (pw - 1)) < pp.W;
            mw[w] = __ballot_sync(0xFFFFFFFFu, ok);
        }
        bool full = true;
        int count = 0;
#pragma unroll
        for (int w = 0; w < MW; ++w) {
            full &= mw[w] == 0xFFFFFFFFu;
            count += __popc(mw[w]);
        }
        mbar_wait(P_FULL(st), (uint32_t)(n / G::NST) & 1u);
        const uint32_t *row = reinterpret_cast<const uint32_t *>(smem + (size_t)st * G::TILE) + j + rh * RB * (D / 2);
        // four partial sums / extrema per channel (rows r mod 4): independent dependency
        // chains; the fp64 sums of bf16 values are exact, so the grouping changes nothing.
        // Max/Min on packed bf16 pairs (exact: they return one of the inputs).
        double s0[4] = {0.0, 0.0, 0.0, 0.0}, s1[4] = {0.0, 0.0, 0.0, 0.0};
        const __nv_bfloat162 ninf = __floats2bfloat162_rn(-INFINITY, -INFINITY), pinf = __floats2bfloat162_rn(INFINITY, INFINITY);
        __nv_bfloat162 mx[4] = {ninf, ninf, ninf, ninf}, mn[4] = {pinf, pinf, pinf, pinf};
        auto take = [&](int q, uint32_t v) {
            s0[q] += (double)__uint_as_float(v << 16);
            s1[q] += (double)__uint_as_float(v & 0xFFFF0000u);
            const __nv_bfloat162 b = *reinterpret_cast<const __nv_bfloat162 *>(&v);
            mx[q] = __hmax2(mx[q], b);
            mn[q] = __hmin2(mn[q], b);
        };
        if (full) {
#pragma unroll 8
            for (int r = 0; r < RB; r += 4) {
#pragma unroll
                for (int q = 0; q < 4; ++q) take(q, row[(r + q) * (D / 2)]);
            }
        } else {
#pragma unroll 2
            for (int r = 0; r < RB; r += 4) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int rr = rh * RB + r + q;
                    if ((mw[rr >> 5] >> (rr & 31)) & 1u) take(q, row[(r + q) * (D / 2)]);
                }
            }
        }
        double sum0 = (s0[0] + s0[1]) + (s0[2] + s0[3]), sum1 = (s1[0] + s1[1]) + (s1[2] + s1[3]);
        __nv_bfloat162 mxa = __hmax2(__hmax2(mx[0], mx[1]), __hmax2(mx[2], mx[3]));
        __nv_bfloat162 mna = __hmin2(__hmin2(mn[0], mn[1]), __hmin2(mn[2], mn[3]));
        if (G::RS == 2) {  // the second row half hands its partials to the first
            double2 *xs = reinterpret_cast<double2 *>(xch);
            __nv_bfloat162 *xm = reinterpret_cast<__nv_bfloat162 *>(xch + D * 8);
            if (rh == 1) {
                xs[j] = make_double2(sum0, sum1);
                xm[2 * j] = mxa;
                xm[2 * j + 1] = mna;
            }
            asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * G::GW) : "memory");
            if (rh == 0) {
                const double2 o = xs[j];
                sum0 += o.x;
                sum1 += o.y;
                mxa = __hmax2(mxa, xm[2 * j]);
                mna = __hmin2(mna, xm[2 * j + 1]);
            }
            asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(32 * G::GW) : "memory");
        }
        const float max0 = __low2float(mxa), max1 = __high2float(mxa);
        const float min0 = __low2float(mna), min1 = __high2float(mna);
        __syncwarp();
        if (lane == 0) mbar_arrive(P_EMPTY(st));  // this warp is done with the stage
        if (rh != 0) continue;
        float *zz = (second ? z2 : z) + (size_t)u * 3 * D + 2 * j;
        if (count == 0) {
            *reinterpret_cast<float2 *>(zz) = make_float2(0.f, 0.f);
            *reinterpret_cast<float2 *>(zz + D) = make_float2(0.f, 0.f);
            *reinterpret_cast<float2 *>(zz + 2 * D) = make_float2(0.f, 0.f);
        } else {  // Avg: exact fp64 sum, one division, one rounding (as trippool_kernel)
            *reinterpret_cast<float2 *>(zz) = make_float2((float)(sum0 / (double)count), (float)(sum1 / (double)count));
            *reinterpret_cast<float2 *>(zz + D) = make_float2(max0, max1);
            *reinterpret_cast<float2 *>(zz + 2 * D) = make_float2(min0, min1);
        }
        if (gw == 0 && lane < MW && !second) {  // (rh == 0 here); the counts / masks come from the first tensor
            uint32_t wv = mw[0];
#pragma unroll
            for (int w = 1; w < MW; ++w)
                if (lane == w) wv = mw[w];
            if (mask) mask[(size_t)u * MW + lane] = wv;
            if (cnt && lane == 0) cnt[u] = count;
        }
    }
#undef P_FULL
#undef P_EMPTY
}

template <int D, int BT>
veda_status launch_pool(const uint16_t *x, const uint16_t *x2, int64_t hs, int64_t ts, const HeadCfgs &cf, int Hh,
                        int Hp, int Wp, int T, int H, int W, int NT, float *z, float *z2, int32_t *cnt,
                        uint32_t *mask, cudaStream_t s)
{
    using G = PGeo<D, BT>;
    cudaError_t e = cudaFuncSetAttribute(pool_tma_kernel<D, BT>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    constexpr int MW = BT / 32;
    for (int h0 = 0; h0 < Hh;) {
        static thread_local PoolParams pp;  // ~1.9 KB of kernel parameters, staged per thread
        memset(&pp, 0, sizeof pp);
        int nc = 0, h1 = h0;
        for (; h1 < Hh; ++h1) {
            int c = 0;
            while (c < nc && !(pp.pt[c] == cf.pt[h1] && pp.ph[c] == cf.ph[h1] && pp.pw[c] == cf.pw[h1])) ++c;
            if (c == nc) {
                if (nc == PMAXC) break;
                pp.pt[c] = cf.pt[h1]; pp.ph[c] = cf.ph[h1]; pp.pw[c] = cf.pw[h1];
                ++nc;
            }
            pp.cid[h1 - h0] = (uint8_t)c;
        }
        const int hn = h1 - h0;
        veda_status st;
        int tm = 0;
        for (int c = 0; c < nc; ++c) {
            if ((st = make_tmap_tile_tokens(&pp.map[c], x + (size_t)h0 * hs, hs, ts, hn, T, H, W, D, pp.pt[c], pp.ph[c],
                                            pp.pw[c], &tm, D, false)) != VEDA_OK)
                return st;
            if (x2 && (st = make_tmap_tile_tokens(&pp.map2[c], x2 + (size_t)h0 * hs, hs, ts, hn, T, H, W, D, pp.pt[c],
                                                  pp.ph[c], pp.pw[c], &tm, D, false)) != VEDA_OK)
                return st;
            pp.nbw[c] = (uint32_t)(Wp / pp.pw[c]);
            pp.nbhw[c] = (uint32_t)((Hp / pp.ph[c]) * (Wp / pp.pw[c]));
            auto magic = [](uint32_t n) {
                const unsigned long long m = (0x100000000ull + n - 1) / n;
                return (uint32_t)(m > 0xFFFFFFFFull ? 0xFFFFFFFFull : m);
            };
            pp.mbw[c] = magic(pp.nbw[c]);
            pp.mbhw[c] = magic(pp.nbhw[c]);
        }
        pp.T = T; pp.H = H; pp.W = W; pp.NT = NT; pp.units = hn * NT; pp.tok_major = tm;
        pp.ntensor = x2 ? 2 : 1;
        const int nsm = num_sms();
        const int grid = pp.units * pp.ntensor < nsm ? pp.units * pp.ntensor : nsm;
        pool_tma_kernel<D, BT><<<grid, PTHREADS, G::SMEM, s>>>(
            pp, z + (size_t)h0 * NT * 3 * D, z2 ? z2 + (size_t)h0 * NT * 3 * D : nullptr,
            cnt ? cnt + (size_t)h0 * NT : nullptr, mask ? mask + (size_t)h0 * NT * MW : nullptr);
        count_launch();
        if ((st = check_launch("tile_pool")) != VEDA_OK) return st;
        h0 = h1;
    }
    return VEDA_OK;
}

}  // namespace

veda_status launch_tile_pool_tokens(const uint16_t *x, int64_t hs, int64_t ts, const HeadCfgs &cf, int Hh, int Tp,
                                    int Hp, int Wp, int T, int H, int W, int B, int NT, int d, float *z,
                                    int32_t *cnt, uint32_t *mask, cudaStream_t s)
{
    return launch_tile_pool_tokens2(x, nullptr, hs, ts, cf, Hh, Tp, Hp, Wp, T, H, W, B, NT, d, z, nullptr, cnt, mask, s);
}

veda_status launch_tile_pool_tokens2(const uint16_t *x, const uint16_t *x2, int64_t hs, int64_t ts, const HeadCfgs &cf,
                                     int Hh, int Tp, int Hp, int Wp, int T, int H, int W, int B, int NT, int d,
                                     float *z, float *z2, int32_t *cnt, uint32_t *mask, cudaStream_t s)
{
    (void)Tp;
    // a stride that is never used (one token, or one head) may equal the other one; give it
    // a distinct value so the 5-D tensor map gets a well-ordered dimension set
    if (hs == ts) {
        if ((int64_t)T * H * W == 1)
            ts = hs * Hh;
        else if (Hh == 1)
            hs = ts * ((int64_t)T * H * W);
        else
            return fail(VEDA_ERR_ALIGN, "tile_pool: head_stride == token_stride");
    }
    if (d == 128 && B == 128) return launch_pool<128, 128>(x, x2, hs, ts, cf, Hh, Hp, Wp, T, H, W, NT, z, z2, cnt, mask, s);
    if (d == 128 && B == 64) return launch_pool<128, 64>(x, x2, hs, ts, cf, Hh, Hp, Wp, T, H, W, NT, z, z2, cnt, mask, s);
    if (d == 64 && B == 128) return launch_pool<64, 128>(x, x2, hs, ts, cf, Hh, Hp, Wp, T, H, W, NT, z, z2, cnt, mask, s);
    if (d == 64 && B == 64) return launch_pool<64, 64>(x, x2, hs, ts, cf, Hh, Hp, Wp, T, H, W, NT, z, z2, cnt, mask, s);
    return fail(VEDA_ERR_SHAPE, "tile_pool: unsupported B=%d d=%d", B, d);
}

}  // namespace veda
