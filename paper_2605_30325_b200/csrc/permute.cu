// permute.cu -- head-aware 3D tiling and untiling (steps a1 / a7 of the path).
//
// Tiling, PAPER.md:143-145 (N tokens -> N_T tiles of B tokens), Eq. 8
// (per-head (p_t,p_h,p_w)), Alg. 2; untiling PAPER.md:298, 660.
// Conventions (R1-R5): raster token order n = (t*H+h)*W+w, tiles in raster
// box order, slots raster (dt,dh,dw) inside the box, zero-padded grid shared by all
// heads, padded slots written as +0 and flagged in slot_mask.
//
// One CTA per (head, tile): the tile's box origin is decoded once; each thread moves
// 16-byte vectors (8 bf16), all loads of a thread issued before its stores.  Both
// kernels are pure HBM copies (DESIGN.md roofline: read N*d*2, write N'*d*2 bytes).
#include <cmath>

#include "common.cuh"

namespace veda {
namespace {

struct GridInfo {
    int T, H, W;     // real latent
    int Tp, Hp, Wp;  // padded grid
    int B, NT;
};

__device__ __forceinline__ int ilog2_pow2(int v) { return __ffs(v) - 1; }

// POOL: also compute the tile's TripPool descriptor z = Avg | Max | Min over its real
// tokens (Eq. 5) from the values already in registers -- one HBM pass instead of a
// second read of the tiled tensor.  Same arithmetic as trippool_kernel (fp64 sums).
template <int CH, bool POOL>  // CH = 16-byte chunks per token row (d / 8)
__global__ void __launch_bounds__(256) tile_permute_kernel(const uint16_t *__restrict__ x, int64_t hs,
                                                           int64_t ts, const __grid_constant__ HeadCfgs cf,
                                                           const GridInfo g, uint16_t *__restrict__ xt,
                                                           int32_t *__restrict__ cnt,
                                                           uint32_t *__restrict__ mask, float *__restrict__ z)
{
    constexpr int D = CH * 8, RG = 256 / CH;  // each thread owns one 8-channel chunk, RG row groups
    double psum[8];
    float pmax[8], pmin[8];
    int pn = 0;
    if (POOL) {
#pragma unroll
        for (int q = 0; q < 8; ++q) { psum[q] = 0.0; pmax[q] = -INFINITY; pmin[q] = INFINITY; }
    }
    const int ti = blockIdx.x;  // h * NT + i
    const int h = ti / g.NT, i = ti - h * g.NT;
    const int pt = cf.pt[h], ph = cf.ph[h], pw = cf.pw[h];
    const int nbw = g.Wp / pw, nbh = g.Hp / ph;
    const int it = i / (nbh * nbw), rem = i - it * nbh * nbw;
    const int ih = rem / nbw, iw = rem - ih * nbw;
    const int t0 = it * pt, h0 = ih * ph, w0 = iw * pw;
    const int lpw = ilog2_pow2(pw), lphw = ilog2_pow2(ph * pw);

    constexpr int PER = 8;  // chunks per thread per batch
    const int total = g.B * CH;
    const uint16_t *xh = x + (int64_t)h * hs;
    uint4 *dst = reinterpret_cast<uint4 *>(xt + (int64_t)ti * g.B * CH * 8);
    for (int base = 0; base < total; base += 256 * PER) {
        uint4 v[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int e = base + q * 256 + threadIdx.x;
            v[q] = make_uint4(0, 0, 0, 0);
            if (e < total) {
                const int j = e / CH, c = e % CH;
                const int dt = j >> lphw, dh = (j >> lpw) & (ph - 1), dw = j & (pw - 1);
                const int t = t0 + dt, hh = h0 + dh, w = w0 + dw;
                if (t < g.T && hh < g.H && w < g.W) {
                    const int64_t n = ((int64_t)t * g.H + hh) * g.W + w;
                    v[q] = __ldg(reinterpret_cast<const uint4 *>(xh + n * ts) + c);
                    if (POOL) {
                        const uint32_t wv[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
                        for (int r = 0; r < 4; ++r) {
                            const float lo = __uint_as_float(wv[r] << 16), hi = __uint_as_float(wv[r] & 0xFFFF0000u);
                            psum[2 * r] += (double)lo;
                            psum[2 * r + 1] += (double)hi;
                            pmax[2 * r] = fmaxf(pmax[2 * r], lo);
                            pmax[2 * r + 1] = fmaxf(pmax[2 * r + 1], hi);
                            pmin[2 * r] = fminf(pmin[2 * r], lo);
                            pmin[2 * r + 1] = fminf(pmin[2 * r + 1], hi);
                        }
                        ++pn;
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int e = base + q * 256 + threadIdx.x;
            if (e < total) dst[e] = v[q];
        }
    }
    if (POOL) {
        __shared__ double s_sum[RG][D];
        __shared__ float s_mx[RG][D], s_mn[RG][D];
        __shared__ int s_n[RG];
        const int c8 = threadIdx.x % CH, rg = threadIdx.x / CH;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            s_sum[rg][c8 * 8 + q] = psum[q];
            s_mx[rg][c8 * 8 + q] = pmax[q];
            s_mn[rg][c8 * 8 + q] = pmin[q];
        }
        if (c8 == 0) s_n[rg] = pn;
        __syncthreads();
        float *zz = z + (int64_t)ti * 3 * D;
        for (int c = threadIdx.x; c < D; c += 256) {
            double sm = 0.0;
            float a = -INFINITY, b = INFINITY;
            int n = 0;
#pragma unroll
            for (int gq = 0; gq < RG; ++gq) {
                sm += s_sum[gq][c];
                a = fmaxf(a, s_mx[gq][c]);
                b = fminf(b, s_mn[gq][c]);
                n += s_n[gq];
            }
            if (n == 0) {
                zz[c] = 0.f; zz[D + c] = 0.f; zz[2 * D + c] = 0.f;
            } else {
                zz[c] = (float)(sm / (double)n);  // Avg: exact fp64 sum, one division, one rounding
                zz[D + c] = a;
                zz[2 * D + c] = b;
            }
        }
    }
    if (mask != nullptr || cnt != nullptr) {
        __shared__ int s_cnt;
        if (threadIdx.x == 0) s_cnt = 0;
        __syncthreads();
        const int MW = (g.B + 31) / 32;
        if (threadIdx.x < MW * 32) {
            const int j = threadIdx.x;
            bool valid = false;
            if (j < g.B) {
                const int dt = j >> lphw, dh = (j >> lpw) & (ph - 1), dw = j & (pw - 1);
                valid = (t0 + dt < g.T) && (h0 + dh < g.H) && (w0 + dw < g.W);
            }
            const uint32_t bits = __ballot_sync(0xFFFFFFFFu, valid);
            if ((threadIdx.x & 31) == 0) {
                if (mask) mask[(int64_t)ti * MW + (j >> 5)] = bits;
                atomicAdd(&s_cnt, __popc(bits));
            }
        }
        __syncthreads();
        if (threadIdx.x == 0 && cnt) cnt[ti] = s_cnt;
    }
}

template <int CH>
__global__ void __launch_bounds__(256) tile_unpermute_kernel(const uint16_t *__restrict__ xt,
                                                             const __grid_constant__ HeadCfgs cf,
                                                             const GridInfo g, uint16_t *__restrict__ x,
                                                             int64_t hs, int64_t ts)
{
    const int ti = blockIdx.x;
    const int h = ti / g.NT, i = ti - h * g.NT;
    const int pt = cf.pt[h], ph = cf.ph[h], pw = cf.pw[h];
    const int nbw = g.Wp / pw, nbh = g.Hp / ph;
    const int it = i / (nbh * nbw), rem = i - it * nbh * nbw;
    const int ih = rem / nbw, iw = rem - ih * nbw;
    const int t0 = it * pt, h0 = ih * ph, w0 = iw * pw;
    const int lpw = ilog2_pow2(pw), lphw = ilog2_pow2(ph * pw);
    constexpr int PER = 8;
    const int total = g.B * CH;
    uint16_t *xh = x + (int64_t)h * hs;
    const uint4 *src = reinterpret_cast<const uint4 *>(xt + (int64_t)ti * g.B * CH * 8);
    for (int base = 0; base < total; base += 256 * PER) {
        uint4 v[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int e = base + q * 256 + threadIdx.x;
            if (e < total) v[q] = __ldg(src + e);
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int e = base + q * 256 + threadIdx.x;
            if (e < total) {
                const int j = e / CH, c = e % CH;
                const int dt = j >> lphw, dh = (j >> lpw) & (ph - 1), dw = j & (pw - 1);
                const int t = t0 + dt, hh = h0 + dh, w = w0 + dw;
                if (t < g.T && hh < g.H && w < g.W) {
                    const int64_t n = ((int64_t)t * g.H + hh) * g.W + w;
                    reinterpret_cast<uint4 *>(xh + n * ts)[c] = v[q];
                }
            }
        }
    }
}

GridInfo make_grid(int Tp, int Hp, int Wp, int T, int H, int W, int B, int NT)
{
    GridInfo g;
    g.T = T; g.H = H; g.W = W; g.Tp = Tp; g.Hp = Hp; g.Wp = Wp; g.B = B; g.NT = NT;
    return g;
}

}  // namespace

veda_status launch_tile_permute(const uint16_t *x, int64_t hs, int64_t ts, const HeadCfgs &cf, int Hh,
                                int Tp, int Hp, int Wp, int T, int H, int W, int B, int NT, int d,
                                uint16_t *xt, int32_t *cnt, uint32_t *mask, float *z, cudaStream_t s)
{
    const GridInfo g = make_grid(Tp, Hp, Wp, T, H, W, B, NT);
    const int blocks = Hh * NT;
    if (d == 128 && z == nullptr)
        tile_permute_kernel<16, false><<<blocks, 256, 0, s>>>(x, hs, ts, cf, g, xt, cnt, mask, z);
    else if (d == 128)
        tile_permute_kernel<16, true><<<blocks, 256, 0, s>>>(x, hs, ts, cf, g, xt, cnt, mask, z);
    else if (d == 64 && z == nullptr)
        tile_permute_kernel<8, false><<<blocks, 256, 0, s>>>(x, hs, ts, cf, g, xt, cnt, mask, z);
    else if (d == 64)
        tile_permute_kernel<8, true><<<blocks, 256, 0, s>>>(x, hs, ts, cf, g, xt, cnt, mask, z);
    else
        return fail(VEDA_ERR_SHAPE, "tile_permute: unsupported d=%d", d);
    count_launch();
    return check_launch("tile_permute");
}

veda_status launch_tile_unpermute(const uint16_t *xt, const HeadCfgs &cf, int Hh, int Tp, int Hp,
                                  int Wp, int T, int H, int W, int B, int NT, int d, uint16_t *x,
                                  int64_t hs, int64_t ts, cudaStream_t s)
{
    const GridInfo g = make_grid(Tp, Hp, Wp, T, H, W, B, NT);
    const int blocks = Hh * NT;
    if (d == 128)
        tile_unpermute_kernel<16><<<blocks, 256, 0, s>>>(xt, cf, g, x, hs, ts);
    else if (d == 64)
        tile_unpermute_kernel<8><<<blocks, 256, 0, s>>>(xt, cf, g, x, hs, ts);
    else
        return fail(VEDA_ERR_SHAPE, "tile_unpermute: unsupported d=%d", d);
    count_launch();
    return check_launch("tile_unpermute");
}

}  // namespace veda
