// search.cu -- support kernels of the head-aware tiling search (Alg. 1, PAPER.md:632-670;
// Eq. 8-9).
//
// The search evaluates every pi in Omega with the path's own kernels (tile, target scores,
// top-k, sparse attention, untile).  Two things are new:
//   * per-token fp32 values (the row log-sum-exp of full attention) must follow each
//     candidate tiling.  lse_u is a property of the token, not of the tiling, so ONE dense
//     pass per head serves all |Omega| candidates; these kernels move it between layouts
//     (same box/slot conventions as permute.cu, readings R1-R5);
//   * E[h, pi] += ||O_fu - O_sp||_F^2 (Alg. 1 l.659): a bandwidth-bound fp64 reduction.
#include <cmath>

#include "common.cuh"

namespace veda {
namespace {

struct ScalarGrid {
    int T, H, W, Tp, Hp, Wp, B, NT;
};

// token index held by slot b of tile i of head h, or -1 for a padded slot
__device__ __forceinline__ int64_t slot_token(const HeadCfgs &cf, const ScalarGrid &g, int h, int i, int b)
{
    const int pt = cf.pt[h], ph = cf.ph[h], pw = cf.pw[h];
    const int nbw = g.Wp / pw, nbh = g.Hp / ph;
    const int it = i / (nbh * nbw), rem = i - it * nbh * nbw;
    const int ih = rem / nbw, iw = rem - ih * nbw;
    const int dt = b / (ph * pw), dh = (b / pw) % ph, dw = b % pw;
    const int t = it * pt + dt, hh = ih * ph + dh, w = iw * pw + dw;
    if (t >= g.T || hh >= g.H || w >= g.W) return -1;
    return ((int64_t)t * g.H + hh) * g.W + w;
}

__global__ void __launch_bounds__(256) permute_scalar_kernel(const float *__restrict__ x, int64_t hs,
                                                             const __grid_constant__ HeadCfgs cf, const ScalarGrid g,
                                                             int Hh, float pad, float *__restrict__ xt)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (h, i, b)
    const int64_t per_head = (int64_t)g.NT * g.B;
    if (e >= per_head * Hh) return;
    const int h = (int)(e / per_head);
    const int r = (int)(e - h * per_head), i = r / g.B, b = r - i * g.B;
    const int64_t n = slot_token(cf, g, h, i, b);
    xt[e] = n >= 0 ? __ldg(x + h * hs + n) : pad;
}

__global__ void __launch_bounds__(256) unpermute_scalar_kernel(const float *__restrict__ xt,
                                                               const __grid_constant__ HeadCfgs cf,
                                                               const ScalarGrid g, int Hh, float *__restrict__ x,
                                                               int64_t hs)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per_head = (int64_t)g.NT * g.B;
    if (e >= per_head * Hh) return;
    const int h = (int)(e / per_head);
    const int r = (int)(e - h * per_head), i = r / g.B, b = r - i * g.B;
    const int64_t n = slot_token(cf, g, h, i, b);
    if (n >= 0) x[h * hs + n] = __ldg(xt + e);
}

__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xFFFF0000u); }

// err[h] += sum over the head's n elements of (a - b)^2.  The difference of two bf16
// values and its square are exact in fp64; per-thread and per-CTA sums are fp64; the CTA
// partials meet in one fp64 atomicAdd per CTA (their order is not fixed: run-to-run
// differences are at the 1e-16 relative level).
constexpr int SQ_THREADS = 256;
__global__ void __launch_bounds__(SQ_THREADS) sq_err_kernel(const uint16_t *__restrict__ a,
                                                            const uint16_t *__restrict__ b, int64_t hs, int64_t n,
                                                            double *__restrict__ err)
{
    const int h = blockIdx.y;
    const uint4 *pa = reinterpret_cast<const uint4 *>(a + h * hs);
    const uint4 *pb = reinterpret_cast<const uint4 *>(b + h * hs);
    const int64_t nv = n / 8;
    double acc0 = 0.0, acc1 = 0.0;
    for (int64_t x = (int64_t)blockIdx.x * SQ_THREADS + threadIdx.x; x < nv; x += (int64_t)gridDim.x * SQ_THREADS) {
        const uint4 va = __ldg(pa + x), vb = __ldg(pb + x);
        const uint32_t wa[4] = {va.x, va.y, va.z, va.w}, wb[4] = {vb.x, vb.y, vb.z, vb.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const double d0 = (double)bf_lo(wa[c]) - (double)bf_lo(wb[c]);
            const double d1 = (double)bf_hi(wa[c]) - (double)bf_hi(wb[c]);
            acc0 = fma(d0, d0, acc0);
            acc1 = fma(d1, d1, acc1);
        }
    }
    double acc = acc0 + acc1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    __shared__ double red[SQ_THREADS / 32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < SQ_THREADS / 32; ++w) s += red[w];
        atomicAdd(err + h, s);
    }
}

ScalarGrid make_sgrid(int Tp, int Hp, int Wp, int T, int H, int W, int B, int NT)
{
    ScalarGrid g;
    g.T = T; g.H = H; g.W = W; g.Tp = Tp; g.Hp = Hp; g.Wp = Wp; g.B = B; g.NT = NT;
    return g;
}

}  // namespace

veda_status launch_permute_scalar(const float *x, int64_t hs, const HeadCfgs &cf, int Hh, int Tp, int Hp, int Wp,
                                  int T, int H, int W, int B, int NT, float pad, float *xt, cudaStream_t s)
{
    const ScalarGrid g = make_sgrid(Tp, Hp, Wp, T, H, W, B, NT);
    const int64_t total = (int64_t)Hh * NT * B;
    permute_scalar_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(x, hs, cf, g, Hh, pad, xt);
    count_launch();
    return check_launch("tile_permute_scalar");
}

veda_status launch_unpermute_scalar(const float *xt, const HeadCfgs &cf, int Hh, int Tp, int Hp, int Wp, int T,
                                    int H, int W, int B, int NT, float *x, int64_t hs, cudaStream_t s)
{
    const ScalarGrid g = make_sgrid(Tp, Hp, Wp, T, H, W, B, NT);
    const int64_t total = (int64_t)Hh * NT * B;
    unpermute_scalar_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(xt, cf, g, Hh, x, hs);
    count_launch();
    return check_launch("tile_unpermute_scalar");
}

veda_status launch_sq_err(const uint16_t *a, const uint16_t *b, int64_t hs, int64_t n, int Hh, double *err,
                          cudaStream_t s)
{
    const int64_t nv = n / 8;
    int per_head = (4 * num_sms() + Hh - 1) / Hh;
    const int64_t need = (nv + SQ_THREADS * 4 - 1) / (SQ_THREADS * 4);  // >= 4 vectors per thread
    if (per_head > need) per_head = (int)(need > 0 ? need : 1);
    sq_err_kernel<<<dim3(per_head, Hh), SQ_THREADS, 0, s>>>(a, b, hs, n, err);
    count_launch();
    return check_launch("sq_err");
}

}  // namespace veda
