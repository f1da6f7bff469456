// score.cu -- statistics-aware tile scoring (step a2-a4 of the path).
//
//   TripPool, Eq. 5 (Alg. 2): z = Avg (+) Max (+) Min per
//     channel over a tile's real tokens (readings R6, R7).
//   phi, Eq. 6 (Alg. 2): e = GELU(z W1 + b1) W2 + b2 (R8).
//   S_pred, Eq. 6 (Alg. 2): S_ij = e_q,i . e_k,j / sqrt(d').
//
// Precision (R17): the kept index lists must match the fp64 oracle except at
// near-ties < 1e-5, so every reduction here accumulates in fp64 (fp32 x fp32 products are
// exact in fp64); scores are rounded once to fp32.  This file holds the pooling kernel of
// the tiled form and the FP64-tensor-core (DMMA) GEMMs of phi / S_pred of the exported
// per-stage calls veda_project / veda_pair_scores; the path's scorer GEMMs run on the INT8
// tensor cores (ozaki.cu) and its pooling straight from token order in pool.cu.
#include <cmath>
#include <cstdlib>

#include "common.cuh"

namespace veda {
namespace {

// ---------------------------------------------------------------- TripPool
// One CTA of 128 threads per (head, tile).  Thread = (row group, 8-channel chunk);
// all of a thread's rows are loaded (16-byte, predicated on the slot mask) before any
// arithmetic so B/RG loads are in flight per thread; fp64 sums, exact fp32 max/min;
// partials reduced through smem.
template <int D, int BT>
__global__ void __launch_bounds__(128) trippool_kernel(const uint16_t *__restrict__ xt,
                                                       const uint32_t *__restrict__ mask,
                                                       float *__restrict__ z)
{
    constexpr int CH = D / 8;       // chunks per row
    constexpr int RG = 128 / CH;    // row groups
    constexpr int RPT = BT / RG;    // rows per thread
    constexpr int MW = BT / 32;
    const int ti = blockIdx.x;
    const int c8 = threadIdx.x % CH, rg = threadIdx.x / CH;
    const uint32_t *mk = mask + (size_t)ti * MW;
    const uint4 *src = reinterpret_cast<const uint4 *>(xt + (size_t)ti * BT * D);
    uint32_t mw[MW];
#pragma unroll
    for (int i = 0; i < MW; ++i) mw[i] = __ldg(mk + i);
    uint4 v[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int r = rg + i * RG;
        v[i] = ((mw[r >> 5] >> (r & 31)) & 1u) ? __ldg(src + (size_t)r * CH + c8) : make_uint4(0, 0, 0, 0);
    }
    double sum[8];
    float mx[8], mn[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { sum[q] = 0.0; mx[q] = -INFINITY; mn[q] = INFINITY; }
    int n = 0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int r = rg + i * RG;
        if (!((mw[r >> 5] >> (r & 31)) & 1u)) continue;
        const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float lo = __uint_as_float(w[q] << 16), hi = __uint_as_float(w[q] & 0xFFFF0000u);
            sum[2 * q] += (double)lo;
            sum[2 * q + 1] += (double)hi;
            mx[2 * q] = fmaxf(mx[2 * q], lo);
            mx[2 * q + 1] = fmaxf(mx[2 * q + 1], hi);
            mn[2 * q] = fminf(mn[2 * q], lo);
            mn[2 * q + 1] = fminf(mn[2 * q + 1], hi);
        }
        ++n;
    }
    __shared__ double s_sum[RG][D];
    __shared__ float s_mx[RG][D], s_mn[RG][D];
    __shared__ int s_n[RG];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        s_sum[rg][c8 * 8 + q] = sum[q];
        s_mx[rg][c8 * 8 + q] = mx[q];
        s_mn[rg][c8 * 8 + q] = mn[q];
    }
    if (c8 == 0) s_n[rg] = n;
    __syncthreads();
    float *zz = z + (size_t)ti * 3 * D;
    for (int c = threadIdx.x; c < D; c += 128) {
        double s = 0.0;
        float a = -INFINITY, b = INFINITY;
        int cnt = 0;
#pragma unroll
        for (int g = 0; g < RG; ++g) {
            s += s_sum[g][c];
            a = fmaxf(a, s_mx[g][c]);
            b = fminf(b, s_mn[g][c]);
            cnt += s_n[g];
        }
        if (cnt == 0) {
            zz[c] = 0.f; zz[D + c] = 0.f; zz[2 * D + c] = 0.f;
        } else {
            zz[c] = (float)(s / (double)cnt);  // Avg: exact fp64 sum, one division, one rounding
            zz[D + c] = a;                      // Max
            zz[2 * D + c] = b;                  // Min
        }
    }
}

// ---------------------------------------------------------------- fp64-accumulating GEMM
// C[M,N] = A[M,K] . B  with B stored [K][N] (B_TRANS=false) or [N][K] (B_TRANS=true),
// batched over blockIdx.z, fp64 accumulation, with a fused epilogue.
enum Epi { EPI_GELU_BIAS = 0, EPI_BIAS = 1, EPI_SCORE = 2 };

constexpr int GB_M = 128, GB_N = 128, GB_K = 16;

// The GEMM of veda_project / veda_pair_scores, on the FP64 tensor cores (DMMA,
// mma.sync.m8n8k4.f64: exact fp64 products, fp64 accumulation).  128x128 CTA tile,
// 8 warps as 2 (m) x 4 (n), warp tile 64x32 = 8x4 DMMA tiles, BK = 16 (4 k-steps).
// Shared tiles are k-major with a 4-double row pad: fragment reads are conflict-free.
constexpr int DM_PAD = 4;

__device__ __forceinline__ void dmma_16x8x8(double (&c)[4], const double (&a)[4], const double (&b)[2])
{
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
                 "{%0, %1, %2, %3};"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void dmma_8x8x4(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <typename T>
__device__ __forceinline__ void load4(const T *p, double (&v)[4], bool ok);
template <>
__device__ __forceinline__ void load4<float>(const float *p, double (&v)[4], bool ok)
{
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ok) a = __ldg(reinterpret_cast<const float4 *>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
template <>
__device__ __forceinline__ void load4<double>(const double *p, double (&v)[4], bool ok)
{
    double2 x = make_double2(0.0, 0.0), y = x;
    if (ok) {
        x = __ldg(reinterpret_cast<const double2 *>(p));
        y = __ldg(reinterpret_cast<const double2 *>(p) + 1);
    }
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
}

constexpr int DM_THREADS = 512;

template <typename TA, typename TB, bool B_TRANS, int EPI>
__global__ void __launch_bounds__(DM_THREADS, 1) gemm_dmma_kernel(const TA *__restrict__ A,
                                                                  const TB *__restrict__ Bm,
                                                                  const float *__restrict__ bias,
                                                                  const int32_t *__restrict__ cnt, void *C,
                                                                  int M, int N, int K, int64_t sA, int64_t sB,
                                                                  int64_t sBias, int64_t sC, double den)
{
    // 128x128 CTA tile, 16 warps as 4 (m) x 4 (n), warp tile 32x32 = 2 x 4 tiles of
    // mma.m16n8k8.f64, BK = 16.  Shared tiles k-major with a 4-double pad.
    __shared__ __align__(16) double As[GB_K][GB_M + DM_PAD];
    __shared__ __align__(16) double Bs[GB_K][GB_N + DM_PAD];
    const int z = blockIdx.z;
    A += z * sA;
    Bm += z * sB;
    const int m0 = blockIdx.y * GB_M, n0 = blockIdx.x * GB_N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = (warp >> 2) * 32, wn = (warp & 3) * 32;
    const int g = lane >> 2, tg = lane & 3;
    const int ar = tid >> 2, ak = (tid & 3) * 4;   // A / B^T staging: 128 rows x 16 k
    const int bk = tid >> 5, bn = (tid & 31) * 4;  // B staging: 16 k x 128 n
    double ra[4], rb[4];
    auto fetch = [&](int k0) {
        const int gm = m0 + ar;
        load4<TA>(A + (int64_t)gm * K + k0 + ak, ra, gm < M && k0 + ak < K);
        if (!B_TRANS) {
            const int gk = k0 + bk;
            if (gk < K && (N % 4) == 0 && n0 + bn + 4 <= N) {
                load4<TB>(Bm + (int64_t)gk * N + n0 + bn, rb, true);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    rb[q] = (gk < K && n0 + bn + q < N) ? (double)Bm[(int64_t)gk * N + n0 + bn + q] : 0.0;
            }
        } else {
            const int gn = n0 + ar;
            load4<TB>(Bm + (int64_t)gn * K + k0 + ak, rb, gn < N && k0 + ak < K);
        }
    };
    auto stash = [&]() {
#pragma unroll
        for (int q = 0; q < 4; ++q) As[ak + q][ar] = ra[q];
        if (!B_TRANS) {
            *reinterpret_cast<double2 *>(&Bs[bk][bn]) = make_double2(rb[0], rb[1]);
            *reinterpret_cast<double2 *>(&Bs[bk][bn + 2]) = make_double2(rb[2], rb[3]);
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) Bs[ak + q][ar] = rb[q];
        }
    };
    double acc[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[i][j][e] = 0.0;

    fetch(0);
    for (int k0 = 0; k0 < K; k0 += GB_K) {
        stash();
        __syncthreads();
        if (k0 + GB_K < K) fetch(k0 + GB_K);
#pragma unroll
        for (int ks = 0; ks < GB_K / 8; ++ks) {
            double a[2][4], b[4][2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int m = wm + i * 16 + g, k = ks * 8 + tg;
                a[i][0] = As[k][m];
                a[i][1] = As[k][m + 8];
                a[i][2] = As[k + 4][m];
                a[i][3] = As[k + 4][m + 8];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = wn + j * 8 + g, k = ks * 8 + tg;
                b[j][0] = Bs[k][n];
                b[j][1] = Bs[k + 4][n];
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_16x8x8(acc[i][j], a[i], b[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int gm = m0 + wm + i * 16 + g + (e >> 1) * 8, gn = n0 + wn + j * 8 + tg * 2 + (e & 1);
                if (gm >= M || gn >= N) continue;
                const int64_t o = z * sC + (int64_t)gm * N + gn;
                const double v = acc[i][j][e];
                if (EPI == EPI_GELU_BIAS) {
                    const double x = v + (double)bias[z * sBias + gn];
                    static_cast<double *>(C)[o] = 0.5 * x * (1.0 + erf(x * 0.70710678118654752440));
                } else if (EPI == EPI_BIAS) {
                    static_cast<double *>(C)[o] = v + (double)bias[z * sBias + gn];
                } else {
                    const bool empty = cnt[z * (int64_t)N + gn] == 0;
                    static_cast<float *>(C)[o] = empty ? -INFINITY : (float)(v / den);
                }
            }
}

#define VEDA_GEMM_LAUNCH(TA, TB, TR_, EPI_, grid, ...) \
    gemm_dmma_kernel<TA, TB, TR_, EPI_><<<grid, DM_THREADS, 0, s>>>(__VA_ARGS__)

}  // namespace

veda_status launch_trippool(const uint16_t *xt, const uint32_t *mask, int Hh, int NT, int B, int d,
                            float *z, cudaStream_t s)
{
    const int blocks = Hh * NT;
    if (d == 128 && B == 128)
        trippool_kernel<128, 128><<<blocks, 128, 0, s>>>(xt, mask, z);
    else if (d == 128 && B == 64)
        trippool_kernel<128, 64><<<blocks, 128, 0, s>>>(xt, mask, z);
    else if (d == 64 && B == 128)
        trippool_kernel<64, 128><<<blocks, 128, 0, s>>>(xt, mask, z);
    else if (d == 64 && B == 64)
        trippool_kernel<64, 64><<<blocks, 128, 0, s>>>(xt, mask, z);
    else
        return fail(VEDA_ERR_SHAPE, "trippool: unsupported B=%d d=%d", B, d);
    count_launch();
    return check_launch("trippool");
}

veda_status launch_project(const float *z, int Hh, int NT, int din, int dh, int dl, const float *w1,
                           const float *b1, const float *w2, const float *b2, double *hidden,
                           double *e, cudaStream_t s)
{
    if ((din % 8) || (dh % 8)) return fail(VEDA_ERR_SHAPE, "project: d_in and d_hidden must be multiples of 8");
    dim3 g1((dh + GB_N - 1) / GB_N, (NT + GB_M - 1) / GB_M, Hh);
    VEDA_GEMM_LAUNCH(float, float, false, EPI_GELU_BIAS, g1, z, w1, b1, nullptr, hidden, NT, dh, din,
                     (int64_t)NT * din, (int64_t)din * dh, dh, (int64_t)NT * dh, 1.0);
    count_launch();
    veda_status st = check_launch("project/layer1");
    if (st != VEDA_OK) return st;
    dim3 g2((dl + GB_N - 1) / GB_N, (NT + GB_M - 1) / GB_M, Hh);
    VEDA_GEMM_LAUNCH(double, float, false, EPI_BIAS, g2, hidden, w2, b2, nullptr, e, NT, dl, dh,
                     (int64_t)NT * dh, (int64_t)dh * dl, dl, (int64_t)NT * dl, 1.0);
    count_launch();
    return check_launch("project/layer2");
}

veda_status launch_pair_scores(const double *eq, const double *ek, const int32_t *cnt, int Hh, int NT,
                               int dl, float *scores, cudaStream_t s)
{
    if (dl % 8) return fail(VEDA_ERR_SHAPE, "pair_scores: d_lat must be a multiple of 8");
    dim3 g((NT + GB_N - 1) / GB_N, (NT + GB_M - 1) / GB_M, Hh);
    VEDA_GEMM_LAUNCH(double, double, true, EPI_SCORE, g, eq, ek, nullptr, cnt, scores, NT, NT, dl,
                     (int64_t)NT * dl, (int64_t)NT * dl, 0, (int64_t)NT * NT, sqrt((double)dl));
    count_launch();
    return check_launch("pair_scores");
}

}  // namespace veda
