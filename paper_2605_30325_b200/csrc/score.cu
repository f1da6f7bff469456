// score.cu -- statistics-aware tile scoring (step a2-a4 of the path).
//
//   TripPool, Eq. 5 (Alg. 2): z = Avg (+) Max (+) Min per
//     channel over a tile's real tokens (readings R6, R7).
//   phi, Eq. 6 (Alg. 2): e = GELU(z W1 + b1) W2 + b2 (R8).
//   S_pred, Eq. 6 (Alg. 2): S_ij = e_q,i . e_k,j / sqrt(d').
//
// Precision (R17): the kept index lists must match the fp64 oracle except at
// near-ties < 1e-5, so every reduction here accumulates in fp64 on the FP64 pipe
// (fp32 x fp32 products are exact in fp64); scores are rounded once to fp32.
#include <cmath>

#include "common.cuh"

namespace veda {
namespace {

// ---------------------------------------------------------------- TripPool
// One CTA of 128 threads per (head, tile).  Thread = (row group, 8-channel chunk);
// 16-byte loads; fp64 sums, exact fp32 max/min; partials reduced through smem.
template <int D>
__global__ void __launch_bounds__(128) trippool_kernel(const uint16_t *__restrict__ xt,
                                                       const uint32_t *__restrict__ mask, int B,
                                                       float *__restrict__ z)
{
    constexpr int CH = D / 8;       // chunks per row
    constexpr int RG = 128 / CH;    // row groups
    const int ti = blockIdx.x;
    const int c8 = threadIdx.x % CH, rg = threadIdx.x / CH;
    const int MW = B / 32;
    const uint32_t *mk = mask + (size_t)ti * MW;
    const uint4 *src = reinterpret_cast<const uint4 *>(xt + (size_t)ti * B * D);
    double sum[8];
    float mx[8], mn[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { sum[q] = 0.0; mx[q] = -INFINITY; mn[q] = INFINITY; }
    int n = 0;
    for (int r = rg; r < B; r += RG) {
        if (!((__ldg(mk + (r >> 5)) >> (r & 31)) & 1u)) continue;
        const uint4 v = __ldg(src + (size_t)r * CH + c8);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
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
// batched over blockIdx.z.  64x64 CTA tile, BK=16, 256 threads, 4x4 outputs per thread
// at stride 16 (conflict-free smem reads).  Operands are widened to fp64 in smem.
enum Epi { EPI_GELU_BIAS = 0, EPI_BIAS = 1, EPI_SCORE = 2 };

template <typename TA, typename TB, bool B_TRANS, int EPI>
__global__ void __launch_bounds__(256) gemm_f64acc_kernel(const TA *__restrict__ A,
                                                          const TB *__restrict__ Bm,
                                                          const float *__restrict__ bias,
                                                          const int32_t *__restrict__ cnt, void *C,
                                                          int M, int N, int K, int64_t sA, int64_t sB,
                                                          int64_t sBias, int64_t sC, double inv_den)
{
    constexpr int BM = 64, BN = 64, BK = 16;
    __shared__ double As[BK][BM + 1];
    __shared__ double Bs[BK][BN];
    const int z = blockIdx.z;
    A += z * sA;
    Bm += z * sB;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    for (int k0 = 0; k0 < K; k0 += BK) {
        // A tile: 64 rows x 16 k, 4 elements per thread (k fastest for coalescing)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = threadIdx.x + q * 256;
            const int r = e / BK, kk = e % BK;
            const int gm = m0 + r, gk = k0 + kk;
            As[kk][r] = (gm < M && gk < K) ? (double)A[(int64_t)gm * K + gk] : 0.0;
        }
        if (!B_TRANS) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = threadIdx.x + q * 256;
                const int kk = e / BN, c = e % BN;
                const int gk = k0 + kk, gn = n0 + c;
                Bs[kk][c] = (gk < K && gn < N) ? (double)Bm[(int64_t)gk * N + gn] : 0.0;
            }
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = threadIdx.x + q * 256;
                const int c = e / BK, kk = e % BK;
                const int gk = k0 + kk, gn = n0 + c;
                Bs[kk][c] = (gk < K && gn < N) ? (double)Bm[(int64_t)gn * K + gk] : 0.0;
            }
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty + 16 * i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx + 16 * j;
            if (gn >= N) continue;
            const int64_t o = z * sC + (int64_t)gm * N + gn;
            if (EPI == EPI_GELU_BIAS) {
                const double x = acc[i][j] + (double)bias[z * sBias + gn];
                static_cast<double *>(C)[o] = 0.5 * x * (1.0 + erf(x * 0.70710678118654752440));
            } else if (EPI == EPI_BIAS) {
                static_cast<double *>(C)[o] = acc[i][j] + (double)bias[z * sBias + gn];
            } else {
                const bool empty = cnt[z * (int64_t)N + gn] == 0;
                static_cast<float *>(C)[o] = empty ? -INFINITY : (float)(acc[i][j] / inv_den);
            }
        }
    }
}

}  // namespace

veda_status launch_trippool(const uint16_t *xt, const uint32_t *mask, int Hh, int NT, int B, int d,
                            float *z, cudaStream_t s)
{
    const int blocks = Hh * NT;
    if (d == 128)
        trippool_kernel<128><<<blocks, 128, 0, s>>>(xt, mask, B, z);
    else if (d == 64)
        trippool_kernel<64><<<blocks, 128, 0, s>>>(xt, mask, B, z);
    else
        return fail(VEDA_ERR_SHAPE, "trippool: unsupported d=%d", d);
    count_launch();
    return check_launch("trippool");
}

veda_status launch_project(const float *z, int Hh, int NT, int din, int dh, int dl, const float *w1,
                           const float *b1, const float *w2, const float *b2, double *hidden,
                           double *e, cudaStream_t s)
{
    dim3 g1((dh + 63) / 64, (NT + 63) / 64, Hh);
    gemm_f64acc_kernel<float, float, false, EPI_GELU_BIAS><<<g1, 256, 0, s>>>(
        z, w1, b1, nullptr, hidden, NT, dh, din, (int64_t)NT * din, (int64_t)din * dh, dh,
        (int64_t)NT * dh, 1.0);
    count_launch();
    veda_status st = check_launch("project/layer1");
    if (st != VEDA_OK) return st;
    dim3 g2((dl + 63) / 64, (NT + 63) / 64, Hh);
    gemm_f64acc_kernel<double, float, false, EPI_BIAS><<<g2, 256, 0, s>>>(
        hidden, w2, b2, nullptr, e, NT, dl, dh, (int64_t)NT * dh, (int64_t)dh * dl, dl,
        (int64_t)NT * dl, 1.0);
    count_launch();
    return check_launch("project/layer2");
}

veda_status launch_pair_scores(const double *eq, const double *ek, const int32_t *cnt, int Hh, int NT,
                               int dl, float *scores, cudaStream_t s)
{
    dim3 g((NT + 63) / 64, (NT + 63) / 64, Hh);
    gemm_f64acc_kernel<double, double, true, EPI_SCORE><<<g, 256, 0, s>>>(
        eq, ek, nullptr, cnt, scores, NT, NT, dl, (int64_t)NT * dl, (int64_t)NT * dl, 0,
        (int64_t)NT * NT, sqrt((double)dl));
    count_launch();
    return check_launch("pair_scores");
}

}  // namespace veda
