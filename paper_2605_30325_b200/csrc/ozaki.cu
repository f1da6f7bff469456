// ozaki.cu -- the scorer's GEMMs (phi layers and S_pred, Eq. 6) at fp64
// accuracy on the INT8 tensor cores (tcgen05.mma kind::i8), Ozaki-style splitting.
//
// Why: the kept-tile lists must equal the fp64 oracle's except on < 1e-5 near-ties
// (reading R17), which rules out bf16/tf32 operands with fp32 accumulation; the FP64
// tensor pipe (DMMA, ~37 TFLOP/s) made the scorer the second-largest step of the path.
//
// Scheme (per GEMM C = A . B^T, A [M][K], B [N][K], per batch = head):
//   * every row of A (and of B) gets a power-of-two scale 2^e with |x| < 2^e (the frexp
//     exponent of the row's max |x|) and is written as NS = 5 signed digits
//       x = 2^e * sum_s a_s 2^-(7s+6),  a_0 = rint(64 y), a_s = rint(128 r_s)  (|a_s| <= 64)
//     i.e. 6 + 4*7 = 34 bits below the row maximum, round-to-nearest (unbiased);
//   * C = 2^(e_A + e_B) * sum_{s+t <= NS-1} 2^-(7(s+t)+12) (A_s . B_t^T): 15 int8 GEMMs with
//     EXACT int32 accumulation (|a_s b_t| <= 4096, K <= 768, <= 5 products per sum), the
//     5 accumulators u = s + t kept side by side in TMEM and combined in fp64 in the
//     epilogue; products with s + t >= NS are below 2^-47 of the row scales and dropped.
//   Simulated on the Waver synthetic heads (fp64 reference): max |S error| 1.0e-8 with
//   NS = 5 (1.3e-6 with NS = 4), vs 7.9e-7 for fp32-stored phi.
//
// Kernels: split_rows / split_cols (row or column digits of an fp32/fp64 matrix; int8
// slices [batch][NS][R][Kp], Kp = K rounded up to 64, zero padded) and oz_gemm_kernel
// (one 128 x BN output tile per CTA; warp 0 TMA producer, warp 1 tcgen05 issuer, all four
// warps the epilogue; 3-stage ring of 64-byte K slabs, SWIZZLE_64B, all five A and B
// slices of a slab in one 4-D TMA box each; epilogues: +bias and erf-GELU -> fp64 hidden,
// +bias -> fp64 phi, /sqrt(d') with -inf for empty key tiles -> fp32 S).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "sm100.cuh"

namespace veda {
namespace oz {
using namespace sm100;

constexpr int NS = 5;       // int8 digits per value
constexpr int BM = 128;     // output rows per CTA (TMEM lanes)
constexpr int BKB = 64;     // K bytes per stage (one SWIZZLE_64B row)
constexpr int NSTAGE = 3;

enum { EPI_GELU_BIAS = 0, EPI_BIAS = 1, EPI_SCORE = 2 };

// ---------------------------------------------------------------- splitting
__device__ __forceinline__ int row_exponent(double m)
{
    int e = 0;
    if (m > 0.0) frexp(m, &e);  // m = f 2^e, f in [0.5, 1): every |x| <= m < 2^e
    return e;
}

// the NS digits of x (|x| < 2^e), packed: digit s of value q goes to byte q of word s
__device__ __forceinline__ void digits4(const double (&x)[4], int e, uint32_t (&w)[NS])
{
#pragma unroll
    for (int s = 0; s < NS; ++s) w[s] = 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        double y = ldexp(x[q], -e);  // exact, |y| < 1
#pragma unroll
        for (int s = 0; s < NS; ++s) {
            y *= (s == 0) ? 64.0 : 128.0;
            const double a = rint(y);
            y -= a;  // exact
            w[s] |= (uint32_t)(uint8_t)(int8_t)(int)a << (8 * q);
        }
    }
}

// A row per warp, K contiguous (element (b, r, k) at X[b*sb + r*sr + k])
template <typename T>
__global__ void __launch_bounds__(256) split_rows_kernel(const T *__restrict__ X, int R, int K, int64_t sr,
                                                         int64_t sb, int Kp, int8_t *__restrict__ out,
                                                         int32_t *__restrict__ ex)
{
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5), b = blockIdx.y;
    if (r >= R) return;
    const T *x = X + b * sb + (int64_t)r * sr;
    double m = 0.0;
    for (int k = lane; k < K; k += 32) m = fmax(m, fabs((double)__ldg(x + k)));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    const int e = row_exponent(m);
    if (lane == 0) ex[(int64_t)b * R + r] = e;
    int8_t *o = out + ((int64_t)b * NS * R + r) * Kp;
    for (int k = lane * 4; k < Kp; k += 128) {
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = (k + q < K) ? (double)__ldg(x + k + q) : 0.0;
        uint32_t w[NS];
        digits4(v, e, w);
#pragma unroll
        for (int s = 0; s < NS; ++s) *reinterpret_cast<uint32_t *>(o + (int64_t)s * R * Kp + k) = w[s];
    }
}

// Matrices stored with the row index contiguous (element (b, r, k) at X[b*sb + k*sk + r]),
// e.g. W1 [d_in][d_h] read as B^T rows n = 0..d_h-1: a block of 32 rows x 8 k-groups; the
// row maximum is reduced across the k-groups in shared memory; loads coalesce over rows
template <typename T>
__global__ void __launch_bounds__(256) split_cols_kernel(const T *__restrict__ X, int R, int K, int64_t sk,
                                                         int64_t sb, int Kp, int8_t *__restrict__ out,
                                                         int32_t *__restrict__ ex)
{
    __shared__ double s_m[8][32];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int r = blockIdx.x * 32 + tx, b = blockIdx.y;
    const bool ok = r < R;
    const T *x = X + b * sb + (ok ? r : 0);
    double m = 0.0;
    if (ok)
        for (int k = ty; k < K; k += 8) m = fmax(m, fabs((double)__ldg(x + (int64_t)k * sk)));
    s_m[ty][tx] = m;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) m = fmax(m, s_m[j][tx]);
    if (!ok) return;
    const int e = row_exponent(m);
    if (ty == 0) ex[(int64_t)b * R + r] = e;
    int8_t *o = out + ((int64_t)b * NS * R + r) * Kp;
    for (int k = ty * 4; k < Kp; k += 32) {
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = (k + q < K) ? (double)__ldg(x + (int64_t)(k + q) * sk) : 0.0;
        uint32_t w[NS];
        digits4(v, e, w);
#pragma unroll
        for (int s = 0; s < NS; ++s) *reinterpret_cast<uint32_t *>(o + (int64_t)s * R * Kp + k) = w[s];
    }
}

// ---------------------------------------------------------------- GEMM
struct GemmArgs {
    const int32_t *ea, *eb;  // row exponents of A [batch][M] and B [batch][N]
    const float *bias;       // [batch][N] (EPI_GELU_BIAS / EPI_BIAS)
    const int32_t *cnt;      // [batch][N] key-tile counts (EPI_SCORE)
    void *C;                 // [batch][M][N]: fp64 (hidden / phi) or fp32 (scores)
    int M, N, nk;            // nk = Kp / 64
    double den;              // EPI_SCORE: sqrt(d')
};

template <int BN>
struct GemmGeo {
    static constexpr int A_BYTES = NS * BM * BKB;
    static constexpr int B_BYTES = NS * BN * BKB;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int SMEM = NSTAGE * STAGE + 1024 + 64;
    static_assert(NS * BN <= 512, "accumulators exceed TMEM");
};

template <int BN, int EPI>
__global__ void __launch_bounds__(128, 1) oz_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB, const GemmArgs g)
{
    using G = GemmGeo<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t sbar = sbase + NSTAGE * G::STAGE;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + NSTAGE * G::STAGE + 8 * (2 * NSTAGE + 1));
#define OZ_FULL(i) (sbar + 8u * (i))
#define OZ_EMPTY(i) (sbar + 8u * (NSTAGE + (i)))
#define OZ_DONE (sbar + 8u * (2 * NSTAGE))
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM, b = blockIdx.z;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(OZ_FULL(i), 1);
            mbar_init(OZ_EMPTY(i), 1);
        }
        mbar_init(OZ_DONE, 1);
        fence_barrier_init();
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // TMA producer: all NS slices of A and of B for one 64-byte K slab
            for (int kc = 0; kc < g.nk; ++kc) {
                const int st = kc % NSTAGE;
                const uint32_t ph = (uint32_t)(kc / NSTAGE) & 1u;
                mbar_wait(OZ_EMPTY(st), ph ^ 1u);
                mbar_expect_tx(OZ_FULL(st), G::STAGE);
                const uint32_t sa = sbase + st * G::STAGE;
                tma_load_4d(sa, &tmA, kc * BKB, m0, 0, b, OZ_FULL(st));
                tma_load_4d(sa + G::A_BYTES, &tmB, kc * BKB, n0, 0, b, OZ_FULL(st));
            }
        }
        __syncwarp();
    } else if (warp == 1) {  // MMA issuer (warp-uniform loop, one elected lane issues)
        constexpr uint32_t idesc = idesc_s8_s32(BM, BN);
        for (int kc = 0; kc < g.nk; ++kc) {
            const int st = kc % NSTAGE;
            mbar_wait(OZ_FULL(st), (uint32_t)(kc / NSTAGE) & 1u);
            tc_fence_after();
            const uint32_t sa = sbase + st * G::STAGE, sb = sa + G::A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BKB / 32; ++kk) {
#pragma unroll
                for (int s = 0; s < NS; ++s) {
                    const uint64_t ad = sdesc_sw64(sa + s * BM * BKB + kk * 32, 512);
#pragma unroll
                    for (int t = 0; t + s < NS; ++t) {
                        const uint64_t bd = sdesc_sw64(sb + t * BN * BKB + kk * 32, 512);
                        mma_i8_ss_w(tbase + (uint32_t)((s + t) * BN), ad, bd, idesc,
                                    (kc > 0 || kk > 0 || s > 0) ? 1u : 0u);
                    }
                }
            }
            tc_commit_w(OZ_EMPTY(st));
        }
        tc_commit_w(OZ_DONE);
        __syncwarp();
    }
    // ---- epilogue (all four warps; warp w owns TMEM lanes / tile rows 32w .. 32w+31).
    // Per-column data (exponent of B's row, bias or key-tile count) staged in smem once per
    // tile: read from global inside the element loop, the loads could not be hoisted above
    // the output stores (possible aliasing) and serialised the epilogue.
    __shared__ int s_eb[BN];
    __shared__ double s_col[BN];
    for (int c = threadIdx.x; c < BN; c += 128) {
        const int n = n0 + c;
        const bool ok = n < g.N;
        s_eb[c] = ok ? __ldg(g.eb + (int64_t)b * g.N + n) : 0;
        if (EPI == EPI_SCORE)
            s_col[c] = (ok && __ldg(g.cnt + (int64_t)b * g.N + n) != 0) ? 1.0 / g.den : -INFINITY;
        else
            s_col[c] = ok ? (double)__ldg(g.bias + (int64_t)b * g.N + n) : 0.0;
    }
    __syncthreads();
    mbar_wait(OZ_DONE, 0);
    tc_fence_after();
    const int row = warp * 32 + lane, m = m0 + row;
    const bool mok = m < g.M;
    const int ea = mok ? __ldg(g.ea + (int64_t)b * g.M + m) : 0;
    const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t acc[NS][16];
#pragma unroll
        for (int u = 0; u < NS; ++u) tmem_ld16(tl + (uint32_t)(u * BN + c0), acc[u]);
        tmem_wait_ld();
        if (!mok) continue;
        const int64_t orow = ((int64_t)b * g.M + m) * g.N;
        // vector stores only when the whole 16-column run is in range and the row base is aligned
        const bool full = n0 + c0 + 16 <= g.N && (g.N % 4) == 0;
        double out[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            // sum_u acc_u 2^-(7u+12) = 2^-40 * sum_u acc_u 2^(7(4-u)): |acc_u| < 2^24, so the
            // weighted sum is an exact int64 below 2^53 and converts to fp64 exactly
            int64_t iv = 0;
#pragma unroll
            for (int u = 0; u < NS; ++u) iv += (int64_t)(int32_t)acc[u][i] << (7 * (NS - 1 - u));
            const int sc = ea + s_eb[c0 + i] - (7 * (NS - 1) + 12) + 1023;  // biased exponent of the scale
            const double v = (double)iv * __longlong_as_double((long long)sc << 52);
            if (EPI == EPI_GELU_BIAS) {
                const double x = v + s_col[c0 + i];
                out[i] = 0.5 * x * (1.0 + erf(x * 0.70710678118654752440));
            } else if (EPI == EPI_BIAS) {
                out[i] = v + s_col[c0 + i];
            } else {
                const double f = s_col[c0 + i];  // 1/sqrt(d'), or -inf for an empty key tile
                out[i] = (f == -INFINITY) ? -INFINITY : v * f;
            }
        }
        if (EPI == EPI_SCORE) {
            float *dst = static_cast<float *>(g.C) + orow + n0 + c0;
            if (full) {
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    *reinterpret_cast<float4 *>(dst + i) =
                        make_float4((float)out[i], (float)out[i + 1], (float)out[i + 2], (float)out[i + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (n0 + c0 + i < g.N) dst[i] = (float)out[i];
            }
        } else {
            double *dst = static_cast<double *>(g.C) + orow + n0 + c0;
            if (full) {
#pragma unroll
                for (int i = 0; i < 16; i += 2) *reinterpret_cast<double2 *>(dst + i) = make_double2(out[i], out[i + 1]);
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    if (n0 + c0 + i < g.N) dst[i] = out[i];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
#undef OZ_FULL
#undef OZ_EMPTY
#undef OZ_DONE
}

// ---------------------------------------------------------------- host side
veda_status make_slices_map(CUtensorMap *map, const int8_t *base, int rows, int Kp, int batch, int box_rows);

int kpad(int K) { return (K + BKB - 1) / BKB * BKB; }

template <typename T>
veda_status split_rows(const T *X, int R, int K, int64_t sr, int64_t sb, int batch, int8_t *out, int32_t *ex,
                       cudaStream_t s)
{
    dim3 grid((R + 7) / 8, batch);
    split_rows_kernel<T><<<grid, 256, 0, s>>>(X, R, K, sr, sb, kpad(K), out, ex);
    count_launch();
    return check_launch("ozaki split_rows");
}

template <typename T>
veda_status split_cols(const T *X, int R, int K, int64_t sk, int64_t sb, int batch, int8_t *out, int32_t *ex,
                       cudaStream_t s)
{
    dim3 grid((R + 31) / 32, batch);
    split_cols_kernel<T><<<grid, 256, 0, s>>>(X, R, K, sk, sb, kpad(K), out, ex);
    count_launch();
    return check_launch("ozaki split_cols");
}

template <int BN, int EPI>
veda_status gemm(const int8_t *As, const int8_t *Bs, int M, int N, int K, int batch, const GemmArgs &a0,
                 cudaStream_t s)
{
    using G = GemmGeo<BN>;
    CUtensorMap ma, mb;
    veda_status st;
    if ((st = make_slices_map(&ma, As, M, kpad(K), batch, BM)) != VEDA_OK) return st;
    if ((st = make_slices_map(&mb, Bs, N, kpad(K), batch, BN)) != VEDA_OK) return st;
    static bool attr = false;
    if (!attr) {
        const cudaError_t e =
            cudaFuncSetAttribute(oz_gemm_kernel<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute(oz_gemm): %s", cudaGetErrorString(e));
        attr = true;
    }
    GemmArgs a = a0;
    a.M = M;
    a.N = N;
    a.nk = kpad(K) / BKB;
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
    oz_gemm_kernel<BN, EPI><<<grid, 128, G::SMEM, s>>>(ma, mb, a);
    count_launch();
    return check_launch("ozaki gemm");
}

}  // namespace oz

veda_status oz::make_slices_map(CUtensorMap *map, const int8_t *base, int rows, int Kp, int batch, int box_rows)
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return fail(VEDA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    cuuint64_t dims[4] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)NS, (cuuint64_t)batch};
    cuuint64_t strides[3] = {(cuuint64_t)Kp, (cuuint64_t)Kp * rows, (cuuint64_t)Kp * rows * NS};
    cuuint32_t box[4] = {(cuuint32_t)BKB, (cuuint32_t)box_rows, (cuuint32_t)NS, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t *>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(VEDA_ERR_CUDA, "cuTensorMapEncodeTiled (int8 slices) failed (%d)", (int)r);
    return VEDA_OK;
}

size_t ozaki_workspace(int Hh, int NT, int din, int dh, int dl)
{
    const size_t k1 = oz::kpad(din), k2 = oz::kpad(dh), k3 = oz::kpad(dl);
    size_t amax = std::max(k1, std::max(k2, k3)) * NT;
    size_t bmax = std::max(dh * k1, std::max(dl * k2, NT * k3));
    size_t emax = std::max((size_t)NT, std::max((size_t)dh, (size_t)dl));
    return align256((size_t)Hh * oz::NS * amax) + align256((size_t)Hh * oz::NS * bmax) +
           align256((size_t)Hh * NT * 4) + align256((size_t)Hh * emax * 4);
}

// phi_q, phi_k and S_pred from pooled descriptors on the INT8 tensor cores.
// hidden [Hh][NT][dh], eq / ek [Hh][NT][dl] are fp64 buffers; scratch >= ozaki_workspace.
veda_status launch_ozaki_score(const float *zq, const float *zk, const int32_t *cnt, int Hh, int NT, int din, int dh,
                               int dl, const float *const w_q[4], const float *const w_k[4], double *hidden,
                               double *eq, double *ek, float *scores, void *scratch, cudaStream_t s)
{
    const size_t k1 = oz::kpad(din), k2 = oz::kpad(dh), k3 = oz::kpad(dl);
    const size_t amax = std::max(k1, std::max(k2, k3)) * NT;
    const size_t bmax = std::max(dh * k1, std::max(dl * k2, NT * k3));
    char *p = static_cast<char *>(scratch);
    int8_t *As = reinterpret_cast<int8_t *>(p); p += align256((size_t)Hh * oz::NS * amax);
    int8_t *Bs = reinterpret_cast<int8_t *>(p); p += align256((size_t)Hh * oz::NS * bmax);
    int32_t *ea = reinterpret_cast<int32_t *>(p); p += align256((size_t)Hh * NT * 4);
    int32_t *eb = reinterpret_cast<int32_t *>(p);
    veda_status st;
    for (int side = 0; side < 2; ++side) {
        const float *z = side ? zk : zq;
        const float *const *w = side ? w_k : w_q;
        double *e = side ? ek : eq;
        // layer 1: hidden = GELU(z W1 + b1)
        if ((st = oz::split_rows<float>(z, NT, din, din, (int64_t)NT * din, Hh, As, ea, s)) != VEDA_OK) return st;
        if ((st = oz::split_cols<float>(w[0], dh, din, dh, (int64_t)din * dh, Hh, Bs, eb, s)) != VEDA_OK) return st;
        oz::GemmArgs a{};
        a.ea = ea; a.eb = eb; a.bias = w[1]; a.C = hidden;
        if ((st = oz::gemm<96, oz::EPI_GELU_BIAS>(As, Bs, NT, dh, din, Hh, a, s)) != VEDA_OK) return st;
        // layer 2: e = hidden W2 + b2
        if ((st = oz::split_rows<double>(hidden, NT, dh, dh, (int64_t)NT * dh, Hh, As, ea, s)) != VEDA_OK) return st;
        if ((st = oz::split_cols<float>(w[2], dl, dh, dl, (int64_t)dh * dl, Hh, Bs, eb, s)) != VEDA_OK) return st;
        a.bias = w[3]; a.C = e;
        if ((st = oz::gemm<64, oz::EPI_BIAS>(As, Bs, NT, dl, dh, Hh, a, s)) != VEDA_OK) return st;
    }
    // S_pred = e_q e_k^T / sqrt(d'), -inf on empty key tiles
    if ((st = oz::split_rows<double>(eq, NT, dl, dl, (int64_t)NT * dl, Hh, As, ea, s)) != VEDA_OK) return st;
    if ((st = oz::split_rows<double>(ek, NT, dl, dl, (int64_t)NT * dl, Hh, Bs, eb, s)) != VEDA_OK) return st;
    oz::GemmArgs a{};
    a.ea = ea; a.eb = eb; a.cnt = cnt; a.C = scores; a.den = std::sqrt((double)dl);
    return oz::gemm<96, oz::EPI_SCORE>(As, Bs, NT, NT, dl, Hh, a, s);
}

}  // namespace veda
