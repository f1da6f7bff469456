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
// Kernels: split_rows / split_cols (row or column digits of an fp32/fp64 matrix, from a
// 35-bit fixed-point rounding; int8 slices [batch][NS][R][Kp], Kp = K rounded up to 64,
// zero padded; split_rows optionally applies the erf-GELU of layer 1 first) and the
// persistent oz_gemm_kernel (128 x BN output tiles; warp 0 TMA producer, warp 1 tcgen05
// issuer, warps 2-9 epilogue; 3-stage ring of 64-byte K slabs, SWIZZLE_64B, all five A and
// B slices of a slab in one 4-D TMA box each; epilogues: +bias -> fp64 (layer-1
// pre-activation, phi), x 1/sqrt(d') with -inf for empty key tiles -> fp32 S).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
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

enum { EPI_GELU = 0, EPI_BIAS = 1, EPI_SCORE = 2 };

// ---------------------------------------------------------------- splitting
__device__ __forceinline__ int row_exponent(double m)
{
    int e = 0;
    if (m > 0.0) frexp(m, &e);  // m = f 2^e, f in [0.5, 1): every |x| <= m < 2^e
    return e;
}

// The NS digits of x (|x| < 2^e): Y = rint(x 2^(34-e)) is a 35-bit fixed-point integer
// (|Y| <= 2^34, error <= 2^(e-35)); balanced base-128 digits are peeled off from the low
// end, a_4 .. a_1 in [-64, 63], and a_0 = the rest (|a_0| <= 64), so
// x ~ 2^e sum_s a_s 2^-(7s+6).  Digit s of value q goes to byte q of word s.
// Peeling is a carry chain, Y_{j+1} = (Y_j + 64) >> 7, a_{4-j} = ((Y_j + 64) & 127) - 64,
// whose closed form is offset binary: with C = 64 (128^5 - 1) / 127 and Z = Y + C >= 0,
// a_{4-j} = bits [7j, 7j + 7) of Z minus 64 (j < 4) and a_0 = (Z >> 28) - 64.  Z comes from
// ONE fma: x 2^(34-e) + (2^52 + C) lands in [2^52, 2^53), where the fp64 ulp is 1, so the
// fma rounds x 2^(34-e) to the nearest integer (ties to even: 2^52 + C is even) exactly
// like rint, and the low mantissa bits of the result are Z.  The four 7-bit fields of a
// value are spread to the bytes of one word, the 4 x 4 bytes transposed with PRMTs, and
// v - 64 taken per byte as the sign extension of the 7-bit v ^ 0x40.
__device__ __forceinline__ void digits4(const double (&x)[4], int e, uint32_t (&w)[NS])
{
    static_assert(NS == 5, "digit layout");
    const double scale = __longlong_as_double((long long)(1023 + 34 - e) << 52);  // 2^(34-e)
    constexpr double MAGIC = 4503599627370496.0 + 17315143744.0;                  // 2^52 + C
    uint32_t sp[4], a0[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double t = fma(x[q], scale, MAGIC);
        const uint32_t lo = (uint32_t)__double2loint(t), hi = (uint32_t)__double2hiint(t);
        a0[q] = __funnelshift_r(lo, hi, 28) - 64u;  // byte 0: a_0 (Z < 2^36: bits 28..35)
        sp[q] = (lo & 0x7Fu) | ((lo << 1) & 0x7F00u) | ((lo << 2) & 0x7F0000u) | ((lo << 3) & 0x7F000000u);
    }
    const uint32_t l01 = __byte_perm(sp[0], sp[1], 0x5140), h01 = __byte_perm(sp[0], sp[1], 0x7362);
    const uint32_t l23 = __byte_perm(sp[2], sp[3], 0x5140), h23 = __byte_perm(sp[2], sp[3], 0x7362);
    w[4] = __byte_perm(l01, l23, 0x5410);  // field 0 of values 0..3
    w[3] = __byte_perm(l01, l23, 0x7632);
    w[2] = __byte_perm(h01, h23, 0x5410);
    w[1] = __byte_perm(h01, h23, 0x7632);
#pragma unroll
    for (int s = 1; s < NS; ++s) {
        const uint32_t u = w[s] ^ 0x40404040u;
        w[s] = u | ((u & 0x40404040u) << 1);
    }
    w[0] = __byte_perm(__byte_perm(a0[0], a0[1], 0x0040), __byte_perm(a0[2], a0[3], 0x0040), 0x5410);
}

// Digit images: the split kernels write each operand pre-tiled in exactly the shared-memory
// image one GEMM ring stage holds -- per (batch, block of BR rows, 64-byte K slab): NS
// slices x BR rows x 64 bytes, 16-byte chunks SWIZZLE_64B-permuted (chunk c of row rr at
// c ^ ((rr >> 1) & 3)) -- so the producer moves a stage with one contiguous bulk copy per
// operand instead of NS x BR 64-byte TMA rows.  Rows R .. ceil(R/BR)*BR - 1 are written 0.
struct Img {
    int BR, nblk, nslab;  // rows per block, blocks per batch, 64-byte slabs per row
    __device__ __forceinline__ int64_t word(int b, int r, int k, int s) const  // byte offset of the word at k (k % 4 == 0)
    {
        const int blk = r / BR, rr = r - blk * BR, slab = k >> 6, kb = k & 63;
        const int c = (kb >> 4) ^ ((rr >> 1) & 3);
        return ((((int64_t)(b * nblk + blk) * nslab + slab) * NS + s) * BR + rr) * 64 + (c << 4) + (kb & 15);
    }
};

// GELU(x) = x Phi(x) (erf form, reading R8) in fp64 without the libdevice erf (which costs
// ~70 FP64 instructions and made the layer-2 split FP64-bound): Phi on [-8, 8] by degree-4
// Taylor polynomials around the centres c of 768 intervals of width 1/48 (truncation
// <= (1/96)^5/120 max|Phi^(5)| ~ 1.2e-12 absolute, below the 2^-35 digit quantum of a row).
// Every derivative of Phi is phi times a Hermite polynomial, Phi^(n+1)(c) = (-1)^n He_n(c)
// phi(c), so an interval needs only {Phi(c), phi(c)} (16 bytes: ONE shared-memory load,
// the split being bound by these loads) and
//   Phi(c + h) = Phi(c) + phi(c) h (1 + h (-c/2 + h ((c^2-1)/6 - h (c^3-3c)/24)))
// with the h^2 term in fp64 and the h^3, h^4 terms in fp32 (|h| <= 1/96: they are
// < 2e-6 phi(c), so fp32 adds < 1e-13); table built once on the host from erfc / exp;
// |x| >= 8: Phi = 0 or 1 (error < 7e-16).
constexpr int PHI_N = 768;
constexpr double PHI_SCALE = 48.0;        // intervals per unit of x: PHI_N = 16 * PHI_SCALE
constexpr double PHI_W = 1.0 / 48.0;      // interval width (rounded); centre i: fma(i + 0.5, PHI_W, -8), host and device
static_assert(PHI_N == 16 * 48, "Phi table layout");
struct __align__(16) PhiEntry {
    double Phi, phi;  // Phi(c), phi(c) = exp(-c^2/2) / sqrt(2 pi)
};
static_assert(sizeof(PhiEntry) == 16, "one 16-byte load per interval");
__device__ PhiEntry g_phi_tab[PHI_N];

__device__ __forceinline__ double gelu_tab(double x, const PhiEntry *tab)
{
    if (x >= 8.0) return x;
    if (x <= -8.0) return 0.0;
    int i = (int)((x + 8.0) * PHI_SCALE);
    if (i > PHI_N - 1) i = PHI_N - 1;
    const double c = fma((double)i + 0.5, PHI_W, -8.0);
    const double h = x - c;  // no fp64 division
    const uint4 a = *reinterpret_cast<const uint4 *>(tab + i);
    const double P0 = __hiloint2double(a.y, a.x), p0 = __hiloint2double(a.w, a.z);
    const float cf = (float)c, c2 = cf * cf, hf = (float)h;
    const float t = fmaf(-cf * (c2 - 3.f) * (1.f / 24.f), hf, (c2 - 1.f) * (1.f / 6.f));
    const double q = fma((double)t, h, -0.5 * c);
    return x * fma(p0, h * fma(q, h, 1.0), P0);
}

// the same from the global table (L1-resident) -- used in the layer-1 GEMM epilogue, where
// it overlaps the next tile's MMAs
__device__ __forceinline__ double gelu_tab_g(double x) { return gelu_tab(x, g_phi_tab); }

// A row per warp, K contiguous (element (b, r, k) at X[b*sb + r*sr + k]); the row is held
// in registers (J x 4 values per lane, K <= 128 J).  GELU: the row is the layer-1
// pre-activation and the digits are those of GELU(x) (erf form, reading R8).
template <typename T, int J, bool GELU, int WPR>
__global__ void __launch_bounds__(256, GELU ? 4 : 1) split_rows_kernel(const T *__restrict__ X, int R, int K, int64_t sr,
                                                         int64_t sb, int Kp, int batch, int8_t *__restrict__ out,
                                                         int32_t *__restrict__ ex, const Img img)
{
    // WPR warps share a row (each holds J/WPR of its 128-column chunks, fewer registers ->
    // more resident warps); the row maximum is combined through shared memory.
    // GELU: the Phi table is staged in shared memory once per block, and the block loops
    // over row groups (grid = resident blocks) so that staging is paid once per block.
    constexpr int JW = J / WPR, RPB = 8 / WPR;
    __shared__ PhiEntry s_tab[GELU ? PHI_N : 1];
    __shared__ double s_max[2][8];  // by iteration parity: one __syncthreads per iteration suffices
    if (GELU) {
        const uint4 *g = reinterpret_cast<const uint4 *>(g_phi_tab);
        uint4 *d = reinterpret_cast<uint4 *>(s_tab);
        for (int i = threadIdx.x; i < PHI_N; i += 256) d[i] = g[i];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, part = wi % WPR;
    const int Rp = img.nblk * img.BR;  // rows of the image (R real + zero padding)
    const int nbx = (Rp + RPB - 1) / RPB;
    // without GELU: one row group per block (grid nbx x batch), the loop runs once
    const int nblk = GELU ? nbx * batch : 1;
    int it = 0;
    for (int blk = GELU ? (int)blockIdx.x : 0; blk < nblk; blk += GELU ? (int)gridDim.x : 1, ++it) {
        const int b = GELU ? blk / nbx : (int)blockIdx.y;
        const int r = (GELU ? blk - b * nbx : (int)blockIdx.x) * RPB + wi / WPR;
        const bool ok = r < R, inimg = r < Rp;
        const T *x = X + b * sb + (int64_t)(ok ? r : 0) * sr;
        double v[JW][4];
        double m = 0.0;
#pragma unroll
        for (int jj = 0; jj < JW; ++jj)  // all loads first (K and the row start are multiples of 4)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = 128 * (part + WPR * jj) + 4 * lane + q;
                v[jj][q] = (ok && k < K) ? (double)__ldg(x + k) : 0.0;
            }
#pragma unroll
        for (int jj = 0; jj < JW; ++jj)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (GELU && 128 * (part + WPR * jj) + 4 * lane + q < K) v[jj][q] = gelu_tab(v[jj][q], s_tab);
                m = fmax(m, fabs(v[jj][q]));
            }
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (WPR > 1) {
            if (lane == 0) s_max[it & 1][wi] = m;
            __syncthreads();
#pragma unroll
            for (int p2 = 0; p2 < WPR; ++p2) m = fmax(m, s_max[it & 1][(wi / WPR) * WPR + p2]);
        }
        if (!inimg) continue;
        const int e = row_exponent(m);  // padding rows: all values 0 -> all digits 0
        if (ok && lane == 0 && part == 0) ex[(int64_t)b * R + r] = e;
#pragma unroll
        for (int jj = 0; jj < JW; ++jj) {
            const int k = 128 * (part + WPR * jj) + 4 * lane;
            if (k >= Kp) break;
            uint32_t w[NS];
            digits4(v[jj], e, w);
#pragma unroll
            for (int s = 0; s < NS; ++s) *reinterpret_cast<uint32_t *>(out + img.word(b, r, k, s)) = w[s];
        }
    }
}

// Matrices stored with the row index contiguous (element (b, r, k) at X[b*sb + k*sk + r]),
// e.g. W1 [d_in][d_h] read as B^T rows n = 0..d_h-1: a block of 32 rows x 8 k-groups.  The
// row maximum is reduced across the k-groups in shared memory; loads coalesce over rows;
// the digits of a 128-wide k chunk are transposed through shared memory so every slice row
// is written as contiguous 128-byte runs.
template <typename T>
__global__ void __launch_bounds__(256) split_cols_kernel(const T *__restrict__ X, int R, int K, int64_t sk,
                                                         int64_t sb, int Kp, int8_t *__restrict__ out,
                                                         int32_t *__restrict__ ex, const Img img)
{
    __shared__ double s_m[8][32];
    __shared__ uint32_t s_d[NS][32][33];  // [slice][row][k word], padded
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int r0 = blockIdx.x * 32, b = blockIdx.y;
    const int r = r0 + tx;
    const bool ok = r < R;
    const T *x = X + b * sb + (ok ? r : 0);
    double m = 0.0;
    if (ok)
        for (int k = ty; k < K; k += 8) m = fmax(m, fabs((double)__ldg(x + (int64_t)k * sk)));
    s_m[ty][tx] = m;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j) m = fmax(m, s_m[j][tx]);
    const int e = row_exponent(m);
    if (ty == 0 && ok) ex[(int64_t)b * R + r] = e;
    for (int kc = 0; kc < Kp; kc += 128) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // k words ty + 8j of this chunk: 4 values each
            const int wk = ty + 8 * j, k = kc + 4 * wk;
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = (ok && k + q < K) ? (double)__ldg(x + (int64_t)(k + q) * sk) : 0.0;
            uint32_t w[NS];
            digits4(v, e, w);
#pragma unroll
            for (int s = 0; s < NS; ++s) s_d[s][tx][wk] = w[s];
        }
        __syncthreads();
        // write: slice s, row rr, word ww (rows past R: zero digits, already in s_d)
        for (int i = threadIdx.x; i < NS * 32 * 32; i += 256) {
            const int ww = i & 31, rr = (i >> 5) & 31, s = i >> 10;
            if (r0 + rr < img.nblk * img.BR && kc + 4 * ww < Kp)
                *reinterpret_cast<uint32_t *>(out + img.word(b, r0 + rr, kc + 4 * ww, s)) = s_d[s][rr][ww];
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- GEMM
struct GemmArgs {
    const int32_t *ea, *eb;  // row exponents of A [batch][M] and B [batch][N]
    const float *bias;       // [batch][N] (EPI_BIAS)
    const int32_t *cnt;      // [batch][N] key-tile counts (EPI_SCORE)
    void *C;                 // [batch][M][N]: fp64 (hidden / phi) or fp32 (scores)
    int M, N, nk, batch;     // nk = Kp / 64
    double den;              // EPI_SCORE: sqrt(d')
};

template <int BN>
struct GemmGeo {
    static constexpr int A_BYTES = NS * BM * BKB;
    static constexpr int B_BYTES = NS * BN * BKB;
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int SMEM = NSTAGE * STAGE + 1024 + 128;
    static_assert(NS * BN <= 512, "accumulators exceed TMEM");
    static_assert((BN / 2) % 16 == 0, "each epilogue column half is a whole number of 16-column chunks");
};

// Persistent: one CTA per SM walks the (batch, m-block, n-block) tiles (n fastest, so an
// A slab is re-read from L2 by the neighbouring tiles).  Warp 0: TMA producer running ahead
// across tile boundaries through the 3-stage ring; warp 1: MMA issuer (waits until the
// epilogue has drained the accumulators of the previous tile); warps 2-9: epilogue, two
// warps per TMEM lane quarter splitting the tile's columns (so the accumulators drain in
// half the time and the next tile's MMAs start sooner) (warp w
// reads TMEM lane quarter w % 4), releasing TMEM as soon as the last accumulator chunk is
// in registers.
constexpr int EPI_WARPS = 8;
constexpr int GEMM_THREADS = 64 + 32 * EPI_WARPS;

// Epilogue of one 128 x BN output tile, run by the EPI_WARPS epilogue warps: stage the
// per-column data, wait for the tile's accumulators (done_bar), read this warp's column
// half from TMEM (releasing TMEM through tfree_bar once all of it is in registers),
// combine the 5 accumulators exactly, scale, apply the epilogue op and store.  The TMEM
// reads use the 16x256b shape: lane t holds rows rbase + t/4 + {0, 8, 16, 24} and columns
// 2(t%4) + {0, 1} and 8 + 2(t%4) + {0, 1} of each 16-column chunk, so four neighbouring
// threads store 8 consecutive outputs of a row (64 B of fp64) -- a warp store touches 8
// rows instead of 32 (the 32x32b row-per-thread form made every store 32 separate
// L1 wavefronts, which competed with the tensor core's shared-memory operand reads).
template <int BN, int EPI>
__device__ __forceinline__ void epi_tile(const GemmArgs &g, uint32_t tl, int b, int m0, int n0, int cbeg, int cend,
                                         int rbase, const int (&ea)[4], uint32_t done_bar, uint32_t done_parity,
                                         uint32_t tfree_bar, const int *s_eb, const double *s_col)
{
    // s_eb / s_col: this tile's per-column data (exponent of B's row, bias / score factor),
    // staged in shared memory by the caller one tile ahead; ea: the A exponents of this
    // thread's four rows rbase + t/4 + 8i
    const int lane = threadIdx.x & 31, tr = lane >> 2, tc = 2 * (lane & 3);
    const bool vec = (g.N % 2) == 0;  // 2-element vector stores stay aligned
    mbar_wait(done_bar, done_parity);
    tc_fence_after();
#pragma unroll 1
    for (int c0 = cbeg; c0 < cend; c0 += 16) {
        uint32_t acc[NS][2][8];  // [accumulator][lane half: rows +0 / +16][register]
#pragma unroll
        for (int u = 0; u < NS; ++u)
#pragma unroll
            for (int h = 0; h < 2; ++h) tmem_ld16x256b_x2(tl + ((uint32_t)(16 * h) << 16) + (uint32_t)(u * BN + c0), acc[u][h]);
        tmem_wait_ld();
        if (c0 + 16 >= cend) {  // this warp's accumulator columns are in registers
            tc_fence_before();
            mbar_arrive(tfree_bar);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int rs = 0; rs < 2; ++rs) {  // row rbase + 16h + 8rs + t/4
                const int m = m0 + rbase + 16 * h + 8 * rs + tr;
                if (m >= g.M) continue;
                const int64_t orow = ((int64_t)b * g.M + m) * g.N;
#pragma unroll
                for (int cb = 0; cb < 2; ++cb) {  // columns c0 + 8cb + 2(t%4) + {0, 1}
                    const int cl = c0 + 8 * cb + tc;
                    double o2[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int j = 4 * cb + 2 * rs + e;
                        // sum_u acc_u 2^-(7u+12) = 2^-40 * sum_u acc_u 2^(7(4-u)): |acc_u| < 2^24, so
                        // the weighted sum is an exact int64 below 2^53 and converts to fp64 exactly
                        int64_t iv = 0;
#pragma unroll
                        for (int u = 0; u < NS; ++u) iv += (int64_t)(int32_t)acc[u][h][j] << (7 * (NS - 1 - u));
                        const int sc = ea[2 * h + rs] + s_eb[cl + e] - (7 * (NS - 1) + 12) + 1023;  // biased exponent
                        const double v = (double)iv * __longlong_as_double((long long)sc << 52);
                        if (EPI == EPI_SCORE) {
                            const double f = s_col[cl + e];  // 1/sqrt(d'), or -inf for an empty key tile
                            o2[e] = (f == -INFINITY) ? -INFINITY : v * f;
                        } else if (EPI == EPI_GELU) {
                            o2[e] = gelu_tab_g(v + s_col[cl + e]);  // hidden = GELU(z W1 + b1)
                        } else {
                            o2[e] = v + s_col[cl + e];  // + bias
                        }
                    }
                    const int n = n0 + cl;
                    if (EPI == EPI_SCORE) {
                        float *dst = static_cast<float *>(g.C) + orow + n;
                        if (vec && n + 2 <= g.N)
                            *reinterpret_cast<float2 *>(dst) = make_float2((float)o2[0], (float)o2[1]);
                        else {
                            if (n < g.N) dst[0] = (float)o2[0];
                            if (n + 1 < g.N) dst[1] = (float)o2[1];
                        }
                    } else {
                        double *dst = static_cast<double *>(g.C) + orow + n;
                        if (vec && n + 2 <= g.N)
                            *reinterpret_cast<double2 *>(dst) = make_double2(o2[0], o2[1]);
                        else {
                            if (n < g.N) dst[0] = o2[0];
                            if (n + 1 < g.N) dst[1] = o2[1];
                        }
                    }
                }
            }
    }
}

template <int BN, int EPI>
__global__ void __launch_bounds__(GEMM_THREADS, 1) oz_gemm_kernel(const int8_t *__restrict__ As,
                                                                  const int8_t *__restrict__ Bs, const GemmArgs g)
{
    using G = GemmGeo<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t sbar = sbase + NSTAGE * G::STAGE;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + NSTAGE * G::STAGE + 8 * (2 * NSTAGE + 2));
#define OZ_FULL(i) (sbar + 8u * (i))
#define OZ_EMPTY(i) (sbar + 8u * (NSTAGE + (i)))
#define OZ_DONE (sbar + 8u * (2 * NSTAGE))
#define OZ_TFREE (sbar + 8u * (2 * NSTAGE + 1))
    __shared__ int s_eb[2][BN];  // per-column data of the current / next tile (epilogue)
    __shared__ double s_col[2][BN];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nmb = (g.M + BM - 1) / BM, nnb = (g.N + BN - 1) / BN;
    const int ntiles = nmb * nnb * g.batch;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(OZ_FULL(i), 1);
            mbar_init(OZ_EMPTY(i), 1);
        }
        mbar_init(OZ_DONE, 1);
        mbar_init(OZ_TFREE, 32 * EPI_WARPS);
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    auto tile_coords = [&](int t, int &b, int &m0, int &n0) {
        const int nb = t % nnb, r = t / nnb;
        m0 = (r % nmb) * BM;
        b = r / nmb;
        n0 = nb * BN;
    };

    if (warp == 0) {
        if (lane == 0) {  // producer: the pre-tiled images of A and B for one 64-byte K slab
            int it = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int b, m0, n0;
                tile_coords(t, b, m0, n0);
                const int8_t *a = As + ((int64_t)(b * nmb + m0 / BM) * g.nk) * G::A_BYTES;
                const int8_t *bb = Bs + ((int64_t)(b * nnb + n0 / BN) * g.nk) * G::B_BYTES;
                for (int kc = 0; kc < g.nk; ++kc, ++it) {
                    const int st = it % NSTAGE;
                    mbar_wait(OZ_EMPTY(st), ((uint32_t)(it / NSTAGE) & 1u) ^ 1u);
                    mbar_expect_tx(OZ_FULL(st), G::STAGE);
                    const uint32_t sa = sbase + st * G::STAGE;
                    bulk_load(sa, a + (int64_t)kc * G::A_BYTES, G::A_BYTES, OZ_FULL(st));
                    bulk_load(sa + G::A_BYTES, bb + (int64_t)kc * G::B_BYTES, G::B_BYTES, OZ_FULL(st));
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {  // MMA issuer (warp-uniform loop, one elected lane issues)
        constexpr uint32_t idesc = idesc_s8_s32(BM, BN);
        int it = 0, nt = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
            mbar_wait(OZ_TFREE, ((uint32_t)nt & 1u) ^ 1u);  // accumulators drained by the epilogue
            tc_fence_after();
            for (int kc = 0; kc < g.nk; ++kc, ++it) {
                const int st = it % NSTAGE;
                mbar_wait(OZ_FULL(st), (uint32_t)(it / NSTAGE) & 1u);
                tc_fence_after();
                const uint32_t sa = sbase + st * G::STAGE, sb = sa + G::A_BYTES;
#pragma unroll
                for (int kk = 0; kk < BKB / 32; ++kk) {
#pragma unroll
                    for (int s = 0; s < NS; ++s) {
                        const uint64_t ad = sdesc_sw64(sa + s * BM * BKB + kk * 32, 512);
#pragma unroll
                        for (int tt = 0; tt + s < NS; ++tt) {
                            const uint64_t bd = sdesc_sw64(sb + tt * BN * BKB + kk * 32, 512);
                            mma_i8_ss_w(tbase + (uint32_t)((s + tt) * BN), ad, bd, idesc,
                                        (kc > 0 || kk > 0 || s > 0) ? 1u : 0u);
                        }
                    }
                }
                tc_commit_w(OZ_EMPTY(st));
            }
            tc_commit_w(OZ_DONE);
        }
        __syncwarp();
    } else {  // ---- epilogue warps 2-9
        const int q = warp & 3;  // TMEM lane quarter (rows 32q .. 32q+31)
        const int cbeg = ((warp - 2) >> 2) * (BN / 2), cend = cbeg + BN / 2;  // this warp's column half
        const int rbase = q * 32, tr = lane >> 2;  // this thread's rows: rbase + tr + 8i (16x256b reads)
        const uint32_t tl = tbase + ((uint32_t)(q * 32) << 16);
        // per-column (and per-row) data of a tile is loaded into registers one tile ahead, so
        // its global-load latency overlaps the previous tile's epilogue; staged to shared
        // memory (double-buffered) behind one named barrier per tile
        const int tid = threadIdx.x - 64;
        int eb_r = 0, ea_r[4] = {0, 0, 0, 0};
        double col_r = 0.0;
        auto load_cols = [&](int t) {
            int b, m0, n0;
            tile_coords(t, b, m0, n0);
            if (tid < BN) {
                const int n = n0 + tid;
                const bool ok = n < g.N;
                eb_r = ok ? __ldg(g.eb + (int64_t)b * g.N + n) : 0;
                if (EPI == EPI_SCORE)
                    col_r = (ok && __ldg(g.cnt + (int64_t)b * g.N + n) != 0) ? 1.0 / g.den : -INFINITY;
                else
                    col_r = ok ? (double)__ldg(g.bias + (int64_t)b * g.N + n) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int m = m0 + rbase + tr + 8 * i;
                ea_r[i] = (m < g.M) ? __ldg(g.ea + (int64_t)b * g.M + m) : 0;
            }
        };
        if (blockIdx.x < ntiles) load_cols(blockIdx.x);
        int nt = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++nt) {
            int b, m0, n0;
            tile_coords(t, b, m0, n0);
            const int buf = nt & 1;  // last read two tiles ago: every warp passed the previous barrier
            if (tid < BN) {
                s_eb[buf][tid] = eb_r;
                s_col[buf][tid] = col_r;
            }
            const int ea[4] = {ea_r[0], ea_r[1], ea_r[2], ea_r[3]};
            asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI_WARPS) : "memory");
            if (t + (int)gridDim.x < ntiles) load_cols(t + gridDim.x);
            epi_tile<BN, EPI>(g, tl, b, m0, n0, cbeg, cend, rbase, ea, OZ_DONE, (uint32_t)nt & 1u, OZ_TFREE,
                              s_eb[buf], s_col[buf]);
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
#undef OZ_TFREE
}

// ---------------------------------------------------------------- host side

int kpad(int K) { return (K + BKB - 1) / BKB * BKB; }

inline Img image_of(int R, int K, int BR) { return Img{BR, (R + BR - 1) / BR, kpad(K) / BKB}; }

template <typename T, bool GELU = false>
veda_status split_rows(const T *X, int R, int K, int64_t sr, int64_t sb, int batch, int8_t *out, int32_t *ex,
                       int BR, cudaStream_t s)
{
    const int Kp = kpad(K);
    const Img img = image_of(R, K, BR);
    const int Rp = img.nblk * BR;
    // one block per row group, or (GELU) as many as are resident, each looping over groups
    auto go = [&](auto kern, int rpb) {
        const int nbx = (Rp + rpb - 1) / rpb, total = nbx * batch;
        dim3 grid(nbx, batch);
        if (GELU) {
            static std::atomic<int> cached{0};  // per instantiation of split_rows<T, GELU>
            int per_sm = cached.load(std::memory_order_relaxed);
            if (per_sm == 0) {
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) != cudaSuccess || per_sm < 1)
                    per_sm = 1;
                cached.store(per_sm, std::memory_order_relaxed);
            }
            grid = dim3(std::min(total, per_sm * num_sms()), 1);
        }
        kern<<<grid, 256, 0, s>>>(X, R, K, sr, sb, Kp, batch, out, ex, img);
    };
    if (Kp <= 128)
        go(split_rows_kernel<T, 1, GELU, 1>, 8);
    else if (Kp <= 256)
        go(split_rows_kernel<T, 2, GELU, 1>, 8);
    else if (Kp <= 512)
        go(split_rows_kernel<T, 4, GELU, 1>, 8);
    else if (Kp <= 1024)  // two warps per row: half the registers per thread
        go(split_rows_kernel<T, 8, GELU, 2>, 4);
    else
        return fail(VEDA_ERR_SHAPE, "ozaki scorer: K=%d > 1024 unsupported", K);
    count_launch();
    return check_launch("ozaki split_rows");
}

template <typename T>
veda_status split_cols(const T *X, int R, int K, int64_t sk, int64_t sb, int batch, int8_t *out, int32_t *ex,
                       int BR, cudaStream_t s)
{
    const Img img = image_of(R, K, BR);
    dim3 grid((img.nblk * BR + 31) / 32, batch);
    split_cols_kernel<T><<<grid, 256, 0, s>>>(X, R, K, sk, sb, kpad(K), out, ex, img);
    count_launch();
    return check_launch("ozaki split_cols");
}

template <int BN, int EPI>
veda_status gemm(const int8_t *As, const int8_t *Bs, int M, int N, int K, int batch, const GemmArgs &a0,
                 cudaStream_t s)
{
    using G = GemmGeo<BN>;
    if ((reinterpret_cast<uintptr_t>(As) | reinterpret_cast<uintptr_t>(Bs)) & 15u)
        return fail(VEDA_ERR_ALIGN, "ozaki gemm: digit images must be 16-byte aligned");
    {  // set per launch: the attribute belongs to the current device's context
        const cudaError_t e =
            cudaFuncSetAttribute(oz_gemm_kernel<BN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute(oz_gemm): %s", cudaGetErrorString(e));
    }
    GemmArgs a = a0;
    a.M = M;
    a.N = N;
    a.nk = kpad(K) / BKB;
    a.batch = batch;
    const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN) * batch;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    oz_gemm_kernel<BN, EPI><<<grid, GEMM_THREADS, G::SMEM, s>>>(As, Bs, a);
    count_launch();
    return check_launch("ozaki gemm");
}

}  // namespace oz

// Taylor table of Phi for gelu_tab, uploaded once per device (static module memory)
static veda_status phi_table_ready(cudaStream_t s)
{
    static std::atomic<bool> done[64];  // zero-initialised (static storage); set once per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (done[dev].load(std::memory_order_acquire)) return VEDA_OK;
    oz::PhiEntry tab[oz::PHI_N];  // 12 KB host staging; the upload below is synchronised before return
    const double inv_sqrt2pi = 0.39894228040143267794;
    for (int i = 0; i < oz::PHI_N; ++i) {
        const double c = std::fma((double)i + 0.5, oz::PHI_W, -8.0);  // the device's centre, bit for bit
        tab[i] = oz::PhiEntry{0.5 * std::erfc(-c / std::sqrt(2.0)), inv_sqrt2pi * std::exp(-0.5 * c * c)};
    }
    const cudaError_t e = cudaMemcpyToSymbolAsync(oz::g_phi_tab, tab, sizeof tab, 0, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "ozaki: Phi table upload: %s", cudaGetErrorString(e));
    if (cudaStreamSynchronize(s) != cudaSuccess) return fail(VEDA_ERR_CUDA, "ozaki: Phi table upload failed");
    done[dev].store(true, std::memory_order_release);  // a concurrent first call uploads the same bytes
    return VEDA_OK;
}

// rows rounded up to whole image blocks: A operands in blocks of BM, B operands of the GEMM's BN
static size_t rup(size_t r, size_t b) { return (r + b - 1) / b * b; }
static size_t img_a_bytes(int NT, int din, int dh, int dl)
{
    return rup(NT, oz::BM) * std::max(oz::kpad(din), std::max(oz::kpad(dh), oz::kpad(dl)));
}
static size_t img_b_bytes(int NT, int din, int dh, int dl)
{
    return std::max(rup(dh, 96) * oz::kpad(din), std::max(rup(dl, 64) * oz::kpad(dh), rup(NT, 96) * oz::kpad(dl)));
}

size_t ozaki_workspace(int Hh, int NT, int din, int dh, int dl)
{
    size_t amax = img_a_bytes(NT, din, dh, dl);
    size_t bmax = img_b_bytes(NT, din, dh, dl);
    size_t emax = std::max((size_t)NT, std::max((size_t)dh, (size_t)dl));
    return align256((size_t)Hh * oz::NS * amax) + align256((size_t)Hh * oz::NS * bmax) +
           align256((size_t)Hh * NT * 4) + align256((size_t)Hh * emax * 4);
}

// Prepared weights (veda_scorer_prepare): the digit images and row exponents of W1 and W2
// of both sides, split once instead of on every call.  Layout for Hh heads (each region
// 256-byte aligned): W1q image, W2q image, W1k image, W2k image (B operands: d_h rows in
// blocks of 96 over d_in, d_lat rows in blocks of 64 over d_h), then the int32 exponents
// e1q [Hh][d_h], e2q [Hh][d_lat], e1k, e2k.
struct Prepared {
    const int8_t *img[4];  // W1q, W2q, W1k, W2k
    const int32_t *ex[4];
};
static size_t prep_img_bytes(int which, int din, int dh, int dl)  // per head
{
    const oz::Img m = (which & 1) ? oz::image_of(dl, dh, 64) : oz::image_of(dh, din, 96);
    return (size_t)m.nblk * m.BR * oz::NS * m.nslab * oz::BKB;
}
size_t ozaki_prepared_bytes(int Hh, int din, int dh, int dl)
{
    size_t b = 0;
    for (int i = 0; i < 4; ++i) b += align256((size_t)Hh * prep_img_bytes(i, din, dh, dl));
    for (int i = 0; i < 4; ++i) b += align256((size_t)Hh * ((i & 1) ? dl : dh) * sizeof(int32_t));
    return b;
}
static Prepared prepared_layout(const void *base, int Hh, int din, int dh, int dl)
{
    Prepared P;
    const char *p = static_cast<const char *>(base);
    for (int i = 0; i < 4; ++i) {
        P.img[i] = reinterpret_cast<const int8_t *>(p);
        p += align256((size_t)Hh * prep_img_bytes(i, din, dh, dl));
    }
    for (int i = 0; i < 4; ++i) {
        P.ex[i] = reinterpret_cast<const int32_t *>(p);
        p += align256((size_t)Hh * ((i & 1) ? dl : dh) * sizeof(int32_t));
    }
    return P;
}
veda_status launch_ozaki_prepare(const float *const w_q[4], const float *const w_k[4], int Hh, int din, int dh, int dl,
                                 void *prepared, cudaStream_t s)
{
    const Prepared P = prepared_layout(prepared, Hh, din, dh, dl);
    veda_status st;
    for (int side = 0; side < 2; ++side) {
        const float *const *w = side ? w_k : w_q;
        int8_t *i1 = const_cast<int8_t *>(P.img[2 * side]), *i2 = const_cast<int8_t *>(P.img[2 * side + 1]);
        int32_t *e1 = const_cast<int32_t *>(P.ex[2 * side]), *e2 = const_cast<int32_t *>(P.ex[2 * side + 1]);
        if ((st = oz::split_cols<float>(w[0], dh, din, dh, (int64_t)din * dh, Hh, i1, e1, 96, s)) != VEDA_OK) return st;
        if ((st = oz::split_cols<float>(w[2], dl, dh, dl, (int64_t)dh * dl, Hh, i2, e2, 64, s)) != VEDA_OK) return st;
    }
    return VEDA_OK;
}

// phi_q, phi_k (Eq. 6's MLPs) from pooled descriptors on the INT8 tensor cores.
// hidden [Hh][NT][dh], eq / ek [Hh][NT][dl] are fp64 buffers; scratch >= ozaki_workspace.
// prepared: the weights' images from launch_ozaki_prepare, or NULL (split here).
veda_status launch_ozaki_phi(const float *zq, const float *zk, int Hh, int NT, int din, int dh, int dl,
                             const float *const w_q[4], const float *const w_k[4], const void *prepared,
                             double *hidden, double *eq, double *ek, void *scratch, cudaStream_t s)
{
    const size_t amax = img_a_bytes(NT, din, dh, dl);
    const size_t bmax = img_b_bytes(NT, din, dh, dl);
    char *p = static_cast<char *>(scratch);
    int8_t *As = reinterpret_cast<int8_t *>(p); p += align256((size_t)Hh * oz::NS * amax);
    int8_t *Bs = reinterpret_cast<int8_t *>(p); p += align256((size_t)Hh * oz::NS * bmax);
    int32_t *ea = reinterpret_cast<int32_t *>(p); p += align256((size_t)Hh * NT * 4);
    int32_t *eb = reinterpret_cast<int32_t *>(p);
    Prepared P{};
    if (prepared) P = prepared_layout(prepared, Hh, din, dh, dl);
    veda_status st;
    if ((st = phi_table_ready(s)) != VEDA_OK) return st;
    for (int side = 0; side < 2; ++side) {
        const float *z = side ? zk : zq;
        const float *const *w = side ? w_k : w_q;
        double *e = side ? ek : eq;
        // layer 1: pre-activation z W1 + b1
        if ((st = oz::split_rows<float>(z, NT, din, din, (int64_t)NT * din, Hh, As, ea, oz::BM, s)) != VEDA_OK) return st;
        const int8_t *b1 = Bs;
        const int32_t *x1 = eb;
        if (prepared) {
            b1 = P.img[2 * side];
            x1 = P.ex[2 * side];
        } else if ((st = oz::split_cols<float>(w[0], dh, din, dh, (int64_t)din * dh, Hh, Bs, eb, 96, s)) != VEDA_OK) {
            return st;
        }
        oz::GemmArgs a{};
        a.ea = ea; a.eb = x1; a.bias = w[1]; a.C = hidden;  // pre-activation z W1 + b1
        if ((st = oz::gemm<96, oz::EPI_BIAS>(As, b1, NT, dh, din, Hh, a, s)) != VEDA_OK) return st;
        // layer 2: e = GELU(pre) W2 + b2 (the GELU is applied while splitting the rows)
        if ((st = oz::split_rows<double, true>(hidden, NT, dh, dh, (int64_t)NT * dh, Hh, As, ea, oz::BM, s)) != VEDA_OK)
            return st;
        const int8_t *b2 = Bs;
        const int32_t *x2 = eb;
        if (prepared) {
            b2 = P.img[2 * side + 1];
            x2 = P.ex[2 * side + 1];
        } else if ((st = oz::split_cols<float>(w[2], dl, dh, dl, (int64_t)dh * dl, Hh, Bs, eb, 64, s)) != VEDA_OK) {
            return st;
        }
        a.eb = x2; a.bias = w[3]; a.C = e;
        if ((st = oz::gemm<64, oz::EPI_BIAS>(As, b2, NT, dl, dh, Hh, a, s)) != VEDA_OK) return st;
    }
    return VEDA_OK;
}

// Digit images of e_q (A) and e_k (B) for all Hh heads (scratch >= ozaki_workspace).
veda_status launch_ozaki_split_e(const double *eq, const double *ek, int Hh, int NT, int din, int dh, int dl,
                                 void *scratch, cudaStream_t s)
{
    const size_t amax = img_a_bytes(NT, din, dh, dl);
    const size_t bmax = img_b_bytes(NT, din, dh, dl);
    char *p = static_cast<char *>(scratch);
    int8_t *As = reinterpret_cast<int8_t *>(p); p += align256((size_t)Hh * oz::NS * amax);
    int8_t *Bs = reinterpret_cast<int8_t *>(p); p += align256((size_t)Hh * oz::NS * bmax);
    int32_t *ea = reinterpret_cast<int32_t *>(p); p += align256((size_t)Hh * NT * 4);
    int32_t *eb = reinterpret_cast<int32_t *>(p);
    veda_status st;
    if ((st = oz::split_rows<double>(eq, NT, dl, dl, (int64_t)NT * dl, Hh, As, ea, oz::BM, s)) != VEDA_OK) return st;
    return oz::split_rows<double>(ek, NT, dl, dl, (int64_t)NT * dl, Hh, Bs, eb, 96, s);
}

// S_pred = e_q e_k^T / sqrt(d'), -inf on empty key tiles, for heads [h0, h0 + hn) of the
// Hh-head images launch_ozaki_split_e wrote (scores: the chunk's [hn][NT][NT]).
veda_status launch_ozaki_score_gemm(const int32_t *cnt, int Hh, int h0, int hn, int NT, int din, int dh, int dl,
                                    float *scores, const void *scratch, cudaStream_t s)
{
    const size_t amax = img_a_bytes(NT, din, dh, dl);
    const size_t bmax = img_b_bytes(NT, din, dh, dl);
    const char *p = static_cast<const char *>(scratch);
    const int8_t *As = reinterpret_cast<const int8_t *>(p); p += align256((size_t)Hh * oz::NS * amax);
    const int8_t *Bs = reinterpret_cast<const int8_t *>(p); p += align256((size_t)Hh * oz::NS * bmax);
    const int32_t *ea = reinterpret_cast<const int32_t *>(p); p += align256((size_t)Hh * NT * 4);
    const int32_t *eb = reinterpret_cast<const int32_t *>(p);
    // per-head image strides (whole blocks of BM / 96 rows, 64-byte slabs of d_lat)
    const size_t a_head = (size_t)oz::image_of(NT, dl, oz::BM).nblk * oz::BM * oz::NS * oz::kpad(dl);
    const size_t b_head = (size_t)oz::image_of(NT, dl, 96).nblk * 96 * oz::NS * oz::kpad(dl);
    oz::GemmArgs a{};
    a.ea = ea + (size_t)h0 * NT; a.eb = eb + (size_t)h0 * NT; a.cnt = cnt + (size_t)h0 * NT;
    a.C = scores; a.den = std::sqrt((double)dl);
    return oz::gemm<96, oz::EPI_SCORE>(As + h0 * a_head, Bs + h0 * b_head, NT, NT, dl, hn, a, s);
}

veda_status launch_ozaki_pair_scores(const double *eq, const double *ek, const int32_t *cnt, int Hh, int NT, int din,
                                     int dh, int dl, float *scores, void *scratch, cudaStream_t s)
{
    veda_status st = launch_ozaki_split_e(eq, ek, Hh, NT, din, dh, dl, scratch, s);
    if (st != VEDA_OK) return st;
    return launch_ozaki_score_gemm(cnt, Hh, 0, Hh, NT, din, dh, dl, scores, scratch, s);
}

// phi_q, phi_k and S_pred for all heads (the unfused form of veda_tile_score)
veda_status launch_ozaki_score(const float *zq, const float *zk, const int32_t *cnt, int Hh, int NT, int din, int dh,
                               int dl, const float *const w_q[4], const float *const w_k[4], const void *prepared,
                               double *hidden, double *eq, double *ek, float *scores, void *scratch, cudaStream_t s)
{
    veda_status st = launch_ozaki_phi(zq, zk, Hh, NT, din, dh, dl, w_q, w_k, prepared, hidden, eq, ek, scratch, s);
    if (st != VEDA_OK) return st;
    return launch_ozaki_pair_scores(eq, ek, cnt, Hh, NT, din, dh, dl, scores, scratch, s);
}

}  // namespace veda
