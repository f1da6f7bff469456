// topk.cu -- per-query-tile exact top-k selection (step a5 of the path).
//
// PAPER.md:146-149 (exactly k kept key tiles per query tile), PAPER.md:280 ("retain the
// k highest-scoring key tiles for each query tile"), Alg. 2 line 697.  Readings R10/R11/
// R16: exactly k; among equal scores the lower key-tile index wins; output ascending;
// -0.0 == +0.0.
//
// One CTA (256 threads) per row.  Scores become order-preserving uint32 keys in smem;
// a 4-pass 8-bit MSB radix select finds the k-th largest key T and how many keys equal
// to T must be taken; a final pass in index order emits {key > T} plus the first
// `need` keys == T, compacted with warp ballots -- so the output is ascending by
// construction and identical to "sort by (S desc, j asc), take k, sort by j".
#include "common.cuh"


namespace veda {
namespace {

__device__ __forceinline__ uint32_t order_key(float f)
{
    uint32_t u = __float_as_uint(f);
    if (u == 0x80000000u) u = 0u;  // -0 -> +0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

constexpr int TK_THREADS = 256;
constexpr int TK_WARPS = TK_THREADS / 32;

__global__ void __launch_bounds__(TK_THREADS) topk_kernel(const float *__restrict__ S, int NT, int k,
                                                          int32_t *__restrict__ idx)
{
    extern __shared__ uint32_t keys[];
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_prefix, s_kk;
    __shared__ uint32_t s_w_eq[TK_WARPS], s_w_sel[TK_WARPS];
    const int row = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float *s = S + (size_t)row * NT;
    for (int j = tid; j < NT; j += TK_THREADS) keys[j] = order_key(__ldg(s + j));

    uint32_t prefix = 0, pmask = 0, kk = (uint32_t)k;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        hist[tid] = 0;  // TK_THREADS == 256 bins
        __syncthreads();
        for (int j = tid; j < NT; j += TK_THREADS) {
            const uint32_t key = keys[j];
            if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (warp == 0) {
            // lane l owns bins 255-8l ... 248-8l (descending)
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) { c[q] = hist[255 - 8 * lane - q]; tot += c[q]; }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= o) incl += v;
            }
            uint32_t run = incl - tot;  // keys with a larger digit than this lane's first bin
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (run < kk && kk <= run + c[q]) {
                    s_prefix = prefix | ((uint32_t)(255 - 8 * lane - q) << shift);
                    s_kk = kk - run;
                }
                run += c[q];
            }
        }
        __syncthreads();
        prefix = s_prefix;
        kk = s_kk;
        pmask |= 255u << shift;
    }
    const uint32_t T = prefix;  // the k-th largest key; kk keys equal to T are taken
    uint32_t out_base = 0, eq_base = 0;
    int32_t *out = idx + (size_t)row * k;
    for (int base = 0; base < NT; base += TK_THREADS) {
        const int j = base + tid;
        const uint32_t key = j < NT ? keys[j] : 0u;
        const bool gt = j < NT && key > T;
        const bool eq = j < NT && key == T;
        const uint32_t beq = __ballot_sync(0xFFFFFFFFu, eq);
        if (lane == 0) s_w_eq[warp] = __popc(beq);
        __syncthreads();
        uint32_t eq_before = eq_base, eq_tot = 0;
#pragma unroll
        for (int w = 0; w < TK_WARPS; ++w) {
            if (w < warp) eq_before += s_w_eq[w];
            eq_tot += s_w_eq[w];
        }
        eq_before += __popc(beq & ((1u << lane) - 1u));
        const bool sel = gt || (eq && eq_before < kk);
        const uint32_t bsel = __ballot_sync(0xFFFFFFFFu, sel);
        if (lane == 0) s_w_sel[warp] = __popc(bsel);
        __syncthreads();
        uint32_t pos = out_base, sel_tot = 0;
#pragma unroll
        for (int w = 0; w < TK_WARPS; ++w) {
            if (w < warp) pos += s_w_sel[w];
            sel_tot += s_w_sel[w];
        }
        pos += __popc(bsel & ((1u << lane) - 1u));
        if (sel) out[pos] = j;
        out_base += sel_tot;
        eq_base += eq_tot;
        __syncthreads();  // s_w_* reused next chunk
    }
}


// Warp-per-row variant for n_tiles <= 32*C: lane l holds keys j = 32*i + l (i < C) in
// registers.  The k-th largest key T is built bit by bit from the MSB: a candidate bit is
// kept while at least k keys are >= the candidate (one compare per key plus a redux.sync
// per bit); the search stops as soon as exactly k keys are >= the candidate.  The index-
// order pass then takes keys > T plus the first (k - #{> T}) keys == T, compacted by
// ballots over i -- the same contract as topk_kernel above, without smem or CTA syncs.
constexpr int TKW_WARPS = 8;

// #{i : key[i] >= c} for this lane (c >= 1, or c = 0 meaning "none": see the caller): key +
// (2^32 - c) carries out iff key >= c, so each key costs one add-with-carry-out and one
// add of the carry (two instructions) instead of compare + select + add, and four
// independent accumulators keep the adds off a single dependency chain.
template <int C>
__device__ __forceinline__ uint32_t count_ge(const uint32_t (&key)[C], uint32_t c)
{
    const uint32_t negc = 0u - c;
    uint32_t n[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < C; ++i)
        asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, 0;\n\t}"
            : "+r"(n[i & 3])
            : "r"(key[i]), "r"(negc));
    return (n[0] + n[1]) + (n[2] + n[3]);
}

template <int C>
__global__ void __launch_bounds__(TKW_WARPS * 32, 3) topk_warp_kernel(const float *__restrict__ S, int rows, int NT,
                                                                   int k, int32_t *__restrict__ idx)
{
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * TKW_WARPS + (threadIdx.x >> 5);
    if (row >= rows) return;
    const float *s = S + (size_t)row * NT;
    uint32_t key[C];
#pragma unroll
    for (int i = 0; i < C; ++i) {
        const int j = 32 * i + lane;
        key[i] = j < NT ? order_key(__ldg(s + j)) : 0u;  // 0 sorts below every finite or -inf key
    }
    const uint32_t kk = (uint32_t)k;
    uint32_t T = 0;
#pragma unroll 1
    for (int b = 31; b >= 0; --b) {
        const uint32_t c = T | (1u << b);
        const uint32_t n = __reduce_add_sync(0xFFFFFFFFu, count_ge<C>(key, c));
        if (n >= kk) {
            T = c;
            if (n == kk) break;  // {key >= T} is exactly the answer
        }
    }
    // keys > T = keys >= T + 1 (T + 1 wraps to 0 only for T = 2^32 - 1, where none is greater:
    // count_ge(0) adds 2^32 - 0 = 0 and never carries)
    const uint32_t ngt = __reduce_add_sync(0xFFFFFFFFu, count_ge<C>(key, T + 1u));
    const uint32_t need = kk - ngt;  // keys == T to take, lowest indices first
    const uint32_t lt = (1u << lane) - 1u;
    int32_t *out = idx + (size_t)row * k;
    uint32_t base = 0, eq_seen = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) {
        const int j = 32 * i + lane;
        const bool eq = j < NT && key[i] == T;
        const uint32_t beq = __ballot_sync(0xFFFFFFFFu, eq);
        const bool sel = (j < NT && key[i] > T) || (eq && eq_seen + __popc(beq & lt) < need);
        eq_seen += __popc(beq);
        const uint32_t bsel = __ballot_sync(0xFFFFFFFFu, sel);
        if (sel) out[base + __popc(bsel & lt)] = j;
        base += __popc(bsel);
    }
}


// Candidate-filter select (the path's top-k for n_tiles <= 2048, one warp per row; same
// contract and result as topk_warp_kernel).  The bitwise search above costs ~30 passes over
// all keys of the row; here:
//   1. the row is read with 16-byte loads (lane l holds scores 128m + 4l + e);
//   2. a threshold T0 below the k-th largest score is guessed from the mean and deviation of
//      a 128-score sample (a normal-quantile guess aiming at ~1.5k + 32 scores >= T0) and
//      corrected by counting; one pass sets a per-lane 64-bit candidate mask (one compare and
//      one bit-set per score);
//   3. the k-th largest key is found among the candidates (~8 % of the row, re-read from L1)
//      by interpolation search over the order-preserving keys (count of keys >= a probe),
//      which ends on a probe with exactly k keys >= it or on a key whose ties straddle rank k.
// Rows where no threshold works in a few tries (ties, few finite scores, k close to n_tiles)
// run the full bitwise search.  The output goes through a bitmap over key-tile indices, so
// it is ascending with ties resolved to the lower index.
constexpr int TKF_WARPS = 8;
constexpr int TKF_CL = 16;  // candidate keys per lane held in registers for the search

// inverse of the standard normal upper tail, z with P(X > z) = p, 0 < p <= 0.5
// (Abramowitz-Stegun 26.2.23, |error| < 4.5e-4 -- only a starting guess, corrected by counting)
__device__ __forceinline__ float upper_quantile(float p)
{
    const float t = sqrtf(-2.f * __logf(p));
    return t - (2.515517f + t * (0.802853f + t * 0.010328f)) / (1.f + t * (1.432788f + t * (0.189269f + t * 0.001308f)));
}
__device__ __forceinline__ float warp_sum(float v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
// k-th largest of the keys (per lane C of them) by the MSB-first bitwise search
template <int C>
__device__ __forceinline__ uint32_t kth_largest(const uint32_t (&key)[C], uint32_t kk)
{
    uint32_t T = 0;
#pragma unroll 1
    for (int b = 31; b >= 0; --b) {
        const uint32_t c = T | (1u << b);
        const uint32_t n = __reduce_add_sync(0xFFFFFFFFu, count_ge<C>(key, c));
        if (n >= kk) {
            T = c;
            if (n == kk) break;
        }
    }
    return T;
}

// V = float4 loads per lane (n_tiles <= 128 V <= 2048)
template <int V>
__global__ void __launch_bounds__(TKF_WARPS * 32, V >= 16 ? 2 : 3) topk_filter_kernel(const float *__restrict__ S,
                                                                                       int rows, int NT, int k,
                                                                                       int32_t *__restrict__ idx)
{
    static_assert(V <= 16, "64-bit candidate mask");
    constexpr int NW = 4 * V;  // bitmap words: word i covers key tiles 32i .. 32i+31
    __shared__ uint32_t s_gt[TKF_WARPS][NW], s_eq[TKF_WARPS][NW];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int row = blockIdx.x * TKF_WARPS + w;
    if (row >= rows) return;
    const float *s = S + (size_t)row * NT;
    const bool vec = (NT & 3) == 0 && (reinterpret_cast<uintptr_t>(s) & 15u) == 0;
    float x[4 * V];  // x[4m + e] = S[128m + 4 lane + e]
#pragma unroll
    for (int m = 0; m < V; ++m) {
        const int j = 128 * m + 4 * lane;
        if (vec && j + 3 < NT) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(s + j));
            x[4 * m] = v.x; x[4 * m + 1] = v.y; x[4 * m + 2] = v.z; x[4 * m + 3] = v.w;
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) x[4 * m + e] = j + e < NT ? __ldg(s + j + e) : -INFINITY;
        }
    }
    const uint32_t kk = (uint32_t)k;
    // threshold from a 128-score sample spread over the row (4 per lane, V/4 loads apart)
    float sum = 0.f, sq = 0.f, nf = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const float a = x[4 * (e * V / 4) + e];
        if (isfinite(a)) { sum += a; sq = fmaf(a, a, sq); nf += 1.f; }
    }
    sum = warp_sum(sum);
    sq = warp_sum(sq);
    nf = warp_sum(nf);
    bool ok = false;
    float t0 = 0.f, mu = 0.f, sd = 0.f;
    unsigned long long cm = 0;  // candidate mask: bit 4m + e
    uint32_t c = 0;
    if (nf >= 32.f && (float)k <= 0.2f * (float)NT) {
        mu = sum / nf;
        sd = sqrtf(fmaxf(sq / nf - mu * mu, 0.f));
        float z = upper_quantile(fminf((1.5f * (float)k + 32.f) / (float)NT, 0.5f));
#pragma unroll 1
        for (int tries = 0; tries < 4 && sd > 0.f; ++tries) {
            t0 = fmaf(z, sd, mu);
            uint32_t lo32 = 0, hi32 = 0;
#pragma unroll
            for (int b = 0; b < 4 * V; ++b) {
                if (b < 32)
                    lo32 |= (x[b] >= t0 ? 1u : 0u) << b;
                else
                    hi32 |= (x[b] >= t0 ? 1u : 0u) << (b - 32);
            }
            cm = ((unsigned long long)hi32 << 32) | lo32;
            const uint32_t nl = __popcll(cm);
            c = __reduce_add_sync(0xFFFFFFFFu, nl);
            const uint32_t nmax = __reduce_max_sync(0xFFFFFFFFu, nl);
            if (c >= kk && nmax <= (uint32_t)TKF_CL) { ok = true; break; }
            z += (c < kk) ? -0.5f : 0.3f;
        }
    }
    uint32_t T;
    if (ok) {
        // candidate keys in registers (re-read from L1) with their key-tile indices
        uint32_t key[TKF_CL];
        uint16_t jj[TKF_CL];
        unsigned long long mm = cm;
#pragma unroll
        for (int q = 0; q < TKF_CL; ++q) {
            key[q] = 0u;
            jj[q] = 0;
            if (mm) {
                const int b = __ffsll((long long)mm) - 1;
                mm &= mm - 1;
                const int j = 128 * (b >> 2) + 4 * lane + (b & 3);
                jj[q] = (uint16_t)j;
                key[q] = order_key(s[j]);
            }
        }
        // interpolation search: count(>= lo) >= k > count(>= hi); the first probe comes from
        // the normal model, the next ones alternate secant and bisection steps
        uint32_t kmax = 0;
#pragma unroll
        for (int q = 0; q < TKF_CL; ++q) kmax = max(kmax, key[q]);
        kmax = __reduce_max_sync(0xFFFFFFFFu, kmax);
        uint32_t lo = order_key(t0), clo = c, chi = 0;
        unsigned long long hi = (unsigned long long)kmax + 1ull;  // count(>= kmax + 1) = 0 < k
        uint32_t guess = order_key(fmaf(upper_quantile(fminf(((float)k - 0.5f) / (float)NT, 0.5f)), sd, mu));
        int step = 0;
#pragma unroll 1
        while (clo != kk && hi - lo > 1ull) {
            const uint32_t span = (uint32_t)(hi - lo - 1ull);  // probes lie in (lo, hi)
            uint32_t mid;
            if (step == 0 && guess > lo && (unsigned long long)guess < hi) {
                mid = guess;
            } else {
                uint32_t d = (step & 1) ? span / 2u + 1u
                                        : (uint32_t)((float)span * ((float)(clo - kk) / (float)(clo - chi))) + 1u;
                if (d > span) d = span;
                mid = lo + d;
            }
            const uint32_t cmid = __reduce_add_sync(0xFFFFFFFFu, count_ge<TKF_CL>(key, mid));
            if (cmid >= kk) { lo = mid; clo = cmid; } else { hi = mid; chi = cmid; }
            ++step;
            if (clo != kk && clo - chi <= 32u) {
                // band finish: the <= 32 keys in [lo, hi) one per lane; the (k - chi)-th largest
                // of them is the answer
                uint32_t nb = 0;
#pragma unroll
                for (int q = 0; q < TKF_CL; ++q) nb += (key[q] >= lo && (unsigned long long)key[q] < hi) ? 1u : 0u;
                uint32_t pb = nb;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t a = __shfl_up_sync(0xFFFFFFFFu, pb, o);
                    if (lane >= o) pb += a;
                }
                pb -= nb;
                __shared__ uint32_t s_band[TKF_WARPS][32];
#pragma unroll
                for (int q = 0; q < TKF_CL; ++q)
                    if (key[q] >= lo && (unsigned long long)key[q] < hi) s_band[w][pb++] = key[q];
                __syncwarp();
                const uint32_t nbt = clo - chi, needb = kk - chi;
                const uint32_t mine = (uint32_t)lane < nbt ? s_band[w][lane] : 0u;
                uint32_t ngt_b = 0, nge_b = 0;
#pragma unroll 8
                for (int i2 = 0; i2 < 32; ++i2) {
                    const uint32_t o = (uint32_t)i2 < nbt ? s_band[w][i2] : 0u;
                    ngt_b += ((uint32_t)i2 < nbt && o > mine) ? 1u : 0u;
                    nge_b += ((uint32_t)i2 < nbt && o >= mine) ? 1u : 0u;
                }
                const bool hit = (uint32_t)lane < nbt && ngt_b < needb && needb <= nge_b;
                const uint32_t hb = __ballot_sync(0xFFFFFFFFu, hit);
                lo = __shfl_sync(0xFFFFFFFFu, mine, __ffs(hb) - 1);
                __syncwarp();
                break;
            }
        }
        // T = the k-th largest key: the smallest candidate key >= lo
        uint32_t tmin = 0xFFFFFFFFu;
#pragma unroll
        for (int q = 0; q < TKF_CL; ++q)
            if (key[q] >= lo) tmin = min(tmin, key[q]);
        T = __reduce_min_sync(0xFFFFFFFFu, tmin);
        // bitmaps of the candidates > T and == T
#pragma unroll
        for (int q = lane; q < NW; q += 32) { s_gt[w][q] = 0u; s_eq[w][q] = 0u; }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < TKF_CL; ++q)
            if (key[q] >= T && key[q] != 0u) {
                const uint32_t j = jj[q];
                atomicOr(key[q] > T ? &s_gt[w][j >> 5] : &s_eq[w][j >> 5], 1u << (j & 31));
            }
    } else {
        uint32_t key[4 * V];
#pragma unroll
        for (int b = 0; b < 4 * V; ++b) key[b] = 128 * (b >> 2) + 4 * lane + (b & 3) < NT ? order_key(x[b]) : 0u;
        T = kth_largest<4 * V>(key, kk);
#pragma unroll
        for (int q = lane; q < NW; q += 32) { s_gt[w][q] = 0u; s_eq[w][q] = 0u; }
        __syncwarp();
#pragma unroll
        for (int b = 0; b < 4 * V; ++b)
            if (key[b] >= T && key[b] != 0u) {
                const uint32_t j = 128 * (b >> 2) + 4 * lane + (b & 3);
                atomicOr(key[b] > T ? &s_gt[w][j >> 5] : &s_eq[w][j >> 5], 1u << (j & 31));
            }
    }
    __syncwarp();
    // ordered output: lane l owns bitmap words [l*WPL, (l+1)*WPL) (key tiles in index order)
    constexpr int WPL = (NW + 31) / 32;
    uint32_t gw[WPL], ew[WPL], ngt = 0, neq = 0;
#pragma unroll
    for (int q = 0; q < WPL; ++q) {
        const int wi = lane * WPL + q;
        gw[q] = wi < NW ? s_gt[w][wi] : 0u;
        ew[q] = wi < NW ? s_eq[w][wi] : 0u;
        ngt += __popc(gw[q]);
        neq += __popc(ew[q]);
    }
    uint32_t gex = ngt, eex = neq;  // inclusive, then exclusive prefix sums over lanes
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a = __shfl_up_sync(0xFFFFFFFFu, gex, o), b = __shfl_up_sync(0xFFFFFFFFu, eex, o);
        if (lane >= o) { gex += a; eex += b; }
    }
    gex -= ngt;
    eex -= neq;
    const uint32_t gt_total = __shfl_sync(0xFFFFFFFFu, gex + ngt, 31);
    const uint32_t need = kk - gt_total;  // keys == T to take, lowest indices first
    int take = (int)need - (int)eex;      // this lane's share of them
#pragma unroll
    for (int q = 0; q < WPL; ++q) {
        uint32_t e = ew[q], kept = 0;
        while (e && take > 0) {
            const uint32_t bit = e & (0u - e);
            kept |= bit;
            e ^= bit;
            --take;
        }
        gw[q] |= kept;
    }
    uint32_t nsel = 0;
#pragma unroll
    for (int q = 0; q < WPL; ++q) nsel += __popc(gw[q]);
    uint32_t pos = nsel;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a = __shfl_up_sync(0xFFFFFFFFu, pos, o);
        if (lane >= o) pos += a;
    }
    pos -= nsel;
    int32_t *out = idx + (size_t)row * k;
#pragma unroll
    for (int q = 0; q < WPL; ++q) {
        uint32_t m = gw[q];
        const int jb = (lane * WPL + q) * 32;
        while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            out[pos++] = jb + b;
        }
    }
}

}  // namespace

template <int C>
static veda_status launch_topk_warp(const float *scores, int rows, int NT, int k, int32_t *idx, cudaStream_t s)
{
    topk_warp_kernel<C><<<(rows + TKW_WARPS - 1) / TKW_WARPS, TKW_WARPS * 32, 0, s>>>(scores, rows, NT, k, idx);
    count_launch();
    return check_launch("select_topk");
}

veda_status launch_topk(const float *scores, int Hh, int NT, int k, int32_t *idx, cudaStream_t s)
{
    const int rows = Hh * NT;
    if (NT <= 32 * 4) return launch_topk_warp<4>(scores, rows, NT, k, idx, s);
    if (NT <= 32 * 64) {
        const int grid = (rows + TKF_WARPS - 1) / TKF_WARPS;
        if (NT <= 128 * 4)
            topk_filter_kernel<4><<<grid, TKF_WARPS * 32, 0, s>>>(scores, rows, NT, k, idx);
        else if (NT <= 128 * 8)
            topk_filter_kernel<8><<<grid, TKF_WARPS * 32, 0, s>>>(scores, rows, NT, k, idx);
        else
            topk_filter_kernel<16><<<grid, TKF_WARPS * 32, 0, s>>>(scores, rows, NT, k, idx);
        count_launch();
        return check_launch("select_topk");
    }
    const size_t smem = (size_t)NT * sizeof(uint32_t);
    if (smem > 200 * 1024) return fail(VEDA_ERR_SHAPE, "select_topk: n_tiles=%d too large", NT);
    if (smem > 48 * 1024) {  // per launch: the attribute belongs to the current device's context
        cudaError_t e = cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
    topk_kernel<<<rows, TK_THREADS, smem, s>>>(scores, NT, k, idx);
    count_launch();
    return check_launch("select_topk");
}

}  // namespace veda
