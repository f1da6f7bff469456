// attn_fwd_alt.cu -- opt-in attention schedules, measured against the default two-slot
// kernel of attn_fwd.cu and kept behind VEDA_ATTN (profiles/r01_attn_experiments.md):
//   hs  64-key half-steps: S of one half per slot, P double-buffered in TMEM (842 TFLOP/s)
//   ps  P in shared memory, P V as an SS MMA, QK(t+1) issued at S_FREE(t) (1077 TFLOP/s)
// Both compute Eq. 2 over the kept tiles exactly as the default kernel
// and pass the same parity tests (tests/test_gpu_parity.py::test_alt_schedule_parity).
#include "attn_common.cuh"

namespace veda {
namespace attn {
using namespace sm100;

// ==========================================================================================
// Half-step schedule ("hs", VEDA_ATTN=hs): each kept key tile is processed as two halves of
// B/2 keys.  Per slot the TMEM holds S for ONE half (B/2 columns), P in two separate
// buffers (B/4 columns each) and O (D columns): 2 x (64 + 64 + 128) = 512 at B = D = 128.
// Because S is free as soon as the softmax has copied it to registers (S_FREE) and P lives
// in its own double buffer, QK of the next half never waits for P V of the current one:
// the MMA issues QK(g+1) during softmax(g), and softmax(g+1) starts as soon as softmax(g)
// ends.  Static MMA order per half-step g: QK(s, g+1) for both slots, then PV(s, g) for both
// slots; ring stages are committed free by the MMA thread (K after its 2nd half's QK, V
// after its 2nd half's PV).  Producer order: K(s,0); then per tile t: V(s,t), K(s,t+1).
// The half-step softmax holds 64 scores per thread (not 128), so registers move from the
// softmax warpgroups to the control warpgroup, whose MMA thread keeps per-slot state for
// both slots (104 + 2 x 200 = 504 per thread slot, as 72 + 2 x 216).
constexpr int REGS_CTRL_HS = 104, REGS_SOFTMAX_HS = 200;

template <int B, int D>
struct GeoHS {
    static constexpr int HB = B / 2;                  // keys per half
    static constexpr int QCHUNK = 128 * 128;
    static constexpr int Q_BYTES = QCHUNK * (D / 64);
    static constexpr int KCHUNK = B * 128;
    static constexpr int TILE_BYTES = KCHUNK * (D / 64);
    static constexpr int NST_FIT = (VEDA_RING_BUDGET_KB * 1024 - NSLOT * Q_BYTES) / TILE_BYTES;
    static constexpr int NST = NST_FIT > 8 ? 8 : NST_FIT;
    static constexpr int MW = B / 32;
    static constexpr int NBAR = 2 * NST + 9 * NSLOT;
    static constexpr int SMEM = NSLOT * Q_BYTES + NST * TILE_BYTES + NBAR * 8 + 16 + 1024;
    // TMEM columns inside a slot's 256
    static constexpr int T_S = 0, T_P0 = 64, T_P1 = 96, T_O = 128;
    static_assert(HB <= 64 && HB / 2 <= 32 && D <= 128, "half-step TMEM layout");
    static_assert(NST >= 3, "ring too shallow");
};

template <int B, int D, bool TOK>
__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_attn_fwd_hs_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                              const __grid_constant__ CUtensorMap tmV, const Params p,
                              const __grid_constant__ TokParams tp)
{
    using G = GeoHS<B, D>;
    constexpr int HB = G::HB;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sRing = sQ + NSLOT * G::Q_BYTES;
    const uint32_t sBar = sRing + G::NST * G::TILE_BYTES;
    uint32_t *tmem_slot =
        reinterpret_cast<uint32_t *>(smem + NSLOT * G::Q_BYTES + G::NST * G::TILE_BYTES + G::NBAR * 8);
#define H_RING_FULL(i) (sBar + 8u * (i))
#define H_RING_EMPTY(i) (sBar + 8u * (G::NST + (i)))
#define H_BAR(k, s) (sBar + 8u * (2 * G::NST + (k) * NSLOT + (s)))
#define H_Q_FULL(s) H_BAR(0, s)
#define H_Q_EMPTY(s) H_BAR(1, s)
#define H_S_FULL(s) H_BAR(2, s)
#define H_S_FREE(s) H_BAR(3, s)
#define H_P_FULL(s, b) H_BAR(4 + (b), s)
#define H_P_EMPTY(s, b) H_BAR(6 + (b), s)
#define H_O_FULL(s) H_BAR(8, s)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (B < 128) {
        uint4 *q4 = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < NSLOT * G::Q_BYTES / 16; i += NTHREADS) q4[i] = make_uint4(0, 0, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G::NST; ++i) {
            mbar_init(H_RING_FULL(i), 1);
            mbar_init(H_RING_EMPTY(i), 1);
        }
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(H_Q_FULL(s), 1);
            mbar_init(H_Q_EMPTY(s), 1);
            mbar_init(H_S_FULL(s), 1);
            mbar_init(H_S_FREE(s), 128);
            mbar_init(H_P_FULL(s, 0), 128);
            mbar_init(H_P_FULL(s, 1), 128);
            mbar_init(H_P_EMPTY(s, 0), 1);
            mbar_init(H_P_EMPTY(s, 1), 1);
            mbar_init(H_O_FULL(s), 1);
        }
        fence_barrier_init();
        if (!TOK) {
            tma_prefetch_desc(&tmQ);
            tma_prefetch_desc(&tmK);
            tma_prefetch_desc(&tmV);
        }
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    const int NT = p.NT, K = p.k, total = p.unit0 + p.total_units;  // units end
    const int gslots = gridDim.x * NSLOT;
    const int rounds = (p.total_units + gslots - 1) / gslots;
#define H_UNIT(r, s) (p.unit0 + (r) * gslots + blockIdx.x * NSLOT + (s))

    if (warp < 4) {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS_CTRL_HS));
#endif
        if (warp == 0) {
            // ============================ TMA producer ============================
            if (lane == 0) {
                uint32_t stage = 0, ph = 0, qe_bits = 0;
                auto load_tile = [&](const CUtensorMap *tm, int h, int j) {
                    mbar_wait(H_RING_EMPTY(stage), ph ^ 1);
                    mbar_expect_tx(H_RING_FULL(stage), G::TILE_BYTES);
                    if (TOK)
                        tma_tile_tok<D / 64>(sRing + stage * G::TILE_BYTES, G::KCHUNK, tm == &tmK ? tp.k : tp.v, tp,
                                             h, j, H_RING_FULL(stage));
                    else
#pragma unroll
                        for (int c = 0; c < D / 64; ++c)
                            tma_load_2d(sRing + stage * G::TILE_BYTES + c * G::KCHUNK, tm, c * 64, (h * NT + j) * B,
                                        H_RING_FULL(stage));
                    if (++stage == G::NST) { stage = 0; ph ^= 1; }
                };
                for (int r = 0; r < rounds; ++r) {
                    int u[NSLOT], hh[NSLOT];
                    bool act[NSLOT];
                    const int32_t *il[NSLOT];
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        u[s] = H_UNIT(r, s);
                        act[s] = u[s] < total;
                        hh[s] = act[s] ? u[s] / NT : 0;
                        il[s] = p.idx + (size_t)(act[s] ? u[s] : 0) * K;
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!act[s]) continue;
                        mbar_wait(H_Q_EMPTY(s), ((qe_bits >> s) & 1u) ^ 1u);
                        qe_bits ^= 1u << s;
                        mbar_expect_tx(H_Q_FULL(s), B * D * 2);
                        if (TOK)
                            tma_tile_tok<D / 64>(sQ + s * G::Q_BYTES, G::QCHUNK, tp.q, tp, hh[s], u[s] - hh[s] * NT,
                                                 H_Q_FULL(s));
                        else
                            for (int c = 0; c < D / 64; ++c)
                                tma_load_2d(sQ + s * G::Q_BYTES + c * G::QCHUNK, &tmQ, c * 64, u[s] * B, H_Q_FULL(s));
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s)
                        if (act[s]) load_tile(&tmK, hh[s], __ldg(il[s]));
                    for (int t = 0; t < K; ++t) {
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if (act[s]) load_tile(&tmV, hh[s], __ldg(il[s] + t));
                        if (t + 1 < K)
#pragma unroll
                            for (int s = 0; s < NSLOT; ++s)
                                if (act[s]) load_tile(&tmK, hh[s], __ldg(il[s] + t + 1));
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            // ============================ MMA issuer ============================
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, HB, 0, 0);
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D, 0, 1);
            uint32_t stage = 0, ph = 0, qf_bits = 0;
            uint32_t sfree_cnt[NSLOT] = {0, 0}, pfull_cnt[NSLOT] = {0, 0};
            bool have_prev[NSLOT] = {false, false};  // an un-waited S_FREE of the previous unit's last half
            auto next_stage = [&](uint32_t &st, uint32_t &sp) {
                st = stage;
                sp = ph;
                if (++stage == G::NST) { stage = 0; ph ^= 1; }
            };
            // S(half) = Q K_half^T: keys [half*HB, half*HB + HB) of the tile in stage st
            auto issue_qk = [&](int s, uint32_t st, int half) {
                // shfl from lane 0: lets ptxas treat the operands as warp-uniform (UR registers,
                // MMAs back to back) instead of converting them per MMA
                const uint64_t ad0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sQ + s * G::Q_BYTES, 16, 1024), 0);
                const uint64_t bd0 = __shfl_sync(
                    0xFFFFFFFFu, sdesc_sw128(sRing + st * G::TILE_BYTES + (uint32_t)(half * HB * 128), 16, 1024), 0);
                const uint32_t tS = __shfl_sync(0xFFFFFFFFu, tbase + s * 256 + G::T_S, 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint64_t ao = (uint64_t)(((kk >> 2) * G::QCHUNK + (kk & 3) * 32) >> 4);
                    const uint64_t bo = (uint64_t)(((kk >> 2) * G::KCHUNK + (kk & 3) * 32) >> 4);
                    mma_ss_w(tS, ad0 + ao, bd0 + bo, idesc_qk, kk > 0 ? 1u : 0u);
                }
            };
            // O += P(half) V_half: P from TMEM buffer half&1... (global half parity), V keys of the half
            auto issue_pv = [&](int s, uint32_t st, int half, int pbuf, bool first) {
                const uint64_t vd0 = __shfl_sync(
                    0xFFFFFFFFu,
                    sdesc_sw128(sRing + st * G::TILE_BYTES + (uint32_t)(half * HB * 128), G::KCHUNK, 1024), 0);
                const uint32_t tP = __shfl_sync(0xFFFFFFFFu, tbase + s * 256 + (pbuf ? G::T_P1 : G::T_P0), 0);
                const uint32_t tO = __shfl_sync(0xFFFFFFFFu, tbase + s * 256 + G::T_O, 0);
#pragma unroll
                for (int kk = 0; kk < HB / 16; ++kk)  // 16 keys = 16 rows of 128 B of the V half
                    mma_ts_w(tO, tP + kk * 8, vd0 + (uint64_t)((kk * 2048) >> 4), idesc_pv, (!first || kk > 0) ? 1u : 0u);
            };
            uint32_t kst[NSLOT] = {0, 0}, kph[NSLOT] = {0, 0}, vst[NSLOT] = {0, 0}, vph[NSLOT] = {0, 0};
            for (int r = 0; r < rounds; ++r) {
                uint32_t act = 0;
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) act |= (H_UNIT(r, s) < total ? 1u : 0u) << s;
                // prologue: half 0 of tile 0 (after the previous unit's last S is in registers)
#pragma unroll
                for (int s = 0; s < NSLOT; ++s)
                    if ((act >> s) & 1u) next_stage(kst[s], kph[s]);
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) {
                    if (!((act >> s) & 1u)) continue;
                    if (have_prev[s]) { mbar_wait(H_S_FREE(s), sfree_cnt[s] & 1u); ++sfree_cnt[s]; }
                    mbar_wait(H_Q_FULL(s), (qf_bits >> s) & 1u);
                    qf_bits ^= 1u << s;
                    mbar_wait(H_RING_FULL(kst[s]), kph[s]);
                    tc_fence_after();
                    issue_qk(s, kst[s], 0);
                    tc_commit_w(H_S_FULL(s));
                }
                const int NH = 2 * K;
                for (int g = 0; g < NH; ++g) {
                    const int trs = r * NH + g;
                    if (lane == 0) TR(0, trs, 0);
                    // QK of half g+1 for both slots, once each slot's S(g) is in registers
                    if (g + 1 < NH) {
                        const int hn = (g + 1) & 1, tn = (g + 1) >> 1;
                        (void)tn;
                        if (hn == 0) {
#pragma unroll
                            for (int s = 0; s < NSLOT; ++s)
                                if ((act >> s) & 1u) next_stage(kst[s], kph[s]);
                        }
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s) {
                            if (!((act >> s) & 1u)) continue;
                            mbar_wait(H_S_FREE(s), sfree_cnt[s] & 1u);
                            ++sfree_cnt[s];
                            if (hn == 0) mbar_wait(H_RING_FULL(kst[s]), kph[s]);
                            tc_fence_after();
                            issue_qk(s, kst[s], hn);
                            tc_commit_w(H_S_FULL(s));
                            if (hn == 1) tc_commit_w(H_RING_EMPTY(kst[s]));  // both halves of this K tile issued
                            if (g + 1 == NH - 1) tc_commit_w(H_Q_EMPTY(s));
                        }
                    }
                    if (lane == 0) TR(0, trs, 1);
                    // P V of half g for both slots
                    const int h = g & 1;
                    if (h == 0) {
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if ((act >> s) & 1u) next_stage(vst[s], vph[s]);
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!((act >> s) & 1u)) continue;
                        // one P_FULL per P buffer: a single barrier could complete twice (halves g
                        // and g+1) before this wait, as QK(g+1) is already issued
                        mbar_wait(H_P_FULL(s, pfull_cnt[s] & 1u), (pfull_cnt[s] >> 1) & 1u);
                        ++pfull_cnt[s];
                        if (lane == 0) TR(0, trs, 2 + s);
                        if (h == 0) mbar_wait(H_RING_FULL(vst[s]), vph[s]);
                        tc_fence_after();
                        issue_pv(s, vst[s], h, g & 1, g == 0);
                        tc_commit_w(H_P_EMPTY(s, g & 1));
                        if (h == 1) tc_commit_w(H_RING_EMPTY(vst[s]));  // both halves of this V tile issued
                        if (g == NH - 1) tc_commit_w(H_O_FULL(s));
                    }
                    if (lane == 0) TR(0, trs, 4);
                }
#pragma unroll
                for (int s = 0; s < NSLOT; ++s)
                    if ((act >> s) & 1u) have_prev[s] = true;
            }
            __syncwarp();
        }
    } else {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_SOFTMAX_HS));
#endif
        // ============================ softmax warpgroups ============================
        const int slot = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const uint32_t tSl = tbase + lane_off + slot * 256;
        const uint32_t tS = tSl + G::T_S, tO = tSl + G::T_O;
        const float sl2 = p.scale_log2;
        uint32_t sfull_cnt = 0, gh = 0, of_ph = 0;  // gh: global half counter of this slot
        for (int r = 0; r < rounds; ++r) {
            const int u = H_UNIT(r, slot);
            if (u >= total) break;
            const int h = u / NT;
            const int32_t *il = p.idx + (size_t)u * K;
            const uint32_t *mbase = p.slot_mask + (size_t)h * NT * G::MW;
            float m = -INFINITY, l = 0.f;
            uint32_t mk[G::MW];
            const int NH = 2 * K;
            for (int g = 0; g < NH; ++g, ++gh) {
                const int half = g & 1;
                if (half == 0) {
                    const int j = __ldg(il + (g >> 1));
#pragma unroll
                    for (int w = 0; w < G::MW; ++w) mk[w] = __ldg(mbase + (size_t)j * G::MW + w);
                }
                const int trs = r * NH + g, trr = 1 + slot * 4 + quarter;
                if (lane == 0) TR(trr, trs, 0);
                mbar_wait(H_S_FULL(slot), sfull_cnt & 1u);
                ++sfull_cnt;
                if (lane == 0) TR(trr, trs, 1);
                tc_fence_after();
                uint32_t sr[HB / 32][32];
#pragma unroll
                for (int c = 0; c < HB / 32; ++c) tmem_ld32(tS + c * 32, sr[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < HB / 32; ++c) reg_fence(sr[c]);
                tc_fence_before();
                mbar_arrive(H_S_FREE(slot));  // S may take the next half's QK
                if (lane == 0) TR(trr, trs, 2);
                // padded key slots of this half -> -inf
#pragma unroll
                for (int c = 0; c < HB / 32; ++c) {
                    const uint32_t word = mk[half * (HB / 32) + c];
                    if (word != 0xFFFFFFFFu) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!((word >> i) & 1u)) sr[c][i] = f2u(-INFINITY);
                    }
                }
                float pm[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pm[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < HB / 32; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) pm[i & 7] = fmaxf(pm[i & 7], u2f(sr[c][i]));
                const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
                const float mnew = fmaxf(m, mx * sl2);
                if (g == 0) {
                    m = mnew;
                } else if (__any_sync(0xFFFFFFFFu, mnew > m + 8.0f)) {
                    const float f = (mnew == -INFINITY) ? 1.f : ex2(m - mnew);
                    // O must be quiescent: P V of the previous half complete (its commit covers
                    // every earlier MMA of the issuing thread)
                    const uint32_t pb = (gh - 1) & 1u, n = (gh - 1 - pb) >> 1;
                    mbar_wait(H_P_EMPTY(slot, pb), n & 1u);
                    tc_fence_after();
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_wait_ld();
                        reg_fence(o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = f2u(u2f(o[i]) * f);
                        tmem_st32(tO + c * 32, o);
                    }
                    l *= f;
                    m = mnew;
                }
                if (lane == 0) TR(trr, trs, 3);
                const float mu = (m == -INFINITY) ? 0.f : m;
                float ps[4] = {0.f, 0.f, 0.f, 0.f};
                uint32_t pk[HB / 2];
#pragma unroll
                for (int i = 0; i < HB / 2; ++i) {
                    const int c = i >> 4, e = (i & 15) * 2;
                    float x0, x1;
                    ffma2_bc(x0, x1, u2f(sr[c][e]), u2f(sr[c][e + 1]), sl2, -mu);
                    const float a = ex2(x0), b2 = ex2(x1);
                    fadd2_acc(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, b2);
                    pk[i] = pack_bf16(a, b2);
                }
                l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
                if (lane == 0) TR(trr, trs, 4);
                // P buffer gh&1 is free once P V of half gh-2 completed
                const uint32_t pbuf = gh & 1u;
                if (gh >= 2) {
                    const uint32_t n = (gh - 2 - pbuf) >> 1;
                    mbar_wait(H_P_EMPTY(slot, pbuf), n & 1u);
                }
                if (lane == 0) TR(trr, trs, 5);
                const uint32_t tP = tSl + (pbuf ? G::T_P1 : G::T_P0);
                if (HB / 2 == 32) {
                    uint32_t (&pk32)[32] = *reinterpret_cast<uint32_t (*)[32]>(pk);
                    tmem_st32(tP, pk32);
                } else {
                    uint32_t (&pk16)[16] = *reinterpret_cast<uint32_t (*)[16]>(pk);
                    tmem_st16(tP, pk16);
                }
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(H_P_FULL(slot, pbuf));
                if (lane == 0) TR(trr, trs, 6);
            }
            // ---- epilogue: O / l -> bf16, padded query rows -> 0
            mbar_wait(H_O_FULL(slot), of_ph);
            of_ph ^= 1;
            tc_fence_after();
            bool qvalid = false;
            if (row < B) qvalid = (__ldg(p.slot_mask + (size_t)u * G::MW + (row >> 5)) >> (row & 31)) & 1u;
            const float inv = (qvalid && l > 0.f) ? 1.f / l : 0.f;
            uint16_t *orow = p.out + ((size_t)u * B + (row < B ? row : 0)) * D;
            bool store = row < B;
            if (TOK) {
                const TileOrigin o = tile_origin(tp, h, u - h * NT);
                const int lpw = __ffs(tp.pw[o.c]) - 1, lphw = lpw + __ffs(tp.ph[o.c]) - 1;
                const int t = o.t0 + (row >> lphw), hq = o.h0 + ((row >> lpw) & (tp.ph[o.c] - 1)),
                          w = o.w0 + (row & (tp.pw[o.c] - 1));
                store = store && qvalid;
                orow = p.out + (size_t)h * tp.o_hs + (((size_t)t * tp.H + hq) * tp.W + w) * tp.o_ts;
            }
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + c * 32, o);
                tmem_wait_ld();
                reg_fence(o);
                if (store) {
                    uint32_t pk2[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) pk2[i] = pack_bf16(u2f(o[2 * i]) * inv, u2f(o[2 * i + 1]) * inv);
                    uint4 *dst = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        dst[v] = make_uint4(pk2[4 * v], pk2[4 * v + 1], pk2[4 * v + 2], pk2[4 * v + 3]);
                }
            }
            if (p.lse != nullptr && row < B)
                p.lse[(size_t)u * B + row] = (qvalid && l > 0.f) ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
        }
    }
#undef H_UNIT
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, TMEM_COLS);
    }
#undef H_RING_FULL
#undef H_RING_EMPTY
#undef H_BAR
#undef H_Q_FULL
#undef H_Q_EMPTY
#undef H_S_FULL
#undef H_S_FREE
#undef H_P_FULL
#undef H_P_EMPTY
#undef H_O_FULL
}

// ==========================================================================================
// P-in-shared-memory schedule ("ps", VEDA_ATTN=ps; B = d = 128): the softmax writes P (bf16,
// the SW128 K-major image a TMA load of a 128x128 tile would produce) to a per-slot shared
// buffer and P V is an SS MMA, so S is free as soon as the softmax has copied it to
// registers: QK(t+1) is issued at S_FREE(t), during softmax(t), instead of after P V(t)
// (the chain of the two-slot kernel).  TMEM per slot: S 128 + O 128 columns.  Shared
// memory: Q 2 x 32 KB + P 2 x 32 KB + a 3-stage K/V ring.  Static MMA order per kept tile t:
// QK(s, t+1) for both slots, then PV(s, t) for both slots; ring stages are committed free by
// the MMA thread.  Producer order: Q, K(s,0); then per tile t: K(s,t+1), V(s,t).
template <int B, int D>
struct GeoPS {
    static constexpr int QCHUNK = 128 * 128;  // 64-column chunk of a 128-row bf16 tile
    static constexpr int Q_BYTES = QCHUNK * (D / 64);
    static constexpr int P_BYTES = QCHUNK * (B / 64);
    static constexpr int KCHUNK = B * 128;
    static constexpr int TILE_BYTES = KCHUNK * (D / 64);
    static constexpr int NST_FIT = (VEDA_RING_BUDGET_KB * 1024 - NSLOT * (Q_BYTES + P_BYTES)) / TILE_BYTES;
    static constexpr int NST = NST_FIT > 8 ? 8 : NST_FIT;
    static constexpr int MW = B / 32;
    static constexpr int NBAR = 2 * NST + 8 * NSLOT;
    static constexpr int SMEM = NSLOT * (Q_BYTES + P_BYTES) + NST * TILE_BYTES + NBAR * 8 + 16 + 1024;
    static_assert(NST >= 3, "ring too shallow");
};

template <int B, int D, bool TOK>
__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_attn_fwd_ps_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                              const __grid_constant__ CUtensorMap tmV, const Params p,
                              const __grid_constant__ TokParams tp)
{
    static_assert(B == 128 && D == 128, "ps schedule: B = d = 128 only");
    using G = GeoPS<B, D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sP = sQ + NSLOT * G::Q_BYTES;
    const uint32_t sRing = sP + NSLOT * G::P_BYTES;
    const uint32_t sBar = sRing + G::NST * G::TILE_BYTES;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + NSLOT * (G::Q_BYTES + G::P_BYTES) +
                                                       G::NST * G::TILE_BYTES + G::NBAR * 8);
#define X_RING_FULL(i) (sBar + 8u * (i))
#define X_RING_EMPTY(i) (sBar + 8u * (G::NST + (i)))
#define X_BAR(k, s) (sBar + 8u * (2 * G::NST + (k) * NSLOT + (s)))
#define X_Q_FULL(s) X_BAR(0, s)
#define X_Q_EMPTY(s) X_BAR(1, s)
#define X_S_FULL(s) X_BAR(2, s)
#define X_S_FREE(s) X_BAR(3, s)
#define X_P_FULL(s) X_BAR(4, s)
#define X_P_EMPTY(s) X_BAR(5, s)
#define X_O_FULL(s) X_BAR(6, s)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G::NST; ++i) {
            mbar_init(X_RING_FULL(i), 1);
            mbar_init(X_RING_EMPTY(i), 1);
        }
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(X_Q_FULL(s), 1);
            mbar_init(X_Q_EMPTY(s), 1);
            mbar_init(X_S_FULL(s), 1);
            mbar_init(X_S_FREE(s), 128);
            mbar_init(X_P_FULL(s), 128);
            mbar_init(X_P_EMPTY(s), 1);
            mbar_init(X_O_FULL(s), 1);
        }
        fence_barrier_init();
        if (!TOK) {
            tma_prefetch_desc(&tmQ);
            tma_prefetch_desc(&tmK);
            tma_prefetch_desc(&tmV);
        }
    }
    if (warp == 1) {
        tmem_alloc(smem_u32(tmem_slot), TMEM_COLS);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tmem_slot;
    const int NT = p.NT, K = p.k, total = p.unit0 + p.total_units;  // units end
    const int gslots = gridDim.x * NSLOT;
    const int rounds = (p.total_units + gslots - 1) / gslots;
#define X_UNIT(r, s) (p.unit0 + (r) * gslots + blockIdx.x * NSLOT + (s))

    if (warp < 4) {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS_CTRL));
#endif
        if (warp == 0) {
            // ============================ TMA producer ============================
            if (lane == 0) {
                uint32_t stage = 0, ph = 0, qe_bits = 0;
                auto load_tile = [&](const CUtensorMap *tm, int h, int j) {
                    mbar_wait(X_RING_EMPTY(stage), ph ^ 1);
                    mbar_expect_tx(X_RING_FULL(stage), G::TILE_BYTES);
                    if (TOK)
                        tma_tile_tok<D / 64>(sRing + stage * G::TILE_BYTES, G::KCHUNK, tm == &tmK ? tp.k : tp.v, tp,
                                             h, j, X_RING_FULL(stage));
                    else
#pragma unroll
                        for (int c = 0; c < D / 64; ++c)
                            tma_load_2d(sRing + stage * G::TILE_BYTES + c * G::KCHUNK, tm, c * 64, (h * NT + j) * B,
                                        X_RING_FULL(stage));
                    if (++stage == G::NST) { stage = 0; ph ^= 1; }
                };
                for (int r = 0; r < rounds; ++r) {
                    int u[NSLOT], hh[NSLOT];
                    bool act[NSLOT];
                    const int32_t *il[NSLOT];
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        u[s] = X_UNIT(r, s);
                        act[s] = u[s] < total;
                        hh[s] = act[s] ? u[s] / NT : 0;
                        il[s] = p.idx + (size_t)(act[s] ? u[s] : 0) * K;
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!act[s]) continue;
                        mbar_wait(X_Q_EMPTY(s), ((qe_bits >> s) & 1u) ^ 1u);
                        qe_bits ^= 1u << s;
                        mbar_expect_tx(X_Q_FULL(s), B * D * 2);
                        if (TOK)
                            tma_tile_tok<D / 64>(sQ + s * G::Q_BYTES, G::QCHUNK, tp.q, tp, hh[s], u[s] - hh[s] * NT,
                                                 X_Q_FULL(s));
                        else
                            for (int c = 0; c < D / 64; ++c)
                                tma_load_2d(sQ + s * G::Q_BYTES + c * G::QCHUNK, &tmQ, c * 64, u[s] * B, X_Q_FULL(s));
                    }
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s)
                        if (act[s]) load_tile(&tmK, hh[s], __ldg(il[s]));
                    for (int t = 0; t < K; ++t) {
                        if (t + 1 < K)
#pragma unroll
                            for (int s = 0; s < NSLOT; ++s)
                                if (act[s]) load_tile(&tmK, hh[s], __ldg(il[s] + t + 1));
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if (act[s]) load_tile(&tmV, hh[s], __ldg(il[s] + t));
                    }
                }
            }
            __syncwarp();
        } else if (warp == 1) {
            // ============================ MMA issuer ============================
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, B, 0, 0);  // Q, K both K-major
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D, 0, 1);  // P K-major (smem), V MN-major
            uint32_t stage = 0, ph = 0, qf_bits = 0;
            uint32_t sfree_cnt[NSLOT] = {0, 0}, pfull_cnt[NSLOT] = {0, 0};
            bool have_prev[NSLOT] = {false, false};
            auto next_stage = [&](uint32_t &st, uint32_t &sp) {
                st = stage;
                sp = ph;
                if (++stage == G::NST) { stage = 0; ph ^= 1; }
            };
            auto issue_qk = [&](int s, uint32_t st) {
                // operands broadcast from lane 0: ptxas keeps them uniform (MMAs back to back)
                const uint64_t ad0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sQ + s * G::Q_BYTES, 16, 1024), 0);
                const uint64_t bd0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sRing + st * G::TILE_BYTES, 16, 1024), 0);
                const uint32_t tS = __shfl_sync(0xFFFFFFFFu, tbase + s * 256, 0);
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint64_t ao = (uint64_t)(((kk >> 2) * G::QCHUNK + (kk & 3) * 32) >> 4);
                    const uint64_t bo = (uint64_t)(((kk >> 2) * G::KCHUNK + (kk & 3) * 32) >> 4);
                    mma_ss_w(tS, ad0 + ao, bd0 + bo, idesc_qk, kk > 0 ? 1u : 0u);
                }
            };
            auto issue_pv = [&](int s, uint32_t st, bool first) {
                const uint64_t pd0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sP + s * G::P_BYTES, 16, 1024), 0);
                const uint64_t vd0 = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sRing + st * G::TILE_BYTES, G::KCHUNK, 1024), 0);
                const uint32_t tO = __shfl_sync(0xFFFFFFFFu, tbase + s * 256 + 128, 0);
#pragma unroll
                for (int kk = 0; kk < B / 16; ++kk) {
                    const uint64_t ao = (uint64_t)(((kk >> 2) * G::QCHUNK + (kk & 3) * 32) >> 4);
                    mma_ss_w(tO, pd0 + ao, vd0 + (uint64_t)((kk * 2048) >> 4), idesc_pv, (!first || kk > 0) ? 1u : 0u);
                }
            };
            uint32_t kst[NSLOT] = {0, 0}, kph[NSLOT] = {0, 0}, vst[NSLOT] = {0, 0}, vph[NSLOT] = {0, 0};
            for (int r = 0; r < rounds; ++r) {
                uint32_t act = 0;
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) act |= (X_UNIT(r, s) < total ? 1u : 0u) << s;
#pragma unroll
                for (int s = 0; s < NSLOT; ++s)
                    if ((act >> s) & 1u) next_stage(kst[s], kph[s]);
#pragma unroll
                for (int s = 0; s < NSLOT; ++s) {
                    if (!((act >> s) & 1u)) continue;
                    if (have_prev[s]) { mbar_wait(X_S_FREE(s), sfree_cnt[s] & 1u); ++sfree_cnt[s]; }
                    mbar_wait(X_Q_FULL(s), (qf_bits >> s) & 1u);
                    qf_bits ^= 1u << s;
                    mbar_wait(X_RING_FULL(kst[s]), kph[s]);
                    tc_fence_after();
                    issue_qk(s, kst[s]);
                    tc_commit_w(X_S_FULL(s));
                    tc_commit_w(X_RING_EMPTY(kst[s]));
                    if (K == 1) tc_commit_w(X_Q_EMPTY(s));
                }
                for (int t = 0; t < K; ++t) {
                    if (lane == 0) TR(0, r * K + t, 0);
                    if (t + 1 < K) {
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s)
                            if ((act >> s) & 1u) next_stage(kst[s], kph[s]);
#pragma unroll
                        for (int s = 0; s < NSLOT; ++s) {
                            if (!((act >> s) & 1u)) continue;
                            mbar_wait(X_S_FREE(s), sfree_cnt[s] & 1u);  // S(t) is in registers
                            ++sfree_cnt[s];
                            mbar_wait(X_RING_FULL(kst[s]), kph[s]);
                            tc_fence_after();
                            issue_qk(s, kst[s]);
                            tc_commit_w(X_S_FULL(s));
                            tc_commit_w(X_RING_EMPTY(kst[s]));
                            if (t + 1 == K - 1) tc_commit_w(X_Q_EMPTY(s));
                        }
                    }
                    if (lane == 0) TR(0, r * K + t, 1);
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s)
                        if ((act >> s) & 1u) next_stage(vst[s], vph[s]);
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (!((act >> s) & 1u)) continue;
                        mbar_wait(X_P_FULL(s), pfull_cnt[s] & 1u);
                        ++pfull_cnt[s];
                        if (lane == 0) TR(0, r * K + t, 2 + s);
                        mbar_wait(X_RING_FULL(vst[s]), vph[s]);
                        if (lane == 0) TR(0, r * K + t, 4 + s);
                        tc_fence_after();
                        issue_pv(s, vst[s], t == 0);
                        tc_commit_w(X_P_EMPTY(s));
                        tc_commit_w(X_RING_EMPTY(vst[s]));
                        if (t == K - 1) tc_commit_w(X_O_FULL(s));
                    }
                }
#pragma unroll
                for (int s = 0; s < NSLOT; ++s)
                    if ((act >> s) & 1u) have_prev[s] = true;
            }
            __syncwarp();
        }
    } else {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_SOFTMAX));
#endif
        // ============================ softmax warpgroups ============================
        const int slot = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const uint32_t tS = tbase + lane_off + slot * 256, tO = tS + 128;
        // this row's 128-byte lines in the two 64-key chunks of the P buffer (SW128: 16-byte
        // unit c of row r sits at unit c ^ (r & 7))
        const uint32_t pRow = sP + slot * G::P_BYTES + row * 128;
        const float sl2 = p.scale_log2;
        uint32_t sfull_cnt = 0, g = 0, of_ph = 0;  // g: this slot's global kept-tile counter
        for (int r = 0; r < rounds; ++r) {
            const int u = X_UNIT(r, slot);
            if (u >= total) break;
            const int h = u / NT;
            const int32_t *il = p.idx + (size_t)u * K;
            const uint32_t *mbase = p.slot_mask + (size_t)h * NT * G::MW;
            float m = -INFINITY, l = 0.f;
            for (int t = 0; t < K; ++t, ++g) {
                const int j = __ldg(il + t);
                uint32_t mk[G::MW];
#pragma unroll
                for (int w = 0; w < G::MW; ++w) mk[w] = __ldg(mbase + (size_t)j * G::MW + w);
                const int trs = r * K + t, trr = 1 + slot * 4 + quarter;
                if (lane == 0) TR(trr, trs, 0);
                mbar_wait(X_S_FULL(slot), sfull_cnt & 1u);
                ++sfull_cnt;
                if (lane == 0) TR(trr, trs, 1);
                tc_fence_after();
                uint32_t sr[B / 32][32];
#pragma unroll
                for (int c = 0; c < B / 32; ++c) tmem_ld32(tS + c * 32, sr[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < B / 32; ++c) reg_fence(sr[c]);
                tc_fence_before();
                mbar_arrive(X_S_FREE(slot));  // S may take QK(t+1)
                if (lane == 0) TR(trr, trs, 2);
                bool full = true;
#pragma unroll
                for (int w = 0; w < G::MW; ++w) full &= (mk[w] == 0xFFFFFFFFu);
                if (!full) {
#pragma unroll
                    for (int c = 0; c < B / 32; ++c)
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (!((mk[c] >> i) & 1u)) sr[c][i] = f2u(-INFINITY);
                }
                float pm[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pm[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < B / 32; ++c)
#pragma unroll
                    for (int i = 0; i < 32; ++i) pm[i & 7] = fmaxf(pm[i & 7], u2f(sr[c][i]));
                const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
                const float mnew = fmaxf(m, mx * sl2);
                // P buffer and O are both quiescent once P V(t-1) completed (P_EMPTY phase g-1)
                if (g > 0) {
                    mbar_wait(X_P_EMPTY(slot), (g - 1) & 1u);
                    tc_fence_after();
                }
                if (lane == 0) TR(trr, trs, 3);
                bool rescale = false;
                if (t == 0) {
                    m = mnew;
                } else if (__any_sync(0xFFFFFFFFu, mnew > m + 8.0f)) {
                    const float f = (mnew == -INFINITY) ? 1.f : ex2(m - mnew);
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_wait_ld();
                        reg_fence(o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = f2u(u2f(o[i]) * f);
                        tmem_st32(tO + c * 32, o);
                    }
                    rescale = true;
                    l *= f;
                    m = mnew;
                }
                const float mu = (m == -INFINITY) ? 0.f : m;
                float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c2 = 0; c2 < B / 64; ++c2) {
                    uint32_t pk[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int c = 2 * c2 + (i >> 4), e = (i & 15) * 2;
                        float x0, x1;
                        ffma2_bc(x0, x1, u2f(sr[c][e]), u2f(sr[c][e + 1]), sl2, -mu);
                        const float a = ex2(x0), b = ex2(x1);
                        fadd2_acc(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, b);
                        pk[i] = pack_bf16(a, b);
                    }
                    // keys 64*c2 .. 64*c2+63: eight 16-byte units of this row's line in chunk c2
#pragma unroll
                    for (int v = 0; v < 8; ++v) {
                        const uint32_t addr = pRow + c2 * G::QCHUNK + (uint32_t)(((v ^ (row & 7)) & 7) << 4);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(pk[4 * v]),
                                     "r"(pk[4 * v + 1]), "r"(pk[4 * v + 2]), "r"(pk[4 * v + 3])
                                     : "memory");
                    }
                }
                l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
                if (lane == 0) TR(trr, trs, 4);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // P visible to the MMA
                if (rescale) tmem_wait_st();
                tc_fence_before();
                mbar_arrive(X_P_FULL(slot));
                if (lane == 0) TR(trr, trs, 5);
            }
            // ---- epilogue: O / l -> bf16, padded query rows -> 0
            mbar_wait(X_O_FULL(slot), of_ph);
            of_ph ^= 1;
            tc_fence_after();
            bool qvalid = false;
            if (row < B) qvalid = (__ldg(p.slot_mask + (size_t)u * G::MW + (row >> 5)) >> (row & 31)) & 1u;
            const float inv = (qvalid && l > 0.f) ? 1.f / l : 0.f;
            uint16_t *orow = p.out + ((size_t)u * B + (row < B ? row : 0)) * D;
            bool store = row < B;
            if (TOK) {
                const TileOrigin o = tile_origin(tp, h, u - h * NT);
                const int lpw = __ffs(tp.pw[o.c]) - 1, lphw = lpw + __ffs(tp.ph[o.c]) - 1;
                const int t = o.t0 + (row >> lphw), hq = o.h0 + ((row >> lpw) & (tp.ph[o.c] - 1)),
                          w = o.w0 + (row & (tp.pw[o.c] - 1));
                store = store && qvalid;
                orow = p.out + (size_t)h * tp.o_hs + (((size_t)t * tp.H + hq) * tp.W + w) * tp.o_ts;
            }
#pragma unroll
            for (int c = 0; c < D / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + c * 32, o);
                tmem_wait_ld();
                reg_fence(o);
                if (store) {
                    uint32_t pk2[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) pk2[i] = pack_bf16(u2f(o[2 * i]) * inv, u2f(o[2 * i + 1]) * inv);
                    uint4 *dst = reinterpret_cast<uint4 *>(orow + c * 32);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        dst[v] = make_uint4(pk2[4 * v], pk2[4 * v + 1], pk2[4 * v + 2], pk2[4 * v + 3]);
                }
            }
            if (p.lse != nullptr && row < B)
                p.lse[(size_t)u * B + row] = (qvalid && l > 0.f) ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
        }
    }
#undef X_UNIT
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, TMEM_COLS);
    }
#undef X_RING_FULL
#undef X_RING_EMPTY
#undef X_BAR
#undef X_Q_FULL
#undef X_Q_EMPTY
#undef X_S_FULL
#undef X_S_FREE
#undef X_P_FULL
#undef X_P_EMPTY
#undef X_O_FULL
}

template <int B, int D, bool TOK>
veda_status launch_alt(int which, const CUtensorMap &mq, const CUtensorMap &mk, const CUtensorMap &mv,
                       const Params &p, const TokParams &tp, int units, cudaStream_t stream)
{
    int grid = (units + NSLOT - 1) / NSLOT;
    const int nsm = num_sms();
    if (grid > nsm) grid = nsm;
    if (which == 1) {
        using GH = GeoHS<B, D>;
        static bool attr = false;
        if (!attr) {
            cudaError_t e = cudaFuncSetAttribute(sparse_attn_fwd_hs_kernel<B, D, TOK>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, GH::SMEM);
            if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
            attr = true;
        }
        sparse_attn_fwd_hs_kernel<B, D, TOK><<<grid, NTHREADS, GH::SMEM, stream>>>(mq, mk, mv, p, tp);
        count_launch();
        return check_launch("sparse_attn_fwd (hs)");
    }
    if constexpr (B == 128 && D == 128) {
        if (which == 2) {
            using GP = GeoPS<B, D>;
            static bool attr = false;
            if (!attr) {
                cudaError_t e = cudaFuncSetAttribute(sparse_attn_fwd_ps_kernel<B, D, TOK>,
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, GP::SMEM);
                if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
                attr = true;
            }
            sparse_attn_fwd_ps_kernel<B, D, TOK><<<grid, NTHREADS, GP::SMEM, stream>>>(mq, mk, mv, p, tp);
            count_launch();
            return check_launch("sparse_attn_fwd (ps)");
        }
    }
    return fail(VEDA_ERR_CONFIG, "attention: schedule %d unavailable for B=%d d=%d", which, B, D);
}

#define VEDA_ALT(B, D, TOK)                                                                                    \
    template veda_status launch_alt<B, D, TOK>(int, const CUtensorMap &, const CUtensorMap &,                 \
                                                const CUtensorMap &, const Params &, const TokParams &, int, \
                                                cudaStream_t);
VEDA_ALT(64, 64, false)
VEDA_ALT(64, 128, false)
VEDA_ALT(128, 64, false)
VEDA_ALT(128, 128, false)
VEDA_ALT(64, 64, true)
VEDA_ALT(64, 128, true)
VEDA_ALT(128, 64, true)
VEDA_ALT(128, 128, true)
#undef VEDA_ALT

}  // namespace attn
}  // namespace veda
