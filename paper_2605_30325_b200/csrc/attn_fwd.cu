// attn_fwd.cu -- tile-skipping FlashAttention forward for sm_100a (B200).
//
// Computes Eq. 2 of the paper: for every (head h, query tile i)
//     O_i = softmax(Q~_i K^_i^T * scale) V^_i,   K^_i / V^_i = concat of the k kept tiles
// visiting ONLY the kept key tiles named by idx[h][i][:] (producer
// fetches "only the selected non-contiguous key/value tiles" into a circular buffer).
//
// B200 design:
//  * persistent, one CTA per SM, 384 threads = 3 warpgroups:
//      warp 0      TMA producer: Q tiles and the kept K/V tiles -> SMEM ring (SWIZZLE_128B)
//      warp 1      MMA issuer (warp-uniform, one elected lane): tcgen05.mma,
//                  S = Q K^T (SS) and O += P V (TS)
//      warps 2-3   ring-stage release for slot 0 / slot 1 (warpgroup 0 gives its spare
//                  registers to the softmax warpgroups with setmaxnreg)
//      warps 4-11  two softmax warpgroups ("slots"), one query tile each, one row per thread
//  * two addressing modes: tiled tensors [Hh][N_T][B][d] (2-D TMA boxes, tiled output), or
//    TOK: tiles gathered from token order by one 5-D TMA box each and output rows stored
//    straight to token order (no tiled copies; the path's mode)
//  * each slot owns 256 TMEM columns: S (fp32, 128 cols; P aliases its first B/2 columns
//    as packed bf16) and O (fp32, D cols).  The two slots work on different query
//    tiles with independent kept lists, so one slot's softmax overlaps the other's MMAs.
//  * online softmax in the log2 domain with lazy rescaling: O (in TMEM) is rescaled
//    only when a row max grows by more than 8 (2^8 head-room in fp32/bf16).
//  * padded key slots (slot_mask bit clear) get -inf; padded query rows are written 0.
//  * ordering: the commit after S_{t} = Q K_t^T also covers the previous O += P_{t-1} V,
//    so when softmax sees S_t, O is quiescent and may be rescaled in place.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "attn_common.cuh"

namespace veda {
namespace attn {
using namespace sm100;

// 32 bytes (words w0 .. w0 + 7 of pk) to global memory in one 256-bit store
__device__ __forceinline__ void st_global_v8(void *dst, const uint32_t (&pk)[16], int w0)
{
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst), "r"(pk[w0]), "r"(pk[w0 + 1]),
                 "r"(pk[w0 + 2]), "r"(pk[w0 + 3]), "r"(pk[w0 + 4]), "r"(pk[w0 + 5]), "r"(pk[w0 + 6]), "r"(pk[w0 + 7])
                 : "memory");
}

// A kept-tile list entry outside [0, n_tiles) (a caller bug; debug mode reports it as
// VEDA_ERR_INDEX) is clamped, so the TMA coordinates and slot-mask reads stay inside the head.
__device__ __forceinline__ int clamp_tile(int j, int NT) { return min(max(j, 0), NT - 1); }

template <int B, int D>
struct Geo {
    static constexpr int QCHUNK = 128 * 128;         // one 64-col chunk of the 128-row Q buffer
    static constexpr int Q_BYTES = QCHUNK * (D / 64);
    static constexpr int KCHUNK = B * 128;           // one 64-col chunk of a B-row K/V tile
    static constexpr int TILE_BYTES = KCHUNK * (D / 64);
    static constexpr int NST_FIT = (VEDA_RING_BUDGET_KB * 1024 - NSLOT * Q_BYTES) / TILE_BYTES;
    static constexpr int NST = NST_FIT > 8 ? 8 : NST_FIT;
    static constexpr int MW = B / 32;
    static constexpr int NPH = B / 64;                // P hand-off halves (64 keys each)
    static constexpr int NBAR = 2 * NST + (4 + NPH) * NSLOT;
    static constexpr int SMEM = NSLOT * Q_BYTES + NST * TILE_BYTES + NBAR * 8 + 16 + 1024;
    static_assert(NST >= 2, "ring too shallow");
};

template <int B, int D, bool TOK>
__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, const Params p,
                           const __grid_constant__ TokParams tp)
{
    using G = Geo<B, D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sRing = sQ + NSLOT * G::Q_BYTES;
    const uint32_t sBar = sRing + G::NST * G::TILE_BYTES;
    uint32_t *tmem_slot =
        reinterpret_cast<uint32_t *>(smem + NSLOT * G::Q_BYTES + G::NST * G::TILE_BYTES + G::NBAR * 8);
    // barrier addresses
#define RING_FULL(i) (sBar + 8u * (i))
#define RING_EMPTY(i) (sBar + 8u * (G::NST + (i)))
#define Q_FULL(s) (sBar + 8u * (2 * G::NST + (s)))
#define Q_EMPTY(s) (sBar + 8u * (2 * G::NST + NSLOT + (s)))
#define S_FULL(s) (sBar + 8u * (2 * G::NST + 2 * NSLOT + (s)))
#define O_FULL(s) (sBar + 8u * (2 * G::NST + 3 * NSLOT + (s)))
#define P_FULL(s, hf) (sBar + 8u * (2 * G::NST + (4 + (hf)) * NSLOT + (s)))

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (B < 128) {  // rows B..127 of the M=128 Q operand are never loaded: keep them zero
        uint4 *q4 = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < NSLOT * G::Q_BYTES / 16; i += NTHREADS) q4[i] = make_uint4(0, 0, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G::NST; ++i) {
            mbar_init(RING_FULL(i), 1);
            mbar_init(RING_EMPTY(i), 1);
        }
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(Q_FULL(s), 1);
            mbar_init(Q_EMPTY(s), 1);
            mbar_init(S_FULL(s), 1);
            for (int hf = 0; hf < G::NPH; ++hf) mbar_init(P_FULL(s, hf), 128);
            mbar_init(O_FULL(s), 1);
        }
        fence_barrier_init();
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
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
    // unit u = h*NT + i; consecutive CTAs/slots take consecutive query tiles of one head (L2 reuse)
#define UNIT_OF(r, s) (p.unit0 + (r) * gslots + blockIdx.x * NSLOT + (s))

    if (warp < 4) {
#ifndef VEDA_NO_SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS_CTRL));
#endif
    if (lane == 0) DBG("w%d ctrl start tbase=%x\n", warp, tbase);
    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            uint32_t stage = 0, ph = 0;
            uint32_t qe_bits = 0;  // per-slot phase bits of Q_EMPTY
            // Load order (the ring is a FIFO; the MMA thread and the release warps follow it):
            //   round 0:  Q(s), K(s, 0) for each slot s
            //   round r, tile t, slot s:  V(s, t), then K(s, t + 1) -- or, at t = K - 1, the next
            //   round's Q(s) and K(s, 0), so the next unit's first QK can follow PV(s, K - 1) at once
            int hh[NSLOT], jv[NSLOT];
            const int32_t *il[NSLOT];
            auto load_q = [&](int s, int u) {
                mbar_wait(Q_EMPTY(s), ((qe_bits >> s) & 1u) ^ 1u);
                qe_bits ^= 1u << s;
                mbar_expect_tx(Q_FULL(s), B * D * 2);
                if (TOK)
                    tma_tile_tok<D / 64>(sQ + s * G::Q_BYTES, G::QCHUNK, tp.q, tp, u / NT, u - (u / NT) * NT, Q_FULL(s));
                else
#pragma unroll
                    for (int c = 0; c < D / 64; ++c)
                        tma_load_2d(sQ + s * G::Q_BYTES + c * G::QCHUNK, &tmQ, c * 64, u * B, Q_FULL(s));
            };
            auto load_tile = [&](const CUtensorMap *tm, int h, int j) {
                mbar_wait(RING_EMPTY(stage), ph ^ 1);
                mbar_expect_tx(RING_FULL(stage), G::TILE_BYTES);
                const int row = (h * NT + j) * B;
                if (TOK)
                    tma_tile_tok<D / 64>(sRing + stage * G::TILE_BYTES, G::KCHUNK, tm == &tmK ? tp.k : tp.v, tp,
                                         h, j, RING_FULL(stage));
                else
#pragma unroll
                    for (int c = 0; c < D / 64; ++c)
                        tma_load_2d(sRing + stage * G::TILE_BYTES + c * G::KCHUNK, tm, c * 64, row,
                                    RING_FULL(stage));
                if (++stage == G::NST) { stage = 0; ph ^= 1; }
            };
            // unit u's index list, head and first K tile into the slot's registers
            auto start_unit = [&](int s, int u) {
                hh[s] = u / NT;
                il[s] = p.idx + (size_t)u * K;
                jv[s] = clamp_tile(__ldg(il[s]), NT);
            };
            // r = -1 is round 0's prologue (Q and first K only); one call site per load kind
            // keeps the producer's code small (the token-layout TMA issue is long)
            for (int r = -1; r < rounds; ++r) {
                for (int t = (r < 0 ? K - 1 : 0); t < K; ++t) {
#pragma unroll
                    for (int s = 0; s < NSLOT; ++s) {
                        if (r >= 0) {
                            if (UNIT_OF(r, s) >= total) continue;
                            load_tile(&tmV, hh[s], jv[s]);
                        }
                        if (t + 1 < K) {
                            jv[s] = clamp_tile(__ldg(il[s] + t + 1), NT);
                        } else {
                            if (UNIT_OF(r + 1, s) >= total) continue;
                            load_q(s, UNIT_OF(r + 1, s));
                            start_unit(s, UNIT_OF(r + 1, s));
                        }
                        load_tile(&tmK, hh[s], jv[s]);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == 2 || warp == 3) {
        // ============================ ring-stage release ============================
        // Warp 2 (slot 0) / warp 3 (slot 1): S_FULL(s) of tile t lands only when QK(s,t)
        // and every earlier MMA of the issuing thread -- in particular PV(s,t-1) -- are
        // complete, so the stages of K(s,t) and V(s,t-1) can go back to the producer at
        // once (O_FULL releases the unit's last V).  Keeping this off the MMA thread and
        // off the softmax keeps stage hold times short with a 5-stage ring.
        if (lane == 0) {
            const int s = warp - 2;
            uint32_t sf_ph = 0, of_ph = 0;
            // global load index of K(s, t) / V(s, t) in the producer's order (see there)
            uint32_t base = (UNIT_OF(0, 1) < total) ? 2 : 1;  // after round 0's first K tiles
            uint32_t gk0 = s;                                  // K(s, 0) of the current round
            for (int r = 0; r < rounds; ++r) {
                if (UNIT_OF(r, s) >= total) break;
                const int A = (UNIT_OF(r, 1) < total) ? 2 : 1;
                const int An = (UNIT_OF(r + 1, 0) < total) ? ((UNIT_OF(r + 1, 1) < total) ? 2 : 1) : 0;
                const uint32_t tail = base + 2 * A * (K - 1);  // first load of tile K - 1
                auto gk = [&](int t) -> uint32_t { return t == 0 ? gk0 : base + 2 * A * (t - 1) + 2 * s + 1; };
                auto gv = [&](int t) -> uint32_t {
                    return t < K - 1 ? base + 2 * A * t + 2 * s : tail + s + (s < An ? s : An);
                };
                for (int t = 0; t < K; ++t) {
                    mbar_wait(S_FULL(s), sf_ph);
                    sf_ph ^= 1;
                    mbar_arrive(RING_EMPTY(gk(t) % G::NST));
                    if (t > 0) mbar_arrive(RING_EMPTY(gv(t - 1) % G::NST));
                }
                mbar_wait(O_FULL(s), of_ph);
                of_ph ^= 1;
                mbar_arrive(RING_EMPTY(gv(K - 1) % G::NST));
                gk0 = gv(K - 1) + 1;
                base = tail + A + An;
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ============================ MMA issuer ============================
        // One thread issues, slot by slot, groups [PV(s,t) ; QK(s,t+1)] back to back (the
        // QK reuses the S/P columns, so it must follow the PV: same thread => in order).
        // Before a group, the three barriers it needs (P(s,t), the V stage, the next K
        // stage) are probed in ONE asm block so their latencies overlap; only a barrier
        // that is not yet complete is then waited on.  Ring stages are released by the
        // softmax warps; the MMA thread only commits S_FULL (+ Q_EMPTY / O_FULL).
        // The whole warp runs the loop (warp-uniform values, one lane issues via elect.sync:
        // see sm100.cuh mma_ss_w); descriptors are advanced by constant offsets.
        {
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, B, 0, 0);  // Q, K both K-major
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D, 0, 1);  // P K-major (TMEM), V MN-major
            uint32_t stage = 0, ph = 0;
            uint32_t qf_bits = 0, pf_bits = 0;  // per-slot phase bits of Q_FULL / P_FULL
            int nqk = 0, npv = 0;
            (void)nqk; (void)npv;
            auto next_stage = [&](uint32_t &st, uint32_t &sp) {
                st = stage;
                sp = ph;
                if (++stage == G::NST) { stage = 0; ph ^= 1; }
            };
            auto issue_qk = [&](int s, int t, uint32_t st) {
                const uint64_t ad0 = sdesc_sw128(sQ + s * G::Q_BYTES, 16, 1024);
                const uint64_t bd0 = sdesc_sw128(sRing + st * G::TILE_BYTES, 16, 1024);
                const uint32_t tS = tbase + s * 256;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint64_t ao = (uint64_t)(((kk >> 2) * G::QCHUNK + (kk & 3) * 32) >> 4);
                    const uint64_t bo = (uint64_t)(((kk >> 2) * G::KCHUNK + (kk & 3) * 32) >> 4);
                    mma_ss_w(tS, ad0 + ao, bd0 + bo, idesc_qk, kk > 0 ? 1u : 0u);
                }
                tc_commit_w(S_FULL(s));
                if (t == K - 1) tc_commit_w(Q_EMPTY(s));
            };
            auto issue_pv = [&](int s, int t, uint32_t st, int hf) {
                // V tile as the MN-major B operand: 16 keys = 16 rows of 128 B; the second
                // 64-wide chunk of d sits one KCHUNK further (LBO).  Half hf = keys
                // [64 hf, 64 hf + 64), i.e. the P columns of hand-off hf.
                const uint64_t vd0 = sdesc_sw128(sRing + st * G::TILE_BYTES, G::KCHUNK, 1024);
                const uint32_t tP = tbase + s * 256, tO = tbase + s * 256 + 128;
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {
                    const int kk = hf * 4 + k4;
                    mma_ts_w(tO, tP + kk * 8, vd0 + (uint64_t)((kk * 2048) >> 4), idesc_pv, (t > 0 || kk > 0) ? 1u : 0u);
                }
                if (t == K - 1 && hf == G::NPH - 1) tc_commit_w(O_FULL(s));
            };
            // round 0's first QKs; every later unit's first QK follows its slot's last PV
            for (int s = 0; s < NSLOT; ++s) {
                if (UNIT_OF(0, s) >= total) continue;
                uint32_t st, sp;
                next_stage(st, sp);
                mbar_wait(Q_FULL(s), (qf_bits >> s) & 1u);
                qf_bits ^= 1u << s;
                mbar_wait(RING_FULL(st), sp);
                TR(0, nqk, 0);
                tc_fence_after();
                issue_qk(s, 0, st);
                TR(0, nqk, 2);
                ++nqk;
            }
            for (int r = 0; r < rounds; ++r) {
                for (int t = 0; t < K; ++t) {
                    for (int s = 0; s < NSLOT; ++s) {
                        if (UNIT_OF(r, s) >= total) continue;
                        const bool more = t + 1 < K, next = !more && UNIT_OF(r + 1, s) < total;
                        uint32_t sv, vp, sk = 0, kp = 0;
                        next_stage(sv, vp);
                        if (more || next) next_stage(sk, kp);
                        const uint32_t pp = (pf_bits >> s) & 1u;
                        pf_bits ^= 1u << s;
                        TR(0, npv, 3);
                        // non-blocking probe of the group's barriers (test_wait: an incomplete
                        // P_FULL must not put the thread to sleep), then wait for the rest
                        const uint32_t ok = mbar_try_wait4(P_FULL(s, 0), pp, RING_FULL(sv), vp,
                                                           RING_FULL((more || next) ? sk : sv), (more || next) ? kp : vp,
                                                           RING_FULL(sv), vp);
                        if (!(ok & 1u)) mbar_wait(P_FULL(s, 0), pp);
                        if (!(ok & 2u)) mbar_wait(RING_FULL(sv), vp);
                        if ((more || next) && !(ok & 4u)) mbar_wait(RING_FULL(sk), kp);
                        TR(0, npv, 4);
                        tc_fence_after();
                        // P arrives in two halves: the first half's PV runs while the softmax
                        // still exponentiates the second (shortens the S -> P -> S chain per slot)
                        issue_pv(s, t, sv, 0);
                        if (G::NPH == 2) {
                            mbar_wait(P_FULL(s, 1), pp);
                            TR(0, npv, 6);
                            tc_fence_after();
                            issue_pv(s, t, sv, 1);
                        }
                        if (more) {
                            issue_qk(s, t + 1, sk);
                        } else if (next) {  // the slot's next unit: its S is ready by the end of the epilogue
                            mbar_wait(Q_FULL(s), (qf_bits >> s) & 1u);
                            qf_bits ^= 1u << s;
                            tc_fence_after();
                            issue_qk(s, 0, sk);
                            ++nqk;
                        }
                        TR(0, npv, 5);
                        ++npv;
                    }
                }
            }
        }
        __syncwarp();
    }
    } else {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_SOFTMAX));
#endif
        if (lane == 0) DBG("w%d softmax start\n", warp);
        // ============================ softmax warpgroups ============================
        const int slot = (warp - 4) >> 2;
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const uint32_t tS = tbase + lane_off + slot * 256;
        const uint32_t tO = tS + 128;
        const float sl2 = p.scale_log2;
        uint32_t sf_ph = 0, of_ph = 0;
        for (int r = 0; r < rounds; ++r) {
            const int u = UNIT_OF(r, slot);
            if (u >= total) break;
            const int h = u / NT;
            const int32_t *il = p.idx + (size_t)u * K;
            const uint32_t *mbase = p.slot_mask + (size_t)h * NT * G::MW;
            float m = -INFINITY, l = 0.f;
            int jn = clamp_tile(__ldg(il), NT);
            for (int t = 0; t < K; ++t) {
                uint32_t mk[G::MW];
#pragma unroll
                for (int w = 0; w < G::MW; ++w) mk[w] = __ldg(mbase + (size_t)jn * G::MW + w);
                if (t + 1 < K) jn = clamp_tile(__ldg(il + t + 1), NT);

                const int trs = r * K + t, trr = 1 + slot * 4 + quarter;  // trace role per softmax warp
                if (lane == 0) TR(trr, trs, 0);
                mbar_wait(S_FULL(slot), sf_ph);
                if (lane == 0) TR(trr, trs, 1);
                sf_ph ^= 1;
                if (lane == 0) DBG("w%d slot%d t%d S ok\n", warp, slot, t);
                tc_fence_after();
                uint32_t sr[B / 32][32];
#pragma unroll
                for (int c = 0; c < B / 32; ++c) tmem_ld32(tS + c * 32, sr[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < B / 32; ++c) reg_fence(sr[c]);
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
                // row max with 8 independent partial maxima (no 128-long dependency chain)
                float pm[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) pm[q] = -INFINITY;
#pragma unroll
                for (int c = 0; c < B / 32; ++c)
#pragma unroll
                    for (int i = 0; i < 32; i += 2)  // three-input maxima (FMNMX3): half the instructions
                        pm[(i >> 1) & 7] = fmax3f(pm[(i >> 1) & 7], u2f(sr[c][i]), u2f(sr[c][i + 1]));
                const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                                       fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
                const float mnew = fmaxf(m, mx * sl2);
                if (lane == 0 && mnew != 1.2345f) TR(trr, trs, 3);
                // lazy rescale: only when some row of this warp grew its max by > 8 (log2 units)
                float f = 1.f;
                bool rescale = false;
                if (t == 0) {
                    m = mnew;
                } else if (__any_sync(0xFFFFFFFFu, mnew > m + 8.0f)) {
                    f = (mnew == -INFINITY) ? 1.f : ex2(m - mnew);
                    rescale = true;
                    l *= f;
                    m = mnew;
                }
                const float mu = (m == -INFINITY) ? 0.f : m;
                float ps[4] = {0.f, 0.f, 0.f, 0.f};
                // P is handed to the MMA thread in halves of 64 keys (P_FULL(slot, half)):
                // P V of the first half runs while the second half is exponentiated
#pragma unroll
                for (int c2 = 0; c2 < B / 64; ++c2) {
                    uint32_t pk[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int c = 2 * c2 + (i >> 4), e = (i & 15) * 2;
                        float x0, x1;
                        ffma2_bc(x0, x1, u2f(sr[c][e]), u2f(sr[c][e + 1]), sl2, -mu);
                        const float a = ex2(x0), b = ex2(x1);  // MUFU (FMA-pipe emulation measured slower)
                        fadd2_acc(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, b);
                        pk[i] = pack_bf16(a, b);
                    }
                    tmem_st32(tS + c2 * 32, pk);  // P (bf16 pairs) over S columns already read
                    if (c2 == 0 && rescale) {  // O is quiescent (see header); scale it before PV_t accumulates
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
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(P_FULL(slot, c2));
                    if (lane == 0) TR(trr, trs, 4 + c2);
                }
                l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
                if (lane == 0 && rescale) TR(trr, trs, 6);
                if (lane == 0) DBG("w%d slot%d t%d P arrive l=%f m=%f\n", warp, slot, t, l, m);
            }
            // ---- epilogue: O / l -> bf16, padded query rows -> 0.  The row's destination and
            // validity do not depend on O: computed (global load included) before the wait
            bool qvalid = false;
            if (row < B) qvalid = (__ldg(p.slot_mask + (size_t)u * G::MW + (row >> 5)) >> (row & 31)) & 1u;
            uint16_t *orow = p.out + ((size_t)u * B + (row < B ? row : 0)) * D;
            bool store = row < B;
            if (TOK) {  // row -> its token (reading R3); padded query slots have none
                const TileOrigin o = tile_origin(tp, h, u - h * NT);
                const int lpw = __ffs(tp.pw[o.c]) - 1, lphw = lpw + __ffs(tp.ph[o.c]) - 1;
                const int t = o.t0 + (row >> lphw), hq = o.h0 + ((row >> lpw) & (tp.ph[o.c] - 1)),
                          w = o.w0 + (row & (tp.pw[o.c] - 1));
                store = store && qvalid;
                orow = p.out + (size_t)h * tp.o_hs + (((size_t)t * tp.H + hq) * tp.W + w) * tp.o_ts;
            }
            const float inv = (qvalid && l > 0.f) ? 1.f / l : 0.f;
            mbar_wait(O_FULL(slot), of_ph);
            of_ph ^= 1;
            tc_fence_after();
            {
                uint32_t o[D / 32][32];  // all of the row's O in flight at once, one wait
#pragma unroll
                for (int c = 0; c < D / 32; ++c) tmem_ld32(tO + c * 32, o[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < D / 32; ++c) reg_fence(o[c]);
                if (store) {
#pragma unroll
                    for (int c = 0; c < D / 32; ++c) {
                        uint32_t pk[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i) pk[i] = pack_bf16(u2f(o[c][2 * i]) * inv, u2f(o[c][2 * i + 1]) * inv);
                        st_global_v8(orow + c * 32, pk, 0);   // 32-byte stores: whole sectors
                        st_global_v8(orow + c * 32 + 16, pk, 8);
                    }
                }
            }
            if (p.lse != nullptr && row < B)
                p.lse[(size_t)u * B + row] = (qvalid && l > 0.f) ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
        }
    }
#undef UNIT_OF
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, TMEM_COLS);
    }
}

static unsigned long long *g_attn_trace = nullptr;

template <int B, int D, bool TOK>
static veda_status launch_kernel(const CUtensorMap &mq, const CUtensorMap &mk, const CUtensorMap &mv, const Params &p,
                                 const TokParams &tp, int units, cudaStream_t stream)
{
    using G = Geo<B, D>;
    // set per launch: the attribute belongs to the current device's context
    cudaError_t e = cudaFuncSetAttribute(sparse_attn_fwd_kernel<B, D, TOK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    if (e != cudaSuccess) return fail(VEDA_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    int grid = (units + NSLOT - 1) / NSLOT;
    const int nsm = num_sms();
    if (grid > nsm) grid = nsm;
    sparse_attn_fwd_kernel<B, D, TOK><<<grid, NTHREADS, G::SMEM, stream>>>(mq, mk, mv, p, tp);
    count_launch();
    return check_launch("sparse_attn_fwd");
}

static Params make_params(const int32_t *idx, const uint32_t *mask, uint16_t *o, float *lse, int Hh, int NT, int kk,
                          float scale)
{
    Params p;
    p.idx = idx;
    p.slot_mask = mask;
    p.out = o;
    p.lse = lse;
    p.NT = NT;
    p.k = kk;
    p.total_units = Hh * NT;
    p.unit0 = 0;
    p.scale_log2 = scale * 1.4426950408889634f;
    p.trace = g_attn_trace;
    return p;
}

template <int B, int D>
static veda_status launch(const uint16_t *q, const uint16_t *k, const uint16_t *v, const int32_t *idx,
                          const uint32_t *mask, int Hh, int NT, int kk, float scale, uint16_t *o,
                          float *lse, cudaStream_t stream)
{
    CUtensorMap mq, mk, mv;
    const uint64_t rows = (uint64_t)Hh * NT * B;
    veda_status st;
    if ((st = make_tmap_bf16(&mq, q, rows, D, B)) != VEDA_OK) return st;
    if ((st = make_tmap_bf16(&mk, k, rows, D, B)) != VEDA_OK) return st;
    if ((st = make_tmap_bf16(&mv, v, rows, D, B)) != VEDA_OK) return st;
    static TokParams tp_unused;  // zero-initialised; the tiled instantiation never reads it
    return launch_kernel<B, D, false>(mq, mk, mv, make_params(idx, mask, o, lse, Hh, NT, kk, scale), tp_unused,
                                      Hh * NT, stream);
}

// Token-layout launch: heads are split into consecutive groups with at most MAXC distinct
// tile shapes; each group is one launch on pointers offset to its first head.
template <int B, int D>
static veda_status launch_tok(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t hs, int64_t ts,
                              const HeadCfgs &cf, int Hh, int Hp, int Wp, int T, int H, int W, int NT,
                              const int32_t *idx, const uint32_t *mask, int kk, float scale, uint16_t *o,
                              int64_t o_hs, int64_t o_ts, float *lse, int u_begin, int u_end, cudaStream_t stream)
{
    TokParams tp{};  // host staging (3-4 KB, per call: thread-safe), passed by value to the kernel
    CUtensorMap dummy;
    memset(&dummy, 0, sizeof dummy);
    const int MW = B / 32;
    for (int h0 = 0; h0 < Hh;) {
        int nc = 0, h1 = h0;
        for (; h1 < Hh; ++h1) {
            int c = 0;
            while (c < nc && !(tp.pt[c] == cf.pt[h1] && tp.ph[c] == cf.ph[h1] && tp.pw[c] == cf.pw[h1])) ++c;
            if (c == nc) {
                if (nc == MAXC) break;
                tp.pt[c] = cf.pt[h1]; tp.ph[c] = cf.ph[h1]; tp.pw[c] = cf.pw[h1];
                ++nc;
            }
            tp.cid[h1 - h0] = (uint8_t)c;
        }
        const int hn = h1 - h0;
        // units of this head group that fall in [u_begin, u_end) (flattened head x query tile)
        const int g_lo = std::max(u_begin, h0 * NT), g_hi = std::min(u_end, h1 * NT);
        if (g_lo >= g_hi) {
            h0 = h1;
            continue;
        }
        veda_status st;
        int tm = 0;
        for (int c = 0; c < nc; ++c) {
            if ((st = make_tmap_tile_tokens(&tp.q[c], q + (size_t)h0 * hs, hs, ts, hn, T, H, W, D, tp.pt[c], tp.ph[c],
                                            tp.pw[c], &tm)) != VEDA_OK ||
                (st = make_tmap_tile_tokens(&tp.k[c], k + (size_t)h0 * hs, hs, ts, hn, T, H, W, D, tp.pt[c], tp.ph[c],
                                            tp.pw[c], &tm)) != VEDA_OK ||
                (st = make_tmap_tile_tokens(&tp.v[c], v + (size_t)h0 * hs, hs, ts, hn, T, H, W, D, tp.pt[c], tp.ph[c],
                                            tp.pw[c], &tm)) != VEDA_OK)
                return st;
        }
        for (int c = 0; c < nc; ++c) {
            tp.nbw[c] = (uint32_t)(Wp / tp.pw[c]);
            tp.nbhw[c] = (uint32_t)((Hp / tp.ph[c]) * (Wp / tp.pw[c]));
            auto magic = [](uint32_t n) {  // ceil(2^32 / n), saturated for n = 1 (div_magic corrects by one)
                const unsigned long long m = (0x100000000ull + n - 1) / n;
                return (uint32_t)(m > 0xFFFFFFFFull ? 0xFFFFFFFFull : m);
            };
            tp.mbw[c] = magic(tp.nbw[c]);
            tp.mbhw[c] = magic(tp.nbhw[c]);
        }
        tp.T = T; tp.H = H; tp.W = W; tp.Hp = Hp; tp.Wp = Wp;
        tp.tok_major = tm;
        tp.o_hs = o_hs;
        tp.o_ts = o_ts;
        Params p = make_params(idx + (size_t)h0 * NT * kk, mask + (size_t)h0 * NT * MW, o + (size_t)h0 * o_hs,
                               lse ? lse + (size_t)h0 * NT * B : nullptr, hn, NT, kk, scale);
        p.unit0 = g_lo - h0 * NT;
        p.total_units = g_hi - g_lo;
        if ((st = launch_kernel<B, D, true>(dummy, dummy, dummy, p, tp, p.total_units, stream)) != VEDA_OK) return st;
        h0 = h1;
    }
    return VEDA_OK;
}

}  // namespace attn

#ifdef VEDA_ATTN_TRACE
extern "C" __attribute__((visibility("default"))) void veda_dbg_set_attn_trace(void *dev_buf)
{
    attn::g_attn_trace = static_cast<unsigned long long *>(dev_buf);
}
#endif

veda_status launch_sparse_attn(const uint16_t *q, const uint16_t *k, const uint16_t *v,
                               const int32_t *idx, const uint32_t *mask, int Hh, int NT, int B, int d,
                               int kk, float scale, uint16_t *o, float *lse, cudaStream_t s)
{
    if (B == 128 && d == 128) return attn::launch<128, 128>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    if (B == 128 && d == 64) return attn::launch<128, 64>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    if (B == 64 && d == 128) return attn::launch<64, 128>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    if (B == 64 && d == 64) return attn::launch<64, 64>(q, k, v, idx, mask, Hh, NT, kk, scale, o, lse, s);
    return fail(VEDA_ERR_CONFIG, "sparse_attn_fwd: unsupported (B=%d, d=%d)", B, d);
}

veda_status launch_sparse_attn_tok(const uint16_t *q, const uint16_t *k, const uint16_t *v, int64_t hs, int64_t ts,
                                   const HeadCfgs &cf, int Hh, int Tp, int Hp, int Wp, int T, int H, int W, int B,
                                   int NT, int d, const int32_t *idx, const uint32_t *mask, int kk, float scale,
                                   uint16_t *o, int64_t o_hs, int64_t o_ts, float *lse, int u_begin, int u_end,
                                   cudaStream_t s)
{
    (void)Tp;
    // a stride that is never used (one token, or one head) may equal the other one; give it
    // a distinct value so the 5-D tensor maps get a well-ordered dimension set
    if (hs == ts) {
        if ((int64_t)T * H * W == 1)
            ts = hs * Hh;
        else if (Hh == 1)
            hs = ts * ((int64_t)T * H * W);
        else
            return fail(VEDA_ERR_ALIGN, "sparse_attn_fwd_tokens: head_stride == token_stride");
    }
#define VEDA_TOK_ARGS q, k, v, hs, ts, cf, Hh, Hp, Wp, T, H, W, NT, idx, mask, kk, scale, o, o_hs, o_ts, lse, u_begin, u_end, s
    if (B == 128 && d == 128) return attn::launch_tok<128, 128>(VEDA_TOK_ARGS);
    if (B == 128 && d == 64) return attn::launch_tok<128, 64>(VEDA_TOK_ARGS);
    if (B == 64 && d == 128) return attn::launch_tok<64, 128>(VEDA_TOK_ARGS);
    if (B == 64 && d == 64) return attn::launch_tok<64, 64>(VEDA_TOK_ARGS);
#undef VEDA_TOK_ARGS
    return fail(VEDA_ERR_CONFIG, "sparse_attn_fwd_tokens: unsupported (B=%d, d=%d)", B, d);
}

}  // namespace veda
