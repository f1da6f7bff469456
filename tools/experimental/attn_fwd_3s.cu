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

// Warp roles in warpgroup 0 (warp w runs on SM sub-partition w % 4, whose TMEM lane quarter
// is also softmax quarter w % 4): producer warp 0, MMA issuer, Q loader; the fourth is idle.
#ifndef VEDA_MMA_WARP
#define VEDA_MMA_WARP 1
#endif
constexpr int MMA_WARP = VEDA_MMA_WARP;
constexpr int QL_WARP = MMA_WARP == 2 ? 3 : 2;
#ifndef VEDA_MMA_SLEEP_NS
#define VEDA_MMA_SLEEP_NS 0
#endif
constexpr int MMA_SLEEP_NS = VEDA_MMA_SLEEP_NS;  // < 0: suspending try_wait
#ifndef VEDA_CTRL_TRYWAIT
#define VEDA_CTRL_TRYWAIT 0
#endif
constexpr bool CTRL_TRYWAIT = VEDA_CTRL_TRYWAIT;  // producer / Q loader wait with try_wait
// exp2 emulation also on the lane quarter that shares its sub-partition with the MMA issuer
#ifndef VEDA_EMU_MMA_QUARTER
#define VEDA_EMU_MMA_QUARTER 1
#endif
constexpr bool EMU_MMA_QUARTER = VEDA_EMU_MMA_QUARTER;

template <int B, int D>
struct Geo {
    static constexpr int QCHUNK = 128 * 128;         // one 64-col chunk of the 128-row Q buffer
    static constexpr int Q_BYTES = QCHUNK * (D / 64);
    static constexpr int KCHUNK = B * 128;           // one 64-col chunk of a B-row K/V tile
    static constexpr int TILE_BYTES = KCHUNK * (D / 64);
    static constexpr int NBAR = 2 * 8 + 2 + 2 * NSB + NOD + 1;
    // mailboxes (64-bit {value, sequence} words, one per row): reference maxima for the next
    // tile, chained (C) and unit-start (T) slots; final row sums of the set that does not run
    // the unit's epilogue (L)
    static constexpr int MBOX_WORDS = 4 * 32 * (1 + 2 + 4);
    static constexpr int MISC = NBAR * 8 + MBOX_WORDS * 8 + 16;
    static constexpr int NST_FIT = (VEDA_RING_BUDGET_KB * 1024 - Q_BYTES - MISC - 1024) / TILE_BYTES;
    static constexpr int NST = NST_FIT > 8 ? 8 : NST_FIT;
    static constexpr int MW = B / 32;
    static constexpr int SMEM = Q_BYTES + NST * TILE_BYTES + MISC + 1024;
    static constexpr uint32_t COL_O = NSB * B;  // S/P buffers at columns b*B, O after them
    static_assert(NST >= 3, "ring too shallow");
    static_assert(NSB * B + D <= 512, "TMEM budget");
};

// Ring position (TMA load order = MMA consumption order) of the K and V tiles of the CTA's
// g-th kept tile, for a CTA with G tiles: K(0), K(1), K(2), then V(g), K(g+3) for g = 0, 1, ...
__device__ __forceinline__ uint32_t ring_pos_k(int g) { return g < NSB ? (uint32_t)g : (uint32_t)(2 * g - NSB + 1); }
__device__ __forceinline__ uint32_t ring_pos_v(int g, int G)
{
    const int a = 2 * g + NSB, b = G + g;
    return (uint32_t)(a < b ? a : b);
}

// (unit, tile-within-unit) cursor over a CTA's flattened tile sequence g = n*k + t
struct Cursor {
    int n, t;
    __device__ __forceinline__ void step(int d, int K)
    {
        t += d;
        while (t >= K) { t -= K; ++n; }
    }
};

template <int B, int D, bool TOK>
__global__ void __launch_bounds__(NTHREADS, 1)
    sparse_attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV, const Params p,
                           const __grid_constant__ TokParams tp)
{
    using G_ = Geo<B, D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~uintptr_t(1023));
    const uint32_t sQ = smem_u32(smem);
    const uint32_t sRing = sQ + G_::Q_BYTES;
    const uint32_t sBar = sRing + G_::NST * G_::TILE_BYTES;
    unsigned long long *mbox =
        reinterpret_cast<unsigned long long *>(smem + G_::Q_BYTES + G_::NST * G_::TILE_BYTES + G_::NBAR * 8);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mbox + G_::MBOX_WORDS);
    // barriers
#define RING_FULL(i) (sBar + 8u * (i))
#define RING_EMPTY(i) (sBar + 8u * (8 + (i)))
#define Q_FULL (sBar + 8u * 16)
#define Q_EMPTY (sBar + 8u * 17)
#define S_FULL(b) (sBar + 8u * (18 + (b)))
#define P_FULL(b) (sBar + 8u * (18 + NSB + (b)))
#define O_DONE(i) (sBar + 8u * (18 + 2 * NSB + (i)))
#define O_FREE (sBar + 8u * (18 + 2 * NSB + NOD))
    // mailbox word of row 32q + lane: chained slot C, unit-start slots T[2], row-sum slots L[4]
#define MB_C(q) smem_u32(mbox + (q) * 32 + lane)
#define MB_T(q, i) smem_u32(mbox + 128 + ((q) * 2 + (i)) * 32 + lane)
#define MB_L(q, i) smem_u32(mbox + 384 + ((q) * 4 + (i)) * 32 + lane)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (B < 128) {  // rows B..127 of the M=128 Q operand are never loaded: keep them zero
        uint4 *q4 = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < G_::Q_BYTES / 16; i += NTHREADS) q4[i] = make_uint4(0, 0, 0, 0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    for (int i = threadIdx.x; i < G_::MBOX_WORDS; i += NTHREADS) mbox[i] = 0ull;
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < G_::NST; ++i) {
            mbar_init(RING_FULL(i), 1);
            mbar_init(RING_EMPTY(i), 1);
        }
        mbar_init(Q_FULL, 1);
        mbar_init(Q_EMPTY, 1);
        for (int b = 0; b < NSB; ++b) {
            mbar_init(S_FULL(b), 1);
            mbar_init(P_FULL(b), 4);  // one arrival per warp of the softmax set
        }
        for (int i = 0; i < NOD; ++i) mbar_init(O_DONE(i), 1);
        mbar_init(O_FREE, 4);
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

    const int NT = p.NT, K = p.k;
    const int grid = gridDim.x;
    // this CTA's units: u_n = unit0 + n*grid + blockIdx.x (consecutive CTAs take consecutive
    // query tiles of one head: the ~148 tiles in flight share their heads' hub K/V tiles in L2)
    const int NU = (p.total_units - (int)blockIdx.x + grid - 1) / grid;
    const int G = NU * K;
#define UNIT_OF(n) (p.unit0 + (n) * grid + (int)blockIdx.x)

    if (warp < 4) {
#ifndef VEDA_NO_SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(REGS_CTRL));
#endif
    if (warp == 0) {
        // ============================ TMA producer (K/V ring) ============================
        if (lane == 0) {
            uint32_t pos = 0;
            // K / V streams: cursors over (unit, tile), head and index list of the current unit
            Cursor ck{0, 0}, cv{0, 0};
            int hk = UNIT_OF(0) / NT, hv = hk;
            const int32_t *ilk = p.idx + (size_t)UNIT_OF(0) * K, *ilv = ilk;
            auto load_item = [&](bool isK) {
                const uint32_t st = pos % G_::NST, ph = (pos / G_::NST) & 1u;
                const int h = isK ? hk : hv;
                const int j = __ldg(isK ? ilk + ck.t : ilv + cv.t);
                if (CTRL_TRYWAIT)
                    mbar_wait(RING_EMPTY(st), ph ^ 1u);
                else
                    mbar_wait_sleep(RING_EMPTY(st), ph ^ 1u, 32);
                mbar_expect_tx(RING_FULL(st), G_::TILE_BYTES);
                if (TOK)
                    tma_tile_tok<D / 64>(sRing + st * G_::TILE_BYTES, G_::KCHUNK, isK ? tp.k : tp.v, tp, h, j,
                                         RING_FULL(st));
                else
#pragma unroll
                    for (int c = 0; c < D / 64; ++c)
                        tma_load_2d(sRing + st * G_::TILE_BYTES + c * G_::KCHUNK, isK ? &tmK : &tmV, c * 64,
                                    (h * NT + j) * B, RING_FULL(st));
                ++pos;
                Cursor &cc = isK ? ck : cv;
                const int n0 = cc.n;
                cc.step(1, K);
                if (cc.n != n0 && cc.n < NU) {
                    const int u = UNIT_OF(cc.n);
                    (isK ? hk : hv) = u / NT;
                    (isK ? ilk : ilv) = p.idx + (size_t)u * K;
                }
            };
            const int pro = G < NSB ? G : NSB;
            for (int g = 0; g < pro; ++g) load_item(true);
            for (int g = 0; g < G; ++g) {
                load_item(false);
                if (g + NSB < G) load_item(true);
            }
        }
        __syncwarp();
    } else if (warp == QL_WARP) {
        // ============================ Q loader ============================
        // Q of unit n+1 goes into the (single) Q buffer as soon as unit n's last QK has
        // completed (Q_EMPTY); it was prefetched into L2 when Q of unit n was loaded.
        if (lane == 0) {
            for (int n = 0; n < NU; ++n) {
                if (n > 0) {
                    if (CTRL_TRYWAIT)
                        mbar_wait(Q_EMPTY, (uint32_t)(n - 1) & 1u);
                    else
                        mbar_wait_sleep(Q_EMPTY, (uint32_t)(n - 1) & 1u, 64);
                }
                const int u = UNIT_OF(n), h = u / NT, i = u - h * NT;
                mbar_expect_tx(Q_FULL, B * D * 2);
                if (TOK)
                    tma_tile_tok<D / 64>(sQ, G_::QCHUNK, tp.q, tp, h, i, Q_FULL);
                else
#pragma unroll
                    for (int c = 0; c < D / 64; ++c) tma_load_2d(sQ + c * G_::QCHUNK, &tmQ, c * 64, u * B, Q_FULL);
                if (n + 1 < NU) {
                    const int u2 = UNIT_OF(n + 1), h2 = u2 / NT;
                    if (TOK) {
                        const TileOrigin o = tile_origin(tp, h2, u2 - h2 * NT);
#pragma unroll
                        for (int c = 0; c < D / 64; ++c) {
                            if (tp.tok_major)
                                tma_prefetch_5d(&tp.q[o.c], c * 64, h2, o.w0, o.h0, o.t0);
                            else
                                tma_prefetch_5d(&tp.q[o.c], c * 64, o.w0, o.h0, o.t0, h2);
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < D / 64; ++c) tma_prefetch_2d(&tmQ, c * 64, u2 * B);
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == MMA_WARP) {
        // ============================ MMA issuer ============================
        // Flat over the CTA's tiles g: QK(0..2), then [PV(g) ; QK(g+3)] for g = 0, 1, ...
        // QK(g+3) writes S buffer g%3, whose P(g) the PV(g) just issued reads: same thread,
        // so the tensor pipe executes them in order.  Before each group the three barriers it
        // needs (P(g), the V(g) stage, the K(g+3) stage) are probed in one asm block and only
        // an incomplete one is waited on: the tcgen05 queue holds only ~250 clk of work, so
        // every clock the issuing thread spends outside issue can idle the tensor core.
        // Commits: ring stage + O_DONE after a PV, ring stage + S_FULL after a QK, Q_EMPTY
        // after a unit's last QK.  The whole warp runs the loop (elect.sync inside the asm).
        constexpr uint32_t idesc_qk = idesc_bf16_f32(128, B, 0, 0);  // Q, K both K-major
        constexpr uint32_t idesc_pv = idesc_bf16_f32(128, D, 0, 1);  // P K-major (TMEM), V MN-major
        const uint64_t qdesc = sdesc_sw128(sQ, 16, 1024);
        Cursor cq{0, 0}, cp{0, 0};
        auto issue_qk = [&](int g, bool k_ready) {
            const int b = g % NSB;
            if (cq.t == 0) mbar_wait_spin(Q_FULL, (uint32_t)cq.n & 1u);
            const uint32_t pk = ring_pos_k(g), st = pk % G_::NST;
            if (!k_ready) mbar_wait_spin(RING_FULL(st), (pk / G_::NST) & 1u);
            TR(0, g, 3);
            tc_fence_after();
            mma_group_ss<D / 16, G_::QCHUNK / 16, 2, G_::KCHUNK / 16, 2>(
                tbase + (uint32_t)(b * B), qdesc, sdesc_sw128(sRing + st * G_::TILE_BYTES, 16, 1024), idesc_qk, 0u);
            tc_commit_w(RING_EMPTY(st));
            tc_commit_w(S_FULL(b));
            if (cq.t == K - 1) tc_commit_w(Q_EMPTY);
            cq.step(1, K);
        };
        const int pro = G < NSB ? G : NSB;
        for (int g = 0; g < pro; ++g) issue_qk(g, false);
        for (int g = 0; g < G; ++g) {
            const int b = g % NSB;
            TR(0, g, 0);
            if (cp.t == 0 && cp.n > 0) mbar_wait_spin(O_FREE, (uint32_t)(cp.n - 1) & 1u);
            const uint32_t pv = ring_pos_v(g, G), sv = pv % G_::NST;
            const bool more = g + NSB < G;
            const uint32_t pk = more ? ring_pos_k(g + NSB) : pv;
            const uint32_t ok = mbar_test3(P_FULL(b), (uint32_t)(g / NSB) & 1u, RING_FULL(sv), (pv / G_::NST) & 1u,
                                           RING_FULL(pk % G_::NST), (pk / G_::NST) & 1u);
            if (!(ok & 1u)) {
                if (MMA_SLEEP_NS < 0)
                    mbar_wait(P_FULL(b), (uint32_t)(g / NSB) & 1u);
                else if (MMA_SLEEP_NS > 0)
                    mbar_wait_sleep(P_FULL(b), (uint32_t)(g / NSB) & 1u, MMA_SLEEP_NS);
                else
                    mbar_wait_spin(P_FULL(b), (uint32_t)(g / NSB) & 1u);
            }
            TR(0, g, 4);
            if (!(ok & 2u)) mbar_wait_spin(RING_FULL(sv), (pv / G_::NST) & 1u);
            TR(0, g, 1);
            tc_fence_after();
            // V tile as the MN-major B operand: 16 keys = 16 rows of 128 B (2048 B per step);
            // the second 64-wide chunk of d sits one KCHUNK further (LBO).
            mma_group_ts<B / 16, 8, 2048 / 16>(tbase + G_::COL_O, tbase + (uint32_t)(b * B),
                                               sdesc_sw128(sRing + sv * G_::TILE_BYTES, G_::KCHUNK, 1024), idesc_pv,
                                               cp.t > 0 ? 1u : 0u);
            tc_commit_w(RING_EMPTY(sv));
            tc_commit_w(O_DONE(g % NOD));
            cp.step(1, K);
            TR(0, g + NSB, 2);
            if (more) issue_qk(g + NSB, (ok & 4u) != 0);
        }
        __syncwarp();
    }
    // warp 3: no role
    } else {
#ifndef VEDA_NO_SETMAXNREG
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(REGS_SOFTMAX));
#endif
        // ============================ softmax sets ============================
        // Set s (warps 4-7 / 8-11) takes the CTA's tiles g with g % 2 == s; warp (s, q) owns
        // TMEM lanes 32q..32q+31, i.e. rows 32q+lane of the query tile, all B columns.
        const int set = (warp - 4) >> 2;
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int row = q * 32 + lane;
        const uint32_t lane_off = uint32_t(q * 32) << 16;
        const uint32_t tO = tbase + lane_off + G_::COL_O;
        const float sl2 = p.scale_log2;
        float m_run = -INFINITY, l = 0.f;  // this set's reference max (log2 units) and row sum
        Cursor c{0, set};
        c.step(0, K);
        // slot mask of a tile's key tile, loaded one tile ahead (two dependent global loads)
        auto key_mask = [&](const Cursor &cc, uint32_t (&mk)[G_::MW]) {
            if (cc.n >= NU) return;
            const int u = UNIT_OF(cc.n), hh = u / NT;
            const int jj = __ldg(p.idx + (size_t)u * K + cc.t);
            const uint32_t *mb = p.slot_mask + ((size_t)hh * NT + jj) * G_::MW;
#pragma unroll
            for (int w = 0; w < G_::MW; ++w) mk[w] = __ldg(mb + w);
        };
        int n_cur = -1, h = 0;
        uint32_t mk_next[G_::MW];
        key_mask(c, mk_next);
        for (int g = set; g < G; g += 2, c.step(2, K)) {
            const int t = c.t;
            if (c.n != n_cur) {
                n_cur = c.n;
                h = UNIT_OF(n_cur) / NT;
            }
            if (t < 2) { m_run = -INFINITY; l = 0.f; }  // this set's first tile of the unit
            uint32_t mk[G_::MW];
#pragma unroll
            for (int w = 0; w < G_::MW; ++w) mk[w] = mk_next[w];
            {
                Cursor cn = c;
                cn.step(2, K);
                key_mask(cn, mk_next);
            }

            const int b = g % NSB;
            const uint32_t tS = tbase + lane_off + (uint32_t)(b * B);
            const int trr = 1 + set * 4 + q;
            if (lane == 0) TR(trr, g >> 1, 0);
            // reference max of the previous tile (the other set's): published long before this
            // tile's S lands, so its shared-memory round trip is taken off the critical path
            float m_prev = -INFINITY;
            if (t > 0)
                m_prev = mbox_get(t == 1 ? MB_T(q, c.n & 1) : MB_C(q), t == 1 ? (uint32_t)c.n + 1u : (uint32_t)g);
            mbar_wait(S_FULL(b), (uint32_t)(g / NSB) & 1u);
            if (lane == 0) TR(trr, g >> 1, 1);
            tc_fence_after();
            uint32_t sr[B / 32][32];
#pragma unroll
            for (int cc = 0; cc < B / 32; ++cc) tmem_ld32(tS + cc * 32, sr[cc]);
            tmem_wait_ld();
#pragma unroll
            for (int cc = 0; cc < B / 32; ++cc) reg_fence(sr[cc]);

            bool full = true;
#pragma unroll
            for (int w = 0; w < G_::MW; ++w) full &= (mk[w] == 0xFFFFFFFFu);
            if (!full) {
#pragma unroll
                for (int cc = 0; cc < B / 32; ++cc)
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (!((mk[cc] >> i) & 1u)) sr[cc][i] = f2u(-INFINITY);
            }
            // row max: 8 independent chains of three-input maxima
            float pm[8];
#pragma unroll
            for (int k8 = 0; k8 < 8; ++k8) pm[k8] = -INFINITY;
#pragma unroll
            for (int cc = 0; cc < B / 32; ++cc)
#pragma unroll
                for (int i = 0; i < 32; i += 2)
                    pm[((cc * 32 + i) >> 1) & 7] = fmax3f(pm[((cc * 32 + i) >> 1) & 7], u2f(sr[cc][i]), u2f(sr[cc][i + 1]));
            const float mx = fmaxf(fmax3f(pm[0], pm[1], pm[2]), fmax3f(fmax3f(pm[3], pm[4], pm[5]), pm[6], pm[7]));
            const float xm = mx * sl2;
            if (lane == 0 && xm != 1.2345f) TR(trr, g >> 1, 2);
            // the reference max is raised lazily: only when a row of this warp exceeds it by more
            // than RESCALE_THR (log2 units)
            if (lane == 0 && m_prev != 1.2345f) TR(trr, g >> 1, 6);
            const bool need = __any_sync(0xFFFFFFFFu, xm > m_prev + (float)RESCALE_THR);
            if (lane == 0 && need != (xm == 1.2345f)) TR(trr, g >> 1, 7);
            const float m_new = need ? fmaxf(m_prev, xm) : m_prev;
            if (t + 1 < K) {  // publish for the next tile (the other set)
                if (t == 0)
                    mbox_put(MB_T(q, c.n & 1), m_new, (uint32_t)c.n + 1u);
                else
                    mbox_put(MB_C(q), m_new, (uint32_t)g + 1u);
            }
            if (lane == 0) TR(trr, g >> 1, 3);
            if (t > 0 && need) {
                // rows whose reference grew from a finite value hold a non-zero O: scale it
                // once PV(g-1) is complete (PV(g) waits for this set's P(g))
                const float f = (m_prev == -INFINITY || m_new == m_prev) ? 1.f : ex2(m_prev - m_new);
                if (__any_sync(0xFFFFFFFFu, f != 1.f)) {
                    mbar_wait(O_DONE((g - 1) % NOD), (uint32_t)((g - 1) / NOD) & 1u);
                    tc_fence_after();
#pragma unroll
                    for (int cc = 0; cc < D / 32; ++cc) {
                        uint32_t o[32];
                        tmem_ld32(tO + cc * 32, o);
                        tmem_wait_ld();
                        reg_fence(o);
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = f2u(u2f(o[i]) * f);
                        tmem_st32(tO + cc * 32, o);
                    }
                }
            }
            if (m_new != m_run) {
                l = (m_run == -INFINITY) ? 0.f : l * ex2(m_run - m_new);
                m_run = m_new;
            }
            const float mu = (m_new == -INFINITY) ? 0.f : m_new;
            float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int cc = 0; cc < B / 32; ++cc) {
                uint32_t pk[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    float x0, x1;
                    ffma2_bc(x0, x1, u2f(sr[cc][2 * i]), u2f(sr[cc][2 * i + 1]), sl2, -mu);
                    float a, bb;
                    if (EMU_EVERY > 0 && (i % EMU_EVERY) == EMU_EVERY - 1 && (EMU_MMA_QUARTER || q != MMA_WARP)) {
                        ex2_emu2(a, bb, x0, x1);  // FMA-pipe polynomial: unloads the MUFU unit
                    } else {
                        a = ex2(x0);
                        bb = ex2(x1);
                    }
                    fadd2_acc(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, bb);
                    pk[i] = pack_bf16(a, bb);
                }
                tmem_st16(tS + cc * 16, pk);  // P (bf16 pairs) over S columns already read
            }
            l += (ps[0] + ps[1]) + (ps[2] + ps[3]);
            if (lane == 0) TR(trr, g >> 1, 4);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(P_FULL(b));
            if (lane == 0) TR(trr, g >> 1, 5);
            if (t == K - 2)  // this set's last tile of the unit; the other set finishes it
                mbox_put(MB_L(q, c.n & 3), l, (uint32_t)c.n + 1u);
            if (t == K - 1) {
                // ---- epilogue: this set ran the unit's last tile
                float lt = l;
                if (K >= 2) {
                    const float lo = mbox_get(MB_L(q, c.n & 3), (uint32_t)c.n + 1u);
                    // the other set's sum is relative to m_prev (its last published reference)
                    if (m_prev != -INFINITY) lt += (m_prev == m_run) ? lo : lo * ex2(m_prev - m_run);
                }
                mbar_wait(O_DONE(g % NOD), (uint32_t)(g / NOD) & 1u);
                tc_fence_after();
                uint32_t o[D / 32][32];
#pragma unroll
                for (int cc = 0; cc < D / 32; ++cc) tmem_ld32(tO + cc * 32, o[cc]);
                tmem_wait_ld();
#pragma unroll
                for (int cc = 0; cc < D / 32; ++cc) reg_fence(o[cc]);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(O_FREE);
                const int u = UNIT_OF(c.n);
                bool qvalid = false;
                if (row < B) qvalid = (__ldg(p.slot_mask + (size_t)u * G_::MW + (row >> 5)) >> (row & 31)) & 1u;
                const float inv = (qvalid && lt > 0.f) ? 1.f / lt : 0.f;
                uint16_t *orow = p.out + ((size_t)u * B + (row < B ? row : 0)) * D;
                bool store = row < B;
                if (TOK) {  // row -> its token (reading R3); padded query slots have none
                    const TileOrigin o2 = tile_origin(tp, h, u - h * NT);
                    const int lpw = __ffs(tp.pw[o2.c]) - 1, lphw = lpw + __ffs(tp.ph[o2.c]) - 1;
                    const int tt = o2.t0 + (row >> lphw), hq = o2.h0 + ((row >> lpw) & (tp.ph[o2.c] - 1)),
                              w = o2.w0 + (row & (tp.pw[o2.c] - 1));
                    store = store && qvalid;
                    orow = p.out + (size_t)h * tp.o_hs + (((size_t)tt * tp.H + hq) * tp.W + w) * tp.o_ts;
                }
                if (store) {
#pragma unroll
                    for (int cc = 0; cc < D / 32; ++cc) {
                        uint32_t pk[16];
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            pk[i] = pack_bf16(u2f(o[cc][2 * i]) * inv, u2f(o[cc][2 * i + 1]) * inv);
                        uint4 *dst = reinterpret_cast<uint4 *>(orow + cc * 32);
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            dst[v] = make_uint4(pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
                    }
                }
                if (p.lse != nullptr && row < B)
                    p.lse[(size_t)u * B + row] =
                        (qvalid && lt > 0.f) ? (m_run + __log2f(lt)) * 0.69314718055994531f : -INFINITY;
            }
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
    const int nsm = num_sms();
    const int grid = units < nsm ? units : nsm;
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
