// sm100.cuh -- thin inline-PTX wrappers for the Blackwell (sm_100a) features the
// attention kernel uses: mbarrier, TMA (cp.async.bulk.tensor), tcgen05 MMA / TMEM.
// Bit layouts follow the PTX ISA descriptors (cross-checked against the CuTe
// headers vendored with flashinfer: cute/arch/mma_sm100_desc.hpp).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>

namespace veda { namespace sm100 {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
// Probe three mbarrier phases in one asm block: the three TRYWAITs are issued back to
// back, so their latencies overlap instead of adding up.
__device__ __forceinline__ void mbar_try_wait3(uint32_t b0, uint32_t p0, uint32_t b1, uint32_t p1, uint32_t b2,
                                               uint32_t p2, uint32_t &ok0, uint32_t &ok1, uint32_t &ok2)
{
    asm volatile(
        "{\n\t.reg .pred q0, q1, q2;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 q0, [%3], %4;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 q1, [%5], %6;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 q2, [%7], %8;\n\t"
        "selp.u32 %0, 1, 0, q0;\n\t"
        "selp.u32 %1, 1, 0, q1;\n\t"
        "selp.u32 %2, 1, 0, q2;\n\t}"
        : "=r"(ok0), "=r"(ok1), "=r"(ok2)
        : "r"(b0), "r"(p0), "r"(b1), "r"(p1), "r"(b2), "r"(p2)
        : "memory");
}
// Probe four mbarrier phases in one asm block without blocking (test_wait never suspends,
// unlike try_wait, which sleeps up to a HW time limit on an incomplete phase); latencies
// overlap.  Bit i of the result is set iff barrier i's phase is complete.
__device__ __forceinline__ uint32_t mbar_try_wait4(uint32_t b0, uint32_t p0, uint32_t b1, uint32_t p1, uint32_t b2,
                                                   uint32_t p2, uint32_t b3, uint32_t p3)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred q0, q1, q2, q3;\n\t.reg .b32 t0, t1, t2, t3;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 q0, [%1], %2;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 q1, [%3], %4;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 q2, [%5], %6;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 q3, [%7], %8;\n\t"
        "selp.u32 t0, 1, 0, q0;\n\t"
        "selp.u32 t1, 2, 0, q1;\n\t"
        "selp.u32 t2, 4, 0, q2;\n\t"
        "selp.u32 t3, 8, 0, q3;\n\t"
        "or.b32 t0, t0, t1;\n\t"
        "or.b32 t2, t2, t3;\n\t"
        "or.b32 %0, t0, t2;\n\t}"
        : "=r"(ok)
        : "r"(b0), "r"(p0), "r"(b1), "r"(p1), "r"(b2), "r"(p2), "r"(b3), "r"(p3)
        : "memory");
    return ok;
}
// Spin on an mbarrier phase.  A wait that never completes (a pipeline bug) traps
// after ~2^26 polls instead of hanging the GPU, reporting the barrier it was stuck on.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    uint32_t spins = 0;
    while (!mbar_try_wait(bar, parity)) {
        if (++spins == (1u << 26)) {
#ifdef VEDA_ATTN_DEBUG
            printf("veda: mbarrier wait timeout block %d thread %d bar 0x%x parity %u\n", blockIdx.x,
                   threadIdx.x, bar, parity);
#endif
            __trap();
        }
    }
}

// Non-suspending probe of one mbarrier phase (test_wait never sleeps, unlike try_wait).
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
// Spin on an mbarrier phase with test_wait (for latency-critical single-thread waiters);
// traps after ~2^27 polls (a pipeline bug) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait_spin(uint32_t bar, uint32_t parity)
{
    uint32_t spins = 0;
    while (!mbar_test(bar, parity)) {
        if (++spins == (1u << 27)) __trap();
    }
}
// Wait on an mbarrier phase with a sleep between probes: for waiters that are off the
// critical path (producer, loaders), so that their polling does not take issue slots from
// the softmax warps sharing their SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, uint32_t ns)
{
    uint32_t spins = 0;
    while (!mbar_test(bar, parity)) {
        __nanosleep(ns);
        if (++spins == (1u << 26)) __trap();
    }
}
// CTA-scope release store / acquire load of a shared-memory word (mailbox sequence numbers)
__device__ __forceinline__ void st_release_shared(uint32_t addr, uint32_t v)
{
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_shared(uint32_t addr)
{
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
// named barrier `id` (1..15) over `n` threads (a multiple of 32)
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// three-input max (FMNMX3 on sm_100)
__device__ __forceinline__ float fmax3f(float a, float b, float c)
{
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// ------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_prefetch_desc(const void *tmap)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// 2-D tiled load, completes `bytes` on mbarrier `bar`; coordinates are (inner, outer).
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void *tmap, int32_t c0, int32_t c1,
                                            uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
// 5-D tiled load (coordinates innermost first); out-of-bounds elements are zero-filled.
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const void *tmap, int32_t c0, int32_t c1, int32_t c2,
                                            int32_t c3, int32_t c4, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
        : "memory");
}
// 4-D tiled load (coordinates innermost first)
// plain (non-tensor) bulk copy global -> shared, completing on an mbarrier; bytes % 16 == 0
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void *tmap, int32_t c0, int32_t c1, int32_t c2,
                                            int32_t c3, uint32_t bar)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}
// L2 prefetch of a 5-D / 2-D tensor box (no shared-memory destination, no barrier)
__device__ __forceinline__ void tma_prefetch_5d(const void *tmap, int32_t c0, int32_t c1, int32_t c2, int32_t c3,
                                                int32_t c4)
{
    asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const void *tmap, int32_t c0, int32_t c1)
{
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(tmap)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const void *tmap, int32_t c0,
                                                 int32_t c1, uint32_t bar, uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ------------------------------------------------------------------ tcgen05 / TMEM
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst_smem),
                 "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tmem_relinquish()
{
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before()
{
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after()
{
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// all prior tcgen05 async ops of this thread arrive on `bar` when complete
__device__ __forceinline__ void tc_commit(uint32_t bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     bar)
                 : "memory");
}
// D[tmem] (+)= A[smem] . B[smem]
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Warp-uniform variants: executed by ALL 32 lanes of the issuing warp with warp-uniform
// operands; elect.sync picks one lane inside the asm.  Keeping the issue code convergent
// lets ptxas hold descriptors / TMEM addresses in uniform registers instead of wrapping
// every tcgen05 instruction in an ELECT + R2UR + branch loop (the divergent lane-0 form
// costs ~80 clk per MMA, more than a 128x128x16 MMA takes to execute).
__device__ __forceinline__ void mma_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void tc_commit_w(uint32_t bar)
{
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}

// NK (4 or 8) back-to-back kind::f16 MMAs -- the K-steps of one 64- or 128-deep
// contraction -- under ONE elect.sync.  Step kk uses A = a0 + kk*ASTEP, B = b0 + BOFF(kk)
// with BOFF(kk) = (kk / 4) * BCH + (kk % 4) * BIN (descriptor units of 16 bytes, or TMEM
// columns for a TMEM A operand).  Only step 0 takes `accumulate`; the rest accumulate.
// One election per group keeps the issuing thread's per-MMA cost to two adds.
// SS: A and B descriptors (shared memory); A steps like B with (ACH, AIN).
template <int NK, uint32_t ACH, uint32_t AIN, uint32_t BCH, uint32_t BIN>
__device__ __forceinline__ void mma_group_ss(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc,
                                             uint32_t accumulate)
{
    static_assert(NK == 4 || NK == 8, "NK");
#define VEDA_AO(k) ((k) / 4 * ACH + (k) % 4 * AIN)
#define VEDA_BO(k) ((k) / 4 * BCH + (k) % 4 * BIN)
    if constexpr (NK == 8) {
        asm volatile(
            "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a, b;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "setp.eq.b32 t, %4, %4;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
            "add.s64 a, %1, %5;\n\tadd.s64 b, %2, %6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
            "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
            "add.s64 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
            "add.s64 a, %1, %11;\n\tadd.s64 b, %2, %12;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
            "add.s64 a, %1, %13;\n\tadd.s64 b, %2, %14;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
            "add.s64 a, %1, %15;\n\tadd.s64 b, %2, %16;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
            "add.s64 a, %1, %17;\n\tadd.s64 b, %2, %18;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t}" ::"r"(d_tmem),
            "l"(a0), "l"(b0), "r"(idesc), "r"(accumulate), "n"(VEDA_AO(1)), "n"(VEDA_BO(1)), "n"(VEDA_AO(2)),
            "n"(VEDA_BO(2)), "n"(VEDA_AO(3)), "n"(VEDA_BO(3)), "n"(VEDA_AO(4)), "n"(VEDA_BO(4)), "n"(VEDA_AO(5)),
            "n"(VEDA_BO(5)), "n"(VEDA_AO(6)), "n"(VEDA_BO(6)), "n"(VEDA_AO(7)), "n"(VEDA_BO(7))
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a, b;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "setp.eq.b32 t, %4, %4;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
            "add.s64 a, %1, %5;\n\tadd.s64 b, %2, %6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
            "add.s64 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
            "add.s64 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t}" ::"r"(d_tmem),
            "l"(a0), "l"(b0), "r"(idesc), "r"(accumulate), "n"(VEDA_AO(1)), "n"(VEDA_BO(1)), "n"(VEDA_AO(2)),
            "n"(VEDA_BO(2)), "n"(VEDA_AO(3)), "n"(VEDA_BO(3))
            : "memory");
    }
#undef VEDA_AO
#undef VEDA_BO
}
// TS: A in TMEM (a0 = TMEM address, +ASTEP columns per step), B descriptor (shared memory).
template <int NK, uint32_t ASTEP, uint32_t BSTEP>
__device__ __forceinline__ void mma_group_ts(uint32_t d_tmem, uint32_t a0, uint64_t b0, uint32_t idesc,
                                             uint32_t accumulate)
{
    static_assert(NK == 4 || NK == 8, "NK");
    if constexpr (NK == 8) {
        asm volatile(
            "{\n\t.reg .pred e, p, t;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "setp.eq.b32 t, %4, %4;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
            "add.s32 a, %1, %5;\n\tadd.s64 b, %2, %6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t"
            "add.s32 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t"
            "add.s32 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t"
            "add.s32 a, %1, %11;\n\tadd.s64 b, %2, %12;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t"
            "add.s32 a, %1, %13;\n\tadd.s64 b, %2, %14;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t"
            "add.s32 a, %1, %15;\n\tadd.s64 b, %2, %16;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t"
            "add.s32 a, %1, %17;\n\tadd.s64 b, %2, %18;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t}" ::"r"(d_tmem),
            "r"(a0), "l"(b0), "r"(idesc), "r"(accumulate), "n"(ASTEP), "n"(BSTEP), "n"(2 * ASTEP), "n"(2 * BSTEP),
            "n"(3 * ASTEP), "n"(3 * BSTEP), "n"(4 * ASTEP), "n"(4 * BSTEP), "n"(5 * ASTEP), "n"(5 * BSTEP),
            "n"(6 * ASTEP), "n"(6 * BSTEP), "n"(7 * ASTEP), "n"(7 * BSTEP)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred e, p, t;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "setp.eq.b32 t, %4, %4;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
            "add.s32 a, %1, %5;\n\tadd.s64 b, %2, %6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t"
            "add.s32 a, %1, %7;\n\tadd.s64 b, %2, %8;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t"
            "add.s32 a, %1, %9;\n\tadd.s64 b, %2, %10;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, t;\n\t}" ::"r"(d_tmem),
            "r"(a0), "l"(b0), "r"(idesc), "r"(accumulate), "n"(ASTEP), "n"(BSTEP), "n"(2 * ASTEP), "n"(2 * BSTEP),
            "n"(3 * ASTEP), "n"(3 * BSTEP)
            : "memory");
    }
}
// Non-blocking probe of three mbarrier phases in one asm block (test_wait: latencies
// overlap, the thread never suspends); bit i set iff barrier i's phase is complete.
__device__ __forceinline__ uint32_t mbar_test3(uint32_t b0, uint32_t p0, uint32_t b1, uint32_t p1, uint32_t b2,
                                               uint32_t p2)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred q0, q1, q2;\n\t.reg .b32 t0, t1, t2;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 q0, [%1], %2;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 q1, [%3], %4;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 q2, [%5], %6;\n\t"
        "selp.u32 t0, 1, 0, q0;\n\t"
        "selp.u32 t1, 2, 0, q1;\n\t"
        "selp.u32 t2, 4, 0, q2;\n\t"
        "or.b32 t0, t0, t1;\n\t"
        "or.b32 %0, t0, t2;\n\t}"
        : "=r"(ok)
        : "r"(b0), "r"(p0), "r"(b1), "r"(p1), "r"(b2), "r"(p2)
        : "memory");
    return ok;
}
// 64-bit shared-memory mailbox word {value bits, sequence}: one naturally aligned 64-bit
// access is single-copy atomic, so a reader that sees the expected sequence also sees the
// value written with it -- no fence needed between writer and reader lanes.
__device__ __forceinline__ void mbox_put(uint32_t addr, float v, uint32_t seq)
{
    const unsigned long long w = ((unsigned long long)seq << 32) | __float_as_uint(v);
    asm volatile("st.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(addr), "l"(w) : "memory");
}
__device__ __forceinline__ float mbox_get(uint32_t addr, uint32_t seq)
{
    unsigned long long w;
    uint32_t spins = 0;
    do {
        asm volatile("ld.relaxed.cta.shared::cta.b64 %0, [%1];" : "=l"(w) : "r"(addr) : "memory");
        if (++spins == (1u << 27)) __trap();
    } while ((uint32_t)(w >> 32) != seq);
    return __uint_as_float((uint32_t)w);
}

// D[tmem] (+)= A[smem] . B[smem], kind::i8 (signed 8-bit A/B, s32 D, K = 32 per instruction);
// warp-uniform form as mma_ss_w
__device__ __forceinline__ void mma_i8_ss_w(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate)
{
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Instruction descriptor, kind::i8: s8 A/B (format 1), s32 D (format 2), both K-major.
__host__ __device__ constexpr uint32_t idesc_s8_s32(int M, int N)
{
    return (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
// Shared-memory matrix descriptor, SWIZZLE_64B K-major (64-byte rows, 8-row atoms of 512 B)
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr, uint32_t sbo)
{
    return (uint64_t((saddr >> 4) & 0x3FFF)) | (uint64_t(1) << 16) | (uint64_t((sbo >> 4) & 0x3FFF) << 32) |
           (uint64_t(1) << 46) | (uint64_t(4) << 61);
}
// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
// 16 lanes x 16 consecutive 32-bit columns (16x256b.x2) -> 8 registers per thread.  Thread t
// gets lane t/4 (r0, r1, r4, r5) and lane t/4 + 8 (r2, r3, r6, r7), columns 2(t%4) + {0, 1}
// (r0-r3) and 8 + 2(t%4) + {0, 1} (r4-r7): four threads hold 8 consecutive columns of a lane
// (layout measured on the B200: tools/micro/tmem_shape.cu)
__device__ __forceinline__ void tmem_ld16x256b_x2(uint32_t taddr, uint32_t (&r)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}

// Instruction descriptor, kind::f16: bf16 A/B, fp32 D.
//  [4,6) D fmt (1 = f32) | [7,10) A fmt (1 = bf16) | [10,13) B fmt (1 = bf16)
//  [15] A major (0 = K) | [16] B major (0 = K, 1 = MN) | [17,23) N>>3 | [24,29) M>>4
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N, int a_mn_major, int b_mn_major)
{
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(a_mn_major) << 15) |
           (uint32_t(b_mn_major) << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bits = 1.
//  [0,14) addr>>4 | [16,30) LBO>>4 | [32,46) SBO>>4 | [46,48) version=1 | [61,64) layout=2
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    return (uint64_t((saddr >> 4) & 0x3FFF)) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

#define VEDA_R32(a) \
    "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]), \
    "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]),        \
    "=r"(a[15]), "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]), "=r"(a[21]),      \
    "=r"(a[22]), "=r"(a[23]), "=r"(a[24]), "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]),      \
    "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
#define VEDA_W32(a) \
    "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]), "r"(a[8]), \
    "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]), "r"(a[15]), "r"(a[16]),   \
    "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]), "r"(a[23]), "r"(a[24]),  \
    "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]), "r"(a[31])

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
        "%30, %31}, [%32];"
        : VEDA_R32(r)
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, "
        "%29, %30, %31, %32};" ::"r"(taddr),
        VEDA_W32(r)
        : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// Registers written by tcgen05.ld are only valid after tcgen05.wait::ld; the empty
// volatile asm makes every later use depend on the wait (the compiler cannot hoist it).
template <int N>
__device__ __forceinline__ void reg_fence(uint32_t (&r)[N])
{
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}

__device__ __forceinline__ float ex2(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi)
{
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t *>(&v);
}

}}  // namespace veda::sm100
