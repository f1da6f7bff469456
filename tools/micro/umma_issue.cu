// Micro-benchmark: what the single MMA-issuing thread of the attention kernel pays per kept
// tile besides the MMAs themselves.  One warp per SM issues groups of 16 tcgen05.mma
// (the kernel's [8 x PV (TS, N = 128) ; 8 x QK (SS, N = 128)], 1024 clk of tensor work at
// the nominal rate) and, per group, one of:
//   0  nothing                                   (baseline: 64 clk per MMA)
//   1  4 x tcgen05.commit to an mbarrier          (the kernel's per-tile commits)
//   2  1 mbarrier.test_wait of a completed phase  (one probe, result consumed at once)
//   3  3 test_waits in one asm block              (batched probes)
//   4  a clock64 spin of DELAY clk between groups (how much idle time the tcgen05 queue hides)
// It also records, for the first group after idle, the clock64 after each MMA issue returns
// (shows how many MMAs the issue queue accepts before the issuing thread blocks).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_issue umma_issue.cu && ./umma_issue
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_30325_b200/csrc/sm100.cuh"

using namespace veda::sm100;

constexpr int CHUNK = 128 * 128;

template <int MODE>
__global__ void __launch_bounds__(128, 1) umma_issue(long long *clk, long long *extra, long long *issue_t, int reps, int delay)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar, cbar[4], done_bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4 * CHUNK / 16; i += 128)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        for (int i = 0; i < 4; ++i) mbar_init(smem_u32(&cbar[i]), 1);
        mbar_init(smem_u32(&done_bar), 1);
        fence_barrier_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tslot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tslot;
    if (warp == 0) {
        // a completed phase to probe: arrive once on `bar` (phase 0 completes)
        if (lane == 0) mbar_arrive(smem_u32(&bar));
        __syncwarp();
        const uint32_t sQ = smem_u32(smem), sK = sQ + 2 * CHUNK;
        const uint64_t qd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sQ, 16, 1024), 0);
        const uint64_t kd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sK, 16, 1024), 0);
        const uint64_t vd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sK, CHUNK, 1024), 0);
        constexpr uint32_t id_qk = idesc_bf16_f32(128, 128, 0, 0), id_pv = idesc_bf16_f32(128, 128, 0, 1);
        const uint32_t tS = tbase, tO = tbase + 128, tP = tbase + 256;
        const uint32_t b = smem_u32(&bar);
        long long probe_clk = 0;
        uint32_t okacc = 0;
        // first group from idle: clock after each issue
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            mma_ts_w(tO, tP + kk * 8, vd + (uint64_t)((kk * 2048) >> 4), id_pv, 1u);
            if (lane == 0 && blockIdx.x == 0) issue_t[kk] = clock64();
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const uint64_t o = (uint64_t)(((kk >> 2) * CHUNK + (kk & 3) * 32) >> 4);
            mma_ss_w(tS, qd + o, kd + o, id_qk, kk > 0 ? 1u : 0u);
            if (lane == 0 && blockIdx.x == 0) issue_t[8 + kk] = clock64();
        }
        tc_commit_w(smem_u32(&done_bar));
        mbar_wait(smem_u32(&done_bar), 0);
        const long long t0 = clock64();
        if (lane == 0 && blockIdx.x == 0) issue_t[16] = t0;
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                mma_ts_w(tO, tP + kk * 8, vd + (uint64_t)((kk * 2048) >> 4), id_pv, 1u);
            if (MODE == 1) {
                tc_commit_w(smem_u32(&cbar[0]));
                tc_commit_w(smem_u32(&cbar[1]));
            }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint64_t o = (uint64_t)(((kk >> 2) * CHUNK + (kk & 3) * 32) >> 4);
                mma_ss_w(tS, qd + o, kd + o, id_qk, kk > 0 ? 1u : 0u);
            }
            if (MODE == 1) {
                tc_commit_w(smem_u32(&cbar[2]));
                tc_commit_w(smem_u32(&cbar[3]));
            }
            if (MODE == 2) {
                const long long a = clock64();
                okacc += mbar_test(b, 0) ? 1u : 0u;
                probe_clk += clock64() - a;
            }
            if (MODE == 3) {
                const long long a = clock64();
                uint32_t o0, o1, o2;
                mbar_try_wait3(b, 0, b, 0, b, 0, o0, o1, o2);  // (try_wait on complete phases)
                okacc += o0 + o1 + o2;
                probe_clk += clock64() - a;
            }
            if (MODE == 4) {
                const long long a = clock64();
                while (clock64() - a < delay) { }
            }
        }
        tc_commit_w(smem_u32(&done_bar));
        mbar_wait(smem_u32(&done_bar), 1);
        const long long t1 = clock64();
        if (lane == 0) {
            clk[blockIdx.x] = t1 - t0;
            extra[blockIdx.x] = probe_clk + (okacc == 0x7fffffff ? 1 : 0);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

template <int MODE>
static void run(int grid, int reps, int delay, long long *d, long long *e, long long *it, const char *name)
{
    const int smem = 4 * CHUNK + 1024;
    cudaFuncSetAttribute(umma_issue<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    umma_issue<MODE><<<grid, 128, smem>>>(d, e, it, reps, delay);
    umma_issue<MODE><<<grid, 128, smem>>>(d, e, it, reps, delay);
    cudaDeviceSynchronize();
    long long h[256], he[256], hi[17];
    cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaMemcpy(he, e, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    cudaMemcpy(hi, it, 17 * sizeof(long long), cudaMemcpyDeviceToHost);
    double m = 0, me = 0;
    for (int i = 0; i < grid; ++i) { m += h[i]; me += he[i]; }
    printf("%-44s delay %4d: %7.1f clk per group of 16 MMAs (nominal 1024)", name, delay, m / grid / reps);
    if (MODE == 2 || MODE == 3) printf(", probe %5.1f clk", me / grid / reps);
    printf("\n");
    if (MODE == 0 && delay == 0) {
        printf("   first group from idle, clk after each issue returns (rel. to first):");
        for (int i = 0; i < 16; ++i) printf(" %lld", hi[i] - hi[0]);
        printf("\n");
    }
}


// Latency of shared-memory accesses made by another warp while warp 0 streams MMAs:
// FORM 0 = QK SS (A and B from shared memory, 128 B/clk), 1 = PV TS (B only, 64 B/clk),
// 2 = QK TS (Q in TMEM, B from shared memory), 3 = no MMAs.  Warp 2 times a dependent chain
// of ld.shared (one load at a time) and of mbarrier.test_wait probes.
template <int FORM>
__global__ void __launch_bounds__(128, 1) smem_lat(long long *out, int reps)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar, done_bar;
    __shared__ volatile int stop;
    __shared__ uint32_t chain[64];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4 * CHUNK / 16; i += 128)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    if (threadIdx.x < 64) chain[threadIdx.x] = (threadIdx.x + 1) & 63;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        stop = 0;
        mbar_init(smem_u32(&bar), 1);
        mbar_init(smem_u32(&done_bar), 1);
        fence_barrier_init();
        mbar_arrive(smem_u32(&bar));
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tslot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tslot;
    if (warp == 0) {
        const uint32_t sQ = smem_u32(smem), sK = sQ + 2 * CHUNK;
        const uint64_t qd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sQ, 16, 1024), 0);
        const uint64_t kd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sK, 16, 1024), 0);
        const uint64_t vd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sK, CHUNK, 1024), 0);
        constexpr uint32_t id_qk = idesc_bf16_f32(128, 128, 0, 0), id_pv = idesc_bf16_f32(128, 128, 0, 1);
        if (FORM != 3)
            for (int r = 0; r < reps; ++r) {
                if (FORM == 0) mma_group_ss<8, CHUNK / 16, 2, CHUNK / 16, 2>(tbase, qd, kd, id_qk, 0u);
                if (FORM == 1) mma_group_ts<8, 8, 128>(tbase + 128, tbase + 256, vd, id_pv, 1u);
                if (FORM == 2) mma_group_ss<8, CHUNK / 16, 2, CHUNK / 16, 2>(tbase, qd, kd, id_qk, 0u);
            }
        tc_commit_w(smem_u32(&done_bar));
        mbar_wait(smem_u32(&done_bar), 0);
        if (lane == 0) stop = 1;
    } else if (warp == 2) {
        long long lds_clk = 0, tw_clk = 0, n = 0;
        uint32_t idx = lane & 63;
        const uint32_t b = smem_u32(&bar);
        uint32_t okacc = 0;
        while (!stop && n < 4000) {
            long long a = clock64();
#pragma unroll
            for (int i = 0; i < 8; ++i) idx = chain[idx];
            long long c = clock64();
            lds_clk += c - a;
#pragma unroll
            for (int i = 0; i < 8; ++i) okacc += mbar_test(b, 0) ? 1u : 0u;
            tw_clk += clock64() - c;
            ++n;
        }
        if (lane == 0 && blockIdx.x == 0) {
            out[0] = lds_clk;
            out[1] = tw_clk;
            out[2] = n * 8;
            out[3] = idx + okacc;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

template <int FORM>
static void run_lat(int grid, long long *d, const char *name)
{
    const int smem = 4 * CHUNK + 1024;
    cudaFuncSetAttribute(smem_lat<FORM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    smem_lat<FORM><<<grid, 128, smem>>>(d, 400);
    cudaDeviceSynchronize();
    long long h[4];
    cudaMemcpy(h, d, 4 * sizeof(long long), cudaMemcpyDeviceToHost);
    printf("%-44s ld.shared %6.1f clk, mbarrier.test_wait %6.1f clk (dependent, %lld samples)\n", name,
           (double)h[0] / h[2], (double)h[1] / h[2], h[2]);
}

// Does a warp that issues tcgen05.mma into a full queue slow the other warps of its SM
// sub-partition?  Warp 1 (SMSP 1) streams MMA groups (MODE 1) or idles (MODE 0); warps
// 4-7 (one per SMSP) each run the same FFMA2/MUFU loop and time it.
template <int MODE, int WORK = 0>
__global__ void __launch_bounds__(256, 1) smsp_share(long long *out, int reps)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long done_bar;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4 * CHUNK / 16; i += 256)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        stop = 0;
        mbar_init(smem_u32(&done_bar), 1);
        fence_barrier_init();
    }
    if (warp == 0) {
        tmem_alloc(smem_u32(&tslot), 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tslot;
    if (warp == 1) {
        const uint32_t sQ = smem_u32(smem), sK = sQ + 2 * CHUNK;
        const uint64_t qd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sQ, 16, 1024), 0);
        const uint64_t kd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sK, 16, 1024), 0);
        const uint64_t vd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sK, CHUNK, 1024), 0);
        constexpr uint32_t id_qk = idesc_bf16_f32(128, 128, 0, 0), id_pv = idesc_bf16_f32(128, 128, 0, 1);
        if (MODE == 1)
            while (stop < 4) {
                mma_group_ts<8, 8, 128>(tbase + 128, tbase + 256, vd, id_pv, 1u);
                mma_group_ss<8, CHUNK / 16, 2, CHUNK / 16, 2>(tbase, qd, kd, id_qk, 0u);
            }
        tc_commit_w(smem_u32(&done_bar));
        mbar_wait(smem_u32(&done_bar), 0);
    } else if (warp >= 4) {
        float a = lane * 0.001f, b = 1.0001f, c2 = 0.5f, d = 0.25f;
        const uint32_t tl = tbase + (uint32_t((warp & 3) * 32) << 16) + 384;  // columns the MMAs do not touch
        uint32_t v[32];
        __syncwarp();
        const long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            if (WORK == 0) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    a = fmaf(a, b, c2);
                    d = ex2(d * 0.5f);
                    c2 = fmaf(c2, b, d);
                }
            } else if (WORK == 1) {  // TMEM load round trips
                tmem_ld32(tl, v);
                tmem_wait_ld();
                a += __uint_as_float(v[lane & 31]);
            } else {  // TMEM stores
                v[0] = __float_as_uint(a);
                tmem_st16(tl, *reinterpret_cast<uint32_t(*)[16]>(v));
                tmem_wait_st();
                a += 1.0f;
            }
        }
        const long long t1 = clock64();
        if (lane == 0) {
            out[blockIdx.x * 4 + (warp - 4)] = t1 - t0 + (a == 12345.f ? 1 : 0);
            atomicAdd((int *)&stop, 1);  // the MMA stream runs until all four timing warps are done
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

template <int MODE, int WORK = 0>
static void run_share(int grid, long long *d, const char *name)
{
    const int smem = 4 * CHUNK + 1024;
    cudaFuncSetAttribute(smsp_share<MODE, WORK>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    smsp_share<MODE, WORK><<<grid, 256, smem>>>(d, 2000);
    cudaDeviceSynchronize();
    long long h[4 * 148];
    cudaMemcpy(h, d, 4 * grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double m[4] = {0, 0, 0, 0};
    for (int b = 0; b < grid; ++b)
        for (int w = 0; w < 4; ++w) m[w] += h[b * 4 + w];
    printf("%-40s clk of the timed loop per SMSP: %8.0f %8.0f %8.0f %8.0f\n", name, m[0] / grid, m[1] / grid, m[2] / grid,
           m[3] / grid);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *d, *e, *it;
    cudaMalloc(&d, 256 * sizeof(long long));
    cudaMalloc(&e, 256 * sizeof(long long));
    cudaMalloc(&it, 32 * sizeof(long long));
    const int reps = 1000;
    run<0>(sms, reps, 0, d, e, it, "baseline");
    run<1>(sms, reps, 0, d, e, it, "+ 4 commits per group");
    run<2>(sms, reps, 0, d, e, it, "+ 1 test_wait probe per group");
    run<3>(sms, reps, 0, d, e, it, "+ 3 try_wait probes (one asm) per group");
    for (int dl : {50, 100, 200, 300, 400, 600, 800, 1200})
        run<4>(sms, reps, dl, d, e, it, "+ spin delay per group");
    long long *dd;
    cudaMalloc(&dd, 4 * 148 * sizeof(long long));
    run_share<0>(sms, dd, "warp 1 idle");
    run_share<1>(sms, dd, "warp 1 streaming MMAs (SMSP 1)");
    run_share<0, 1>(sms, dd, "tcgen05.ld x32 loop, warp 1 idle");
    run_share<1, 1>(sms, dd, "tcgen05.ld x32 loop, warp 1 MMAs");
    run_share<0, 2>(sms, dd, "tcgen05.st x16 loop, warp 1 idle");
    run_share<1, 2>(sms, dd, "tcgen05.st x16 loop, warp 1 MMAs");
    run_lat<3>(sms, d, "latency, no MMAs");
    run_lat<0>(sms, d, "latency under QK SS MMAs (128 B/clk operands)");
    run_lat<1>(sms, d, "latency under PV TS MMAs (64 B/clk)");
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
