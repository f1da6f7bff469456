// Micro-benchmark: tcgen05.mma (kind::f16, bf16 -> fp32, cta_group::1, M = 128) issue-to-
// completion rate for the operand forms the attention kernel uses, with the same SMEM
// descriptors (SWIZZLE_128B, 64-column chunks) and TMEM addresses:
//   QK-SS  : A = Q tile in SMEM (K-major), B = K tile in SMEM (K-major), N = 128 / 64
//   QK-TS  : A = Q in TMEM, B = K tile in SMEM                              (N = 128)
//   PV-TS  : A = P in TMEM, B = V tile in SMEM (MN-major)                    (N = 128)
//   group  : the production group [PV (8 x TS) ; QK (8 x SS)]
// One CTA per SM; one warp issues R x 8 MMAs (the 8 K-steps of d = 128 or of a 128-key
// tile), commits once, waits; clk per MMA = clock64 delta / MMAs.  The nominal rate is
// 128 * N / 256 clk per 128xNx16 MMA (64 clk at N = 128).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_rate umma_rate.cu && ./umma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_30325_b200/csrc/sm100.cuh"

using namespace veda::sm100;

constexpr int CHUNK_Q = 128 * 128;  // one 64-column chunk of a 128-row bf16 tile (bytes)

// INTF: what warps 4-7 do while warp 0 issues: 0 nothing, 1 tcgen05.ld 32 columns in a
// loop (the softmax's S loads), 2 tcgen05.ld + tcgen05.st (S load + P store), 3 st.shared
// 16 B per lane in a loop, 4 ld.shared 16 B per lane in a loop, 5 warp 1 streams 32 KB
// cp.async.bulk copies global -> shared (the TMA writes of the K/V ring) in a loop.
template <int MODE, int INTF>
__global__ void __launch_bounds__(256, 1) umma_rate(long long *clk, int reps, const uint8_t *gsrc, long long *nbytes)
{
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar, tbar;
    const int warp = threadIdx.x >> 5;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    for (int i = threadIdx.x; i < 3 * 2 * CHUNK_Q / 16; i += 256)
        reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&bar), 1);
        mbar_init(smem_u32(&tbar), 1);
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
        const uint32_t sQ = smem_u32(smem), sK = sQ + 2 * CHUNK_Q, sV = sK + 2 * CHUNK_Q;
        const uint64_t qd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sQ, 16, 1024), 0);
        const uint64_t kd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sK, 16, 1024), 0);
        const uint64_t vd = __shfl_sync(0xFFFFFFFFu, sdesc_sw128(sV, CHUNK_Q, 1024), 0);
        constexpr uint32_t id_qk = idesc_bf16_f32(128, 128, 0, 0), id_qk64 = idesc_bf16_f32(128, 64, 0, 0);
        constexpr uint32_t id_pv = idesc_bf16_f32(128, 128, 0, 1);
        const uint32_t tS = tbase, tO = tbase + 128, tA = tbase + 256;  // tA: Q or P operand in TMEM
        __syncwarp();
        const long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            if (MODE == 0 || MODE == 1 || MODE == 4) {
                if (MODE == 4) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        mma_ts_w(tO, tA + kk * 8, vd + (uint64_t)((kk * 2048) >> 4), id_pv, 1u);
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t o = (uint64_t)(((kk >> 2) * CHUNK_Q + (kk & 3) * 32) >> 4);
                    mma_ss_w(tS, qd + o, kd + o, MODE == 1 ? id_qk64 : id_qk, kk > 0 ? 1u : 0u);
                }
            } else if (MODE == 2) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t o = (uint64_t)(((kk >> 2) * CHUNK_Q + (kk & 3) * 32) >> 4);
                    mma_ts_w(tS, tA + kk * 8, kd + o, id_qk, kk > 0 ? 1u : 0u);
                }
            } else if (MODE == 3) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    mma_ts_w(tO, tA + kk * 8, vd + (uint64_t)((kk * 2048) >> 4), id_pv, 1u);
            } else if (MODE == 5) {  // half-tile group: [4 PV-TS (64 keys) ; 8 QK-SS N = 64]
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_ts_w(tO, tA + kk * 8, vd + (uint64_t)((kk * 2048) >> 4), id_pv, 1u);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t o = (uint64_t)(((kk >> 2) * CHUNK_Q + (kk & 3) * 32) >> 4);
                    mma_ss_w(tS, qd + o, kd + o, id_qk64, kk > 0 ? 1u : 0u);
                }
            }
        }
        tc_commit_w(smem_u32(&bar));
        mbar_wait(smem_u32(&bar), 0);
        const long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) {
            clk[blockIdx.x] = t1 - t0;
            done = 1;
        }
    } else if (warp == 1 && INTF == 5) {
        // bulk copies into the second half of the V area... (a region the MMAs do not read)
        const uint32_t dst = smem_u32(smem) + 6 * CHUNK_Q;
        long long n = 0;
        uint32_t ph = 0;
        int i = 0;
        while (!done) {
            if ((threadIdx.x & 31) == 0) {
                mbar_expect_tx(smem_u32(&tbar), 32768);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32768, [%2];"
                             ::"r"(dst), "l"(gsrc + (size_t)((blockIdx.x * 64 + i) % 8192) * 32768), "r"(smem_u32(&tbar))
                             : "memory");
            }
            __syncwarp();
            mbar_wait(smem_u32(&tbar), ph);
            ph ^= 1;
            n += 32768;
            ++i;
        }
        if ((threadIdx.x & 31) == 0) nbytes[blockIdx.x] = n;
    } else if (warp >= 4 && INTF > 0 && INTF < 5) {
        const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
        const uint32_t tR = tbase + lane_off + 384;  // columns 384-511: not touched by the MMAs
        uint32_t acc = 0, v[32];
        uint4 *sp = reinterpret_cast<uint4 *>(smem) + 5 * CHUNK_Q / 16 + (threadIdx.x - 128);  // V area
        uint4 x = make_uint4(threadIdx.x, 1, 2, 3);
        while (!done) {
            if (INTF == 1 || INTF == 2) {
                tmem_ld32(tR, v);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) acc += v[i];
                if (INTF == 2) {
                    tmem_st32(tR + 64, v);
                    tmem_wait_st();
                }
            } else if (INTF == 3) {
#pragma unroll
                for (int i = 0; i < 16; ++i) sp[(i * 128) % (CHUNK_Q / 16)] = x;
            } else if (INTF == 4) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const uint4 y = sp[(i * 128) % (CHUNK_Q / 16)];
                    acc += y.x ^ y.w;
                }
            }
        }
        if (acc == 0x12345678u) clk[255] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

template <int MODE, int INTF = 0>
static double run(int grid, int reps, long long *d)
{
    const int smem = 6 * CHUNK_Q + 32768 + 1024;
    static uint8_t *gsrc = nullptr;
    static long long *nb = nullptr;
    if (!gsrc) {
        cudaMalloc(&gsrc, (size_t)8192 * 32768);  // 256 MB: beyond L2, like the gathered K/V
        cudaMemset(gsrc, 0, (size_t)8192 * 32768);
        cudaMalloc(&nb, 256 * sizeof(long long));
    }
    cudaMemset(nb, 0, 256 * sizeof(long long));
    cudaFuncSetAttribute(umma_rate<MODE, INTF>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    umma_rate<MODE, INTF><<<grid, 256, smem>>>(d, reps, gsrc, nb);  // warm
    umma_rate<MODE, INTF><<<grid, 256, smem>>>(d, reps, gsrc, nb);
    if (INTF == 5) {
        cudaDeviceSynchronize();
        long long hb[256], hc[256];
        cudaMemcpy(hb, nb, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        cudaMemcpy(hc, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        printf("   (bulk-copy stream: %.1f B/clk per SM during the MMAs)\n", (double)hb[0] / hc[0]);
    }
    cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < grid; ++i) m += h[i];
    const int per_rep = MODE == 4 ? 16 : (MODE == 5 ? 12 : 8);
    return m / grid / ((double)reps * per_rep);
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long *d;
    cudaMalloc(&d, 256 * sizeof(long long));
    const int reps = 2000;
    const char *names[] = {"QK-SS N=128 (Q, K in SMEM)", "QK-SS N=64", "QK-TS N=128 (Q in TMEM)", "PV-TS N=128 (P in TMEM, V MN-major)",
                           "group [8 PV-TS ; 8 QK-SS]"};
    for (int grid : {1, sms}) {
        double c[5];
        c[0] = run<0>(grid, reps, d);
        c[1] = run<1>(grid, reps, d);
        c[2] = run<2>(grid, reps, d);
        c[3] = run<3>(grid, reps, d);
        c[4] = run<4>(grid, reps, d);
        for (int m = 0; m < 5; ++m) printf("grid %3d  %-40s %7.1f clk per MMA\n", grid, names[m], c[m]);
    }
    {
        const double h0 = run<5, 0>(sms, reps, d), h2 = run<5, 2>(sms, reps, d), h5 = run<5, 5>(sms, reps, d);
        printf("half-tile group [4 PV-TS ; 8 QK-SS N=64]: %.1f / %.1f / %.1f clk per MMA (alone / + tcgen05.ld+st / + bulk copies) = %.0f clk per group (nominal 4x64 + 8x32 = 512)\n",
               h0, h2, h5, h0 * 12);
    }
    const char *intf[] = {"none", "tcgen05.ld x32 loop (4 warps)", "tcgen05.ld + st x32 loop", "st.shared 16 B loop", "ld.shared 16 B loop",
                          "bulk copies global->shared"};
    for (int g = 0; g < 4; ++g) {
        double c[6];
        if (g == 0) {
            c[0] = run<0, 0>(sms, reps, d); c[1] = run<0, 1>(sms, reps, d); c[2] = run<0, 2>(sms, reps, d);
            c[3] = run<0, 3>(sms, reps, d); c[4] = run<0, 4>(sms, reps, d); c[5] = run<0, 5>(sms, reps, d);
        } else if (g == 1) {
            c[0] = run<4, 0>(sms, reps, d); c[1] = run<4, 1>(sms, reps, d); c[2] = run<4, 2>(sms, reps, d);
            c[3] = run<4, 3>(sms, reps, d); c[4] = run<4, 4>(sms, reps, d); c[5] = run<4, 5>(sms, reps, d);
        } else if (g == 2) {
            c[0] = run<1, 0>(sms, reps, d); c[1] = run<1, 1>(sms, reps, d); c[2] = run<1, 2>(sms, reps, d);
            c[3] = run<1, 3>(sms, reps, d); c[4] = run<1, 4>(sms, reps, d); c[5] = run<1, 5>(sms, reps, d);
        } else {
            c[0] = run<3, 0>(sms, reps, d); c[1] = run<3, 1>(sms, reps, d); c[2] = run<3, 2>(sms, reps, d);
            c[3] = run<3, 3>(sms, reps, d); c[4] = run<3, 4>(sms, reps, d); c[5] = run<3, 5>(sms, reps, d);
        }
        const char *gn[] = {"QK-SS N=128", "group [8 PV-TS ; 8 QK-SS]", "QK-SS N=64", "PV-TS N=128"};
        for (int i = 0; i < 6; ++i)
            printf("%-28s with %-32s %7.1f clk per MMA\n", gn[g], intf[i], c[i]);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
