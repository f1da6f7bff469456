// Micro-benchmark: the attention softmax's exp phase (128 scores per thread -> packed bf16
// P + fp32 row sum, as in csrc/attn_fwd.cu) on registers only, timed per warp with
// clock64.  Configurations: W warps per SMSP (1 or 2) running the phase at the same time,
// and EMU = 0 / 4 (one pair in 4 through the FMA-pipe exp2 polynomial).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o softmax_exp softmax_exp.cu && ./softmax_exp
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2f(float x)
{
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void ex2_emu2(float &y0, float &y1, float x0, float x1)
{
    x0 = fmaxf(x0, -125.0f);
    x1 = fmaxf(x1, -125.0f);
    float j0, j1, p0, p1;
    asm("{\n\t.reg .b64 rx, rm, rj, rt, rf, rp, c3, c2, c1, c0;\n\t"
        "mov.b64 rx, {%4, %5};\n\tmov.b64 rm, {%6, %6};\n\t"
        "add.rn.f32x2 rj, rx, rm;\n\tsub.rn.f32x2 rt, rj, rm;\n\tsub.rn.f32x2 rf, rx, rt;\n\t"
        "mov.b64 c3, {%7, %7};\n\tmov.b64 c2, {%8, %8};\n\tmov.b64 c1, {%9, %9};\n\tmov.b64 c0, {%10, %10};\n\t"
        "fma.rn.f32x2 rp, rf, c3, c2;\n\tfma.rn.f32x2 rp, rp, rf, c1;\n\tfma.rn.f32x2 rp, rp, rf, c0;\n\t"
        "mov.b64 {%0, %1}, rj;\n\tmov.b64 {%2, %3}, rp;\n\t}"
        : "=f"(j0), "=f"(j1), "=f"(p0), "=f"(p1)
        : "f"(x0), "f"(x1), "f"(12582912.0f), "f"(0.05517162f), "f"(0.24261113f), "f"(0.69326097f),
          "f"(0.99992806f));
    y0 = __int_as_float(__float_as_int(p0) + (__float_as_int(j0) << 23));
    y1 = __int_as_float(__float_as_int(p1) + (__float_as_int(j1) << 23));
}
__device__ __forceinline__ void ffma2(float &d0, float &d1, float a0, float a1, float b, float c)
{
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\t"
        "mov.b64 rc, {%5, %5};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
__device__ __forceinline__ void fadd2(float &s0, float &s1, float a, float b)
{
    asm("{\n\t.reg .b64 ra, rs;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rs, {%0, %1};\n\t"
        "add.rn.f32x2 rs, rs, ra;\n\tmov.b64 {%0, %1}, rs;\n\t}"
        : "+f"(s0), "+f"(s1) : "f"(a), "f"(b));
}
__device__ __forceinline__ uint32_t pack(float lo, float hi)
{
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(lo), "f"(hi));
    return r;
}

template <int EMU>
__global__ void kern(const float *in, uint32_t *out, long long *cyc, int reps)
{
    float s[128];
    for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x * 7 + i) & 1023] * 0.01f;
    uint32_t acc = 0;
    float tot = 0.f;
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        const float sl2 = 0.127f + r * 1e-9f, mu = 3.0f;
        float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
            uint32_t pk[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int e = c2 * 64 + 2 * i;
                float x0, x1, a, b;
                ffma2(x0, x1, s[e], s[e + 1], sl2, -mu);
                if (EMU > 0 && (i % EMU) == EMU - 1) {
                    ex2_emu2(a, b, x0, x1);
                } else {
                    a = ex2f(x0);
                    b = ex2f(x1);
                }
                fadd2(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, b);
                pk[i] = pack(a, b);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) acc ^= pk[i];
        }
        tot += (ps[0] + ps[1]) + (ps[2] + ps[3]);
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(tot);
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}

// Interference probe: warps 0-3 (one per SMSP) run the exp phase; warps 4-7 (one more per
// SMSP) run an interference loop until the exp warps finish: MODE 1 = mbarrier try_wait on
// a phase that never completes (an idle waiter), MODE 2 = FMNMX3 chains (another warp's
// row-max phase), MODE 3 = the exp phase itself (MUFU contention).
template <int MODE>
__global__ void interfere(const float *in, uint32_t *out, long long *cyc, int reps)
{
    __shared__ unsigned long long bar;
    __shared__ volatile int done;
    if (threadIdx.x == 0) {
        done = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    }
    __syncthreads();
    const int w = threadIdx.x >> 5;
    if (w >= 4) {
        float a = in[threadIdx.x & 1023], b = a + 1.f, c = a - 1.f;
        uint32_t spins = 0;
        while (!done) {
            if (MODE == 1) {
                uint32_t ok;
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
                spins += ok;
            } else if (MODE == 2) {
#pragma unroll
                for (int i = 0; i < 64; ++i) {
                    float d;
                    asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
                    a = b; b = c; c = d;
                }
            } else if (MODE == 3) {
#pragma unroll
                for (int i = 0; i < 32; ++i) { a = ex2f(a * 0.5f); b = ex2f(b * 0.5f); }
            }
        }
        out[blockIdx.x * blockDim.x + threadIdx.x] = __float_as_uint(a + b + c) + spins;
        return;
    }
    float s[128];
    for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x * 7 + i) & 1023] * 0.01f;
    uint32_t acc = 0;
    float tot = 0.f;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        const float sl2 = 0.127f + r * 1e-9f, mu = 3.0f;
        float ps[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c2 = 0; c2 < 2; ++c2) {
            uint32_t pk[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int e = c2 * 64 + 2 * i;
                float x0, x1;
                ffma2(x0, x1, s[e], s[e + 1], sl2, -mu);
                const float a = ex2f(x0), b = ex2f(x1);
                fadd2(ps[(i & 1) * 2], ps[(i & 1) * 2 + 1], a, b);
                pk[i] = pack(a, b);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) acc ^= pk[i];
        }
        tot += (ps[0] + ps[1]) + (ps[2] + ps[3]);
    }
    const long long t1 = clock64();
    asm volatile("bar.sync 1, 128;");
    if (threadIdx.x == 0) done = 1;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(tot);
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 4 + w] = t1 - t0;
}

int main()
{
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *in;
    uint32_t *out;
    long long *cyc;
    cudaMalloc(&in, 1024 * 4);
    cudaMemset(in, 0, 1024 * 4);
    cudaMalloc(&out, sms * 512 * 4);
    cudaMalloc(&cyc, sms * 16 * 8);
    const int reps = 200;
    for (int wps = 1; wps <= 2; ++wps) {
        for (int emu = 0; emu <= 4; emu += 4) {
            const int threads = 128 * wps;  // wps warps per SMSP
            if (emu == 0) kern<0><<<sms, threads>>>(in, out, cyc, reps);
            else kern<4><<<sms, threads>>>(in, out, cyc, reps);
            cudaDeviceSynchronize();
            long long h[32];
            cudaMemcpy(h, cyc, (threads / 32) * 8, cudaMemcpyDeviceToHost);
            double m = 0;
            for (int w = 0; w < threads / 32; ++w) m += h[w];
            m /= threads / 32;
            printf("warps/SMSP=%d emu=%d: %.0f clk per 128-element exp phase per warp (%.0f per SMSP-tile)\n", wps,
                   emu, m / reps, m / reps / wps);
        }
    }
    for (int mode = 0; mode <= 3; ++mode) {
        if (mode == 0) interfere<0><<<sms, 256>>>(in, out, cyc, reps);
        if (mode == 1) interfere<1><<<sms, 256>>>(in, out, cyc, reps);
        if (mode == 2) interfere<2><<<sms, 256>>>(in, out, cyc, reps);
        if (mode == 3) interfere<3><<<sms, 256>>>(in, out, cyc, reps);
        cudaDeviceSynchronize();
        long long h[4];
        cudaMemcpy(h, cyc, 4 * 8, cudaMemcpyDeviceToHost);
        const double m = (h[0] + h[1] + h[2] + h[3]) / 4.0 / reps;
        const char *names[] = {"none", "mbarrier try_wait spinner", "FMNMX3 chains", "MUFU ex2 loop"};
        printf("exp phase with one interfering warp per SMSP (%s): %.0f clk\n", names[mode], m);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
