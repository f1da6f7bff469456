// Micro-benchmark: one softmax warp's exp stream (FFMA2 scale, 2 x MUFU.EX2, FADD2 row sum,
// F2FP pack per key pair) with the compiler's order vs a hand-interleaved order (volatile
// asm: MUFU, FFMA2 of the next pair, MUFU, F2FP / FADD2 of the previous pair), W warps per SMSP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exp_order exp_order.cu && ./exp_order
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define NP 64  // pairs per tile row (128 keys)

__device__ __forceinline__ void ffma2v(float &d0, float &d1, float a0, float a1, float b, float c)
{
    asm volatile("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\t"
                 "mov.b64 rc, {%5, %5};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
                 : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
__device__ __forceinline__ void fadd2v(float &s0, float &s1, float a, float b)
{
    asm volatile("{\n\t.reg .b64 ra, rs;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rs, {%0, %1};\n\t"
                 "add.rn.f32x2 rs, rs, ra;\n\tmov.b64 {%0, %1}, rs;\n\t}" : "+f"(s0), "+f"(s1) : "f"(a), "f"(b));
}
__device__ __forceinline__ float ex2v(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t packv(float lo, float hi) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float ex2n(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ void ffma2n(float &d0, float &d1, float a0, float a1, float b, float c)
{
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\t"
        "mov.b64 rc, {%5, %5};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
__device__ __forceinline__ void fadd2n(float &s0, float &s1, float a, float b)
{
    asm("{\n\t.reg .b64 ra, rs;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rs, {%0, %1};\n\t"
        "add.rn.f32x2 rs, rs, ra;\n\tmov.b64 {%0, %1}, rs;\n\t}" : "+f"(s0), "+f"(s1) : "f"(a), "f"(b));
}
__device__ __forceinline__ uint32_t packn(float lo, float hi) { uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(r) : "f"(lo), "f"(hi)); return r; }

template <int MODE>
__global__ void kern(const float *in, uint32_t *out, long long *cyc, int reps)
{
    float s[2 * NP];
    for (int i = 0; i < 2 * NP; ++i) s[i] = in[(threadIdx.x * 7 + i) & 1023] * 0.01f;
    const float sl2 = 1.3f, mu = 0.7f;
    uint32_t acc = 0;
    float ps0 = 0.f, ps1 = 0.f, ps2 = 0.f, ps3 = 0.f;
    __syncwarp();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        uint32_t pk[NP];
        if (MODE == 0) {  // compiler order
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                float x0, x1;
                ffma2n(x0, x1, s[2 * i], s[2 * i + 1], sl2, -mu);
                const float a = ex2n(x0), b = ex2n(x1);
                if (i & 1) fadd2n(ps2, ps3, a, b); else fadd2n(ps0, ps1, a, b);
                pk[i] = packn(a, b);
            }
        } else {  // software pipelined, volatile: MUFU a(i), FFMA2 x(i+2), MUFU b(i), F2FP+FADD2 (i-1)
            float x0[NP], x1[NP], a[NP], b[NP];
            ffma2v(x0[0], x1[0], s[0], s[1], sl2, -mu);
            ffma2v(x0[1], x1[1], s[2], s[3], sl2, -mu);
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                a[i] = ex2v(x0[i]);
                if (i + 2 < NP) ffma2v(x0[i + 2], x1[i + 2], s[2 * i + 4], s[2 * i + 5], sl2, -mu);
                b[i] = ex2v(x1[i]);
                if (i >= MODE) {
                    const int j = i - MODE;
                    pk[j] = packv(a[j], b[j]);
                    if (j & 1) fadd2v(ps2, ps3, a[j], b[j]); else fadd2v(ps0, ps1, a[j], b[j]);
                }
            }
#pragma unroll
            for (int j = NP - MODE; j < NP; ++j) {
                pk[j] = packv(a[j], b[j]);
                if (j & 1) fadd2v(ps2, ps3, a[j], b[j]); else fadd2v(ps0, ps1, a[j], b[j]);
            }
        }
#pragma unroll
        for (int i = 0; i < NP; ++i) acc ^= pk[i];
#pragma unroll
        for (int i = 0; i < 2 * NP; ++i) s[i] += 1e-7f;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(ps0 + ps1 + ps2 + ps3);
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
}

template <int MODE>
void run(const char *name, float *in, uint32_t *out, long long *cyc, int W)
{
    const int reps = 64;
    kern<MODE><<<148, 128 * W>>>(in, out, cyc, reps);
    kern<MODE><<<148, 128 * W>>>(in, out, cyc, reps);
    cudaDeviceSynchronize();
    long long h[32];
    cudaMemcpy(h, cyc, sizeof(long long) * 4 * W, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < 4 * W; ++i) m += h[i];
    m /= 4 * W;
    printf("%-40s W=%d  %6.2f clk per pair per warp  (%6.1f clk per 64-pair tile row per SMSP)\n", name, W,
           m / (reps * NP), m / reps / W);
}

int main()
{
    float *in; uint32_t *out; long long *cyc;
    cudaMalloc(&in, 1024 * 4); cudaMemset(in, 0, 1024 * 4);
    cudaMalloc(&out, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 32 * 8);
    for (int W = 1; W <= 2; ++W) {
        run<0>("compiler order", in, out, cyc, W);
        run<1>("pipelined, pack/sum lag 1", in, out, cyc, W);
        run<2>("pipelined, pack/sum lag 2", in, out, cyc, W);
        run<4>("pipelined, pack/sum lag 4", in, out, cyc, W);
    }
    return 0;
}
