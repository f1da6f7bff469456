// Micro-benchmark: issue cost per warp-instruction on one SMSP of the softmax's instruction
// classes (MUFU.EX2, FFMA2, FADD2, FMNMX / FMNMX3, F2FP bf16x2 pack) alone and mixed, with
// W warps per SMSP.  Each loop body carries 8 independent chains so latency is hidden;
// the figure printed is clk per instruction of the class named first per warp... (see table).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates pipe_rates.cu && ./pipe_rates
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define N_IT 256

__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float mx3(float a, float b, float c) { float d; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float mx2(float a, float b) { float d; asm volatile("max.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ uint32_t pk(float a, float b) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void ffma2(float &a, float &b, float s, float c)
{
    asm volatile("{\n\t.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %2};\n\tmov.b64 rc, {%3, %3};\n\t"
                 "fma.rn.f32x2 ra, ra, rb, rc;\n\tmov.b64 {%0, %1}, ra;\n\t}" : "+f"(a), "+f"(b) : "f"(s), "f"(c));
}
__device__ __forceinline__ void fadd2(float &a, float &b, float c, float d)
{
    asm volatile("{\n\t.reg .b64 ra, rb;\n\tmov.b64 ra, {%0, %1};\n\tmov.b64 rb, {%2, %3};\n\t"
                 "add.rn.f32x2 ra, ra, rb;\n\tmov.b64 {%0, %1}, ra;\n\t}" : "+f"(a), "+f"(b) : "f"(c), "f"(d));
}
__device__ __forceinline__ float ffma(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }

__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2b2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
// MODE: 0 ex2, 1 ffma2, 2 fadd2, 3 fmnmx3, 4 fmnmx, 5 f2fp, 6 ffma, 7 ex2+fmnmx3 (1:1),
// 8 ex2+f2fp (2:1), 9 ex2+ffma2 (2:1), 10 full softmax mix per pair (ffma2, 2 ex2, fadd2, f2fp),
// 11 mode 10 + 2 fmnmx3 per pair
template <int MODE>
__global__ void kern(float *out, long long *cyc, float seed)
{
    float v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = seed * (threadIdx.x + i) * 1e-3f - 0.5f;
    uint32_t acc = 0;
    __syncwarp();
    const long long t0 = clock64();
    for (int it = 0; it < N_IT; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float &a = v[2 * j], &b = v[2 * j + 1];
            if (MODE == 0) { a = ex2f(a); }
            if (MODE == 12) { a = __uint_as_float(ex2h2(__float_as_uint(a))); }
            if (MODE == 13) { a = __uint_as_float(ex2b2(__float_as_uint(a))); }
            if (MODE == 1) { ffma2(a, b, 0.999f, -0.001f); }
            if (MODE == 2) { fadd2(a, b, v[(2 * j + 2) & 15], v[(2 * j + 3) & 15]); }
            if (MODE == 3) { a = mx3(a, b, v[(2 * j + 5) & 15]); }
            if (MODE == 4) { a = mx2(a, b); }
            if (MODE == 5) { acc += pk(a, b); a += 1e-7f; }
            if (MODE == 6) { a = ffma(a, 0.999f, b); }
            if (MODE == 7) { b = ex2f(a); a = mx3(a, b, v[(2 * j + 5) & 15]); }
            if (MODE == 8) { a = ex2f(a); b = ex2f(b); acc ^= pk(a, b); }
            if (MODE == 9) { a = ex2f(a); b = ex2f(b); ffma2(a, b, 0.999f, -0.001f); }
            if (MODE == 10 || MODE == 11) {
                float x0 = a, x1 = b;
                ffma2(x0, x1, 0.999f, -0.5f);
                x0 = ex2f(x0); x1 = ex2f(x1);
                fadd2(a, b, x0, x1);
                acc ^= pk(x0, x1);
                if (MODE == 11) { v[(2 * j + 4) & 15] = mx3(v[(2 * j + 4) & 15], x0, a); v[(2 * j + 6) & 15] = mx3(v[(2 * j + 6) & 15], x1, b); }
            }
        }
    }
    const long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)acc;
    if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32] = t1 - t0;
}

template <int MODE>
void run(const char *name, int per_iter, float *out, long long *cyc, int W)
{
    const int threads = 128 * W;
    kern<MODE><<<148, threads>>>(out, cyc, 1.0f);
    kern<MODE><<<148, threads>>>(out, cyc, 1.0f);
    cudaDeviceSynchronize();
    long long h[64];
    cudaMemcpy(h, cyc, sizeof(long long) * 4 * W, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < 4 * W; ++i) mean += h[i];
    mean /= 4 * W;
    // per SMSP: W warps each issued N_IT * 8 * per_iter instructions of the class
    printf("%-34s W=%d  %7.2f clk per warp-instr per SMSP (all W warps)\n", name, W,
           mean / ((double)N_IT * 8 * per_iter * W));
}

int main()
{
    float *out;
    long long *cyc;
    cudaMalloc(&out, 148 * 1024 * sizeof(float));
    cudaMalloc(&cyc, 148 * 64 * sizeof(long long));
    for (int W = 1; W <= 2; ++W) {
        run<0>("ex2 (MUFU)", 1, out, cyc, W);
        run<12>("ex2.approx.f16x2 (per pair)", 1, out, cyc, W);
        run<13>("ex2.approx.ftz.bf16x2 (per pair)", 1, out, cyc, W);
        run<1>("ffma2", 1, out, cyc, W);
        run<2>("fadd2", 1, out, cyc, W);
        run<3>("fmnmx3", 1, out, cyc, W);
        run<4>("fmnmx", 1, out, cyc, W);
        run<5>("f2fp bf16x2 (+fadd)", 2, out, cyc, W);
        run<6>("ffma", 1, out, cyc, W);
        run<7>("ex2+fmnmx3 (per pair of instr)", 2, out, cyc, W);
        run<8>("2 ex2 + f2fp (per instr, 3)", 3, out, cyc, W);
        run<9>("2 ex2 + ffma2 (per instr, 3)", 3, out, cyc, W);
        run<10>("softmax pair: 5 instr", 5, out, cyc, W);
        run<11>("softmax pair + 2 fmnmx3: 7 instr", 7, out, cyc, W);
    }
    printf("(clk per exp pair = 5 x or 7 x the last two figures)\n");
    return 0;
}
