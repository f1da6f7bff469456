// Micro-benchmark: FP64 DFMA and DMMA (m8n8k4) throughput on the current GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters) {
    double a[8], b = 1.0000001, c = 0.9999999;
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 123.0) out[0] = s;
}
__global__ void dmma_loop(double *out, int iters) {
    double c[8][2], a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 123.0) out[0] = s;
}
int main() {
    double *o; cudaMalloc(&o, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps = 4; warps <= 32; warps *= 2) {
        dim3 grid(sms * 2), block(32 * warps / 2);
        dfma_loop<<<grid, block>>>(o, 10); cudaDeviceSynchronize();
        cudaEventRecord(e0); dfma_loop<<<grid, block>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)grid.x * block.x;
        printf("DFMA  warps/SM=%2d: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
        dmma_loop<<<grid, block>>>(o, 10); cudaDeviceSynchronize();
        cudaEventRecord(e0); dmma_loop<<<grid, block>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 256 * 8 * iters * (double)grid.x * (block.x / 32);
        printf("DMMA  warps/SM=%2d: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
    }
    return 0;
}
