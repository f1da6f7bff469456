// Micro-benchmark: MUFU.EX2 throughput with 8-32 independent chains per warp and 1-4 warps per
// SMSP (clk per warp-instruction per SMSP; 8.0 = 16 ex2 per clock per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_tput mufu_tput.cu && ./mufu_tput
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float ex2v(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int NCH>
__global__ void k(float *out, long long *clk, int iters) {
  float v[NCH];
  for (int i = 0; i < NCH; ++i) v[i] = -0.001f * (threadIdx.x + i);
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) v[i] = ex2v(v[i]) - 1.0f;
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NCH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int NCH> void run(int W) {
  float *o; long long *c; cudaMalloc(&o, 148*1024*4); cudaMalloc(&c, 148*8);
  int iters = 2048;
  k<NCH><<<148, 128*W>>>(o, c, iters); k<NCH><<<148, 128*W>>>(o, c, iters); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  // per SMSP: W warps x iters x NCH MUFU instructions (+ NCH FADD)
  printf("chains %2d  W=%d: %.2f clk per MUFU warp-instr per SMSP\n", NCH, W, (double)h / ((double)iters * NCH * W));
}
int main() { for (int W = 1; W <= 4; W *= 2) { run<8>(W); run<16>(W); run<32>(W); } return 0; }
