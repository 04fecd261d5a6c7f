// Probe: MUFU.EX2 throughput per SM (ex2.approx.ftz.f32), vs FFMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_probe mufu_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ex2k(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int i = 0; i < iters; ++i) {
#define E(x) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x));
    E(a0) E(a1) E(a2) E(a3) E(a4) E(a5) E(a6) E(a7)
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void ex2bf(float* out, int iters) {
  unsigned a[8];
  for (int k = 0; k < 8; ++k) a[k] = 0x3c003c00u + threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[k]));
  }
  unsigned s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void ex2h(float* out, int iters) {
  unsigned a[8];
  for (int k = 0; k < 8; ++k) a[k] = 0x3c003c00u + threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[k]));
  }
  unsigned s = 0;
  for (int k = 0; k < 8; ++k) s += a[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
int main() {
  float* o;
  cudaMalloc(&o, 148 * 1024 * 4 * 8);
  int iters = 4096;
  for (int threads : {256, 512, 1024}) {
    cudaEvent_t s, e;
    cudaEventCreate(&s); cudaEventCreate(&e);
    ex2k<<<148, threads>>>(o, iters);
    cudaEventRecord(s);
    ex2k<<<148, threads>>>(o, iters);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    double ops = 148.0 * threads * iters * 8;
    printf("f32 ex2: threads/SM %d: %.3f ms, %.1f ex2/clk/SM (at 1.965 GHz)\n", threads, ms, ops / (ms * 1e-3) / 148 / 1.965e9);
    ex2bf<<<148, threads>>>(o, iters);
    cudaEventRecord(s);
    ex2bf<<<148, threads>>>(o, iters);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("bf16x2 ex2: threads/SM %d: %.3f ms, %.1f instr/clk/SM (x2 values)\n", threads, ms, ops / (ms * 1e-3) / 148 / 1.965e9);
    ex2h<<<148, threads>>>(o, iters);
    cudaEventRecord(s);
    ex2h<<<148, threads>>>(o, iters);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("f16x2 ex2: threads/SM %d: %.3f ms, %.1f instr/clk/SM (x2 values)\n", threads, ms, ops / (ms * 1e-3) / 148 / 1.965e9);
  }
  return 0;
}
