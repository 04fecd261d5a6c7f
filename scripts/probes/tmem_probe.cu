// Probe: tcgen05.ld round-trip latency (ld.32x32b.x32 + wait::ld) and throughput.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2505_19342_b200/csrc -o tmem_probe tmem_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace astra;
__global__ void k(long long* out, int iters, int mode) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[32];
    if (mode == 0) {  // dependent: ld, wait, use
      tmem_ld32(t + ((i * 32 + acc) & 127), r);
      tmem_ld_wait();
      acc += r[0] & 1;
    } else {          // two loads in flight per wait
      uint32_t r2[32];
      tmem_ld32(t + ((i * 32) & 127), r);
      tmem_ld32(t + ((i * 32 + 64) & 127), r2);
      tmem_ld_wait();
      acc += (r[0] ^ r2[5]) & 1;
    }
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 8 + warp] = (t1 - t0) / iters + (acc & 0);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(slot); }
}
int main() {
  long long* o; cudaMalloc(&o, 148 * 8 * 8);
  long long h[8];
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {1, 4, 8}) {
      k<<<1, warps * 32>>>(o, 1000, mode);
      cudaDeviceSynchronize();
      cudaMemcpy(h, o, 8 * 8, cudaMemcpyDeviceToHost);
      printf("mode %d (%s), %d warps: %lld cycles per iteration (warp 0)\n", mode,
             mode ? "2 loads/wait" : "1 load/wait", warps, h[0]);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
