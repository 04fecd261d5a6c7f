// Probe: throughput of the attention softmax inner loop on TMEM-resident scores.
// Per warp, repeated over groups of 32 columns: tcgen05.ld 32x32b.x32 (+wait), 32 exp2, bf16 pack,
// tcgen05.st 32x32b.x16.  Modes switch parts off to find the binding resource.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2505_19342_b200/csrc -o softmax_probe softmax_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace astra;

template <int kMode>
__global__ void k(long long* out, int iters, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (warp == 0) tmem_alloc<256>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int half = warp >> 2, halves = nw >> 2;
  const uint32_t t = slot + ((uint32_t)((warp & 3) * 32) << 16);
  float2 acc = make_float2(0.f, 0.f);
  const float2 sl = make_float2(0.18f, 0.18f), nm = make_float2(-1.f, -1.f);
  long long t0 = clock64();
  if (kMode == 4) {   // software-pipelined: group g+1 loads while group g computes
    for (int i = 0; i < iters; ++i) {
      uint32_t ra[32], rb[32], pk[16];
      int g = half;
      tmem_ld32(t + g * 32, ra);
      tmem_ld_wait();
      while (true) {
        const bool more = g + halves < 8;
        if (more) tmem_ld32(t + (g + halves) * 32, rb);
#pragma unroll
        for (int j = 0; j < 32; ++j) asm volatile("" : "+r"(ra[j]));
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 x = ffma2(make_float2(__uint_as_float(ra[j]), __uint_as_float(ra[j + 1])), sl, nm);
          const float2 e = make_float2(ex2_approx(x.x), ex2_approx(x.y));
          pk[j >> 1] = pack_bf16x2(e.x, e.y);
          acc = fadd2(acc, e);
        }
        tmem_st16(t + g * 16, pk);
        g += halves;
        if (!more) break;
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) ra[j] = rb[j];
      }
      tmem_st_wait();
    }
  } else if (kMode == 5) {   // two groups per load round trip
    for (int i = 0; i < iters; ++i) {
      for (int g = half; g < 8; g += 2 * halves) {
        uint32_t ra[32], rb[32], pk[16], pk2[16];
        tmem_ld32(t + g * 32, ra);
        tmem_ld32(t + (g + halves) * 32, rb);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) asm volatile("" : "+r"(ra[j]), "+r"(rb[j]));
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 x = ffma2(make_float2(__uint_as_float(ra[j]), __uint_as_float(ra[j + 1])), sl, nm);
          const float2 y = ffma2(make_float2(__uint_as_float(rb[j]), __uint_as_float(rb[j + 1])), sl, nm);
          const float2 e = make_float2(ex2_approx(x.x), ex2_approx(x.y));
          const float2 f = make_float2(ex2_approx(y.x), ex2_approx(y.y));
          pk[j >> 1] = pack_bf16x2(e.x, e.y);
          pk2[j >> 1] = pack_bf16x2(f.x, f.y);
          acc = fadd2(acc, fadd2(e, f));
        }
        tmem_st16(t + g * 16, pk);
        tmem_st16(t + (g + halves) * 16, pk2);
      }
      tmem_st_wait();
    }
  } else if (kMode >= 6) {   // ld + exp (kMode-5 of every 4 pairs by polynomial) + st
    constexpr int kP = kMode - 5;
    for (int i = 0; i < iters; ++i) {
      for (int g = half; g < 8; g += halves) {
        uint32_t r[32], pk[16];
        tmem_ld32(t + g * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) asm volatile("" : "+r"(r[j]));
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 x = ffma2(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), sl, nm);
          const float2 e = ((j >> 1) & 3) < kP ? exp2_poly2(x) : make_float2(ex2_approx(x.x), ex2_approx(x.y));
          pk[j >> 1] = pack_bf16x2(e.x, e.y);
          acc = fadd2(acc, e);
        }
        tmem_st16(t + g * 16, pk);
      }
      tmem_st_wait();
    }
  } else
  for (int i = 0; i < iters; ++i) {
    for (int g = half; g < 8; g += halves) {
      uint32_t r[32], pk[16];
      if (kMode != 3) {
        tmem_ld32(t + g * 32, r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) asm volatile("" : "+r"(r[j]));
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint((float)(j + i + g));
      }
      if (kMode == 1) {   // load only
#pragma unroll
        for (int j = 0; j < 32; ++j) acc.x += __uint_as_float(r[j]);
        continue;
      }
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 x = ffma2(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), sl, nm);
        const float2 e = make_float2(ex2_approx(x.x), ex2_approx(x.y));
        pk[j >> 1] = pack_bf16x2(e.x, e.y);
        acc = fadd2(acc, e);
      }
      if (kMode == 0 || kMode == 3) tmem_st16(t + g * 16, pk);
      else acc.x += __uint_as_float(pk[3] ^ pk[9]);
    }
    if (kMode == 0 || kMode == 3) tmem_st_wait();
  }
  long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + warp] = (t1 - t0) / iters;
  if (acc.x == 1234.5f) sink[threadIdx.x] = acc.y;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(slot); }
}

__global__ void acc_check(float* err) {
  float worst = 0.f;
  for (int i = threadIdx.x; i < 200000; i += blockDim.x) {
    const float x = -40.f + 40.f * i / 200000.f;
    const float2 e = exp2_poly2(make_float2(x, x - 0.37f));
    worst = fmaxf(worst, fabsf(e.x / exp2f(x) - 1.f));
    worst = fmaxf(worst, fabsf(e.y / exp2f(x - 0.37f) - 1.f));
  }
  atomicMax(reinterpret_cast<int*>(err), __float_as_int(worst));
}
int main() {
  { float* e; cudaMalloc(&e, 4); cudaMemset(e, 0, 4); acc_check<<<1, 256>>>(e); float h; cudaMemcpy(&h, e, 4, cudaMemcpyDeviceToHost); printf("poly max rel err %.3g\n", h); }
  long long* o; cudaMalloc(&o, 148 * 16 * 8);
  float* sink; cudaMalloc(&sink, 4096);
  long long h[16];
  const char* names[] = {"ld+exp+st", "ld only", "ld+exp (no st)", "exp+st (no ld)", "pipelined", "2 per wait", "poly 1/4", "poly 2/4", "poly 3/4"};
  for (int mode = 0; mode < 9; ++mode)
    for (int warps : {4, 8}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, warps * 32>>>(o, 200, sink);
        if (mode == 1) k<1><<<148, warps * 32>>>(o, 200, sink);
        if (mode == 2) k<2><<<148, warps * 32>>>(o, 200, sink);
        if (mode == 3) k<3><<<148, warps * 32>>>(o, 200, sink);
        if (mode == 4) k<4><<<148, warps * 32>>>(o, 200, sink);
        if (mode == 5) k<5><<<148, warps * 32>>>(o, 200, sink);
        if (mode == 6) k<6><<<148, warps * 32>>>(o, 200, sink);
        if (mode == 7) k<7><<<148, warps * 32>>>(o, 200, sink);
        if (mode == 8) k<8><<<148, warps * 32>>>(o, 200, sink);
      }
      cudaDeviceSynchronize();
      cudaMemcpy(h, o, 16 * 8, cudaMemcpyDeviceToHost);
      // cycles per pass over 8 groups (= 128 rows x 256 keys), i.e. per attention unit
      printf("%-16s %d warps: %lld cycles per 128x256 pass (MUFU bound 2048)\n", names[mode], warps, h[0]);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
