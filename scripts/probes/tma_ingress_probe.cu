// Probe: TMA load ingress per SM (bytes/clk) with a bare load ring (no MMA): one CTA per SM,
// one thread issues 2-D tiled loads (SW128, 64 bf16 columns x box_rows rows) into an S-stage
// ring, one thread releases each stage as soon as it lands.  Source sized to stay in L2 or not.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2505_19342_b200/csrc -o tma_ingress_probe tma_ingress_probe.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace astra;

__global__ void __launch_bounds__(64, 1) k(const __grid_constant__ CUtensorMap map, int stages,
                                           int box_rows, int loads, int row_blocks, int col_blocks,
                                           long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  const int bytes = box_rows * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < loads; ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      mbar_arrive_expect_tx(&full[s], bytes);
      const int t = blockIdx.x + i * gridDim.x;   // spread tiles over the grid
      const int rb = t % row_blocks, cb = (t / row_blocks) % col_blocks;
      tma_load_2d(sm + s * bytes, &map, &full[s], cb * 64, rb * box_rows, 0x1000000000000000ull);
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < loads; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}


// GEMM-like: CTA pairs (cluster 2), per stage each CTA loads an A box (128 rows of a 12608x768
// operand) and a B box (128 rows of a 2304x768 operand), pair loads completing on the leader's
// barrier; the leader releases the stage in both CTAs (no MMA).  mode 1: per-CTA barriers.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64, 1)
    kpair(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int stages,
          int ksteps, int tiles_m, int tiles_n, int mode, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  cluster_sync();
  const uint32_t full0 = mapa_shared(full, 0);
  long long t0 = clock64();
  const int pair = blockIdx.x / 2, pairs = gridDim.x / 2;
  const int total = tiles_m * tiles_n;
  int it = 0;
  for (int t = pair; t < total; t += pairs) {
    const int mt = t / tiles_n, nt = t % tiles_n;
    for (int kb = 0; kb < ksteps; ++kb, ++it) {
      const int s = it % stages;
      const uint32_t ph = (it / stages) & 1;
      if (threadIdx.x == 0) {
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = sm + s * 32768;
        if (mode == 0) {
          if (leader) mbar_arrive_expect_tx(&full[s], 65536);
          tma_load_2d_pair(st, &ma, full0 + s * 8, kb * 64, (mt * 2 + rank) * 128, kEvictNormal);
          tma_load_2d_pair(st + 16384, &mb, full0 + s * 8, kb * 64, nt * 256 + rank * 128, kEvictLast);
        } else {
          mbar_arrive_expect_tx(&full[s], 32768);
          tma_load_2d(st, &ma, &full[s], kb * 64, (mt * 2 + rank) * 128, kEvictNormal);
          tma_load_2d(st + 16384, &mb, &full[s], kb * 64, nt * 256 + rank * 128, kEvictLast);
        }
      } else if (threadIdx.x == 32) {
        if (mode == 0) {
          if (leader) {
            mbar_wait(&full[s], ph);
            mbar_arrive(&empty[s]);
            mbar_arrive_cluster(mapa_shared(&empty[s], 1));
          }
        } else {
          mbar_wait(&full[s], ph);
          mbar_arrive(&empty[s]);
        }
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  cluster_sync();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / (it ? it : 1);
}


// 16 lanes of one warp each issue a 16-row box per stage (the attention producer's pattern)
__global__ void __launch_bounds__(64, 1) k16(const __grid_constant__ CUtensorMap map, int stages, int loads,
                                             int lanes, int row_blocks, int col_blocks, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  const int lane = threadIdx.x & 31;
  const int bytes = lanes * 2048;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    for (int i = 0; i < loads; ++i) {
      const int s = i % stages;
      const uint32_t ph = (i / stages) & 1;
      mbar_wait(&empty[s], ph ^ 1);
      if (lane == 0) mbar_arrive_expect_tx(&full[s], bytes);
      __syncwarp();
      if (lane < lanes) {
        const int t = (blockIdx.x + i * gridDim.x) * lanes + lane;
        tma_load_2d(sm + s * bytes + lane * 2048, &map, &full[s], (t / row_blocks) % col_blocks * 64,
                    (t % row_blocks) * 16, 0x1000000000000000ull);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < loads; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  const size_t rows = 65536, cols = 3072;   // 384 MB: rows limited below to choose L2 / HBM
  void* buf; cudaMalloc(&buf, rows * cols * 2); cudaMemset(buf, 0, rows * cols * 2);
  long long* out; cudaMalloc(&out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  long long h[148];

  {
    void* A; void* B;
    cudaMalloc(&A, 12608ull * 768 * 2); cudaMalloc(&B, 2304ull * 768 * 2);
    cudaMemset(A, 0, 12608ull * 768 * 2); cudaMemset(B, 0, 2304ull * 768 * 2);
    CUtensorMap ma, mb;
    cuuint64_t ga[2] = {768, 12608}, gb[2] = {768, 2304}, gs[1] = {768 * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&ma, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, A, ga, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, B, gb, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(kpair, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int mode = 0; mode < 0; ++mode)
      for (int stages : {3, 4, 5, 6}) {
        for (int rep = 0; rep < 2; ++rep)
          kpair<<<148, 64, stages * 32768 + 1024>>>(ma, mb, stages, 12, 12608 / 256, 2304 / 256, mode, out);
        cudaDeviceSynchronize();
        cudaMemcpy(h, out, 148 * 8, cudaMemcpyDeviceToHost);
        double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
        printf("QKV-like %s stages %d: %.0f clk per k-step per CTA = %.1f B/clk/SM (MMA needs 512 clk)\n",
               mode ? "per-CTA barriers" : "pair loads", stages, avg, 32768.0 / avg);
      }
  }

  {
    CUtensorMap map;
    cuuint64_t gdim[2] = {cols, 4096};
    cuuint64_t gstr[1] = {cols * 2};
    cuuint32_t box[2] = {64, 16};
    cuuint32_t es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(k16, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int lanes : {1, 4, 16, 32}) {
      const int stages = lanes == 32 ? 2 : 4, loads = 400;
      for (int rep = 0; rep < 2; ++rep)
        k16<<<148, 64, stages * lanes * 2048 + 1024>>>(map, stages, loads, lanes, 4096 / 16, cols / 64, out);
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, 148 * 8, cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
      printf("16-row boxes, %2d lanes issuing per step: %.0f clk per box, %.1f B/clk/SM\n", lanes,
             avg / (loads * lanes), (double)loads * lanes * 2048 / avg);
    }
  }
  for (int use_rows : {4096}) {      // 24 MB (L2-resident) / 384 MB (HBM)
    for (int box_rows : {16}) {
      CUtensorMap map;
      cuuint64_t gdim[2] = {cols, (cuuint64_t)use_rows};
      cuuint64_t gstr[1] = {cols * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int stages : {4, 8, 16}) {
        const int bytes = box_rows * 128;
        if (stages * bytes > 190 * 1024) continue;
        const int loads = bytes >= 8192 ? (64 << 20) / bytes / 148 * 4 : 2000;
        for (int rep = 0; rep < 2; ++rep)
          k<<<148, 64, stages * bytes + 1024>>>(map, stages, box_rows, loads, use_rows / box_rows, cols / 64, out);
        cudaDeviceSynchronize();
        cudaMemcpy(h, out, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0; double avg = 0;
        for (int i = 0; i < 148; ++i) { mx = h[i] > mx ? h[i] : mx; avg += h[i] / 148.0; }
        printf("%s box %3dx64 (%2d KB) stages %2d: %.1f B/clk/SM (avg CTA), %.1f (slowest)\n",
               use_rows == 4096 ? "L2 " : "HBM", box_rows, bytes / 1024, stages,
               (double)loads * bytes / avg, (double)loads * bytes / mx);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
