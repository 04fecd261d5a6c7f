// Probe: does a TMA box of ONE row (and a gather4 of 4 rows) landing at a 128-byte (512-byte)
// aligned offset inside a 1024-byte SW128 atom get the address-based 128B swizzle?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/tma_probe tma_swizzle_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstring>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap m1, const __grid_constant__ CUtensorMap m4,
                      uint16_t* out) {
  __shared__ __align__(1024) uint16_t sm[2][8 * 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(2 * 8 * 128));
    // buffer 0: row r of smem <- global row (7 - r), one-row boxes
    for (int r = 0; r < 8; ++r)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
          ::"r"(smem_u32(&sm[0][r * 64])), "l"(&m1), "r"(smem_u32(&bar)), "r"(0), "r"(7 - r) : "memory");
    // buffer 1: rows 0-3 <- gather4 {3, 9, 1, 12}; rows 4-7 <- gather4 {5, 0, 14, 2}
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
        ::"r"(smem_u32(&sm[1][0])), "l"(&m4), "r"(smem_u32(&bar)), "r"(0), "r"(3), "r"(9), "r"(1), "r"(12) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
        ::"r"(smem_u32(&sm[1][4 * 64])), "l"(&m4), "r"(smem_u32(&bar)), "r"(0), "r"(5), "r"(0), "r"(14), "r"(2) : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}\n" ::"r"(smem_u32(&bar)));
  for (int i = threadIdx.x; i < 2 * 8 * 64; i += blockDim.x) out[i] = (&sm[0][0])[i];
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int R = 16;
  uint16_t h[R * 64];
  for (int i = 0; i < R * 64; ++i) h[i] = (uint16_t)i;  // value = row*64 + col
  uint16_t *d, *o;
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, 2 * 8 * 64 * 2);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m1, m4;
  cuuint64_t gdim[2] = {64, R}, gstr[1] = {128};
  cuuint32_t box1[2] = {64, 1}, box4[2] = {64, 1}, es[2] = {1, 1};
  CUresult r1 = enc(&m1, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, gdim, gstr, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r4 = enc(&m4, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, gdim, gstr, box4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r4);
  probe<<<1, 128>>>(m1, m4, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  uint16_t res[2 * 8 * 64];
  cudaMemcpy(res, o, sizeof(res), cudaMemcpyDeviceToHost);
  const int g4[8] = {3, 9, 1, 12, 5, 0, 14, 2};
  for (int b = 0; b < 2; ++b) {
    int ok_sw = 1, ok_lin = 1;
    for (int r = 0; r < 8; ++r) {
      const int src = b == 0 ? 7 - r : g4[r];
      for (int c = 0; c < 8; ++c)
        for (int e2 = 0; e2 < 8; ++e2) {
          const uint16_t want = (uint16_t)(src * 64 + c * 8 + e2);
          if (res[b * 512 + r * 64 + ((c ^ r) * 8) + e2] != want) ok_sw = 0;
          if (res[b * 512 + r * 64 + c * 8 + e2] != want) ok_lin = 0;
        }
    }
    printf("buffer %d (%s): address-swizzled=%d linear=%d  row0:", b, b ? "gather4" : "1-row boxes", ok_sw, ok_lin);
    for (int i = 0; i < 16; ++i) printf(" %d", res[b * 512 + 64 + i * 8]);
    printf("\n");
  }
  return 0;
}
