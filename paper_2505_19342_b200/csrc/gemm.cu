// Projection / MLP GEMMs of the Astra block with fused epilogues
// (reference: tensor.matmul tensor.py:142-155, add_bias :186-190, gelu :348-358,
// residual adds cluster.py:213 and :216).
#include "host_common.h"
#include "tc_gemm.cuh"

namespace astra {

struct StdEpilogue {
  int M, N;
  const float* bias;
  const float* residual;
  int ld_res;
  float* out_f32;
  int ld_f32;
  __nv_bfloat16* out_hi;
  __nv_bfloat16* out_lo;
  int ld_bf;
  int gelu;
  int BN;

  __device__ __forceinline__ void operator()(const TileCoord& tc, int row_in_tile,
                                             uint32_t taddr) const {
    const int row = tc.m_blk * kBM + row_in_tile;
    const bool row_ok = row < M;
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(taddr + c0, r);
      tmem_ld_wait();
      const int col0 = tc.n_blk * BN + c0;
      if (!row_ok || col0 >= N) continue;
      float v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
      const bool full = (col0 + 32 <= N);
      if (bias) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (full || col0 + j < N) v[j] += __ldg(bias + col0 + j);
      }
      if (gelu) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
      }
      if (residual) {
        const float* rp = residual + (size_t)row * ld_res + col0;
        if (full && ((reinterpret_cast<uintptr_t>(rp) & 15) == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 q = *reinterpret_cast<const float4*>(rp + j);
            v[j] = q.x + v[j];
            v[j + 1] = q.y + v[j + 1];
            v[j + 2] = q.z + v[j + 2];
            v[j + 3] = q.w + v[j + 3];
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (col0 + j < N) v[j] = rp[j] + v[j];
        }
      }
      if (out_f32) {
        float* op = out_f32 + (size_t)row * ld_f32 + col0;
        if (full && ((reinterpret_cast<uintptr_t>(op) & 15) == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(op + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
          for (int j = 0; j < 32; ++j)
            if (col0 + j < N) op[j] = v[j];
        }
      }
      if (out_hi) {
        __nv_bfloat16 hi[32], lo[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) split_bf16(v[j], hi[j], lo[j]);
        __nv_bfloat16* hp = out_hi + (size_t)row * ld_bf + col0;
        __nv_bfloat16* lp = out_lo ? out_lo + (size_t)row * ld_bf + col0 : nullptr;
        if (full && ((reinterpret_cast<uintptr_t>(hp) & 15) == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            *reinterpret_cast<uint4*>(hp + j) = *reinterpret_cast<const uint4*>(hi + j);
            if (lp) *reinterpret_cast<uint4*>(lp + j) = *reinterpret_cast<const uint4*>(lo + j);
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (col0 + j < N) {
              hp[j] = hi[j];
              if (lp) lp[j] = lo[j];
            }
        }
      }
    }
  }
};

template <int BN, int PASSES, int STAGES>
static int launch_std(const CUtensorMap& ta, const CUtensorMap& talo, const CUtensorMap& tb,
                      const CUtensorMap& tblo, int M, int N, int K, StdEpilogue epi,
                      cudaStream_t stream) {
  auto kern = tc_gemm_kernel<BN, PASSES, STAGES, StdEpilogue>;
  constexpr int smem = gemm_smem_bytes<BN, PASSES, STAGES>();
  static bool configured = false;
  if (!configured) {
    ASTRA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  TileSched sched{(M + kBM - 1) / kBM, (N + BN - 1) / BN, 1};
  const int tiles = sched.num_m * sched.num_n;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  epi.BN = BN;
  kern<<<grid, kGemmThreads, smem, stream>>>(ta, talo, tb, tblo, K, sched, 0, 0, epi);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

}  // namespace astra

using namespace astra;

extern "C" int astra_gemm(const void* a_hi, const void* a_lo, int lda, const void* b_hi,
                          const void* b_lo, int ldb, int M, int N, int K, int passes,
                          const float* bias, const float* residual, int ld_res, float* out_f32,
                          int ld_f32, void* out_hi, void* out_lo, int ld_bf, int gelu,
                          void* stream) {
  ASTRA_REQUIRE(M > 0 && N > 0 && K > 0, ASTRA_ERR_SHAPE, "astra_gemm: empty problem %dx%dx%d", M,
                N, K);
  ASTRA_REQUIRE(K % 8 == 0, ASTRA_ERR_SHAPE, "astra_gemm: K=%d must be a multiple of 8", K);
  ASTRA_REQUIRE(passes == 1 || passes == 3, ASTRA_ERR_SHAPE, "astra_gemm: passes must be 1 or 3");
  ASTRA_REQUIRE(passes == 1 || (a_lo && b_lo), ASTRA_ERR_SHAPE,
                "astra_gemm: passes=3 needs lo operands");
  ASTRA_REQUIRE(out_lo == nullptr || out_hi != nullptr, ASTRA_ERR_SHAPE,
                "astra_gemm: out_lo requires out_hi");
  // Wide N: 256-column tiles if that still fills the machine, else 128.
  const int num_m = (M + kBM - 1) / kBM;
  const bool wide = (N >= 256) && ((long)num_m * ((N + 255) / 256) >= num_sms());
  const int BN = wide ? 256 : 128;
  CUtensorMap ta, talo, tb, tblo;
  int st;
  if ((st = make_tmap_2d(&ta, a_hi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, K, lda, kBM, kBK, true)))
    return st;
  if ((st = make_tmap_2d(&tb, b_hi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, N, K, ldb, BN, kBK, true)))
    return st;
  if (passes == 3) {
    if ((st = make_tmap_2d(&talo, a_lo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, K, lda, kBM, kBK,
                           true)))
      return st;
    if ((st = make_tmap_2d(&tblo, b_lo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, N, K, ldb, BN, kBK,
                           true)))
      return st;
  } else {
    talo = ta;
    tblo = tb;
  }
  StdEpilogue epi{M,      N,      bias,
                  residual, ld_res, out_f32,
                  ld_f32, reinterpret_cast<__nv_bfloat16*>(out_hi),
                  reinterpret_cast<__nv_bfloat16*>(out_lo), ld_bf, gelu, 0};
  cudaStream_t s = as_stream(stream);
  if (passes == 1)
    return wide ? launch_std<256, 1, 4>(ta, talo, tb, tblo, M, N, K, epi, s)
                : launch_std<128, 1, 6>(ta, talo, tb, tblo, M, N, K, epi, s);
  return wide ? launch_std<256, 3, 2>(ta, talo, tb, tblo, M, N, K, epi, s)
              : launch_std<128, 3, 3>(ta, talo, tb, tblo, M, N, K, epi, s);
}
