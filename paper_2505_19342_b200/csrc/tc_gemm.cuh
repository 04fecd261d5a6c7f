// Persistent warp-specialised tcgen05 GEMM mainloop for sm_100a.
//
//   D[M, N] = A[M, K] * B[N, K]^T      (both operands K-major bf16, f32 accumulate in TMEM)
//
// PASSES == 1 : plain bf16 GEMM (fast mode).
// PASSES == 3 : split-precision "bf16x3": A = Ahi + Alo, B = Bhi + Blo (each bf16) and
//               D = Ahi*Bhi + Ahi*Blo + Alo*Bhi, which reproduces an fp32 GEMM to
//               ~2^-16 relative per product (parity mode / VQ distance scores).
//
// Roles (192 threads, one CTA per SM, persistent over output tiles):
//   warp 0      : TMA producer (one lane)            smem ring of STAGES {A[,Alo],B[,Blo]} tiles
//   warp 1      : TMEM allocator + UMMA issuer (one lane)
//   warps 2..5  : epilogue; warp w drains TMEM lanes 32*(w%4) .. +31 (one output row per thread)
// Two TMEM accumulators (2*BN columns) let the epilogue of tile i overlap the MMAs of tile i+1.
#pragma once
#include <cuda.h>
#include "ptx.cuh"

namespace astra {

constexpr int kBM = 128;  // UMMA M (rows per tile)
constexpr int kBK = 64;   // bf16 elements per 128-byte swizzle row
constexpr int kUK = 16;   // UMMA K for kind::f16
constexpr int kEpiWarps = 16;     // four warps per TMEM lane quarter, each owns 1/4 of the columns
constexpr int kEpiParts = kEpiWarps / 4;
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiStageBytes = 2048 + 64;   // per-epilogue-warp smem: 32x16 fp32 tile + 16 floats

template <int BN, int PASSES>
struct GemmSmem {
  static constexpr int kATile = kBM * kBK * 2;       // bytes
  static constexpr int kBTile = BN * kBK * 2;
  static constexpr int kOperands = (PASSES == 3) ? 2 : 1;
  static constexpr int kStageBytes = kOperands * (kATile + kBTile);
};

template <int BN, int PASSES, int STAGES>
constexpr int gemm_smem_bytes() {
  return STAGES * GemmSmem<BN, PASSES>::kStageBytes + kEpiWarps * kEpiStageBytes +
         1024 /*align*/ + 256 /*barriers*/;
}

struct TileCoord {
  int m_blk, n_blk, batch;
};

// Tile scheduler: tiles enumerate (batch, m_blk, n_blk) with n fastest.  B (weights, a
// codebook) is a few MB and stays L2-resident; A (activations, up to ~80 MB) is the stream,
// so the CTAs that share an A row-block run concurrently and A crosses HBM once
// (m-fastest order re-read the 77 MB W2 operand from DRAM once per column tile).
struct TileSched {
  int num_m, num_n, num_b;
  __device__ int total() const { return num_m * num_n * num_b; }
  __device__ TileCoord get(int t) const {
    TileCoord c;
    c.n_blk = t % num_n;
    t /= num_n;
    c.m_blk = t % num_m;
    c.batch = t / num_m;
    return c;
  }
};

// Epi must provide:
//   __device__ void operator()(const TileCoord&, int row_in_tile /*0..127*/,
//                              uint32_t tmem_row_addr /*lane-qualified TMEM address of col 0*/,
//                              int col_begin, int col_end, int part /*this warp's column
//                              quarter (BN/4 columns)*/,
//                              uint8_t* stage /*kEpiStageBytes of warp-private smem*/) const;
// It reads its accumulator row via tmem_ld32 (warp-collective) and writes results.
template <int BN, int PASSES, int STAGES, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAlo,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBlo,
                   int K, TileSched sched, int a_batch_rows, int b_batch_rows, Epi epi) {
  using S = GemmSmem<BN, PASSES>;
  constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                 : (2 * BN <= 256) ? 256 : 512;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_stage = smem + STAGES * S::kStageBytes;
  uint64_t* full_bar =
      reinterpret_cast<uint64_t*>(epi_stage + kEpiWarps * kEpiStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int num_kb = (K + kBK - 1) / kBK;
  const int total = sched.total();

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (PASSES == 3) {
      tma_prefetch_desc(&tmAlo);
      tma_prefetch_desc(&tmBlo);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 32 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        TileCoord tc = sched.get(t);
        const int arow = tc.batch * a_batch_rows + tc.m_blk * kBM;
        const int brow = tc.batch * b_batch_rows + tc.n_blk * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * S::kStageBytes;
          mbar_arrive_expect_tx(&full_bar[stage], S::kStageBytes);
          tma_load_2d(st, &tmA, &full_bar[stage], kb * kBK, arow, kEvictNormal);
          tma_load_2d(st + S::kATile, &tmB, &full_bar[stage], kb * kBK, brow, kEvictLast);
          if (PASSES == 3) {
            tma_load_2d(st + S::kATile + S::kBTile, &tmAlo, &full_bar[stage], kb * kBK, arow,
                        kEvictNormal);
            tma_load_2d(st + 2 * S::kATile + S::kBTile, &tmBlo, &full_bar[stage], kb * kBK, brow,
                        kEvictLast);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------ MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t st = smem_u32(smem + stage * S::kStageBytes);
          const uint32_t a_hi = st, b_hi = st + S::kATile;
          const uint32_t a_lo = st + S::kATile + S::kBTile, b_lo = st + 2 * S::kATile + S::kBTile;
#pragma unroll
          for (int kk = 0; kk < kBK / kUK; ++kk) {
            const uint32_t koff = kk * kUK * 2;  // bytes inside the 128B swizzle row
            const uint32_t accum = (kb > 0 || kk > 0) ? 1u : 0u;
            umma_f16(d_tmem, sdesc_kmajor_sw128(a_hi + koff), sdesc_kmajor_sw128(b_hi + koff), idesc,
                     accum);
            if (PASSES == 3) {
              umma_f16(d_tmem, sdesc_kmajor_sw128(a_hi + koff), sdesc_kmajor_sw128(b_lo + koff),
                       idesc, 1u);
              umma_f16(d_tmem, sdesc_kmajor_sw128(a_lo + koff), sdesc_kmajor_sw128(b_hi + koff),
                       idesc, 1u);
            }
          }
          umma_commit(&empty_bar[stage]);  // smem slot free once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const uint32_t quarter = warp & 3;
    const int row_in_tile = quarter * 32 + lane;
    const int part = (warp - 2) / 4;
    const int col_begin = part * (BN / kEpiParts), col_end = col_begin + BN / kEpiParts;
    uint8_t* stage = epi_stage + (warp - 2) * kEpiStageBytes;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      TileCoord tc = sched.get(t);
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + acc * BN;
      epi(tc, row_in_tile, taddr, col_begin, col_end, part, stage);
      tc_fence_before();
      mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace astra
