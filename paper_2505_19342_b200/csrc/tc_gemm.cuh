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
#include <cstdio>
#include <cstdlib>
#include "ptx.cuh"

namespace astra {

constexpr int kBM = 128;  // UMMA M (rows per tile)
constexpr int kBK = 64;   // bf16 elements per 128-byte swizzle row
constexpr int kUK = 16;   // UMMA K for kind::f16
constexpr int kEpiWarps = 16;     // four warps per TMEM lane quarter, each owns 1/4 of the columns
constexpr int kEpiParts = kEpiWarps / 4;
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiStageBytes = 2048 + 64;   // per-epilogue-warp smem: 32x16 fp32 tile + 16 floats

// Per-CTA smem stage: A tile (128 rows) and this CTA's share of the B tile (all BN rows,
// or BN/2 when a CTA pair splits B across its two SMs), times 2 for the bf16x3 lo operands.
template <int BN, int PASSES, int CLUSTER = 1>
struct GemmSmem {
  static constexpr int kATile = kBM * kBK * 2;       // bytes
  static constexpr int kBTile = (CLUSTER == 1 ? BN : BN / 2) * kBK * 2;
  static constexpr int kOperands = (PASSES == 3) ? 2 : 1;
  static constexpr int kStageBytes = kOperands * (kATile + kBTile);
};

template <int BN, int PASSES, int STAGES, int CLUSTER = 1>
constexpr int gemm_smem_bytes() {
  return STAGES * GemmSmem<BN, PASSES, CLUSTER>::kStageBytes + kEpiWarps * kEpiStageBytes +
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
  int cluster;  // CTAs per cluster: 1, 2 (a pair along M) or 4 (two pairs along N)
  int runs = 0;  // 1: a CTA (pair) takes a row block and ALL its column tiles in order (a "run"),
                 // so a stateful epilogue can reduce across the columns of a row
  __device__ int cm() const { return cluster >= 2 ? 2 : 1; }
  __device__ int cn() const { return cluster == 4 ? 2 : 1; }
  __device__ int num_units_m() const { return (num_m + cm() - 1) / cm(); }
  __device__ int num_units_n() const { return (num_n + cn() - 1) / cn(); }
  __device__ int total() const { return num_units_m() * num_units_n() * num_b; }
  // rank bit 0 = row block within the pair, bit 1 = column tile within the cluster
  __device__ TileCoord get(int t, int rank) const {
    TileCoord c;
    const int un = num_units_n();
    c.n_blk = (t % un) * cn() + (rank >> 1);
    t /= un;
    const int mu = num_units_m();
    c.m_blk = (t % mu) * cm() + (rank & 1);
    c.batch = t / mu;
    return c;
  }
};

// Tile sequence of one persistent CTA: tiles t = unit0, unit0 + units, ... (runs = 0: every
// tile is a run of its own) or, with runs, row-block units rb = unit0, unit0 + units, ... each
// followed through all its column tiles (t = rb * units_n + n).
struct TileIter {
  int t, n, un, rb, step, total, runs;
  __device__ TileIter(const TileSched& s, int unit0, int units) {
    un = s.num_units_n();
    runs = s.runs;
    step = units;
    total = s.total();
    rb = unit0;
    n = 0;
    t = runs ? rb * un : unit0;
  }
  __device__ bool valid() const { return t < total; }
  __device__ bool first() const { return !runs || n == 0; }
  __device__ bool last() const { return !runs || n == un - 1; }
  __device__ void next() {
    if (!runs) {
      t += step;
      return;
    }
    if (++n == un) {
      n = 0;
      rb += step;
    }
    t = rb * un + n;
  }
};

// Epi::kStateful == false: stateless, per tile.  true: the epilogue keeps a per-thread
// Epi::State across the tiles of a run (TileSched::runs) and is told the run's first / last
// tile (e.g. the VQ argmin reducing a row over every code tile).
// Epi must provide:
//   __device__ void operator()(const TileCoord&, int row_in_tile /*0..127*/,
//                              uint32_t tmem_row_addr /*lane-qualified TMEM address of col 0*/,
//                              int col_begin, int col_end, int part /*this warp's column
//                              quarter (BN/4 columns)*/,
//                              uint8_t* stage /*kEpiStageBytes of warp-private smem*/) const;
// It reads its accumulator row via tmem_ld* (warp-collective) and writes results.
//
// CLUSTER == 4: two such pairs side by side along N.  The CTAs with the same row block in
// both pairs need the same A tile: each loads half of it (64 rows) and multicasts it to both,
// so per SM the TMA request traffic drops to (64 + BN/2) rows per k-step.  Bytes landing in a
// pair complete on that pair's leader barrier; a stage is free once BOTH pairs' MMAs have
// retired it (the leaders' commits are multicast to all four CTAs; empty count 2).
//
// CLUSTER == 2: a CTA pair (cta_group::2).  The two CTAs of a cluster own adjacent 128-row
// blocks of one 256-row tile; each loads its A rows and HALF of the B tile into its own smem,
// and the leader (even rank) issues M=256 UMMAs that read both CTAs' operands and write each
// CTA's TMEM rows.  Per SM the operand traffic drops from (128 + BN) to (128 + BN/2) rows per
// k-step — these GEMMs are bound by L2->SM bandwidth (~6.3 KB/clk chip-wide), not by the
// tensor pipe.  Barriers: the leader's full barrier counts both CTAs' TMA bytes; its MMA
// commits (multicast) release the stage / publish the accumulator in both CTAs; both CTAs'
// epilogue warps arrive on the leader's TMEM-empty barrier.
// Bench-only isolation switch (ASTRA_GEMM_DEBUG, gemm.cu): bit 0 skips the UMMAs (stages are
// still consumed and released), bit 1 skips the epilogue work, bit 2 skips the TMA loads.
// 0 in production.
static __device__ int g_gemm_debug = 0;

template <int BN, int PASSES, int STAGES, int CLUSTER, class Epi>
__global__ void __launch_bounds__(kGemmThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAlo,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBlo,
                   int K, TileSched sched, int a_batch_rows, int b_batch_rows,
                   const __grid_constant__ Epi epi) {
  using S = GemmSmem<BN, PASSES, CLUSTER>;
  static_assert(CLUSTER == 1 || CLUSTER == 2 || CLUSTER == 4, "cluster of 1, 2 or 4");
  constexpr bool kPair = CLUSTER >= 2;
  constexpr bool kQuad = CLUSTER == 4;
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
  const int dbg = g_gemm_debug;   // read once: the loops below clobber memory
  const int rank = kPair ? (int)cluster_ctarank() : 0;
  const bool leader = (rank & 1) == 0;   // issues the pair's UMMAs
  const int pair_leader = rank & ~1;
  const int unit0 = blockIdx.x / CLUSTER, units = gridDim.x / CLUSTER;
  const int num_kb = (K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (PASSES == 3) {
      tma_prefetch_desc(&tmAlo);
      tma_prefetch_desc(&tmBlo);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kQuad ? 2 : 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], kPair ? 2 * kEpiWarps : 32 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    if (kPair)
      tmem_alloc_pair<kTmemCols>(tmem_slot);
    else
      tmem_alloc<kTmemCols>(tmem_slot);
  }
  tc_fence_before();
  if (kPair)
    cluster_sync();  // the peer touches our barriers / TMEM only after they exist
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL (ptx.cuh): barriers, TMEM and descriptors were set up while the previous kernel of the
  // stream drained; every operand / epilogue access follows the wait
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer (both CTAs)
      const uint32_t full0 = kPair ? mapa_shared(full_bar, pair_leader) : smem_u32(full_bar);
      const uint16_t a_mask = (uint16_t)((1u << (rank & 1)) | (1u << ((rank & 1) + 2)));
      const uint32_t full_pb = smem_u32(full_bar) & kPeerBitMask;   // multicast form
      int stage = 0;
      uint32_t phase = 0;
      for (TileIter it(sched, unit0, units); it.valid(); it.next()) {
        TileCoord tc = sched.get(it.t, rank);
        const int arow = tc.batch * a_batch_rows + tc.m_blk * kBM;
        const int brow = tc.batch * b_batch_rows + tc.n_blk * BN + (kPair ? (rank & 1) * (BN / 2) : 0);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* st = smem + stage * S::kStageBytes;
          const int kc = kb * kBK;
          if (dbg & 4) {   // no loads: the stage is "full" at once (MMA on stale data)
            if (leader) mbar_arrive(&full_bar[stage]);
          } else if (kQuad) {
            // this CTA's half of the A tile goes to both pairs; B half to itself
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * S::kStageBytes);
            const uint32_t fb = full_pb + stage * 8, fl = full0 + stage * 8;
            const int half = rank >> 1;
            tma_load_2d_pair_mc(st + half * (S::kATile / 2), &tmA, fb, kc, arow + half * (kBM / 2),
                                a_mask, kEvictNormal);
            tma_load_2d_pair(st + S::kATile, &tmB, fl, kc, brow, kEvictLast);
            if (PASSES == 3) {
              tma_load_2d_pair_mc(st + S::kATile + S::kBTile + half * (S::kATile / 2), &tmAlo, fb,
                                  kc, arow + half * (kBM / 2), a_mask, kEvictNormal);
              tma_load_2d_pair(st + 2 * S::kATile + S::kBTile, &tmBlo, fl, kc, brow, kEvictLast);
            }
          } else if (kPair) {
            // both CTAs' bytes land on the leader's full barrier
            if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * S::kStageBytes);
            const uint32_t fb = full0 + stage * 8;
            tma_load_2d_pair(st, &tmA, fb, kc, arow, kEvictNormal);
            tma_load_2d_pair(st + S::kATile, &tmB, fb, kc, brow, kEvictLast);
            if (PASSES == 3) {
              tma_load_2d_pair(st + S::kATile + S::kBTile, &tmAlo, fb, kc, arow, kEvictNormal);
              tma_load_2d_pair(st + 2 * S::kATile + S::kBTile, &tmBlo, fb, kc, brow, kEvictLast);
            }
          } else {
            mbar_arrive_expect_tx(&full_bar[stage], S::kStageBytes);
            tma_load_2d(st, &tmA, &full_bar[stage], kc, arow, kEvictNormal);
            tma_load_2d(st + S::kATile, &tmB, &full_bar[stage], kc, brow, kEvictLast);
            if (PASSES == 3) {
              tma_load_2d(st + S::kATile + S::kBTile, &tmAlo, &full_bar[stage], kc, arow,
                          kEvictNormal);
              tma_load_2d(st + 2 * S::kATile + S::kBTile, &tmBlo, &full_bar[stage], kc, brow,
                          kEvictLast);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ------------------------------------------------------------ MMA issuer (leader)
      constexpr uint32_t idesc = idesc_bf16_f32(kBM * (kPair ? 2 : 1), BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (TileIter it(sched, unit0, units); it.valid(); it.next()) {
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
            if (dbg & 1) break;
            const uint32_t koff = kk * kUK * 2;  // bytes inside the 128B swizzle row
            const uint32_t accum = (kb > 0 || kk > 0) ? 1u : 0u;
            if (kPair) {
              umma_f16_pair(d_tmem, sdesc_kmajor_sw128(a_hi + koff),
                            sdesc_kmajor_sw128(b_hi + koff), idesc, accum);
              if (PASSES == 3) {
                umma_f16_pair(d_tmem, sdesc_kmajor_sw128(a_hi + koff),
                              sdesc_kmajor_sw128(b_lo + koff), idesc, 1u);
                umma_f16_pair(d_tmem, sdesc_kmajor_sw128(a_lo + koff),
                              sdesc_kmajor_sw128(b_hi + koff), idesc, 1u);
              }
            } else {
              umma_f16(d_tmem, sdesc_kmajor_sw128(a_hi + koff), sdesc_kmajor_sw128(b_hi + koff),
                       idesc, accum);
              if (PASSES == 3) {
                umma_f16(d_tmem, sdesc_kmajor_sw128(a_hi + koff), sdesc_kmajor_sw128(b_lo + koff),
                         idesc, 1u);
                umma_f16(d_tmem, sdesc_kmajor_sw128(a_lo + koff), sdesc_kmajor_sw128(b_hi + koff),
                         idesc, 1u);
              }
            }
          }
          // the smem slot is free once these MMAs retire (in both CTAs of a pair)
          if (kPair)
            umma_commit_pair_mc(&empty_bar[stage], kQuad ? 0xF : 0x3);
          else
            umma_commit(&empty_bar[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        // accumulator ready for the epilogue (of both CTAs)
        if (kPair)
          umma_commit_pair_mc(&tfull_bar[acc], (uint16_t)(0x3u << pair_leader));
        else
          umma_commit(&tfull_bar[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // -------------------------------------------------------------- epilogue (both CTAs)
    const uint32_t quarter = warp & 3;
    const int row_in_tile = quarter * 32 + lane;
    const int part = (warp - 2) / 4;
    const int col_begin = part * (BN / kEpiParts), col_end = col_begin + BN / kEpiParts;
    uint8_t* stage = epi_stage + (warp - 2) * kEpiStageBytes;
    const uint32_t tempty0 = kPair ? mapa_shared(tempty_bar, pair_leader) : 0u;
    int acc = 0;
    uint32_t acc_phase = 0;
    typename Epi::State est{};
    for (TileIter it(sched, unit0, units); it.valid(); it.next()) {
      TileCoord tc = sched.get(it.t, rank);
      // stateful epilogues stage their per-tile inputs while the accumulator is still being
      // computed (their global-load latency hides behind the wait)
      if constexpr (Epi::kStateful) epi.pre(tc, row_in_tile, col_begin, col_end, part, stage, est, it.first());
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((quarter * 32u) << 16) + acc * BN;
      if constexpr (Epi::kStateful) {
        epi(tc, row_in_tile, taddr, col_begin, col_end, part, stage, est, it.first(), it.last());
      } else {
        if (!(dbg & 2)) epi(tc, row_in_tile, taddr, col_begin, col_end, part, stage);
      }
      tc_fence_before();
      if (kPair) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);  // one arrival per warp
      } else {
        mbar_arrive(&tempty_bar[acc]);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait<0>();   // epilogues that store by TMA: complete before exit
  }

  tc_fence_before();
  if (kPair)
    cluster_sync();  // no CTA leaves (or frees TMEM) while its peer may still use the pair
  else
    __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if (kPair)
      tmem_dealloc_pair<kTmemCols>(tmem_base);
    else
      tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// Host launcher: persistent grid of at most one CTA per SM (pairs when CLUSTER == 2).
template <int BN, int PASSES, int STAGES, int CLUSTER, class Epi>
inline cudaError_t launch_tc_gemm(const CUtensorMap& ta, const CUtensorMap& talo,
                                  const CUtensorMap& tb, const CUtensorMap& tblo, int K,
                                  TileSched sched, int a_batch_rows, int b_batch_rows,
                                  const Epi& epi, cudaStream_t stream, int sms) {
  auto kern = tc_gemm_kernel<BN, PASSES, STAGES, CLUSTER, Epi>;
  constexpr int smem = gemm_smem_bytes<BN, PASSES, STAGES, CLUSTER>();
  static_assert(smem <= 232448, "GEMM smem budget exceeded");
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  sched.cluster = CLUSTER;
  const int cm = CLUSTER >= 2 ? 2 : 1, cn = CLUSTER == 4 ? 2 : 1;
  const long units_m = (sched.num_m + cm - 1) / cm;
  const long total = units_m * ((sched.num_n + cn - 1) / cn) * sched.num_b;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kGemmThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CLUSTER;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // Persistent grid = the clusters that can be co-resident.  Clusters live inside one GPC, so
  // with GPCs of odd / non-multiple SM counts fewer than sms / CLUSTER fit; launching more
  // would run the surplus as a second, mostly empty wave.
  static int max_clusters = 0;
  if (max_clusters == 0) {
    cfg.gridDim = dim3(CLUSTER * (sms / CLUSTER), 1, 1);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) n = sms / CLUSTER;
    max_clusters = n;
    if (getenv("ASTRA_GEMM_VERBOSE"))
      fprintf(stderr, "tc_gemm<BN=%d,P=%d,C=%d>: %d co-resident clusters (%d SMs)\n", BN, PASSES,
              CLUSTER, n, sms);
  }
  cfg.numAttrs = pdl_persistent() ? 2 : 1;
  const long max_units = max_clusters;
  const long work = sched.runs ? units_m * sched.num_b : total;   // runs: one unit per row block
  const int grid = (int)((work < max_units ? work : max_units) * CLUSTER);
  cfg.gridDim = dim3(grid, 1, 1);
  return cudaLaunchKernelEx(&cfg, kern, ta, talo, tb, tblo, K, sched, a_batch_rows, b_batch_rows,
                            epi);
}

}  // namespace astra
