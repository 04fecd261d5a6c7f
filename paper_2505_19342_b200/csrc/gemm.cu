// Projection / MLP GEMMs of the Astra block with fused epilogues
// (reference: tensor.matmul tensor.py:142-155, add_bias :186-190, gelu :348-358,
// residual adds cluster.py:213 and :216).
//
// Epilogue I/O is staged through a warp-private 4 KB shared-memory tile (128B-swizzled, so
// both the row-per-thread TMEM side and the coalesced global side are bank-conflict free):
// residual tiles are read with fully coalesced 16-byte loads, results leave as fully
// coalesced 16-byte stores (a warp writes 4 fp32 rows x 128 B or 8 bf16 rows x 64 B per
// instruction) instead of 32 scattered row segments.
#include <cstdlib>

#include "host_common.h"
#include "tc_gemm.cuh"

namespace astra {

// Warp-private staging (kEpiStageBytes): a 32-row x 16-column tile, 64 B (fp32) or 32 B (bf16)
// per row, with 16-byte chunks XOR-swizzled so the row-per-thread side and the coalesced
// side are both conflict-free (4 wavefronts per 512 B).
__device__ __forceinline__ float4* st_f32(uint8_t* stage, int r, int c) {  // c in 0..3
  return reinterpret_cast<float4*>(stage + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}
__device__ __forceinline__ uint4* st_bf(uint8_t* stage, int r, int c) {    // c in 0..1
  return reinterpret_cast<uint4*>(stage + r * 32 + ((c ^ ((r >> 2) & 1)) << 4));
}

// Epilogue flags: 0 = generic (the pointers / gelu field decide at run time); otherwise a
// compile-time specialisation for the block's hot GEMMs (no dead branches, no lo split when the
// output is bf16 only) — the W1 epilogue was instruction-bound at ~27 instructions per output.
constexpr int kEpBias = 1, kEpGeluFast = 2, kEpGeluExact = 4, kEpResid = 8, kEpF32 = 16,
              kEpHi = 32, kEpLo = 64;

template <int kF>
struct StdEpilogueT {
  // Stateful only to carry the residual prefetch: the warp's slice of the next 16-column
  // residual chunk (4 rows x 16 B per lane) is loaded one chunk ahead, and the first chunk of a
  // tile in pre(), before the accumulator is ready — the Wo / W2 epilogues stream 77 MB of
  // fp32 residual per launch, and one exposed HBM round trip per chunk left the per-SM
  // bandwidth share two-thirds idle.
  static constexpr bool kStateful = true;
  // (the generic form keeps the synchronous residual load: the prefetch registers made it spill)
  static constexpr bool kPrefetch = (kF & kEpResid) != 0;
  struct State {
    float4 res[kPrefetch ? 4 : 1];
    float bias2[2];   // this warp's column part (<= 64 columns): lane l holds cols l and 32 + l
  };
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
  int vec;  // all row pitches / bases allow 16-byte vectors
  // bf16-only outputs of the specialised epilogues (Q|K|V, W1): the warp's 32x16 chunk goes
  // out as one TMA store from a row-major staging buffer (two per warp, alternating) instead of
  // a shared-memory round trip and per-lane global stores
  static constexpr bool kTmaOut = kF != 0 && (kF & kEpHi) && !(kF & (kEpF32 | kEpLo));
  alignas(64) CUtensorMap tm_hi;   // out_hi [M, N], box 32 rows x 16 columns (set by the host)

  __device__ __forceinline__ void store_bf16(uint8_t* stage, __nv_bfloat16* out, int row0,
                                             int col0, const uint32_t (&h)[8]) const {
    const int lane = threadIdx.x & 31;
    *st_bf(stage, lane, 0) = make_uint4(h[0], h[1], h[2], h[3]);
    *st_bf(stage, lane, 1) = make_uint4(h[4], h[5], h[6], h[7]);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int rr = i * 16 + (lane >> 1), ch = lane & 1, grow = row0 + rr;
      if (grow < M)
        *reinterpret_cast<uint4*>(out + (size_t)grow * ld_bf + col0 + ch * 8) = *st_bf(stage, rr, ch);
    }
    __syncwarp();
  }

  // residual slice of the chunk at col0 for this lane: rows row0 + 8 i + lane / 4, 16 B chunk
  // lane % 4 (the coalesced pattern the staging tile transposes)
  __device__ __forceinline__ void load_res(float4 (&res)[kPrefetch ? 4 : 1], int row0, int col0) const {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < (kPrefetch ? 4 : 1); ++i) {
      const int grow = row0 + i * 8 + (lane >> 2);
      res[i] = grow < M ? __ldg(reinterpret_cast<const float4*>(residual + (size_t)grow * ld_res + col0) +
                                (lane & 3))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }

  __device__ __forceinline__ void pre(const TileCoord& tc, int row_in_tile, int cb, int ce,
                                      int /*part*/, uint8_t* /*stage*/, State& st,
                                      bool /*first*/) const {
    const int col0 = tc.n_blk * BN + cb;
    if (kPrefetch && col0 + 16 <= N)
      load_res(st.res, tc.m_blk * kBM + row_in_tile - (threadIdx.x & 31), col0);
    // the part's bias, loaded once per tile before the accumulator is ready (a per-chunk load
    // left one L2 round trip exposed per 16 columns: +6-8 us on the W1 / Q|K|V shapes)
    if (kF ? bool(kF & kEpBias) : bias != nullptr) {
      const int lane = threadIdx.x & 31, w = ce - cb;
      st.bias2[0] = (lane < w && col0 + lane < N) ? __ldg(bias + col0 + lane) : 0.f;
      st.bias2[1] = (32 + lane < w && col0 + 32 + lane < N) ? __ldg(bias + col0 + 32 + lane) : 0.f;
    }
  }

  __device__ __forceinline__ void operator()(const TileCoord& tc, int row_in_tile, uint32_t taddr,
                                             int cb, int ce, int /*part*/, uint8_t* stage,
                                             State& st, bool /*first*/, bool /*last*/) const {
    if (g_gemm_debug & 2) return;   // bench-only isolation switch (tc_gemm.cuh)
    const bool has_bias = kF ? bool(kF & kEpBias) : bias != nullptr;
    const int gmode = kF ? ((kF & kEpGeluFast) ? 2 : (kF & kEpGeluExact) ? 1 : 0) : gelu;
    const bool has_res = kF ? bool(kF & kEpResid) : residual != nullptr;
    const bool has_f32 = kF ? bool(kF & kEpF32) : out_f32 != nullptr;
    const bool has_hi = kF ? bool(kF & kEpHi) : out_hi != nullptr;
    const bool has_lo = kF ? bool(kF & kEpLo) : out_lo != nullptr;
    const bool vec_ok = kF ? true : vec != 0;
    const int lane = threadIdx.x & 31;
    const int row0 = tc.m_blk * kBM + row_in_tile - lane;  // first row of this warp's slab
    const int row = row0 + lane;
    const bool row_ok = row < M;
#pragma unroll 1
    for (int c0 = cb; c0 < ce; c0 += 16) {
      const int col0 = tc.n_blk * BN + c0;
      uint32_t r[16];
      tmem_ld16(taddr + c0, r);
      tmem_ld_wait();
      if (col0 >= N) continue;  // warp-uniform
      const bool full = (col0 + 16 <= N);
      const bool fast = full && vec_ok;
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
      if (has_bias) {   // broadcast from the lanes holding the part's bias (pre())
        const float bsrc = (c0 - cb) < 32 ? st.bias2[0] : st.bias2[1];
        const int l0 = (c0 - cb) & 31;
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] += __shfl_sync(0xffffffffu, bsrc, l0 + j);
      }
      if (gmode == 1) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = gelu_erf(v[j]);
      } else if (gmode == 2) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = gelu_erf_bf16(v[j]);
      }
      if constexpr (kPrefetch && (kF & kEpF32) && !(kF & kEpHi)) {
        if (fast) {
          // residual + fp32 output in the coalesced layout: one smem transpose of the
          // accumulator, then out = residual + acc per 16-byte chunk (the residual of this
          // chunk arrived with the previous one; the next chunk's loads go out first)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *st_f32(stage, lane, c) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          float4 rv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) rv[i] = st.res[i];
          if (c0 + 16 < ce && col0 + 32 <= N) load_res(st.res, row0, col0 + 16);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = i * 8 + (lane >> 2), ch = lane & 3, grow = row0 + rr;
            const float4 a = *st_f32(stage, rr, ch);
            if (grow < M)
              *(reinterpret_cast<float4*>(out_f32 + (size_t)grow * ld_f32 + col0) + ch) =
                  make_float4(rv[i].x + a.x, rv[i].y + a.y, rv[i].z + a.z, rv[i].w + a.w);
          }
          __syncwarp();
          continue;
        }
      }
      if (has_res) {
        if (fast) {
          if constexpr (kPrefetch) {
            // this chunk's residual arrived with the previous chunk (or pre()); the next
            // chunk's loads go out before this one is consumed
#pragma unroll
            for (int i = 0; i < 4; ++i) *st_f32(stage, i * 8 + (lane >> 2), lane & 3) = st.res[i];
            if (c0 + 16 < ce && col0 + 32 <= N) load_res(st.res, row0, col0 + 16);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int rr = i * 8 + (lane >> 2), ch = lane & 3, grow = row0 + rr;
              if (grow < M)
                *st_f32(stage, rr, ch) =
                    __ldg(reinterpret_cast<const float4*>(residual + (size_t)grow * ld_res + col0) + ch);
            }
          }
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const float4 q = *st_f32(stage, lane, c);
            v[4 * c] = q.x + v[4 * c];
            v[4 * c + 1] = q.y + v[4 * c + 1];
            v[4 * c + 2] = q.z + v[4 * c + 2];
            v[4 * c + 3] = q.w + v[4 * c + 3];
          }
          __syncwarp();
        } else if (row_ok) {
          const float* rp = residual + (size_t)row * ld_res + col0;
          for (int j = 0; j < 16; ++j)
            if (col0 + j < N) v[j] = rp[j] + v[j];
        }
      }
      if (has_f32) {
        if (fast) {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            *st_f32(stage, lane, c) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int rr = i * 8 + (lane >> 2), ch = lane & 3, grow = row0 + rr;
            if (grow < M)
              *(reinterpret_cast<float4*>(out_f32 + (size_t)grow * ld_f32 + col0) + ch) =
                  *st_f32(stage, rr, ch);
          }
          __syncwarp();
        } else if (row_ok) {
          float* op = out_f32 + (size_t)row * ld_f32 + col0;
          for (int j = 0; j < 16; ++j)
            if (col0 + j < N) op[j] = v[j];
        }
      }
      if (has_hi) {
        uint32_t hp[8], lp[8];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          __nv_bfloat162 h2 = __floats2bfloat162_rn(v[j], v[j + 1]);
          hp[j >> 1] = *reinterpret_cast<uint32_t*>(&h2);
          if (has_lo) {
            __nv_bfloat162 l2 = __floats2bfloat162_rn(v[j] - __low2float(h2), v[j + 1] - __high2float(h2));
            lp[j >> 1] = *reinterpret_cast<uint32_t*>(&l2);
          }
        }
        if (kTmaOut && fast) {
          // TMA needs a 128-byte aligned source: warp stages are 2112 B apart, so odd warps'
          // buffers start 64 B in (the stage's last 64 B are free: the bias is in registers)
          const uint32_t s0 = smem_u32(stage);
          const uint32_t buf = ((s0 + 127u) & ~127u) + (((c0 - cb) >> 4) & 1) * 1024;
          if (lane == 0) bulk_wait_read<1>();   // the store that read this buffer is done
          __syncwarp();
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 32), "r"(hp[0]),
                       "r"(hp[1]), "r"(hp[2]), "r"(hp[3]) : "memory");
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + lane * 32 + 16),
                       "r"(hp[4]), "r"(hp[5]), "r"(hp[6]), "r"(hp[7]) : "memory");
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tm_hi, buf, col0, row0);
            bulk_commit();
          }
        } else if (fast) {
          store_bf16(stage, out_hi, row0, col0, hp);
          if (has_lo) store_bf16(stage, out_lo, row0, col0, lp);
        } else if (row_ok) {
          __nv_bfloat16* hq = out_hi + (size_t)row * ld_bf + col0;
          __nv_bfloat16* lq = has_lo ? out_lo + (size_t)row * ld_bf + col0 : nullptr;
          const __nv_bfloat16* hs = reinterpret_cast<const __nv_bfloat16*>(hp);
          const __nv_bfloat16* ls = reinterpret_cast<const __nv_bfloat16*>(lp);
          for (int j = 0; j < 16; ++j)
            if (col0 + j < N) {
              hq[j] = hs[j];
              if (lq) lq[j] = ls[j];
            }
        }
      }
    }
  }
};

using StdEpilogue = StdEpilogueT<0>;

// Deepest operand ring that fits next to the epilogue staging (<= 192 KB of stages).
template <int BN, int PASSES, int CLUSTER>
constexpr int gemm_stages() {
  constexpr int per = GemmSmem<BN, PASSES, CLUSTER>::kStageBytes;
  constexpr int n = 196608 / per;
  return n > 8 ? 8 : n;
}

template <int BN, int PASSES, class Epi>
static int launch_std(const CUtensorMap& ta, const CUtensorMap& talo, const CUtensorMap& tb,
                      const CUtensorMap& tblo, int M, int N, int K, Epi epi,
                      cudaStream_t stream, int cluster) {
  TileSched sched{(M + kBM - 1) / kBM, (N + BN - 1) / BN, 1, 1};
  epi.BN = BN;
  const cudaError_t e =
      cluster == 4   ? launch_tc_gemm<BN, PASSES, gemm_stages<BN, PASSES, 4>(), 4>(
                         ta, talo, tb, tblo, K, sched, 0, 0, epi, stream, num_sms())
      : cluster == 2 ? launch_tc_gemm<BN, PASSES, gemm_stages<BN, PASSES, 2>(), 2>(
                         ta, talo, tb, tblo, K, sched, 0, 0, epi, stream, num_sms())
                     : launch_tc_gemm<BN, PASSES, gemm_stages<BN, PASSES, 1>(), 1>(
                         ta, talo, tb, tblo, K, sched, 0, 0, epi, stream, num_sms());
  ASTRA_CUDA_CHECK(e);
  return ASTRA_OK;
}

// A compile-time-specialised epilogue for the hot fast-mode GEMMs (CTA pairs, 1 pass).
template <int kF>
static int launch_spec(int BN, const CUtensorMap& ta, const CUtensorMap& talo,
                       const CUtensorMap& tb, const CUtensorMap& tblo, int M, int N, int K,
                       const StdEpilogue& g, cudaStream_t stream) {
  StdEpilogueT<kF> epi{g.M, g.N, g.bias, g.residual, g.ld_res, g.out_f32, g.ld_f32, g.out_hi,
                       g.out_lo, g.ld_bf, g.gelu, BN, g.vec};
  if constexpr (StdEpilogueT<kF>::kTmaOut) {
    const int st = make_tmap_2d(&epi.tm_hi, g.out_hi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, g.M, g.N,
                                g.ld_bf, 32, 16, false);
    if (st) return st;
  }
  TileSched sched{(M + kBM - 1) / kBM, (N + BN - 1) / BN, 1, 1};
  // (BN = 128: one rank's few token rows at N >= 8 — the generic epilogue spilled there)
  const cudaError_t e =
      BN == 256 ? launch_tc_gemm<256, 1, gemm_stages<256, 1, 2>(), 2>(ta, talo, tb, tblo, K, sched,
                                                                      0, 0, epi, stream, num_sms())
      : BN == 192 ? launch_tc_gemm<192, 1, gemm_stages<192, 1, 2>(), 2>(ta, talo, tb, tblo, K, sched,
                                                                        0, 0, epi, stream, num_sms())
                  : launch_tc_gemm<128, 1, gemm_stages<128, 1, 2>(), 2>(ta, talo, tb, tblo, K, sched,
                                                                        0, 0, epi, stream, num_sms());
  ASTRA_CUDA_CHECK(e);
  return ASTRA_OK;
}

// Cluster shape and tile width.  Measured on B200 (scripts/gemm_bench.py): the 1-pass
// mainloop moves ~29 B/clk of TMA operands per SM for every tile shape, and the 2x2 cluster
// with A multicast does not raise that (and only 33 four-CTA clusters are co-resident, i.e.
// 132 SMs), so the CTA pair is the default whenever there are two row blocks; cluster 4
// stays selectable (ASTRA_GEMM_CLUSTER=4) for A/B runs.  Tile width minimises persistent
// waves x per-SM operand rows per k-step (W1 12608x3072x768: BN 256 55.5 us vs 192 61.7 us).
static void pick_tile(int M, int N, int* bn_out, int* cluster_out) {
  const int sms = num_sms();
  const int num_m = (M + kBM - 1) / kBM;
  const int cl = num_m >= 2 ? 2 : 1;
  const int cands[3] = {256, 192, 128};
  double best_cost = 1e30;
  *bn_out = 128;
  *cluster_out = cl;
  for (int i = 0; i < 3; ++i) {
    const int bn = cands[i];
    if (bn > 128 && N < bn) continue;
    const long units = (long)((num_m + cl - 1) / cl) * ((N + bn - 1) / bn);
    const long slots = sms / cl;
    const long waves = (units + slots - 1) / slots;
    // a tile's k-step costs the operand rows this SM requests (ingress-bound mainloop)
    const double cost = (double)waves * (cl == 2 ? 128 + bn / 2 : 128 + bn);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      *bn_out = bn;
    }
  }
}

// General-shape fallback (K not a multiple of 8 or rows not 16-byte aligned: the small
// configs of the reference's own tests, e.g. hidden 4/12).  One thread per output element,
// A = hi (+ lo) and B = hi (+ lo) reconstructed in fp32, fp32 accumulation, the same
// epilogue as the tcgen05 kernel (bias, GELU, residual, fp32 / bf16 split outputs).
__global__ void gemm_simt_kernel(const __nv_bfloat16* __restrict__ a_hi,
                                 const __nv_bfloat16* __restrict__ a_lo, int lda,
                                 const __nv_bfloat16* __restrict__ b_hi,
                                 const __nv_bfloat16* __restrict__ b_lo, int ldb, int M, int N,
                                 int K, const float* __restrict__ bias,
                                 const float* __restrict__ residual, int ld_res,
                                 float* __restrict__ out_f32, int ld_f32,
                                 __nv_bfloat16* __restrict__ out_hi,
                                 __nv_bfloat16* __restrict__ out_lo, int ld_bf, int gelu) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (n >= N || m >= M) return;
  const __nv_bfloat16* ah = a_hi + (size_t)m * lda;
  const __nv_bfloat16* bh = b_hi + (size_t)n * ldb;
  float acc = 0.f;
  for (int k = 0; k < K; ++k) {
    float a = __bfloat162float(ah[k]), b = __bfloat162float(bh[k]);
    if (a_lo) a += __bfloat162float(a_lo[(size_t)m * lda + k]);
    if (b_lo) b += __bfloat162float(b_lo[(size_t)n * ldb + k]);
    acc = fmaf(a, b, acc);
  }
  float v = acc;
  if (bias) v += bias[n];
  if (gelu == 1) v = gelu_erf(v);
  else if (gelu == 2) v = gelu_erf_bf16(v);
  if (residual) v = residual[(size_t)m * ld_res + n] + v;
  if (out_f32) out_f32[(size_t)m * ld_f32 + n] = v;
  if (out_hi) {
    __nv_bfloat16 hi, lo;
    split_bf16(v, hi, lo);
    out_hi[(size_t)m * ld_bf + n] = hi;
    if (out_lo) out_lo[(size_t)m * ld_bf + n] = lo;
  }
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
  ASTRA_REQUIRE(passes == 1 || passes == 3, ASTRA_ERR_SHAPE, "astra_gemm: passes must be 1 or 3");
  ASTRA_REQUIRE(passes == 1 || (a_lo && b_lo), ASTRA_ERR_SHAPE,
                "astra_gemm: passes=3 needs lo operands");
  ASTRA_REQUIRE(out_lo == nullptr || out_hi != nullptr, ASTRA_ERR_SHAPE,
                "astra_gemm: out_lo requires out_hi");
  {
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const bool tma_ok = K % 8 == 0 && lda % 8 == 0 && ldb % 8 == 0 && al16(a_hi) && al16(b_hi) &&
                        (passes == 1 || (al16(a_lo) && al16(b_lo)));
    if (!tma_ok) {
      dim3 grid((N + 127) / 128, M);
      launch_k(gemm_simt_kernel, grid, 128, 0, as_stream(stream), 
          reinterpret_cast<const __nv_bfloat16*>(a_hi),
          passes == 3 ? reinterpret_cast<const __nv_bfloat16*>(a_lo) : nullptr, lda,
          reinterpret_cast<const __nv_bfloat16*>(b_hi),
          passes == 3 ? reinterpret_cast<const __nv_bfloat16*>(b_lo) : nullptr, ldb, M, N, K, bias,
          residual, ld_res, out_f32, ld_f32, reinterpret_cast<__nv_bfloat16*>(out_hi),
          reinterpret_cast<__nv_bfloat16*>(out_lo), ld_bf, gelu);
      ASTRA_CUDA_CHECK(cudaGetLastError());
      return ASTRA_OK;
    }
  }
  static int debug_set = -1;
  if (debug_set < 0) {   // bench-only isolation switch, see tc_gemm.cuh
    const char* d = getenv("ASTRA_GEMM_DEBUG");
    debug_set = d ? atoi(d) : 0;
    if (debug_set) ASTRA_CUDA_CHECK(cudaMemcpyToSymbol(g_gemm_debug, &debug_set, sizeof(int)));
  }
  int BN, cluster;
  pick_tile(M, N, &BN, &cluster);
  if (const char* f = getenv("ASTRA_GEMM_BN")) {   // A/B hook (benchmarks)
    const int b = atoi(f);
    if ((b == 128 || b == 192 || b == 256) && (b == 128 || N >= b)) BN = b;
  }
  if (const char* f = getenv("ASTRA_GEMM_CLUSTER")) {   // A/B hook (benchmarks)
    const int c = atoi(f);
    if ((c == 1) || (c == 2 && M > kBM) || (c == 4 && M > kBM && (N + BN - 1) / BN >= 2)) cluster = c;
  }
  const int brows = cluster == 1 ? BN : BN / 2;
  const int arows = cluster == 4 ? kBM / 2 : kBM;
  CUtensorMap ta, talo, tb, tblo;
  int st;
  if ((st = make_tmap_2d(&ta, a_hi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, K, lda, arows, kBK, true)))
    return st;
  if ((st = make_tmap_2d(&tb, b_hi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, N, K, ldb, brows, kBK,
                         true)))
    return st;
  if (passes == 3) {
    if ((st = make_tmap_2d(&talo, a_lo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, M, K, lda, arows, kBK,
                           true)))
      return st;
    if ((st = make_tmap_2d(&tblo, b_lo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, N, K, ldb, brows, kBK,
                           true)))
      return st;
  } else {
    talo = ta;
    tblo = tb;
  }
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const int vec = (!residual || (ld_res % 4 == 0 && al16(residual))) &&
                  (!out_f32 || (ld_f32 % 4 == 0 && al16(out_f32))) &&
                  (!out_hi || (ld_bf % 8 == 0 && al16(out_hi) && (!out_lo || al16(out_lo))));
  StdEpilogue epi{M,      N,      bias,
                  residual, ld_res, out_f32,
                  ld_f32, reinterpret_cast<__nv_bfloat16*>(out_hi),
                  reinterpret_cast<__nv_bfloat16*>(out_lo), ld_bf, gelu, 0, vec};
  cudaStream_t s = as_stream(stream);
  if (passes == 1 && cluster == 2 && vec && (BN == 256 || BN == 192 || BN == 128)) {
    const int flags = (bias ? kEpBias : 0) | (gelu == 2 ? kEpGeluFast : 0) |
                      (gelu == 1 ? kEpGeluExact : 0) | (residual ? kEpResid : 0) |
                      (out_f32 ? kEpF32 : 0) | (out_hi ? kEpHi : 0) | (out_lo ? kEpLo : 0);
    int st2 = -1;
    switch (flags) {   // the fast-mode block GEMMs: Q|K|V, W1, Wo, W2
      case kEpHi: st2 = launch_spec<kEpHi>(BN, ta, talo, tb, tblo, M, N, K, epi, s); break;
      case kEpBias | kEpGeluFast | kEpHi:
        st2 = launch_spec<kEpBias | kEpGeluFast | kEpHi>(BN, ta, talo, tb, tblo, M, N, K, epi, s);
        break;
      case kEpResid | kEpF32:
        st2 = launch_spec<kEpResid | kEpF32>(BN, ta, talo, tb, tblo, M, N, K, epi, s);
        break;
      case kEpBias | kEpResid | kEpF32:
        st2 = launch_spec<kEpBias | kEpResid | kEpF32>(BN, ta, talo, tb, tblo, M, N, K, epi, s);
        break;
      default: break;
    }
    if (st2 >= 0) return st2;
  }
  if (passes == 1) {
    if (BN == 256) return launch_std<256, 1>(ta, talo, tb, tblo, M, N, K, epi, s, cluster);  // 230 KB
    if (BN == 192) return launch_std<192, 1>(ta, talo, tb, tblo, M, N, K, epi, s, cluster);
    return launch_std<128, 1>(ta, talo, tb, tblo, M, N, K, epi, s, cluster);
  }
  if (BN == 256) return launch_std<256, 3>(ta, talo, tb, tblo, M, N, K, epi, s, cluster);
  if (BN == 192) return launch_std<192, 3>(ta, talo, tb, tblo, M, N, K, epi, s, cluster);
  return launch_std<128, 3>(ta, talo, tb, tblo, M, N, K, epi, s, cluster);
}
