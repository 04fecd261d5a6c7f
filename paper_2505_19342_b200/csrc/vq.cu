// VQ encode / decode and the packed-index wire format.
//
// Reference: vq._nearest (vq.py:126-131) scores d2 = ||p||^2 - 2 p.c + ||c||^2 in
// fp64 and takes argmin with ties -> lowest index; vq.quantize (vq.py:207-222)
// runs it per group; vq.dequantize (vq.py:225-233) gathers centroid rows.
//
// Encode on B200 = three kernels (plus the fp64 re-rank of multi-candidate rows):
//   1. vq_split      fp32 token rows -> bf16 hi/lo split, one zero-padded [M, 64k] slab per
//                    group, and ||x_g|| (for the error window).
//   2. tc_gemm<VqEpilogue>  tcgen05 bf16x3 distance GEMM (scores = ||c||^2 - 2 x.c, the
//                    row-constant ||x||^2 dropped) with a fused per-row argmin epilogue that
//                    records, per 256-code chunk, the best score and every code inside the
//                    window best + 2*Delta.
//   3. vq_finalize   merge the chunks; a row with one surviving candidate is decided; rows
//                    with several are re-ranked in exact fp64 (reference formula and order);
//                    a chunk that overflowed its candidate list falls back to a full fp64 scan.
//
// Error window.  With x = xh + xl, c = ch + cl (bf16, RN) the computed xh.ch + xh.cl + xl.ch
// differs from x.c by at most 3.02 * 2^-16 * sum|x_i c_i| <= 3.02 * 2^-16 ||x|| ||c||
// (Cauchy-Schwarz) plus fp32 accumulation error; kTau = 2^-14 covers the former with 30%
// headroom left for the latter (measured |err| ~ 1.3e-6 ||x|| ||c||).  Score error is 2x
// that plus fp32 rounding of the epilogue arithmetic — bounded PER CODE with ||c_k|| (see
// window_a), so a code is a candidate iff its lower bound s_k - D_k reaches the best upper
// bound min_j (s_j + D_j).
#include <cstdlib>

#include "host_common.h"
#include "tc_gemm.cuh"

namespace astra {

constexpr int kVqBN = 256;      // distance-GEMM tile width (codes); 128 for small token counts
constexpr int kVqBNMin = 128;
constexpr int kVqCap = 4;          // candidates recorded per (row, chunk)
constexpr int kRRCands = 8;        // candidates handed to the re-rank kernel directly
constexpr int kRREntry = 2 + kRRCands;
constexpr float kTau = 1.0f / 16384.0f;

struct VqWorkspace {
  __nv_bfloat16* x_hi;
  __nv_bfloat16* x_lo;
  float* x_norm;      // [G, M]
  float* rec_best;    // [G, M, nchunk] U_chunk = min_j (s_j + D_j): an upper bound of the true
                      // best score among the chunk's codes
  float* rec_lmin;    // [G, M, nchunk] min_j (s_j - D_j) over the chunk
  int* rec_cnt;       // [G, M, nchunk]
  int* rec_idx;       // [G, M, nchunk, cap]
  float* rec_score;   // [G, M, nchunk, cap] lower bounds L_k = s_k - D_k of the candidates
  int* rr_list;       // [G * M][kRREntry] items whose window holds > 1 candidate (fp64 re-rank):
                      // {item, n (-1: scan the records), candidate codes ...}
  int* rr_count;      // [1]
  int* row_tok;       // [M] source row -> token (-1: not a token row); run mode over pre-split rows
  // run-mode items that need an exact scan of every code (a part's candidate list overflowed,
  // or > 8 candidates): split over kOvSub code ranges scanned by different warps of the re-rank
  // kernel; the warp finishing an item's last range reduces the partial argmins
  int* ov_list;       // [kOvCap] items
  int* ov_count;      // [2] items listed, range units claimed
  int* ov_done;       // [kOvCap] ranges finished per item
  double* ov_d;       // [kOvCap * kOvSub] partial best distance
  int* ov_k;          // [kOvCap * kOvSub] partial best code
};
constexpr int kOvCap = 1024, kOvSub = 16;

static inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t carve(VqWorkspace* w, void* base, int M, int G, int K, int gdp) {
  const int nchunk = kEpiParts * ((K + kVqBNMin - 1) / kVqBNMin);   // sized for the narrow tile
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  size_t o_hi = take((size_t)G * M * gdp * 2);
  size_t o_lo = take((size_t)G * M * gdp * 2);
  size_t o_norm = take((size_t)G * M * 4);
  size_t o_best = take((size_t)G * M * nchunk * 4);
  size_t o_lmin = take((size_t)G * M * nchunk * 4);
  size_t o_cnt = take((size_t)G * M * nchunk * 4);
  size_t o_idx = take((size_t)G * M * nchunk * kVqCap * 4);
  size_t o_sc = take((size_t)G * M * nchunk * kVqCap * 4);
  size_t o_rl = take((size_t)G * M * kRREntry * 4);
  size_t o_rc = take(4);
  size_t o_rt = take((size_t)M * 4);
  size_t o_ol = take((size_t)kOvCap * 4);
  size_t o_oc = take(8);
  size_t o_od = take((size_t)kOvCap * 4);
  size_t o_odd = take((size_t)kOvCap * kOvSub * 8);
  size_t o_ok = take((size_t)kOvCap * kOvSub * 4);
  if (w && base) {
    uint8_t* b = reinterpret_cast<uint8_t*>(base);
    w->x_hi = reinterpret_cast<__nv_bfloat16*>(b + o_hi);
    w->x_lo = reinterpret_cast<__nv_bfloat16*>(b + o_lo);
    w->x_norm = reinterpret_cast<float*>(b + o_norm);
    w->rec_best = reinterpret_cast<float*>(b + o_best);
    w->rec_lmin = reinterpret_cast<float*>(b + o_lmin);
    w->rec_cnt = reinterpret_cast<int*>(b + o_cnt);
    w->rec_idx = reinterpret_cast<int*>(b + o_idx);
    w->rec_score = reinterpret_cast<float*>(b + o_sc);
    w->rr_list = reinterpret_cast<int*>(b + o_rl);
    w->rr_count = reinterpret_cast<int*>(b + o_rc);
    w->row_tok = reinterpret_cast<int*>(b + o_rt);
    w->ov_list = reinterpret_cast<int*>(b + o_ol);
    w->ov_count = reinterpret_cast<int*>(b + o_oc);
    w->ov_done = reinterpret_cast<int*>(b + o_od);
    w->ov_d = reinterpret_cast<double*>(b + o_odd);
    w->ov_k = reinterpret_cast<int*>(b + o_ok);
  }
  return off;
}

// Error bound of the computed score s_k = ||c_k||^2 - 2 x.c_k (bf16x3 dot product, fp32
// epilogue) for a token of norm <= xn and a code of norm <= n_k:
//   D_k = 2 tau xn n_k + eps (n_k^2 + 2 xn n_k) = n_k (a + eps n_k) + tiny, a = (2 tau + 2 eps) xn.
// Per code, not per codebook: the true argmin k* satisfies s_k* - D_k* <= true score of k* <=
// true score of any j <= s_j + D_j, so every code with L_k = s_k - D_k above
// U = min_j (s_j + D_j) is excluded — a window of D_best + D_k instead of 4 tau xn max||c||
// (layer-input codebooks span ||c|| from ~0.2x to 1x of the max, so this is 2-6x tighter).
constexpr float kEps = 4.8e-7f;
__device__ __forceinline__ float window_a(float xn) { return (2.0f * kTau + 2.0f * kEps) * xn; }

// ------------------------------------------------------------ prepare
__global__ void vq_prepare_kernel(AstraCodebook cb) {
  pdl_wait();
  pdl_trigger();
  // one warp per (g, k) code row
  const int warps = (blockDim.x >> 5);
  const int code = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int G = cb.groups, K = cb.size, gd = cb.group_dim, gdp = cb.padded_dim;
  if (code >= G * K) return;
  const float* c = cb.centroids + (size_t)code * gd;
  __nv_bfloat16* hi = (__nv_bfloat16*)cb.c_hi + (size_t)code * gdp;
  __nv_bfloat16* lo = (__nv_bfloat16*)cb.c_lo + (size_t)code * gdp;
  double s64 = 0.0;
  for (int e = lane; e < gdp; e += 32) {
    float v = e < gd ? c[e] : 0.0f;
    __nv_bfloat16 h, l;
    split_bf16(v, h, l);
    hi[e] = h;
    lo[e] = l;
    s64 += (double)v * (double)v;
  }
  for (int o = 16; o; o >>= 1) s64 += __shfl_xor_sync(0xffffffffu, s64, o);
  if (lane == 0) {
    ((double*)cb.c_sq64)[code] = s64;
    ((float*)cb.c_sq)[code] = (float)s64;
    // per-code window terms: ||c|| rounded up, and the fp32-epilogue rounding term
    const float n = (float)sqrt(s64) * (1.0f + 1e-6f);
    ((float4*)cb.c_win)[code] = make_float4((float)s64, n, kEps * n * n, 0.f);
  }
}

__global__ void vq_normmax_kernel(AstraCodebook cb) {
  pdl_wait();
  pdl_trigger();
  const int g = blockIdx.x;
  float m = 0.f;
  for (int k = threadIdx.x; k < cb.size; k += blockDim.x)
    m = fmaxf(m, sqrtf((float)cb.c_sq64[(size_t)g * cb.size + k]));
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float r = 0.f;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmaxf(r, red[i]);
    // round up a hair so the window bound stays an upper bound
    ((float*)cb.c_norm_max)[g] = r * (1.0f + 1e-6f);
  }
}

// -------------------------------------------------------------- split
// one warp per token row: gather, split to bf16 hi/lo per group (zero padded), ||x_g||.
__global__ void vq_split_kernel(const float* __restrict__ x, int M, int ldx,
                                const int32_t* __restrict__ rows, int G, int gd, int gdp,
                                VqWorkspace w) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int r = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  // the re-rank list is appended to by the GEMM epilogue that follows: reset here
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *w.rr_count = 0;
    w.ov_count[0] = 0;
    w.ov_count[1] = 0;
  }
  if (r >= M) return;
  const int src = rows ? rows[r] : r;
  const float* xr = x + (size_t)src * ldx;
  for (int g = 0; g < G; ++g) {
    __nv_bfloat16* hi = w.x_hi + ((size_t)g * M + r) * gdp;
    __nv_bfloat16* lo = w.x_lo + ((size_t)g * M + r) * gdp;
    float ss = 0.f;
    for (int e = lane; e < gdp; e += 32) {
      float v = e < gd ? __ldg(xr + g * gd + e) : 0.0f;
      __nv_bfloat16 h, l;
      split_bf16(v, h, l);
      hi[e] = h;
      lo[e] = l;
      ss = fmaf(v, v, ss);
    }
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) w.x_norm[(size_t)g * M + r] = sqrtf(ss) * (1.0f + 1e-6f);
  }
}

// Vectorised form for unpadded groups (gd == gdp, gd % 4 == 0, gd/4 dividing or divisible by
// 32): float4 loads, 8-byte hi/lo stores, per-group norms by a segmented shuffle reduction.
// `per` = float4s per group; a warp covers 32 / per groups per step (per <= 32) or one group
// in per / 32 steps.
__global__ void vq_split_v4_kernel(const float* __restrict__ x, int M, int ldx,
                                   const int32_t* __restrict__ rows, int G, int gd, VqWorkspace w) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int r = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  // the re-rank list is appended to by the GEMM epilogue that follows: reset here
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *w.rr_count = 0;
    w.ov_count[0] = 0;
    w.ov_count[1] = 0;
  }
  if (r >= M) return;
  const int src = rows ? rows[r] : r;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)src * ldx);
  const int per = gd >> 2;
  auto put = [&](int g, int q, float4 v) {   // group g, float4 q of the group
    __nv_bfloat16 h[4], l[4];
    split_bf16(v.x, h[0], l[0]);
    split_bf16(v.y, h[1], l[1]);
    split_bf16(v.z, h[2], l[2]);
    split_bf16(v.w, h[3], l[3]);
    const size_t o = ((size_t)g * M + r) * gd + 4 * q;
    *reinterpret_cast<uint2*>(w.x_hi + o) = *reinterpret_cast<const uint2*>(h);
    *reinterpret_cast<uint2*>(w.x_lo + o) = *reinterpret_cast<const uint2*>(l);
    return fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, v.w * v.w)));
  };
  if (per <= 32) {
    const int gpi = 32 / per;
    for (int g0 = 0; g0 < G; g0 += gpi) {
      const int g = g0 + lane / per, q = lane % per;
      float ss = 0.f;
      if (g < G) ss = put(g, q, __ldg(xr + g * per + q));
      for (int o = per >> 1; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (g < G && q == 0) w.x_norm[(size_t)g * M + r] = sqrtf(ss) * (1.0f + 1e-6f);
    }
  } else {
    for (int g = 0; g < G; ++g) {
      float ss = 0.f;
      for (int q = lane; q < per; q += 32) ss += put(g, q, __ldg(xr + g * per + q));
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) w.x_norm[(size_t)g * M + r] = sqrtf(ss) * (1.0f + 1e-6f);
    }
  }
}

// Inverse of the token -> source-row map for the run-mode GEMM over pre-split stack rows
// (two launches: every row to -1, then the token rows; also resets the re-rank count).
__global__ void vq_row_tok_fill_kernel(int* row_tok, int R, int* rr_count, int* ov_count) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0) {
    *rr_count = 0;
    ov_count[0] = 0;
    ov_count[1] = 0;
  }
  if (r < R) row_tok[r] = -1;
}
__global__ void vq_row_tok_scatter_kernel(const int32_t* __restrict__ rows, int M, int* row_tok) {
  pdl_wait();
  pdl_trigger();
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m < M) row_tok[rows[m]] = m;
}

// ---------------------------------------------------------- epilogue
__device__ __forceinline__ void vq_decide(const AstraCodebook& cb, const float* __restrict__ x,
                                          int ldx, int src_row, int tok, int g, int Mtok,
                                          size_t rec0, int nchunk, const VqWorkspace& w,
                                          int32_t* __restrict__ idx_out, int32_t* __restrict__ stats,
                                          bool inline_rr, int lane);

__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_s32(uint32_t a, int v) {
  asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int lds_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float4 lds_v4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_v4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w) : "memory");
}
// Records epilogue (G = 1 over all 148 SMs; a row's codes span several tiles on different CTA
// pairs): per (row, 64-code part) the window's upper bound, min lower bound and up to kVqCap
// candidates; vq_finalize_kernel merges them.  (Finalizing inside the GEMM — the CTA completing
// a row block decides its rows — measured 141 us vs 52 + 7: the latency-bound decisions land
// on a few CTAs' critical paths.)
template <int BN>
struct VqEpilogue {
  static constexpr bool kStateful = true;
  static constexpr int kPartCols = BN / kEpiParts;   // 64 (BN 256) or 32 (BN 128)
  static constexpr int kCh = kPartCols / 32;
  struct State {
    float a;   // the row's window slope (2 tau + 2 eps) ||x||
  };
  int M, K, nchunk;         // nchunk = records per (g, row): kEpiParts per BN-code tile
  const float4* c_win;      // [G, K] {||c||^2, ||c||, eps ||c||^2, 0}
  VqWorkspace w;

  // While the MMAs run: the part's window terms into smem, SoA [0, 256) ||c||^2,
  // [256, 512) ||c||, [512, 768) -eps ||c||^2, [768, 1024) eps ||c||^2 (columns >= K:
  // ||c||^2 = +inf, never a candidate, U unaffected), and the row's window slope.
  __device__ __forceinline__ void pre(const TileCoord& tc, int row_in_tile, int cb, int ce,
                                      int part, uint8_t* stage, State& st, bool) const {
    const int lane = threadIdx.x & 31;
    const int g = tc.batch;
    const int col0 = tc.n_blk * BN + cb + lane;
    const float4* cw = c_win + (size_t)g * K;
    const float4 inf4 = make_float4(INFINITY, 0.f, 0.f, 0.f);
    const float4 c0 = col0 < K ? __ldg(cw + col0) : inf4;
    const float4 c1 = (kCh > 1 && col0 + 32 < K) ? __ldg(cw + col0 + 32) : inf4;
    const int row = tc.m_blk * kBM + row_in_tile;
    st.a = window_a(row < M ? w.x_norm[(size_t)g * M + row] : 0.f);
    const uint32_t s_scs = smem_u32(stage);
    __syncwarp();   // the previous tile's reads of the staged terms are done
    sts_f32(s_scs + 4 * lane, c0.x);
    sts_f32(s_scs + 256 + 4 * lane, c0.y);
    sts_f32(s_scs + 512 + 4 * lane, -c0.z);
    sts_f32(s_scs + 768 + 4 * lane, c0.z);
    if (kCh > 1) {
      sts_f32(s_scs + 128 + 4 * lane, c1.x);
      sts_f32(s_scs + 384 + 4 * lane, c1.y);
      sts_f32(s_scs + 640 + 4 * lane, -c1.z);
      sts_f32(s_scs + 896 + 4 * lane, c1.z);
    }
    __syncwarp();
  }

  // One TMEM read of the part; s_j = ||c_j||^2 - 2 x.c_j, U = min_j (s_j + D_j), candidates
  // L_j = s_j - D_j <= U (the part's own U; the finalize applies the global one) in code
  // order, and the part's min L — every expression the same single-rounding FMA/add as the
  // scalar form, in packed pairs (FFMA2 / FADD2).
  __device__ __forceinline__ void operator()(const TileCoord& tc, int row_in_tile, uint32_t taddr,
                                             int cb, int ce, int part, uint8_t* stage, State& st,
                                             bool, bool) const {
    const int row = tc.m_blk * kBM + row_in_tile;
    const bool ok = row < M;
    const int g = tc.batch;
    // the re-rank list count for the finalize kernel that follows (stream order): reset by
    // one thread here instead of a memset node in front of this GEMM
    if (tc.m_blk == 0 && tc.n_blk == 0 && g == 0 && row_in_tile == 0 && cb == 0) {
      *w.rr_count = 0;
      w.ov_count[0] = 0;   // (no overflow list in records mode)
    }
    const uint32_t s_scs = smem_u32(stage);
    const float a = st.a;
    // s_j of a 32-code chunk from a fresh TMEM read (two reads per chunk keep the epilogue
    // inside the kernel's 96-register budget)
    auto scores = [&](int c, float (&sv)[32]) {
      uint32_t r[32];
      tmem_ld32(taddr + cb + 32 * c, r);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 n2 = lds_v4(s_scs + 128 * c + 16 * q);
        const int j = 4 * q;
        const float2 t01 = ffma2(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])),
                                 make_float2(-2.0f, -2.0f), make_float2(n2.x, n2.y));
        const float2 t23 = ffma2(make_float2(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3])),
                                 make_float2(-2.0f, -2.0f), make_float2(n2.z, n2.w));
        sv[j] = t01.x;
        sv[j + 1] = t01.y;
        sv[j + 2] = t23.x;
        sv[j + 3] = t23.y;
      }
    };
    // pass 1: U = min_j (s_j + D_j)
    float u4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#pragma unroll 1
    for (int c = 0; c < kCh; ++c) {
      float sv[32];
      scores(c, sv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 nn = lds_v4(s_scs + 256 + 128 * c + 16 * q);
        const float4 ee = lds_v4(s_scs + 768 + 128 * c + 16 * q);
        const int j = 4 * q;
        const float2 u01 = fadd2(make_float2(sv[j], sv[j + 1]),
                                 ffma2(make_float2(a, a), make_float2(nn.x, nn.y), make_float2(ee.x, ee.y)));
        const float2 u23 = fadd2(make_float2(sv[j + 2], sv[j + 3]),
                                 ffma2(make_float2(a, a), make_float2(nn.z, nn.w), make_float2(ee.z, ee.w)));
        u4[q & 1] = fmin3(u4[q & 1], u01.x, u01.y);
        u4[2 + (q & 1)] = fmin3(u4[2 + (q & 1)], u23.x, u23.y);
      }
    }
    const float U = fminf(fminf(u4[0], u4[1]), fminf(u4[2], u4[3])) + 1e-30f;
    const size_t rec = ((size_t)g * M + row) * nchunk + tc.n_blk * kEpiParts + part;
    const int col0 = tc.n_blk * BN + cb;
    const int nvalid = K - col0;   // columns j >= nvalid are padding
    // pass 2: L = s - D = s + (-a ||c|| - eps ||c||^2), candidates in code order
    int cnt = 0;
    float l4[2] = {INFINITY, INFINITY};
#pragma unroll 1
    for (int c = 0; c < kCh; ++c) {
      float sv[32];
      scores(c, sv);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 nn = lds_v4(s_scs + 256 + 128 * c + 16 * q);
        const float4 ne = lds_v4(s_scs + 512 + 128 * c + 16 * q);
        const int j = 4 * q;
        const float2 l01 = fadd2(make_float2(sv[j], sv[j + 1]),
                                 ffma2(make_float2(-a, -a), make_float2(nn.x, nn.y), make_float2(ne.x, ne.y)));
        const float2 l23 = fadd2(make_float2(sv[j + 2], sv[j + 3]),
                                 ffma2(make_float2(-a, -a), make_float2(nn.z, nn.w), make_float2(ne.z, ne.w)));
        l4[0] = fmin3(l4[0], l01.x, l01.y);
        l4[1] = fmin3(l4[1], l23.x, l23.y);
        const float lo[4] = {l01.x, l01.y, l23.x, l23.y};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int jj = 32 * c + j + t;
          if (lo[t] <= U && jj < nvalid) {
            if (ok && cnt < kVqCap) {
              w.rec_idx[rec * kVqCap + cnt] = col0 + jj;
              w.rec_score[rec * kVqCap + cnt] = lo[t];
            }
            ++cnt;
          }
        }
      }
    }
    if (ok) {
      w.rec_best[rec] = U;
      w.rec_lmin[rec] = fminf(l4[0], l4[1]);
      w.rec_cnt[rec] = cnt;
    }
  }
};

// Grouped codebooks (G > 1): the GEMM runs in "runs" (TileSched::runs) — a CTA pair takes a
// 128-row block of one group and sweeps every code tile of it — and this epilogue keeps each
// (row, column part)'s window state in registers across the sweep, then merges the four parts
// of the row through shared memory and DECIDES the row: one surviving candidate is written as
// the index; several go to the fp64 re-rank list.  No per-chunk records, no finalize pass
// (G = 16 at ViT-L: 16 records x 40 B per token-group were 190 MB of HBM traffic per layer).
constexpr int kRunCap = 4;
struct VqRunState {
  float a, dmax2;   // the row's window slope (2 tau + 2 eps) ||x_g|| and 2 Dmax (run constants)
  float U;       // min (s_k + D_k) over the codes examined in detail (only decreases)
  float smin;    // min score s_k over every code swept so far
  float ovl;     // smallest lower bound of a candidate dropped for want of a slot (+inf: none)
  int n;         // live candidate slots (kept in the warp's stage smem, [slot][lane])
};

// r[j] for a run-time j in [0, 32): a 5-level select tree (keeps r in registers)
__device__ __forceinline__ float pick32(const uint32_t (&r)[32], int j) {
  float t16[16], t8[8], t4[4], t2[2];
#pragma unroll
  for (int i = 0; i < 16; ++i) t16[i] = __uint_as_float((j & 1) ? r[2 * i + 1] : r[2 * i]);
#pragma unroll
  for (int i = 0; i < 8; ++i) t8[i] = (j & 2) ? t16[2 * i + 1] : t16[2 * i];
#pragma unroll
  for (int i = 0; i < 4; ++i) t4[i] = (j & 4) ? t8[2 * i + 1] : t8[2 * i];
#pragma unroll
  for (int i = 0; i < 2; ++i) t2[i] = (j & 8) ? t4[2 * i + 1] : t4[2 * i];
  return (j & 16) ? t2[1] : t2[0];
}

// Stage layout of one epilogue warp (kEpiStageBytes): [0, 1024) the window terms of the tile
// part's (up to) 64 codes (float4 per code, broadcast reads), staged by pre() while the MMAs
// run; [1024, 1536) candidate codes [kRunCap][32 lanes]; [1536, 2048) their lower bounds.  The
// end-of-run merge reuses [0, 1536) as [lane][12] words.
//
// Filter (exact superset of the window test).  With D_k = a n_k + e_k <= Dmax (the group's max
// code norm) and U' = min (s_k + D_k) over the codes examined in detail, a code with
// s_k > smin + 2 Dmax has L_k = s_k - D_k > smin + Dmax >= (s + D) of the code holding smin
// >= U' — never a candidate.  So the common path per score is one FFMA (s = ||c||^2 - 2 x.c)
// and one FMNMX; only a 32-code chunk holding a score <= smin + 2 Dmax (a new running minimum
// or a near tie; ~2-3 of a part's chunks per row) takes the per-code bounds.
template <int BN>
struct VqRunEpilogue {
  static constexpr bool kStateful = true;
  using State = VqRunState;
  int M, K;
  const float4* c_win;      // [G, K] {||c||^2, ||c||, eps ||c||^2, 0}
  const float* c_norm_max;  // [G] max ||c|| (rounded up)
  VqWorkspace w;
  int32_t* idx_out;         // [Mtok, G]
  int32_t* stats;           // nullable: stats[2] += window candidates
  int G;
  const int32_t* row_tok;   // nullable: GEMM row -> token (pre-split stack rows); else identity
  int Mtok;

  // Before the tile's accumulator is ready: the window terms of this part's codes into smem
  // and, on a run's first tile, the row's window constants.
  __device__ __forceinline__ void pre(const TileCoord& tc, int row_in_tile, int cb, int ce,
                                      int part, uint8_t* stage, State& st, bool first) const {
    const int lane = threadIdx.x & 31;
    const int g = tc.batch;
    const int col0 = tc.n_blk * BN + cb + lane;
    const float4* cw = c_win + (size_t)g * K;
    const float4 c0 = col0 < K ? __ldg(cw + col0) : make_float4(INFINITY, 0.f, 0.f, 0.f);
    const float4 c1 = (cb + 32 < ce && col0 + 32 < K) ? __ldg(cw + col0 + 32)
                                                      : make_float4(INFINITY, 0.f, 0.f, 0.f);
    if (first) {
      const int row = tc.m_blk * kBM + row_in_tile;
      const float xn = row < M ? w.x_norm[(size_t)g * M + row] : 0.f;
      st.a = window_a(xn);
      const float nmax = __ldg(c_norm_max + g);
      st.dmax2 = 2.0f * (nmax * (st.a + kEps * nmax)) * (1.0f + 1e-6f);
    }
    const uint32_t s_scs = smem_u32(stage);
    __syncwarp();   // the previous tile's reads of the staged terms are done
    // SoA: [0, 256) ||c||^2, [256, 512) ||c||, [512, 768) eps ||c||^2 of the part's <= 64 codes
    // (the common path reads four ||c||^2 per 16-byte load)
    sts_f32(s_scs + 4 * lane, c0.x);
    sts_f32(s_scs + 256 + 4 * lane, c0.y);
    sts_f32(s_scs + 512 + 4 * lane, c0.z);
    sts_f32(s_scs + 128 + 4 * lane, c1.x);
    sts_f32(s_scs + 384 + 4 * lane, c1.y);
    sts_f32(s_scs + 640 + 4 * lane, c1.z);
    __syncwarp();
  }

  __device__ __forceinline__ void operator()(const TileCoord& tc, int row_in_tile, uint32_t taddr,
                                             int cb, int ce, int part, uint8_t* stage, State& st,
                                             bool first, bool last) const {
    const int row = tc.m_blk * kBM + row_in_tile;
    const bool ok = row < M;
    const int g = tc.batch;
    const int col_base = tc.n_blk * BN;
    const int lane = threadIdx.x & 31;
    const uint32_t s_stage = smem_u32(stage), s_idx = s_stage + 1024 + 4 * lane,
                   s_lo = s_stage + 1536 + 4 * lane;
    const float a = st.a, dmax2 = st.dmax2;
    if (first) {
      st.U = INFINITY;
      st.smin = INFINITY;
      st.ovl = INFINITY;
      st.n = 0;
    }
#pragma unroll 1
    for (int c0 = cb; c0 < ce; c0 += 32) {
      const int col0 = col_base + c0;
      const uint32_t s_cn = s_stage + (c0 - cb) * 4;   // this chunk's 32 staged ||c||^2
      uint32_t r[32];
      tmem_ld32(taddr + c0, r);
      float cn[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {   // (shared-memory loads overlap the TMEM load)
        const float4 v = lds_v4(s_cn + 16 * q);
        cn[4 * q] = v.x;
        cn[4 * q + 1] = v.y;
        cn[4 * q + 2] = v.z;
        cn[4 * q + 3] = v.w;
      }
      tmem_ld_wait();
      // r[j] <- s_j = ||c_j||^2 - 2 x.c_j (the same single-rounding FMA per lane of FFMA2)
      float m4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 sc = ffma2(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])),
                                make_float2(-2.0f, -2.0f), make_float2(cn[j], cn[j + 1]));
        r[j] = __float_as_uint(sc.x);
        r[j + 1] = __float_as_uint(sc.y);
        m4[(j >> 1) & 3] = fmin3(m4[(j >> 1) & 3], sc.x, sc.y);
      }
      const float cmin = fminf(fminf(m4[0], m4[1]), fminf(m4[2], m4[3]));
      st.smin = fminf(st.smin, cmin);
      // + a rounding margin of 2^-21 (|smin| + 2 Dmax): the comparisons stay exact supersets
      const float thr = (st.smin + dmax2) + kEps * (fabsf(st.smin) + dmax2);
      if (cmin > thr) continue;   // common case: nothing in this chunk can compete
      // bit j = (s_j <= thr) = sign of s_j - thr' (thr' the next float above thr; the difference
      // of finite floats is exact in sign, +inf scores give +inf), packed pairwise and shifted
      // in with one funnel shift per code
      const float2 nthr = make_float2(-nextafterf(thr, INFINITY), -nextafterf(thr, INFINITY));
      uint32_t m = 0;
#pragma unroll
      for (int j = 30; j >= 0; j -= 2) {
        const float2 dd = fadd2(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])), nthr);
        m = __funnelshift_l(__float_as_uint(dd.y), m, 1);
        m = __funnelshift_l(__float_as_uint(dd.x), m, 1);
      }
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const float sc = pick32(r, j);
        const uint32_t o = (uint32_t)(c0 - cb + j) * 4;
        const float d = fmaf(a, lds_f32(s_stage + 256 + o), lds_f32(s_stage + 512 + o));
        const float up = sc + d + 1e-30f, lo = sc - d;
        if (up < st.U) {   // tighter bound: prune the kept codes
          st.U = up;
          int k = 0;
          for (int i = 0; i < st.n; ++i) {
            const float li = lds_f32(s_lo + 128 * i);
            if (li <= up) {
              sts_f32(s_lo + 128 * k, li);
              sts_s32(s_idx + 128 * k, lds_s32(s_idx + 128 * i));
              ++k;
            }
          }
          st.n = k;
        }
        if (lo <= st.U) {
          if (st.n < kRunCap) {
            sts_s32(s_idx + 128 * st.n, col0 + j);
            sts_f32(s_lo + 128 * st.n, lo);
            ++st.n;
          } else {
            st.ovl = fminf(st.ovl, lo);
          }
        }
      }
    }
    if (!last) return;
    // ---- end of the run: merge the row's kEpiParts column parts (warps quarter + 4 p)
    int ci[kRunCap];
    float cl[kRunCap];
#pragma unroll
    for (int i = 0; i < kRunCap; ++i) {
      ci[i] = i < st.n ? lds_s32(s_idx + 128 * i) : 0;
      cl[i] = i < st.n ? lds_f32(s_lo + 128 * i) : INFINITY;
    }
    float* sh = reinterpret_cast<float*>(stage);          // [lane][12] words, this warp's part
    float* my = sh + lane * 12;
    __syncwarp();
    my[0] = st.U;
    my[1] = st.ovl;
    reinterpret_cast<int*>(my)[2] = st.n;
#pragma unroll
    for (int i = 0; i < kRunCap; ++i) {
      reinterpret_cast<int*>(my)[4 + i] = ci[i];
      my[8 + i] = cl[i];
    }
    const int quarter = row_in_tile >> 5;
    asm volatile("bar.sync %0, %1;" ::"r"(1 + quarter), "r"(32 * kEpiParts) : "memory");
    const int tok = !ok ? -1 : row_tok ? __ldg(row_tok + row) : row;
    if (part == 0 && tok >= 0) {
      // stage areas of the warps of this quarter are kEpiStageBytes * 4 apart (warp + 4 p)
      float U = INFINITY;
#pragma unroll
      for (int p = 0; p < kEpiParts; ++p) U = fminf(U, (sh + p * 4 * (kEpiStageBytes / 4))[lane * 12]);
      int n = 0, only = 0x7FFFFFFF, ovf = 0, list[8];
#pragma unroll
      for (int p = 0; p < kEpiParts; ++p) {
        const float* o = sh + p * 4 * (kEpiStageBytes / 4) + lane * 12;
        if (o[1] <= U) ovf = 1;                 // a dropped code is still a candidate
        const int pn = reinterpret_cast<const int*>(o)[2];
#pragma unroll
        for (int i = 0; i < kRunCap; ++i)
          if (i < pn && o[8 + i] <= U) {
            const int k = reinterpret_cast<const int*>(o)[4 + i];
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (q == n) list[q] = k;
            ++n;
            only = min(only, k);
          }
      }
      if (stats) atomicAdd(&stats[2], n);
      if (n == 1 && !ovf) {
        idx_out[(size_t)tok * G + g] = only;
      } else {
        const bool direct = !ovf && n >= 1 && n <= 8;
        // exact scan of every code: split over the re-rank kernel's warps (ov list) while it
        // has room, else one warp scans the whole group (-2 entry)
        const int os = direct ? kOvCap : atomicAdd(w.ov_count, 1);
        if (os < kOvCap) {
          w.ov_list[os] = g * Mtok + tok;
          w.ov_done[os] = 0;
        } else {
          const int slot = atomicAdd(w.rr_count, 1);
          int* ent = w.rr_list + (size_t)slot * kRREntry;
          ent[0] = g * Mtok + tok;
          if (direct) {
            ent[1] = n;
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (i < n) ent[2 + i] = list[i];
          } else {
            ent[1] = -2;                        // full fp64 scan of the group's codes
          }
        }
      }
    }
    asm volatile("bar.sync %0, %1;" ::"r"(1 + quarter), "r"(32 * kEpiParts) : "memory");
  }
};

// ---------------------------------------------------------- finalize
__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum_e a[e] b[e] over this lane's elements e = lane, lane + 32, ... in fp64 (the warp sum of
// it is the dot product); loads batched 8 per lane so a 768-wide row costs 3 round trips, not 24
__device__ __forceinline__ double lane_dot64(const float* a, const float* b, int gd, int lane) {
  double acc = 0.0;
  for (int base = 0; base < gd; base += 256) {
    float av[8], bv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = base + lane + 32 * i;
      av[i] = e < gd ? __ldg(a + e) : 0.0f;
      bv[i] = e < gd ? __ldg(b + e) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (base + lane + 32 * i < gd) acc = fma((double)av[i], (double)bv[i], acc);
  }
  return acc;
}

// exact reference distance (vq.py:130 evaluation order): (pp - 2 pc) + cc, fp64
__device__ __forceinline__ double exact_d2(const float* xr, const float* c, int gd, double pp,
                                           double cc, int lane) {
  const double pc = warp_sum_d(lane_dot64(xr, c, gd, lane));
  return (pp - 2.0 * pc) + cc;
}

// Decide one (g, token) item from its chunk records (one warp; lane c reads record c): a single
// window survivor is the answer.  Several go to the fp64 re-rank — inline (inline_rr: the warp
// scores the <= kRRCands candidates itself with the reference expression, vq.py:130) or as an
// entry of the re-rank list; an overflowed record list always goes to the list.
__device__ __forceinline__ void vq_decide(const AstraCodebook& cb, const float* __restrict__ x,
                                          int ldx, int src_row, int tok, int g, int Mtok,
                                          size_t rec0, int nchunk, const VqWorkspace& w,
                                          int32_t* __restrict__ idx_out, int32_t* __restrict__ stats,
                                          bool inline_rr, int lane) {
  const int G = cb.groups;
  const int item = g * Mtok + tok, row = tok;
  // one round of independent loads: lane c holds chunk record c (nchunk <= 32 for K <= 2048;
  // larger codebooks loop)
  // U = min over chunks of U_chunk bounds the true best score from above; a chunk matters if
  // its min lower bound reaches U, a candidate if its own lower bound L_k does
  float best = INFINITY;
  int n = 0, only = 0x7FFFFFFF;
  int overflow = 0;
  uint32_t live = 0;
  int ix[kVqCap];
  if (nchunk <= 32) {
    float rb = INFINITY, rl = INFINITY, sc[kVqCap];
    int rc = 0;
    if (lane < nchunk) {
      rb = w.rec_best[rec0 + lane];
      rl = w.rec_lmin[rec0 + lane];
      rc = w.rec_cnt[rec0 + lane];
#pragma unroll
      for (int i = 0; i < kVqCap; ++i) {
        sc[i] = w.rec_score[(rec0 + lane) * kVqCap + i];
        ix[i] = w.rec_idx[(rec0 + lane) * kVqCap + i];
      }
    }
    best = rb;
    for (int o = 16; o; o >>= 1) best = fminf(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane < nchunk && rl <= best) {
      if (rc > kVqCap) overflow = 1;
#pragma unroll
      for (int i = 0; i < kVqCap; ++i)
        if (i < rc && sc[i] <= best) {
          ++n;
          only = min(only, ix[i]);
          live |= 1u << i;
        }
    }
  } else {
    // wide codebooks (> 32 records per row): a single surviving candidate still decides here;
    // several go to the re-rank kernel, which scans the records (no compacted list)
    for (int c = lane; c < nchunk; c += 32) best = fminf(best, w.rec_best[rec0 + c]);
    for (int o = 16; o; o >>= 1) best = fminf(best, __shfl_xor_sync(0xffffffffu, best, o));
    for (int c = lane; c < nchunk; c += 32) {
      if (w.rec_lmin[rec0 + c] > best) continue;
      const int cnt = w.rec_cnt[rec0 + c];
      if (cnt > kVqCap) overflow = 1;
      const int m = cnt < kVqCap ? cnt : kVqCap;
      for (int i = 0; i < m; ++i)
        if (w.rec_score[(rec0 + c) * kVqCap + i] <= best) {
          ++n;
          only = min(only, w.rec_idx[(rec0 + c) * kVqCap + i]);
        }
    }
  }
  for (int o = 16; o; o >>= 1) {
    n += __shfl_xor_sync(0xffffffffu, n, o);
    only = min(only, __shfl_xor_sync(0xffffffffu, only, o));
    overflow |= __shfl_xor_sync(0xffffffffu, overflow, o);
  }
  const bool wide = nchunk > 32;   // no per-lane candidate slots (ix / live) were filled
  if (inline_rr && !wide && !overflow && n > 1 && n <= kRRCands) {
    // several window candidates: the warp re-ranks them now, exact fp64 with the reference's
    // expression (||p||^2 - 2 p.c) + ||c||^2, ties to the lowest index
    const int gd = cb.group_dim, K = cb.size;
    const float* xr = x + (size_t)src_row * ldx + (size_t)g * gd;
    const float* cents = cb.centroids + (size_t)g * K * gd;
    const double pp = warp_sum_d(lane_dot64(xr, xr, gd, lane));
    double bd = INFINITY;
    int bi = 0x7FFFFFFF;
#pragma unroll
    for (int i = 0; i < kVqCap; ++i) {
      uint32_t m = __ballot_sync(0xffffffffu, (live >> i) & 1u);
      while (m) {
        const int srcl = __ffs(m) - 1;
        m &= m - 1;
        const int k = __shfl_sync(0xffffffffu, ix[i], srcl);
        const double d = exact_d2(xr, cents + (size_t)k * gd, gd, pp, cb.c_sq64[(size_t)g * K + k], lane);
        if (d < bd || (d == bd && k < bi)) {
          bd = d;
          bi = k;
        }
      }
    }
    if (lane == 0) {
      idx_out[(size_t)row * G + g] = bi;
      if (stats) atomicAdd(&stats[0], 1);
    }
  } else if (overflow || n > 1) {
    // several window candidates: exact fp64 re-rank by vq_rerank_kernel, handed the compacted
    // candidate list (codes in increasing order) when it fits
    int slot = 0;
    if (lane == 0) slot = atomicAdd(w.rr_count, 1);
    slot = __shfl_sync(0xffffffffu, slot, 0);
    int* ent = w.rr_list + (size_t)slot * kRREntry;
    const bool direct = !wide && !overflow && n <= kRRCands;
    if (direct) {
      const int cnt = __popc(live);
      int pre = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += t;
      }
      pre -= cnt;
#pragma unroll
      for (int i = 0; i < kVqCap; ++i)
        if ((live >> i) & 1u) ent[2 + pre++] = ix[i];
    }
    if (lane == 0) {
      ent[0] = item;
      ent[1] = direct ? n : -1;
    }
  } else if (lane == 0) {
    idx_out[(size_t)row * G + g] = only;
  }
  if (lane == 0 && stats) atomicAdd(&stats[2], n);
}

__global__ void vq_finalize_kernel(AstraCodebook cb, const float* __restrict__ x, int M, int ldx,
                                   const int32_t* __restrict__ rows, VqWorkspace w, int nchunk,
                                   int32_t* __restrict__ idx_out, int32_t* __restrict__ stats,
                                   int Mrec, int rec_by_row) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int item = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int G = cb.groups;
  if (item >= G * M) return;
  const int g = item / M, row = item % M;
  // records are indexed by token (gathered split) or by source row (pre-split stack)
  const int rr = rec_by_row ? rows[row] : row;
  const size_t rec0 = ((size_t)g * Mrec + rr) * nchunk;
  // (re-ranking the multi-candidate rows in place measured slower: 27.7 vs 7.4 + 10.2 us — the
  // re-rank kernel's batched loads beat the per-row warps' dependent round trips)
  vq_decide(cb, x, ldx, rows ? rows[row] : row, row, g, M, rec0, nchunk, w, idx_out, stats, false,
            lane);
}

// vq_finalize for <= 16 records per row (K <= 1024 at BN = 256): two rows per warp, a
// half-warp per row, so every lane carries a record and the grid is one resident wave at
// ViT-B (the per-row work is one round trip of record loads; a full warp per row left half
// the lanes idle and needed 1.3 waves).  Same decisions as vq_decide without inline re-rank:
// one surviving candidate is the index, several (or an overflowed part) go to the re-rank
// list, the candidate codes compacted in code order when they fit.
__global__ void vq_finalize_half_kernel(AstraCodebook cb, int M, const int32_t* __restrict__ rows,
                                        VqWorkspace w, int nchunk, int32_t* __restrict__ idx_out,
                                        int32_t* __restrict__ stats, int Mrec, int rec_by_row) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31, hl = lane & 15, lead = lane & 16;
  const int G = cb.groups;
  const int item = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 2 + (lane >> 4);
  const bool on = item < G * M;
  const int g = on ? item / M : 0, row = on ? item - g * M : 0;
  const bool has = on && hl < nchunk;
  float rb = INFINITY, rl = INFINITY, sc[kVqCap];
  int rc = 0, ix[kVqCap];
  if (has) {
    const int rr = rec_by_row ? rows[row] : row;
    const size_t rec = ((size_t)g * Mrec + rr) * nchunk + hl;
    rb = w.rec_best[rec];
    rl = w.rec_lmin[rec];
    rc = w.rec_cnt[rec];
#pragma unroll
    for (int i = 0; i < kVqCap; ++i) {
      sc[i] = w.rec_score[rec * kVqCap + i];
      ix[i] = w.rec_idx[rec * kVqCap + i];
    }
  }
  float best = rb;
#pragma unroll
  for (int o = 8; o; o >>= 1) best = fminf(best, __shfl_xor_sync(0xffffffffu, best, o));
  int n = 0, only = 0x7FFFFFFF, overflow = 0;
  uint32_t live = 0;
  if (has && rl <= best) {
    overflow = rc > kVqCap;
#pragma unroll
    for (int i = 0; i < kVqCap; ++i)
      if (i < rc && sc[i] <= best) {
        ++n;
        only = min(only, ix[i]);
        live |= 1u << i;
      }
  }
  int pre = __popc(live);
  const int mine = pre;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, pre, o, 16);
    if (hl >= o) pre += t;
  }
  pre -= mine;
#pragma unroll
  for (int o = 8; o; o >>= 1) {
    n += __shfl_xor_sync(0xffffffffu, n, o);
    only = min(only, __shfl_xor_sync(0xffffffffu, only, o));
    overflow |= __shfl_xor_sync(0xffffffffu, overflow, o);
  }
  const bool rr = on && (overflow || n > 1);
  int slot = 0;
  if (rr && hl == 0) slot = atomicAdd(w.rr_count, 1);
  slot = __shfl_sync(0xffffffffu, slot, lead);
  if (rr) {
    int* ent = w.rr_list + (size_t)slot * kRREntry;
    const bool direct = !overflow && n <= kRRCands;
    if (direct) {
#pragma unroll
      for (int i = 0; i < kVqCap; ++i)
        if ((live >> i) & 1u) ent[2 + pre++] = ix[i];
    }
    if (hl == 0) {
      ent[0] = item;
      ent[1] = direct ? n : -1;
    }
  } else if (on && hl == 0) {
    idx_out[(size_t)row * G + g] = only;
  }
  if (on && hl == 0 && stats) atomicAdd(&stats[2], n);
}

// Exact fp64 re-rank of the listed items (one warp per item, grid-stride over the list): the
// window's candidate codes are compacted into a per-warp list and each is scored with the
// reference expression (||p||^2 - 2 p.c) + ||c||^2 (vq.py:130), ties to the lowest index.
// For group widths <= 1024 each lane loads its slice of the token and of a candidate row in
// one batch of independent loads (one memory round trip per candidate, not one per 32
// elements); a chunk whose candidate list overflowed contributes all of its 64 codes.
// Grid (blocks per SM): the generic variant's 239 registers fit one 256-thread block per SM,
// and its G = 1 lists are short (~560 items per ViT-B layer, one per warp), so the grid is the
// co-resident blocks (4 per SM spent ~1 us retiring empty blocks one at a time: 4.4 -> 3.3 us).
// The narrow variant serves the long grouped-codebook lists, where queued blocks balance the
// statically strided items better (G = 32 with 2 per SM: 430 -> 483 us).
constexpr int kRerankBlocks = 1, kRerankBlocksNarrow = 8;
template <bool kNarrow>
__global__ void __launch_bounds__(256) vq_rerank_kernel(AstraCodebook cb, const float* __restrict__ x,
                                                        int M, int ldx,
                                                        const int32_t* __restrict__ rows,
                                                        VqWorkspace w, int nchunk,
                                                        int32_t* __restrict__ idx_out,
                                                        int32_t* __restrict__ stats, int Mrec,
                                                        int rec_by_row, int part_codes) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) int s_cand[8][32 * kVqCap];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int G = cb.groups, K = cb.size, gd = cb.group_dim;
  const int total = *w.rr_count;
  for (int li = blockIdx.x * 8 + wib; li < total; li += gridDim.x * 8) {
    const int* ent = w.rr_list + (size_t)li * kRREntry;
    const int ev = __ldg(ent + min(lane, kRREntry - 1));   // whole entry in one round trip
    const int item = __shfl_sync(0xffffffffu, ev, 0);
    const int nd = __shfl_sync(0xffffffffu, ev, 1);
    const int g = item / M, row = item % M;
    if (kNarrow && nd > 0) {
      // narrow groups: lane q holds float4 q of the token slice; the slice and every candidate
      // row load in one round trip, then one fp64 dot product per candidate
      const int src = rows ? rows[row] : row;
      const float4* xr = reinterpret_cast<const float4*>(x + (size_t)src * ldx + (size_t)g * gd);
      const float4* cents = reinterpret_cast<const float4*>(cb.centroids + (size_t)g * K * gd);
      const bool on = lane < (gd >> 2);
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 xv = on ? __ldg(xr + lane) : z;
      int kk[kRRCands];
      float4 cv[kRRCands];
#pragma unroll
      for (int i = 0; i < kRRCands; ++i) {
        kk[i] = __shfl_sync(0xffffffffu, ev, 2 + min(i, nd - 1));
        cv[i] = (on && i < nd) ? __ldg(cents + (size_t)kk[i] * (gd >> 2) + lane) : z;
      }
      double pp = fma((double)xv.x, (double)xv.x, fma((double)xv.y, (double)xv.y,
                  fma((double)xv.z, (double)xv.z, (double)xv.w * (double)xv.w)));
      pp = warp_sum_d(pp);
      double bd = INFINITY;
      int bi = -1;
#pragma unroll
      for (int i = 0; i < kRRCands; ++i) {
        if (i >= nd) break;
        double pc = fma((double)xv.x, (double)cv[i].x, fma((double)xv.y, (double)cv[i].y,
                    fma((double)xv.z, (double)cv[i].z, (double)xv.w * (double)cv[i].w)));
        const double d = (pp - 2.0 * warp_sum_d(pc)) + cb.c_sq64[(size_t)g * K + kk[i]];
        if (d < bd || (d == bd && kk[i] < bi)) {
          bd = d;
          bi = kk[i];
        }
      }
      if (lane == 0) {
        idx_out[(size_t)row * G + g] = bi;
        if (stats) atomicAdd(&stats[0], 1);
      }
      continue;
    }
    if (!kNarrow && nd > 0 && cb.group_dim <= 1024) {
      // direct: token slice and two candidate rows per round trip, fp64 dot products
      const int src = rows ? rows[row] : row;
      const float* xr = x + (size_t)src * ldx + (size_t)g * gd;
      const float* cents = cb.centroids + (size_t)g * K * gd;
      // the token slice and the first candidate pair load in the same round trip
      float xs[32], c0[32], c1[32];
      int k0 = __shfl_sync(0xffffffffu, ev, 2);
      int k1 = nd > 1 ? __shfl_sync(0xffffffffu, ev, 3) : k0;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int e = lane + 32 * i;
        xs[i] = e < gd ? __ldg(xr + e) : 0.0f;
        c0[i] = e < gd ? __ldg(cents + (size_t)k0 * gd + e) : 0.0f;
        c1[i] = e < gd ? __ldg(cents + (size_t)k1 * gd + e) : 0.0f;
      }
      double pp = 0.0;
#pragma unroll
      for (int i = 0; i < 32; ++i) pp = fma((double)xs[i], (double)xs[i], pp);
      pp = warp_sum_d(pp);
      double bd = INFINITY;
      int bi = -1;
      for (int q = 0; q < nd; q += 2) {
        if (q > 0) {
          k0 = __shfl_sync(0xffffffffu, ev, 2 + q);
          k1 = q + 1 < nd ? __shfl_sync(0xffffffffu, ev, 3 + q) : k0;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int e = lane + 32 * i;
            c0[i] = e < gd ? __ldg(cents + (size_t)k0 * gd + e) : 0.0f;
            c1[i] = e < gd ? __ldg(cents + (size_t)k1 * gd + e) : 0.0f;
          }
        }
        const double cc0 = cb.c_sq64[(size_t)g * K + k0], cc1 = cb.c_sq64[(size_t)g * K + k1];
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          d0 = fma((double)xs[i], (double)c0[i], d0);
          d1 = fma((double)xs[i], (double)c1[i], d1);
        }
        d0 = (pp - 2.0 * warp_sum_d(d0)) + cc0;
        d1 = (pp - 2.0 * warp_sum_d(d1)) + cc1;
        if (d0 < bd || (d0 == bd && k0 < bi)) {
          bd = d0;
          bi = k0;
        }
        if (d1 < bd || (d1 == bd && k1 < bi)) {
          bd = d1;
          bi = k1;
        }
      }
      if (lane == 0) {
        idx_out[(size_t)row * G + g] = bi;
        if (stats) atomicAdd(&stats[0], 1);
      }
      continue;
    }
    if (nd == -2) {
      // run-mode overflow (grouped codebooks): exact fp64 scan of every code of the group, the
      // lanes over the codes (lane k scores codes k, k + 32, ...; token slice broadcast from
      // shared memory), then a lowest-index argmin across the warp
      const int src = rows ? rows[row] : row;
      const float* xr = x + (size_t)src * ldx + (size_t)g * gd;
      const float* cents = cb.centroids + (size_t)g * K * gd;
      double pp = 0.0;
      for (int e = lane; e < gd; e += 32) pp = fma((double)__ldg(xr + e), (double)__ldg(xr + e), pp);
      pp = warp_sum_d(pp);
      double bd = INFINITY;
      int bi = 0x7FFFFFFF;
      if (gd <= 32 * kVqCap && gd % 4 == 0) {
        // narrow groups, 16-byte rows: lane k scores codes k, k + 32, ... with float4 loads of
        // the code row (4 in flight per code, two codes per step) against the token slice
        // broadcast from shared memory
        float* xsh = reinterpret_cast<float*>(s_cand[wib]);
        for (int e = lane; e < gd; e += 32) xsh[e] = __ldg(xr + e);
        __syncwarp();
        const int q4 = gd >> 2;
        const float4* c4 = reinterpret_cast<const float4*>(cents);
        const float4* x4 = reinterpret_cast<const float4*>(xsh);
        for (int k = lane; k < K; k += 64) {
          const int k2 = min(k + 32, K - 1);
          const float4* ca = c4 + (size_t)k * q4;
          const float4* cb2 = c4 + (size_t)k2 * q4;
          double pa = 0.0, pb = 0.0;
          for (int q = 0; q < q4; q += 4) {
            float4 va[4], vb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              va[i] = q + i < q4 ? __ldg(ca + q + i) : make_float4(0.f, 0.f, 0.f, 0.f);
              vb[i] = q + i < q4 ? __ldg(cb2 + q + i) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (q + i >= q4) break;
              const float4 xv = x4[q + i];
              pa = fma((double)xv.x, (double)va[i].x, pa);
              pa = fma((double)xv.y, (double)va[i].y, pa);
              pa = fma((double)xv.z, (double)va[i].z, pa);
              pa = fma((double)xv.w, (double)va[i].w, pa);
              pb = fma((double)xv.x, (double)vb[i].x, pb);
              pb = fma((double)xv.y, (double)vb[i].y, pb);
              pb = fma((double)xv.z, (double)vb[i].z, pb);
              pb = fma((double)xv.w, (double)vb[i].w, pb);
            }
          }
          const double d = (pp - 2.0 * pa) + cb.c_sq64[(size_t)g * K + k];
          if (d < bd) {   // ascending k per lane: strict < keeps the lowest index
            bd = d;
            bi = k;
          }
          const double d2 = (pp - 2.0 * pb) + cb.c_sq64[(size_t)g * K + k2];
          if (k + 32 < K && d2 < bd) {
            bd = d2;
            bi = k2;
          }
        }
        __syncwarp();
        for (int o = 16; o; o >>= 1) {
          const double od = __shfl_xor_sync(0xffffffffu, bd, o);
          const int ok_ = __shfl_xor_sync(0xffffffffu, bi, o);
          if (od < bd || (od == bd && ok_ < bi)) {
            bd = od;
            bi = ok_;
          }
        }
      } else if (gd <= 32 * kVqCap) {
        float* xsh = reinterpret_cast<float*>(s_cand[wib]);
        for (int e = lane; e < gd; e += 32) xsh[e] = __ldg(xr + e);
        __syncwarp();
        for (int k = lane; k < K; k += 64) {   // codes k and k + 32 (independent chains)
          const int k2 = min(k + 32, K - 1);
          const float* c = cents + (size_t)k * gd;
          const float* c2 = cents + (size_t)k2 * gd;
          double pc = 0.0, pc2 = 0.0;
          for (int e = 0; e < gd; ++e) {
            const double xe = (double)xsh[e];
            pc = fma(xe, (double)__ldg(c + e), pc);
            pc2 = fma(xe, (double)__ldg(c2 + e), pc2);
          }
          const double d = (pp - 2.0 * pc) + cb.c_sq64[(size_t)g * K + k];
          if (d < bd) {   // ascending k per lane: strict < keeps the lowest index
            bd = d;
            bi = k;
          }
          const double d2 = (pp - 2.0 * pc2) + cb.c_sq64[(size_t)g * K + k2];
          if (k + 32 < K && d2 < bd) {
            bd = d2;
            bi = k2;
          }
        }
        __syncwarp();
        for (int o = 16; o; o >>= 1) {
          const double od = __shfl_xor_sync(0xffffffffu, bd, o);
          const int ok_ = __shfl_xor_sync(0xffffffffu, bi, o);
          if (od < bd || (od == bd && ok_ < bi)) {
            bd = od;
            bi = ok_;
          }
        }
      } else {
        for (int k = 0; k < K; ++k) {
          const double d = exact_d2(xr, cents + (size_t)k * gd, gd, pp, cb.c_sq64[(size_t)g * K + k], lane);
          if (d < bd) {
            bd = d;
            bi = k;
          }
        }
      }
      if (lane == 0) {
        idx_out[(size_t)row * G + g] = bi;
        if (stats) atomicAdd(&stats[1], 1);
      }
      continue;
    }
    if (kNarrow) continue;   // (run mode hands over direct lists and full scans only)
    const int rr = rec_by_row ? rows[row] : row;
    const size_t rec0 = ((size_t)g * Mrec + rr) * nchunk;
    float thr = INFINITY;   // U: min over the chunks' upper bounds
    for (int c = lane; c < nchunk; c += 32) thr = fminf(thr, w.rec_best[rec0 + c]);
    for (int o = 16; o; o >>= 1) thr = fminf(thr, __shfl_xor_sync(0xffffffffu, thr, o));
    const int src = rows ? rows[row] : row;
    const float* xr = x + (size_t)src * ldx + (size_t)g * gd;
    const float* cents = cb.centroids + (size_t)g * K * gd;
    const double* cc = cb.c_sq64 + (size_t)g * K;
    const bool vec = gd <= 1024;
    float xs[32];   // this lane's slice of the token (fp32 inputs, fp64 arithmetic)
    double pp = 0.0;
    if (vec) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int e = lane + 32 * i;
        xs[i] = e < gd ? __ldg(xr + e) : 0.0f;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) pp = fma((double)xs[i], (double)xs[i], pp);
    } else {
      for (int e = lane; e < gd; e += 32) pp = fma((double)__ldg(xr + e), (double)__ldg(xr + e), pp);
    }
    pp = warp_sum_d(pp);
    double bd = INFINITY;
    int bi = -1, overflowed = 0;
    auto score = [&](int k) {
      const float* c = cents + (size_t)k * gd;
      double pc = 0.0;
      if (vec) {
        float cv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int e = lane + 32 * i;
          cv[i] = e < gd ? __ldg(c + e) : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) pc = fma((double)xs[i], (double)cv[i], pc);
      } else {
        for (int e = lane; e < gd; e += 32) pc = fma((double)__ldg(xr + e), (double)__ldg(c + e), pc);
      }
      pc = warp_sum_d(pc);
      const double d = (pp - 2.0 * pc) + cc[k];
      if (d < bd || (d == bd && k < bi)) {
        bd = d;
        bi = k;
      }
    };
    // candidates of the window, chunk by chunk (lane c reads chunk c), compacted in order
    for (int c0 = 0; c0 < nchunk; c0 += 32) {
      const int c = c0 + lane;
      uint32_t live = 0;
      int ix[kVqCap];
      int full_part = 0;
      if (c < nchunk && w.rec_lmin[rec0 + c] <= thr) {
        const int m = w.rec_cnt[rec0 + c];
        if (m > kVqCap) {
          full_part = 1;
        } else {
#pragma unroll
          for (int i = 0; i < kVqCap; ++i)
            if (i < m && w.rec_score[(rec0 + c) * kVqCap + i] <= thr) {
              live |= 1u << i;
              ix[i] = w.rec_idx[(rec0 + c) * kVqCap + i];
            }
        }
      }
      const int cnt = __popc(live);
      int pre = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += t;
      }
      const int tot = __shfl_sync(0xffffffffu, pre, 31);
      pre -= cnt;
      int k_ = 0;
#pragma unroll
      for (int i = 0; i < kVqCap; ++i)
        if ((live >> i) & 1u) s_cand[wib][pre + k_++] = ix[i];
      __syncwarp();
      for (int q = 0; q < tot; ++q) score(s_cand[wib][q]);
      __syncwarp();
      // overflowed chunks: every code of the 64-code part (rare; exact in any order since
      // ties resolve to the lowest index)
      uint32_t fb = __ballot_sync(0xffffffffu, full_part);
      overflowed |= fb != 0;
      while (fb) {
        const int cc_ = c0 + __ffs(fb) - 1;
        fb &= fb - 1;
        const int k_lo = cc_ * part_codes;   // chunk c = codes [c * part, (c + 1) * part)
        const int k_hi = min(K, k_lo + part_codes);
        for (int k = k_lo; k < k_hi; ++k) score(k);
      }
    }
    if (lane == 0) {
      idx_out[(size_t)row * G + g] = bi;
      if (stats) atomicAdd(&stats[overflowed ? 1 : 0], 1);
    }
  }
  // Exact scans of the overflow list (run mode): unit u = (item u / kOvSub, code range
  // u % kOvSub), claimed by warps as they finish their entries.  Each range's fp64 argmin goes
  // to ov_d / ov_k; the warp completing an item's last range reduces them in range order
  // (lowest code on equal distance, as the reference's argmin).
  const int n_ov = min(w.ov_count[0], kOvCap);
  if (n_ov == 0) return;
  const int sc = (K + kOvSub - 1) / kOvSub;
  while (true) {
    int u = 0;
    if (lane == 0) u = atomicAdd(&w.ov_count[1], 1);
    u = __shfl_sync(0xffffffffu, u, 0);
    if (u >= n_ov * kOvSub) break;
    const int slot = u / kOvSub, sub = u % kOvSub;
    const int item = __ldcg(w.ov_list + slot);
    const int g = item / M, row = item % M;
    const int src = rows ? rows[row] : row;
    const float* xr = x + (size_t)src * ldx + (size_t)g * gd;
    const float* cents = cb.centroids + (size_t)g * K * gd;
    const double* cc = cb.c_sq64 + (size_t)g * K;
    const int k_lo = sub * sc, k_hi = min(K, k_lo + sc);
    double pp = 0.0;
    for (int e = lane; e < gd; e += 32) pp = fma((double)__ldg(xr + e), (double)__ldg(xr + e), pp);
    pp = warp_sum_d(pp);
    double bd = INFINITY;
    int bi = 0x7FFFFFFF;
    if (gd <= 32 * kVqCap && gd % 4 == 0) {
      // lanes over codes, token slice broadcast from shared memory, 16-byte code-row loads
      float* xsh = reinterpret_cast<float*>(s_cand[wib]);
      __syncwarp();
      for (int e = lane; e < gd; e += 32) xsh[e] = __ldg(xr + e);
      __syncwarp();
      const int q4 = gd >> 2;
      const float4* x4 = reinterpret_cast<const float4*>(xsh);
      for (int k = k_lo + lane; k < k_hi; k += 32) {
        const float4* c4 = reinterpret_cast<const float4*>(cents + (size_t)k * gd);
        double pc = 0.0;
        for (int q = 0; q < q4; q += 4) {
          float4 v[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) v[i] = q + i < q4 ? __ldg(c4 + q + i) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (q + i >= q4) break;
            const float4 xv = x4[q + i];
            pc = fma((double)xv.x, (double)v[i].x, pc);
            pc = fma((double)xv.y, (double)v[i].y, pc);
            pc = fma((double)xv.z, (double)v[i].z, pc);
            pc = fma((double)xv.w, (double)v[i].w, pc);
          }
        }
        const double d = (pp - 2.0 * pc) + cc[k];
        if (d < bd) {   // ascending k per lane
          bd = d;
          bi = k;
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, bd, o);
        const int ok_ = __shfl_xor_sync(0xffffffffu, bi, o);
        if (od < bd || (od == bd && ok_ < bi)) {
          bd = od;
          bi = ok_;
        }
      }
      __syncwarp();
    } else {
      for (int k = k_lo; k < k_hi; ++k) {   // lanes over the dimensions
        const double d = exact_d2(xr, cents + (size_t)k * gd, gd, pp, cc[k], lane);
        if (d < bd) {
          bd = d;
          bi = k;
        }
      }
    }
    int last = 0;
    if (lane == 0) {
      w.ov_d[u] = bd;
      w.ov_k[u] = bi;
      __threadfence();
      last = atomicAdd(w.ov_done + slot, 1) == kOvSub - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence();
      double d = INFINITY;
      int k = 0x7FFFFFFF;
      if (lane < kOvSub) {
        d = __ldcg(w.ov_d + (size_t)slot * kOvSub + lane);
        k = __ldcg(w.ov_k + (size_t)slot * kOvSub + lane);
      }
      for (int o = 16; o; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, d, o);
        const int ok_ = __shfl_xor_sync(0xffffffffu, k, o);
        if (od < d || (od == d && ok_ < k)) {
          d = od;
          k = ok_;
        }
      }
      if (lane == 0) {
        idx_out[(size_t)row * G + g] = k;
        if (stats) atomicAdd(&stats[1], 1);
      }
    }
  }
}

// ------------------------------------------------------------ decode
// out[m, g*gd + e] = centroids[g][idx[m, g]][e]; one warp per (m, g), float4 when aligned.
__global__ void vq_decode_kernel(AstraCodebook cb, const int32_t* __restrict__ idx, int M,
                                 float* __restrict__ out, int ldo, int32_t* err) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int item = blockIdx.x * warps + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int G = cb.groups, K = cb.size, gd = cb.group_dim;
  if (item >= M * G) return;
  const int m = item / G, g = item % G;
  const int k = __ldg(idx + item);
  float* o = out + (size_t)m * ldo + (size_t)g * gd;
  if (k < 0 || k >= K) {
    if (lane == 0) atomicExch(err, 1);
    for (int e = lane; e < gd; e += 32) o[e] = 0.f;
    return;
  }
  const float* c = cb.centroids + ((size_t)g * K + k) * gd;
  if ((gd & 3) == 0 && ((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(c)) & 15) == 0) {
    for (int e = lane * 4; e < gd; e += 128)
      *reinterpret_cast<float4*>(o + e) = __ldg(reinterpret_cast<const float4*>(c + e));
  } else {
    for (int e = lane; e < gd; e += 32) o[e] = __ldg(c + e);
  }
}

// 16-byte form (gd % 4 == 0, aligned rows): one thread per output float4, so narrow groups
// (gd = 24..64: 6..16 float4 per group) keep every lane busy and a warp stores 512 contiguous
// bytes of a row; the code of (m, g) is a broadcast load shared by the group's threads.
__global__ void vq_decode_v4_kernel(AstraCodebook cb, const int32_t* __restrict__ idx, int M,
                                    float* __restrict__ out, int ldo, int32_t* err,
                                    uint32_t per_magic) {
  pdl_wait();
  pdl_trigger();
  const int G = cb.groups, K = cb.size, gd = cb.group_dim;
  const int row4 = (G * gd) >> 2, per = gd >> 2;
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)M * row4) return;
  const int m = (int)(t / row4), c4 = (int)(t - (long)m * row4);
  const int g = per == 1 ? c4 : (int)__umulhi((uint32_t)c4, per_magic);   // (magic wraps for 1)
  const int k = __ldg(idx + (size_t)m * G + g);
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (k < 0 || k >= K)
    atomicExch(err, 1);
  else
    v = __ldg(reinterpret_cast<const float4*>(cb.centroids + ((size_t)g * K + k) * gd) + (c4 - g * per));
  *(reinterpret_cast<float4*>(out + (size_t)m * ldo) + c4) = v;
}

// ------------------------------------------------------------ packing
__global__ void pack_kernel(const int32_t* __restrict__ idx, int count, int bits,
                            uint32_t* __restrict__ words, int nwords) {
  pdl_wait();
  pdl_trigger();
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nwords) return;
  const long long b0 = (long long)w * 32, b1 = b0 + 32;
  uint32_t acc = 0;
  if (bits > 0) {
    long long first = b0 / bits, last = (b1 - 1) / bits;
    for (long long i = first; i <= last && i < count; ++i) {
      const uint64_t v = (uint64_t)(uint32_t)idx[i] & ((1ull << bits) - 1);
      const long long pos = i * bits - b0;  // may be negative
      acc |= (uint32_t)(pos >= 0 ? (v << pos) : (v >> (-pos)));
    }
  }
  words[w] = acc;
}

__global__ void unpack_kernel(const uint32_t* __restrict__ words, int count, int bits, int K,
                              int32_t* __restrict__ idx, int32_t* err) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint32_t v = 0;
  if (bits > 0) {
    const long long b = (long long)i * bits;
    const int w = (int)(b >> 5), off = (int)(b & 31);
    uint64_t pair = words[w];
    if (off + bits > 32) pair |= (uint64_t)words[w + 1] << 32;
    v = (uint32_t)((pair >> off) & ((1ull << bits) - 1));
  }
  if ((int)v >= K) {
    atomicExch(err, 1);
    v = 0;
  }
  idx[i] = (int32_t)v;
}

}  // namespace astra

using namespace astra;

extern "C" int astra_vq_prepare(const AstraCodebook* cbp, void* stream) {
  ASTRA_REQUIRE(cbp, ASTRA_ERR_SHAPE, "null codebook");
  AstraCodebook cb = *cbp;
  ASTRA_REQUIRE(cb.groups >= 1 && cb.size >= 1 && cb.group_dim >= 1, ASTRA_ERR_SHAPE,
                "bad codebook shape");
  ASTRA_REQUIRE(cb.padded_dim % 64 == 0 && cb.padded_dim >= cb.group_dim, ASTRA_ERR_SHAPE,
                "padded_dim must be a multiple of 64 >= group_dim");
  cudaStream_t s = as_stream(stream);
  const int rows = cb.groups * cb.size;
  launch_k(vq_prepare_kernel, (rows + 7) / 8, 256, 0, s, cb);
  launch_k(vq_normmax_kernel, cb.groups, 256, 0, s, cb);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int64_t astra_vq_encode_workspace(int M, int groups, int size, int padded_dim) {
  return (int64_t)carve(nullptr, nullptr, M, groups, size, padded_dim);
}

// Distance GEMM + windowed-argmin epilogue over `Mg` operand rows (per group), then the
// finalize over the M tokens.  rec_by_row: records are indexed by source row (pre-split
// operands cover the whole stack) instead of by token.
template <int BN>
static cudaError_t vq_launch_gemm(const AstraCodebook& cb, const CUtensorMap& ta,
                                  const CUtensorMap& talo, int Mg, VqWorkspace w, int nchunk,
                                  int cluster, cudaStream_t s) {
  const int G = cb.groups, K = cb.size, gdp = cb.padded_dim;
  CUtensorMap tb, tblo;
  if (make_tmap_2d(&tb, cb.c_hi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)G * K, gdp, gdp,
                   BN / cluster, kBK, true) ||
      make_tmap_2d(&tblo, cb.c_lo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)G * K, gdp, gdp,
                   BN / cluster, kBK, true))
    return cudaErrorInvalidValue;
  VqEpilogue<BN> epi{Mg, K, nchunk, reinterpret_cast<const float4*>(cb.c_win), w};
  TileSched sched{(Mg + kBM - 1) / kBM, (K + BN - 1) / BN, G, 1};
  return cluster == 2 ? launch_tc_gemm<BN, 3, 3, 2>(ta, talo, tb, tblo, gdp, sched, Mg, K, epi, s,
                                                    num_sms())
                      : launch_tc_gemm<BN, 3, 2, 1>(ta, talo, tb, tblo, gdp, sched, Mg, K, epi, s,
                                                    num_sms());
}

// Grouped codebooks: the run-mode GEMM (a CTA pair sweeps all code tiles of a row block)
// decides every row in its epilogue; only multi-candidate rows reach the re-rank kernel.
template <int BN>
static cudaError_t vq_launch_run(const AstraCodebook& cb, const CUtensorMap& ta,
                                 const CUtensorMap& talo, int M, VqWorkspace w, int32_t* idx_out,
                                 int32_t* stats, int cluster, cudaStream_t s,
                                 const int32_t* row_tok, int Mtok) {
  const int G = cb.groups, K = cb.size, gdp = cb.padded_dim;
  CUtensorMap tb, tblo;
  if (make_tmap_2d(&tb, cb.c_hi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)G * K, gdp, gdp,
                   BN / cluster, kBK, true) ||
      make_tmap_2d(&tblo, cb.c_lo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)G * K, gdp, gdp,
                   BN / cluster, kBK, true))
    return cudaErrorInvalidValue;
  VqRunEpilogue<BN> epi{M, K, reinterpret_cast<const float4*>(cb.c_win),
                         reinterpret_cast<const float*>(cb.c_norm_max), w, idx_out, stats, G,
                         row_tok, Mtok};
  TileSched sched{(M + kBM - 1) / kBM, (K + BN - 1) / BN, G, 1};
  sched.runs = 1;
  return cluster == 2 ? launch_tc_gemm<BN, 3, 3, 2>(ta, talo, tb, tblo, gdp, sched, M, K, epi, s,
                                                    num_sms())
                      : launch_tc_gemm<BN, 3, 2, 1>(ta, talo, tb, tblo, gdp, sched, M, K, epi, s,
                                                    num_sms());
}

// Distance GEMM + windowed-argmin epilogue over `Mg` operand rows (per group), then the
// finalize over the M tokens.  rec_by_row: records are indexed by source row (pre-split
// operands cover the whole stack) instead of by token.  Few token rows (one rank of a wide
// split) take 128-code tiles so the persistent grid still covers the SMs.  Grouped codebooks
// (G > 1, token-gathered operands) take the run-mode GEMM instead (no records, no finalize).
static int vq_gemm_finalize(const AstraCodebook& cb, const void* a_hi, const void* a_lo, int lda,
                            int Mg, VqWorkspace w, const float* x, int M, int ldx,
                            const int32_t* rows, int rec_by_row, int32_t* idx_out, int32_t* stats,
                            cudaStream_t s, const int32_t* row_tok_in = nullptr) {
  const int G = cb.groups, K = cb.size, gdp = cb.padded_dim;
  if (Mg <= 0 || M <= 0) return ASTRA_OK;   // (the GEMM's tile (0, 0) resets the re-rank count)
  static int debug_set = -1;
  if (debug_set < 0) {   // bench-only isolation switch for this unit's GEMMs, see tc_gemm.cuh
    const char* d = getenv("ASTRA_VQ_GEMM_DEBUG");
    debug_set = d ? atoi(d) : 0;
    if (debug_set) ASTRA_CUDA_CHECK(cudaMemcpyToSymbol(g_gemm_debug, &debug_set, sizeof(int)));
  }
  const int cluster = (Mg > kBM) ? 2 : 1;  // CTA pairs split the codebook tile (cta_group::2)
  const long units256 = (long)G * ((Mg + kBM * cluster - 1) / (kBM * cluster)) * ((K + kVqBN - 1) / kVqBN);
  const int bn = (units256 * 2 * cluster <= num_sms()) ? kVqBNMin : kVqBN;
  const int nchunk = kEpiParts * ((K + bn - 1) / bn);   // one record per epilogue column part
  CUtensorMap ta, talo;
  int st;
  if ((st = make_tmap_2d(&ta, a_hi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)G * Mg, gdp,
                         lda, kBM, kBK, true)))
    return st;
  if ((st = make_tmap_2d(&talo, a_lo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)G * Mg, gdp,
                         lda, kBM, kBK, true)))
    return st;
  // G = 1 over the pre-split stack: run mode only when it costs no extra waves (a run keeps a
  // pair for ceil(K / 256) tiles; with fewer row blocks than pairs the idle SMs cost more than
  // the finalize pass saves — ViT-B B=64: 50 blocks on 74 pairs, 58 us vs 51 + 9)
  const long pairs = num_sms() / 2, rblocks = (Mg + 2 * kBM - 1) / (2 * kBM), ct = (K + kVqBN - 1) / kVqBN;
  // (and only up to K = 1024: a run keeps 4 candidate slots per 1/4 of the codebook, and an
  // overflow costs an exact scan of every code — ViT-L K = 4096 saw 25 per step, 5 ms per layer;
  // records bound an overflow to its 64-code part)
  const bool run_g1 = rec_by_row && cluster == 2 && K >= kVqBN && K <= 4 * kVqBN &&
                      ((rblocks + pairs - 1) / pairs) * ct <= (rblocks * ct + pairs - 1) / pairs;
  if (G > 1 || run_g1) {
    // Run mode: grouped codebooks (token-gathered operands), and G = 1 over the pre-split stack
    // (a CTA pair per 256-row block sweeps the whole codebook; rows decided in the epilogue —
    // no records, no finalize pass; the re-rank takes the ~5% multi-candidate rows).
    const int* row_tok = row_tok_in;
    if (rec_by_row && !row_tok) {
      launch_k(vq_row_tok_fill_kernel, (Mg + 255) / 256, 256, 0, s, w.row_tok, Mg, w.rr_count, w.ov_count);
      launch_k(vq_row_tok_scatter_kernel, (M + 255) / 256, 256, 0, s, rows, M, w.row_tok);
      row_tok = w.row_tok;
    } else if (rec_by_row) {   // the caller's map: only the re-rank list count to reset
      launch_k(vq_row_tok_fill_kernel, 1, 32, 0, s, w.row_tok, 0, w.rr_count, w.ov_count);
    }
    const long runs = (long)G * ((Mg + kBM * cluster - 1) / (kBM * cluster));
    const int rbn = (K <= kVqBNMin || (G > 1 && runs * cluster < num_sms())) ? kVqBNMin : kVqBN;
    const cudaError_t er = rbn == kVqBN
        ? vq_launch_run<kVqBN>(cb, ta, talo, Mg, w, idx_out, stats, cluster, s, row_tok, M)
        : vq_launch_run<kVqBNMin>(cb, ta, talo, Mg, w, idx_out, stats, cluster, s, row_tok, M);
    ASTRA_CUDA_CHECK(er);
    const int gd = cb.group_dim;
    if (gd <= 128 && gd % 4 == 0 && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0)
      launch_k(vq_rerank_kernel<true>, num_sms() * kRerankBlocksNarrow, 256, 0, s, cb, x, M, ldx, rows, w, nchunk, idx_out,
                                                           stats, Mg, rec_by_row, bn / kEpiParts);
    else
      launch_k(vq_rerank_kernel<false>, num_sms() * kRerankBlocks, 256, 0, s, cb, x, M, ldx, rows, w, nchunk, idx_out,
                                                            stats, Mg, rec_by_row, bn / kEpiParts);
    ASTRA_CUDA_CHECK(cudaGetLastError());
    return ASTRA_OK;
  }
  const cudaError_t e = bn == kVqBN ? vq_launch_gemm<kVqBN>(cb, ta, talo, Mg, w, nchunk, cluster, s)
                                    : vq_launch_gemm<kVqBNMin>(cb, ta, talo, Mg, w, nchunk, cluster, s);
  ASTRA_CUDA_CHECK(e);
  const int items = G * M;
  if (nchunk <= 16)
    launch_k(vq_finalize_half_kernel, (items + 15) / 16, 256, 0, s, cb, M, rows, w, nchunk, idx_out,
                                                             stats, Mg, rec_by_row);
  else
    launch_k(vq_finalize_kernel, (items + 7) / 8, 256, 0, s, cb, x, M, ldx, rows, w, nchunk, idx_out,
                                                        stats, Mg, rec_by_row);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  launch_k(vq_rerank_kernel<false>, num_sms() * kRerankBlocks, 256, 0, s, cb, x, M, ldx, rows, w, nchunk, idx_out, stats,
                                                 Mg, rec_by_row, bn / kEpiParts);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_vq_encode(const AstraCodebook* cbp, const float* x, int M, int ldx,
                               const int32_t* rows, int32_t* idx_out, int32_t* stats,
                               void* workspace, int64_t workspace_bytes, void* stream) {
  ASTRA_REQUIRE(cbp && x && idx_out, ASTRA_ERR_SHAPE, "astra_vq_encode: null argument");
  const AstraCodebook cb = *cbp;
  ASTRA_REQUIRE(M >= 0, ASTRA_ERR_SHAPE, "astra_vq_encode: M < 0");
  if (M == 0) return ASTRA_OK;
  ASTRA_REQUIRE(ldx >= cb.groups * cb.group_dim, ASTRA_ERR_SHAPE, "astra_vq_encode: ldx too small");
  const int G = cb.groups, K = cb.size, gdp = cb.padded_dim;
  const size_t need = carve(nullptr, nullptr, M, G, K, gdp);
  ASTRA_REQUIRE((size_t)workspace_bytes >= need, ASTRA_ERR_SHAPE,
                "astra_vq_encode: workspace %lld < %zu bytes", (long long)workspace_bytes, need);
  VqWorkspace w;
  carve(&w, workspace, M, G, K, gdp);
  cudaStream_t s = as_stream(stream);
  const int gd = cb.group_dim, per = gd / 4;
  if (gd == gdp && gd % 4 == 0 && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
      (per <= 32 ? 32 % per == 0 : per % 32 == 0))
    launch_k(vq_split_v4_kernel, (M + 7) / 8, 256, 0, s, x, M, ldx, rows, G, gd, w);
  else
    launch_k(vq_split_kernel, (M + 7) / 8, 256, 0, s, x, M, ldx, rows, G, gd, gdp, w);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return vq_gemm_finalize(cb, w.x_hi, w.x_lo, gdp, M, w, x, M, ldx, rows, 0, idx_out, stats, s);
}

extern "C" int64_t astra_vq_encode_split_workspace(int R, int size) {
  return (int64_t)carve(nullptr, nullptr, R, 1, size, 0);
}

extern "C" int astra_vq_encode_split_ex(const AstraCodebook* cbp, const float* x, int ldx,
                                        const void* x_hi, const void* x_lo, int ld_split,
                                        const float* x_norm, int R, const int32_t* rows, int M,
                                        const int32_t* row_token, int32_t* idx_out,
                                        int32_t* stats, void* workspace, int64_t workspace_bytes,
                                        void* stream) {
  ASTRA_REQUIRE(cbp && x && x_hi && x_lo && x_norm && rows && idx_out, ASTRA_ERR_SHAPE,
                "astra_vq_encode_split: null argument");
  const AstraCodebook cb = *cbp;
  ASTRA_REQUIRE(cb.groups == 1 && cb.padded_dim == cb.group_dim, ASTRA_ERR_SHAPE,
                "astra_vq_encode_split: needs G = 1 and D %% 64 == 0");
  if (M == 0) return ASTRA_OK;
  const size_t need = carve(nullptr, nullptr, R, 1, cb.size, 0);
  ASTRA_REQUIRE((size_t)workspace_bytes >= need, ASTRA_ERR_SHAPE,
                "astra_vq_encode_split: workspace %lld < %zu bytes", (long long)workspace_bytes,
                need);
  VqWorkspace w;
  carve(&w, workspace, R, 1, cb.size, 0);
  w.x_hi = nullptr;
  w.x_lo = nullptr;
  w.x_norm = const_cast<float*>(x_norm);
  return vq_gemm_finalize(cb, x_hi, x_lo, ld_split, R, w, x, M, ldx, rows, 1, idx_out, stats,
                          as_stream(stream), row_token);
}

extern "C" int astra_vq_encode_split(const AstraCodebook* cbp, const float* x, int ldx,
                                     const void* x_hi, const void* x_lo, int ld_split,
                                     const float* x_norm, int R, const int32_t* rows, int M,
                                     int32_t* idx_out, int32_t* stats, void* workspace,
                                     int64_t workspace_bytes, void* stream) {
  return astra_vq_encode_split_ex(cbp, x, ldx, x_hi, x_lo, ld_split, x_norm, R, rows, M, nullptr,
                                  idx_out, stats, workspace, workspace_bytes, stream);
}

extern "C" int astra_vq_decode(const AstraCodebook* cbp, const int32_t* idx, int M, float* out,
                               int ldo, int32_t* err_flag, void* stream) {
  ASTRA_REQUIRE(cbp && idx && out && err_flag, ASTRA_ERR_SHAPE, "astra_vq_decode: null argument");
  const AstraCodebook cb = *cbp;
  ASTRA_REQUIRE(ldo >= cb.groups * cb.group_dim, ASTRA_ERR_SHAPE, "astra_vq_decode: ldo too small");
  if (M == 0) return ASTRA_OK;
  const int items = M * cb.groups;
  const int D = cb.groups * cb.group_dim;
  // (wide groups keep the warp per (m, g): 32+ float4 per code already fill the warp)
  if (cb.group_dim < 128 && cb.group_dim % 4 == 0 && ldo % 4 == 0 && D / 4 <= (1 << 20) &&
      ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(cb.centroids)) & 15) == 0) {
    const uint32_t per = (uint32_t)(cb.group_dim / 4);
    const long threads = (long)M * (D / 4);
    launch_k(vq_decode_v4_kernel, (unsigned)((threads + 255) / 256), 256, 0, as_stream(stream), cb,
             idx, M, out, ldo, err_flag, (uint32_t)((0x100000000ull + per - 1) / per));
  } else {
    launch_k(vq_decode_kernel, (items + 7) / 8, 256, 0, as_stream(stream), cb, idx, M, out, ldo, err_flag);
  }
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_pack_indices(const int32_t* idx, int count, int bits, uint32_t* words,
                                  void* stream) {
  ASTRA_REQUIRE(bits >= 0 && bits <= 31, ASTRA_ERR_SHAPE, "pack: bits out of range");
  const int nwords = (int)(((long long)count * bits + 31) / 32);
  if (nwords == 0) return ASTRA_OK;
  launch_k(pack_kernel, (nwords + 255) / 256, 256, 0, as_stream(stream), idx, count, bits, words, nwords);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_unpack_indices(const uint32_t* words, int count, int bits, int size,
                                    int32_t* idx, int32_t* err_flag, void* stream) {
  ASTRA_REQUIRE(bits >= 0 && bits <= 31, ASTRA_ERR_SHAPE, "unpack: bits out of range");
  if (count == 0) return ASTRA_OK;
  launch_k(unpack_kernel, (count + 255) / 256, 256, 0, as_stream(stream), words, count, bits, size, idx,
                                                                    err_flag);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}
