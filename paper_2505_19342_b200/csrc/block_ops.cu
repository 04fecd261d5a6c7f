// Row-wise block operations of the Astra layer that are HBM-bound:
//   - LayerNorm (tensor.layer_norm, tensor.py:318-345) producing the next GEMM's operand
//     (bf16, or the bf16 hi/lo split in parity mode), optionally fp32;
//   - stack assembly x + pos / class replicas (model.py:275-280, cluster.py:189-194, :259-262);
//   - replica merge mean (cluster.py:290-292 -> tensor.mean_rows, tensor.py:200-208);
//   - per-layer key map (G=1 remote keys -> codebook K/V table rows, cluster.py:182-187).
// One warp per row, 16-byte vector accesses; grids sized in multiples of the SM count.
#include "host_common.h"
#include "ptx.cuh"

namespace astra {

// ---------------------------------------------------------------- LayerNorm
// mean, biased variance, 1/sqrt(var + eps), affine — all fp32 like the reference.
// Source rows of the LayerNorm: the stack itself, or (decode fused into LN1) the VQ decode of
// received codes — row r, float4 q of the row = centroids[g][idx[r, g]][4q - g gd], a coalesced
// gather of L2-resident codebook rows (vq.dequantize, vq.py:225-233, then tensor.layer_norm):
// the decoded fp32 row never goes to HBM.  Codes outside [0, K) raise the error flag and read
// as zero rows (the caller raises IndexCorruptionError, vq.py:229-231).
struct LnGather {
  const float* cents;     // [G, K, gd] fp32
  const int32_t* idx;     // [M, G]
  int G, K, gd;
  int32_t* err;
  uint32_t per_magic;     // ceil(2^32 / (gd / 4)): q / (gd / 4) = umulhi(q, magic) for q < 2^8
};

template <int VPL>  // float4 vectors per lane (D = VPL * 128)
__global__ void layernorm_kernel(const float* __restrict__ x, int M, int ldx,
                                 const float* __restrict__ gain, const float* __restrict__ bias,
                                 float eps, float* __restrict__ out_f32, int ld_f32,
                                 __nv_bfloat16* __restrict__ out_hi, __nv_bfloat16* __restrict__ out_lo,
                                 int ld_bf, __nv_bfloat16* __restrict__ xs_hi,
                                 __nv_bfloat16* __restrict__ xs_lo, int ld_xs,
                                 float* __restrict__ x_norm, LnGather gat = LnGather{}) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  // one row per warp, every row of the grid in flight at once (no grid-stride tail: the
  // kernel is HBM-latency bound, and a second partial round doubles the exposed latency)
  const int row = blockIdx.x * warps + (threadIdx.x >> 5);
  if (row < M) {
    float4 v[VPL];
    if (gat.cents) {
      const int per = gat.gd >> 2;   // float4s per group
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        const int q = lane + 32 * i, g = per == 1 ? q : (int)__umulhi((uint32_t)q, gat.per_magic);
        const int k = __ldg(gat.idx + (size_t)row * gat.G + g);
        if (k < 0 || k >= gat.K) {
          atomicExch(gat.err, 1);
          v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
          v[i] = __ldg(reinterpret_cast<const float4*>(gat.cents + ((size_t)g * gat.K + k) * gat.gd) +
                       (q - g * per));
        }
      }
    } else {
      const float4* xr = reinterpret_cast<const float4*>(x + (size_t)row * ldx);
#pragma unroll
      for (int i = 0; i < VPL; ++i) v[i] = __ldg(xr + lane + 32 * i);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
      if (xs_hi) {  // bf16 hi/lo split of the raw row: the VQ-encode GEMM operand
        __nv_bfloat16 h[4], l[4];
        split_bf16(v[i].x, h[0], l[0]);
        split_bf16(v[i].y, h[1], l[1]);
        split_bf16(v[i].z, h[2], l[2]);
        split_bf16(v[i].w, h[3], l[3]);
        const size_t o = (size_t)row * ld_xs + (lane + 32 * i) * 4;
        *reinterpret_cast<uint2*>(xs_hi + o) = *reinterpret_cast<uint2*>(h);
        *reinterpret_cast<uint2*>(xs_lo + o) = *reinterpret_cast<uint2*>(l);
      }
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float D = (float)(VPL * 128);
    const float mu = s / D;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      v[i].x -= mu; v[i].y -= mu; v[i].z -= mu; v[i].w -= mu;
      q += (v[i].x * v[i].x + v[i].y * v[i].y) + (v[i].z * v[i].z + v[i].w * v[i].w);
    }
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = 1.0f / sqrtf(q / D + eps);
    // ||x|| upper bound for the VQ error window: ||x||^2 = sum (x-mu)^2 + D mu^2
    if (x_norm && lane == 0) x_norm[row] = sqrtf(q + D * mu * mu) * (1.0f + 1e-5f);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = (lane + 32 * i) * 4;
      const float4 g = __ldg(reinterpret_cast<const float4*>(gain + c));
      const float4 b = __ldg(reinterpret_cast<const float4*>(bias + c));
      float4 y;
      y.x = __fadd_rn(__fmul_rn(__fmul_rn(v[i].x, inv), g.x), b.x);
      y.y = __fadd_rn(__fmul_rn(__fmul_rn(v[i].y, inv), g.y), b.y);
      y.z = __fadd_rn(__fmul_rn(__fmul_rn(v[i].z, inv), g.z), b.z);
      y.w = __fadd_rn(__fmul_rn(__fmul_rn(v[i].w, inv), g.w), b.w);
      if (out_f32) *reinterpret_cast<float4*>(out_f32 + (size_t)row * ld_f32 + c) = y;
      if (out_hi) {
        __nv_bfloat16 h[4], l[4];
        split_bf16(y.x, h[0], l[0]);
        split_bf16(y.y, h[1], l[1]);
        split_bf16(y.z, h[2], l[2]);
        split_bf16(y.w, h[3], l[3]);
        *reinterpret_cast<uint2*>(out_hi + (size_t)row * ld_bf + c) = *reinterpret_cast<uint2*>(h);
        if (out_lo)
          *reinterpret_cast<uint2*>(out_lo + (size_t)row * ld_bf + c) = *reinterpret_cast<uint2*>(l);
      }
    }
  }
}

// generic-width fallback (D % 4 == 0 but not a multiple of 128)
__global__ void layernorm_generic_kernel(const float* __restrict__ x, int M, int D, int ldx,
                                         const float* __restrict__ gain,
                                         const float* __restrict__ bias, float eps,
                                         float* __restrict__ out_f32, int ld_f32,
                                         __nv_bfloat16* __restrict__ out_hi,
                                         __nv_bfloat16* __restrict__ out_lo, int ld_bf) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int row = blockIdx.x * warps + (threadIdx.x >> 5); row < M; row += gridDim.x * warps) {
    const float* xr = x + (size_t)row * ldx;
    float s = 0.f;
    for (int c = lane; c < D; c += 32) s += xr[c];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / (float)D;
    float q = 0.f;
    for (int c = lane; c < D; c += 32) {
      const float d = xr[c] - mu;
      q += d * d;
    }
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = 1.0f / sqrtf(q / (float)D + eps);
    for (int c = lane; c < D; c += 32) {
      const float y = __fadd_rn(__fmul_rn(__fmul_rn(xr[c] - mu, inv), gain[c]), bias[c]);
      if (out_f32) out_f32[(size_t)row * ld_f32 + c] = y;
      if (out_hi) {
        __nv_bfloat16 h, l;
        split_bf16(y, h, l);
        out_hi[(size_t)row * ld_bf + c] = h;
        if (out_lo) out_lo[(size_t)row * ld_bf + c] = l;
      }
    }
  }
}

// --------------------------------------------------------------- stack build
// row_src[r] >= 0 : content row = x[row_src[r]] + pos[row_pos[r]]   (x is [B*T, D])
// row_src[r] <  0 : class replica = cls
__global__ void embed_stack_kernel(const float* __restrict__ x, const float* __restrict__ pos,
                                   const float* __restrict__ cls, const int32_t* __restrict__ row_src,
                                   const int32_t* __restrict__ row_pos, int rows, int D,
                                   float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < rows; r += gridDim.x * warps) {
    const int src = row_src[r];
    float* o = out + (size_t)r * D;
    if ((D & 3) != 0) {   // general width (small reference configs): scalar path
      const float* a = src >= 0 ? x + (size_t)src * D : cls;
      const float* p = pos + (size_t)(src >= 0 ? row_pos[r] : 0) * D;
      for (int c = lane; c < D; c += 32) o[c] = src >= 0 ? a[c] + p[c] : a[c];
    } else if (src >= 0) {
      const float* a = x + (size_t)src * D;
      const float* p = pos + (size_t)row_pos[r] * D;
      for (int c = lane * 4; c < D; c += 128) {
        float4 va = __ldg(reinterpret_cast<const float4*>(a + c));
        float4 vp = __ldg(reinterpret_cast<const float4*>(p + c));
        *reinterpret_cast<float4*>(o + c) =
            make_float4(va.x + vp.x, va.y + vp.y, va.z + vp.z, va.w + vp.w);
      }
    } else {
      for (int c = lane * 4; c < D; c += 128)
        *reinterpret_cast<float4*>(o + c) = __ldg(reinterpret_cast<const float4*>(cls + c));
    }
  }
}

// ------------------------------------------------------------- replica mean
// reps: [N, B, D] in device order -> out [B, D] = (((r0 + r1) + r2) + ...) / N
__global__ void replica_mean_kernel(const float* __restrict__ reps, int N, int BD,
                                    float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= BD) return;
  float s = reps[i];
  for (int n = 1; n < N; ++n) s += reps[(size_t)n * BD + i];
  out[i] = s / (float)N;
}

// gather rows: out[r] = src[idx[r]]   (D floats, float4)
__global__ void gather_rows_kernel(const float* __restrict__ src, int lds,
                                   const int32_t* __restrict__ idx, int rows, int D,
                                   float* __restrict__ out, int ldo) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < rows; r += gridDim.x * warps) {
    const float* s = src + (size_t)idx[r] * lds;
    float* o = out + (size_t)r * ldo;
    if (((D | lds | ldo) & 3) != 0) {
      for (int c = lane; c < D; c += 32) o[c] = s[c];
    } else {
      for (int c = lane * 4; c < D; c += 128)
        *reinterpret_cast<float4*>(o + c) = __ldg(reinterpret_cast<const float4*>(s + c));
    }
  }
}

// ------------------------------------------------------------------ key map
// key_map[j] >= 0 : local key row (copied)
// key_map[j] <  0 : remote content token t = -(key_map[j]+1); key_src[j] = -(codes[t]+1)
//                   (G = 1: the K/V table row of its code)  or  -(t+1) when codes == NULL
__global__ void key_map_kernel(const int32_t* __restrict__ key_map, int n,
                               const int32_t* __restrict__ codes, int32_t* __restrict__ key_src) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int m = key_map[j];
  key_src[j] = (m >= 0 || codes == nullptr) ? m : -(codes[-(m + 1)] + 1);
}

// ---------------------------------------------------------- decode support
// (greedy generation on the device holding the last prompt token: cluster.py:297-308,
//  DecodeState / _decode_one model.py:324-358)

// 16-byte vector copy of `bytes` (multiple of 16) by one warp
__device__ __forceinline__ void warp_copy16(void* dst, const void* src, int bytes, int lane) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* d = reinterpret_cast<uint4*>(dst);
  for (int i = lane; i < bytes / 16; i += 32) d[i] = __ldg(s + i);
}

// cache row (i / n_per) * ld_blocks + i % n_per  <-  [K | V] of key i, gathered via key_src
__global__ void gather_kv_kernel(const int32_t* __restrict__ key_src, int n, int n_per,
                                 int ld_blocks, const uint8_t* __restrict__ k_local,
                                 const uint8_t* __restrict__ v_local, int ld_local,
                                 const uint8_t* __restrict__ k_remote,
                                 const uint8_t* __restrict__ v_remote, int ld_remote,
                                 int row_bytes, uint8_t* __restrict__ cache, int ld_cache) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * warps + (threadIdx.x >> 5); i < n; i += gridDim.x * warps) {
    const int src = key_src[i];
    const uint8_t *kp, *vp;
    if (src >= 0) {
      kp = k_local + (size_t)src * ld_local;
      vp = v_local + (size_t)src * ld_local;
    } else {
      kp = k_remote + (size_t)(-(src + 1)) * ld_remote;
      vp = v_remote + (size_t)(-(src + 1)) * ld_remote;
    }
    uint8_t* dst = cache + ((size_t)(i / n_per) * ld_blocks + i % n_per) * ld_cache;
    warp_copy16(dst, kp, row_bytes, lane);
    warp_copy16(dst + row_bytes, vp, row_bytes, lane);
  }
}

// append the new token's K|V (row b of the projection buffer) at cache row b*ld_blocks + pos[b]
__global__ void append_kv_kernel(const uint8_t* __restrict__ k_new, const uint8_t* __restrict__ v_new,
                                 int ld_new, int rows, const int32_t* __restrict__ pos,
                                 int ld_blocks, int row_bytes, uint8_t* __restrict__ cache,
                                 int ld_cache) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= rows) return;
  uint8_t* dst = cache + ((size_t)b * ld_blocks + pos[b]) * ld_cache;
  warp_copy16(dst, k_new + (size_t)b * ld_new, row_bytes, lane);
  warp_copy16(dst + row_bytes, v_new + (size_t)b * ld_new, row_bytes, lane);
}

// np.argmax order (model.py:358 / cluster.py:302): NaN ranks above every number (the first
// NaN wins), then the larger value, then the lower index on ties.  An all -inf row picks 0.
__device__ __forceinline__ bool argmax_better(float v, int i, float bv, int bi) {
  const bool vn = isnan(v), bn = isnan(bv);
  if (vn != bn) return vn;
  if (vn) return i < bi;
  return v > bv || (v == bv && i < bi);
}

// greedy argmax per row, lowest index on ties
__global__ void argmax_rows_kernel(const float* __restrict__ logits, int cols, int ld,
                                   int32_t* __restrict__ out, int out_stride,
                                   const int32_t* __restrict__ step_pos, int pos_base,
                                   int32_t* __restrict__ next_tok) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x;
  const float* lr = logits + (size_t)row * ld;
  float bv = -INFINITY;
  int bi = 0x7FFFFFFF;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float v = lr[c];
    if (argmax_better(v, c, bv, bi)) {
      bv = v;
      bi = c;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (argmax_better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[w] = bv;
    si[w] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i)
      if (argmax_better(sv[i], si[i], bv, bi)) {
        bv = sv[i];
        bi = si[i];
      }
    if (bi == 0x7FFFFFFF) bi = 0;   // cols == 0 cannot happen; keep the id in range anyway
    const int slot = step_pos ? step_pos[row] - pos_base : 0;
    out[(size_t)row * out_stride + slot] = bi;
    if (next_tok) next_tok[row] = bi;
  }
}

// one decode step done: every image's position and key count advance by one
__global__ void decode_advance_kernel(int32_t* __restrict__ pos, int32_t* __restrict__ segs,
                                      int rows) {
  pdl_wait();
  pdl_trigger();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= rows) return;
  pos[b] += 1;
  segs[b * 6 + 2] += 1;  // query position
  segs[b * 6 + 5] += 1;  // key count
}

static int grid_rows(int rows, int warps_per_block) {
  int g = (rows + warps_per_block - 1) / warps_per_block;
  const int cap = num_sms() * 8;
  return g < cap ? (g > 0 ? g : 1) : cap;
}

}  // namespace astra

using namespace astra;

// Lloyd centroid update (vq.py:160-165 `pts[assign == k].mean(axis=0)`): thread per
// (cluster, dim) sums its cluster's points in ascending sample order in fp64 — NumPy's
// axis-0 reduction order — then divides by the count, so the result is bit-identical to the
// reference's mean for the same assignment.  `order` lists the sample ids sorted by cluster
// (stable), seg[k]..seg[k+1] the range of cluster k.  Empty clusters keep `mean` unchanged.
__global__ void segment_mean_f64_kernel(const double* __restrict__ pts, int ld,
                                        const int32_t* __restrict__ order,
                                        const int32_t* __restrict__ seg, int k, int dim,
                                        double* __restrict__ mean, double* __restrict__ sums) {
  pdl_wait();
  pdl_trigger();
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (d >= dim || c >= k) return;
  const int s0 = seg[c], s1 = seg[c + 1];
  double acc = 0.0;
  for (int i = s0; i < s1; ++i) acc += pts[(size_t)order[i] * ld + d];
  if (sums) sums[(size_t)c * dim + d] = acc;
  if (s1 > s0) mean[(size_t)c * dim + d] = acc / (double)(s1 - s0);
}

// LM embed (model.py:283-288): out[r] = emb[ids[row_src[r]]] + pos[row_pos[r]].  ids are this
// step's token ids [B*T] in HBM (staged by one H2D copy), row_src the static stack-row ->
// (b*T + t) map of the layout, so a new batch needs no host-side index rebuild.
__global__ void embed_tokens_kernel(const float* __restrict__ emb, const float* __restrict__ pos,
                                    const int32_t* __restrict__ ids,
                                    const int32_t* __restrict__ row_src,
                                    const int32_t* __restrict__ row_pos, int rows, int D,
                                    float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < rows; r += gridDim.x * warps) {
    const float* a = emb + (size_t)ids[row_src[r]] * D;
    const float* p = pos + (size_t)row_pos[r] * D;
    float* o = out + (size_t)r * D;
    if ((D & 3) != 0) {
      for (int c = lane; c < D; c += 32) o[c] = a[c] + p[c];
    } else {
      for (int c = lane * 4; c < D; c += 128) {
        const float4 va = __ldg(reinterpret_cast<const float4*>(a + c));
        const float4 vp = __ldg(reinterpret_cast<const float4*>(p + c));
        *reinterpret_cast<float4*>(o + c) =
            make_float4(va.x + vp.x, va.y + vp.y, va.z + vp.z, va.w + vp.w);
      }
    }
  }
}

extern "C" int astra_layernorm_ex(const float* x, int M, int D, int ldx, const float* gain,
                                  const float* bias, float eps, float* out_f32, int ld_f32,
                                  void* out_hi, void* out_lo, int ld_bf, void* xs_hi, void* xs_lo,
                                  int ld_xs, float* x_norm, void* stream) {
  ASTRA_REQUIRE(M >= 0 && D > 0, ASTRA_ERR_SHAPE, "layernorm: bad shape");
  ASTRA_REQUIRE(eps > 0.f, ASTRA_ERR_SHAPE, "layer_norm: eps must be positive");
  ASTRA_REQUIRE((xs_hi == nullptr) == (xs_lo == nullptr), ASTRA_ERR_SHAPE,
                "layernorm: split outputs come in pairs");
  if (M == 0) return ASTRA_OK;
  cudaStream_t s = as_stream(stream);
  auto hi = reinterpret_cast<__nv_bfloat16*>(out_hi);
  auto lo = reinterpret_cast<__nv_bfloat16*>(out_lo);
  auto xh = reinterpret_cast<__nv_bfloat16*>(xs_hi);
  auto xl = reinterpret_cast<__nv_bfloat16*>(xs_lo);
  const bool vec = (D % 128 == 0) && (ldx % 4 == 0) && (!out_f32 || ld_f32 % 4 == 0) &&
                   (!out_hi || ld_bf % 4 == 0) && (!xs_hi || ld_xs % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  const int grid = grid_rows(M, 8);
  const int grid1 = (M + 3) / 4;   // vector kernels: one row per warp, 4 warps per block
  if (vec && D == 768)
    launch_k(layernorm_kernel<6>, grid1, 128, 0, s, x, M, ldx, gain, bias, eps, out_f32, ld_f32, hi, lo,
                                             ld_bf, xh, xl, ld_xs, x_norm, LnGather{});
  else if (vec && D == 1024)
    launch_k(layernorm_kernel<8>, grid1, 128, 0, s, x, M, ldx, gain, bias, eps, out_f32, ld_f32, hi, lo,
                                             ld_bf, xh, xl, ld_xs, x_norm, LnGather{});
  else if (vec && D == 512)
    launch_k(layernorm_kernel<4>, grid1, 128, 0, s, x, M, ldx, gain, bias, eps, out_f32, ld_f32, hi, lo,
                                             ld_bf, xh, xl, ld_xs, x_norm, LnGather{});
  else {
    ASTRA_REQUIRE(xs_hi == nullptr && x_norm == nullptr, ASTRA_ERR_SHAPE,
                  "layernorm: split / norm outputs need D in {512, 768, 1024}");
    launch_k(layernorm_generic_kernel, grid, 256, 0, s, x, M, D, ldx, gain, bias, eps, out_f32, ld_f32,
                                                  hi, lo, ld_bf);
  }
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_vq_decode_layernorm(const AstraCodebook* cbp, const int32_t* idx, int M,
                                         const float* gain, const float* bias, float eps,
                                         void* out_hi, void* out_lo, int ld_bf, int32_t* err_flag,
                                         void* stream) {
  ASTRA_REQUIRE(cbp && idx && gain && bias && out_hi && err_flag, ASTRA_ERR_SHAPE,
                "decode_layernorm: null argument");
  const AstraCodebook cb = *cbp;
  const int D = cb.groups * cb.group_dim;
  ASTRA_REQUIRE(M >= 0, ASTRA_ERR_SHAPE, "decode_layernorm: M < 0");
  ASTRA_REQUIRE(eps > 0.f, ASTRA_ERR_SHAPE, "layer_norm: eps must be positive");
  ASTRA_REQUIRE((D == 512 || D == 768 || D == 1024) && cb.group_dim % 4 == 0 && ld_bf % 4 == 0 &&
                    (reinterpret_cast<uintptr_t>(cb.centroids) & 15) == 0,
                ASTRA_ERR_SHAPE, "decode_layernorm: needs D in {512, 768, 1024} and D/G %% 4 == 0");
  if (M == 0) return ASTRA_OK;
  cudaStream_t s = as_stream(stream);
  auto hi = reinterpret_cast<__nv_bfloat16*>(out_hi);
  auto lo = reinterpret_cast<__nv_bfloat16*>(out_lo);
  const uint32_t per = (uint32_t)(cb.group_dim / 4);
  const LnGather gat{cb.centroids, idx, cb.groups, cb.size, cb.group_dim, err_flag,
                     (uint32_t)((0x100000000ull + per - 1) / per)};
  const int grid1 = (M + 3) / 4;
  if (D == 768)
    launch_k(layernorm_kernel<6>, grid1, 128, 0, s, nullptr, M, 0, gain, bias, eps, nullptr, 0, hi, lo,
                                             ld_bf, nullptr, nullptr, 0, nullptr, gat);
  else if (D == 1024)
    launch_k(layernorm_kernel<8>, grid1, 128, 0, s, nullptr, M, 0, gain, bias, eps, nullptr, 0, hi, lo,
                                             ld_bf, nullptr, nullptr, 0, nullptr, gat);
  else
    launch_k(layernorm_kernel<4>, grid1, 128, 0, s, nullptr, M, 0, gain, bias, eps, nullptr, 0, hi, lo,
                                             ld_bf, nullptr, nullptr, 0, nullptr, gat);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_layernorm(const float* x, int M, int D, int ldx, const float* gain,
                               const float* bias, float eps, float* out_f32, int ld_f32,
                               void* out_hi, void* out_lo, int ld_bf, void* stream) {
  return astra_layernorm_ex(x, M, D, ldx, gain, bias, eps, out_f32, ld_f32, out_hi, out_lo, ld_bf,
                            nullptr, nullptr, 0, nullptr, stream);
}

extern "C" int astra_embed_stack(const float* x, const float* pos, const float* cls,
                                 const int32_t* row_src, const int32_t* row_pos, int rows, int D,
                                 float* out, void* stream) {
  ASTRA_REQUIRE(D >= 1, ASTRA_ERR_SHAPE, "embed: bad width");
  if (rows == 0) return ASTRA_OK;
  launch_k(embed_stack_kernel, grid_rows(rows, 8), 256, 0, as_stream(stream), x, pos, cls, row_src,
                                                                       row_pos, rows, D, out);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_replica_mean(const float* reps, int N, int B, int D, float* out,
                                  void* stream) {
  ASTRA_REQUIRE(N >= 1, ASTRA_ERR_SHAPE, "no class-token replicas to aggregate");
  const int bd = B * D;
  if (bd == 0) return ASTRA_OK;
  launch_k(replica_mean_kernel, (bd + 255) / 256, 256, 0, as_stream(stream), reps, N, bd, out);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_gather_rows(const float* src, int lds, const int32_t* idx, int rows, int D,
                                 float* out, int ldo, void* stream) {
  ASTRA_REQUIRE(D >= 1 && lds >= D && ldo >= D, ASTRA_ERR_SHAPE, "gather_rows: bad widths");
  if (rows == 0) return ASTRA_OK;
  launch_k(gather_rows_kernel, grid_rows(rows, 8), 256, 0, as_stream(stream), src, lds, idx, rows, D,
                                                                       out, ldo);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

// G = 1 exchange, fused: remote key -> codebook row straight from the all-gathered packed
// words (sender e's payload at words[e * wmax]; its code i at bit i * bits), replacing the
// per-sender unpack launches + key map.  Corrupt codes (>= K) raise *err and map to row 0.
__global__ void key_map_packed_kernel(const int32_t* __restrict__ key_map, int n,
                                      const uint32_t* __restrict__ words, int wmax, int bits, int K,
                                      const int32_t* __restrict__ gofs, int nsend,
                                      int32_t* __restrict__ key_src, int32_t* err) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int m = key_map[j];
  if (m >= 0) {
    key_src[j] = m;
    return;
  }
  const int slot = -(m + 1);
  int e = 0;
  while (e + 1 < nsend && __ldg(gofs + e + 1) <= slot) ++e;
  const long long b = (long long)e * wmax * 32 + (long long)(slot - __ldg(gofs + e)) * bits;
  const uint32_t* wp = words + (b >> 5);
  const int off = (int)(b & 31);
  uint64_t pair = __ldg(wp);
  if (off + bits > 32) pair |= (uint64_t)__ldg(wp + 1) << 32;
  int code = (int)((pair >> off) & ((1ull << bits) - 1));
  if (code >= K) {
    atomicExch(err, 1);
    code = 0;
  }
  key_src[j] = -(code + 1);
}

extern "C" int astra_key_map_packed(const int32_t* key_map, int n, const uint32_t* words, int wmax,
                                    int bits, int size, const int32_t* gofs, int nsend,
                                    int32_t* key_src, int32_t* err_flag, void* stream) {
  ASTRA_REQUIRE(bits >= 1 && bits <= 31 && nsend >= 1, ASTRA_ERR_SHAPE, "key_map_packed: bad shape");
  if (n == 0) return ASTRA_OK;
  launch_k(key_map_packed_kernel, (n + 255) / 256, 256, 0, as_stream(stream), 
      key_map, n, words, wmax, bits, size, gofs, nsend, key_src, err_flag);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_key_map(const int32_t* key_map, int n, const int32_t* codes,
                             int32_t* key_src, void* stream) {
  if (n == 0) return ASTRA_OK;
  launch_k(key_map_kernel, (n + 255) / 256, 256, 0, as_stream(stream), key_map, n, codes, key_src);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_gather_kv(const int32_t* key_src, int n, int n_per, int ld_blocks,
                               const void* k_local, const void* v_local, int ld_local_bytes,
                               const void* k_remote, const void* v_remote, int ld_remote_bytes,
                               int row_bytes, void* cache, int ld_cache_bytes, void* stream) {
  ASTRA_REQUIRE(row_bytes % 16 == 0 && n_per > 0, ASTRA_ERR_SHAPE, "gather_kv: bad row size");
  if (n == 0) return ASTRA_OK;
  launch_k(gather_kv_kernel, grid_rows(n, 8), 256, 0, as_stream(stream), 
      key_src, n, n_per, ld_blocks, (const uint8_t*)k_local, (const uint8_t*)v_local,
      ld_local_bytes, (const uint8_t*)k_remote, (const uint8_t*)v_remote, ld_remote_bytes,
      row_bytes, (uint8_t*)cache, ld_cache_bytes);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_append_kv(const void* k_new, const void* v_new, int ld_new_bytes, int rows,
                               const int32_t* pos, int ld_blocks, int row_bytes, void* cache,
                               int ld_cache_bytes, void* stream) {
  ASTRA_REQUIRE(row_bytes % 16 == 0, ASTRA_ERR_SHAPE, "append_kv: bad row size");
  if (rows == 0) return ASTRA_OK;
  launch_k(append_kv_kernel, (rows + 7) / 8, 256, 0, as_stream(stream), 
      (const uint8_t*)k_new, (const uint8_t*)v_new, ld_new_bytes, rows, pos, ld_blocks, row_bytes,
      (uint8_t*)cache, ld_cache_bytes);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_argmax_rows(const float* logits, int rows, int cols, int ld, int32_t* out,
                                 int out_stride, const int32_t* step_pos, int pos_base,
                                 int32_t* next_tok, void* stream) {
  if (rows == 0) return ASTRA_OK;
  launch_k(argmax_rows_kernel, rows, 1024, 0, as_stream(stream), logits, cols, ld, out, out_stride,
                                                            step_pos, pos_base, next_tok);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_decode_advance(int32_t* pos, int32_t* segs, int rows, void* stream) {
  if (rows == 0) return ASTRA_OK;
  launch_k(decode_advance_kernel, (rows + 127) / 128, 128, 0, as_stream(stream), pos, segs, rows);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_segment_mean_f64(const double* pts, int ld, const int32_t* order,
                                      const int32_t* seg, int k, int dim, double* mean,
                                      double* sums, void* stream) {
  ASTRA_REQUIRE(k >= 0 && dim >= 0 && ld >= dim, ASTRA_ERR_SHAPE, "segment_mean: bad shape");
  if (k == 0 || dim == 0) return ASTRA_OK;
  dim3 grid((dim + 127) / 128, k);
  launch_k(segment_mean_f64_kernel, grid, 128, 0, as_stream(stream), pts, ld, order, seg, k, dim, mean,
                                                              sums);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_embed_tokens(const float* emb, const float* pos, const int32_t* ids,
                                  const int32_t* row_src, const int32_t* row_pos, int rows, int D,
                                  float* out, void* stream) {
  ASTRA_REQUIRE(rows >= 0 && D >= 1, ASTRA_ERR_SHAPE, "embed_tokens: bad shape");
  if (rows == 0) return ASTRA_OK;
  launch_k(embed_tokens_kernel, grid_rows(rows, 8), 256, 0, as_stream(stream), emb, pos, ids, row_src,
                                                                        row_pos, rows, D, out);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}
