// Mixed-precision attention with distributed class tokens
// (reference: attention.multihead_attention attention.py:50-73 + tensor.masked_softmax
// tensor.py:295-315, called from cluster._device_layer_compute cluster.py:201-212).
//
// One launch covers every (segment, head, 64-query tile).  A segment is one device's view of
// one image: its local query rows (content + optional class replica) and its key list of
// T tokens + replica key.  Each key is gathered by `key_src`:
//     key_src >= 0 : a local row of the K/V projection buffer (full precision)
//     key_src <  0 : row -(key_src+1) of the remote K/V buffer — for G = 1 that is the per-layer
//                    codebook K/V table indexed directly by the received VQ code, i.e. the VQ
//                    decode is fused into the K/V tile load; for G > 1 the decoded K^/V^ rows.
// Masking: key visible iff !causal || key_pos <= query_pos (class replica key has pos -1 and
// replica queries pos INT_MAX), so masked weights are exactly zero like the reference.
//
// v1 is an fp32 SIMT flash-style kernel (online softmax over 64-key tiles, 64x64 fp32 K/V tiles
// in padded shared memory).  It is exact enough for the fp32 parity mode and general in T.
#include <climits>

#include "host_common.h"
#include "ptx.cuh"

namespace astra {

struct AttnArgs {
  const void* q;
  int ldq;
  const void* k_local;
  const void* v_local;
  int ld_local;
  const void* k_remote;
  const void* v_remote;
  int ld_remote;
  const int32_t* key_src;
  const int32_t* key_pos;
  const int32_t* segs;  // [S, 6] q0, nq, qpos0, ncontent, k0, nk
  int num_segs, heads, head_dim, causal, in_bf16;
  float scale;
  float* out_f32;
  __nv_bfloat16* out_hi;
  __nv_bfloat16* out_lo;
  int ld_out;
};

constexpr int kAQ = 64;    // queries per CTA
constexpr int kAK = 64;    // keys per tile

template <bool BF16>
__device__ __forceinline__ float ld_elem(const void* base, size_t off) {
  if (BF16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[off]);
  return reinterpret_cast<const float*>(base)[off];
}

template <bool BF16, int kDH>
__global__ void __launch_bounds__(256) attention_simt_kernel(AttnArgs a) {
  constexpr int kPad = kDH + 1;
  constexpr int kDPT = kDH / 4;   // output dims per thread
  extern __shared__ float smem_f[];
  float* sK = smem_f;
  float* sV = sK + kAK * kPad;
  float* sP = sV + kAK * kPad;
  int* sKpos = reinterpret_cast<int*>(sP + kAQ * (kAK + 1));

  const int seg = blockIdx.x, h = blockIdx.y, qt = blockIdx.z;
  const int* sg = a.segs + seg * 6;
  const int q0 = sg[0], nq = sg[1], qpos0 = sg[2], ncontent = sg[3], k0 = sg[4], nk = sg[5];
  if (qt * kAQ >= nq) return;
  const int tid = threadIdx.x;
  const int r = tid >> 2, part = tid & 3;
  const int qi = qt * kAQ + r;
  const bool qvalid = qi < nq;
  const int qpos = qi < ncontent ? qpos0 + qi : INT_MAX;
  const int hoff = h * kDH;

  float q[kDH];
  {
    const size_t base = (size_t)(q0 + (qvalid ? qi : 0)) * a.ldq + hoff;
#pragma unroll
    for (int d = 0; d < kDH; ++d) q[d] = ld_elem<BF16>(a.q, base + d);
  }
  float m = -INFINITY, l = 0.f;
  float acc[kDPT];
#pragma unroll
  for (int i = 0; i < kDPT; ++i) acc[i] = 0.f;

  for (int kt = 0; kt < nk; kt += kAK) {
    // ---- gather K/V tile (64 keys x 64 dims): thread -> key tid/4, 16 dims
    {
      const int kj = tid >> 2, c0 = (tid & 3) * kDPT;
      const int j = kt + kj;
      if (j < nk) {
        const int src = a.key_src[k0 + j];
        const void *kb, *vb;
        size_t off;
        if (src >= 0) {
          kb = a.k_local;
          vb = a.v_local;
          off = (size_t)src * a.ld_local + hoff + c0;
        } else {
          kb = a.k_remote;
          vb = a.v_remote;
          off = (size_t)(-(src + 1)) * a.ld_remote + hoff + c0;
        }
#pragma unroll
        for (int d = 0; d < kDPT; ++d) {
          sK[kj * kPad + c0 + d] = ld_elem<BF16>(kb, off + d);
          sV[kj * kPad + c0 + d] = ld_elem<BF16>(vb, off + d);
        }
        if ((tid & 3) == 0) sKpos[kj] = a.key_pos[k0 + j];
      } else if ((tid & 3) == 0) {
        sKpos[kj] = INT_MAX;  // padding key: never visible
      }
    }
    __syncthreads();
    // ---- scores for keys part + 4i
    float s[16];
    float tmax = -INFINITY;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int kj = part + 4 * i;
      const int kp = sKpos[kj];
      const bool vis = (kt + kj < nk) && (!a.causal || kp <= qpos) && kp != INT_MAX;
      float dot = 0.f;
#pragma unroll
      for (int d = 0; d < kDH; ++d) dot = fmaf(q[d], sK[kj * kPad + d], dot);
      s[i] = vis ? dot * a.scale : -INFINITY;
      tmax = fmaxf(tmax, s[i]);
    }
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
    const float mnew = fmaxf(m, tmax);
    const float corr = (m == -INFINITY) ? 0.f : expf(m - mnew);
    float lsum = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const float p = (s[i] == -INFINITY) ? 0.f : expf(s[i] - mnew);
      sP[r * (kAK + 1) + part + 4 * i] = p;
      lsum += p;
    }
    l = l * corr + lsum;
    m = mnew;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kDPT; ++i) acc[i] *= corr;
    for (int kj = 0; kj < kAK; ++kj) {
      const float p = sP[r * (kAK + 1) + kj];
#pragma unroll
      for (int i = 0; i < kDPT; ++i) acc[i] = fmaf(p, sV[kj * kPad + part + 4 * i], acc[i]);
    }
    __syncthreads();
  }
  l += __shfl_xor_sync(0xffffffffu, l, 1);
  l += __shfl_xor_sync(0xffffffffu, l, 2);
  if (!qvalid) return;
  const float inv = 1.0f / l;
  const size_t ob = (size_t)(q0 + qi) * a.ld_out + hoff;
#pragma unroll
  for (int i = 0; i < kDPT; ++i) {
    const float o = acc[i] * inv;
    const int d = part + 4 * i;
    if (a.out_f32) a.out_f32[ob + d] = o;
    if (a.out_hi) {
      __nv_bfloat16 hi, lo;
      split_bf16(o, hi, lo);
      a.out_hi[ob + d] = hi;
      if (a.out_lo) a.out_lo[ob + d] = lo;
    }
  }
}

template <int DH>
static int launch_attn(const AttnArgs& a, dim3 grid, cudaStream_t st) {
  constexpr int smem = 2 * kAK * (DH + 1) * 4 + kAQ * (kAK + 1) * 4 + kAK * 4;
  static bool configured = false;
  if (!configured) {
    ASTRA_CUDA_CHECK(cudaFuncSetAttribute(attention_simt_kernel<true, DH>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    ASTRA_CUDA_CHECK(cudaFuncSetAttribute(attention_simt_kernel<false, DH>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  if (a.in_bf16)
    attention_simt_kernel<true, DH><<<grid, 256, smem, st>>>(a);
  else
    attention_simt_kernel<false, DH><<<grid, 256, smem, st>>>(a);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

}  // namespace astra

using namespace astra;

extern "C" int astra_attention(const void* q, int ldq, const void* k_local, const void* v_local,
                               int ld_local, const void* k_remote, const void* v_remote,
                               int ld_remote, const int32_t* key_src, const int32_t* key_pos,
                               const int32_t* segs, int num_segs, int max_nq, int heads,
                               int head_dim, int causal, int in_bf16, float scale, float* out_f32,
                               void* out_hi, void* out_lo, int ld_out, void* stream) {
  ASTRA_REQUIRE(head_dim == 8 || head_dim == 16 || head_dim == 32 || head_dim == 64 ||
                    head_dim == 128,
                ASTRA_ERR_SHAPE, "attention: head_dim %d unsupported", head_dim);
  ASTRA_REQUIRE(heads >= 1 && num_segs >= 0 && max_nq >= 0, ASTRA_ERR_SHAPE, "attention: bad shape");
  if (num_segs == 0 || max_nq == 0) return ASTRA_OK;
  AttnArgs a{q,       ldq,     k_local, v_local, ld_local, k_remote, v_remote, ld_remote,
             key_src, key_pos, segs,    num_segs, heads,   head_dim, causal,   in_bf16,
             scale,   out_f32, reinterpret_cast<__nv_bfloat16*>(out_hi),
             reinterpret_cast<__nv_bfloat16*>(out_lo), ld_out};
  dim3 grid(num_segs, heads, (max_nq + kAQ - 1) / kAQ);
  cudaStream_t st = as_stream(stream);
  int rc = ASTRA_OK;
  switch (head_dim) {
    case 8: rc = launch_attn<8>(a, grid, st); break;
    case 16: rc = launch_attn<16>(a, grid, st); break;
    case 32: rc = launch_attn<32>(a, grid, st); break;
    case 64: rc = launch_attn<64>(a, grid, st); break;
    default: rc = launch_attn<128>(a, grid, st); break;
  }
  if (rc) return rc;
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}
