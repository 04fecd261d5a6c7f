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
#include <cmath>
#include <vector>

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
  const uint8_t* mask;  // optional dense mask [rows, mask_ld] indexed by (q0 + qi, key)
  int mask_ld;
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
      } else {
        // padding key: never visible, and zeroed so 0-weight * stale smem cannot make a NaN
#pragma unroll
        for (int d = 0; d < kDPT; ++d) {
          sK[kj * kPad + c0 + d] = 0.f;
          sV[kj * kPad + c0 + d] = 0.f;
        }
        if ((tid & 3) == 0) sKpos[kj] = INT_MAX;
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
      bool vis = (kt + kj < nk) && (!a.causal || kp <= qpos) && kp != INT_MAX;
      if (a.mask && vis) vis = a.mask[(size_t)(q0 + (qvalid ? qi : 0)) * a.mask_ld + kt + kj] != 0;
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

// ----------------------------------------------------------------------------------------
// tcgen05 flash attention (bf16 fast path, head_dim 64).  One CTA (4 warps) per
// (segment, head, 128-query tile); keys stream in chunks of 128:
//   S = Q K^T on the tensor core (M=128, N=128, K=64) into TMEM,
//   softmax in registers (thread = query row, tcgen05.ld of its TMEM lane),
//   P (bf16) written to shared memory in the UMMA K-major SW128 layout,
//   O_chunk = P V on the tensor core (M=128, N=64, K=128; V used MN-major as stored),
//   online-softmax rescale of the running output in registers.
// K/V rows are gathered with cp.async through key_src, which fuses the VQ decode
// (codebook K/V table rows) into the tile load.
constexpr int kTQ = 128, kTK = 128;
static bool g_force_simt_attention = false;  // test hook (astra_attention_force_simt)
// 16 KB Q + 2 x (16 KB K + 16 KB V) + 32 KB P + 2 x 128 int16 key positions + barrier:
// 115,264 B, so two CTAs (and their 2 x 256 TMEM columns) share an SM.  The dynamic smem base
// is 1024-byte aligned (checked at run time), as the SW128 layouts require.
constexpr int kTcSmem = 16384 + 2 * 32768 + 32768 + 2 * 256 + 64;
constexpr short kPosNever = 0x7FFF;  // padding key: never visible

__host__ __device__ constexpr uint32_t idesc_bf16_f32_bmn(uint32_t M, uint32_t N) {
  return idesc_bf16_f32(M, N) | (1u << 16);  // B operand MN-major
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Issue the cp.async gather of key chunk [kc, kc+128) into (sK, sV) and its positions.
// Key descriptor of key `key` of the segment (loaded ahead of use: src < 0 marks a remote
// (codebook-table) row, INT_MIN a padding key).
struct KeyRef {
  int src;
  short pos;
};
__device__ __forceinline__ KeyRef attn_key_ref(const AttnArgs& a, int k0, int nk, int key) {
  KeyRef r;
  if (key < nk) {
    r.src = __ldg(a.key_src + k0 + key);
    r.pos = a.causal ? (short)__ldg(a.key_pos + k0 + key) : (short)0;
  } else {
    r.src = INT_MIN;
    r.pos = kPosNever;
  }
  return r;
}

// Issue the cp.async gather of one key row per thread (2 x 8 16-byte copies) into the chunk
// buffers (sK, sV) and record its position; padding keys are zero-filled.
__device__ __forceinline__ void attn_load_chunk(const AttnArgs& a, KeyRef kr, int hoff,
                                                uint32_t k_s, uint32_t v_s, uint8_t* sK,
                                                uint8_t* sV, short* kpos, int tid) {
  if (kr.src != INT_MIN) {
    const __nv_bfloat16 *kp, *vp;
    if (kr.src >= 0) {
      kp = reinterpret_cast<const __nv_bfloat16*>(a.k_local) + (size_t)kr.src * a.ld_local + hoff;
      vp = reinterpret_cast<const __nv_bfloat16*>(a.v_local) + (size_t)kr.src * a.ld_local + hoff;
    } else {
      kp = reinterpret_cast<const __nv_bfloat16*>(a.k_remote) +
           (size_t)(-(kr.src + 1)) * a.ld_remote + hoff;
      vp = reinterpret_cast<const __nv_bfloat16*>(a.v_remote) +
           (size_t)(-(kr.src + 1)) * a.ld_remote + hoff;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      cp_async16(k_s + sw128_offset(tid, c), kp + c * 8);
      cp_async16(v_s + sw128_offset(tid, c), vp + c * 8);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      *reinterpret_cast<uint4*>(sK + sw128_offset(tid, c)) = make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(sV + sw128_offset(tid, c)) = make_uint4(0, 0, 0, 0);
    }
  }
  kpos[tid] = kr.pos;
}

__global__ void __launch_bounds__(128) attention_tc_kernel(AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw;
  if (smem_u32(sm) & 1023) __trap();      // SW128 tiles need a 1024-byte aligned base
  uint8_t* sQ = sm;                       // 16 KB
  uint8_t* sK0 = sm + 16384;              // 2 x 16 KB
  uint8_t* sV0 = sm + 16384 + 32768;      // 2 x 16 KB
  uint8_t* sP = sm + 16384 + 65536;       // 32 KB
  short* sKpos = reinterpret_cast<short*>(sm + 16384 + 98304);   // 2 x 128
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 16384 + 98304 + 512);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);

  const int seg = blockIdx.x, h = blockIdx.y, qt = blockIdx.z;
  const int* sg = a.segs + seg * 6;
  const int q0 = sg[0], nq = sg[1], qpos0 = sg[2], ncontent = sg[3], k0 = sg[4], nk = sg[5];
  if (qt * kTQ >= nq) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hoff = h * 64;
  const __nv_bfloat16* Q = reinterpret_cast<const __nv_bfloat16*>(a.q);

  if (warp == 0) tmem_alloc<256>(tslot);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  const uint32_t q_s = smem_u32(sQ), p_s = smem_u32(sP);
  // key descriptors of the first two chunks: loads issued now, consumed after the Q copies
  const KeyRef kr0 = attn_key_ref(a, k0, nk, tid);
  const KeyRef kr1 = attn_key_ref(a, k0, nk, kTK + tid);
  // prologue: group 0 = Q + key chunk 0, group 1 = key chunk 1
  {
    const int qr = qt * kTQ + tid;  // one query row per thread
    if (qr < nq) {
      const __nv_bfloat16* qp = Q + (size_t)(q0 + qr) * a.ldq + hoff;
#pragma unroll
      for (int c = 0; c < 8; ++c) cp_async16(q_s + sw128_offset(tid, c), qp + c * 8);
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(sQ + sw128_offset(tid, c)) = make_uint4(0, 0, 0, 0);
    }
  }
  const int nchunks = (nk + kTK - 1) / kTK;
  attn_load_chunk(a, kr0, hoff, smem_u32(sK0), smem_u32(sV0), sK0, sV0, sKpos, tid);
  cp_async_commit();
  if (nchunks > 1)
    attn_load_chunk(a, kr1, hoff, smem_u32(sK0 + 16384), smem_u32(sV0 + 16384), sK0 + 16384,
                    sV0 + 16384, sKpos + 128, tid);
  cp_async_commit();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 128;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;

  const int r = warp * 32 + lane;
  const int qi = qt * kTQ + r;
  const int qpos = qi < ncontent ? qpos0 + qi : 0x7FFE;  // replica / pad queries see all keys
  const float sl2 = a.scale * 1.4426950408889634f;  // exp(x) = exp2(x * log2 e)
  float m = -INFINITY, l = 0.f;
  float o[64];
#pragma unroll
  for (int d = 0; d < 64; ++d) o[d] = 0.f;
  uint32_t phase = 0;

  for (int c = 0; c < nchunks; ++c) {
    const int buf = c & 1, kc = c * kTK;
    uint8_t* sK = sK0 + buf * 16384;
    uint8_t* sV = sV0 + buf * 16384;
    const short* kpos = sKpos + buf * 128;
    cp_async_wait_group<1>();   // this chunk's group has landed (the next may be in flight)
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_f16(tS, sdesc_kmajor_sw128(q_s + kk * 32), sdesc_kmajor_sw128(smem_u32(sK) + kk * 32),
                 idesc_bf16_f32(128, 128), kk > 0 ? 1u : 0u);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();

    // ---- softmax of row r over this chunk, branch-free: a 32-bit visibility mask per
    // 32-column group (non-causal: only the chunk tail; causal: key_pos <= query position,
    // replica keys have position -1) turns masked scores into -inf, so max and exp2 need no
    // control flow and masked weights come out exactly 0.
    const int valid = min(kTK, nk - kc);
    uint32_t vm[4];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int left = valid - cc * 32;
      uint32_t m32 = left >= 32 ? 0xffffffffu : (left <= 0 ? 0u : ((1u << left) - 1u));
      if (a.causal && m32) {
        uint32_t c32 = 0;
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const short2 kp2 = *reinterpret_cast<const short2*>(kpos + cc * 32 + j);
          c32 |= (uint32_t)(kp2.x <= qpos) << j;
          c32 |= (uint32_t)(kp2.y <= qpos) << (j + 1);
        }
        m32 &= c32;
      }
      vm[cc] = m32;
    }
    const int ngroups = (valid + 31) >> 5;
    float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      if (cc < ngroups) {
        uint32_t rr[32];
        tmem_ld32(tS + lane_off + cc * 32, rr);
        tmem_ld_wait();
        const uint32_t m32 = vm[cc];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float x = ((m32 >> j) & 1u) ? __uint_as_float(rr[j]) : -INFINITY;
          mx[j & 3] = fmaxf(mx[j & 3], x);
        }
      }
    }
    const float cmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
    const float mnew = fmaxf(m, cmax * sl2);
    const float corr = (m == -INFINITY) ? 0.f : ex2_approx(m - mnew);
    const float mref = (mnew == -INFINITY) ? 0.f : mnew;  // fully masked so far: all p = 0
    float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t pk[16];
      if (cc < ngroups) {
        uint32_t rr[32];
        tmem_ld32(tS + lane_off + cc * 32, rr);
        tmem_ld_wait();
        const uint32_t m32 = vm[cc];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float x0 = ((m32 >> j) & 1u) ? __uint_as_float(rr[j]) : -INFINITY;
          const float x1 = ((m32 >> (j + 1)) & 1u) ? __uint_as_float(rr[j + 1]) : -INFINITY;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(ex2_approx(fmaf(x0, sl2, -mref)),
                                                    ex2_approx(fmaf(x1, sl2, -mref)));
          // sum what the tensor core multiplies (the bf16-rounded probabilities)
          ls[(j >> 1) & 3] += __low2float(b2) + __high2float(b2);
          pk[j >> 1] = *reinterpret_cast<uint32_t*>(&b2);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = 0u;
      }
      const int col0 = cc * 32;
      uint8_t* blk = sP + (col0 >> 6) * 16384;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int chunk = ((col0 & 63) >> 3) + q;
        *reinterpret_cast<uint4*>(blk + sw128_offset(r, chunk)) =
            make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
      }
    }
    l = l * corr + ((ls[0] + ls[1]) + (ls[2] + ls[3]));
    m = mnew;
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_f16(tO, sdesc_kmajor_sw128(p_s + (kk >> 2) * 16384 + (kk & 3) * 32),
                 sdesc_mnmajor_sw128(smem_u32(sV) + kk * 2048, 8192), idesc_bf16_f32_bmn(128, 64),
                 kk > 0 ? 1u : 0u);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    {
      uint32_t r0[32], r1[32];
      tmem_ld32(tO + lane_off, r0);
      tmem_ld32(tO + lane_off + 32, r1);
      tmem_ld_wait();
#pragma unroll
      for (int d = 0; d < 32; ++d) {
        o[d] = fmaf(o[d], corr, __uint_as_float(r0[d]));
        o[32 + d] = fmaf(o[32 + d], corr, __uint_as_float(r1[d]));
      }
    }
    tc_fence_before();
    __syncthreads();   // buffers of this chunk are free
    if (c + 2 < nchunks)
      attn_load_chunk(a, attn_key_ref(a, k0, nk, (c + 2) * kTK + tid), hoff, smem_u32(sK),
                      smem_u32(sV), sK, sV, sKpos + buf * 128, tid);
    cp_async_commit();
  }

  if (qi < nq) {
    const float inv = 1.0f / l;
    const size_t ob = (size_t)(q0 + qi) * a.ld_out + hoff;
    if (a.out_hi) {
#pragma unroll
      for (int d = 0; d < 64; d += 8) {
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          __nv_bfloat162 b2 = __floats2bfloat162_rn(o[d + 2 * u] * inv, o[d + 2 * u + 1] * inv);
          w[u] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(a.out_hi + ob + d) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    if (a.out_f32) {
#pragma unroll
      for (int d = 0; d < 64; ++d) a.out_f32[ob + d] = o[d] * inv;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
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
  ASTRA_REQUIRE(head_dim == 4 || head_dim == 8 || head_dim == 16 || head_dim == 32 || head_dim == 64 ||
                    head_dim == 128,
                ASTRA_ERR_SHAPE, "attention: head_dim %d unsupported", head_dim);
  ASTRA_REQUIRE(heads >= 1 && num_segs >= 0 && max_nq >= 0, ASTRA_ERR_SHAPE, "attention: bad shape");
  if (num_segs == 0 || max_nq == 0) return ASTRA_OK;
  AttnArgs a{q,       ldq,     k_local, v_local, ld_local, k_remote, v_remote, ld_remote,
             key_src, key_pos, segs,    num_segs, heads,   head_dim, causal,   in_bf16,
             scale,   out_f32, reinterpret_cast<__nv_bfloat16*>(out_hi),
             reinterpret_cast<__nv_bfloat16*>(out_lo), ld_out};
  cudaStream_t st = as_stream(stream);
  const bool aligned = (ldq % 8 == 0) && (ld_local % 8 == 0) && (ld_remote % 8 == 0) &&
                       ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k_local) |
                         reinterpret_cast<uintptr_t>(v_local) |
                         reinterpret_cast<uintptr_t>(k_remote) |
                         reinterpret_cast<uintptr_t>(v_remote)) & 15) == 0;
  if (in_bf16 && head_dim == 64 && out_lo == nullptr && aligned && !g_force_simt_attention) {
    static bool configured = false;
    if (!configured) {
      ASTRA_CUDA_CHECK(cudaFuncSetAttribute(attention_tc_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
      configured = true;
    }
    dim3 tgrid(num_segs, heads, (max_nq + kTQ - 1) / kTQ);
    attention_tc_kernel<<<tgrid, 128, kTcSmem, st>>>(a);
    ASTRA_CUDA_CHECK(cudaGetLastError());
    return ASTRA_OK;
  }
  dim3 grid(num_segs, heads, (max_nq + kAQ - 1) / kAQ);
  int rc = ASTRA_OK;
  switch (head_dim) {
    case 4: rc = launch_attn<4>(a, grid, st); break;
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

extern "C" int astra_attention_force_simt(int enable) {
  g_force_simt_attention = enable != 0;
  return ASTRA_OK;
}

// Dense-mask multi-head attention for the drop-in operator API
// (attention.multihead_attention, attention.py:50-73): one segment, fp32 in/out.
extern "C" int astra_attention_masked(const float* q, const float* k, const float* v, int R, int C,
                                      int D, int heads, const uint8_t* mask, int32_t* scratch,
                                      float* out, void* stream) {
  ASTRA_REQUIRE(heads >= 1 && D % heads == 0, ASTRA_ERR_SHAPE, "width %d not divisible by %d heads",
                D, heads);
  const int dk = D / heads;
  ASTRA_REQUIRE(dk == 4 || dk == 8 || dk == 16 || dk == 32 || dk == 64 || dk == 128, ASTRA_ERR_SHAPE,
                "attention: head_dim %d unsupported", dk);
  if (R == 0) return ASTRA_OK;
  std::vector<int32_t> h(6 + 2 * (size_t)C);
  h[0] = 0; h[1] = R; h[2] = 0; h[3] = R; h[4] = 0; h[5] = C;
  for (int j = 0; j < C; ++j) {
    h[6 + j] = j;
    h[6 + C + j] = j;
  }
  cudaStream_t st = as_stream(stream);
  ASTRA_CUDA_CHECK(cudaMemcpyAsync(scratch, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st));
  AttnArgs a{q, D, k, v, D, k, v, D, scratch + 6, scratch + 6 + C, scratch, 1, heads, dk, 0, 0,
             (float)(1.0 / sqrt((double)dk)), out, nullptr, nullptr, D, mask, C};
  dim3 grid(1, heads, (R + kAQ - 1) / kAQ);
  int rc;
  switch (dk) {
    case 4: rc = launch_attn<4>(a, grid, st); break;
    case 8: rc = launch_attn<8>(a, grid, st); break;
    case 16: rc = launch_attn<16>(a, grid, st); break;
    case 32: rc = launch_attn<32>(a, grid, st); break;
    case 64: rc = launch_attn<64>(a, grid, st); break;
    default: rc = launch_attn<128>(a, grid, st); break;
  }
  return rc;
}
