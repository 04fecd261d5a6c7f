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
#include <algorithm>
#include <climits>
#include <cstdlib>
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
  pdl_wait();
  pdl_trigger();
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
  const int hd = a.head_dim;   // <= kDH; dims hd..kDH-1 are zero padding
  const int hoff = h * hd;

  float q[kDH];
  {
    const size_t base = (size_t)(q0 + (qvalid ? qi : 0)) * a.ldq + hoff;
#pragma unroll
    for (int d = 0; d < kDH; ++d) q[d] = d < hd ? ld_elem<BF16>(a.q, base + d) : 0.f;
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
          const bool in = c0 + d < hd;
          sK[kj * kPad + c0 + d] = in ? ld_elem<BF16>(kb, off + d) : 0.f;
          sV[kj * kPad + c0 + d] = in ? ld_elem<BF16>(vb, off + d) : 0.f;
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
    if (d >= hd) continue;
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
// tcgen05 attention (bf16 fast path, head_dim 64).  One CTA (8 warps) per
// (segment, head, 128-query tile); keys stream in chunks of up to 256, so one chunk covers
// a whole ViT-B segment (197 keys) and its softmax needs no rescaling:
//   S = Q K^T        UMMA M=128, N=round16(keys in chunk), K=64      -> TMEM cols [0, 256)
//   softmax          thread = query row (its TMEM lane); the two warps of a lane quarter
//                    split the key columns and exchange row max / row sum through smem
//   P (bf16)         stored back into TMEM over the S columns it was computed from
//                    (keys 0-127 -> cols 0-63, keys 128-255 -> cols 128-191)
//   O = P V          UMMA with A read from TMEM, V used MN-major as gathered -> cols [64,128)
// S, P and O share 256 TMEM columns and ~84 KB of smem: two CTAs (16 warps) per SM.
// Segments with more than 256 keys take further chunks with the online-softmax rescale of
// the 32 output columns each thread keeps in registers.
// K/V rows are gathered with cp.async through key_src, which fuses the VQ decode (codebook
// K/V table rows) into the tile load.
constexpr int kTQ = 128, kTKC = 256, kTcThreads = 256;
static bool g_force_simt_attention = false;  // test hook (astra_attention_force_simt)
static int g_attention_variant = 0;  // 0 persistent two pipelines, 1 one CTA per tile, 2 persistent single pipeline + correction warps
// Q 16 KB + K 32 KB + V 32 KB + 256 key positions + row max / sum exchange (4 x 128 floats)
// + barrier and TMEM slot, plus 1 KB to align the base for the SW128 layouts.
constexpr int kTcSmemUsed = 16384 + 32768 + 32768 + 512 + 2048 + 64;
constexpr int kTcSmem = kTcSmemUsed + 1024;
constexpr short kPosNever = 0x7FFF;  // padding key: never visible

__host__ __device__ constexpr uint32_t idesc_bf16_f32_bmn(uint32_t M, uint32_t N) {
  return idesc_bf16_f32(M, N) | (1u << 16);  // B operand MN-major
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Key descriptor of key `key` of the segment: src < 0 marks a remote (codebook-table) row,
// INT_MIN a padding key.
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

// cp.async gather of one key row (its K and V head slices, 2 x 8 16-byte copies) into row
// `row` of the SW128 chunk buffers; padding keys are zero-filled (P is 0 there, and 0 * a
// stale NaN would not be).
__device__ __forceinline__ void attn_load_key(const AttnArgs& a, KeyRef kr, int hoff, int row,
                                              uint8_t* sK, uint8_t* sV, short* kpos) {
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
    const uint32_t k_s = smem_u32(sK), v_s = smem_u32(sV);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      cp_async16(k_s + sw128_offset(row, c), kp + c * 8);
      cp_async16(v_s + sw128_offset(row, c), vp + c * 8);
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      *reinterpret_cast<uint4*>(sK + sw128_offset(row, c)) = make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(sV + sw128_offset(row, c)) = make_uint4(0, 0, 0, 0);
    }
  }
  kpos[row] = kr.pos;
}

// Visibility bits of the 32 key columns [col0, col0 + 32) of the chunk for a query at
// position qpos: the chunk tail (non-causal) or key_pos <= qpos (causal; replica keys have
// position -1, replica / padding queries see everything).
__device__ __forceinline__ uint32_t attn_vis32(const short* kpos, int col0, int valid, int qpos,
                                               int causal) {
  const int left = valid - col0;
  uint32_t m32 = left >= 32 ? 0xffffffffu : (left <= 0 ? 0u : ((1u << left) - 1u));
  if (causal && m32) {
    uint32_t c32 = 0;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const short2 kp2 = *reinterpret_cast<const short2*>(kpos + col0 + j);
      c32 |= (uint32_t)(kp2.x <= qpos) << j;
      c32 |= (uint32_t)(kp2.y <= qpos) << (j + 1);
    }
    m32 &= c32;
  }
  return m32;
}

__global__ void __launch_bounds__(kTcThreads, 2) attention_tc_kernel(AttnArgs a) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* sQ = sm;                        // 16 KB: 128 query rows x 64 dims, SW128
  uint8_t* sK = sm + 16384;                // 32 KB: 256 key rows
  uint8_t* sV = sm + 16384 + 32768;        // 32 KB
  short* sKpos = reinterpret_cast<short*>(sm + 81920);
  float* sRed = reinterpret_cast<float*>(sm + 81920 + 512);   // [max | sum][half][128 rows]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 81920 + 512 + 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);

  const int seg = blockIdx.x, h = blockIdx.y, qt = blockIdx.z;
  const int* sg = a.segs + seg * 6;
  const int q0 = sg[0], nq = sg[1], qpos0 = sg[2], ncontent = sg[3], k0 = sg[4], nk = sg[5];
  if (qt * kTQ >= nq) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int hoff = h * 64;

  if (warp == 0) tmem_alloc<256>(tslot);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  // Q tile: thread -> row tid/2, four of its eight 16-byte chunks
  {
    const int row = tid >> 1, c0 = (tid & 1) * 4, qr = qt * kTQ + row;
    const uint32_t q_s = smem_u32(sQ);
    if (qr < nq) {
      const __nv_bfloat16* qp =
          reinterpret_cast<const __nv_bfloat16*>(a.q) + (size_t)(q0 + qr) * a.ldq + hoff;
#pragma unroll
      for (int c = 0; c < 4; ++c) cp_async16(q_s + sw128_offset(row, c0 + c), qp + (c0 + c) * 8);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4*>(sQ + sw128_offset(row, c0 + c)) = make_uint4(0, 0, 0, 0);
    }
  }

  const int row = quarter * 32 + lane;             // this thread's query row = TMEM lane
  const int qi = qt * kTQ + row;
  const bool warp_rows = qt * kTQ + quarter * 32 < nq;   // warp-uniform: any valid row
  const int qpos = qi < ncontent ? qpos0 + qi : 0x7FFE;  // replica / pad queries see all keys
  const float sl2 = a.scale * 1.4426950408889634f;       // exp(x) = exp2(x * log2 e)
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  float m_run = -INFINITY, l_half = 0.f;
  float o[32];
#pragma unroll
  for (int d = 0; d < 32; ++d) o[d] = 0.f;
  tc_fence_before();
  __syncthreads();   // TMEM address and barrier init visible to all
  tc_fence_after();
  pdl_trigger();   // after the TMEM allocation (ptx.cuh)
  const uint32_t tmem = *tslot, tS = tmem, tO = tmem + 64;
  uint32_t phase = 0;

  const int nchunks = (nk + kTKC - 1) / kTKC;
  for (int c = 0; c < nchunks; ++c) {
    const int kc = c * kTKC;
    const int valid = min(kTKC, nk - kc);
    const int ncols = (valid + 15) & ~15;
    if (tid < ncols) attn_load_key(a, attn_key_ref(a, k0, nk, kc + tid), hoff, tid, sK, sV, sKpos);
    cp_async_commit();
    cp_async_wait_group<0>();
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_f16(tS, sdesc_kmajor_sw128(smem_u32(sQ) + kk * 32),
                 sdesc_kmajor_sw128(smem_u32(sK) + kk * 32), idesc_bf16_f32(128, ncols),
                 kk > 0 ? 1u : 0u);
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();

    // ---- pass 1: row max over this warp's half of the columns (masked scores -> -inf)
    float mx = -INFINITY;
    if (warp_rows) {
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {
        const int g = half * 4 + gg;
        if (g * 32 < valid) {
          uint32_t rr[32];
          tmem_ld32(tS + lane_off + g * 32, rr);
          const uint32_t m32 = attn_vis32(sKpos, g * 32, valid, qpos, a.causal);
          tmem_ld_wait();
          float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int j = 0; j < 32; ++j)
            m4[j & 3] = fmaxf(m4[j & 3], ((m32 >> j) & 1u) ? __uint_as_float(rr[j]) : -INFINITY);
          mx = fmaxf(mx, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])));
        }
      }
    }
    sRed[half * 128 + row] = mx;
    __syncthreads();
    const float cmax = fmaxf(sRed[row], sRed[128 + row]);
    const float mnew = fmaxf(m_run, cmax * sl2);
    const float corr = (m_run == -INFINITY) ? 0.f : ex2_approx(m_run - mnew);
    const float mref = (mnew == -INFINITY) ? 0.f : mnew;  // fully masked so far: all p = 0

    // ---- pass 2: p = exp2(s * scale * log2e - m) as bf16, summed as rounded, stored into TMEM
    float ls[4] = {0.f, 0.f, 0.f, 0.f};
    if (warp_rows) {
#pragma unroll
      for (int gg = 0; gg < 4; ++gg) {
        const int g = half * 4 + gg;
        if (g * 32 < valid) {
          uint32_t rr[32], pk[16];
          tmem_ld32(tS + lane_off + g * 32, rr);
          const uint32_t m32 = attn_vis32(sKpos, g * 32, valid, qpos, a.causal);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float x0 = ((m32 >> j) & 1u) ? __uint_as_float(rr[j]) : -INFINITY;
            const float x1 = ((m32 >> (j + 1)) & 1u) ? __uint_as_float(rr[j + 1]) : -INFINITY;
            __nv_bfloat162 b2 = __floats2bfloat162_rn(ex2_approx(fmaf(x0, sl2, -mref)),
                                                      ex2_approx(fmaf(x1, sl2, -mref)));
            ls[(j >> 1) & 3] += __low2float(b2) + __high2float(b2);
            pk[j >> 1] = *reinterpret_cast<uint32_t*>(&b2);
          }
          // keys 0-127 -> P cols 0-63, keys 128-255 -> P cols 128-191: every column written
          // here was already read by this thread (same or an earlier group)
          const int pcol = g < 4 ? g * 16 : 128 + (g - 4) * 16;
          tmem_st16(tS + lane_off + pcol, pk);
        }
      }
      tmem_st_wait();
    }
    l_half = l_half * corr + ((ls[0] + ls[1]) + (ls[2] + ls[3]));
    m_run = mnew;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      const int ksteps = ncols >> 4;
      for (int kk = 0; kk < ksteps; ++kk) {
        const uint32_t acol = kk < 8 ? kk * 8 : 128 + (kk - 8) * 8;
        umma_f16_ts(tO, tS + acol, sdesc_mnmajor_sw128(smem_u32(sV) + kk * 2048, 8192),
                    idesc_bf16_f32_bmn(128, 64), kk > 0 ? 1u : 0u);
      }
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    if (warp_rows) {
      uint32_t r0[32];
      tmem_ld32(tO + lane_off + half * 32, r0);
      tmem_ld_wait();
#pragma unroll
      for (int d = 0; d < 32; ++d) o[d] = fmaf(o[d], corr, __uint_as_float(r0[d]));
    }
    tc_fence_before();
    __syncthreads();   // K/V buffers and TMEM columns are free for the next chunk
  }

  sRed[256 + half * 128 + row] = l_half;
  __syncthreads();
  if (qi < nq) {
    const float inv = 1.0f / (sRed[256 + row] + sRed[384 + row]);
    const size_t ob = (size_t)(q0 + qi) * a.ld_out + hoff + half * 32;
    if (a.out_hi) {
#pragma unroll
      for (int d = 0; d < 32; d += 8) {
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
      for (int d = 0; d < 32; ++d) a.out_f32[ob + d] = o[d] * inv;
    }
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<256>(tmem);
  }
}

// ----------------------------------------------------------------------------------------
// Persistent form of the same computation (the default tcgen05 path): one CTA per SM runs TWO
// independent attention pipelines side by side, so one's softmax hides the other's MMA and
// gather latencies.  Pipeline w (w = 0, 1) owns smem stage w, TMEM slot w (256 columns) and
// the items t = blockIdx.x + (2k + w) * gridDim.x — (segment, head, 128-query tile) — taken
// 256 keys ("chunk") at a time:
//   warps 4w..4w+3   softmax: thread = query row = TMEM lane, all key columns of its row
//                    (no cross-warp exchange): pass 1 row max, pass 2 P = exp2(...) as bf16
//                    written back into TMEM over the S columns it was computed from, then
//                    O(chunk) = P V read back into registers with the online-softmax rescale;
//                    the item's last chunk normalises and stores
//   warp 8 + w       producer: TMA gather4 of 4 rows per instruction (SW128 applied by smem
//                    address) — Q rows clamped into the segment, K/V rows through key_src
//                    (local rows of the projection buffer or codebook-table rows: the fused
//                    VQ decode); per-thread cp.async would top out at the SM's outstanding-
//                    miss limit (~16 KB in flight), the TMA engine does not
//   warp 10 + w      MMA issuer (one thread): S = Q K^T into the slot, O = P V with A = P
//                    read from TMEM, into columns [128, 192) of the slot
constexpr int kPThreads = 384;
constexpr int kPStageBytes = 16384 + 32768 + 32768;     // Q, K, V of one chunk
constexpr int kPSmemUsed = 2 * kPStageBytes + 2 * 2 * 256 * 4 + 512 + 384 * 32 + 2 * 16384;
constexpr int kPSmem = kPSmemUsed + 1024;

// Debug timeline (astra_attention_trace): CTA 0 records globaltimer stamps per chunk.
__device__ long long* g_attn_trace = nullptr;
__device__ int g_attn_pipe_delay = 0;   // ns: pipeline 1 starts this late (ASTRA_ATTN_PIPE_DELAY)
__device__ __forceinline__ void p_trace(long long* tr, int slot, uint32_t u) {
  if (tr != nullptr && u < 32) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[u * 16 + slot] = t;
  }
}

struct PBars {   // per pipeline
  uint64_t qk_full, v_full, qk_empty, v_empty, s_full, p_full, o_full, t_empty, kp_full[2];
};
struct PMaps {
  CUtensorMap q;             // box {64, 128}: a query tile
  CUtensorMap kl, vl, kr, vr;   // box {64, 1}: gather4 / single rows (local, codebook table)
  CUtensorMap kl16, vl16;    // box {64, 16}: runs of consecutive local keys
};

// Item table: at kernel start the CTA decodes its items t = blockIdx.x + i * gridDim.x —
// (segment, head, 128-query tile) with the q-tile fastest (concurrent CTAs share a segment's
// K/V in L2) — into shared memory, so the roles' per-item bookkeeping never waits on a global
// load.  Item i belongs to pipeline i % 2; items past the table capacity are decoded from
// global memory.
constexpr int kPItemCap = 384;
struct PItem {
  int q0, nq, qpos0, ncontent, k0, nk, h, qt;
};
struct PUnit {
  int q0, nq, qpos0, ncontent, k0, nk, h, qt, kc, cs;   // cs: keys per chunk
  bool ok;
};
__device__ __forceinline__ PItem p_decode(const AttnArgs& a, int qtiles, int t) {
  PItem r;
  r.qt = t % qtiles;
  r.h = (t / qtiles) % a.heads;
  const int* sg = a.segs + (t / qtiles / a.heads) * 6;
  r.q0 = __ldg(sg);
  r.nq = __ldg(sg + 1);
  r.qpos0 = __ldg(sg + 2);
  r.ncontent = __ldg(sg + 3);
  r.k0 = __ldg(sg + 4);
  r.nk = __ldg(sg + 5);
  return r;
}
struct PIter {
  int i, n_items, qtiles, step = 2, cs = kTKC;
  const PItem* table;
  PUnit cur;
  __device__ __forceinline__ void next_item(const AttnArgs& a) {
    cur.ok = false;
    for (; i < n_items; i += step) {
      const PItem e = i < kPItemCap ? table[i] : p_decode(a, qtiles, blockIdx.x + i * gridDim.x);
      if (e.qt * kTQ < e.nq && e.nk > 0) {
        cur.q0 = e.q0;
        cur.nq = e.nq;
        cur.qpos0 = e.qpos0;
        cur.ncontent = e.ncontent;
        cur.k0 = e.k0;
        cur.nk = e.nk;
        if (a.causal == 2) {   // prefix keys (key j at position j): later keys are invisible
          const int last = min(e.nq, (e.qt + 1) * kTQ) - 1;
          if (last < e.ncontent) cur.nk = min(e.nk, e.qpos0 + last + 1);
        }
        cur.h = e.h;
        cur.qt = e.qt;
        cur.kc = 0;
        cur.cs = cs;
        cur.ok = true;
        i += step;
        return;
      }
    }
  }
  __device__ __forceinline__ void init(const AttnArgs& a, int qt_, int pipe, const PItem* tab,
                                       int n) {
    qtiles = qt_;
    table = tab;
    n_items = n;
    i = pipe;
    next_item(a);
  }
  __device__ __forceinline__ void advance(const AttnArgs& a) {
    if (!cur.ok) return;
    cur.kc += cs;
    if (cur.kc >= cur.nk) next_item(a);
  }
};

// key_src of the 16 key rows 16*lane .. 16*lane+15 of a chunk (lanes 0-15).  Rows past the
// chunk end (inside its last 16-key MMA step) continue a local run (rows of the next segment,
// or zero-filled past the buffer) or repeat the last codebook row: finite data that P = 0
// multiplies away.
__device__ __forceinline__ void p_fetch_rows(const AttnArgs& a, const PUnit& un, int lane,
                                             int (&r)[16]) {
  const int valid = min(un.cs, un.nk - un.kc);
  const int32_t* ks = a.key_src + un.k0 + un.kc;
  const int last = __ldg(ks + valid - 1);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int j = 16 * lane + i;
    r[i] = j < valid ? __ldg(ks + j) : (last >= 0 ? last + (j - valid + 1) : last);
  }
}

// Gather this lane's 16 key rows (K or V) into `dst`: one 16-row box when they are a run of
// consecutive local rows (N = 1: every group), else a TMA gather4 per 4 rows from one source,
// else single rows.
template <bool kV>
__device__ __forceinline__ void p_gather_keys(const PMaps& mp, const PUnit& un, const int (&r)[16],
                                              uint8_t* dst, uint64_t* bar, int lane) {
  const int ncols = (min(un.cs, un.nk - un.kc) + 15) & ~15;
  if (16 * lane >= ncols) return;
  const int col = un.h * 64;
  uint8_t* d = dst + lane * 2048;
  bool run = r[0] >= 0;
#pragma unroll
  for (int i = 1; i < 16; ++i) run &= r[i] == r[0] + i;
  if (run) {
    tma_load_2d(d, kV ? &mp.vl16 : &mp.kl16, bar, col, r[0], kEvictNormal);
    return;
  }
  const CUtensorMap* ml = kV ? &mp.vl : &mp.kl;
  const CUtensorMap* mr = kV ? &mp.vr : &mp.kr;
#pragma unroll
  for (int qd = 0; qd < 4; ++qd) {
    const int* q = r + 4 * qd;
    const bool all_local = (q[0] >= 0) & (q[1] >= 0) & (q[2] >= 0) & (q[3] >= 0);
    const bool all_remote = (q[0] < 0) & (q[1] < 0) & (q[2] < 0) & (q[3] < 0);
    if (all_local) {
      tma_gather4(d + qd * 512, ml, bar, col, q[0], q[1], q[2], q[3]);
    } else if (all_remote) {
      tma_gather4(d + qd * 512, mr, bar, col, -(q[0] + 1), -(q[1] + 1), -(q[2] + 1), -(q[3] + 1));
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        tma_load_2d(d + qd * 512 + i * 128, q[i] >= 0 ? ml : mr, bar, col,
                    q[i] >= 0 ? q[i] : -(q[i] + 1), kEvictNormal);
    }
  }
}

// Producer warp of one pipeline: Q + K of chunk n once S(n-1) retired, V once O(n-1) retired.
template <bool kCausal>
__device__ __forceinline__ void p_producer(const AttnArgs& a, const PMaps& mp, int qtiles, int pipe,
                                           const PItem* items, int n_items, uint8_t* st,
                                           int* kpos2, PBars* b, int lane, long long* trace) {
  PIter it;
  it.init(a, qtiles, pipe, items, n_items);
  if (pipe == 1 && g_attn_pipe_delay > 0) __nanosleep(g_attn_pipe_delay);
  for (uint32_t n = 0; it.cur.ok; ++n, it.advance(a)) {
    const PUnit un = it.cur;
    const uint32_t ph = n & 1;
    const int valid = min(kTKC, un.nk - un.kc), ncols = (valid + 15) & ~15;
    int rows[16];   // this lane's key rows, loaded before the stage wait (latency hidden)
    if (lane < 16) p_fetch_rows(a, un, lane, rows);
    int kpv[8];
    if (kCausal) {
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int j = lane + 32 * m;
        kpv[m] = j < valid ? __ldg(a.key_pos + un.k0 + un.kc + j) : 0x7FFFFFFF;
      }
    }
    mbar_wait_spin(&b->qk_empty, ph ^ 1);
    if (lane == 0) p_trace(trace, 6 + pipe * 8, n);
    if (kCausal) {
      // key positions (plain stores + release arrive).  Buffer n%2 was last read by the
      // softmax of chunk n-2, which ended before S(n-1) (just retired) was issued.
      int* kp = kpos2 + (n & 1) * 256;
#pragma unroll
      for (int m = 0; m < 8; ++m) kp[lane + 32 * m] = kpv[m];
      __syncwarp();
      if (lane == 0) mbar_arrive(&b->kp_full[n & 1]);
    }
    if (lane == 0) mbar_arrive_expect_tx(&b->qk_full, (128 + ncols) * 128);
    __syncwarp();
    // Q: one 128-row box (rows past nq belong to the next segment or are zero-filled past the
    // buffer; they are computed and never stored)
    if (lane == 16) tma_load_2d(st, &mp.q, &b->qk_full, un.h * 64, un.q0 + un.qt * kTQ, kEvictNormal);
    if (lane < 16) p_gather_keys<false>(mp, un, rows, st + 16384, &b->qk_full, lane);
    if (lane == 0) p_trace(trace, 0 + pipe * 8, n);
    mbar_wait_spin(&b->v_empty, ph ^ 1);
    if (lane == 0) mbar_arrive_expect_tx(&b->v_full, ncols * 128);
    __syncwarp();
    if (lane < 16) p_gather_keys<true>(mp, un, rows, st + 16384 + 32768, &b->v_full, lane);
  }
}

// MMA issuer of one pipeline (one thread): S(n) = Q K^T, then O(n) = P V once P is in TMEM.
__device__ __forceinline__ void p_mma(const AttnArgs& a, int qtiles, int pipe, const PItem* items,
                                      int n_items, uint8_t* st, uint32_t tS, PBars* b,
                                      long long* trace) {
  PIter it;
  it.init(a, qtiles, pipe, items, n_items);
  const uint32_t q_s = smem_u32(st), k_s = q_s + 16384, v_s = k_s + 32768;
  for (uint32_t n = 0; it.cur.ok; ++n, it.advance(a)) {
    const uint32_t ph = n & 1;
    const int ncols = (min(kTKC, it.cur.nk - it.cur.kc) + 15) & ~15;
    mbar_wait_spin(&b->t_empty, ph ^ 1);   // O(n-1) read back: the slot is free
    mbar_wait_spin(&b->qk_full, ph);
    tc_fence_after();
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      umma_f16(tS, sdesc_kmajor_sw128(q_s + kk * 32), sdesc_kmajor_sw128(k_s + kk * 32),
               idesc_bf16_f32(128, ncols), kk > 0 ? 1u : 0u);
    umma_commit(&b->s_full);
    umma_commit(&b->qk_empty);
    p_trace(trace, 1 + pipe * 8, n);
    if (trace) {   // debug: when does S actually complete?
      mbar_wait_spin(&b->s_full, ph);
      p_trace(trace, 5 + pipe * 8, n);
    }
    mbar_wait_spin(&b->p_full, ph);
    mbar_wait_spin(&b->v_full, ph);
    tc_fence_after();
    // P V into two accumulators (even / odd 16-key steps, summed at read-back): the N=64 TS
    // UMMAs are issue-bound when each depends on the previous one's accumulator
    // (scripts/probes/pv_probe.cu: 13 steps 3018 -> 2304 cycles).  O_a / O_b sit on S columns
    // 128..255, all read by the softmax before it published P.
    for (int kk = 0; kk < (ncols >> 4); ++kk)
      umma_f16_ts(tS + 128 + (kk & 1) * 64, tS + kk * 8, sdesc_mnmajor_sw128(v_s + kk * 2048, 8192),
                  idesc_bf16_f32_bmn(128, 64), kk > 1 ? 1u : 0u);
    umma_commit(&b->o_full);
    umma_commit(&b->v_empty);
    p_trace(trace, 2 + pipe * 8, n);
  }
}

// Visibility bits of 32 key columns: the chunk tail (`left` keys remain) and, when causal,
// key_pos <= the query's position.
template <bool kCausal>
__device__ __forceinline__ uint32_t p_vis(const int* kpos, int left, int qpos) {
  uint32_t m32 = left >= 32 ? 0xffffffffu : ((1u << left) - 1u);
  if (kCausal) {
    uint32_t c32 = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) c32 |= (uint32_t)(kpos[j] <= qpos) << j;
    m32 &= c32;
  }
  return m32;
}

// Softmax warpgroup of one pipeline.
template <bool kCausal>
__device__ __forceinline__ void p_softmax(const AttnArgs& a, int qtiles, int pipe,
                                          const PItem* items, int n_items, uint32_t tS,
                                          const int* kpos2, PBars* b, uint8_t* ostage,
                                          int quarter, int lane, long long* trace) {
  const int row = quarter * 32 + lane;
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  const float sl2 = a.scale * 1.4426950408889634f;
  float o[64];
#pragma unroll
  for (int d = 0; d < 64; ++d) o[d] = 0.f;
  float m_run = -INFINITY, l = 0.f;
  PIter it;
  it.init(a, qtiles, pipe, items, n_items);
  for (uint32_t n = 0; it.cur.ok; ++n, it.advance(a)) {
    const PUnit un = it.cur;
    const uint32_t ph = n & 1;
    const int valid = min(kTKC, un.nk - un.kc);
    const int qi = un.qt * kTQ + row;
    const bool warp_rows = un.qt * kTQ + quarter * 32 < un.nq;
    const int qpos = qi < un.ncontent ? un.qpos0 + qi : 0x7FFE;
    const int* kpos = kpos2 + (n & 1) * 256;
    if (un.kc == 0) {
      m_run = -INFINITY;
      l = 0.f;
    }
    if (quarter == 0 && lane == 0) p_trace(trace, 7 + pipe * 8, n);
    if (kCausal) mbar_wait_spin(&b->kp_full[n & 1], (n >> 1) & 1);
    mbar_wait_spin(&b->s_full, ph);
    tc_fence_after();
    if (quarter == 0 && lane == 0) p_trace(trace, 3 + pipe * 8, n);
    float corr = 0.f, mref = 0.f, mnew = m_run;
    if (warp_rows) {
      // pass 1: row max (fully visible groups skip the mask selects)
      float mx = -INFINITY;
#pragma unroll 1
      for (int g = 0; g * 32 < valid; ++g) {
        uint32_t rr[32];
        tmem_ld32(tS + lane_off + g * 32, rr);
        const int left = valid - g * 32;
        const uint32_t m32 = p_vis<kCausal>(kpos + g * 32, left, qpos);
        tmem_ld_wait();
        float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        if (!kCausal && left >= 32) {
#pragma unroll
          for (int j = 0; j < 32; ++j) m4[j & 3] = fmaxf(m4[j & 3], __uint_as_float(rr[j]));
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            m4[j & 3] = fmaxf(m4[j & 3], ((m32 >> j) & 1u) ? __uint_as_float(rr[j]) : -INFINITY);
        }
        mx = fmaxf(mx, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])));
      }
      mnew = fmaxf(m_run, mx * sl2);
      corr = (m_run == -INFINITY) ? 0.f : ex2_approx(m_run - mnew);
      mref = (mnew == -INFINITY) ? 0.f : mnew;
      // pass 2: P = exp2(s*scale*log2e - m) in bf16, group g packed into TMEM cols 16g..16g+15
      // (already read by this thread in group g/2); packed fp32 pairs for the affine step and
      // the row sum (of the unrounded probabilities)
      const float2 sl2x2 = make_float2(sl2, sl2), nm2 = make_float2(-mref, -mref);
      float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                       make_float2(0.f, 0.f)};
#pragma unroll 1
      for (int g = 0; g * 32 < valid; ++g) {
        uint32_t rr[32], pk[16];
        tmem_ld32(tS + lane_off + g * 32, rr);
        const int left = valid - g * 32;
        const uint32_t m32 = p_vis<kCausal>(kpos + g * 32, left, qpos);
        tmem_ld_wait();
        if (!kCausal && left >= 32) {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float2 t = ffma2(make_float2(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1])),
                                   sl2x2, nm2);
            const float2 e = make_float2(ex2_approx(t.x), ex2_approx(t.y));
            pk[j >> 1] = pack_bf16x2(e.x, e.y);
            acc[(j >> 1) & 3] = fadd2(acc[(j >> 1) & 3], e);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float x0 = ((m32 >> j) & 1u) ? __uint_as_float(rr[j]) : -INFINITY;
            const float x1 = ((m32 >> (j + 1)) & 1u) ? __uint_as_float(rr[j + 1]) : -INFINITY;
            const float2 t = ffma2(make_float2(x0, x1), sl2x2, nm2);
            const float2 e = make_float2(ex2_approx(t.x), ex2_approx(t.y));
            pk[j >> 1] = pack_bf16x2(e.x, e.y);
            acc[(j >> 1) & 3] = fadd2(acc[(j >> 1) & 3], e);
          }
        }
        tmem_st16(tS + lane_off + g * 16, pk);
      }
      tmem_st_wait();
      const float2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
      l = l * corr + ((s01.x + s01.y) + (s23.x + s23.y));
    }
    m_run = mnew;
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&b->p_full);
    mbar_wait_spin(&b->o_full, ph);
    tc_fence_after();
    if (warp_rows) {
      const bool two = valid > 16;   // O_b holds the odd 16-key steps (p_mma)
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) {
        uint32_t r0[16], r1[16];
        tmem_ld16(tS + 128 + lane_off + hh * 16, r0);
        if (two) tmem_ld16(tS + 192 + lane_off + hh * 16, r1);
        tmem_ld_wait();
        // corr = 0 on an item's first chunk clears what the previous item left in o
#pragma unroll
        for (int d = 0; d < 16; ++d)
          o[hh * 16 + d] = fmaf(o[hh * 16 + d], corr,
                                two ? __uint_as_float(r0[d]) + __uint_as_float(r1[d]) : __uint_as_float(r0[d]));
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&b->t_empty);
    if (un.kc + kTKC >= un.nk && warp_rows) {
      const float inv = 1.0f / l;
      if (a.out_hi) {
        // stage the warp's 32 output rows (128 B each, 16-byte chunks XOR-swizzled by row) and
        // write them back as whole rows: 4 rows per warp instruction instead of 32 scattered
        // 16-byte pieces
        uint8_t* stg = ostage + quarter * 4096;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 w;
          w.x = pack_bf16x2(o[8 * c] * inv, o[8 * c + 1] * inv);
          w.y = pack_bf16x2(o[8 * c + 2] * inv, o[8 * c + 3] * inv);
          w.z = pack_bf16x2(o[8 * c + 4] * inv, o[8 * c + 5] * inv);
          w.w = pack_bf16x2(o[8 * c + 6] * inv, o[8 * c + 7] * inv);
          *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) = w;
        }
        __syncwarp();
        const int rbase = un.qt * kTQ + quarter * 32;
#pragma unroll
        for (int it2 = 0; it2 < 8; ++it2) {
          const int r = 4 * it2 + (lane >> 3), c = lane & 7;
          if (rbase + r < un.nq)
            *reinterpret_cast<uint4*>(a.out_hi + (size_t)(un.q0 + rbase + r) * a.ld_out + un.h * 64 + 8 * c) =
                *reinterpret_cast<const uint4*>(stg + r * 128 + ((c ^ (r & 7)) << 4));
        }
        __syncwarp();
      }
      if (a.out_f32 && qi < un.nq) {
        const size_t ob = (size_t)(un.q0 + qi) * a.ld_out + un.h * 64;
#pragma unroll
        for (int d = 0; d < 64; ++d) a.out_f32[ob + d] = o[d] * inv;
      }
    }
    if (quarter == 0 && lane == 0) p_trace(trace, 4 + pipe * 8, n);
  }
}

template <bool kCausal>
__global__ void __launch_bounds__(kPThreads, 1)
    attention_tcp_kernel(AttnArgs a, const __grid_constant__ PMaps mp, int qtiles) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  int* sKpos = reinterpret_cast<int*>(sm + 2 * kPStageBytes);          // [pipe][2][256]
  PBars* bars = reinterpret_cast<PBars*>(sKpos + 2 * 2 * 256);         // [pipe]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2);
  PItem* items = reinterpret_cast<PItem*>(sm + 2 * kPStageBytes + 2 * 2 * 256 * 4 + 512);
  uint8_t* ostage = reinterpret_cast<uint8_t*>(items + kPItemCap);   // [pipe][4 warps][4 KB]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  long long* const trace = blockIdx.x == 0 ? g_attn_trace : nullptr;   // debug timeline
  if (g_attn_trace != nullptr && tid == 0) {   // per-CTA start / end stamps
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    g_attn_trace[512 + blockIdx.x * 2] = t0;
  }

  if (tid == 0) {
    for (int w = 0; w < 2; ++w) {
      PBars* b = bars + w;
      mbar_init(&b->qk_full, 1);
      mbar_init(&b->v_full, 1);
      mbar_init(&b->qk_empty, 1);
      mbar_init(&b->v_empty, 1);
      mbar_init(&b->s_full, 1);
      mbar_init(&b->p_full, 4);
      mbar_init(&b->o_full, 1);
      mbar_init(&b->t_empty, 4);
      mbar_init(&b->kp_full[0], 1);
      mbar_init(&b->kp_full[1], 1);
    }
    fence_barrier_init();
  }
  const int total = a.num_segs * a.heads * qtiles;
  const int n_items = total > (int)blockIdx.x ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  for (int i = tid; i < min(n_items, kPItemCap); i += kPThreads)
    items[i] = p_decode(a, qtiles, blockIdx.x + i * gridDim.x);
  if (warp == 10) tmem_alloc<512>(tslot);
  if (tid == 256) {
    tma_prefetch_desc(&mp.q);
    tma_prefetch_desc(&mp.kl);
    tma_prefetch_desc(&mp.vl);
    tma_prefetch_desc(&mp.kr);
    tma_prefetch_desc(&mp.vr);
    tma_prefetch_desc(&mp.kl16);
    tma_prefetch_desc(&mp.vl16);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();   // after the TMEM allocation (ptx.cuh)
  const uint32_t tmem = *tslot;

  if (warp < 8) {
    const int pipe = warp >> 2;
    p_softmax<kCausal>(a, qtiles, pipe, items, n_items, tmem + pipe * 256, sKpos + pipe * 512,
                       bars + pipe, ostage + pipe * 16384, warp & 3, lane, trace);
  } else if (warp < 10) {
    const int pipe = warp - 8;
    p_producer<kCausal>(a, mp, qtiles, pipe, items, n_items, sm + pipe * kPStageBytes,
                        sKpos + pipe * 512, bars + pipe, lane, trace);
  } else if (lane == 0) {
    const int pipe = warp - 10;
    p_mma(a, qtiles, pipe, items, n_items, sm + pipe * kPStageBytes, tmem + pipe * 256,
          bars + pipe, trace);
  }
  tc_fence_before();
  __syncthreads();
  if (g_attn_trace != nullptr && tid == 0) {
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    g_attn_trace[512 + blockIdx.x * 2 + 1] = t1;
  }
  if (warp == 10) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ----------------------------------------------------------------------------------------
// Single-pipeline variant (astra_attention_variant 2; parity-tested, same speed as the default
// two-pipeline kernel on ViT-B/16: 37.0 vs 37.1 us per launch, 42.0 vs 41.4 inside the step).
// What bounds it (scripts/attn_trace_s.py, scripts/probes/pv_probe.cu): the P V MMAs
// (13 x 128x64x16, N = head width) cost 120-185 cycles each against a 32-cycle floor, so
// P V(u) + S(u+2) take ~1.2 us of tensor time per unit, and the softmax (MUFU-bound at
// 16 ex2/clk/SM, softmax_probe.cu) ~1.9 us.
// Warps 0..kSW-1 softmax (kSW/4 per TMEM lane quarter, interleaved 32-key groups), then four
// correction warps (one per lane quarter: O readback, o = o * corr + PV, normalise + store),
// a Q+K TMA producer, a V TMA producer and the MMA issuer.  Unit u (one 224-key chunk of one
// 128-query tile) uses smem stage and S/P slot u%2; O has its own TMEM columns.  The MMA warp
// issues S(u+2) right behind P V(u) (same slot, in-order tensor pipe), so the scores of the
// next unit are ready when the softmax of this one ends, and O(u) drains during the next
// softmax: the softmax warps (the MUFU exp2 consumers) do not wait on the tensor core.
constexpr int kSW = 8;                     // softmax warps
constexpr int kSHalves = kSW / 4;          // softmax warps per lane quarter
// TMEM columns: S/P slot 0 at 0..223, O at 224..287, S/P slot 1 at 288..511
constexpr int kSKC = 224;                  // keys per chunk
constexpr int kSOCol = 224, kSSlot1 = 288;
constexpr int kSProd = kSW + 4, kSProdV = kSW + 5, kSMma = kSW + 6;
constexpr int kSThreads = (kSW + 7) * 32;
constexpr int kSSmemUsed = 2 * kPStageBytes + 4 * 256 * 4 + 2 * 2 * 128 * 4 + 4 * 3 * 128 * 4 +
                           512 + kPItemCap * 32 + 4 * 4096;
constexpr int kSSmem = kSSmemUsed + 1024;

struct SBars {
  uint64_t qk_full[2], v_full[2], qk_empty[2], v_empty[2], s_full[2], p_full[2], o_full[2],
      t_empty[2], kp_full[4], cl_full[4];
};

__device__ __forceinline__ void softmax_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kSW * 32) : "memory");
}

// P column of 32-key group g when two warps share a lane quarter: each half owns alternate
// groups and packs a group's 32 probabilities into 16 columns of a region it already read.
__device__ __forceinline__ int p_col2(int g) {
  if (kSHalves == 1) return g << 4;
  return ((g >> 2) << 6) | ((g & 1) << 5) | (((g >> 1) & 1) << 4);
}

__device__ __forceinline__ void reg_fence32(uint32_t (&r)[32]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) asm volatile("" : "+r"(r[j]));
}

// max over the visible scores of one 32-key group
template <bool kCausal>
__device__ __forceinline__ float s_group_max(const uint32_t (&rr)[32], uint32_t m32, bool full) {
  float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  if (!kCausal && full) {
#pragma unroll
    for (int j = 0; j < 32; ++j) m4[j & 3] = fmaxf(m4[j & 3], __uint_as_float(rr[j]));
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      m4[j & 3] = fmaxf(m4[j & 3], ((m32 >> j) & 1u) ? __uint_as_float(rr[j]) : -INFINITY);
  }
  return fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
}

// P = exp2(s * scale*log2e - m) of one group, packed bf16; row sum accumulated in acc
template <bool kCausal>
__device__ __forceinline__ void s_group_exp(const uint32_t (&rr)[32], uint32_t m32, bool full,
                                            float2 sl2x2, float2 nm2, uint32_t (&pk)[16],
                                            float2 (&acc)[4]) {
  if (!kCausal && full) {
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const float2 t = ffma2(make_float2(__uint_as_float(rr[j]), __uint_as_float(rr[j + 1])),
                             sl2x2, nm2);
      const float2 e = make_float2(ex2_approx(t.x), ex2_approx(t.y));
      pk[j >> 1] = pack_bf16x2(e.x, e.y);
      acc[(j >> 1) & 3] = fadd2(acc[(j >> 1) & 3], e);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      const float x0 = ((m32 >> j) & 1u) ? __uint_as_float(rr[j]) : -INFINITY;
      const float x1 = ((m32 >> (j + 1)) & 1u) ? __uint_as_float(rr[j + 1]) : -INFINITY;
      const float2 t = ffma2(make_float2(x0, x1), sl2x2, nm2);
      const float2 e = make_float2(ex2_approx(t.x), ex2_approx(t.y));
      pk[j >> 1] = pack_bf16x2(e.x, e.y);
      acc[(j >> 1) & 3] = fadd2(acc[(j >> 1) & 3], e);
    }
  }
}

template <bool kCausal>
__global__ void __launch_bounds__(kSThreads, 1)
    attention_tcs_kernel(AttnArgs a, const __grid_constant__ PMaps mp, int qtiles) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  int* sKpos = reinterpret_cast<int*>(sm + 2 * kPStageBytes);          // [4][256]
  float* sRed = reinterpret_cast<float*>(sKpos + 4 * 256);             // [2 par][2 half][128]
  // [4 units][corr, l half 0, l half 1][128]: 4 deep, because the softmax may run up to three
  // units ahead of the correction warps (softmax(u+4) needs S(u+4) <- P V(u+2) <- O(u+1) read)
  float* sCL = sRed + 2 * 2 * 128;
  SBars* bars = reinterpret_cast<SBars*>(sCL + 4 * 3 * 128);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 1);
  PItem* items = reinterpret_cast<PItem*>(reinterpret_cast<uint8_t*>(bars) + 512);
  uint8_t* ostage = reinterpret_cast<uint8_t*>(items + kPItemCap);     // [4 warps][4 KB]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  long long* const trace = blockIdx.x == 0 ? g_attn_trace : nullptr;
  if (g_attn_trace != nullptr && tid == 0) {
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    g_attn_trace[512 + blockIdx.x * 2] = t0;
  }
  const int total = a.num_segs * a.heads * qtiles;
  const int n_items = total > (int)blockIdx.x ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  for (int i = tid; i < min(n_items, kPItemCap); i += kSThreads)
    items[i] = p_decode(a, qtiles, blockIdx.x + i * gridDim.x);
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars->qk_full[s], 1);
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->qk_empty[s], 1);
      mbar_init(&bars->v_empty[s], 1);
      mbar_init(&bars->s_full[s], 1);
      mbar_init(&bars->p_full[s], kSW);
      mbar_init(&bars->o_full[s], 1);
      mbar_init(&bars->t_empty[s], 4);
    }
    for (int s = 0; s < 4; ++s) {
      mbar_init(&bars->kp_full[s], 1);
      mbar_init(&bars->cl_full[s], kSW);
    }
    fence_barrier_init();
  }
  if (warp == kSMma) tmem_alloc<512>(tslot);
  if (tid == kSProd * 32) {
    tma_prefetch_desc(&mp.q);
    tma_prefetch_desc(&mp.kl);
    tma_prefetch_desc(&mp.vl);
    tma_prefetch_desc(&mp.kr);
    tma_prefetch_desc(&mp.vr);
    tma_prefetch_desc(&mp.kl16);
    tma_prefetch_desc(&mp.vl16);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();   // after the TMEM allocation (ptx.cuh)
  const uint32_t tmem = *tslot;
  PIter it;
  it.step = 1;
  it.cs = kSKC;
  it.init(a, qtiles, 0, items, n_items);

  if (warp == kSProd || warp == kSProdV) {
    // -------------------------------------------------------------- TMA producers (Q+K, V)
    const bool pv = warp == kSProdV;
    for (uint32_t u = 0; it.cur.ok; ++u, it.advance(a)) {
      const PUnit un = it.cur;
      const int s = u & 1;
      const uint32_t ph = (u >> 1) & 1;
      const int valid = min(kSKC, un.nk - un.kc), ncols = (valid + 15) & ~15;
      uint8_t* st = sm + s * kPStageBytes;
      int rows[16];
      if (lane < 16) p_fetch_rows(a, un, lane, rows);
      if (pv) {
        mbar_wait(&bars->v_empty[s], ph ^ 1);
        if (lane == 0) mbar_arrive_expect_tx(&bars->v_full[s], ncols * 128);
        if (lane == 0) p_trace(trace, 5, u);
        __syncwarp();
        if (lane < 16)
          p_gather_keys<true>(mp, un, rows, st + 16384 + 32768, &bars->v_full[s], lane);
        continue;
      }
      int kpv[8];
      if (kCausal) {
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const int j = lane + 32 * m;
          kpv[m] = j < valid ? __ldg(a.key_pos + un.k0 + un.kc + j) : 0x7FFFFFFF;
        }
      }
      mbar_wait(&bars->qk_empty[s], ph ^ 1);
      if (kCausal) {
        // buffer u%4 was last read by the softmax of unit u-4, which ended before S(u-2)
        // (just retired) could be issued
        int* kp = sKpos + (u & 3) * 256;
#pragma unroll
        for (int m = 0; m < 8; ++m) kp[lane + 32 * m] = kpv[m];
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->kp_full[u & 3]);
      }
      if (lane == 0) mbar_arrive_expect_tx(&bars->qk_full[s], (128 + ncols) * 128);
      __syncwarp();
      if (lane == 16)
        tma_load_2d(st, &mp.q, &bars->qk_full[s], un.h * 64, un.q0 + un.qt * kTQ, kEvictNormal);
      if (lane < 16) p_gather_keys<false>(mp, un, rows, st + 16384, &bars->qk_full[s], lane);
    }
  } else if (warp == kSMma) {
    // -------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      PIter si = it;   // S runs two units ahead of PV
      uint32_t su = 0;
      auto issue_s = [&]() {
        const int s = su & 1;
        const uint32_t ph = (su >> 1) & 1;
        const int ncols = (min(kSKC, si.cur.nk - si.cur.kc) + 15) & ~15;
        // slot s was last read by P V of unit su-2, issued (and so executed) before this
        p_trace(trace, 0, su);
        mbar_wait(&bars->qk_full[s], ph);
        tc_fence_after();
        p_trace(trace, 9, su);
        const uint32_t q_s = smem_u32(sm + s * kPStageBytes), k_s = q_s + 16384;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_f16(tmem + s * kSSlot1, sdesc_kmajor_sw128(q_s + kk * 32),
                   sdesc_kmajor_sw128(k_s + kk * 32), idesc_bf16_f32(128, ncols),
                   kk > 0 ? 1u : 0u);
        umma_commit(&bars->s_full[s]);
        umma_commit(&bars->qk_empty[s]);
        p_trace(trace, 1, su);
        ++su;
        si.advance(a);
      };
      if (si.cur.ok) issue_s();
      if (si.cur.ok) issue_s();
      for (uint32_t u = 0; it.cur.ok; ++u, it.advance(a)) {
        const int s = u & 1;
        const uint32_t ph = (u >> 1) & 1;
        const int ncols = (min(kSKC, it.cur.nk - it.cur.kc) + 15) & ~15;
        mbar_wait(&bars->p_full[s], ph);
        p_trace(trace, 10, u);
        mbar_wait(&bars->v_full[s], ph);
        mbar_wait(&bars->t_empty[0], (u & 1) ^ 1);   // O(u-1) read back
        tc_fence_after();
        p_trace(trace, 11, u);
        const uint32_t tS = tmem + s * kSSlot1;
        const uint32_t v_s = smem_u32(sm + s * kPStageBytes + 16384 + 32768);
        for (int kk = 0; kk < (ncols >> 4); ++kk)
          umma_f16_ts(tmem + kSOCol, tS + p_col2(kk >> 1) + (kk & 1) * 8,
                      sdesc_mnmajor_sw128(v_s + kk * 2048, 8192), idesc_bf16_f32_bmn(128, 64),
                      kk > 0 ? 1u : 0u);
        umma_commit(&bars->o_full[0]);
        umma_commit(&bars->v_empty[s]);
        p_trace(trace, 2, u);
        if (si.cur.ok) issue_s();   // S(u+2) into the slot P V(u) just read
      }
    }
  } else if (warp >= kSW) {
    // -------------------------------------------------------------- correction warps
    const int quarter = warp & 3, row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    uint8_t* stg = ostage + quarter * 4096;
    float o[64];
#pragma unroll
    for (int d = 0; d < 64; ++d) o[d] = 0.f;
    for (uint32_t u = 0; it.cur.ok; ++u, it.advance(a)) {
      const PUnit un = it.cur;
      const int s = u & 1;
      const uint32_t ph = (u >> 1) & 1;
      const int c4 = u & 3;
      mbar_wait(&bars->cl_full[c4], (u >> 2) & 1);   // corr / l of this unit visible
      const float corr = sCL[c4 * 384 + row];
      const float l = kSHalves == 1 ? sCL[c4 * 384 + 128 + row]
                                    : sCL[c4 * 384 + 128 + row] + sCL[c4 * 384 + 256 + row];
      mbar_wait(&bars->o_full[0], u & 1);
      tc_fence_after();
      if (quarter == 0 && lane == 0) p_trace(trace, 7, u);
      const bool rows_live = un.qt * kTQ + quarter * 32 < un.nq;
      if (rows_live) {
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
          uint32_t r0[16];
          tmem_ld16(tmem + kSOCol + lane_off + hh * 16, r0);
          tmem_ld_wait();
#pragma unroll
          for (int d = 0; d < 16; ++d) asm volatile("" : "+r"(r0[d]));
          // corr = 0 on an item's first chunk clears what the previous item left in o
#pragma unroll
          for (int d = 0; d < 16; ++d)
            o[hh * 16 + d] = fmaf(o[hh * 16 + d], corr, __uint_as_float(r0[d]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->t_empty[0]);
      if (rows_live && un.kc + kSKC >= un.nk) {
        const float inv = 1.0f / l;
        // stage this warp's 32 rows x 64 dims (128 B per row, 16 B chunks XOR-swizzled by row)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 w;
          w.x = pack_bf16x2(o[8 * c] * inv, o[8 * c + 1] * inv);
          w.y = pack_bf16x2(o[8 * c + 2] * inv, o[8 * c + 3] * inv);
          w.z = pack_bf16x2(o[8 * c + 4] * inv, o[8 * c + 5] * inv);
          w.w = pack_bf16x2(o[8 * c + 6] * inv, o[8 * c + 7] * inv);
          *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) = w;
        }
        __syncwarp();
        const int rbase = un.qt * kTQ + quarter * 32;
#pragma unroll
        for (int it2 = 0; it2 < 8; ++it2) {
          const int r = 4 * it2 + (lane >> 3), c = lane & 7;
          if (a.out_hi && rbase + r < un.nq)
            *reinterpret_cast<uint4*>(a.out_hi + (size_t)(un.q0 + rbase + r) * a.ld_out +
                                      un.h * 64 + 8 * c) =
                *reinterpret_cast<const uint4*>(stg + r * 128 + ((c ^ (r & 7)) << 4));
        }
        __syncwarp();
        const int qi = un.qt * kTQ + row;
        if (a.out_f32 && qi < un.nq) {
          const size_t ob = (size_t)(un.q0 + qi) * a.ld_out + un.h * 64;
#pragma unroll
          for (int d = 0; d < 64; ++d) a.out_f32[ob + d] = o[d] * inv;
        }
      }
      if (quarter == 0 && lane == 0) p_trace(trace, 8, u);
    }
  } else {
    // -------------------------------------------------------------- softmax warps
    const int quarter = warp & 3, half = warp >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = a.scale * 1.4426950408889634f;
    float m_run = -INFINITY, l_half = 0.f;
    for (uint32_t u = 0; it.cur.ok; ++u, it.advance(a)) {
      const PUnit un = it.cur;
      const int s = u & 1;
      const uint32_t ph = (u >> 1) & 1;
      const uint32_t tS = tmem + s * kSSlot1 + lane_off;
      const int valid = min(kSKC, un.nk - un.kc);
      const int qi = un.qt * kTQ + row;
      const bool warp_rows = un.qt * kTQ + quarter * 32 < un.nq;
      const int qpos = qi < un.ncontent ? un.qpos0 + qi : 0x7FFE;
      const int* kpos = sKpos + (u & 3) * 256;
      if (un.kc == 0) {
        m_run = -INFINITY;
        l_half = 0.f;
      }
      if (tid == 0) p_trace(trace, 12, u);
      if (kCausal) mbar_wait(&bars->kp_full[u & 3], (u >> 2) & 1);
      mbar_wait(&bars->s_full[s], ph);
      if (tid == 0) p_trace(trace, 13, u);
      tc_fence_after();
      if (tid == 0) p_trace(trace, 3, u);
      // pass 1: max of keys 0..127 (groups 0-3, this half's two in one TMEM round trip).
      // P is packed into the columns of groups 0-3 only, so the scores of keys 128.. stay in
      // TMEM through pass 2.  The max of keys 0..127 is the exponent reference: any m with no
      // score more than 2^64 above it gives the same softmax (P and l scale together; bf16
      // and f32 share the exponent range).  If a later key does exceed it by more than 64
      // (log2 units), the softmax warps vote and redo keys 128.. from their intact scores with
      // the exact max, rescaling the P already written.
      float mx = -INFINITY;
      if (warp_rows && half * 32 < valid) {
        uint32_t ra[32], rb[32];
        const int g2 = half + kSHalves;
        const bool two = kSHalves == 2 && g2 < 4 && g2 * 32 < valid;
        tmem_ld32(tS + half * 32, ra);
        if (two) tmem_ld32(tS + g2 * 32, rb);
        const uint32_t ma = p_vis<kCausal>(kpos + half * 32, valid - half * 32, qpos);
        const uint32_t mb = two ? p_vis<kCausal>(kpos + g2 * 32, valid - g2 * 32, qpos) : 0u;
        tmem_ld_wait();
        reg_fence32(ra);
        mx = s_group_max<kCausal>(ra, ma, valid - half * 32 >= 32);
        if (two) {
          reg_fence32(rb);
          mx = fmaxf(mx, s_group_max<kCausal>(rb, mb, valid - g2 * 32 >= 32));
        }
        if (kSHalves == 1) {   // one warp per row: groups 2, 3 as well
          for (int g = 2; g < 4 && g * 32 < valid; ++g) {
            tmem_ld32(tS + g * 32, ra);
            const uint32_t m32 = p_vis<kCausal>(kpos + g * 32, valid - g * 32, qpos);
            tmem_ld_wait();
            reg_fence32(ra);
            mx = fmaxf(mx, s_group_max<kCausal>(ra, m32, valid - g * 32 >= 32));
          }
        }
      }
      if (tid == 0) p_trace(trace, 14, u);
      float cmax = mx;
      if (kSHalves == 2) {
        sRed[(s * 2 + half) * 128 + row] = mx;
        softmax_bar();
        cmax = fmaxf(sRed[s * 256 + row], sRed[s * 256 + 128 + row]);
      }
      if (tid == 0) p_trace(trace, 6, u);
      float mnew = fmaxf(m_run, cmax * sl2);
      float mref = (mnew == -INFINITY) ? 0.f : mnew;
      // pass 2: P = exp2(s*scale*log2e - m) in bf16, into TMEM over already-read S columns
      // (one group per load round trip: the loop is MUFU-bound, prefetching the next group
      // measured slower — scripts/probes/softmax_probe.cu)
      float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                       make_float2(0.f, 0.f)};
      float usum_lo = 0.f;   // keys 0..127
      if (warp_rows) {
        const float2 sl2x2 = make_float2(sl2, sl2), nm2 = make_float2(-mref, -mref);
#pragma unroll 1
        for (int g = half; g * 32 < valid; g += kSHalves) {
          uint32_t rr[32], pk[16];
          tmem_ld32(tS + g * 32, rr);
          const uint32_t m32 = p_vis<kCausal>(kpos + g * 32, valid - g * 32, qpos);
          tmem_ld_wait();
          reg_fence32(rr);
          s_group_exp<kCausal>(rr, m32, valid - g * 32 >= 32, sl2x2, nm2, pk, acc);
          tmem_st16(tS + p_col2(g), pk);
          if (g + kSHalves >= 4 && g < 4) {
            const float2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
            usum_lo = (s01.x + s01.y) + (s23.x + s23.y);
          }
        }
        tmem_st_wait();
      }
      const float2 s01 = fadd2(acc[0], acc[1]), s23 = fadd2(acc[2], acc[3]);
      float usum = (s01.x + s01.y) + (s23.x + s23.y);
      if (valid > 128) {
        uint32_t bad = !(usum <= 1.8446744e19f), any_bad;   // a P above 2^64, or inf / NaN
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
            "bar.red.or.pred p, 2, %2, p;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(any_bad) : "r"(bad), "n"(kSW * 32) : "memory");
        if (any_bad) {   // rare: exact max over keys 128.., then redo them
          float mx2 = mx;
          if (warp_rows) {
#pragma unroll 1
            for (int g = 4 + ((half - 4 % kSHalves + kSHalves) % kSHalves); g * 32 < valid; g += kSHalves) {
              uint32_t rr[32];
              tmem_ld32(tS + g * 32, rr);
              const uint32_t m32 = p_vis<kCausal>(kpos + g * 32, valid - g * 32, qpos);
              tmem_ld_wait();
              reg_fence32(rr);
              mx2 = fmaxf(mx2, s_group_max<kCausal>(rr, m32, valid - g * 32 >= 32));
            }
          }
          float cmax2 = mx2;
          if (kSHalves == 2) {
            __syncwarp();
            softmax_bar();   // every half is done reading sRed of this unit
            sRed[(s * 2 + half) * 128 + row] = mx2;
            softmax_bar();
            cmax2 = fmaxf(sRed[s * 256 + row], sRed[s * 256 + 128 + row]);
          }
          const float mnew2 = fmaxf(m_run, cmax2 * sl2);
          const float mref2 = (mnew2 == -INFINITY) ? 0.f : mnew2;
          const float resc = ex2_approx(mref - mref2);
          usum = usum_lo * resc;
          if (warp_rows) {
            // rescale the P of keys 0..127
#pragma unroll 1
            for (int g = half; g < 4 && g * 32 < valid; g += kSHalves) {
              uint32_t pk[16];
              tmem_ld16(tS + p_col2(g), pk);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float lo = __uint_as_float(pk[j] << 16), hi = __uint_as_float(pk[j] & 0xFFFF0000u);
                pk[j] = pack_bf16x2(lo * resc, hi * resc);
              }
              tmem_st16(tS + p_col2(g), pk);
            }
            // recompute keys 128..
            float2 acc2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                              make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            const float2 sl2x2 = make_float2(sl2, sl2), nm2 = make_float2(-mref2, -mref2);
#pragma unroll 1
            for (int g = 4 + ((half - 4 % kSHalves + kSHalves) % kSHalves); g * 32 < valid; g += kSHalves) {
              uint32_t rr[32], pk[16];
              tmem_ld32(tS + g * 32, rr);
              const uint32_t m32 = p_vis<kCausal>(kpos + g * 32, valid - g * 32, qpos);
              tmem_ld_wait();
              reg_fence32(rr);
              s_group_exp<kCausal>(rr, m32, valid - g * 32 >= 32, sl2x2, nm2, pk, acc2);
              tmem_st16(tS + p_col2(g), pk);
            }
            tmem_st_wait();
            const float2 t01 = fadd2(acc2[0], acc2[1]), t23 = fadd2(acc2[2], acc2[3]);
            usum += (t01.x + t01.y) + (t23.x + t23.y);
          }
          mnew = mnew2;
        }
      }
      const float corr = (m_run == -INFINITY) ? 0.f : ex2_approx(m_run - mnew);
      l_half = l_half * corr + usum;
      m_run = mnew;
      if (half == 0) sCL[(u & 3) * 384 + row] = corr;
      sCL[(u & 3) * 384 + 128 + half * 128 + row] = l_half;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&bars->p_full[s]);
        mbar_arrive(&bars->cl_full[u & 3]);
      }
      if (tid == 0) p_trace(trace, 4, u);

    }
  }
  tc_fence_before();
  __syncthreads();
  if (g_attn_trace != nullptr && tid == 0) {
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    g_attn_trace[512 + blockIdx.x * 2 + 1] = t1;
  }
  if (warp == kSMma) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// ----------------------------------------------------------------------------------------
// fp32-class (parity mode) attention on tcgen05: the split-bf16 ("bf16x3") scheme of the
// GEMMs applied to both products of attention (reference op order attention.py:66-72,
// tensor.py:295-315):
//   S = Qh Kh^T + Qh Kl^T + Ql Kh^T         (fp32 operands split x = hi + lo on load)
//   x = S * scale (fp32), p = exp(x - m) (accurate expf), l = sum p in fp32
//   O = Ph Vh + Ph Vl + Pl Vh               (p = Ph + Pl, split in registers)
//   out = O / l, written as an fp32 row and/or a bf16 hi/lo split (the next GEMM's operand).
// One CTA (8 warps) per (segment, head, 128-query tile); keys in 128-key chunks with the
// online-softmax rescale (ViT-B: 197 keys = 2 chunks), so Q, K and V (hi and lo) take 96 KB
// of smem and 256 TMEM columns: two CTAs per SM overlap one's softmax with the other's MMAs
// and gathers.  K/V rows are gathered through key_src (local projection rows or codebook
// K/V-table rows: the VQ decode fused into the load) from fp32 buffers, split to bf16 hi/lo
// in registers and stored in the SW128 layout the UMMA descriptors read.  Causal: chunks with
// no key visible to any query of the tile are skipped.
// TMEM (256 cols): S [0,128) fp32 with Ph packed over it (keys 0-63 -> cols 0-31, keys
// 64-127 -> cols 64-95), Pl at [128,192), O at [192,256).
constexpr int kT3Q = 128, kT3KC = 128, kT3Threads = 256;
constexpr int kT3Tile = 16384;   // 128 rows x 64 bf16, SW128
constexpr int kT3SmemUsed = 6 * kT3Tile + 2 * 128 * 2 + 2 * 128 * 4 + 4 * 128 * 4 + 64;
constexpr int kT3Smem = kT3SmemUsed + 1024;

// 8 fp32 values -> bf16 hi and lo 16-byte chunks at chunk c of row r of two SW128 tiles.
__device__ __forceinline__ void t3_store_split(const float4& a, const float4& b, uint8_t* hi,
                                               uint8_t* lo, int r, int c) {
  const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __nv_bfloat162 hh = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    const __nv_bfloat162 ll = __floats2bfloat162_rn(v[2 * i] - __low2float(hh),
                                                    v[2 * i + 1] - __high2float(hh));
    h[i] = *reinterpret_cast<const uint32_t*>(&hh);
    l[i] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  const uint32_t off = sw128_offset(r, c);
  *reinterpret_cast<uint4*>(hi + off) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(lo + off) = make_uint4(l[0], l[1], l[2], l[3]);
}

__device__ __forceinline__ const float* t3_key_row(const AttnArgs& a, int src, bool v, int hoff) {
  if (src >= 0)
    return reinterpret_cast<const float*>(v ? a.v_local : a.k_local) + (size_t)src * a.ld_local + hoff;
  return reinterpret_cast<const float*>(v ? a.v_remote : a.k_remote) +
         (size_t)(-(src + 1)) * a.ld_remote + hoff;
}

__global__ void __launch_bounds__(kT3Threads, 2) attention_tc3_kernel(AttnArgs a) {
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  uint8_t* sQh = sm;
  uint8_t* sQl = sm + kT3Tile;
  uint8_t* sKh = sm + 2 * kT3Tile;
  uint8_t* sKl = sm + 3 * kT3Tile;
  uint8_t* sVh = sm + 4 * kT3Tile;
  uint8_t* sVl = sm + 5 * kT3Tile;
  short* sKposB = reinterpret_cast<short*>(sm + 6 * kT3Tile);        // [2][128] key positions
  int* sSrc = reinterpret_cast<int*>(sm + 6 * kT3Tile + 512);         // [2][128] key sources
  float* sRed = reinterpret_cast<float*>(sm + 6 * kT3Tile + 1536);   // [max|sum][half][128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 6 * kT3Tile + 1536 + 2048);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);

  // query tile fastest: the tiles of one (segment, head) run together and share its K/V rows
  // through L2 instead of re-reading them a wave later
  const int qt = blockIdx.x, seg = blockIdx.y, h = blockIdx.z;
  const int* sg = a.segs + seg * 6;
  const int q0 = sg[0], nq = sg[1], qpos0 = sg[2], ncontent = sg[3], k0 = sg[4], nk = sg[5];
  if (qt * kT3Q >= nq) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, half = warp >> 2;
  const int hoff = h * 64;

  if (warp == 0) tmem_alloc<256>(tslot);
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (tid < kT3KC) {   // first chunk's key sources / positions (published by the barrier below)
    const bool in = tid < nk;
    sSrc[tid] = in ? __ldg(a.key_src + k0 + tid) : 0;
    sKposB[tid] = in ? (a.causal ? (short)__ldg(a.key_pos + k0 + tid) : (short)0) : kPosNever;
  }
  // Q tile: 128 rows x 8 chunks, four (row, chunk) units per thread, loads issued first
  {
    float4 qa[4], qb[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int u = tid + i * kT3Threads, r = u >> 3, c = u & 7, qr = qt * kT3Q + r;
      if (qr < nq) {
        const float* qp = reinterpret_cast<const float*>(a.q) + (size_t)(q0 + qr) * a.ldq + hoff + c * 8;
        qa[i] = __ldg(reinterpret_cast<const float4*>(qp));
        qb[i] = __ldg(reinterpret_cast<const float4*>(qp + 4));
      } else {
        qa[i] = qb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int u = tid + i * kT3Threads;
      t3_store_split(qa[i], qb[i], sQh, sQl, u >> 3, u & 7);
    }
  }

  const int row = quarter * 32 + lane;             // this thread's query row = TMEM lane
  const int qi = qt * kT3Q + row;
  const bool warp_rows = qt * kT3Q + quarter * 32 < nq;
  const int qpos = qi < ncontent ? qpos0 + qi : 0x7FFE;
  const int last_q = min(nq, (qt + 1) * kT3Q) - 1;  // causal chunk skipping: tile's last query
  const int qpos_max = last_q < ncontent ? qpos0 + last_q : 0x7FFE;
  const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
  float m_run = -INFINITY, l_half = 0.f;
  float o[32];
#pragma unroll
  for (int d = 0; d < 32; ++d) o[d] = 0.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();   // after the TMEM allocation (ptx.cuh)
  const uint32_t tmem = *tslot, tS = tmem, tPl = tmem + 128, tO = tmem + 192;
  uint32_t phase = 0;

  const int nchunks = (nk + kT3KC - 1) / kT3KC;
  for (int c = 0; c < nchunks; ++c) {
    const int kc = c * kT3KC, buf = c & 1;
    const int valid = min(kT3KC, nk - kc);
    const int* cSrc = sSrc + buf * kT3KC;
    const short* sKpos = sKposB + buf * kT3KC;
    // next chunk's key sources / positions: loads issued now, stored into the other buffer at
    // the end of this chunk (its latency hides behind this chunk's work)
    int nsrc = 0;
    short npos = kPosNever;
    if (tid < kT3KC && kc + kT3KC + tid < nk) {
      nsrc = __ldg(a.key_src + k0 + kc + kT3KC + tid);
      npos = a.causal ? (short)__ldg(a.key_pos + k0 + kc + kT3KC + tid) : (short)0;
    }
    // causal: a chunk none of whose keys is visible to any query of the tile contributes
    // nothing (p = 0 for all of it) and is skipped; replica keys (position -1) stay visible
    const bool run = !a.causal || __syncthreads_or(tid < valid && (int)sKpos[tid] <= qpos_max);
    if (run) {
    const int ncols = (valid + 15) & ~15;
    // ---- K chunk: 128 rows x 8 chunks = 1024 units, 4 per thread; S = Q K^T issued as soon
    // as K is in place, the V chunk is loaded and split while those MMAs run
    {
      float4 ka[4], kb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int u = tid + i * kT3Threads, r = u >> 3, cc = u & 7;
        if (r < valid) {
          const float* p = t3_key_row(a, cSrc[r], false, hoff) + cc * 8;
          ka[i] = __ldg(reinterpret_cast<const float4*>(p));
          kb[i] = __ldg(reinterpret_cast<const float4*>(p + 4));
        } else {
          ka[i] = kb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int u = tid + i * kT3Threads;
        t3_store_split(ka[i], kb[i], sKh, sKl, u >> 3, u & 7);
      }
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      const uint32_t id = idesc_bf16_f32(128, ncols);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        umma_f16(tS, sdesc_kmajor_sw128(smem_u32(sQh) + kk * 32),
                 sdesc_kmajor_sw128(smem_u32(sKh) + kk * 32), id, kk > 0 ? 1u : 0u);
        umma_f16(tS, sdesc_kmajor_sw128(smem_u32(sQh) + kk * 32),
                 sdesc_kmajor_sw128(smem_u32(sKl) + kk * 32), id, 1u);
        umma_f16(tS, sdesc_kmajor_sw128(smem_u32(sQl) + kk * 32),
                 sdesc_kmajor_sw128(smem_u32(sKh) + kk * 32), id, 1u);
      }
      umma_commit(bar);
    }
    {
      float4 va[4], vb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int u = tid + i * kT3Threads, r = u >> 3, cc = u & 7;
        if (r < valid) {
          const float* p = t3_key_row(a, cSrc[r], true, hoff) + cc * 8;
          va[i] = __ldg(reinterpret_cast<const float4*>(p));
          vb[i] = __ldg(reinterpret_cast<const float4*>(p + 4));
        } else {
          va[i] = vb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int u = tid + i * kT3Threads;
        t3_store_split(va[i], vb[i], sVh, sVl, u >> 3, u & 7);
      }
    }
    fence_proxy_async();   // V tiles: published to the P.V MMAs by the barrier below
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();

    // ---- pass 1: row max of x = s * scale over this warp's half of the columns
    float mx = -INFINITY;
    if (warp_rows) {
#pragma unroll
      for (int gg = 0; gg < 2; ++gg) {
        const int g = half * 2 + gg;
        if (g * 32 < valid) {
          uint32_t rr[32];
          tmem_ld32(tS + lane_off + g * 32, rr);
          const uint32_t m32 = attn_vis32(sKpos, g * 32, valid, qpos, a.causal);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if ((m32 >> j) & 1u) mx = fmaxf(mx, __uint_as_float(rr[j]) * a.scale);
        }
      }
    }
    sRed[half * 128 + row] = mx;
    // only the two warps sharing these TMEM lanes (quarter, halves 0 and 1) exchange maxima
    asm volatile("bar.sync %0, 64;" ::"r"(1 + quarter) : "memory");
    const float cmax = fmaxf(sRed[row], sRed[128 + row]);
    const float mnew = fmaxf(m_run, cmax);
    const float corr = (m_run == -INFINITY) ? 0.f : expf(m_run - mnew);
    const float mref = (mnew == -INFINITY) ? 0.f : mnew;

    // ---- pass 2: p = exp(x - m) in fp32, l += p, P = Ph + Pl into TMEM
    float ls = 0.f;
    if (warp_rows) {
#pragma unroll
      for (int gg = 0; gg < 2; ++gg) {
        const int g = half * 2 + gg;
        if (g * 32 < valid) {
          uint32_t rr[32], ph[16], pl[16];
          tmem_ld32(tS + lane_off + g * 32, rr);
          const uint32_t m32 = attn_vis32(sKpos, g * 32, valid, qpos, a.causal);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            const float p0 = ((m32 >> j) & 1u) ? expf(__uint_as_float(rr[j]) * a.scale - mref) : 0.f;
            const float p1 =
                ((m32 >> (j + 1)) & 1u) ? expf(__uint_as_float(rr[j + 1]) * a.scale - mref) : 0.f;
            ls += p0 + p1;
            const __nv_bfloat162 hh = __floats2bfloat162_rn(p0, p1);
            const __nv_bfloat162 ll =
                __floats2bfloat162_rn(p0 - __low2float(hh), p1 - __high2float(hh));
            ph[j >> 1] = *reinterpret_cast<const uint32_t*>(&hh);
            pl[j >> 1] = *reinterpret_cast<const uint32_t*>(&ll);
          }
          const int pcol = g < 2 ? g * 16 : 64 + (g - 2) * 16;
          tmem_st16(tS + lane_off + pcol, ph);
          tmem_st16(tPl + lane_off + g * 16, pl);
        }
      }
      tmem_st_wait();
    }
    l_half = l_half * corr + ls;
    m_run = mnew;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      const int ksteps = ncols >> 4;
      const uint32_t id = idesc_bf16_f32_bmn(128, 64);
      for (int kk = 0; kk < ksteps; ++kk) {
        const uint32_t acol = kk < 4 ? kk * 8 : 64 + (kk - 4) * 8;
        const uint64_t dvh = sdesc_mnmajor_sw128(smem_u32(sVh) + kk * 2048, 8192);
        const uint64_t dvl = sdesc_mnmajor_sw128(smem_u32(sVl) + kk * 2048, 8192);
        umma_f16_ts(tO, tS + acol, dvh, id, kk > 0 ? 1u : 0u);
        umma_f16_ts(tO, tS + acol, dvl, id, 1u);
        umma_f16_ts(tO, tPl + kk * 8, dvh, id, 1u);
      }
      umma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
    if (warp_rows) {
      uint32_t r0[32];
      tmem_ld32(tO + lane_off + half * 32, r0);
      tmem_ld_wait();
#pragma unroll
      for (int d = 0; d < 32; ++d) o[d] = fmaf(o[d], corr, __uint_as_float(r0[d]));
    }
    }   // run
    if (tid < kT3KC) {
      sSrc[(buf ^ 1) * kT3KC + tid] = nsrc;
      sKposB[(buf ^ 1) * kT3KC + tid] = npos;
    }
    tc_fence_before();
    __syncthreads();   // K/V tiles, TMEM columns and the staged key buffer free for the next chunk
  }

  sRed[256 + half * 128 + row] = l_half;
  __syncthreads();
  if (qi < nq) {
    const float inv = 1.0f / (sRed[256 + row] + sRed[384 + row]);
    const size_t ob = (size_t)(q0 + qi) * a.ld_out + hoff + half * 32;
    if (a.out_hi) {
#pragma unroll
      for (int d = 0; d < 32; d += 8) {
        uint32_t wh[4], wl[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float v0 = o[d + 2 * u] * inv, v1 = o[d + 2 * u + 1] * inv;
          const __nv_bfloat162 hh = __floats2bfloat162_rn(v0, v1);
          const __nv_bfloat162 ll = __floats2bfloat162_rn(v0 - __low2float(hh), v1 - __high2float(hh));
          wh[u] = *reinterpret_cast<const uint32_t*>(&hh);
          wl[u] = *reinterpret_cast<const uint32_t*>(&ll);
        }
        *reinterpret_cast<uint4*>(a.out_hi + ob + d) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
        if (a.out_lo)
          *reinterpret_cast<uint4*>(a.out_lo + ob + d) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
      }
    }
    if (a.out_f32) {
#pragma unroll
      for (int d = 0; d < 32; d += 4)
        *reinterpret_cast<float4*>(a.out_f32 + ob + d) =
            make_float4(o[d] * inv, o[d + 1] * inv, o[d + 2] * inv, o[d + 3] * inv);
    }
  }
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
    launch_k(attention_simt_kernel<true, DH>, grid, 256, smem, st, a);
  else
    launch_k(attention_simt_kernel<false, DH>, grid, 256, smem, st, a);
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

// SIMT kernel instance for any head width 1..128: the smallest padded width >= head_dim.
static int launch_attn_any(const AttnArgs& a, dim3 grid, cudaStream_t st) {
  const int hd = a.head_dim;
  if (hd <= 4) return launch_attn<4>(a, grid, st);
  if (hd <= 8) return launch_attn<8>(a, grid, st);
  if (hd <= 16) return launch_attn<16>(a, grid, st);
  if (hd <= 32) return launch_attn<32>(a, grid, st);
  if (hd <= 64) return launch_attn<64>(a, grid, st);
  return launch_attn<128>(a, grid, st);
}

}  // namespace astra

using namespace astra;

extern "C" int astra_attention(const void* q, int ldq, const void* k_local, const void* v_local,
                               int ld_local, const void* k_remote, const void* v_remote,
                               int ld_remote, const int32_t* key_src, const int32_t* key_pos,
                               const int32_t* segs, int num_segs, int max_nq, int heads,
                               int head_dim, int causal, int in_bf16, float scale, float* out_f32,
                               void* out_hi, void* out_lo, int ld_out, int q_rows,
                               int local_rows, int remote_rows, void* stream) {
  ASTRA_REQUIRE(head_dim >= 1 && head_dim <= 128, ASTRA_ERR_SHAPE,
                "attention: head_dim %d unsupported (1..128)", head_dim);
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
      ASTRA_CUDA_CHECK(cudaFuncSetAttribute(attention_tcp_kernel<false>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
      ASTRA_CUDA_CHECK(cudaFuncSetAttribute(attention_tcp_kernel<true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, kPSmem));
      ASTRA_CUDA_CHECK(cudaFuncSetAttribute(attention_tcs_kernel<false>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, kSSmem));
      ASTRA_CUDA_CHECK(cudaFuncSetAttribute(attention_tcs_kernel<true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, kSSmem));
      configured = true;
    }
    const int qtiles = (max_nq + kTQ - 1) / kTQ;
    static int delay_set = -1;
    if (delay_set < 0) {   // bench-only experiment switch (default 0: both pipelines start at once)
      const char* d = getenv("ASTRA_ATTN_PIPE_DELAY");
      delay_set = d ? atoi(d) : 0;
      if (delay_set) ASTRA_CUDA_CHECK(cudaMemcpyToSymbol(g_attn_pipe_delay, &delay_set, sizeof(int)));
    }
    if (g_attention_variant != 1) {
      const long items = (long)num_segs * heads * qtiles;
      const int grid = (int)std::min<long>(items, num_sms());
      // gather maps (SW128, true row extents: boxes running past a buffer are zero-filled)
      PMaps mp;
      const auto bf = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
      const uint64_t qr = std::max(q_rows, 1), lr = std::max(local_rows, 1),
                     rr = std::max(remote_rows, 1);
      int rc;
      if ((rc = make_tmap_2d(&mp.q, q, bf, 2, qr, ldq, ldq, kTQ, 64, true)) ||
          (rc = make_tmap_2d(&mp.kl, k_local, bf, 2, lr, ld_local, ld_local, 1, 64, true)) ||
          (rc = make_tmap_2d(&mp.vl, v_local, bf, 2, lr, ld_local, ld_local, 1, 64, true)) ||
          (rc = make_tmap_2d(&mp.kl16, k_local, bf, 2, lr, ld_local, ld_local, 16, 64, true)) ||
          (rc = make_tmap_2d(&mp.vl16, v_local, bf, 2, lr, ld_local, ld_local, 16, 64, true)) ||
          (rc = make_tmap_2d(&mp.kr, k_remote, bf, 2, rr, ld_remote, ld_remote, 1, 64, true)) ||
          (rc = make_tmap_2d(&mp.vr, v_remote, bf, 2, rr, ld_remote, ld_remote, 1, 64, true)))
        return rc;
      if (g_attention_variant == 2) {
        if (causal)
          launch_kp(attention_tcs_kernel<true>, grid, kSThreads, kSSmem, st, a, mp, qtiles);
        else
          launch_kp(attention_tcs_kernel<false>, grid, kSThreads, kSSmem, st, a, mp, qtiles);
      } else if (causal) {
        launch_kp(attention_tcp_kernel<true>, grid, kPThreads, kPSmem, st, a, mp, qtiles);
      } else {
        launch_kp(attention_tcp_kernel<false>, grid, kPThreads, kPSmem, st, a, mp, qtiles);
      }
    } else {
      dim3 tgrid(num_segs, heads, qtiles);
      launch_kp(attention_tc_kernel, tgrid, kTcThreads, kTcSmem, st, a);
    }
    ASTRA_CUDA_CHECK(cudaGetLastError());
    return ASTRA_OK;
  }
  // fp32 inputs (parity mode): the split-bf16 tcgen05 kernel for 64-wide heads
  const bool aligned32 = (ldq % 4 == 0) && (ld_local % 4 == 0) && (ld_remote % 4 == 0) &&
                         (ld_out % 8 == 0) &&
                         ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k_local) |
                           reinterpret_cast<uintptr_t>(v_local) |
                           reinterpret_cast<uintptr_t>(k_remote) |
                           reinterpret_cast<uintptr_t>(v_remote) |
                           reinterpret_cast<uintptr_t>(out_f32) |
                           reinterpret_cast<uintptr_t>(out_hi) |
                           reinterpret_cast<uintptr_t>(out_lo)) & 15) == 0;
  if (!in_bf16 && head_dim == 64 && aligned32 && !g_force_simt_attention) {
    static bool configured3 = false;
    if (!configured3) {
      ASTRA_CUDA_CHECK(cudaFuncSetAttribute(attention_tc3_kernel,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, kT3Smem));
      configured3 = true;
    }
    dim3 tgrid((max_nq + kT3Q - 1) / kT3Q, num_segs, heads);
    launch_kp(attention_tc3_kernel, tgrid, kT3Threads, kT3Smem, st, a);
    ASTRA_CUDA_CHECK(cudaGetLastError());
    return ASTRA_OK;
  }
  dim3 grid(num_segs, heads, (max_nq + kAQ - 1) / kAQ);
  const int rc = launch_attn_any(a, grid, st);
  if (rc) return rc;
  ASTRA_CUDA_CHECK(cudaGetLastError());
  return ASTRA_OK;
}

extern "C" int astra_attention_trace(void* buf) {
  long long* p = reinterpret_cast<long long*>(buf);
  ASTRA_CUDA_CHECK(cudaMemcpyToSymbol(g_attn_trace, &p, sizeof(p)));
  return ASTRA_OK;
}

extern "C" int astra_attention_variant(int variant) {
  g_attention_variant = variant;
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
  ASTRA_REQUIRE(dk >= 1 && dk <= 128, ASTRA_ERR_SHAPE, "attention: head_dim %d unsupported", dk);
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
  return launch_attn_any(a, grid, st);
}
