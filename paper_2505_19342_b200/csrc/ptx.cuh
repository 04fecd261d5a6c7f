// Thin inline-PTX layer for sm_100a: mbarriers, TMA, tcgen05 (UMMA + TMEM).
// Everything the hot kernels need, nothing else.  Encodings follow the
// PTX ISA for tcgen05 (instruction descriptor kind::f16, shared-memory matrix
// descriptor version 1) as used by the sm_100a tensor-core path.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define ASTRA_DEVICE __device__ __forceinline__

namespace astra {

ASTRA_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

ASTRA_DEVICE uint32_t lane_id() { return threadIdx.x & 31; }
ASTRA_DEVICE uint32_t warp_id() {
  return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
}

ASTRA_DEVICE bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- programmatic dependent launch
// Every kernel of the library is launched with programmatic stream serialisation (host
// launch_k / launch_tc_gemm): its CTAs may start while the previous kernel of the stream is
// still draining.  pdl_wait() blocks until that kernel has completed and its writes are
// visible (a no-op without the attribute), so it precedes every global-memory access;
// pdl_trigger() lets the next kernel's CTAs start their prologue.  Kernels that allocate TMEM
// trigger only after their allocation: a dependent CTA that allocated first on the same SM
// would otherwise hold the columns while waiting on this kernel (deadlock).
ASTRA_DEVICE void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
ASTRA_DEVICE void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---------------------------------------------------------------- mbarrier
ASTRA_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
ASTRA_DEVICE void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
ASTRA_DEVICE void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
ASTRA_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
ASTRA_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Blocks until the phase with `parity` completes (try_wait spin: the hardware already parks a
// waiting warp for a short, system-dependent time per probe).
ASTRA_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Same, polling with mbarrier.test_wait (never parks the warp): try_wait may suspend a warp
// for a system-dependent time and wake it late (~0.5 us measured) — too slow for a
// latency-critical hand-off between warps of a pipeline.
ASTRA_DEVICE void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// --------------------------------------------------------------------- TMA
ASTRA_DEVICE void tma_prefetch_desc(const void* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}
// 2-D tiled load: coordinates are (inner, outer) in elements.
ASTRA_DEVICE void tma_load_2d(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1,
                              uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(cache_hint)
      : "memory");
}
// Gather of four rows (r0..r3, any order) of a 2-D tensor whose box is {cols, 1}: the rows
// land back to back at smem_dst with the tensor map's swizzle applied by smem address.
ASTRA_DEVICE void tma_gather4(void* smem_dst, const void* desc, uint64_t* bar, int col, int r0,
                              int r1, int r2, int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1),
      "r"(r2), "r"(r3)
      : "memory");
}
// 2-D tiled store smem -> global (bulk group): rows / columns past the tensor are not written.
ASTRA_DEVICE void tma_store_2d(const void* desc, uint32_t smem_src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(desc)),
               "r"(smem_src), "r"(c0), "r"(c1)
               : "memory");
}
ASTRA_DEVICE void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N committed bulk groups may still be reading their shared-memory source
template <int N>
ASTRA_DEVICE void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
ASTRA_DEVICE void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// 3-D tiled load: (inner, mid, outer).
ASTRA_DEVICE void tma_load_3d(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1,
                              int c2, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "l"(cache_hint)
      : "memory");
}
// 2-D tiled load multicast to every CTA of the cluster in `mask`: the box lands at the same
// CTA-relative smem offset in each destination and signals the mbarrier at the same offset.
ASTRA_DEVICE void tma_load_2d_mc(void* smem_dst, const void* desc, uint64_t* bar, int c0, int c1,
                                 uint16_t mask, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::"
      "cluster.L2::cache_hint [%0], [%1, {%4, %5}], [%2], %3, %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "h"(mask), "r"(c0), "r"(c1),
      "l"(cache_hint)
      : "memory");
}
// CTA-pair (cta_group::2) tiled load: lands in this CTA's smem, completes bytes on the
// mbarrier given as a shared::cluster address (the pair leader's barrier).
ASTRA_DEVICE void tma_load_2d_pair(void* smem_dst, const void* desc, uint32_t bar_cluster_addr,
                                   int c0, int c1, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar_cluster_addr), "r"(c0), "r"(c1),
      "l"(cache_hint)
      : "memory");
}
// CTA-pair load multicast to the CTAs in `mask`: the box lands at the same offset in each
// destination and its bytes complete on the barrier at `bar_offset` in each destination's pair
// leader (CUTLASS SM100_TMA_2SM_LOAD_MULTICAST convention: local barrier address with the
// peer bit, bit 24, cleared).
ASTRA_DEVICE void tma_load_2d_pair_mc(void* smem_dst, const void* desc, uint32_t bar_pair_addr,
                                      int c0, int c1, uint16_t mask, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster.L2::cache_hint [%0], [%1, {%4, %5}], [%2], %3, %6;" ::"r"(
          smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(bar_pair_addr), "h"(mask), "r"(c0), "r"(c1),
      "l"(cache_hint)
      : "memory");
}
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;
// shared::cluster address of the same variable in CTA `rank` of the cluster
ASTRA_DEVICE uint32_t mapa_shared(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// Remote arrive (CUTLASS ClusterBarrier form).  An explicit .release.cluster compiles to a
// GPU-scope MEMBAR that waits for all of the warp's outstanding global stores — measured as the
// top stall of the GEMM epilogue warps (their TMEM-empty signal only orders tcgen05.ld reads,
// which tcgen05.fence::before_thread_sync already covers).
ASTRA_DEVICE void mbar_arrive_cluster(uint32_t bar_cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster_addr) : "memory");
}
template <uint32_t kCols>
ASTRA_DEVICE void tmem_alloc_pair(uint32_t* smem_slot) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t kCols>
ASTRA_DEVICE void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
// D[tmem of both CTAs] (+)= A[smem of both] * B[smem of both]^T, M = 256 across the pair
ASTRA_DEVICE void umma_f16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
ASTRA_DEVICE void umma_commit_pair_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
ASTRA_DEVICE uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
ASTRA_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
constexpr uint64_t kEvictNormal = 0x1000000000000000ull;
constexpr uint64_t kEvictFirst = 0x12F0000000000000ull;
constexpr uint64_t kEvictLast = 0x14F0000000000000ull;

// ----------------------------------------------------------------- tcgen05
template <uint32_t kCols>
ASTRA_DEVICE void tmem_alloc(uint32_t* smem_slot) {
  static_assert(kCols >= 32 && kCols <= 512 && (kCols & (kCols - 1)) == 0, "bad TMEM cols");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(smem_slot)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t kCols>
ASTRA_DEVICE void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
// Per-warp register budget hand-off between warp roles (all warps of a warpgroup together).
template <uint32_t kRegs>
ASTRA_DEVICE void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegs));
}
template <uint32_t kRegs>
ASTRA_DEVICE void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegs));
}
ASTRA_DEVICE void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
ASTRA_DEVICE void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T ; both K-major, kind::f16 (bf16 in, f32 accumulate).
ASTRA_DEVICE void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Arrive on an mbarrier once every previously issued tcgen05.mma of this thread completes.
ASTRA_DEVICE void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Same, arriving on the mbarrier at this offset in every CTA of the cluster in `mask`.
ASTRA_DEVICE void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// Instruction descriptor, kind::f16: bf16 A/B, f32 D, both K-major, shape M x N.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N) {
  return (1u << 4)              // D format = f32
         | (1u << 7)            // A format = bf16
         | (1u << 10)           // B format = bf16
         | ((N >> 3) << 17)     // N / 8
         | ((M >> 4) << 24);    // M / 16
}

// Shared-memory matrix descriptor, K-major, 128-byte swizzle: 8-row core
// groups are 1024 B apart (SBO); LBO unused for swizzled K-major layouts.
ASTRA_DEVICE uint64_t sdesc_kmajor_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                 // LBO (ignored)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// MN-major, 128-byte swizzle: 64 MN elements (128 B) per row, consecutive K rows 128 B apart,
// 8-row K groups 1024 B apart (SBO); LBO = stride between 64-wide MN blocks.
ASTRA_DEVICE uint64_t sdesc_mnmajor_sw128(uint32_t smem_addr, uint32_t lbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Byte offset of 16-byte chunk `c` (0..7) of row `r` inside a 128B-swizzled tile
// (the TMA SWIZZLE_128B / UMMA SW128 pattern; tile base 1024-byte aligned).
ASTRA_DEVICE uint32_t sw128_offset(uint32_t r, uint32_t c) {
  return r * 128u + ((c ^ (r & 7u)) << 4);
}

ASTRA_DEVICE void cp_async16(uint32_t smem_addr, const void* gptr) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr), "l"(gptr) : "memory");
}
ASTRA_DEVICE void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 32 lanes x 32 columns of 32-bit TMEM -> 32 registers per thread.
ASTRA_DEVICE void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 32 lanes x 16 columns -> 16 registers per thread.
ASTRA_DEVICE void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
ASTRA_DEVICE void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 16 registers per thread -> 32 lanes x 16 columns of 32-bit TMEM.
ASTRA_DEVICE void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
ASTRA_DEVICE void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]: A (M x K, K-major) read from TMEM — row m in lane m, two
// bf16 K-elements per 32-bit column — B through a shared-memory descriptor.
ASTRA_DEVICE void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

// --------------------------------------------------------------- numerics
// Packed fp32 pairs (sm_100 FFMA2 / FADD2: two lanes of work per issue slot).
ASTRA_DEVICE float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
// three-input min (FMNMX3, sm_100)
ASTRA_DEVICE float fmin3(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
ASTRA_DEVICE float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// 2^x for a pair on the FMA pipe, leaving the MUFU free: x = n + f by round-to-nearest
// (magic-number add), f in [-0.5, 0.5]; degree-3 fit of 2^f (max rel. error 1.0e-4, below the
// bf16 rounding of P); n added to the exponent field.  x is clamped at -126 (masked scores give
// 2^-126, not 0).
ASTRA_DEVICE float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 r = fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = ffma2(r, make_float2(-1.f, -1.f), x);
  float2 q = ffma2(f, make_float2(0.05500893f, 0.05500893f), make_float2(0.242211f, 0.242211f));
  q = ffma2(f, q, make_float2(0.69328293f, 0.69328293f));
  q = ffma2(f, q, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}
ASTRA_DEVICE float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
ASTRA_DEVICE uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
// Split an fp32 value into bf16 hi + bf16 lo (x ~= hi + lo, |x-hi-lo| <= 2^-16 |x|).
ASTRA_DEVICE void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// Exact-erf GELU of the reference (tensor.py:348-352: x * 0.5 * (1 + erf(x / sqrt 2))),
// evaluated branch-free as x * Phi(x) with Phi(-|x|) = 0.5 * exp(-z^2) * R(z), z = |x|/sqrt 2,
// R(z) = erfc(z) exp(z^2) a degree-14 fit on [0, 4] (|R error| < 5e-8).  Max |error| vs the
// exact GELU is 3.8e-7 over the real line — below the 4.5e-7 of the reference's own fp32
// formula — at ~22 instructions, with no data-dependent branches, so 32 unrolled calls in
// the GEMM epilogue pipeline instead of serialising.
ASTRA_DEVICE float gelu_erf(float x) {
  const float z = fabsf(x) * 0.70710678118654752f;
  const float e = exp2f(-(z * z) * 1.4426950408889634f);
  const float u = fminf(z, 4.0f) - 2.0f;
  float r = 6.649368495352473e-08f;
  r = fmaf(r, u, -2.5338264570453217e-07f);
  r = fmaf(r, u, 1.1481752158355554e-08f);
  r = fmaf(r, u, -1.2186578377952116e-07f);
  r = fmaf(r, u, 5.857062441703646e-06f);
  r = fmaf(r, u, -2.0142884551620198e-05f);
  r = fmaf(r, u, 5.3301944671312905e-05f);
  r = fmaf(r, u, -0.00017814906436665912f);
  r = fmaf(r, u, 0.0005950281527983256f);
  r = fmaf(r, u, -0.0018374285307079506f);
  r = fmaf(r, u, 0.00543942681539313f);
  r = fmaf(r, u, -0.01545844890954592f);
  r = fmaf(r, u, 0.04180300727310504f);
  r = fmaf(r, u, -0.1067967008512302f);
  r = fmaf(r, u, 0.25539566823187454f);
  const float h = 0.5f * e * r;  // Phi(-|x|)
  return x * (x >= 0.0f ? 1.0f - h : h);
}

// bf16-output GELU for the fast path: x * Phi(x) with Phi(x) = 1 / (1 + 2^-v(x)), v an odd
// degree-5 polynomial fitted (minimax, fp32 evaluation) to log2(Phi / (1 - Phi)) on [-5, 5];
// the logistic form has no cancellation on either tail.  Max |error| vs the exact erf GELU
// 2.6e-5 over |x| <= 50 (relative 1.2e-3 where |gelu| > 1e-2, below the bf16 output's half
// ulp).  10 instructions, two of them MUFU (ex2, rcp) — half the issue slots of the erfc
// polynomial, which bound the W1 epilogue.
ASTRA_DEVICE float gelu_erf_bf16(float x) {
  const float xc = fminf(fmaxf(x, -5.0f), 5.0f);
  const float x2 = xc * xc;
  const float p = fmaf(fmaf(-0.0010147804887581664f, x2, 0.10677938108922315f), x2,
                       2.3011167090624842f);
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(p * -xc));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return x * r;
}

}  // namespace astra
