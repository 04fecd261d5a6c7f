// Host-side helpers shared by the C-ABI entry points: status codes, TMA
// descriptor encoding (driver entry point fetched at run time so the library
// does not link libcuda), SM count cache.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <utility>

#include "../../include/astra_b200.h"

namespace astra {

void set_last_error(const char* fmt, ...);

#define ASTRA_CUDA_CHECK(expr)                                                       \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      ::astra::set_last_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,             \
                              cudaGetErrorString(_e));                               \
      return ASTRA_ERR_CUDA;                                                         \
    }                                                                                \
  } while (0)

#define ASTRA_REQUIRE(cond, code, ...)        \
  do {                                        \
    if (!(cond)) {                            \
      ::astra::set_last_error(__VA_ARGS__);   \
      return (code);                          \
    }                                         \
  } while (0)

int num_sms();

// 2-D row-major tensor [rows, cols] of `elem_bytes` elements with row pitch
// `ld` elements; box = [box_rows, box_cols]; 128B swizzle when swizzle128.
int make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, int elem_bytes,
                 uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows, uint32_t box_cols,
                 bool swizzle128);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch: ASTRA_PDL=0 off, 1 every kernel, 2 (default) only the
// persistent tensor-core kernels (GEMM, attention) — see DESIGN §3.5.
int pdl_mode();
int set_pdl_override(int mode);   // -1: back to ASTRA_PDL / the default; returns the previous
inline bool pdl_enabled() { return pdl_mode() == 1; }
inline bool pdl_persistent() { return pdl_mode() >= 1; }

// Kernel launch with programmatic stream serialisation (see ptx.cuh pdl_wait): the kernel's
// CTAs may launch while the stream's previous kernel drains and run their prologue (barrier
// init, TMEM allocation, descriptor prefetch) before pdl_wait().  Errors surface through
// cudaGetLastError() like a <<<>>> launch.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args&&... args) {
  return launch_pdl(pdl_enabled(), kern, grid, block, smem, s, std::forward<Args>(args)...);
}
// persistent tensor-core kernels (attention)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kp(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t s, Args&&... args) {
  return launch_pdl(pdl_persistent(), kern, grid, block, smem, s, std::forward<Args>(args)...);
}

}  // namespace astra
