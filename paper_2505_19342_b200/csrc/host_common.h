// Host-side helpers shared by the C-ABI entry points: status codes, TMA
// descriptor encoding (driver entry point fetched at run time so the library
// does not link libcuda), SM count cache.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <mutex>

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

}  // namespace astra
