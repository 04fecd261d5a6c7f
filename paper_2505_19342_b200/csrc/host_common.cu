#include <cstdarg>
#include <cstdlib>
#include <cudaTypedefs.h>

#include "host_common.h"

namespace astra {

static thread_local char g_last_error[1024] = "";

void set_last_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

static thread_local int g_pdl_override = -1;   // astra_pdl_override (this host thread's launches)

int pdl_mode() {
  static const int mode = [] {
    const char* e = getenv("ASTRA_PDL");
    return e && e[0] >= '0' && e[0] <= '2' ? e[0] - '0' : 2;
  }();
  return g_pdl_override >= 0 ? g_pdl_override : mode;
}

int set_pdl_override(int mode) {
  const int prev = g_pdl_override;
  g_pdl_override = mode >= 0 && mode <= 2 ? mode : -1;
  return prev;
}

int num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached = n > 0 ? n : 148;
  }
  return cached;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
  });
  return fn;
}

int make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, int elem_bytes,
                 uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows, uint32_t box_cols,
                 bool swizzle128) {
  auto fn = get_encode_fn();
  ASTRA_REQUIRE(fn != nullptr, ASTRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  ASTRA_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, ASTRA_ERR_SHAPE,
                "TMA base pointer must be 16-byte aligned");
  ASTRA_REQUIRE((ld * elem_bytes) % 16 == 0, ASTRA_ERR_SHAPE,
                "TMA row pitch must be a multiple of 16 bytes (ld=%llu)", (unsigned long long)ld);
  cuuint64_t gdim[2] = {cols, rows};
  cuuint64_t gstride[1] = {ld * elem_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = fn(map, dtype, 2, const_cast<void*>(base), gdim, gstride, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  ASTRA_REQUIRE(r == CUDA_SUCCESS, ASTRA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ASTRA_OK;
}

}  // namespace astra

extern "C" const char* astra_last_error(void) { return astra::g_last_error; }

extern "C" int astra_abi_version(void) { return ASTRA_ABI_VERSION; }

// Programmatic-dependent-launch policy for the calling host thread's subsequent launches
// (0 none, 1 every kernel, 2 persistent kernels only, -1 back to ASTRA_PDL / the default).
// The runtime turns it off around the Q|K|V GEMM when the VQ chain is on the critical path.
extern "C" int astra_pdl_override(int mode) { return astra::set_pdl_override(mode); }
