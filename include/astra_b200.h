/*
 * astra_b200.h — C ABI of the B200-native Astra Mixed-Precision Attention path.
 *
 * The reference (seqvq, /root/reference/pkg/src/seqvq) is a pure-Python
 * operator API over NumPy arrays; it has no FFI.  This header is the native
 * boundary underneath the Python drop-in (paper_2505_19342_b200), one entry
 * point per reference operator on the hot path.  Each declaration cites the
 * reference interface it replaces.
 *
 * Conventions
 *   - every buffer is a caller-owned DEVICE pointer, row-major, no allocation
 *     happens inside a call; `stream` is a cudaStream_t passed as void*.
 *   - calls are asynchronous on `stream` and deterministic (no atomics in
 *     reductions, fixed summation order).
 *   - return value: ASTRA_OK or one of the status codes below; the message of
 *     the last failure on the calling thread is astra_last_error().
 */
#ifndef ASTRA_B200_H
#define ASTRA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASTRA_ABI_VERSION 1

/* status codes; the Python shim maps them to the reference's exception types
 * (seqvq/errors.py:4-33). */
#define ASTRA_OK 0
#define ASTRA_ERR_SHAPE 1      /* -> ShapeError          */
#define ASTRA_ERR_INDEX 2      /* -> IndexCorruptionError */
#define ASTRA_ERR_CUDA 3       /* -> RuntimeError         */
#define ASTRA_ERR_MASK 5       /* -> MaskError            */

const char* astra_last_error(void);
int astra_abi_version(void);

/* ------------------------------------------------------------------ GEMM
 * Replaces tensor.matmul (tensor.py:142-155) and the elementwise ops fused
 * after it on the hot path: add_bias (tensor.py:186-190), gelu
 * (tensor.py:348-358) and the residual add (cluster.py:213, :216).
 *
 *   v[m, n]  = sum_k A[m, k] * B[n, k]        (B is the weight TRANSPOSED: [N, K])
 *   v       += bias[n]            (bias != NULL)
 *   v        = gelu_erf(v)        (gelu != 0)
 *   v        = residual[m, n] + v (residual != NULL)
 *   out_f32[m, n] = v; out_hi/out_lo[m, n] = bf16 split of v (each optional)
 *
 * passes = 1: A, B are bf16 (fast mode).  passes = 3: A = A_hi + A_lo and
 * B = B_hi + B_lo are split bf16 pairs and the product is computed as
 * hi*hi + hi*lo + lo*hi on tcgen05 (fp32-class parity mode).
 * Requires K % 8 == 0 and 16-byte aligned rows.
 */
int astra_gemm(const void* a_hi, const void* a_lo, int lda, const void* b_hi, const void* b_lo,
               int ldb, int M, int N, int K, int passes, const float* bias,
               const float* residual, int ld_res, float* out_f32, int ld_f32, void* out_hi,
               void* out_lo, int ld_bf, int gelu, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ASTRA_B200_H */
