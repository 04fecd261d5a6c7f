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

#define ASTRA_ABI_VERSION 2

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
 *   v        = gelu_erf(v)        (gelu = 1: fp32-class, |err| < 4e-7;
 *                                  gelu = 2: bf16-output class, |err| < 3e-5)
 *   v        = residual[m, n] + v (residual != NULL)
 *   out_f32[m, n] = v; out_hi/out_lo[m, n] = bf16 split of v (each optional)
 *
 * passes = 1: A, B are bf16 (fast mode).  passes = 3: A = A_hi + A_lo and
 * B = B_hi + B_lo are split bf16 pairs and the product is computed as
 * hi*hi + hi*lo + lo*hi on tcgen05 (fp32-class parity mode).
 * K % 8 == 0 with 16-byte aligned rows runs the tcgen05 kernel; any other shape runs a
 * general SIMT kernel with the same epilogue (fp32 accumulation of hi + lo operands).
 */
int astra_gemm(const void* a_hi, const void* a_lo, int lda, const void* b_hi, const void* b_lo,
               int ldb, int M, int N, int K, int passes, const float* bias,
               const float* residual, int ld_res, float* out_f32, int ld_f32, void* out_hi,
               void* out_lo, int ld_bf, int gelu, void* stream);

/* ------------------------------------------------------------ VQ encode
 * Replaces vq.quantize / vq._nearest (vq.py:126-131, :207-222): per group g,
 * idx = argmin_k ||x_g - c_{g,k}||^2 evaluated in fp64, ties -> lowest k.
 *
 * B200 design: the distance GEMM runs on tcgen05 in split bf16x3 (fp32-class)
 * with a fused per-row argmin epilogue that keeps every code whose approximate
 * score lies inside a proven error window of the best; a second kernel merges
 * the code-chunk candidates and re-ranks the (rare) multi-candidate rows in
 * exact fp64, so the indices are bit-identical to the fp64 reference.
 */
typedef struct AstraCodebook {
  int groups;            /* G                                                */
  int size;              /* K (codes per group)                              */
  int group_dim;         /* D/G                                              */
  int padded_dim;        /* D/G rounded up to 64 (bf16 swizzle row)          */
  const float* centroids;   /* [G, K, D/G] fp32 (Codebook.centroids, vq.py:31-76) */
  const void* c_hi;         /* [G, K, padded] bf16 hi split, zero padded      */
  const void* c_lo;         /* [G, K, padded] bf16 lo split                   */
  const float* c_sq;        /* [G, K] ||c||^2 (fp32, epilogue score)          */
  const double* c_sq64;     /* [G, K] ||c||^2 (fp64, exact re-rank)           */
  const float* c_norm_max;  /* [G] max_k ||c_k||                              */
  const void* c_win;        /* [G, K] float4 {||c||^2, ||c|| (rounded up), 4.8e-7 ||c||^2, 0}:
                               per-code score error window of the encode epilogue */
} AstraCodebook;

/* Fill the derived tables of `cb` (c_hi, c_lo, c_sq, c_sq64, c_norm_max, c_win are
 * caller-allocated device buffers named in cb; cb->centroids is the input). */
int astra_vq_prepare(const AstraCodebook* cb, void* stream);

/* Bytes of scratch astra_vq_encode needs for M tokens. */
int64_t astra_vq_encode_workspace(int M, int groups, int size, int padded_dim);

/* idx_out[m, g] (int32, [M, G] row-major) = nearest code of token row
 * rows ? rows[m] : m of x (fp32, row pitch ldx).  stats (nullable, int32[4],
 * accumulated): {tokens re-ranked in fp64, tokens needing a full fp64 scan,
 * total window candidates, 0}. */
int astra_vq_encode(const AstraCodebook* cb, const float* x, int M, int ldx, const int32_t* rows,
                    int32_t* idx_out, int32_t* stats, void* workspace, int64_t workspace_bytes,
                    void* stream);

/* G = 1 variant fed by pre-split operands: x_hi/x_lo [R, D] bf16 (the LN1 pass
 * writes them, astra_layernorm_ex) and x_norm [R] (an upper bound of ||x_r||).
 * The distance GEMM covers all R source rows; idx_out[m] is produced for the
 * M token rows rows[m] (fp64 re-rank reads x[rows[m]]). */
int64_t astra_vq_encode_split_workspace(int R, int size);
int astra_vq_encode_split(const AstraCodebook* cb, const float* x, int ldx, const void* x_hi,
                          const void* x_lo, int ld_split, const float* x_norm, int R,
                          const int32_t* rows, int M, int32_t* idx_out, int32_t* stats,
                          void* workspace, int64_t workspace_bytes, void* stream);
/* Same, with row_token [R] = the token index of stack row r (-1: not a token row; the inverse
 * of rows), precomputed by the caller.  When the stack has at least as many 256-row blocks as
 * the GPU has CTA pairs, the distance GEMM runs in run mode (a CTA pair sweeps the whole
 * codebook for its rows and decides them in the epilogue; no finalize pass) and uses the map
 * instead of rebuilding it. */
int astra_vq_encode_split_ex(const AstraCodebook* cb, const float* x, int ldx, const void* x_hi,
                             const void* x_lo, int ld_split, const float* x_norm, int R,
                             const int32_t* rows, int M, const int32_t* row_token,
                             int32_t* idx_out, int32_t* stats, void* workspace,
                             int64_t workspace_bytes, void* stream);

/* ------------------------------------------------------------ VQ decode
 * Replaces vq.dequantize (vq.py:225-233): out[m, g*gd:(g+1)*gd] =
 * centroids[g][idx[m, g]].  Out-of-range indices are not dereferenced; they
 * set *err_flag = 1 (caller maps it to IndexCorruptionError). */
int astra_vq_decode(const AstraCodebook* cb, const int32_t* idx, int M, float* out, int ldo,
                    int32_t* err_flag, void* stream);
/* VQ decode fused into LN1 — the K/V projection's A operand for received tokens of grouped
 * codebooks (vq.dequantize vq.py:225-233 -> tensor.layer_norm tensor.py:318-345, as
 * cluster._device_layer_compute does for every remote row, cluster.py:182-198): row m is gathered
 * from the codebook rows idx[m, :] straight into registers, normalised in fp32 exactly like
 * astra_layernorm, and written as bf16 hi[, lo] (pitch ld_bf).  The decoded fp32 row never
 * reaches HBM.  Needs D = G * gd in {512, 768, 1024} and gd % 4 == 0.  Bad codes: *err_flag = 1,
 * the row reads as zeros. */
int astra_vq_decode_layernorm(const AstraCodebook* cb, const int32_t* idx, int M, const float* gain,
                              const float* bias, float eps, void* out_hi, void* out_lo, int ld_bf,
                              int32_t* err_flag, void* stream);

/* ------------------------------------------------------- index wire format
 * The exchanged payload of allgather_indices (cluster.py:144-160; the
 * reference only accounts ceil(log2 K) bits per index, vq.py:24-28): an
 * LSB-first bitstream of `bits`-bit codes in [token, group] order, padded to
 * whole uint32 words. */
int astra_pack_indices(const int32_t* idx, int count, int bits, uint32_t* words, void* stream);
int astra_unpack_indices(const uint32_t* words, int count, int bits, int size, int32_t* idx,
                         int32_t* err_flag, void* stream);

/* ---------------------------------------------------------- block ops
 * tensor.layer_norm (tensor.py:318-345): fp32 row statistics, eps, affine;
 * writes fp32 and/or the bf16 (hi[, lo]) operand of the following GEMM. */
int astra_layernorm(const float* x, int M, int D, int ldx, const float* gain, const float* bias,
                    float eps, float* out_f32, int ld_f32, void* out_hi, void* out_lo, int ld_bf,
                    void* stream);
/* Same, additionally writing the bf16 hi/lo split of the RAW rows (xs_hi/xs_lo,
 * pitch ld_xs) and an upper bound of each row's norm (x_norm) — the operands of
 * astra_vq_encode_split — from the same single read of x. */
int astra_layernorm_ex(const float* x, int M, int D, int ldx, const float* gain, const float* bias,
                       float eps, float* out_f32, int ld_f32, void* out_hi, void* out_lo,
                       int ld_bf, void* xs_hi, void* xs_lo, int ld_xs, float* x_norm,
                       void* stream);

/* Stack assembly: embed_classifier_inputs (model.py:275-280) + replica rows
 * (cluster.py:189-194, :259-262).  row_src[r] >= 0: out[r] = x[row_src[r]] +
 * pos[row_pos[r]];  row_src[r] < 0: out[r] = cls. */
int astra_embed_stack(const float* x, const float* pos, const float* cls, const int32_t* row_src,
                      const int32_t* row_pos, int rows, int D, float* out, void* stream);

/* aggregate_class_tokens / mean_rows (model.py:268-272, tensor.py:200-208):
 * reps [N, B, D] in device order -> out [B, D], summed in device order then / N. */
/* LM embed (replaces embed_lm_inputs, model.py:283-288, on the prefill path):
 * out[r] = emb[ids[row_src[r]]] + pos[row_pos[r]]; ids [B*T] int32 in device memory
 * (validated by the caller), row_src the stack-row -> b*T + t map. */
int astra_embed_tokens(const float* emb, const float* pos, const int32_t* ids,
                       const int32_t* row_src, const int32_t* row_pos, int rows, int D, float* out,
                       void* stream);
int astra_replica_mean(const float* reps, int N, int B, int D, float* out, void* stream);

/* out[r, :D] = src[idx[r], :D] (row gather, 16-byte vectors). */
int astra_gather_rows(const float* src, int lds, const int32_t* idx, int rows, int D, float* out,
                      int ldo, void* stream);

/* Per-layer key map (x_view assembly, cluster.py:182-187): key_map[j] >= 0 is a
 * local key row; < 0 names remote content token t = -(key_map[j]+1), whose key
 * becomes remote row codes[t] (G = 1, codebook K/V table) or t (codes == NULL). */
int astra_key_map(const int32_t* key_map, int n, const int32_t* codes, int32_t* key_src,
                  void* stream);
/* G = 1 fused exchange tail (replaces astra_unpack_indices per sender + astra_key_map):
 * remote keys read their code straight from the all-gathered packed payload — sender e's
 * words start at words[e * wmax], code i of sender e at bit i * bits (LSB first); gofs[e] =
 * first content slot of sender e (nsend + 1 entries).  Codes >= size set *err_flag and map to
 * row 0 (caller raises IndexCorruptionError). */
int astra_key_map_packed(const int32_t* key_map, int n, const uint32_t* words, int wmax, int bits,
                         int size, const int32_t* gofs, int nsend, int32_t* key_src,
                         int32_t* err_flag, void* stream);

/* ------------------------------------------------------ greedy decoding
 * Generation on the device holding the last prompt token (cluster.py:297-308,
 * DecodeState/_decode_one model.py:324-358).  All byte-addressed (any dtype).
 *   gather_kv : cache row (i / n_per) * ld_blocks + i % n_per = [K | V] of key i
 *               picked through key_src (the decoding device's mixed K/V view)
 *   append_kv : cache row b * ld_blocks + pos[b] = [K | V] of the new token b
 *   argmax_rows: out[row * out_stride + (step_pos ? step_pos[row] - pos_base : 0)] =
 *               argmax (lowest index on ties); next_tok[row] too (nullable)
 *   decode_advance: pos[b] += 1; segs[b].qpos0 += 1; segs[b].nk += 1 */
int astra_gather_kv(const int32_t* key_src, int n, int n_per, int ld_blocks, const void* k_local,
                    const void* v_local, int ld_local_bytes, const void* k_remote,
                    const void* v_remote, int ld_remote_bytes, int row_bytes, void* cache,
                    int ld_cache_bytes, void* stream);
int astra_append_kv(const void* k_new, const void* v_new, int ld_new_bytes, int rows,
                    const int32_t* pos, int ld_blocks, int row_bytes, void* cache,
                    int ld_cache_bytes, void* stream);
int astra_argmax_rows(const float* logits, int rows, int cols, int ld, int32_t* out,
                      int out_stride, const int32_t* step_pos, int pos_base, int32_t* next_tok,
                      void* stream);
int astra_decode_advance(int32_t* pos, int32_t* segs, int rows, void* stream);

/* Codebook setup (replaces the centroid update of vq._lloyd, vq.py:160-165, and the
 * per-cluster sums of kmeans_init, vq.py:190-192): mean[c] = sum of pts[order[i]] for
 * i in [seg[c], seg[c+1]) in ascending order, / count — fp64, bit-identical to NumPy's
 * axis-0 mean for the same assignment.  Empty clusters leave mean[c] untouched; sums
 * (optional) receives every cluster's sum. */
int astra_segment_mean_f64(const double* pts, int ld, const int32_t* order, const int32_t* seg,
                           int k, int dim, double* mean, double* sums, void* stream);

/* --------------------------------------------------- mixed-precision attention
 * attention.multihead_attention + tensor.masked_softmax (attention.py:50-73,
 * tensor.py:295-315) over each device's mixed key set (cluster.py:201-212).
 * segs[S, 6] = {q0, nq, qpos0, ncontent, k0, nk} per (device, image) segment;
 * key_src (see astra_key_map) picks local or remote K/V rows; key_pos is the
 * global token position (-1 = class replica key); visible iff !causal ||
 * key_pos <= query_pos.  causal = 2 additionally promises prefix keys (key j of every
 * segment has position j, no replica key), so key chunks past a query tile's last position
 * are skipped.  head_dim 1..128 (64: tcgen05 kernels; fp32 inputs take the split-bf16
 * parity kernel).  in_bf16 selects bf16 inputs; out_hi/out_lo receive the bf16 (split) output,
 * out_f32 the fp32 one. */
int astra_attention(const void* q, int ldq, const void* k_local, const void* v_local, int ld_local,
                    const void* k_remote, const void* v_remote, int ld_remote,
                    const int32_t* key_src, const int32_t* key_pos, const int32_t* segs,
                    int num_segs, int max_nq, int heads, int head_dim, int causal, int in_bf16,
                    float scale, float* out_f32, void* out_hi, void* out_lo, int ld_out,
                    int q_rows, int local_rows, int remote_rows, void* stream);

/* Dense-mask form for the operator API (attention.multihead_attention,
 * attention.py:50-73): q [R, D], k/v [C, D] fp32, mask uint8 [R, C] (nonzero =
 * visible; every row must see a key), scratch >= 6 + 2*C int32 (device). */
int astra_attention_masked(const float* q, const float* k, const float* v, int R, int C, int D,
                           int heads, const uint8_t* mask, int32_t* scratch, float* out,
                           void* stream);

/* Route astra_attention to the fp32 SIMT kernel even when the tcgen05 bf16
 * kernel applies (test / A-B hook). */
int astra_attention_force_simt(int enable);
/* Test hook: tcgen05 variant — 0 persistent two-pipeline (default), 1 one CTA per tile,
   2 persistent single pipeline with correction warps (attention_tcs_kernel). */
int astra_attention_variant(int variant);
/* Programmatic-dependent-launch policy for this host thread's subsequent launches: 0 none,
   1 every kernel, 2 persistent kernels only (default), -1 back to ASTRA_PDL / the default.
   Returns the previous override (-1: none). */
int astra_pdl_override(int mode);
/* Debug hook: CTA 0 of the persistent kernel writes per-unit globaltimer stamps
 * (int64 [64][8]) to buf; NULL disables. */
int astra_attention_trace(void* buf);

#ifdef __cplusplus
}
#endif
#endif /* ASTRA_B200_H */
