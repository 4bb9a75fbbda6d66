/* vecinfer.h -- C ABI of the B200-native VecInfer decode-attention library (libvecinfer.so).
 *
 * VecInfer (arXiv 2510.06175): decode-time self-attention computed directly over a
 * vector-quantized KV cache.  Keys are smoothed (Eq. 3-4) and Hadamard-rotated (Eq. 5-6)
 * before product-VQ encoding (Eq. 2, 8, 9); queries get the matching transform so that
 * q~ K~^T = q K^T (Eq. 7); attention runs over the codes without materialising a dequantized
 * cache (Eq. 10, Algorithm 1).  Citations "P:n" are lines of the paper text PAPER.md.
 *
 * Conventions shared by every entry point
 *  - Every tensor pointer is a DEVICE pointer owned by the caller (e.g. allocated by PyTorch).
 *    The library never allocates device memory, never synchronises the device, and launches
 *    only on the stream it is given.
 *  - Strides are in ELEMENTS; the innermost (head_dim) dimension is always contiguous.
 *  - bf16 tensors are raw IEEE bfloat16 (uint16) buffers.
 *  - A status is returned synchronously after argument validation and before any launch;
 *    VECINFER_ERR_CUDA reports a launch/configuration error (cudaGetLastError); asynchronous
 *    device faults surface at the caller's next synchronisation.  No exception or abort
 *    crosses the ABI.  vecinfer_last_error() returns a thread-local description of the last
 *    non-OK status of the calling thread.
 *  - Thread-safe: no global mutable state except the thread-local error string and a
 *    per-device attribute cache.
 *  - Supported shapes (ABI v6): head_dim D in {128, 64}, sub_dim d = 4, code_bits in {4, 8, 16}
 *    (b1d4, b2d4, b4d4 in BASELINE.json notation = paper d4b4, d4b8, d4b16), K and V
 *    widths independent; GQA group G = H_q / H_kv in 1..8; contiguous or paged code caches.
 *    D = 64: split kernel (residual window, fused append) and, for batch decode without those,
 *    the stream kernel.
 *    The paper's other configurations, D = 128 only:
 *    d8b8 {128, 8, 8}, d8b12 {128, 8, 12}, d4b10 {128, 4, 10}, d2b8 {128, 2, 8}, d8b16
 *    {128, 8, 16} (Table 5's 2-bit row: 65 536 eight-dim centroids, 1 MiB bf16 per book);
 *    attention pairs (f, f) and the mixed K-d4b10 / V-d8b12 and K-d8b12 / V-d8b8 of Table 3, on the split
 *    DEQUANT_MMA kernel (contiguous or paged, residual window allowed; no stream / LUT variant;
 *    decode_step fuses the append for the books held in the kernel's shared tables -- d8b8,
 *    d8b12, d4b10, d2b8 -- and appends d8b16 with a separate encode launch).  The kernel keeps
 *    these books (like the d = 4 ones) as fp16 copies: every centroid value must be exactly
 *    representable in fp16 (0 or 2^-14 <= |c| <= 65504 with <= 11 significant bits; bf16 values
 *    in the fp16 normal range are), else attention and the fused append's codes are not exact.
 *    Anything else returns VECINFER_ERR_UNSUPPORTED.
 *  - ABI v5 adds: n_tokens_max in vecinfer_attn_kernel_kind (the stream/split choice is a cost
 *    model over it), vecinfer_kmeans_step (GPU codebook Lloyd iteration) and the fused
 *    cross-GPU exchange + merge over peer memory (vecinfer_p2p_window_*, vecinfer_merge_lse_p2p).
 *  - ABI v6 adds: the tcgen05 score variant (VECINFER_ATTN_DEQUANT_TC), d8b16, and the
 *    cross-GPU merge fused into the attention launch itself (vecinfer_attn_decode_xr,
 *    vecinfer_decode_step_xr, vecinfer_xr_window_bytes).
 *  - ABI v7 adds: VECINFER_ATTN_FLAG_EARLY_CACHE, OR'ed into the algo argument.
 */
#ifndef VECINFER_H_
#define VECINFER_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VECINFER_ABI_VERSION 7

typedef struct CUstream_st* vecinfer_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  VECINFER_OK = 0,
  VECINFER_ERR_INVALID_ARG = 1, /* NULL / misaligned pointer, bad enum, eps <= 0, bad stride     */
  VECINFER_ERR_SHAPE = 2,       /* non-positive sizes, H_q % H_kv != 0, tok_begin > tok_end, ... */
  VECINFER_ERR_UNSUPPORTED = 3, /* (D, d, code_bits, G) combination without a kernel             */
  VECINFER_ERR_EMPTY = 4,       /* calibration with n_tokens == 0                                */
  VECINFER_ERR_RANGE = 5,       /* (reported through the device err_flags word, see encode_kv)   */
  VECINFER_ERR_WORKSPACE = 6,   /* workspace NULL or smaller than the *_workspace_bytes() query  */
  VECINFER_ERR_CUDA = 7         /* CUDA launch / attribute error                                 */
} vecinfer_status_t;

typedef enum { VECINFER_BF16 = 0, VECINFER_F32 = 1 } vecinfer_dtype_t;

/* Product-VQ configuration: head_dim D, sub-vector dim d, code bits b (2^b centroids).
 * b2d4 = {128, 4, 8}: 256 centroids of 4 dims, one byte per sub-vector. */
typedef struct {
  int32_t head_dim;
  int32_t sub_dim;
  int32_t code_bits;
} vecinfer_vq_t;

/* Score/P.V algorithm of vecinfer_attn_decode.
 *  DEQUANT_MMA: keys are dequantised from a bank-conflict-free replicated codebook into
 *    tensor-core fragments; s = q~ K^T and o = P V both run as fp16 MMAs with hi/lo-split
 *    operands (fp32 accumulate).  Default on sm_100a.
 *  LUT: the paper's Algorithm 1 literally: lut = q~' C_k^T (l.4) in shared
 *    memory, scores by table lookup (l.11), P.V from the dequantised value codebook on CUDA
 *    cores (l.16).  Kept as the paper-faithful variant and for comparison.
 *  DEQUANT_MMA_STREAM: DEQUANT_MMA with the stream partition (units cut into pieces so every
 *    CTA gets the same number of tokens; pieces merged in fixed order).  AUTO selects it for
 *    B*H_kv >= #SMs (batch decode); forcing it here with num_splits = S > 0 gives exactly S
 *    pieces per unit (grid min(B*H_kv*S, #SMs) persistent CTAs).
 *  DEQUANT_TC: the split DEQUANT_MMA kernel with the score contraction (Alg. 1 l.11 as q~ K^T)
 *    on the 5th-generation tensor cores: each 4-warp group stages its 128 gathered K^ rows in
 *    tensor memory (tcgen05.st), one thread issues tcgen05.mma (A = K^ in TMEM, B = q~ hi/lo in
 *    shared memory, fp32 scores in TMEM), the scores return with tcgen05.ld; P.V stays on
 *    mma.sync.  Contiguous caches, D = 128, K codebooks b1d4 / b2d4 (V: b1d4 / b2d4 / b4d4);
 *    anything else is VECINFER_ERR_UNSUPPORTED.  AUTO never selects it: measured slower than
 *    DEQUANT_MMA on B200. */
typedef enum {
  VECINFER_ATTN_AUTO = 0,
  VECINFER_ATTN_DEQUANT_MMA = 1,
  VECINFER_ATTN_LUT = 2,
  VECINFER_ATTN_DEQUANT_MMA_STREAM = 3,
  VECINFER_ATTN_DEQUANT_TC = 4
} vecinfer_attn_algo_t;

/* Launch-ordering hint OR'ed into the algo argument of the attention / decode-step calls (ABI v7):
 * the caller promises that seq_lens, write_pos, the block table and the code caches were NOT
 * written by the kernel immediately preceding this call on the stream (e.g. the preceding kernel
 * is the previous layer's attention or the QKV projection; the step's seq_lens update and the
 * cache writes of earlier launches are at least two kernels back).  The split kernel then reads
 * them, derives its token range and issues its first code tile BEFORE the programmatic-dependent-
 * launch wait, so under PDL these loads overlap the previous kernel's tail; q, k_new / v_new and
 * the residual window are still read after the wait.  The stream kernel does the same for its
 * first round (its segments and first tiles) when no residual window is given.  Results are
 * identical with and without the flag.  Ignored by the LUT kernel and by a decode step that appends
 * with a separate encode launch (that launch writes the cache right before the attention). */
#define VECINFER_ATTN_FLAG_EARLY_CACHE 0x100

/* Paged code cache (serving integration): k_codes / v_codes are a pool of
 * n_pages pages laid out [n_pages, H_kv, page_size, row_bytes]; token t of batch row b lives in
 * page block_table[b * bt_stride + t / page_size] at row t % page_size.  page_size is a power of
 * two >= 32; n_cap (the per-sequence capacity) must not exceed bt_stride * page_size.  Entries
 * outside [0, n_pages) are flagged as VECINFER_FLAG_WRITE_POS by the encoders and must not be
 * reached by attended tokens.  Token ranges must start at a multiple of 32.  The *_paged entry
 * points run the split or the stream attention kernel (the LUT and DEQUANT_TC variants are
 * contiguous-only).
 *   block_table  device int32 [B, bt_stride] (caller owned).                                   */
typedef struct {
  const int32_t* block_table;
  int64_t bt_stride;
  int32_t page_size;
  int32_t n_pages;
} vecinfer_paged_t;

/* Full-precision residual window ("the residual length for all methods is set to 128";
 * SURVEY §8(f) NEXT-1): the newest tokens of each sequence kept as raw bf16 k, v rows next to the
 * VQ cache.  Attention runs one softmax over the quantised tokens [tok range of seq_lens] and the
 * residual rows [0, lens[b]); residual scores use the raw q (q k^T = q~ k~^T, Eq. 7).
 *   k, v        bf16 [B, H_kv, r_cap, D]; element (b, h, t, c) at b*stride_b + h*stride_h + t*D + c.
 *   lens        device int32 [B] rows in use (0 = none).
 *   append_new  vecinfer_decode_step only: 1 = the new token is written to residual row lens[b]-1
 *               (raw bf16 copy, no encode) instead of being encoded into the codes.
 * The caller flushes old residual rows into the codes (vecinfer_encode_kv) when the window fills. */
typedef struct {
  const void* k;
  const void* v;
  int64_t stride_b, stride_h;
  int64_t r_cap;
  const int32_t* lens;
  int32_t append_new;
} vecinfer_residual_t;

/* Device-side error bits written (atomicOr) into the optional err_flags word of encode_kv. */
#define VECINFER_FLAG_RANGE 1u     /* |k * inv_lambda| >= 2^32: outside the pinned fixed point */
#define VECINFER_FLAG_WRITE_POS 2u /* write_pos[b] + t outside [0, n_cap): row not written     */
#define VECINFER_FLAG_P2P_TIMEOUT 4u /* vecinfer_merge_lse_p2p: a peer's partial did not arrive  */

/* Programmatic dependent launch: every kernel is launched with PDL and reads only the static
 * weights (codebooks) before griddepcontrol.wait, so codebooks must not be produced by the
 * kernel immediately preceding a call on the same stream.  All other inputs may be. */

int vecinfer_abi_version(void);
const char* vecinfer_last_error(void);
const char* vecinfer_status_string(vecinfer_status_t status);

/* ---------------------------------------------------------------------------------------
 * Smoothing-factor calibration, Eq. 4: lambda_c = sqrt(max_n |K[n, h, c]|).
 *   k_cal        bf16 [n_tokens, n_kv_heads, head_dim], element (n, h, c) at
 *                n * stride_tok + h * stride_head + c.
 *   eps_floor    > 0; lambda = max(RN32(sqrt(amax)), RN32(eps_floor)) (SPEC S:91 floor).
 *   lambda_out, inv_lambda_out   fp32 [n_kv_heads, head_dim]; inv_lambda = RN32(1 / lambda).
 *   workspace    >= vecinfer_calibrate_workspace_bytes(n_kv_heads, head_dim) bytes; contents
 *                are overwritten (zeroed on the stream before use).
 * Errors: INVALID_ARG (NULL, eps <= 0, stride_head < head_dim when n_kv_heads > 1),
 *         EMPTY (n_tokens == 0), SHAPE (head_dim % 8 != 0 or <= 0), WORKSPACE, CUDA.
 * ------------------------------------------------------------------------------------- */
size_t vecinfer_calibrate_workspace_bytes(int32_t n_kv_heads, int32_t head_dim);
vecinfer_status_t vecinfer_calibrate_smooth(const void* k_cal_bf16, int64_t n_tokens,
                                            int32_t n_kv_heads, int32_t head_dim,
                                            int64_t stride_tok, int64_t stride_head,
                                            float eps_floor, float* lambda_out,
                                            float* inv_lambda_out, void* workspace,
                                            size_t workspace_bytes, vecinfer_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * KV encode + cache store: prefill (Eq. 8, T tokens) and decode append (Eq. 9,
 * P:241-249, T = 1).  Per (b, t, h):
 *   key:   x = (k diag(lambda)^-1) H_D (S then H) on the pinned exact fixed point
 *          (R10): A = rint(k*inv_lambda*2^24) in int64, X = A H_pm (warp-shuffle
 *          FWHT, exact), x = RN32(RN32(X) * 2^-24) * RN32(1/sqrt(D)); then
 *          code[m] = argmin_j ||x_m - C_k[j]||^2 (Eq. 2).
 *   value: code[m] = argmin_j ||v_m - C_v[j]||^2 (values are not transformed, Eq. 8).
 *   Distances: fp32, each op round-to-nearest, no FMA, order ((e0^2+e1^2)+e2^2)+e3^2; ties to
 *   the lowest index (R9).  Codes are bit-identical to the CPU oracle.
 *   k_bf16, v_bf16   [B, T, H_kv, D] with element strides (b, t, h) in k_strides / v_strides.
 *   inv_lambda       fp32 [H_kv, D] (from vecinfer_calibrate_smooth).
 *   ck_bf16, cv_bf16 codebooks [H_kv, 2^b, d] bf16; *_head_stride = elements between heads,
 *                    0 = one codebook shared by all heads.
 *   k_codes, v_codes uint8 [B, H_kv, n_cap, D/d*b/8] token-major packed rows (R11: the row is
 *                    one little-endian bit string, code m in bits [m b, m b + b) -- 8-bit one
 *                    byte per sub-vector; 4-bit sub-vector 2i low nibble, 2i+1 high nibble;
 *                    16-bit little-endian u16; 10/12-bit codes straddle bytes).
 *   (d = 8 / 2 distances sum the d squared differences left to right in the same way; the
 *    NEXT-2 formats are encoded by one CTA per (token-head, K or V) that scans the codebook
 *    with all 256 threads and reduces (dist_bits << 32 | index) minima.)
 *   write_pos        device int32 [B]: cache row of token t = 0 of batch b (e.g. seq_len).
 *   err_flags        device uint32 (may be NULL): VECINFER_FLAG_* bits are OR-ed in.
 *   workspace        >= vecinfer_encode_workspace_bytes(B, T, H_kv, kcfg, vcfg) bytes (0 for
 *                    4/8-bit codebooks, which are searched from shared memory).  16-bit codebooks
 *                    (65 536 entries) are searched in passes of <= 512 token-heads by a tensor-core
 *                    filter (mma bf16 over a_j = ||c_j||^2 - 2 x.c_j with a rigorous error bound)
 *                    that keeps, per sub-vector and 512-centroid chunk, bounds on the chunk's best
 *                    approximate distance, and an exact selection that rescans only the chunks
 *                    that can hold the pinned-distance argmin (codes identical to the full scan):
 *                    min(B*T, max(1, 512/H_kv)) * H_kv * 64 KiB.  Contents on entry are never read
 *                    before written; every word the call writes is zero again on exit (a
 *                    zero-filled workspace stays zero).  ABI v7: was B*T*H_kv*516 bytes.
 * Errors: INVALID_ARG, SHAPE, UNSUPPORTED, WORKSPACE, CUDA.
 * ------------------------------------------------------------------------------------- */
size_t vecinfer_encode_workspace_bytes(int32_t B, int32_t T, int32_t H_kv, vecinfer_vq_t kcfg,
                                       vecinfer_vq_t vcfg);
vecinfer_status_t vecinfer_encode_kv(const void* k_bf16, const void* v_bf16, int32_t B,
                                     int32_t T, int32_t H_kv, const int64_t k_strides[3],
                                     const int64_t v_strides[3], const float* inv_lambda,
                                     const void* ck_bf16, const void* cv_bf16,
                                     int64_t ck_head_stride, int64_t cv_head_stride,
                                     vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes,
                                     uint8_t* v_codes, int64_t n_cap, const int32_t* write_pos,
                                     uint32_t* err_flags, void* workspace, size_t workspace_bytes,
                                     vecinfer_stream_t stream);
/* vecinfer_encode_kv into a paged code cache (vecinfer_paged_t; same arguments otherwise). */
vecinfer_status_t vecinfer_encode_kv_paged(const void* k_bf16, const void* v_bf16, int32_t B,
                                           int32_t T, int32_t H_kv, const int64_t k_strides[3],
                                           const int64_t v_strides[3], const float* inv_lambda,
                                           const void* ck_bf16, const void* cv_bf16,
                                           int64_t ck_head_stride, int64_t cv_head_stride,
                                           vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes,
                                           uint8_t* v_codes, int64_t n_cap, const int32_t* write_pos,
                                           uint32_t* err_flags, void* workspace,
                                           size_t workspace_bytes, vecinfer_stream_t stream,
                                           const vecinfer_paged_t* paged);

/* ---------------------------------------------------------------------------------------
 * Fused decode attention over the VQ cache, Eq. 10 + Algorithm 1,
 * split-KV generalised to a stream partition: the B*H_kv units (b, h_kv) are cut into
 * pieces so that every CTA (one per SM) gets the same number of tokens; the log-sum-exp merge
 * of the pieces of a split unit is fused into the same launch (fixed piece order).
 *   q_bf16      [B, H_q, D] raw queries (strides q_stride_b, q_stride_h); query head i reads
 *               KV head i / G (GQA, G = H_q / H_kv in 1..8; groups of 5..8 run as two virtual KV
 *               heads of <= 4 query heads that share the codes).  The kernel applies
 *               q~ = q diag(lambda) H_D (Eq. 7).
 *   lambda      fp32 [H_kv, D].
 *   codebooks / codes / n_cap as in vecinfer_encode_kv (kcfg, vcfg may differ).
 *   seq_lens    device int32 [B]; tokens [tok_begin, min(tok_end, seq_len)) are attended
 *               (tok_end < 0 means "to seq_len"): the sharding hook for multi-GPU splits.
 *   softmax_scale  usually 1/sqrt(D).
 *   num_splits  0 = heuristic (fill the SMs); S > 0 = exactly S pieces per unit.  Results are
 *               bitwise reproducible for a fixed (shape, num_splits, device SM count).
 *   o           [B, H_q, D] bf16 or fp32 (o_dtype); lse fp32 [B, H_q] natural log.
 *               An empty range yields o = 0, lse = -inf (weight 0 in vecinfer_merge_lse).
 *   residual    optional full-precision window (NULL = none); row t of a unit is attended by
 *               its piece t % P (P = pieces of the unit);
 *               LUT variant: not supported (VECINFER_ERR_UNSUPPORTED).
 *   workspace   >= vecinfer_attn_workspace_bytes(B, H_q, H_kv, D, n_tokens_max, num_splits)
 *               bytes, where n_tokens_max bounds the attended range; MUST be zero-filled once
 *               when first allocated.  Every launch leaves the whole workspace zero on exit, so
 *               one workspace may serve calls of any shape that it is large enough for.
 * Errors: INVALID_ARG, SHAPE, UNSUPPORTED, WORKSPACE, CUDA.
 * ------------------------------------------------------------------------------------- */
/* pieces per unit (num_splits if > 0, else the heuristic's upper bound), and the number of
 * virtual CTAs V of the partition (the grid is min(V, #SMs) persistent CTAs).  These queries and
 * vecinfer_attn_kernel_kind / vecinfer_decode_step_launches take the number of attention units per
 * batch row as H_kv: pass 2 * H_kv when H_q / H_kv > 4 (virtual KV heads). */
int32_t vecinfer_attn_num_splits(int32_t B, int32_t H_kv, int64_t n_tokens_max,
                                 int32_t num_splits);
int32_t vecinfer_attn_num_ctas(int32_t B, int32_t H_kv, int64_t n_tokens_max,
                               int32_t num_splits);
/* which kernel a call with these arguments runs: 0 = split kernel, 1 = stream kernel, 2 = LUT.
 * AUTO picks the stream partition when B*H_kv >= #SMs, and below that when a cost model over
 * n_tokens_max (the attended range) says the split plan's waves leave more SMs idle than the
 * stream partition's fixed costs (e.g. B = 8..16 at 32k tokens, 8 KV heads).  (ABI v5: n_tokens_max
 * added.) */
int32_t vecinfer_attn_kernel_kind(int32_t B, int32_t H_kv, int64_t n_tokens_max, int32_t num_splits,
                                  vecinfer_attn_algo_t algo);
size_t vecinfer_attn_workspace_bytes(int32_t B, int32_t H_q, int32_t H_kv, int32_t D,
                                     int64_t n_tokens_max, int32_t num_splits);
vecinfer_status_t vecinfer_attn_decode(const void* q_bf16, int32_t B, int32_t H_q,
                                       int32_t H_kv, int64_t q_stride_b, int64_t q_stride_h,
                                       const float* lambda, const void* ck_bf16,
                                       const void* cv_bf16, int64_t ck_head_stride,
                                       int64_t cv_head_stride, vecinfer_vq_t kcfg,
                                       vecinfer_vq_t vcfg, const uint8_t* k_codes,
                                       const uint8_t* v_codes, int64_t n_cap,
                                       const int32_t* seq_lens, int64_t tok_begin,
                                       int64_t tok_end, float softmax_scale, int32_t num_splits,
                                       vecinfer_attn_algo_t algo, void* o,
                                       vecinfer_dtype_t o_dtype, float* lse, void* workspace,
                                       size_t workspace_bytes, vecinfer_stream_t stream,
                                       const vecinfer_residual_t* residual);
/* vecinfer_attn_decode over a paged code cache (tok_begin % 32 == 0).  The split kernel and, for
 * batch decode (AUTO's choice or DEQUANT_MMA_STREAM), the stream kernel: every 16-token sub-tile
 * is translated through the block table; results equal the contiguous cache bit for bit. */
vecinfer_status_t vecinfer_attn_decode_paged(const void* q_bf16, int32_t B, int32_t H_q,
                                             int32_t H_kv, int64_t q_stride_b, int64_t q_stride_h,
                                             const float* lambda, const void* ck_bf16,
                                             const void* cv_bf16, int64_t ck_head_stride,
                                             int64_t cv_head_stride, vecinfer_vq_t kcfg,
                                             vecinfer_vq_t vcfg, const uint8_t* k_codes,
                                             const uint8_t* v_codes, int64_t n_cap,
                                             const int32_t* seq_lens, int64_t tok_begin,
                                             int64_t tok_end, float softmax_scale,
                                             int32_t num_splits, vecinfer_attn_algo_t algo, void* o,
                                             vecinfer_dtype_t o_dtype, float* lse, void* workspace,
                                             size_t workspace_bytes, vecinfer_stream_t stream,
                                             const vecinfer_residual_t* residual,
                                             const vecinfer_paged_t* paged);

/* ---------------------------------------------------------------------------------------
 * Fused decode step for one layer: EXACTLY vecinfer_encode_kv(T = 1) of the new token followed
 * by vecinfer_attn_decode over [0, seq_lens[b]) (Eq. 9 then Eq. 10), in one launch.
 * The split of each (b, h_kv) whose range holds row write_pos[b] (else split 0) encodes the new
 * k, v in its prologue (centroid scan split over its 16 warps, bit-identical codes), writes them
 * to the cache and uses them for that row; all other work is the plain attention kernel.
 *   q_bf16     [B, H_q, D] (strides q_strides = {b, h});  k_new_bf16, v_new_bf16 [B, H_kv, D]
 *              (strides {b, h}); inv_lambda as in encode_kv; lambda as in attn_decode.
 *   k_codes, v_codes  the code caches (written at row write_pos[b], read over [0, seq_lens[b])).
 *   Other arguments as in vecinfer_attn_decode (token range = whole sequence) and
 *   vecinfer_encode_kv (err_flags); workspace >= vecinfer_decode_step_workspace_bytes(...), zero-
 *   filled once.  The append runs inside the attention launch for the d = 4 books of 16 / 256
 *   entries (b1d4, b2d4, any K/V mix of them) and for d8b8 / d8b12 / d4b10 / d2b8 and their mixed
 *   pairs when the grid is one wave (the stream partition always budgets it).  Otherwise it runs
 *   first as its own encode (same codes): grids of several waves, the LUT variant, and the
 *   65 536-entry books (b4d4, d8b16) through the tensor-core filter + exact selection of
 *   vecinfer_encode_kv (two launches).  vecinfer_decode_step_launches reports the count.
 * Errors: as vecinfer_encode_kv and vecinfer_attn_decode.
 * ------------------------------------------------------------------------------------- */
/* kernel launches one vecinfer_decode_step call makes (1: the append is fused into attention) */
int32_t vecinfer_decode_step_launches(int32_t B, int32_t H_kv, int64_t n_cap, vecinfer_vq_t kcfg,
                                      vecinfer_vq_t vcfg, int32_t num_splits,
                                      vecinfer_attn_algo_t algo, int32_t residual_append);
size_t vecinfer_decode_step_workspace_bytes(int32_t B, int32_t H_q, int32_t H_kv, int64_t n_cap,
                                            vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, int32_t num_splits);
vecinfer_status_t vecinfer_decode_step(const void* q_bf16, const void* k_new_bf16, const void* v_new_bf16,
                                       int32_t B, int32_t H_q, int32_t H_kv, const int64_t q_strides[2],
                                       const int64_t k_new_strides[2], const int64_t v_new_strides[2],
                                       const float* lambda, const float* inv_lambda, const void* ck_bf16,
                                       const void* cv_bf16, int64_t ck_head_stride, int64_t cv_head_stride,
                                       vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes,
                                       uint8_t* v_codes, int64_t n_cap, const int32_t* write_pos,
                                       const int32_t* seq_lens, float softmax_scale, int32_t num_splits,
                                       vecinfer_attn_algo_t algo, void* o, vecinfer_dtype_t o_dtype,
                                       float* lse, uint32_t* err_flags, void* workspace,
                                       size_t workspace_bytes, vecinfer_stream_t stream,
                                       const vecinfer_residual_t* residual);
/* vecinfer_decode_step over a paged code cache (append row write_pos[b] translated through the
 * block table; split kernel). */
vecinfer_status_t vecinfer_decode_step_paged(
    const void* q_bf16, const void* k_new_bf16, const void* v_new_bf16, int32_t B, int32_t H_q,
    int32_t H_kv, const int64_t q_strides[2], const int64_t k_new_strides[2],
    const int64_t v_new_strides[2], const float* lambda, const float* inv_lambda,
    const void* ck_bf16, const void* cv_bf16, int64_t ck_head_stride, int64_t cv_head_stride,
    vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes, uint8_t* v_codes, int64_t n_cap,
    const int32_t* write_pos, const int32_t* seq_lens, float softmax_scale, int32_t num_splits,
    vecinfer_attn_algo_t algo, void* o, vecinfer_dtype_t o_dtype, float* lse, uint32_t* err_flags,
    void* workspace, size_t workspace_bytes, vecinfer_stream_t stream,
    const vecinfer_residual_t* residual, const vecinfer_paged_t* paged);

/* ---------------------------------------------------------------------------------------
 * Log-sum-exp merge of P normalised partials (cross-GPU sequence shards, residual window):
 *   L = logsumexp_s L_s;  o = sum_s exp(L_s - L) o_s, summed in the fixed order s = 0..P-1
 *   (the online-softmax recurrence of P:745-757 applied to whole partials).
 *   o_parts fp32 [P, B, H_q, D] (normalised), lse_parts fp32 [P, B, H_q] (natural log);
 *   partials with lse = -inf have zero weight; all -inf -> o = 0, lse = -inf.
 *   o [B, H_q, D] bf16 or fp32; lse fp32 [B, H_q] (may be NULL).
 * Errors: INVALID_ARG, SHAPE, CUDA.
 * ------------------------------------------------------------------------------------- */
vecinfer_status_t vecinfer_merge_lse(const float* o_parts, const float* lse_parts, int32_t P,
                                     int32_t B, int32_t H_q, int32_t D, void* o,
                                     vecinfer_dtype_t o_dtype, float* lse,
                                     vecinfer_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * vecinfer_kmeans_step -- one Lloyd iteration of the codebook k-means (offline step of the
 * method: "C_k ... via K-means"; "K-means ... maximum number of iterations set to 30",
 * P:501; empty-cluster re-seeding at the largest-distortion points).  NEXT-3.
 *   X          fp32 [n, d] points (row-major, contiguous), d in {2, 4, 8}; n >= k, n < 2^32 - 1.
 *   C          fp32 [k, d] current centroids, 0 < k <= 65536.
 *   C_new      fp32 [k, d] out: RN32(mean of the cluster's points) for non-empty clusters, the sum
 *              taken exactly in int64 fixed point (each x rounded to a 2^-e grid, e chosen from
 *              max|x|, max|C| and n so that no sum overflows), then / 2^e / count in fp64; the
 *              empty clusters, in increasing index, take the points of largest best distance
 *              (ties: lowest point index).  May alias C.
 *   assign     int32 [n] out: argmin_j of the pinned fp32 distance (the encoder's rule: e = x - c,
 *              ((e_0^2 + e_1^2) + e_2^2) + ..., RN, no FMA), ties to the lowest index.
 *   best       fp32 [n] out: the pinned distance to the assigned centroid.
 *   objective  fp64 device scalar out: sum_i best_i (exact int64 fixed-point sum, as above).
 *   workspace  >= vecinfer_kmeans_workspace_bytes(k, d) bytes, 256-byte aligned, any contents.
 * Bitwise deterministic run to run (integer sums do not depend on the order the atomics land in;
 * SPEC S:128, 187).  C_new is within one fp32 ulp of the exactly rounded mean (the fixed-point
 * rounding of each point, <= 2^-(e+1)).  Launches 4 kernels + 1 memset on `stream`.
 * Errors: INVALID_ARG (NULL / misaligned), UNSUPPORTED (d), SHAPE (k, n), EMPTY (n == 0),
 * WORKSPACE, CUDA.
 * ------------------------------------------------------------------------------------- */
size_t vecinfer_kmeans_workspace_bytes(int32_t k, int32_t d);
vecinfer_status_t vecinfer_kmeans_step(const float* X, int64_t n, int32_t d, const float* C,
                                       int32_t k, float* C_new, int32_t* assign, float* best,
                                       double* objective, void* workspace, size_t workspace_bytes,
                                       vecinfer_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Cross-GPU exchange fused with the LSE merge over peer memory (sequence-sharded
 * 196k decoding, BASELINE configs[3]).  The all-gather + vecinfer_merge_lse pair becomes ONE
 * kernel: every rank stores its partial rows straight into every peer's window (CUDA IPC mapping;
 * NVLink / NVSwitch P2P between GPUs), raises a per-row flag, waits for the P flags of its own
 * window and merges the P partials in rank order with vecinfer_merge_lse's arithmetic (bitwise the
 * same result on every rank, and the same as all-gather + merge_lse).
 *
 * Setup (not on the hot path; these calls allocate / map and synchronise):
 *   vecinfer_p2p_window_bytes(P, rows, D)      window size for P ranks, rows = B * H_q rows of D.
 *   vecinfer_p2p_window_create(bytes, &w, h)   cudaMalloc + zero the own window, export its CUDA
 *                                              IPC handle h (64 bytes) for the peers.
 *   vecinfer_p2p_window_open(h, &w)            map a peer's window (cudaIpcOpenMemHandle).
 *   vecinfer_p2p_window_close(w) / _destroy(w) unmap a peer's window / free the own window.
 * vecinfer_merge_lse_p2p:
 *   o_local, lse_local  this rank's normalised partial fp32 [B, H_q, D] / [B, H_q] (natural log).
 *   windows             DEVICE array of P window pointers as mapped in this process, windows[rank]
 *                       = the own window; every rank must pass the same P, B, H_q, D.
 *   epoch               0 = automatic (a counter in the own window's header, advanced by the
 *                       kernel itself: graph-capturable); else explicit 1, 2, 3, ...  Either way
 *                       every rank must make the same sequence of calls (slots are double-buffered
 *                       by epoch parity; do not mix explicit and automatic on one window).
 *   o, o_dtype, lse     merged output [B, H_q, D] / [B, H_q].
 *   err_flags           device uint32 (may be NULL): VECINFER_FLAG_P2P_TIMEOUT if a peer's rows
 *                       did not arrive within 5 s (outputs are then zero / -inf, never a hang).
 * Errors: INVALID_ARG, SHAPE (P, rank, D <= 1024), CUDA.
 * ------------------------------------------------------------------------------------- */
size_t vecinfer_p2p_window_bytes(int32_t P, int64_t rows, int32_t D);
vecinfer_status_t vecinfer_p2p_window_create(size_t bytes, void** window, void* ipc_handle);
vecinfer_status_t vecinfer_p2p_window_open(const void* ipc_handle, void** window);
vecinfer_status_t vecinfer_p2p_window_close(void* window);
vecinfer_status_t vecinfer_p2p_window_destroy(void* window);
vecinfer_status_t vecinfer_merge_lse_p2p(const float* o_local, const float* lse_local,
                                         void* const* windows, int32_t P, int32_t rank, int32_t B,
                                         int32_t H_q, int32_t D, uint32_t epoch, void* o,
                                         vecinfer_dtype_t o_dtype, float* lse, uint32_t* err_flags,
                                         vecinfer_stream_t stream);

/* ---------------------------------------------------------------------------------------
 * Sequence-sharded attention with the cross-GPU merge fused into the attention launch (SURVEY
 * §8(e): "N4's epilogue stores partials straight into peers' symmetric windows ... then local N5").
 * Each rank attends its own token shard (its own cache, as vecinfer_attn_decode /
 * vecinfer_decode_step); inside the same launch every CTA merges its slice of outputs over the
 * rank's S splits (the single-wave spin merge), stores the slice's rank partial (o_r, L_r) as
 * self-validating 64-bit words straight into every rank's window, waits for the P partials of its
 * slice in its own window, and merges them (log-sum-exp, Alg. 1 l.729-730 / S:314-322) into the
 * FINAL o and lse.  No separate exchange kernel, no host round trip, graph-capturable.
 *   xr.world, xr.rank  P ranks, this rank (0 <= rank < P <= 16); every rank calls with the same
 *                      B, H_q, D and the same sequence of calls (slots alternate by a launch
 *                      counter in the own window's header: a rank may run at most one call ahead).
 *   xr.windows         DEVICE array [P] of window pointers as mapped in this process (windows from
 *                      vecinfer_p2p_window_create / _open, sized by vecinfer_xr_window_bytes;
 *                      windows[rank] = the own window).  Zero-initialised by create; left
 *                      consistent by every call.
 *   xr.rows_max        rows (B * H_q) the windows were sized for.
 *   xr.err_flags       device uint32 (may be NULL): VECINFER_FLAG_P2P_TIMEOUT if a peer's partial
 *                      did not arrive within 5 s (that rank's share then counts as empty).
 * The launch must be a single wave of the split kernel: B * H_kv * S <= #SMs with S >= 2 splits
 * (the planner's S, raised to 2 if it chose 1).  Contiguous caches, DEQUANT_MMA / AUTO (not the
 * stream partition, the LUT or the tcgen05 variant).  Otherwise UNSUPPORTED: use
 * vecinfer_attn_decode + vecinfer_merge_lse_p2p.  o / lse receive the merged result on every rank.
 * ------------------------------------------------------------------------------------- */
typedef struct {
  int32_t world;
  int32_t rank;
  void* const* windows;
  int64_t rows_max;
  uint32_t* err_flags;
} vecinfer_xrank_t;
size_t vecinfer_xr_window_bytes(int32_t P, int64_t rows, int32_t D);
vecinfer_status_t vecinfer_attn_decode_xr(const void* q_bf16, int32_t B, int32_t H_q, int32_t H_kv,
                                          int64_t q_stride_b, int64_t q_stride_h, const float* lambda,
                                          const void* ck_bf16, const void* cv_bf16, int64_t ck_head_stride,
                                          int64_t cv_head_stride, vecinfer_vq_t kcfg, vecinfer_vq_t vcfg,
                                          const uint8_t* k_codes, const uint8_t* v_codes, int64_t n_cap,
                                          const int32_t* seq_lens, int64_t tok_begin, int64_t tok_end,
                                          float softmax_scale, int32_t num_splits, vecinfer_attn_algo_t algo,
                                          void* o, vecinfer_dtype_t o_dtype, float* lse, void* workspace,
                                          size_t workspace_bytes, vecinfer_stream_t stream,
                                          const vecinfer_residual_t* residual, const vecinfer_xrank_t* xr);
vecinfer_status_t vecinfer_decode_step_xr(const void* q_bf16, const void* k_new_bf16, const void* v_new_bf16,
                                          int32_t B, int32_t H_q, int32_t H_kv, const int64_t q_strides[2],
                                          const int64_t k_new_strides[2], const int64_t v_new_strides[2],
                                          const float* lambda, const float* inv_lambda, const void* ck_bf16,
                                          const void* cv_bf16, int64_t ck_head_stride, int64_t cv_head_stride,
                                          vecinfer_vq_t kcfg, vecinfer_vq_t vcfg, uint8_t* k_codes,
                                          uint8_t* v_codes, int64_t n_cap, const int32_t* write_pos,
                                          const int32_t* seq_lens, float softmax_scale, int32_t num_splits,
                                          vecinfer_attn_algo_t algo, void* o, vecinfer_dtype_t o_dtype,
                                          float* lse, uint32_t* err_flags, void* workspace,
                                          size_t workspace_bytes, vecinfer_stream_t stream,
                                          const vecinfer_residual_t* residual, const vecinfer_xrank_t* xr);

/* Diagnostics: how many thread-block clusters of `cluster_size` CTAs of the attention kernel can
 * be co-resident on the current device (0 = not schedulable); used by the split planner. */
int32_t vecinfer_debug_attn_max_clusters(int32_t cluster_size);

#ifdef __cplusplus
}
#endif
#endif /* VECINFER_H_ */
