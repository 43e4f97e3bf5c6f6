/*
 * tadakv_b200.h — C ABI of libtadakv_b200.so, the B200 (sm_100a) implementation of
 * the TaDA KV-cache hot path (arxiv 2506.04642).
 *
 * The reference (tadakv 0.1.0, /root/reference/pkg) is pure Python + numpy and has
 * no FFI of its own; its boundary is the Python API re-exported in
 * pkg/src/tadakv/__init__.py:10-50.  Each entry point below replaces the body of
 * one reference function (cited per function); the Python package
 * paper_2506_04642_b200 binds them with ctypes and keeps the
 * reference names, argument meaning and error types.
 *
 * Conventions
 *  - All pointers are DEVICE pointers owned by the caller (torch tensors in the
 *    Python host); the library never allocates, frees or synchronises.
 *  - Work is enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy).
 *  - Return value: TADA_OK or a TADA_ERR_* code; tada_last_error() has the text.
 *    Argument validation happens before anything is enqueued, so an error return
 *    leaves all buffers untouched (reference errors are raised before mutation).
 *  - Non-finite inputs cannot be detected on the host without a sync: kernels
 *    OR 1 into *err_flag (a device int32) and the host raises DataError when it
 *    reads the flag (quant.py:151-152 semantics).
 *  - Group order is row-major (token, head): group id = t*H + h (quant.py:200-207).
 *  - Packing is LSB-first, 8/bits codes per byte, each group padded to a byte
 *    boundary (quant.py:93-111).  bits = 16 is the raw-f32 pass-through
 *    (quant.py:208-219) with scale = min = 0.
 */
#ifndef TADAKV_B200_H
#define TADAKV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TADA_ABI_VERSION 1

enum tada_status {
  TADA_OK = 0,
  TADA_ERR_SHAPE = 1,  /* ShapeError  (errors.py:8)  */
  TADA_ERR_CONFIG = 2, /* ConfigError (errors.py:12) */
  TADA_ERR_DATA = 3,   /* DataError   (errors.py:16) */
  TADA_ERR_FORMAT = 4, /* FormatError (errors.py:20) */
  TADA_ERR_STATE = 5,  /* StateError  (errors.py:24) */
  TADA_ERR_CUDA = 6    /* launch / runtime failure   */
};

enum tada_dtype { TADA_F32 = 0, TADA_BF16 = 1 };

/*
 * Paged layout of one layer's compressed cache (replaces the growing numpy
 * arrays of CompressedLayerCache, cache.py:130-135).  A page holds
 * `page_tokens` consecutive compressed tokens of one sequence; within a page,
 * for side K then V:
 *   mean  [page_tokens][head_dim]            f32           (cache.py:109)
 *   codes [page_tokens][heads][group_bytes]  packed u8     (quant.py:226)
 *   meta  [page_tokens][heads] {scale, min}  f32 x 2       (quant.py:174)
 * Every block starts 128-byte aligned; page_bytes is a multiple of 256.
 * All layers of a model share one page table (they append the same tokens);
 * each layer has its own pool and layout (its own bit width, PrecisionPlan
 * cache.py:38-63).
 */
typedef struct tada_page_layout {
  int32_t page_tokens;
  int32_t heads;
  int32_t head_dim;
  int32_t bits;        /* 2, 4, 8 or 16 */
  int32_t group_bytes; /* bytes_per_group(head_dim, bits), quant.py:34-38 */
  int32_t reserved;
  int64_t page_bytes;
  int64_t off_mean[2];  /* [side]: 0 = K, 1 = V */
  int64_t off_codes[2];
  int64_t off_meta[2];
} tada_page_layout;

/* ---------------------------------------------------------------- library */
int tada_abi_version(void);
/* Kernels this library has launched so far in this process (all entry points, all streams). */
int64_t tada_launch_count(void);
const char* tada_last_error(void);
/* bytes_per_group (quant.py:34-38); -1 on bad width. */
int64_t tada_bytes_per_group(int32_t group_size, int32_t bits);
/* Fill *out for the given geometry (validate_bits, quant.py:28-31). */
int tada_page_layout_init(int32_t page_tokens, int32_t heads, int32_t head_dim, int32_t bits,
                          tada_page_layout* out);

/* ---------------------------------------------------------------- quantizer
 * quantize_tensor / _quantize_rows / pack_codes (quant.py:200-229, 143-174, 93-111).
 * rows: [n_groups][group_size] (f32 or bf16).  codes: n_groups * group_bytes bytes.
 * scales, mins: [n_groups] f32.  Bit-exact with the reference's fp64 arithmetic. */
int tada_quantize_groups(const void* rows, int32_t dtype, int64_t n_groups, int32_t group_size,
                         int32_t bits, uint8_t* codes, float* scales, float* mins,
                         int32_t* err_flag, void* stream);

/* dequantize_groups / dequantize_tensor (quant.py:232-245, 177-180).
 * select: optional [n_select] int64 group ids (NULL = all n_groups, in order).
 * out: [n_out][group_size] f32 with f32(f64 min + f64 code * f64 scale). */
int tada_dequantize_groups(const uint8_t* codes, const float* scales, const float* mins,
                           int64_t n_groups, int32_t group_size, int32_t bits,
                           const int64_t* select, int64_t n_select, float* out, void* stream);

/* pack_codes / unpack_codes (quant.py:93-111, 114-140); codes are u8 in [0, 2^bits). */
int tada_pack_codes(const uint8_t* codes, int64_t n_groups, int32_t group_size, int32_t bits,
                    uint8_t* packed, void* stream);
int tada_unpack_codes(const uint8_t* packed, int64_t n_groups, int32_t group_size, int32_t bits,
                      const int64_t* select, int64_t n_select, uint8_t* codes, void* stream);

/* mean_center (cache.py:98-111): mean[t][d] = f32(sum_h f64 x / H) in head order,
 * dev[t][h][d] = mean - x. */
int tada_mean_center(const void* x, int32_t dtype, int64_t tokens, int32_t heads, int32_t head_dim,
                     float* mean, float* dev, int32_t* err_flag, void* stream);

/* ---------------------------------------------------------------- K1: quantize-on-append
 * Fused mean_center + quantize + pack of fresh K/V rows straight into the paged
 * layout: the body of _compress_block (cache.py:182-188) for every token that
 * append_tokens (cache.py:154-180) moves into the compressed region.
 * src_k/src_v: [batch][src_seq_stride][heads][head_dim] (f32 or bf16); tokens
 * i in [0, n_tok) of sequence b go to compressed index dst_start[b] + i
 * + dst_offset (dst_start: device int32[batch]) via
 * page_table[b * pt_stride + idx / page_tokens]. */
int tada_quant_append(const tada_page_layout* layout, uint8_t* pool, const void* src_k,
                      const void* src_v, int32_t dtype, int32_t batch, int64_t n_tok,
                      int64_t src_seq_stride, const int32_t* page_table, int32_t pt_stride,
                      const int32_t* dst_start, int64_t dst_offset, int32_t* err_flag,
                      void* stream);

/* ---------------------------------------------------------------- RoPE
 * apply_rope / rotate_heads (tensor.py:63-105): rotate every adjacent (2j, 2j+1) pair of each
 * [n_tok][heads][head_dim] row of token t by position positions[t]; out is f32. rope_cs is the
 * host-built table [rope_rows][head_dim/2] of f32 (cos, sin) pairs, made exactly like tensor.py:84-88
 * (f64 angles, np.cos/np.sin, cast to f32); the rotation is bit-identical to numpy's
 * f32(e*c - o*s), f32(e*s + o*c). Positions outside [0, rope_rows) set bit 1 of err_flag. */
int tada_apply_rope(const void* x, int32_t dtype, int64_t n_tok, int32_t heads, int32_t head_dim,
                    const int32_t* positions, const float* rope_cs, int32_t rope_rows, float* out,
                    int32_t* err_flag, void* stream);

/* K1 with the keys rotated in registers before the mean: append_fused's key path
 * (model.py:167-183 = rotate_heads + append_tokens) without the rotated keys ever reaching HBM.
 * positions: device int32 [batch][pos_stride], token i of sequence b at positions[b * pos_stride + i].
 * Values are appended as given. Needs heads 8, head_dim 128, bits 2/4/8 and 16-byte aligned rows,
 * else TADA_ERR_CONFIG (compose tada_apply_rope + tada_quant_append). Bit-identical to that
 * composition. */
int tada_quant_append_rope(const tada_page_layout* layout, uint8_t* pool, const void* src_k,
                           const void* src_v, int32_t dtype, int32_t batch, int64_t n_tok,
                           int64_t src_seq_stride, const int32_t* page_table, int32_t pt_stride,
                           const int32_t* dst_start, int64_t dst_offset, const int32_t* positions,
                           int64_t pos_stride, const float* rope_cs, int32_t rope_rows,
                           int32_t* err_flag, void* stream);

/* Residual-buffer write (cache.py:174-175): token i of sequence b is copied (as f32)
 * to res[(b * res_seq_stride + pos[b] + pos_offset + i)][heads][head_dim]. */
int tada_residual_write(float* res_k, float* res_v, int64_t res_seq_stride, int32_t heads,
                        int32_t head_dim, const void* src_k, const void* src_v, int32_t dtype,
                        int32_t batch, int64_t n_tok, int64_t src_seq_stride, const int32_t* pos,
                        int32_t pos_offset, void* stream);

/* tada_residual_write at pos[b] (pos_offset 0) followed by pos[b] += n_tok, in one launch:
 * the no-flush branch of append_tokens (cache.py:174-175) for a decode step. */
int tada_residual_append(float* res_k, float* res_v, int64_t res_seq_stride, int32_t heads,
                         int32_t head_dim, const void* src_k, const void* src_v, int32_t dtype,
                         int32_t batch, int64_t n_tok, int64_t src_seq_stride, int32_t* pos,
                         void* stream);

/* arr[b] += delta for b < batch (device-side length bookkeeping, graph-capturable). */
int tada_lengths_add(int32_t* arr, int32_t batch, int32_t delta, void* stream);

/* Export / import of one sequence's compressed region between the paged layout
 * and the reference's dense layout (k_mean, k_dev.codes/scales/mins, ...), used
 * for TADAKV1 serialization (cache.py:311-368).  side: 0 = K, 1 = V. */
int tada_gather_compressed(const tada_page_layout* layout, const uint8_t* pool,
                           const int32_t* page_row, int64_t n_tok, int32_t side, float* mean,
                           uint8_t* codes, float* scales, float* mins, void* stream);
int tada_scatter_compressed(const tada_page_layout* layout, uint8_t* pool, const int32_t* page_row,
                            int64_t n_tok, int32_t side, const float* mean, const uint8_t* codes,
                            const float* scales, const float* mins, void* stream);

/* ---------------------------------------------------------------- K2 + K3: decode attention
 * attend_streaming (attention.py:103-151) for a batch of single-query decodes:
 * out[b][g] = softmax_t(scale * q[b][g] . K̂[b][t][kv(g)]) V̂[b][t][kv(g)], over the
 * comp_len[b] compressed tokens (K̂ = mean - deq(dev), cache.py:193-200) followed by
 * the res_len[b] residual rows (attention.py:94-100).  kv(g) = g*H/Hq (attention.py:47-49).
 * q: [batch][num_q_heads][head_dim] (f32 or bf16).  res_k/res_v: f32
 * [batch][res_seq_stride][heads][head_dim].  The token axis is split `num_splits`
 * ways (split-K flash decoding) and merged by a log-sum-exp combine (K3);
 * workspace must hold tada_decode_attn_workspace_bytes(...) bytes.
 * out: [batch][num_q_heads][head_dim] in out_dtype.
 * mode: 0 = auto, 1 = exact generic kernel (f32 reconstruct-then-dot, any geometry),
 *       2 = fast tensor-core kernel (head_dim 128, bits 2/4/8),
 *       3 = fast tensor-core kernel, previous two-barrier-per-tile variant (A/B comparisons). */
int64_t tada_decode_attn_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t head_dim,
                                         int32_t num_splits);
int tada_decode_attn(const tada_page_layout* layout, const uint8_t* pool, const void* q,
                     int32_t q_dtype, int32_t batch, int32_t num_q_heads, const int32_t* page_table,
                     int32_t pt_stride, const int32_t* comp_len, const int32_t* res_len,
                     const float* res_k, const float* res_v, int64_t res_seq_stride, float scale,
                     int32_t num_splits, void* workspace, void* out, int32_t out_dtype, int32_t mode,
                     void* stream);

/* Same as tada_decode_attn, and also writes lse_out[b][g] = log sum_t exp(scale * q.k_t) (natural
 * log) so that attention over disjoint token sets held by different ranks can be merged exactly
 * (the sequence-axis shard of SURVEY §8e; attend_streaming's online-softmax state,
 * attention.py:139-147, expressed as (out, lse)). */
int tada_decode_attn_lse(const tada_page_layout* layout, const uint8_t* pool, const void* q,
                         int32_t q_dtype, int32_t batch, int32_t num_q_heads,
                         const int32_t* page_table, int32_t pt_stride, const int32_t* comp_len,
                         const int32_t* res_len, const float* res_k, const float* res_v,
                         int64_t res_seq_stride, float scale, int32_t num_splits, void* workspace,
                         void* out, int32_t out_dtype, int32_t mode, float* lse_out, void* stream);

/* Merge n_parts normalised partial attentions: o_parts [n_parts][rows][head_dim] f32 and
 * lse_parts [n_parts][rows] f32 (-inf = the part had no tokens) ->
 * out[rows][head_dim] = sum_p o_p e^(lse_p - M) / sum_p e^(lse_p - M); lse_out (optional) gets the
 * merged log-sum-exp.  This is the online-softmax merge of attention.py:139-147 applied across
 * ranks after the NCCL all-gather of partials. */
int tada_combine_lse(const float* o_parts, const float* lse_parts, int32_t n_parts, int64_t rows,
                     int32_t head_dim, void* out, int32_t out_dtype, float* lse_out, void* stream);

/* Split count for this layer's kernel on the current device: the fewest whole waves of resident
 * CTAs (SM count x CTAs per SM of the instantiation that will run) whose last wave is >= 90% full,
 * with >= 256 tokens per split. */
/* One decode step of a layer in one call: append_tokens of one new token that stays in the residual
 * buffer (no flush: r_prev + 1 < residual_length; cache.py:174-175) followed by attend_streaming
 * (attention.py:103-151). new_k / new_v: [batch][heads][head_dim] (f32 or bf16), already rotated.
 * The K3 combine attends the new row straight from the input, stores it (as f32) at residual row
 * r_prev of every sequence and sets res_len[b] = r_prev + 1 (r_prev: the host-known, batch-uniform
 * residual count before the step). Needs the tensor-core path (head_dim 128), else TADA_ERR_CONFIG
 * with nothing enqueued. Results equal tada_residual_append + tada_decode_attn. */
int tada_decode_attn_append(const tada_page_layout* layout, const uint8_t* pool, const void* q,
                            int32_t q_dtype, int32_t batch, int32_t num_q_heads,
                            const int32_t* page_table, int32_t pt_stride, const int32_t* comp_len,
                            int32_t* res_len, float* res_k, float* res_v, int64_t res_seq_stride,
                            float scale, int32_t num_splits, void* workspace, void* out,
                            int32_t out_dtype, int32_t mode, const void* new_k, const void* new_v,
                            int32_t new_dtype, int32_t r_prev, void* stream);

int32_t tada_decode_attn_plan_splits(const tada_page_layout* layout, int32_t num_q_heads, int32_t batch,
                                     int64_t max_tokens);

/* Suggested split count assuming one CTA per SM on a 148-SM B200 (geometry-agnostic). */
int32_t tada_decode_attn_suggest_splits(int32_t batch, int64_t max_tokens, int32_t page_tokens);

#ifdef __cplusplus
}
#endif
#endif /* TADAKV_B200_H */
