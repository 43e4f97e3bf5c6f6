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

/* Device-planned K1 for a batch of sequences at different lengths (append_tokens, cache.py:154-180, per
 * sequence): every sequence b appends n = seq_n ? seq_n[b] : n_new rows and its flush is planned on the
 * device from res_len[b] (r < residual_length) — the first floor((r + n) / R) * R tokens of [its r
 * residual rows, its new rows] are compressed at comp_len[b] onwards (R = residual_length; R = 0: all n
 * new rows).  part 1 compresses the residual rows (src = the f32 residual buffer, src_seq_stride = its
 * rows per sequence), part 2 the new rows (src = the step input; dst after the part-1 rows).  n_max bounds
 * the rows of any sequence in this launch (grid size).  Lengths are not changed: tada_append_commit
 * follows.  rope_cs / positions (part 2 only, nullable): the keys are rotated in registers first, bit for
 * bit like tada_apply_rope.  range_word (nullable): the layer's two int32 range words, atomicMax'ed with
 * the binary exponent of any stored |mean| >= 2^15 ([0]) or group scale >= 2^8 ([1]); see tada_decode_attn. */
int tada_quant_append_plan(const tada_page_layout* layout, uint8_t* pool, const void* src_k,
                           const void* src_v, int32_t dtype, int32_t batch, int64_t n_max,
                           int64_t src_seq_stride, const int32_t* page_table, int32_t pt_stride,
                           const int32_t* comp_len, const int32_t* res_len, int32_t residual_length,
                           int32_t n_new, const int32_t* seq_n, int32_t part, const int32_t* positions,
                           int64_t pos_stride, const float* rope_cs, int32_t rope_rows,
                           int32_t* err_flag, int32_t* range_word, void* stream);

/* The rest of that append, one CTA per sequence: the new rows that stay raw are stored (f32; keys rotated
 * when rope_cs is given) at their residual rows, then comp_len[b] / res_len[b] advance by the plan. */
int tada_append_commit(float* res_k, float* res_v, int64_t res_seq_stride, int32_t heads, int32_t head_dim,
                       const void* src_k, const void* src_v, int32_t dtype, int32_t batch,
                       int64_t src_seq_stride, int32_t n_new, const int32_t* seq_n,
                       int32_t residual_length, int32_t* comp_len, int32_t* res_len,
                       const int32_t* positions, int64_t pos_stride, const float* rope_cs,
                       int32_t rope_rows, int32_t* err_flag, void* stream);

/* ---------------------------------------------------------------- RoPE
 * apply_rope / rotate_heads (tensor.py:63-105): rotate every adjacent (2j, 2j+1) pair of each
 * [n_tok][heads][head_dim] row of token t by position positions[t]; out is f32. rope_cs is the
 * host-built table [rope_rows][head_dim/2] of f32 (cos, sin) pairs, made exactly like tensor.py:84-88
 * (f64 angles, np.cos/np.sin, cast to f32); the rotation is bit-identical to numpy's
 * f32(e*c - o*s), f32(e*s + o*c). Positions outside [0, rope_rows) set bit 1 of err_flag. */
int tada_apply_rope(const void* x, int32_t dtype, int64_t n_tok, int32_t heads, int32_t head_dim,
                    const int32_t* positions, const float* rope_cs, int32_t rope_rows, float* out,
                    int32_t* err_flag, void* stream);

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
 * range_word (nullable): the layer's two device range words that tada_quant_append_plan maintains; the
 * tensor-core kernels stage q, the means and P' as f16, so a layer with a stored |mean| >= 2^15 or a
 * group scale beyond what its kernel's P' holds (2^15 for the 2/4-bit kernel, 2^8 for the 8-bit one),
 * or a query element >= 2^15, is attended on their exact f32 path instead (mode 0 and 2). 
 * mode: 0 = auto, 1 = exact generic kernel (f32 reconstruct-then-dot, any geometry),
 *       2 = fast tensor-core kernel (head_dim 128, bits 2/4/8, a multiple of 8 KV heads: other group sizes
 *           and head counts run as padded passes / views of 8 KV heads),
 *       3 = fast tensor-core kernel, previous two-barrier-per-tile variant (A/B comparisons). */
int64_t tada_decode_attn_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t head_dim,
                                         int32_t num_splits);
int tada_decode_attn(const tada_page_layout* layout, const uint8_t* pool, const void* q,
                     int32_t q_dtype, int32_t batch, int32_t num_q_heads, const int32_t* page_table,
                     int32_t pt_stride, const int32_t* comp_len, const int32_t* res_len,
                     const float* res_k, const float* res_v, int64_t res_seq_stride, float scale,
                     int32_t num_splits, void* workspace, void* out, int32_t out_dtype, int32_t mode,
                     const int32_t* range_word, void* stream);

/* Same as tada_decode_attn, and also writes lse_out[b][g] = log sum_t exp(scale * q.k_t) (natural
 * log) so that attention over disjoint token sets held by different ranks can be merged exactly
 * (the sequence-axis shard of SURVEY §8e; attend_streaming's online-softmax state,
 * attention.py:139-147, expressed as (out, lse)). */
int tada_decode_attn_lse(const tada_page_layout* layout, const uint8_t* pool, const void* q,
                         int32_t q_dtype, int32_t batch, int32_t num_q_heads,
                         const int32_t* page_table, int32_t pt_stride, const int32_t* comp_len,
                         const int32_t* res_len, const float* res_k, const float* res_v,
                         int64_t res_seq_stride, float scale, int32_t num_splits, void* workspace,
                         void* out, int32_t out_dtype, int32_t mode, float* lse_out,
                         const int32_t* range_word, void* stream);

/* Merge n_parts normalised partial attentions: o_parts [n_parts][rows][head_dim] f32 and
 * lse_parts [n_parts][rows] f32 (-inf = the part had no tokens) ->
 * out[rows][head_dim] = sum_p o_p e^(lse_p - M) / sum_p e^(lse_p - M); lse_out (optional) gets the
 * merged log-sum-exp.  This is the online-softmax merge of attention.py:139-147 applied across
 * ranks after the NCCL all-gather of partials. */
int tada_combine_lse(const float* o_parts, const float* lse_parts, int32_t n_parts, int64_t rows,
                     int32_t head_dim, void* out, int32_t out_dtype, float* lse_out, void* stream);

/* One decode step of a layer for a batch of sequences at ANY mix of lengths (ragged), graph-capturable:
 * append_tokens of one token per sequence (cache.py:154-180) then attend_streaming (attention.py:103-151),
 * every flush decision taken on the device from the sequence's own res_len (seq_plan):
 *  - a sequence whose residual reaches residual_length compresses it and the new row (K1, two launches
 *    over the flushing sequences: the residual rows, then the new row; k1_rows bounds the residual rows
 *    any sequence may flush, residual_length - 1 under graph capture; k1_rows < 0 skips K1 when the caller
 *    knows no sequence compresses a token this step; residual_length 0 compresses every new row);
 *  - K2 attends comp_len[b] plus the tokens this step compresses;
 *  - K3 attends the residual rows and, where no flush happened, the new row read from the input, stores
 *    that row at residual row res_len[b], and the last K3 CTA of each sequence advances comp_len[b] /
 *    res_len[b] (step_sync: device int32[batch] arrival counters, zero-initialised, left at zero).
 * new_k / new_v: [batch][heads][head_dim] (f32 or bf16), already rotated. Needs the tensor-core path
 * (head_dim 128), else TADA_ERR_CONFIG with nothing enqueued (compose tada_quant_append_plan +
 * tada_append_commit + tada_decode_attn). Results equal that composition. */
int tada_decode_step(const tada_page_layout* layout, uint8_t* pool, const void* q, int32_t q_dtype,
                     int32_t batch, int32_t num_q_heads, const int32_t* page_table, int32_t pt_stride,
                     int32_t* comp_len, int32_t* res_len, float* res_k, float* res_v,
                     int64_t res_seq_stride, int32_t residual_length, const void* new_k, const void* new_v,
                     int32_t new_dtype, int32_t k1_rows, int32_t* step_sync, float scale,
                     int32_t num_splits, void* workspace, void* out, int32_t out_dtype, int32_t mode,
                     int32_t* err_flag, int32_t* range_word, void* stream);

/* Split count for this layer's kernel on the current device: the fewest whole waves of resident
 * CTAs (SM count x CTAs per SM of the instantiation that will run) whose last wave is >= 90% full,
 * with >= 256 tokens per split. */
int32_t tada_decode_attn_plan_splits(const tada_page_layout* layout, int32_t num_q_heads, int32_t batch,
                                     int64_t max_tokens);
/* The same for the kernel a given mode runs (mode 1: the exact kernels, which also take splits down to 64
 * tokens when 256-token splits would leave SMs idle, e.g. one sequence). */
int32_t tada_decode_attn_plan_splits_mode(const tada_page_layout* layout, int32_t num_q_heads, int32_t batch,
                                          int64_t max_tokens, int32_t mode);

/* Suggested split count assuming one CTA per SM on a 148-SM B200 (geometry-agnostic). */
int32_t tada_decode_attn_suggest_splits(int32_t batch, int64_t max_tokens, int32_t page_tokens);

#ifdef __cplusplus
}
#endif
#endif /* TADAKV_B200_H */
