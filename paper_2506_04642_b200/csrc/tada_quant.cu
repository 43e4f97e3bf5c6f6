// Quantizer, packer, mean-centering and K1 (fused quantize-on-append) for sm_100a.
//
// Reference: pkg/src/tadakv/quant.py (quantize_tensor 200-229, _quantize_rows 143-174,
// pack_codes 93-111, unpack_codes 114-140, _dequantize_rows 177-180) and
// pkg/src/tadakv/cache.py (mean_center 98-111, append_tokens 154-180,
// _compress_block 182-188).  Codes, scales, mins and means are bit-exact.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <mutex>
#include <string>

#include "tada_common.cuh"

namespace tada {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
// Every kernel launch in the library is followed by exactly one check_launch, so this counts
// launches (tada_launch_count; the bench reports it as gpu_launches).
static std::atomic<int64_t> g_launches{0};
int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return TADA_OK;
}

static bool valid_bits(int b) { return b == 2 || b == 4 || b == 8 || b == 16; }
static bool valid_dtype(int t) { return t == TADA_F32 || t == TADA_BF16; }
static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > 148 * 64) g = 148 * 64;
  return int(g);
}

// Stored values beyond the f16 operand range of the tensor-core decode kernels (tada_attn.cuh: a mean at or
// above 2^15, a group scale at or above 2^8 for the unscaled P' of attn_fast_kernel) record their binary
// exponent in the layer's range words (atomicMax, rare): [0] means, [1] scales.  K2 then attends that layer
// on its exact f32 path.
__device__ __forceinline__ void note_mean(int32_t* range, float v) {
  const float a = fabsf(v);
  if (range && a >= 32768.f && a <= 3.4028235e38f) atomicMax(range, ilogbf(a));
}
__device__ __forceinline__ void note_scale(int32_t* range, float s) {
  if (range && s >= 256.f && s <= 3.4028235e38f) atomicMax(range + 1, ilogbf(s));
}

// ------------------------------------------------------------------ warp group quantizer
//
// One warp quantizes one group of D elements.  Lane l owns elements
// c*128 + 4l .. +3 of chunk c (NCH chunks cover D <= 128*NCH), so each lane packs
// 4 codes = 4*bits bits = whole bytes for every width, exactly like pack_codes'
// zero-padded byte layout (quant.py:101-111).
template <int NCH, typename Load>
__device__ __forceinline__ void quantize_group_warp(Load load, int D, int bits, uint8_t* __restrict__ out,
                                                    float* scale_out, float* min_out, int32_t* err, int lane,
                                                    bool vec_ok, int32_t* range = nullptr) {
  float v[NCH][4];
  float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
  bool bad = false;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int e0 = c * 128 + lane * 4;
    if (vec_ok && e0 + 3 < D) {
      load.vec4(e0, v[c]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[c][k] = (e0 + k < D) ? load(e0 + k) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (e0 + k < D) {
        bad |= !finite(v[c][k]);
        mn = fminf(mn, v[c][k]);
        mx = fmaxf(mx, v[c][k]);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0 && err) atomicOr(err, 1);  // host raises DataError (quant.py:151-152)
  }
  if (bits == 16) {  // raw f32 pass-through (quant.py:208-219)
    float* o = reinterpret_cast<float*>(out);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int e0 = c * 128 + lane * 4;
      if (vec_ok && e0 + 3 < D) {
        *reinterpret_cast<float4*>(o + e0) = make_float4(v[c][0], v[c][1], v[c][2], v[c][3]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (e0 + k < D) o[e0 + k] = v[c][k];
      }
    }
    if (lane == 0) {
      *scale_out = 0.f;
      *min_out = 0.f;
    }
    return;
  }
  mn = warp_min(mn);
  mx = warp_max(mx);
  const float s = group_scale(mn, mx, bits);
  const int cmax = (1 << bits) - 1;
  const bool fast = s >= 0x1p-100f && s <= 0x1p100f;
  const float inv_s = fast ? __frcp_rn(s) : 0.f;
  const int gb = int(group_bytes(D, bits));
  const int nbytes = bits / 2;  // bytes produced by 4 codes
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    const int e0 = c * 128 + lane * 4;
    if (e0 >= D) continue;
    uint32_t word = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t code = 0;
      if (e0 + k < D && s != 0.f) code = quant_code(v[c][k], mn, s, inv_s, fast, cmax);
      word |= code << (bits * k);
    }
    const int off = (e0 * bits) >> 3;
    if (vec_ok && off + nbytes <= gb) {
      if (bits == 2) out[off] = uint8_t(word);
      else if (bits == 4) *reinterpret_cast<uint16_t*>(out + off) = uint16_t(word);
      else *reinterpret_cast<uint32_t*>(out + off) = word;
    } else {
      for (int j = 0; j < nbytes; ++j)
        if (off + j < gb) out[off + j] = uint8_t(word >> (8 * j));
    }
  }
  if (lane == 0) {
    *scale_out = s;
    *min_out = mn;
    note_scale(range, s);
  }
}

template <typename T>
struct GlobalRow {
  const T* p;
  __device__ float operator()(int e) const { return to_f32(p[e]); }
  __device__ void vec4(int e, float (&v)[4]) const { load4(p + e, v); }
};

// dev = mean - x, read from shared memory (cache.py:110)
struct CenteredRow {
  const float* mean;
  const float* x;
  __device__ float operator()(int e) const { return __fsub_rn(mean[e], x[e]); }
  __device__ void vec4(int e, float (&v)[4]) const {
    const float4 m = *reinterpret_cast<const float4*>(mean + e);
    const float4 a = *reinterpret_cast<const float4*>(x + e);
    v[0] = __fsub_rn(m.x, a.x);
    v[1] = __fsub_rn(m.y, a.y);
    v[2] = __fsub_rn(m.z, a.z);
    v[3] = __fsub_rn(m.w, a.w);
  }
};

// ------------------------------------------------------------------ quantize_tensor
template <typename T, int NCH>
__global__ void __launch_bounds__(256) quantize_groups_kernel(const T* __restrict__ rows, int64_t n_groups, int D,
                                                              int bits, uint8_t* __restrict__ codes,
                                                              float* __restrict__ scales, float* __restrict__ mins,
                                                              int32_t* err, bool vec_ok) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int64_t gb = group_bytes(D, bits);
  for (int64_t g = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); g < n_groups; g += warps) {
    GlobalRow<T> ld{rows + g * D};
    quantize_group_warp<NCH>(ld, D, bits, codes + g * gb, scales + g, mins + g, err, lane, vec_ok);
  }
}

// ------------------------------------------------------------------ dequantize / (un)pack
__global__ void dequant_kernel(const uint8_t* __restrict__ codes, const float* __restrict__ scales,
                               const float* __restrict__ mins, int D, int bits, const int64_t* __restrict__ sel,
                               int64_t n_out, float* __restrict__ out) {
  const int64_t gb = group_bytes(D, bits);
  const int64_t total = n_out * D;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = i / D;
    const int e = int(i - j * D);
    const int64_t g = sel ? sel[j] : j;
    const uint8_t* grp = codes + g * gb;
    if (bits == 16) {
      out[i] = reinterpret_cast<const float*>(grp)[e];
    } else {
      out[i] = dequant_exact(get_code(grp, e, bits), scales[g], mins[g]);
    }
  }
}

__global__ void pack_kernel(const uint8_t* __restrict__ codes, int64_t n_groups, int D, int bits,
                            uint8_t* __restrict__ packed) {
  const int gb = int(group_bytes(D, bits));
  const int per = 8 / bits;
  const int64_t total = n_groups * gb;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t g = i / gb;
    const int byte = int(i - g * gb);
    uint32_t w = 0;
    for (int k = 0; k < per; ++k) {
      const int e = byte * per + k;
      if (e < D) w |= (uint32_t(codes[g * D + e]) & ((1u << bits) - 1u)) << (bits * k);
    }
    packed[i] = uint8_t(w);
  }
}

__global__ void unpack_kernel(const uint8_t* __restrict__ packed, int D, int bits, const int64_t* __restrict__ sel,
                              int64_t n_out, uint8_t* __restrict__ codes) {
  const int64_t gb = group_bytes(D, bits);
  const int64_t total = n_out * D;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = i / D;
    const int e = int(i - j * D);
    const int64_t g = sel ? sel[j] : j;
    codes[i] = uint8_t(get_code(packed + g * gb, e, bits));
  }
}

// ------------------------------------------------------------------ mean_center
// mean[t][d] = f32((((0 + x0) + x1) + ... ) / H) with an fp64 sequential head sum
// (numpy reduces the non-contiguous head axis in order).
__device__ __forceinline__ float head_mean(const float* col, int stride, int H) {
  double acc = 0.0;
  for (int h = 0; h < H; ++h) acc = __dadd_rn(acc, double(col[h * stride]));
  return __double2float_rn(__ddiv_rn(acc, double(H)));
}

template <typename T>
__global__ void mean_center_kernel(const T* __restrict__ x, int64_t tokens, int H, int D, float* __restrict__ mean,
                                   float* __restrict__ dev, int32_t* err) {
  const int64_t total = tokens * D;
  bool bad = false;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / D;
    const int d = int(i - t * D);
    const T* col = x + t * H * D + d;
    double acc = 0.0;
    for (int h = 0; h < H; ++h) {
      const float xv = to_f32(col[h * D]);
      bad |= !finite(xv);
      acc = __dadd_rn(acc, double(xv));
    }
    const float m = __double2float_rn(__ddiv_rn(acc, double(H)));
    mean[i] = m;
    for (int h = 0; h < H; ++h) dev[(t * H + h) * D + d] = __fsub_rn(m, to_f32(col[h * D]));
  }
  if (bad && err) atomicOr(err, 1);
}

// ------------------------------------------------------------------ K1: quantize-on-append
//
// CTA = a tile of TT consecutive tokens of one sequence, both sides (blockIdx.y).
//  A: tile [TT][H][D] -> smem (f32), 16B vector loads.
//  B: per (t, d) fp64 head-sum mean -> smem + paged mean block.
//  C: warp per (t, h) group: dev = mean - x, warp-shuffle min/max, fp64 scale +
//     fixed-point refinement, half-up codes, LSB-first pack -> paged codes/meta.
struct AppendArgs {
  tada_page_layout L;
  uint8_t* pool;
  const void* src[2];
  int64_t n_tok;
  int64_t src_seq_stride;
  const int32_t* page_table;
  int pt_stride;
  const int32_t* dst_start;
  int64_t dst_offset;
  int32_t* err;
  int tt;  // tokens per tile
  int tiles_per_seq;
  bool vec_ok;
  // fused RoPE of the keys: rope_cs[pos][j] = (cos, sin) f32, positions[b * pos_stride + i]
  const float* rope_cs;
  int rope_rows;
  const int32_t* positions;
  int64_t pos_stride;
  // device-planned append (seq_plan): part 1 = the residual rows a flush compresses, part 2 = the new rows it
  // compresses (dst at comp_len[b] + the residual rows); part 0 = the caller's n_tok rows at dst_start + offset
  int part;
  const int32_t* plan_res;  // res_len [B]
  const int32_t* plan_n;    // optional per-sequence new-row counts [B]
  int plan_n_new;           // new rows per sequence when plan_n is null
  int plan_R;               // residual_length
  int32_t* range;           // optional: the layer's two range words (note_mean / note_scale)
};

// rows [0, count) of sequence b this launch compresses, and their destination offset after comp_len[b]
__device__ __forceinline__ void append_part(const AppendArgs& a, int b, int64_t& count, int64_t& offset) {
  if (a.part == 0) {
    count = a.n_tok;
    offset = a.dst_offset;
    return;
  }
  const SeqPlan p = seq_plan(a.plan_res[b], a.plan_n ? a.plan_n[b] : a.plan_n_new, a.plan_R);
  count = a.part == 1 ? p.cnt_res : p.cnt_new;
  offset = a.part == 1 ? 0 : p.cnt_res;
  if (count > a.n_tok) count = a.n_tok;  // the launch covers at most n_tok rows per sequence
}

template <typename T, int NCH>
__global__ void __launch_bounds__(256) quant_append_kernel(AppendArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int H = a.L.heads, D = a.L.head_dim, bits = a.L.bits, P = a.L.page_tokens;
  const int side = blockIdx.y;
  const int b = blockIdx.x / a.tiles_per_seq;
  const int64_t i0 = int64_t(blockIdx.x % a.tiles_per_seq) * a.tt;
  int64_t count, offset;
  append_part(a, b, count, offset);
  const int64_t rem = count - i0;
  const int nt = int(rem < a.tt ? rem : a.tt);
  if (nt <= 0) return;
  const int row = H * D;
  float* xs = smem;                  // [tt][H*D]
  float* ms = smem + a.tt * row;     // [tt][D]
  const T* src = reinterpret_cast<const T*>(a.src[side]) + (int64_t(b) * a.src_seq_stride + i0) * row;

  // A: load tile
  const int n_el = nt * row;
  bool bad = false;
  if (a.vec_ok) {
    for (int e = threadIdx.x * 4; e < n_el; e += blockDim.x * 4) {
      float v[4];
      load4(src + e, v);
#pragma unroll
      for (int k = 0; k < 4; ++k) bad |= !finite(v[k]);
      *reinterpret_cast<float4*>(xs + e) = make_float4(v[0], v[1], v[2], v[3]);
    }
  } else {
    for (int e = threadIdx.x; e < n_el; e += blockDim.x) {
      xs[e] = to_f32(src[e]);
      bad |= !finite(xs[e]);
    }
  }
  if (bad && a.err) atomicOr(a.err, 1);
  __syncthreads();

  const int64_t c0 = a.dst_start[b] + offset;
  const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
  // B: means
  for (int e = threadIdx.x; e < nt * D; e += blockDim.x) {
    const int t = e / D, d = e - t * D;
    const float m = head_mean(xs + t * row + d, D, H);
    ms[t * D + d] = m;
    note_mean(a.range, m);
    const int64_t c = c0 + i0 + t;
    uint8_t* page = a.pool + int64_t(pt[c / P]) * a.L.page_bytes;
    reinterpret_cast<float*>(page + a.L.off_mean[side])[(c % P) * D + d] = m;
  }
  __syncthreads();

  // C: groups
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gb = a.L.group_bytes;
  for (int g = warp; g < nt * H; g += nw) {
    const int t = g / H, h = g - t * H;
    const int64_t c = c0 + i0 + t;
    uint8_t* page = a.pool + int64_t(pt[c / P]) * a.L.page_bytes;
    const int64_t grp = (c % P) * H + h;
    float* meta = reinterpret_cast<float*>(page + a.L.off_meta[side]) + 2 * grp;
    CenteredRow ld{ms + t * D, xs + t * row + h * D};
    quantize_group_warp<NCH>(ld, D, bits, page + a.L.off_codes[side] + grp * gb, meta, meta + 1, a.err, lane,
                             a.vec_ok, a.range);
  }
}

// ------------------------------------------------------------------ append commit (residual rows + lengths)
// Commit of a device-planned append (seq_plan), one CTA per sequence: the new rows that stay raw go to
// the residual buffer (keys rotated here when a RoPE table is given, like tada_apply_rope), then the
// sequence's lengths advance.  The CTA reads res_len[b] before anything writes it and is the only writer
// of sequence b, so no other ordering is needed; it runs after the K1 parts that read the same plan.
template <typename T, bool ROPE>
__global__ void __launch_bounds__(256) append_commit_kernel(float* __restrict__ rk, float* __restrict__ rv,
                                                            int64_t res_seq_stride, int H, int D,
                                                            const T* __restrict__ sk, const T* __restrict__ sv,
                                                            int64_t src_seq_stride, int n_new, const int32_t* plan_n,
                                                            int R, int32_t* comp_len, int32_t* res_len,
                                                            const int32_t* __restrict__ positions, int64_t pos_stride,
                                                            const float* __restrict__ rope_cs, int rope_rows,
                                                            int32_t* err) {
  const int b = blockIdx.x;
  const int r = res_len[b];
  const int n = plan_n ? plan_n[b] : n_new;
  const SeqPlan p = seq_plan(r, n, R);
  const bool flush = p.ncomp > 0;
  const int src0 = R > 0 ? (flush ? p.cnt_new : 0) : 0;  // first new row kept raw
  const int dst0 = flush ? 0 : r;                       // its residual row
  const int rows = R > 0 ? (flush ? p.res_after : n) : 0;
  const int row = H * D;
  const T* s0 = sk + int64_t(b) * src_seq_stride * row;
  const T* s1 = sv + int64_t(b) * src_seq_stride * row;
  float* d0 = rk + int64_t(b) * res_seq_stride * row;
  float* d1 = rv + int64_t(b) * res_seq_stride * row;
  const int64_t n_el = int64_t(rows) * row;
  if (!ROPE) {
    for (int64_t e = threadIdx.x; e < n_el; e += blockDim.x) {
      d0[int64_t(dst0) * row + e] = to_f32(s0[int64_t(src0) * row + e]);
      d1[int64_t(dst0) * row + e] = to_f32(s1[int64_t(src0) * row + e]);
    }
  } else {  // keys: one thread per (row, head, pair) with the reference's separately rounded products
    const int half = D >> 1;
    for (int64_t e = threadIdx.x; e < n_el / 2; e += blockDim.x) {
      const int64_t t = e / (int64_t(H) * half);
      const int j = int(e % half);
      const int64_t el = 2 * e;  // = (t * H + h) * D + 2j
      int ps = positions[int64_t(b) * pos_stride + src0 + t];
      if (ps < 0 || ps >= rope_rows) {
        if (err) atomicOr(err, 2);
        ps = 0;
      }
      const float c = rope_cs[int64_t(ps) * D + 2 * j], sn = rope_cs[int64_t(ps) * D + 2 * j + 1];
      const float x0 = to_f32(s0[int64_t(src0) * row + el]), x1 = to_f32(s0[int64_t(src0) * row + el + 1]);
      d0[int64_t(dst0) * row + el] = __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, sn));
      d0[int64_t(dst0) * row + el + 1] = __fadd_rn(__fmul_rn(x0, sn), __fmul_rn(x1, c));
      d1[int64_t(dst0) * row + el] = to_f32(s1[int64_t(src0) * row + el]);
      d1[int64_t(dst0) * row + el + 1] = to_f32(s1[int64_t(src0) * row + el + 1]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    comp_len[b] += p.ncomp;
    res_len[b] = p.res_after;
  }
}

// ------------------------------------------------------------------ paged <-> dense (TADAKV1 export/import)
template <bool kGather>
__global__ void move_compressed_kernel(tada_page_layout L, uint8_t* pool, const int32_t* __restrict__ page_row,
                                       int64_t n_tok, int side, float* mean, uint8_t* codes, float* scales,
                                       float* mins) {
  const int H = L.heads, D = L.head_dim, P = L.page_tokens, gb = L.group_bytes;
  const int64_t per_tok = int64_t(D) + int64_t(H) * gb + 2 * H;  // work items per token
  const int64_t total = n_tok * per_tok;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t t = i / per_tok;
    int64_t k = i - t * per_tok;
    uint8_t* page = pool + int64_t(page_row[t / P]) * L.page_bytes;
    const int64_t r = t % P;
    if (k < D) {
      float* pm = reinterpret_cast<float*>(page + L.off_mean[side]) + r * D + k;
      if (kGather) mean[t * D + k] = *pm; else *pm = mean[t * D + k];
      continue;
    }
    k -= D;
    if (k < int64_t(H) * gb) {
      uint8_t* pc = page + L.off_codes[side] + r * H * gb + k;
      if (kGather) codes[t * H * gb + k] = *pc; else *pc = codes[t * H * gb + k];
      continue;
    }
    k -= int64_t(H) * gb;
    const int h = int(k >> 1);
    float* pmeta = reinterpret_cast<float*>(page + L.off_meta[side]) + 2 * (r * H + h) + (k & 1);
    float* dense = (k & 1) ? mins : scales;
    if (kGather) dense[t * H + h] = *pmeta; else *pmeta = dense[t * H + h];
  }
}

// ------------------------------------------------------------------ host dispatch helpers
template <typename T>
static int launch_quantize(const void* rows, int64_t n, int D, int bits, uint8_t* codes, float* scales, float* mins,
                           int32_t* err, cudaStream_t st) {
  const int wpb = 8;
  const int grid = grid_for(n, wpb);
  const bool vec = (D % 4 == 0) && (reinterpret_cast<uintptr_t>(rows) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(codes) % 4 == 0);
  const T* r = reinterpret_cast<const T*>(rows);
  if (D <= 128)
    quantize_groups_kernel<T, 1><<<grid, 256, 0, st>>>(r, n, D, bits, codes, scales, mins, err, vec);
  else if (D <= 256)
    quantize_groups_kernel<T, 2><<<grid, 256, 0, st>>>(r, n, D, bits, codes, scales, mins, err, vec);
  else if (D <= 512)
    quantize_groups_kernel<T, 4><<<grid, 256, 0, st>>>(r, n, D, bits, codes, scales, mins, err, vec);
  else
    quantize_groups_kernel<T, 8><<<grid, 256, 0, st>>>(r, n, D, bits, codes, scales, mins, err, vec);
  return check_launch("quantize_groups");
}

// ------------------------------------------------------------------ K1 fast path (head_dim 128, 8 heads)
//
// One warp per (token, side).  Lane l owns columns d = 4l .. 4l+3 of all 8 heads, so
//  * the cross-head mean of its 4 columns is a register-only f64 sequential sum (cache.py:109);
//  * each (token, head) group's min / max is one CREDUX.MIN/MAX.F32 across the warp;
//  * lane h computes group h's fp64 scale + refinement (quant.py:153-167) and broadcasts it;
//  * codes use an f32 round-to-nearest estimate q = (d - min) / s through the 2^23 magic add;
//    when |q - RN(q)| is within 2^-12 of a half-integer the lane's group falls back to the
//    exact fp64 half-up sequence (quant_code), which decides every tie like the reference.
// Loads are 8-byte (bf16) / 16-byte (f32) per lane and head, stores 16-bit (4-bit) codes per
// lane and head, a float4 of the mean per lane, and (scale, min) by lanes 0..7.
__device__ __forceinline__ uint32_t prmt(uint32_t x, uint32_t y, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(y), "r"(sel));
  return r;
}
__device__ __forceinline__ float redux_min(float v) {
  float r;
  asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float redux_max(float v) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
  return r;
}

// Each warp streams its tokens' rows (H*D contiguous elements) into a private 3-deep shared
// ring with cp.async.bulk + an mbarrier per slot, so the next rows are in flight while the
// current one is quantized (the kernel is otherwise latency-bound on its global loads).
constexpr int K1_RING = 3;
#ifndef TADA_K1_RECOMP
#define TADA_K1_RECOMP 0  // recompute nd = x - mean from the packed row on each use instead of holding it
#endif
#ifndef TADA_K1_MINB
#define TADA_K1_MINB 3  // resident CTAs per SM the register allocation targets (3: 80 registers)
#endif
#ifndef TADA_K1_PAGE_CACHE
#define TADA_K1_PAGE_CACHE 1  // page base pointer reloaded on page change only
#endif
__device__ __forceinline__ uint32_t k1_su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }


// K1 row of one token as held by lane l: elements 4l .. 4l+3 of each of the 8 heads.  bf16 rows stay packed:
// cvt.f64.bf16 (F2F.F64.BF16) and the mixed-precision sub.f32.bf16 (FHADD) read the halves directly.
struct K1RowBF16 {
  uint32_t w[8][2];
  __device__ __forceinline__ void load(const __nv_bfloat16* p) {
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const uint2 x = *reinterpret_cast<const uint2*>(p + h * 128);
      w[h][0] = x.x;
      w[h][1] = x.y;
    }
  }
  __device__ __forceinline__ double f64(int h, int k) const {
    double r;
    if (k & 1) asm("{.reg .b16 l, u; mov.b32 {l, u}, %1; cvt.f64.bf16 %0, u;}" : "=d"(r) : "r"(w[h][k >> 1]));
    else asm("{.reg .b16 l, u; mov.b32 {l, u}, %1; cvt.f64.bf16 %0, l;}" : "=d"(r) : "r"(w[h][k >> 1]));
    return r;
  }
  __device__ __forceinline__ float minus(int h, int k, float m) const {  // RN(x - m)
    float r;
    if (k & 1) asm("{.reg .b16 l, u; mov.b32 {l, u}, %2; sub.rn.f32.bf16 %0, u, %1;}" : "=f"(r) : "f"(m), "r"(w[h][k >> 1]));
    else asm("{.reg .b16 l, u; mov.b32 {l, u}, %2; sub.rn.f32.bf16 %0, l, %1;}" : "=f"(r) : "f"(m), "r"(w[h][k >> 1]));
    return r;
  }
  __device__ __forceinline__ float add_rd(int h, int k, float acc) const {  // RD(x + acc)
    float r;
    if (k & 1) asm("{.reg .b16 l, u; mov.b32 {l, u}, %2; add.rm.f32.bf16 %0, u, %1;}" : "=f"(r) : "f"(acc), "r"(w[h][k >> 1]));
    else asm("{.reg .b16 l, u; mov.b32 {l, u}, %2; add.rm.f32.bf16 %0, l, %1;}" : "=f"(r) : "f"(acc), "r"(w[h][k >> 1]));
    return r;
  }
  __device__ __forceinline__ float add_ru(int h, int k, float acc) const {  // RU(x + acc)
    float r;
    if (k & 1) asm("{.reg .b16 l, u; mov.b32 {l, u}, %2; add.rp.f32.bf16 %0, u, %1;}" : "=f"(r) : "f"(acc), "r"(w[h][k >> 1]));
    else asm("{.reg .b16 l, u; mov.b32 {l, u}, %2; add.rp.f32.bf16 %0, l, %1;}" : "=f"(r) : "f"(acc), "r"(w[h][k >> 1]));
    return r;
  }
};
struct K1RowF32 {
  float v[8][4];
  __device__ __forceinline__ void load(const float* p) {
#pragma unroll
    for (int h = 0; h < 8; ++h) load4(p + h * 128, v[h]);
  }
  __device__ __forceinline__ void load(const __nv_bfloat16* p) {
#pragma unroll
    for (int h = 0; h < 8; ++h) load4(p + h * 128, v[h]);
  }
  __device__ __forceinline__ double f64(int h, int k) const { return double(v[h][k]); }
  __device__ __forceinline__ float minus(int h, int k, float m) const { return __fsub_rn(v[h][k], m); }
  __device__ __forceinline__ float add_rd(int h, int k, float acc) const { return __fadd_rd(v[h][k], acc); }
  __device__ __forceinline__ float add_ru(int h, int k, float acc) const { return __fadd_ru(v[h][k], acc); }
};
template <typename T> struct K1Row { using type = K1RowF32; };
template <> struct K1Row<__nv_bfloat16> { using type = K1RowBF16; };

// negated deviations held in registers, or recomputed from the packed row on every use (TADA_K1_RECOMP)
struct K1NdRegs {
  float v[8][4];
  __device__ __forceinline__ float operator()(int h, int k) const { return v[h][k]; }
};
template <typename Row>
struct K1NdLazy {
  Row x;
  float m[4];
  __device__ __forceinline__ float operator()(int h, int k) const { return x.minus(h, k, m[k]); }
};

// mean (cache.py:109): the reference sums the 8 heads in f64 from +0.0, divides by 8 (exact) and rounds to f32.
// The f64 sum of 8 bf16/f32 values is exact unless their exponents span more than ~28 bits, so the mean is
// RN32(S) / 8 for the exact sum S.  Two f32 sums rounded down and up bracket S; when they are equal, S is that
// f32 value (every step was exact) and the mean is S * 0.125 (|S| >= 2^-120 keeps the scaling exact).  Other
// columns (rare: a wide exponent spread, an exact zero or tiny sum, or non-finite) take the f64 sequence.  This keeps the F2F conversions off the XU pipe, which they saturated.
template <typename Row>
__device__ __forceinline__ double k1_col_sum64(const Row& x, int k) {
  double acc = 0.0;
#pragma unroll
  for (int h = 0; h < 8; ++h) acc = __dadd_rn(acc, x.f64(h, k));
  return acc;
}
#ifndef TADA_K1_F32_MEAN64
#define TADA_K1_F32_MEAN64 1  // f32 rows (RoPE keys, residual flushes): the f64 sequence directly (measured +4.5% with RoPE)
#endif
template <typename Row>
__device__ __forceinline__ void k1_mean(const Row& x, float (&mean)[4], bool& big) {
  if (TADA_K1_F32_MEAN64 && sizeof(x) == sizeof(float) * 32) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mean[k] = __double2float_rn(__dmul_rn(k1_col_sum64(x, k), 0.125));
      big |= !(fabsf(mean[k]) < 32768.f);
    }
    return;
  }
  bool slow = false;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float dn = 0.f, up = 0.f;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      dn = x.add_rd(h, k, dn);
      up = x.add_ru(h, k, up);
    }
    slow |= (dn != up) | !(fabsf(up) >= 0x1p-120f);  // inexact, tiny (zero included: conservative) or NaN
    mean[k] = __fmaf_rn(dn, 0.125f, 0.f);
  }
  if (__any_sync(0xffffffffu, slow)) {
#pragma unroll
    for (int k = 0; k < 4; ++k) mean[k] = __double2float_rn(__dmul_rn(k1_col_sum64(x, k), 0.125));
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) big |= !(fabsf(mean[k]) < 32768.f);
}
// ... and nd = RN(x - mean)
template <typename Row>
__device__ __forceinline__ void k1_mean_dev(const Row& x, float (&mean)[4], float (&nd)[8][4], bool& big) {
  // any non-finite input makes its column's sum non-finite; |mean| >= 2^15 leaves the f16 range of K2
  k1_mean(x, mean, big);
#pragma unroll
  for (int h = 0; h < 8; ++h)
#pragma unroll
    for (int k = 0; k < 4; ++k) nd[h][k] = x.minus(h, k, mean[k]);
}

// The two bracket ends of 4 codes of one group, packed like pack_codes (LSB-first): t = RN(u * m + 2^23) holds
// RN(u * m) in its low mantissa bits, and the bits above the code field are identical for both ends.
template <int BITS, typename ND>
__device__ __forceinline__ void k1_bracket(const ND& nd, int h, float ndmax, float ml, float mh, uint32_t& wl,
                                           uint32_t& wh) {
  uint32_t tl[4], th[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float u = __fsub_rn(ndmax, nd(h, k));  // RN(dev - min): dev = -nd, min = -ndmax (zero signs aside)
    tl[k] = __float_as_uint(__fmaf_rn(u, ml, 8388608.f));
    th[k] = __float_as_uint(__fmaf_rn(u, mh, 8388608.f));
  }
  if (BITS == 8) {
    wl = prmt(prmt(tl[0], tl[1], 0x0040u), prmt(tl[2], tl[3], 0x0040u), 0x5410u);
    wh = prmt(prmt(th[0], th[1], 0x0040u), prmt(th[2], th[3], 0x0040u), 0x5410u);
  } else {  // code fields < 2^BITS: shifted adds keep the garbage above bit 4 * BITS
    wl = (((tl[3] << BITS) + tl[2]) << (2 * BITS)) + ((tl[1] << BITS) + tl[0]);
    wh = (((th[3] << BITS) + th[2]) << (2 * BITS)) + ((th[1] << BITS) + th[0]);
  }
}
template <int BITS>
__device__ __forceinline__ void k1_store_codes(uint8_t* dst, uint32_t w) {
  if (BITS == 8) *reinterpret_cast<uint32_t*>(dst) = w;
  else if (BITS == 4) *reinterpret_cast<uint16_t*>(dst) = uint16_t(w);
  else *dst = uint8_t(w);
}

// One token of one side after its rows were read: group min / max, scales, codes and stores (K1 fast path).
// ND yields the negated deviations nd(h, k) = RN(x - mean) of the lane's elements, from registers or recomputed.
template <int BITS, typename ND>
__device__ __forceinline__ void k1_token(const AppendArgs& a, const ND& nd, const float (&mean)[4], bool big,
                                         uint8_t* page, int row, int side, int lane) {
  constexpr int H = 8, D = 128, GB = D * BITS / 8;
  if (__any_sync(0xffffffffu, big)) {  // rare: a non-finite input, or a mean beyond K2's f16 range
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bad |= !finite(mean[k]);
      note_mean(a.range, mean[k]);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0 && a.err) atomicOr(a.err, 1);
  }
  // group min / max of dev = -nd: one CREDUX each per head; +0.0 - y keeps the reference's +0.0 for zeros
  float ndmax[H], ndmin[H];  // max / min of nd = -(min / max of dev) per head (uniform across the warp)
#pragma unroll
  for (int h = 0; h < H; ++h) {
    ndmax[h] = redux_max(fmaxf(fmaxf(nd(h, 0), nd(h, 1)), fmaxf(nd(h, 2), nd(h, 3))));
    ndmin[h] = redux_min(fminf(fminf(nd(h, 0), nd(h, 1)), fminf(nd(h, 2), nd(h, 3))));
  }
  // lane h < 8 takes head h's pair: a three-level select tree on the lane bits
  const bool l0 = lane & 1, l1 = lane & 2, l2 = lane & 4;
  auto pick = [&](const float (&v)[H]) {
    const float a0 = l0 ? v[1] : v[0], a1 = l0 ? v[3] : v[2], a2 = l0 ? v[5] : v[4], a3 = l0 ? v[7] : v[6];
    const float b0 = l1 ? a1 : a0, b1 = l1 ? a3 : a2;
    return l2 ? b1 : b0;
  };
  float my_mn = pick(ndmax), my_mx = pick(ndmin);
  my_mn = __fsub_rn(0.f, my_mn);  // group min / max of dev
  my_mx = __fsub_rn(0.f, my_mx);
  // Lane h < 8: group h's f64 scale with the reference's refinement, then the bracket multipliers.
  // Codes (quant.py:169-173): code = floor(W + 1/2), W = (dev - min) / s in f64.  With u = RN32(dev - min),
  // r = RN32(1 / s) and the multipliers r * (1 -+ 2^-22) rounded once more (relative error 2^-24 each, so
  // 3 * 2^-24 < 2^-22 in total), u * r * (1 -+ 2^-22) lies strictly below / above W.  The two FFMAs t = RN(u * m + 2^23) round
  // both bracket ends to integers in t's low mantissa bits; when they agree on every code of a group the
  // common value is floor(W + 1/2) (W sits strictly inside (r - 1/2, r + 1/2)), otherwise the group is
  // recomputed with the exact f64 half-up sequence (quant_code), which also decides every exact tie.
  float my_s = 0.f, my_lo = 0.f, my_hi = 0.f;
  bool special = false;
  if (lane < H) {
    my_s = group_scale_k1(my_mn, my_mx, BITS);
    if (my_s >= 0x1p-100f && my_s <= 0x1p100f) {
      const float r = __frcp_rn(my_s);
      my_lo = __fmul_rn(r, 1.f - 0x1p-22f);
      my_hi = __fmul_rn(r, 1.f + 0x1p-22f);
    }
    // no bracket outside [2^-100, 2^100] (codes forced to 0, then redone); scales beyond the f16 range of
    // attn_fast_kernel are recorded (note_scale)
    special = (my_s != 0.f && my_lo == 0.f) || my_s >= 256.f;
  }
  *reinterpret_cast<float4*>(reinterpret_cast<float*>(page + a.L.off_mean[side]) + row * D + 4 * lane) =
      make_float4(mean[0], mean[1], mean[2], mean[3]);
  if (lane < H)
    *reinterpret_cast<float2*>(page + a.L.off_meta[side] + (row * H + lane) * 8) = make_float2(my_s, my_mn);
  uint8_t* codes = page + a.L.off_codes[side] + row * (H * GB) + lane * (BITS / 2);
  uint32_t diff = 0;
#pragma unroll
  for (int h = 0; h < H; ++h) {
    const float ml = __shfl_sync(0xffffffffu, my_lo, h), mh = __shfl_sync(0xffffffffu, my_hi, h);
    uint32_t wl, wh;
    k1_bracket<BITS>(nd, h, ndmax[h], ml, mh, wl, wh);
    diff |= wl ^ wh;  // the constant bits above the fields cancel
    k1_store_codes<BITS>(codes + h * GB, wl);
  }
  if (__any_sync(0xffffffffu, diff != 0 || special)) {  // rare: a code near a rounding boundary, or a special scale
    if (special && my_s >= 256.f) note_scale(a.range, my_s);
    constexpr int CMAX = (1 << BITS) - 1;
#pragma unroll
    for (int h = 0; h < H; ++h) {  // unrolled: nd stays in registers
      const float ml = __shfl_sync(0xffffffffu, my_lo, h), mh = __shfl_sync(0xffffffffu, my_hi, h);
      const float sh = __shfl_sync(0xffffffffu, my_s, h);
      const bool sp = __shfl_sync(0xffffffffu, special && (my_s != 0.f && my_lo == 0.f), h);
      uint32_t wl, wh;
      k1_bracket<BITS>(nd, h, ndmax[h], ml, mh, wl, wh);
      if (!__any_sync(0xffffffffu, wl != wh) && !sp) continue;
      uint32_t w = 0;
      if (sh != 0.f)
#pragma unroll
        for (int k = 0; k < 4; ++k) w |= quant_code(-nd(h, k), __fsub_rn(0.f, ndmax[h]), sh, 0.f, false, CMAX) << (BITS * k);
      k1_store_codes<BITS>(codes + h * GB, w);
    }
  }
}

template <typename T, int BITS, int MINB, bool ROPE>
__global__ void __launch_bounds__(256, MINB) quant_append_fast_kernel(AppendArgs a, int tpw, int page_shift) {
  constexpr int H = 8, D = 128, GB = D * BITS / 8;
  constexpr uint32_t ROWB = H * D * sizeof(T);  // bytes of one token's rows
  extern __shared__ __align__(128) uint8_t k1_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T* ring = reinterpret_cast<T*>(k1_smem + warp * K1_RING * ROWB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(k1_smem + 8 * K1_RING * ROWB) + warp * K1_RING;
  const int side = blockIdx.y & 1, b = blockIdx.y >> 1;
  const int64_t i_begin = (int64_t(blockIdx.x) * 8 + warp) * tpw;
  int64_t count, offset;
  append_part(a, b, count, offset);
  const int64_t i_end = min(count, i_begin + tpw);
  const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
  const int64_t c0 = a.dst_start[b] + offset;
  const T* src_seq = reinterpret_cast<const T*>(a.src[side]) + int64_t(b) * a.src_seq_stride * (H * D);
  const int P = a.L.page_tokens;
  // lane 0 copies the rows of the next token (fsrc, advanced per copy) into ring slot `slot`
  const T* fsrc = src_seq + i_begin * (H * D);
  const uint32_t ring_s = k1_su32(ring), bars_s = k1_su32(bars);
  auto fetch = [&](int slot) {
    const uint32_t bar = bars_s + 8 * slot;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(ROWB) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ring_s + slot * ROWB),
                 "l"(fsrc), "r"(ROWB), "r"(bar)
                 : "memory");
    fsrc += H * D;
  };
  if (lane == 0) {
    for (int k = 0; k < K1_RING; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(k1_su32(&bars[k])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = 0; k < K1_RING - 1 && i_begin + k < i_end; ++k) fetch(k);
  }
  __syncwarp();
  // ring cursor (slot, phase parity) and page cursor (page index, row) advance incrementally
  int slot = 0, fslot = K1_RING - 1;
  uint32_t parity = 0;
  int64_t pg = 0;
  int row = 0;
  {
    const int64_t c = c0 + i_begin;
    pg = page_shift >= 0 ? (c >> page_shift) : c / P;
    row = int(c - pg * P);
  }
#if TADA_K1_PAGE_CACHE
  // the page base changes once every P tokens: load the page-table entry only then
  uint8_t* page = i_begin < i_end ? a.pool + int64_t(pt[pg]) * a.L.page_bytes : nullptr;
#endif
  for (int64_t i = i_begin; i < i_end; ++i) {
    asm volatile(
        "{\n.reg .pred p;\nK1_WAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra K1_WAIT_%=;\n}\n" ::"r"(
            k1_su32(&bars[slot])),
        "r"(parity)
        : "memory");
    const T* src = ring + slot * (H * D) + 4 * lane;
    // every lane has its rows in registers: refill the slot freed last
    auto refill = [&]() {
      __syncwarp();
      if (lane == 0 && i + K1_RING - 1 < i_end) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        fetch(fslot);
      }
      fslot = fslot == K1_RING - 1 ? 0 : fslot + 1;
    };
    bool big = false;
    if (!ROPE && TADA_K1_RECOMP) {
      K1NdLazy<typename K1Row<T>::type> nd;
      nd.x.load(src);
      refill();
      k1_mean(nd.x, nd.m, big);
      k1_token<BITS>(a, nd, nd.m, big, page, row, side, lane);
    } else {
      float mean[4];
      K1NdRegs nd;  // x - mean = -(mean - x): the negated deviations (dev = -nd exactly, cache.py:110)
      if (ROPE && side == 0) {  // rotate the keys in registers (tensor.py:84-89); lane l holds pairs 2l, 2l+1
        K1RowF32 x;
        x.load(src);
        int p = a.positions[int64_t(b) * a.pos_stride + i];
        if (p < 0 || p >= a.rope_rows) {  // the host validates positions; this guards device-side ones
          if (lane == 0 && a.err) atomicOr(a.err, 2);
          p = 0;
        }
        const float4 cs = *reinterpret_cast<const float4*>(a.rope_cs + int64_t(p) * D + 4 * lane);
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const float e0 = x.v[h][0], o0 = x.v[h][1], e1 = x.v[h][2], o1 = x.v[h][3];
          x.v[h][0] = __fsub_rn(__fmul_rn(e0, cs.x), __fmul_rn(o0, cs.y));
          x.v[h][1] = __fadd_rn(__fmul_rn(e0, cs.y), __fmul_rn(o0, cs.x));
          x.v[h][2] = __fsub_rn(__fmul_rn(e1, cs.z), __fmul_rn(o1, cs.w));
          x.v[h][3] = __fadd_rn(__fmul_rn(e1, cs.w), __fmul_rn(o1, cs.z));
        }
        k1_mean_dev(x, mean, nd.v, big);
      } else {
        typename K1Row<T>::type x;
        x.load(src);
        k1_mean_dev(x, mean, nd.v, big);
      }
      refill();
      k1_token<BITS>(a, nd, mean, big, page, row, side, lane);
    }
    if (++slot == K1_RING) {
      slot = 0;
      parity ^= 1u;
    }
    if (++row == P) {
      row = 0;
      ++pg;
#if TADA_K1_PAGE_CACHE
      if (i + 1 < i_end) page = a.pool + int64_t(pt[pg]) * a.L.page_bytes;
#endif
    }
  }
}

template <typename T, int NCH>
static int launch_append_n(const AppendArgs& a, int batch, size_t smem, cudaStream_t st) {
  auto kern = quant_append_kernel<T, NCH>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("quant_append smem: ") + cudaGetErrorString(e));
  }
  dim3 grid(unsigned(int64_t(batch) * a.tiles_per_seq), 2);
  kern<<<grid, 256, smem, st>>>(a);
  return check_launch("quant_append");
}

template <typename T>
static int launch_append(const AppendArgs& a, int batch, size_t smem, cudaStream_t st) {
  const int D = a.L.head_dim;
  if (D == 128 && a.L.heads == 8 && a.vec_ok && (a.L.bits == 2 || a.L.bits == 4 || a.L.bits == 8)) {
    const int tpw = a.n_tok >= 16384 ? 8 : (a.n_tok >= 2048 ? 4 : 1);  // tokens per warp (streamed through the ring)
    const dim3 grid(unsigned((a.n_tok + 8 * tpw - 1) / (8 * tpw)), unsigned(2 * batch));
    const int P = a.L.page_tokens;
    const int shift = (P & (P - 1)) == 0 ? __builtin_ctz(unsigned(P)) : -1;
    const size_t smem = size_t(8) * K1_RING * 8 * 128 * sizeof(T) + 8 * K1_RING * 8;
    // 3 CTAs per SM (80 registers, a few spills) measured faster than 2 (no spills): 3686 vs 3470 GB/s
    auto k = a.rope_cs ? (a.L.bits == 2 ? quant_append_fast_kernel<T, 2, TADA_K1_MINB, true>
                                        : (a.L.bits == 4 ? quant_append_fast_kernel<T, 4, TADA_K1_MINB, true>
                                                         : quant_append_fast_kernel<T, 8, TADA_K1_MINB, true>))
                       : (a.L.bits == 2 ? quant_append_fast_kernel<T, 2, TADA_K1_MINB, false>
                                        : (a.L.bits == 4 ? quant_append_fast_kernel<T, 4, TADA_K1_MINB, false>
                                                         : quant_append_fast_kernel<T, 8, TADA_K1_MINB, false>));
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("quant_append smem: ") + cudaGetErrorString(e));
    }
    k<<<grid, 256, smem, st>>>(a, tpw, shift);
    return check_launch("quant_append_fast");
  }
  if (a.rope_cs) return fail(TADA_ERR_CONFIG, "fused RoPE append needs 16-byte aligned rows (compose apply_rope + quant_append)");
  if (D <= 128) return launch_append_n<T, 1>(a, batch, smem, st);
  if (D <= 256) return launch_append_n<T, 2>(a, batch, smem, st);
  if (D <= 512) return launch_append_n<T, 4>(a, batch, smem, st);
  return launch_append_n<T, 8>(a, batch, smem, st);
}

}  // namespace tada

using namespace tada;

// ====================================================================== C ABI
extern "C" {

int64_t tada_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int tada_abi_version(void) { return TADA_ABI_VERSION; }
const char* tada_last_error(void) { return g_err.c_str(); }

int64_t tada_bytes_per_group(int32_t group_size, int32_t bits) {
  if (!valid_bits(bits) || group_size < 0) return -1;
  return group_bytes(group_size, bits);
}

int tada_page_layout_init(int32_t page_tokens, int32_t heads, int32_t head_dim, int32_t bits, tada_page_layout* out) {
  if (!out) return fail(TADA_ERR_CONFIG, "null layout");
  if (!valid_bits(bits)) return fail(TADA_ERR_CONFIG, "bit width must be one of (2, 4, 8, 16), got " + std::to_string(bits));
  if (page_tokens <= 0 || heads <= 0 || head_dim <= 0)
    return fail(TADA_ERR_CONFIG, "page_tokens, heads and head_dim must be positive");
  if (head_dim > 1024) return fail(TADA_ERR_CONFIG, "head_dim > 1024 is not supported");
  auto up = [](int64_t x, int64_t a) { return (x + a - 1) / a * a; };
  tada_page_layout L{};
  L.page_tokens = page_tokens;
  L.heads = heads;
  L.head_dim = head_dim;
  L.bits = bits;
  L.group_bytes = int32_t(group_bytes(head_dim, bits));
  int64_t off = 0;
  for (int side = 0; side < 2; ++side) {
    L.off_mean[side] = off;
    off = up(off + int64_t(page_tokens) * head_dim * 4, 128);
    L.off_codes[side] = off;
    off = up(off + int64_t(page_tokens) * heads * L.group_bytes, 128);
    L.off_meta[side] = off;
    off = up(off + int64_t(page_tokens) * heads * 8, 128);
  }
  L.page_bytes = up(off, 256);
  *out = L;
  return TADA_OK;
}

int tada_quantize_groups(const void* rows, int32_t dtype, int64_t n_groups, int32_t group_size, int32_t bits,
                         uint8_t* codes, float* scales, float* mins, int32_t* err_flag, void* stream) {
  if (!valid_bits(bits)) return fail(TADA_ERR_CONFIG, "bit width must be one of (2, 4, 8, 16)");
  if (!valid_dtype(dtype)) return fail(TADA_ERR_CONFIG, "dtype must be f32 or bf16");
  if (n_groups < 0 || group_size <= 0 || group_size > 1024) return fail(TADA_ERR_SHAPE, "bad group geometry");
  if (n_groups == 0) return TADA_OK;
  if (!rows || !codes || !scales || !mins) return fail(TADA_ERR_SHAPE, "null buffer");
  return dtype == TADA_F32
             ? launch_quantize<float>(rows, n_groups, group_size, bits, codes, scales, mins, err_flag, S(stream))
             : launch_quantize<__nv_bfloat16>(rows, n_groups, group_size, bits, codes, scales, mins, err_flag, S(stream));
}

int tada_dequantize_groups(const uint8_t* codes, const float* scales, const float* mins, int64_t n_groups,
                           int32_t group_size, int32_t bits, const int64_t* select, int64_t n_select, float* out,
                           void* stream) {
  if (!valid_bits(bits)) return fail(TADA_ERR_CONFIG, "bit width must be one of (2, 4, 8, 16)");
  if (group_size <= 0 || n_groups < 0) return fail(TADA_ERR_SHAPE, "bad group geometry");
  const int64_t n_out = select ? n_select : n_groups;
  if (n_out <= 0) return TADA_OK;
  dequant_kernel<<<grid_for(n_out * group_size, 256), 256, 0, S(stream)>>>(codes, scales, mins, group_size, bits,
                                                                           select, n_out, out);
  return check_launch("dequantize_groups");
}

int tada_pack_codes(const uint8_t* codes, int64_t n_groups, int32_t group_size, int32_t bits, uint8_t* packed,
                    void* stream) {
  if (bits != 2 && bits != 4 && bits != 8) return fail(TADA_ERR_CONFIG, "packing supports widths (2, 4, 8)");
  if (group_size <= 0 || n_groups < 0) return fail(TADA_ERR_SHAPE, "bad group geometry");
  if (n_groups == 0) return TADA_OK;
  pack_kernel<<<grid_for(n_groups * group_bytes(group_size, bits), 256), 256, 0, S(stream)>>>(codes, n_groups,
                                                                                               group_size, bits, packed);
  return check_launch("pack_codes");
}

int tada_unpack_codes(const uint8_t* packed, int64_t n_groups, int32_t group_size, int32_t bits, const int64_t* select,
                      int64_t n_select, uint8_t* codes, void* stream) {
  if (bits != 2 && bits != 4 && bits != 8) return fail(TADA_ERR_CONFIG, "unpacking supports widths (2, 4, 8)");
  if (group_size <= 0 || n_groups < 0) return fail(TADA_ERR_SHAPE, "bad group geometry");
  const int64_t n_out = select ? n_select : n_groups;
  if (n_out <= 0) return TADA_OK;
  unpack_kernel<<<grid_for(n_out * group_size, 256), 256, 0, S(stream)>>>(packed, group_size, bits, select, n_out,
                                                                          codes);
  return check_launch("unpack_codes");
}

int tada_mean_center(const void* x, int32_t dtype, int64_t tokens, int32_t heads, int32_t head_dim, float* mean,
                     float* dev, int32_t* err_flag, void* stream) {
  if (!valid_dtype(dtype)) return fail(TADA_ERR_CONFIG, "dtype must be f32 or bf16");
  if (tokens < 0 || heads <= 0 || head_dim <= 0) return fail(TADA_ERR_SHAPE, "bad (tokens, heads, head_dim)");
  if (tokens == 0) return TADA_OK;
  const int grid = grid_for(tokens * head_dim, 256);
  if (dtype == TADA_F32)
    mean_center_kernel<float><<<grid, 256, 0, S(stream)>>>(reinterpret_cast<const float*>(x), tokens, heads, head_dim,
                                                             mean, dev, err_flag);
  else
    mean_center_kernel<__nv_bfloat16><<<grid, 256, 0, S(stream)>>>(reinterpret_cast<const __nv_bfloat16*>(x), tokens,
                                                                     heads, head_dim, mean, dev, err_flag);
  return check_launch("mean_center");
}

}  // extern "C"

static int quant_append_impl(const tada_page_layout* layout, uint8_t* pool, const void* src_k, const void* src_v,
                             int32_t dtype, int32_t batch, int64_t n_tok, int64_t src_seq_stride,
                             const int32_t* page_table, int32_t pt_stride, const int32_t* dst_start, int64_t dst_offset,
                             int32_t* err_flag, const float* rope_cs, int32_t rope_rows, const int32_t* positions,
                             int64_t pos_stride, void* stream, int part = 0, const int32_t* plan_res = nullptr,
                             const int32_t* plan_n = nullptr, int plan_n_new = 0, int plan_R = 0,
                             int32_t* range = nullptr) {
  if (!layout) return fail(TADA_ERR_CONFIG, "null layout");
  if (!valid_dtype(dtype)) return fail(TADA_ERR_CONFIG, "dtype must be f32 or bf16");
  if (batch < 0 || n_tok < 0 || src_seq_stride < n_tok) return fail(TADA_ERR_SHAPE, "bad batch/token geometry");
  if (batch == 0 || n_tok == 0) return TADA_OK;
  if (!pool || !src_k || !src_v || !page_table || !dst_start) return fail(TADA_ERR_SHAPE, "null buffer");
  AppendArgs a{};
  a.L = *layout;
  a.pool = pool;
  a.src[0] = src_k;
  a.src[1] = src_v;
  a.n_tok = n_tok;
  a.src_seq_stride = src_seq_stride;
  a.page_table = page_table;
  a.pt_stride = pt_stride;
  a.dst_start = dst_start;
  a.dst_offset = dst_offset;
  a.err = err_flag;
  a.rope_cs = rope_cs;
  a.rope_rows = rope_rows;
  a.positions = positions;
  a.pos_stride = pos_stride;
  a.part = part;
  a.plan_res = plan_res;
  a.plan_n = plan_n;
  a.plan_n_new = plan_n_new;
  a.plan_R = plan_R;
  a.range = range;
  const int row = layout->heads * layout->head_dim;
  const size_t per_tok = size_t(row + layout->head_dim) * 4;
  int tt = int((32 * 1024) / per_tok);
  tt = tt < 1 ? 1 : (tt > 16 ? 16 : tt);
  if (tt > n_tok) tt = int(n_tok);
  const size_t smem = per_tok * tt;
  if (smem > 200 * 1024) return fail(TADA_ERR_CONFIG, "heads*head_dim too large for quant_append");
  a.tt = tt;
  a.tiles_per_seq = int((n_tok + tt - 1) / tt);
  const size_t esz = dtype == TADA_F32 ? 4 : 2;
  a.vec_ok = (layout->head_dim % 4 == 0) && (reinterpret_cast<uintptr_t>(src_k) % 16 == 0) &&
             (reinterpret_cast<uintptr_t>(src_v) % 16 == 0) && ((src_seq_stride * row * esz) % 16 == 0) &&
             (layout->group_bytes % 4 == 0 || layout->bits <= 4);
  return dtype == TADA_F32 ? launch_append<float>(a, batch, smem, S(stream))
                           : launch_append<__nv_bfloat16>(a, batch, smem, S(stream));
}

extern "C" {

int tada_quant_append(const tada_page_layout* layout, uint8_t* pool, const void* src_k, const void* src_v,
                      int32_t dtype, int32_t batch, int64_t n_tok, int64_t src_seq_stride, const int32_t* page_table,
                      int32_t pt_stride, const int32_t* dst_start, int64_t dst_offset, int32_t* err_flag,
                      void* stream) {
  return quant_append_impl(layout, pool, src_k, src_v, dtype, batch, n_tok, src_seq_stride, page_table, pt_stride,
                           dst_start, dst_offset, err_flag, nullptr, 0, nullptr, 0, stream);
}

int tada_quant_append_plan(const tada_page_layout* layout, uint8_t* pool, const void* src_k, const void* src_v,
                           int32_t dtype, int32_t batch, int64_t n_max, int64_t src_seq_stride,
                           const int32_t* page_table, int32_t pt_stride, const int32_t* comp_len,
                           const int32_t* res_len, int32_t residual_length, int32_t n_new, const int32_t* seq_n,
                           int32_t part, const int32_t* positions, int64_t pos_stride, const float* rope_cs,
                           int32_t rope_rows, int32_t* err_flag, int32_t* range_word, void* stream) {
  if (!layout) return fail(TADA_ERR_CONFIG, "null layout");
  if (part != 1 && part != 2) return fail(TADA_ERR_CONFIG, "part must be 1 (residual rows) or 2 (new rows)");
  if (!res_len) return fail(TADA_ERR_SHAPE, "null buffer");
  if (residual_length < 0 || n_new < 0) return fail(TADA_ERR_SHAPE, "bad plan geometry");
  if (rope_cs) {
    if (part != 2) return fail(TADA_ERR_CONFIG, "only the new rows are rotated (residual rows are stored rotated)");
    if (!(layout->head_dim == 128 && layout->heads == 8 && (layout->bits == 2 || layout->bits == 4 || layout->bits == 8)))
      return fail(TADA_ERR_CONFIG, "fused RoPE append needs heads 8, head_dim 128, bits 2/4/8");
    if (!positions || rope_rows <= 0 || pos_stride < n_max) return fail(TADA_ERR_SHAPE, "bad rope arguments");
  }
  return quant_append_impl(layout, pool, src_k, src_v, dtype, batch, n_max, src_seq_stride, page_table, pt_stride,
                           comp_len, 0, err_flag, rope_cs, rope_rows, positions, pos_stride, stream, part, res_len,
                           seq_n, n_new, residual_length, range_word);
}

int tada_append_commit(float* res_k, float* res_v, int64_t res_seq_stride, int32_t heads, int32_t head_dim,
                       const void* src_k, const void* src_v, int32_t dtype, int32_t batch, int64_t src_seq_stride,
                       int32_t n_new, const int32_t* seq_n, int32_t residual_length, int32_t* comp_len,
                       int32_t* res_len, const int32_t* positions, int64_t pos_stride, const float* rope_cs,
                       int32_t rope_rows, int32_t* err_flag, void* stream) {
  if (!valid_dtype(dtype)) return fail(TADA_ERR_CONFIG, "dtype must be f32 or bf16");
  if (batch < 0 || n_new < 0 || heads <= 0 || head_dim <= 0 || residual_length < 0)
    return fail(TADA_ERR_SHAPE, "bad append geometry");
  if (batch == 0) return TADA_OK;
  if (!comp_len || !res_len || (residual_length > 0 && (!res_k || !res_v || !src_k || !src_v)))
    return fail(TADA_ERR_SHAPE, "null buffer");
  if (rope_cs && (head_dim % 2 || !positions || rope_rows <= 0)) return fail(TADA_ERR_SHAPE, "bad rope arguments");
  cudaStream_t st = S(stream);
#define TADA_COMMIT(T, ROPE)                                                                                    \
  append_commit_kernel<T, ROPE><<<batch, 256, 0, st>>>(res_k, res_v, res_seq_stride, heads, head_dim,             \
                                                       reinterpret_cast<const T*>(src_k),                       \
                                                       reinterpret_cast<const T*>(src_v), src_seq_stride, n_new, \
                                                       seq_n, residual_length, comp_len, res_len, positions,     \
                                                       pos_stride, rope_cs, rope_rows, err_flag)
  if (dtype == TADA_F32) {
    if (rope_cs) TADA_COMMIT(float, true);
    else TADA_COMMIT(float, false);
  } else {
    if (rope_cs) TADA_COMMIT(__nv_bfloat16, true);
    else TADA_COMMIT(__nv_bfloat16, false);
  }
#undef TADA_COMMIT
  return check_launch("append_commit");
}

int tada_gather_compressed(const tada_page_layout* layout, const uint8_t* pool, const int32_t* page_row, int64_t n_tok,
                           int32_t side, float* mean, uint8_t* codes, float* scales, float* mins, void* stream) {
  if (!layout || side < 0 || side > 1) return fail(TADA_ERR_CONFIG, "bad layout/side");
  if (n_tok <= 0) return TADA_OK;
  const int64_t per = layout->head_dim + int64_t(layout->heads) * layout->group_bytes + 2 * layout->heads;
  move_compressed_kernel<true><<<grid_for(n_tok * per, 256), 256, 0, S(stream)>>>(
      *layout, const_cast<uint8_t*>(pool), page_row, n_tok, side, mean, codes, scales, mins);
  return check_launch("gather_compressed");
}

int tada_scatter_compressed(const tada_page_layout* layout, uint8_t* pool, const int32_t* page_row, int64_t n_tok,
                            int32_t side, const float* mean, const uint8_t* codes, const float* scales,
                            const float* mins, void* stream) {
  if (!layout || side < 0 || side > 1) return fail(TADA_ERR_CONFIG, "bad layout/side");
  if (n_tok <= 0) return TADA_OK;
  const int64_t per = layout->head_dim + int64_t(layout->heads) * layout->group_bytes + 2 * layout->heads;
  move_compressed_kernel<false><<<grid_for(n_tok * per, 256), 256, 0, S(stream)>>>(
      *layout, pool, page_row, n_tok, side, const_cast<float*>(mean), const_cast<uint8_t*>(codes),
      const_cast<float*>(scales), const_cast<float*>(mins));
  return check_launch("scatter_compressed");
}

}  // extern "C"
