// Shared declarations between the decode-attention translation units.
#pragma once

#include <cuda.h>

#include <atomic>
#include <string>

#include "tada_common.cuh"

namespace tada {

struct AttnArgs {
  tada_page_layout L;
  const uint8_t* pool;
  const void* q;
  int Hq;
  const int32_t* page_table;
  int pt_stride;
  const int32_t* comp_len;
  const int32_t* res_len;
  const float* res_k;
  const float* res_v;
  int64_t res_seq_stride;
  float scale;
  int splits;       // splits over the compressed tokens (fast path) or all tokens (generic)
  int slots;        // partial slots per (b, g) in the workspace (fast path: splits + 1 for the residual)
  float* part_acc;  // [B][Hq][slots][D]
  float* part_ml;   // [B][Hq][slots][2]
  void* out;
  int out_dtype;
  int q_dtype;
  // decode step (tada_decode_step): the step's new K/V row [batch][heads][head_dim], attended by K3 straight
  // from the input and stored at the sequence's next residual row
  const void* new_k;
  const void* new_v;
  int new_dtype;
  int diag;  // diagnostics only (env TADA_ATTN_DIAG): 1 = TMA ring without compute, 2 = compute on one L2-resident page
  float* lse_out;  // optional [B][Hq]: natural-log sum-exp of the scaled logits (cross-rank merge)
  // device-planned decode step (tada_decode_step): one new row per sequence, residual_length step_R; each
  // sequence's flush decision comes from its own res_len (seq_plan), K3 advances the lengths (step_sync:
  // per-sequence arrival counters, zero between steps)
  int step;
  int step_R;
  int32_t* step_sync;
  // the layer's range words (K1's note_range): [0] binary exponent of its largest stored |mean| >= 2^15,
  // [1] of its largest group scale >= 2^8 (0 when below)
  const int32_t* range;
  // a view of KV heads kv_h0 .. kv_h0 + L.heads - 1 of a layout with kv_rh heads per token row (head-group
  // passes, tada_attn.cu): L.off_codes / L.off_meta already point at head kv_h0 of each row; the code and meta
  // rows, the residual rows and the step's new rows are kv_rh heads wide.  Normally kv_rh = L.heads, kv_h0 = 0.
  int kv_rh;
  int kv_h0;
  bool step_commit;  // a decode step's K3 advances the lengths (false for all but the last view / q-head pass)
  int commit_units;  // > 1: that many concurrent (view, pass) launches share the step's arrival counters
};

// The tensor-core kernels stage q and the f32 means (f16 hi + lo / f16) as f16, which holds |x| < 65504, and
// P' = -p * vscale with the lazy softmax's p <= 2^8: attn_v8_kernel pre-scales it by 2^-8 (safe for scales
// below 2^15), attn_fast_kernel does not (safe below 2^8).  A layer whose range words pass those bounds, or a
// query element of magnitude >= 2^15, is attended on the exact f32 path below instead (rare; mode 0 never
// returns inf/NaN for finite inputs).
constexpr int kF16SafeExp = 15;    // |mean|, |q| and (attn_v8_kernel) vscale below 2^15
constexpr int kFastScaleExp = 8;   // attn_fast_kernel: vscale below 2^8
__device__ __forceinline__ bool beyond_f16(const AttnArgs& a, int scale_exp) {
  return a.range && (a.range[0] >= kF16SafeExp || a.range[1] >= scale_exp);
}

// Exact f32 partials of one K2 split over compressed tokens [t_begin, t_end) of sequence b, in the
// tensor-core kernels' slot format (natural-log max, normaliser, unnormalised weighted sum): warp w < H
// attends for KV head w, lane = 4 columns; K̂ = mean - fmaf(code, scale, min) as in the reference's
// reconstruct_slice (cache.py:190-213), logits scaled after the dot (attention.py:118-136).
template <int BITS, int G>
__device__ void exact_split_partials(const AttnArgs& a, int b, int split, int t_begin, int t_end, int warp,
                                     int lane) {
  constexpr int D = 128;
  const int H = a.L.heads, Hq = a.Hq, P = a.L.page_tokens, gb = a.L.group_bytes;
  if (warp >= H) return;
  const int h = warp;
  const float NEG_INF = -__int_as_float(0x7f800000);
  if (a.kv_h0 + h >= a.kv_rh) {  // a view's missing KV head (fewer than 8 in the layout): empty slots
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int64_t slot = (int64_t(b) * Hq + h * G + g) * a.slots + split;
      *reinterpret_cast<float4*>(a.part_acc + slot * D + 4 * lane) = make_float4(0.f, 0.f, 0.f, 0.f);
      if (lane == 0) {
        a.part_ml[slot * 2] = NEG_INF;
        a.part_ml[slot * 2 + 1] = 0.f;
      }
    }
    return;
  }
  float q[G][4], acc[G][4], m[G], l[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int64_t qi = (int64_t(b) * Hq + h * G + g) * D + 4 * lane;
    if (a.q_dtype == TADA_F32) load4(reinterpret_cast<const float*>(a.q) + qi, q[g]);
    else load4(reinterpret_cast<const __nv_bfloat16*>(a.q) + qi, q[g]);
    acc[g][0] = acc[g][1] = acc[g][2] = acc[g][3] = 0.f;
    m[g] = NEG_INF;
    l[g] = 0.f;
  }
  const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
  for (int t = t_begin; t < t_end; ++t) {
    const uint8_t* page = a.pool + int64_t(pt[t / P]) * a.L.page_bytes;
    const int r = t % P;
    float kh[4], vh[4];
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const float4 mean = *reinterpret_cast<const float4*>(page + a.L.off_mean[side] + (int64_t(r) * D + 4 * lane) * 4);
      const uint8_t* grp = page + a.L.off_codes[side] + (int64_t(r) * a.kv_rh + h) * gb;
      const float2 sm = *reinterpret_cast<const float2*>(page + a.L.off_meta[side] + (int64_t(r) * a.kv_rh + h) * 8);
      const float mv[4] = {mean.x, mean.y, mean.z, mean.w};
      float* dst = side ? vh : kh;
#pragma unroll
      for (int e = 0; e < 4; ++e)
        dst[e] = __fsub_rn(mv[e], __fmaf_rn(float(get_code(grp, 4 * lane + e, BITS)), sm.x, sm.y));
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float z = __fmaf_rn(q[g][3], kh[3], __fmaf_rn(q[g][2], kh[2], __fmaf_rn(q[g][1], kh[1], __fmul_rn(q[g][0], kh[0]))));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
      z = __fmul_rn(z, a.scale);
      const float mn = fmaxf(m[g], z);
      const float cf = expf(m[g] - mn), p = expf(z - mn);
      l[g] = l[g] * cf + p;
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[g][e] = fmaf(p, vh[e], acc[g][e] * cf);
      m[g] = mn;
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int64_t slot = (int64_t(b) * Hq + h * G + g) * a.slots + split;
    *reinterpret_cast<float4*>(a.part_acc + slot * D + 4 * lane) = make_float4(acc[g][0], acc[g][1], acc[g][2], acc[g][3]);
    if (lane == 0) {
      a.part_ml[slot * 2] = l[g] > 0.f ? m[g] : NEG_INF;
      a.part_ml[slot * 2 + 1] = l[g];
    }
  }
}

// Compressed tokens K2 attends for sequence b: in a decode step, those a flush of this step adds too (K1
// compressed them just before).
__device__ __forceinline__ int comp_tokens(const AttnArgs& a, int b) {
  return a.comp_len[b] + (a.step ? seq_plan(a.res_len[b], 1, a.step_R).ncomp : 0);
}

// K3 side of a decode step: how many residual rows sequence b attends and which of them
// (r_new, or -1) is the step's new row read from the input.
__device__ __forceinline__ void residual_rows(const AttnArgs& a, int b, int& rows, int& r_new, int h = 0) {
  if (a.kv_h0 + h >= a.kv_rh) {  // a view's missing KV head (fewer than 8 in the layout)
    rows = 0;
    r_new = -1;
    return;
  }
  if (a.step) {
    const int rb = a.res_len[b];
    const SeqPlan p = seq_plan(rb, 1, a.step_R);
    rows = p.res_after;
    r_new = (a.step_R > 0 && p.ncomp == 0) ? rb : -1;
  } else {
    rows = a.res_len[b];
    r_new = -1;
  }
}

// Last of `ctas` CTAs of sequence b in a decode step's K3: advance its lengths (every CTA read them at
// entry, before its arrival; the counter returns to zero for the next step).  Call from one thread after
// the CTA's last global read of the lengths.
__device__ __forceinline__ void step_commit(const AttnArgs& a, int b, int ctas) {
  __threadfence();
  const int old = atomicAdd(&a.step_sync[b], 1);
  if (old == ctas - 1) {
    const SeqPlan p = seq_plan(a.res_len[b], 1, a.step_R);
    const_cast<int32_t*>(a.comp_len)[b] += p.ncomp;
    const_cast<int32_t*>(a.res_len)[b] = p.res_after;
    a.step_sync[b] = 0;
    __threadfence();
  }
}

__device__ __forceinline__ void store_any(void* out, int dtype, int64_t i, float v) {
  if (dtype == TADA_F32) reinterpret_cast<float*>(out)[i] = v;
  else reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(v);
}

// Token range [t0, t1) of split s out of n tokens; chunk boundaries are multiples of `align`.
__device__ __forceinline__ void split_range(int n, int splits, int s, int align, int& t0, int& t1) {
  int chunk = (n + splits - 1) / splits;
  chunk = (chunk + align - 1) / align * align;
  t0 = min(n, s * chunk);
  t1 = min(n, t0 + chunk);
}

// TMA descriptors of one layer pool: [side][region] with region 0 = means, 1 = codes, 2 = scale/min.
struct alignas(64) TmaMaps {
  CUtensorMap m[2][3];
};

// Raise a kernel's dynamic shared-memory limit once per device (thread-safe; `done` is a per-kernel bitmask
// of devices already configured).
// Programmatic dependent launch (PDL): decode launches K2 -> K3 -> next layer's K2 back to back.  Each
// is launched with programmatic stream serialization and, at entry, lets its dependent launch and then
// waits for its prerequisites (griddepcontrol.wait: previous grid complete, its writes visible) before
// any global read, so only the launch and CTA ramp overlap the previous kernel's tail, never data.
// TADA_PDL=0 in the environment turns it off (A/B).
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
bool pdl_enabled();
template <typename Kern, typename... Args>
cudaError_t launch_maybe_pdl(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  if (!pdl_enabled()) {
    kern<<<grid, block, smem, st>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename Kern>
int ensure_smem(Kern kern, int bytes, std::atomic<uint64_t>& done, const char* what) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail(TADA_ERR_CUDA, "cudaGetDevice failed");
  const uint64_t bit = uint64_t(1) << dev;
  if (done.load(std::memory_order_acquire) & bit) return TADA_OK;
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string(what) + " smem: " + cudaGetErrorString(e));
  done.fetch_or(bit, std::memory_order_acq_rel);
  return TADA_OK;
}

// Fast path (tensor-core grouped-head contraction); returns TADA_ERR_CONFIG if the
// geometry is unsupported so the caller can fall back to the generic kernel.
bool fast_supported(const tada_page_layout& L, int Hq);
// tensor-core head mapping: `passes` passes of up to gc q heads per KV head, each padded to gp rows (tada_attn.cu)
struct FastMap {
  int passes, gc, gp, g;
  int hg = 1;         // head groups of 8 KV heads (layouts with 16, 24, 32, ... KV heads run one view per group)
  bool view = false;  // the layout is not 8 KV heads: views (head_group_view; fewer than 8 heads zero-filled)
  bool direct() const { return passes == 1 && gp == g && !view; }
};
// the view of KV heads 8j .. 8j + 7 of a layout with a multiple of 8 heads (AttnArgs::kv_rh / kv_h0)
tada_page_layout head_group_view(const tada_page_layout& L, int j);
bool fast_map(const tada_page_layout& L, int Hq, FastMap* m);
int launch_fast_mapped(const AttnArgs& a, int batch, const FastMap& fm, int mode, void* workspace, cudaStream_t st);
int launch_fast(const AttnArgs& a, int batch, cudaStream_t st);
int fast_tile_tokens(const tada_page_layout& L, int Hq);  // 16 or 32 (0: unsupported)
// One-barrier-per-tile kernel (tada_attn_v8.cu): 2/4-bit (8-bit where two stages fit), Hq in {8, 16, 32}.
bool v8_supported(const tada_page_layout& L, int Hq);
int launch_v8(const AttnArgs& a, int batch, cudaStream_t st);
// Staged exact f32 kernel for any geometry (tada_attn_exact.cu): compressed tokens only, K3 adds the residual.
int exact_smem_bytes(const tada_page_layout& L, int Hq);  // 0: geometry too large (use attn_generic_kernel)
int exact_ctas_per_sm(const tada_page_layout& L, int Hq);
int launch_exact(const AttnArgs& a, int batch, cudaStream_t st);
// Cached TMA descriptors of a layer pool for TT-token tiles (tada_attn_fast.cu).
int get_tma_maps(const AttnArgs& a, TmaMaps* out, int tt);

}  // namespace tada
