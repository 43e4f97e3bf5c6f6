// K2 (split-K decode attention over the compressed paged cache) and K3 (LSE combine).
//
// Reference: pkg/src/tadakv/attention.py attend_streaming (103-151): per KV head,
// tiles over compressed then residual tokens (94-100); logits = (K̂ @ q) * F32(1/sqrt(D));
// running max / normalizer / weighted sum; out = acc / norm.  K̂ = mean - deq(dev)
// (cache.py:193-200) with deq = fmaf(code, scale, min), bit-identical to the
// reference's f32(f64 min + code * f64 scale) (SURVEY §8a "Dequant").
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <string>

#include "tada_attn.cuh"

#ifndef TADA_K3_KV
#define TADA_K3_KV 1  // 0: the per-q-head combine_pair_kernel for every G (A/B)
#endif

namespace tada {

template <int BITS>
__device__ __forceinline__ float khat_elem(const float* mean, const uint8_t* grp, float s, float mn, int d) {
  if (BITS == 16) return __fsub_rn(mean[d], reinterpret_cast<const float*>(grp)[d]);
  return __fsub_rn(mean[d], __fmaf_rn(float(get_code(grp, d, BITS)), s, mn));
}

// ------------------------------------------------------------------ generic exact kernel
// Any (H, Hq, D, bits).  CTA = (split, sequence); f32 reconstruct-then-dot.
constexpr int kGenTile = 32;

template <typename QT, int BITS>
__global__ void __launch_bounds__(256) attn_generic_kernel(AttnArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int H = a.L.heads, D = a.L.head_dim, Hq = a.Hq, G = Hq / H, P = a.L.page_tokens, gb = a.L.group_bytes;
  const int b = blockIdx.y, split = blockIdx.x, tid = threadIdx.x, bd = blockDim.x;
  float* qs = sm;                 // [Hq][D]
  float* acc = qs + Hq * D;       // [Hq][D]
  float* lg = acc + Hq * D;       // [Hq][kGenTile]
  float* mrow = lg + Hq * kGenTile;
  float* lrow = mrow + Hq;
  float* crow = lrow + Hq;
  const int C = a.comp_len[b], n = C + a.res_len[b];
  int t_begin, t_end;
  split_range(n, a.splits, split, kGenTile, t_begin, t_end);
  const QT* q = reinterpret_cast<const QT*>(a.q) + int64_t(b) * Hq * D;
  for (int i = tid; i < Hq * D; i += bd) {
    qs[i] = to_f32(q[i]);
    acc[i] = 0.f;
  }
  for (int g = tid; g < Hq; g += bd) {
    mrow[g] = -__int_as_float(0x7f800000);
    lrow[g] = 0.f;
  }
  __syncthreads();
  const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
  const int64_t res_base = int64_t(b) * a.res_seq_stride;

  for (int t0 = t_begin; t0 < t_end; t0 += kGenTile) {
    const int nt = min(kGenTile, t_end - t0);
    for (int pair = tid; pair < Hq * nt; pair += bd) {
      const int g = pair / nt, j = pair - g * nt, t = t0 + j, h = g / G;
      const float* qg = qs + g * D;
      float dot = 0.f;
      if (t < C) {
        const uint8_t* page = a.pool + int64_t(pt[t / P]) * a.L.page_bytes;
        const int r = t % P;
        const float* mean = reinterpret_cast<const float*>(page + a.L.off_mean[0]) + r * D;
        const uint8_t* grp = page + a.L.off_codes[0] + (int64_t(r) * H + h) * gb;
        const float2 sm2 = reinterpret_cast<const float2*>(page + a.L.off_meta[0])[r * H + h];
        for (int d = 0; d < D; ++d) dot = __fmaf_rn(qg[d], khat_elem<BITS>(mean, grp, sm2.x, sm2.y, d), dot);
      } else {
        const float* kr = a.res_k + ((res_base + (t - C)) * H + h) * D;
        for (int d = 0; d < D; ++d) dot = __fmaf_rn(qg[d], kr[d], dot);
      }
      lg[g * kGenTile + j] = __fmul_rn(dot, a.scale);
    }
    __syncthreads();
    for (int g = tid; g < Hq; g += bd) {
      float tmax = lg[g * kGenTile];
      for (int j = 1; j < nt; ++j) tmax = fmaxf(tmax, lg[g * kGenTile + j]);
      const float m_new = fmaxf(mrow[g], tmax);
      const float corr = expf(mrow[g] - m_new);
      float sum = 0.f;
      for (int j = 0; j < nt; ++j) {
        const float p = expf(lg[g * kGenTile + j] - m_new);
        lg[g * kGenTile + j] = p;
        sum += p;
      }
      lrow[g] = lrow[g] * corr + sum;
      mrow[g] = m_new;
      crow[g] = corr;
    }
    __syncthreads();
    for (int pair = tid; pair < Hq * D; pair += bd) {
      const int g = pair / D, d = pair - g * D, h = g / G;
      float av = acc[pair] * crow[g];
      for (int j = 0; j < nt; ++j) {
        const int t = t0 + j;
        float v;
        if (t < C) {
          const uint8_t* page = a.pool + int64_t(pt[t / P]) * a.L.page_bytes;
          const int r = t % P;
          const float* mean = reinterpret_cast<const float*>(page + a.L.off_mean[1]) + r * D;
          const uint8_t* grp = page + a.L.off_codes[1] + (int64_t(r) * H + h) * gb;
          const float2 sm2 = reinterpret_cast<const float2*>(page + a.L.off_meta[1])[r * H + h];
          v = khat_elem<BITS>(mean, grp, sm2.x, sm2.y, d);
        } else {
          v = a.res_v[((res_base + (t - C)) * H + h) * D + d];
        }
        av = __fmaf_rn(lg[g * kGenTile + j], v, av);
      }
      acc[pair] = av;
    }
    __syncthreads();
  }
  if (a.splits == 1) {
    for (int pair = tid; pair < Hq * D; pair += bd) {
      const int g = pair / D;
      store_any(a.out, a.out_dtype, int64_t(b) * Hq * D + pair, acc[pair] / lrow[g]);
    }
    if (a.lse_out)
      for (int g = tid; g < Hq; g += bd) a.lse_out[int64_t(b) * Hq + g] = mrow[g] + logf(lrow[g]);
  } else {
    for (int pair = tid; pair < Hq * D; pair += bd) {
      const int g = pair / D, d = pair - g * D;
      a.part_acc[((int64_t(b) * Hq + g) * a.slots + split) * D + d] = acc[pair];
    }
    for (int g = tid; g < Hq; g += bd) {
      float* ml = a.part_ml + ((int64_t(b) * Hq + g) * a.slots + split) * 2;
      ml[0] = mrow[g];
      ml[1] = lrow[g];
    }
  }
}

// ------------------------------------------------------------------ K3: split combine
// out = sum_s acc_s * e^{m_s - M} / sum_s l_s * e^{m_s - M}   (log-sum-exp merge)
__global__ void combine_kernel(const float* __restrict__ part_acc, const float* __restrict__ part_ml, int S, int D,
                               void* out, int out_dtype, float* lse_out) {
  const int64_t bg = blockIdx.x;  // b * Hq + g
  const float* ml = part_ml + bg * S * 2;
  float M = -__int_as_float(0x7f800000);
  for (int s = 0; s < S; ++s) M = fmaxf(M, ml[2 * s]);
  float L = 0.f;
  for (int s = 0; s < S; ++s)
    if (ml[2 * s + 1] > 0.f) L += ml[2 * s + 1] * expf(ml[2 * s] - M);
  const float inv = 1.f / L;
  if (lse_out && threadIdx.x == 0) lse_out[bg] = M + logf(L);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float o = 0.f;
    for (int s = 0; s < S; ++s)
      if (ml[2 * s + 1] > 0.f) o += part_acc[(bg * S + s) * D + d] * expf(ml[2 * s] - M);
    store_any(out, out_dtype, bg * D + d, o * inv);
  }
}

// ------------------------------------------------------------------ cross-rank merge of normalised partials
// Each part p holds o_p = softmax-weighted mean over its own tokens and lse_p = log sum exp of its
// logits (-inf: part saw no tokens).  out = sum_p o_p e^{lse_p - M} / sum_p e^{lse_p - M}.
__global__ void combine_lse_kernel(const float* __restrict__ o, const float* __restrict__ lse, int n, int64_t rows,
                                   int D, void* out, int out_dtype, float* lse_out) {
  const int64_t row = blockIdx.x;
  float M = -__int_as_float(0x7f800000);
  for (int p = 0; p < n; ++p) M = fmaxf(M, lse[p * rows + row]);
  float W = 0.f;
  for (int p = 0; p < n; ++p) {
    const float l = lse[p * rows + row];
    if (l > -__int_as_float(0x7f800000)) W += expf(l - M);
  }
  const float inv = 1.f / W;
  if (lse_out && threadIdx.x == 0) lse_out[row] = M + logf(W);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < n; ++p) {
      const float l = lse[p * rows + row];
      if (l > -__int_as_float(0x7f800000)) acc += o[(p * rows + row) * D + d] * expf(l - M);
    }
    store_any(out, out_dtype, row * D + d, acc * inv);
  }
}

// ------------------------------------------------------------------ K3 for the tensor-core path:
// residual rows + split merge, one CTA per (KV head, sequence).
// The raw f32 residual tokens (cache.py:174-180) are attended exactly like the reference's
// residual tiles (attention.py:94-100: f32 dot, scale after the dot) and merged with the
// compressed-token splits by the log-sum-exp rule:
//   out = (Σ_s e^{m_s-M} acc_s + e^{m_r-M} Σ_t p_t v_t) / (Σ_s e^{m_s-M} l_s + e^{m_r-M} l_r)
constexpr int kCombThreads = 256;
__device__ __forceinline__ float block_reduce(float v, float* red, bool is_max) {
  for (int o = 16; o > 0; o >>= 1) {
    const float u = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, u) : v + u;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = red[0];
  for (int w = 1; w < kCombThreads / 32; ++w) r = is_max ? fmaxf(r, red[w]) : r + red[w];
  __syncthreads();
  return r;
}

// One CTA per (q head, sequence), 256 threads.
__global__ void __launch_bounds__(kCombThreads) combine_residual_kernel(AttnArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int H = a.L.heads, D = a.L.head_dim, Hq = a.Hq, G = Hq / H, S = a.splits;
  const int gq = blockIdx.x, b = blockIdx.y, h = gq / G, tid = threadIdx.x;
  const int R = a.res_len[b];
  float* qs = sm;            // [D]
  float* pr = qs + D;        // [rcap] residual logits -> probabilities
  float* ws = pr + a.res_seq_stride;  // [S] split weights
  float* part = ws + S;      // [2][D] partial outputs of the two thread halves
  float* red = part + 2 * D; // [8]
  const int64_t qi = (int64_t(b) * Hq + gq) * D;
  for (int i = tid; i < D; i += kCombThreads)
    qs[i] = a.q_dtype == TADA_F32 ? reinterpret_cast<const float*>(a.q)[qi + i]
                                  : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.q)[qi + i]);
  __syncthreads();
  const int64_t rbase = int64_t(b) * a.res_seq_stride;
  float mx = -__int_as_float(0x7f800000);
  // residual logits: one warp per token, lanes split d (4 each) and reduce by shuffles
  const int warp = tid >> 5, lane = tid & 31;
  for (int t = warp; t < R; t += kCombThreads / 32) {
    const float* kr = a.res_k + ((rbase + t) * a.kv_rh + a.kv_h0 + h) * D;
    float dot = 0.f;
    for (int d = 4 * lane; d < D; d += 128) {  // the fast path has D % 4 == 0
      const float4 k4 = *reinterpret_cast<const float4*>(kr + d);
      const float4 q4 = *reinterpret_cast<const float4*>(qs + d);
      dot = __fmaf_rn(q4.w, k4.w, __fmaf_rn(q4.z, k4.z, __fmaf_rn(q4.y, k4.y, __fmaf_rn(q4.x, k4.x, dot))));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const float sv = __fmul_rn(dot, a.scale);
    if (lane == 0) pr[t] = sv;
    mx = fmaxf(mx, sv);
  }
  const float* ml = a.part_ml + (int64_t(b) * Hq + gq) * a.slots * 2;
  for (int s2 = tid; s2 < S; s2 += kCombThreads)
    if (ml[2 * s2 + 1] > 0.f) mx = fmaxf(mx, ml[2 * s2]);
  const float M = block_reduce(mx, red, true);
  float lsum = 0.f;
  for (int t = tid; t < R; t += kCombThreads) {
    const float p = expf(pr[t] - M);
    pr[t] = p;
    lsum += p;
  }
  for (int s2 = tid; s2 < S; s2 += kCombThreads) {
    const float w = ml[2 * s2 + 1] > 0.f ? expf(ml[2 * s2] - M) : 0.f;
    ws[s2] = w;
    lsum += w * ml[2 * s2 + 1];
  }
  const float L = block_reduce(lsum, red, false);  // its barrier also publishes pr / ws
  // output: thread = (half j, d); with D <= 128 each of two halves takes every other slot and residual token,
  // with D up to 256 one half takes them all
  const int NH = 2 * D <= kCombThreads ? 2 : 1;
  const int j = tid / D, d = tid - j * D;
  if (j < NH) {
    // the partial slots live in L2 (written by K2 just before): issue a batch of loads, then the FMAs
    constexpr int U = 8;
    const float* pa = a.part_acc + (int64_t(b) * Hq + gq) * a.slots * D + d;
    float acc0 = 0.f, acc1 = 0.f;
    for (int s0 = j; s0 < S; s0 += NH * U) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = s0 + NH * u < S ? pa[int64_t(s0 + NH * u) * D] : 0.f;
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        acc0 = fmaf(s0 + NH * u < S ? ws[s0 + NH * u] : 0.f, v[u], acc0);
        acc1 = fmaf(s0 + NH * (u + 1) < S ? ws[s0 + NH * (u + 1)] : 0.f, v[u + 1], acc1);
      }
    }
    const float* vr = a.res_v + (rbase * a.kv_rh + a.kv_h0 + h) * D + d;
    for (int t0 = j; t0 < R; t0 += NH * U) {
      float v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = t0 + NH * u < R ? vr[int64_t(t0 + NH * u) * a.kv_rh * D] : 0.f;
#pragma unroll
      for (int u = 0; u < U; u += 2) {
        acc0 = fmaf(t0 + NH * u < R ? pr[t0 + NH * u] : 0.f, v[u], acc0);
        acc1 = fmaf(t0 + NH * (u + 1) < R ? pr[t0 + NH * (u + 1)] : 0.f, v[u + 1], acc1);
      }
    }
    part[j * D + d] = acc0 + acc1;
  }
  __syncthreads();
  for (int dd = tid; dd < D; dd += kCombThreads) {
    store_any(a.out, a.out_dtype, qi + dd, (NH == 2 ? part[dd] + part[D + dd] : part[dd]) / L);
    if (dd == 0 && a.lse_out) a.lse_out[int64_t(b) * Hq + gq] = M + logf(L);
  }
}

// K3 for head_dim 128: four warps per (q head, sequence), lane l owning d = 4l .. 4l+3.  Warp 0 of the
// group merges the split partials, warps 1..3 attend the residual rows (batches of 8 rows round-robin;
// warp 1 also stores this step's new row); each runs an online softmax whose global loads are all issued
// before their consumers, and the four parts meet in shared memory with one rescale.  The residual grows
// by a row per decode step (up to R = 128 between flushes), so its batches are spread over three warps.
// (The first one-warp version walked ~10 dependent global round trips per row.)
__global__ void __launch_bounds__(256) combine_pair_kernel(AttnArgs a, int n_rows) {
  constexpr int D = 128, U = 8, RW = 3;  // RW residual warps per row
  __shared__ float rx[2][RW][D + 4];      // residual parts of each row: acc[D], m, l
  const float NEG_INF = -__int_as_float(0x7f800000);
  pdl_enter();  // no global reads above this line
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, pair = wib >> 2, role = wib & 3;
  const int row = blockIdx.x * 2 + pair;  // b * Hq + gq
  const bool active = row < n_rows;
  const int Hq = a.Hq, H = a.L.heads, G = Hq / H, S = a.splits;
  const int b = row / Hq, gq = row - b * Hq, h = gq / G;
  float acc[4] = {0.f, 0.f, 0.f, 0.f}, m_run = NEG_INF, l_run = 0.f;
  if (active && role == 0) {  // ---- split partials (natural-log (m, l) per slot)
    const float* ml = a.part_ml + int64_t(row) * a.slots * 2;
    const float* pa = a.part_acc + int64_t(row) * a.slots * D + 4 * lane;
    for (int s0 = 0; s0 < S; s0 += 32) {
      const int s2 = s0 + lane, n = min(32, S - s0);
      float m = NEG_INF, l = 0.f;
      if (s2 < S) {
        m = ml[2 * s2];
        l = ml[2 * s2 + 1];
      }
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = u < n ? *reinterpret_cast<const float4*>(pa + int64_t(s0 + u) * D) : make_float4(0.f, 0.f, 0.f, 0.f);
      float mc = l > 0.f ? m : NEG_INF;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
      const float mn = fmaxf(m_run, mc);
      if (mn == NEG_INF) continue;  // every slot of this chunk (and before) is empty
      const float cf = m_run == NEG_INF ? 0.f : expf(m_run - mn);
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] *= cf;
      l_run *= cf;
      m_run = mn;
      const float w = l > 0.f ? expf(m - mn) : 0.f;
      l_run += w * l;  // lane-partial; reduced below
      for (int j0 = 0; j0 < n; j0 += U) {
        float4 nv[U];
        const bool more = j0 + U < n;
        if (more)
#pragma unroll
          for (int u = 0; u < U; ++u)
            nv[u] = j0 + U + u < n ? *reinterpret_cast<const float4*>(pa + int64_t(s0 + j0 + U + u) * D)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float wu = __shfl_sync(0xffffffffu, w, (j0 + u) & 31);
          acc[0] = fmaf(wu, v[u].x, acc[0]);
          acc[1] = fmaf(wu, v[u].y, acc[1]);
          acc[2] = fmaf(wu, v[u].z, acc[2]);
          acc[3] = fmaf(wu, v[u].w, acc[3]);
        }
        if (more)
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = nv[u];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l_run += __shfl_xor_sync(0xffffffffu, l_run, o);
  }
  if (active && role >= 1) {  // ---- residual rows (raw f32; this step's row read from the input)
    const int rw = role - 1;
    int R, r_new;
    residual_rows(a, b, R, r_new, h);
    auto new_row = [&](const void* src) {  // this lane's 4 columns of the new row of head h, as f32
      float x[4];
      const int64_t off = (int64_t(b) * a.kv_rh + a.kv_h0 + h) * D + 4 * lane;
      if (a.new_dtype == TADA_F32) load4(reinterpret_cast<const float*>(src) + off, x);
      else load4(reinterpret_cast<const __nv_bfloat16*>(src) + off, x);
      return make_float4(x[0], x[1], x[2], x[3]);
    };
    if (r_new >= 0 && gq % G == 0 && rw == 0) {  // one warp per (sequence, KV head) stores the row for later steps
      const int64_t dst = ((int64_t(b) * a.res_seq_stride + r_new) * a.kv_rh + a.kv_h0 + h) * D + 4 * lane;
      *reinterpret_cast<float4*>(const_cast<float*>(a.res_k) + dst) = new_row(a.new_k);
      *reinterpret_cast<float4*>(const_cast<float*>(a.res_v) + dst) = new_row(a.new_v);
      if (!a.step && gq == 0 && lane == 0) const_cast<int32_t*>(a.res_len)[b] = r_new + 1;
    }
    float q[4];
    if (a.q_dtype == TADA_F32) load4(reinterpret_cast<const float*>(a.q) + int64_t(row) * D + 4 * lane, q);
    else load4(reinterpret_cast<const __nv_bfloat16*>(a.q) + int64_t(row) * D + 4 * lane, q);
    const int64_t rbase = int64_t(b) * a.res_seq_stride;
    for (int t0 = U * rw; t0 < R; t0 += U * RW) {
      float4 k4[U], v4[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t0 + u;
        const int64_t o = ((rbase + t) * a.kv_rh + a.kv_h0 + h) * D + 4 * lane;
        k4[u] = t >= R ? make_float4(0.f, 0.f, 0.f, 0.f)
                       : (t == r_new ? new_row(a.new_k) : *reinterpret_cast<const float4*>(a.res_k + o));
        v4[u] = t >= R ? make_float4(0.f, 0.f, 0.f, 0.f)
                       : (t == r_new ? new_row(a.new_v) : *reinterpret_cast<const float4*>(a.res_v + o));
      }
      float sv[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        sv[u] = __fmaf_rn(q[3], k4[u].w, __fmaf_rn(q[2], k4[u].z, __fmaf_rn(q[1], k4[u].y, __fmaf_rn(q[0], k4[u].x, 0.f))));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int u = 0; u < U; ++u) sv[u] += __shfl_xor_sync(0xffffffffu, sv[u], o);
      float bm = NEG_INF;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        sv[u] = t0 + u < R ? __fmul_rn(sv[u], a.scale) : NEG_INF;
        bm = fmaxf(bm, sv[u]);
      }
      const float mn = fmaxf(m_run, bm);  // finite: every batch has a valid row
      const float cf = m_run == NEG_INF ? 0.f : expf(m_run - mn);
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] *= cf;
      l_run *= cf;
      m_run = mn;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float p = t0 + u < R ? expf(sv[u] - mn) : 0.f;
        l_run += p;
        acc[0] = fmaf(p, v4[u].x, acc[0]);
        acc[1] = fmaf(p, v4[u].y, acc[1]);
        acc[2] = fmaf(p, v4[u].z, acc[2]);
        acc[3] = fmaf(p, v4[u].w, acc[3]);
      }
    }
    *reinterpret_cast<float4*>(&rx[pair][rw][4 * lane]) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    if (lane == 0) {
      rx[pair][rw][D] = m_run;  // -inf with l = 0 when this warp had no rows
      rx[pair][rw][D + 1] = l_run;
    }
  }
  __syncthreads();
  if (active && role == 0) {  // ---- merge the parts
    float M = m_run;
#pragma unroll
    for (int w = 0; w < RW; ++w) M = fmaxf(M, rx[pair][w][D]);
    const float fs = m_run == NEG_INF ? 0.f : expf(m_run - M);
    float L = l_run * fs;
    float o[4] = {acc[0] * fs, acc[1] * fs, acc[2] * fs, acc[3] * fs};
#pragma unroll
    for (int w = 0; w < RW; ++w) {
      const float mr = rx[pair][w][D];
      const float fr = mr == NEG_INF ? 0.f : expf(mr - M);
      L += rx[pair][w][D + 1] * fr;
      const float4 ar = *reinterpret_cast<const float4*>(&rx[pair][w][4 * lane]);
      o[0] += ar.x * fr;
      o[1] += ar.y * fr;
      o[2] += ar.z * fr;
      o[3] += ar.w * fr;
    }
    const float inv = 1.f / L;
    const int64_t qi = int64_t(row) * D + 4 * lane;
#pragma unroll
    for (int e = 0; e < 4; ++e) store_any(a.out, a.out_dtype, qi + e, o[e] * inv);
    if (lane == 0 && a.lse_out) a.lse_out[row] = M + logf(L);
  }
  if (a.step && a.step_commit) {  // both rows of this CTA belong to one sequence (Hq is even: a multiple of 8 KV heads)
    __syncthreads();
    if (threadIdx.x == 0 && active) step_commit(a, b, Hq / 2 * (a.commit_units > 1 ? a.commit_units : 1));
  }
}

// K3 for head_dim 128 and G = Hq/H in {1, 2, 4, 8}: one CTA per (sequence, KV head), G + 8 warps.
//  * warps 0..G-1: the split partials of q head h*G + w (natural-log (m, l) per slot), online merge;
//  * warps G..G+7: the residual rows, staged into shared memory by one round of 16-byte cp.async (up to 128
//    rows per chunk), then 8 rows per warp and round with lane = (row, d quarter): each lane forms the 32-d
//    partial dots of its row with all G q rows (broadcast), two shuffles join the quarters, so a K/V row is
//    read once for the whole head group and the dependent FMA chains are 32 long; then lane = 4 d columns
//    for P.V, the weights broadcast by shuffle.  (The lane = row variant with 4 warps ran its 128-long FMA
//    chains on too few warps: 100 rows cost 7 us per layer.)
//  * the parts meet in shared memory; warp w writes q head h*G + w.
// In a fused decode step the new row is read from the input and residual warp 0 stores it.
template <int G>
__global__ void __launch_bounds__((G + 8) * 32) combine_kv_kernel(AttnArgs a, int rch) {
  constexpr int D = 128, RWN = 8, U = 8, RP = D + 4;  // RP: padded staged row (8-row phases hit distinct banks)
  extern __shared__ __align__(16) float rst[];        // staged residual chunk: K rows [rch][RP], then V rows
  __shared__ __align__(16) float qsm[G][D];
  __shared__ __align__(16) float rpart[RWN][G][D];
  __shared__ float rml[RWN][G][2];
  const float NEG_INF = -__int_as_float(0x7f800000);
  pdl_enter();  // no global reads above this line
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = blockIdx.x, b = blockIdx.y, H = a.L.heads, Hq = a.Hq, S = a.splits;
  int R, r_new;
  residual_rows(a, b, R, r_new, h);
  if (warp >= G) {  // the residual warps stage the q rows (named barrier 1: the split warps start at once)
    for (int i = threadIdx.x - G * 32; i < G * D; i += RWN * 32) {
      const int g = i / D, d = i - (i / D) * D;
      const int64_t qi = (int64_t(b) * Hq + h * G + g) * D + d;
      qsm[g][d] = a.q_dtype == TADA_F32 ? reinterpret_cast<const float*>(a.q)[qi]
                                        : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.q)[qi]);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(RWN * 32) : "memory");
  }
  float acc[4] = {0.f, 0.f, 0.f, 0.f}, m_run = NEG_INF, l_run = 0.f;
  if (warp < G) {  // ---- split partials of q head h*G + warp
    const int row = b * Hq + h * G + warp;
    const float* ml = a.part_ml + int64_t(row) * a.slots * 2;
    const float* pa = a.part_acc + int64_t(row) * a.slots * D + 4 * lane;
    for (int s0 = 0; s0 < S; s0 += 32) {
      const int s2 = s0 + lane, n = min(32, S - s0);
      float m = NEG_INF, l = 0.f;
      if (s2 < S) {
        m = ml[2 * s2];
        l = ml[2 * s2 + 1];
      }
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = u < n ? *reinterpret_cast<const float4*>(pa + int64_t(s0 + u) * D) : make_float4(0.f, 0.f, 0.f, 0.f);
      float mc = l > 0.f ? m : NEG_INF;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, o));
      const float mn = fmaxf(m_run, mc);
      if (mn == NEG_INF) continue;
      const float cf = m_run == NEG_INF ? 0.f : expf(m_run - mn);
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] *= cf;
      l_run *= cf;
      m_run = mn;
      const float w = l > 0.f ? expf(m - mn) : 0.f;
      l_run += w * l;
      for (int j0 = 0; j0 < n; j0 += U) {
        float4 nv[U];
        const bool more = j0 + U < n;
        if (more)
#pragma unroll
          for (int u = 0; u < U; ++u)
            nv[u] = j0 + U + u < n ? *reinterpret_cast<const float4*>(pa + int64_t(s0 + j0 + U + u) * D)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float wu = __shfl_sync(0xffffffffu, w, (j0 + u) & 31);
          acc[0] = fmaf(wu, v[u].x, acc[0]);
          acc[1] = fmaf(wu, v[u].y, acc[1]);
          acc[2] = fmaf(wu, v[u].z, acc[2]);
          acc[3] = fmaf(wu, v[u].w, acc[3]);
        }
        if (more)
#pragma unroll
          for (int u = 0; u < U; ++u) v[u] = nv[u];
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l_run += __shfl_xor_sync(0xffffffffu, l_run, o);
  } else {  // ---- residual rows
    const int rw = warp - G;
    const int64_t rbase = int64_t(b) * a.res_seq_stride;
    const int64_t nrow = (int64_t(b) * a.kv_rh + a.kv_h0 + h) * D;  // this head's new row in the step input
    if (r_new >= 0 && rw == 0) {  // store the step's row for later steps
      float x[4];
      const int64_t dst = ((rbase + r_new) * a.kv_rh + a.kv_h0 + h) * D + 4 * lane;
      if (a.new_dtype == TADA_F32) load4(reinterpret_cast<const float*>(a.new_k) + nrow + 4 * lane, x);
      else load4(reinterpret_cast<const __nv_bfloat16*>(a.new_k) + nrow + 4 * lane, x);
      *reinterpret_cast<float4*>(const_cast<float*>(a.res_k) + dst) = make_float4(x[0], x[1], x[2], x[3]);
      if (a.new_dtype == TADA_F32) load4(reinterpret_cast<const float*>(a.new_v) + nrow + 4 * lane, x);
      else load4(reinterpret_cast<const __nv_bfloat16*>(a.new_v) + nrow + 4 * lane, x);
      *reinterpret_cast<float4*>(const_cast<float*>(a.res_v) + dst) = make_float4(x[0], x[1], x[2], x[3]);
      if (!a.step && h == 0 && lane == 0) const_cast<int32_t*>(a.res_len)[b] = r_new + 1;
    }
    float racc[G][4], rm[G], rl[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      racc[g][0] = racc[g][1] = racc[g][2] = racc[g][3] = 0.f;
      rm[g] = NEG_INF;
      rl[g] = 0.f;
    }
    const int tid_r = threadIdx.x - G * 32;  // 0 .. 255 among the residual warps
    for (int cb = 0; cb < R; cb += rch) {   // chunks of rch rows: one round of async copies each
      const int n = min(rch, R - cb);
      if (cb > 0) asm volatile("bar.sync 2, %0;" ::"n"(RWN * 32) : "memory");  // previous chunk consumed
      for (int i = tid_r; i < 2 * n * 32; i += RWN * 32) {
        const int side = i >= n * 32, rem = i - side * n * 32, r = rem >> 5, col = (rem & 31) * 4;
        float* dst = rst + (side * rch + r) * RP + col;
        if (cb + r == r_new) {  // the step's row, from the input (f32 or bf16)
          float x[4];
          const void* src = side ? a.new_v : a.new_k;
          if (a.new_dtype == TADA_F32) load4(reinterpret_cast<const float*>(src) + nrow + col, x);
          else load4(reinterpret_cast<const __nv_bfloat16*>(src) + nrow + col, x);
          *reinterpret_cast<float4*>(dst) = make_float4(x[0], x[1], x[2], x[3]);
        } else {
          const float* src = (side ? a.res_v : a.res_k) + ((rbase + cb + r) * a.kv_rh + a.kv_h0 + h) * D + col;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                       "l"(src)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
      asm volatile("bar.sync 2, %0;" ::"n"(RWN * 32) : "memory");
      // rounds of 8 rows per warp: lane = (row r = lane & 7, d quarter dq = lane >> 3); an 8-lane phase reads 8
      // rows of one quarter (row stride RP = 4 words mod 32: distinct banks), the quarters meet by two shuffles
      const int r8 = lane & 7, dq = lane >> 3;
      for (int c0 = cb + 8 * rw; c0 < cb + n; c0 += 8 * RWN) {
        const int t = c0 + r8;
        const bool valid = t < cb + n;
        float sc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) sc[g] = 0.f;
        if (valid) {  // partial logits of row t over columns 32 dq .. 32 dq + 31
          const float* kr = rst + (t - cb) * RP + 32 * dq;
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 k4 = *reinterpret_cast<const float4*>(kr + j);
#pragma unroll
            for (int g = 0; g < G; ++g) {
              const float4 qv = *reinterpret_cast<const float4*>(&qsm[g][32 * dq + j]);
              sc[g] = __fmaf_rn(qv.w, k4.w, __fmaf_rn(qv.z, k4.z, __fmaf_rn(qv.y, k4.y, __fmaf_rn(qv.x, k4.x, sc[g]))));
            }
          }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          sc[g] += __shfl_xor_sync(0xffffffffu, sc[g], 8);
          sc[g] += __shfl_xor_sync(0xffffffffu, sc[g], 16);
        }
        float p[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float sv = valid ? __fmul_rn(sc[g], a.scale) : NEG_INF;
          float bm = sv;
#pragma unroll
          for (int o = 4; o > 0; o >>= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
          const float mn = fmaxf(rm[g], bm);  // finite: row c0 of every round is valid
          const float cf = rm[g] == NEG_INF ? 0.f : expf(rm[g] - mn);
          racc[g][0] *= cf;
          racc[g][1] *= cf;
          racc[g][2] *= cf;
          racc[g][3] *= cf;
          rl[g] *= cf;
          rm[g] = mn;
          p[g] = valid ? expf(sv - mn) : 0.f;
          if (dq == 0) rl[g] += p[g];  // lane-partial over the quarter-0 lanes; reduced below
        }
        const int nr = min(8, cb + n - c0);
        const float* vr = rst + (rch + (c0 - cb)) * RP + 4 * lane;
        for (int u = 0; u < nr; ++u) {  // P.V: lane = columns 4*lane .. +3, row u's weight from lane u
          const float4 v4 = *reinterpret_cast<const float4*>(vr + u * RP);
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const float pu = __shfl_sync(0xffffffffu, p[g], u);
            racc[g][0] = fmaf(pu, v4.x, racc[g][0]);
            racc[g][1] = fmaf(pu, v4.y, racc[g][1]);
            racc[g][2] = fmaf(pu, v4.z, racc[g][2]);
            racc[g][3] = fmaf(pu, v4.w, racc[g][3]);
          }
        }
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) rl[g] += __shfl_xor_sync(0xffffffffu, rl[g], o);
      *reinterpret_cast<float4*>(&rpart[rw][g][4 * lane]) = make_float4(racc[g][0], racc[g][1], racc[g][2], racc[g][3]);
      if (lane == 0) {
        rml[rw][g][0] = rm[g];  // -inf with l = 0 when this warp had no rows
        rml[rw][g][1] = rl[g];
      }
    }
  }
  __syncthreads();
  if (warp < G) {  // ---- merge the parts of q head h*G + warp
    float M = m_run;
#pragma unroll
    for (int w = 0; w < RWN; ++w) M = fmaxf(M, rml[w][warp][0]);
    const float fs = m_run == NEG_INF ? 0.f : expf(m_run - M);
    float L = l_run * fs;
    float o[4] = {acc[0] * fs, acc[1] * fs, acc[2] * fs, acc[3] * fs};
#pragma unroll
    for (int w = 0; w < RWN; ++w) {
      const float mr = rml[w][warp][0];
      const float fr = mr == NEG_INF ? 0.f : expf(mr - M);
      L += rml[w][warp][1] * fr;
      const float4 ar = *reinterpret_cast<const float4*>(&rpart[w][warp][4 * lane]);
      o[0] += ar.x * fr;
      o[1] += ar.y * fr;
      o[2] += ar.z * fr;
      o[3] += ar.w * fr;
    }
    const float inv = 1.f / L;
    const int row = b * Hq + h * G + warp;
    const int64_t qi = int64_t(row) * D + 4 * lane;
#pragma unroll
    for (int e = 0; e < 4; ++e) store_any(a.out, a.out_dtype, qi + e, o[e] * inv);
    if (lane == 0 && a.lse_out) a.lse_out[row] = M + logf(L);
  }
  if (a.step && a.step_commit) {  // the H CTAs of sequence b: the last one advances its lengths
    __syncthreads();
    if (threadIdx.x == 0) step_commit(a, b, gridDim.x * (a.commit_units > 1 ? a.commit_units : 1));
  }
}

// K3 with residual rows covers this geometry (head_dim % 4 == 0 and, off the D = 128 kernels, the residual
// logits and split weights fit shared memory).
static bool combine_residual_ok(const AttnArgs& a) {
  if (a.L.head_dim % 4) return false;
  if (a.L.head_dim == 128) return true;
  return (size_t(a.L.head_dim) * 3 + size_t(a.res_seq_stride) + size_t(a.splits) + 8) * 4 <= 220 * 1024;
}

static int launch_combine_residual(const AttnArgs& a, int batch, cudaStream_t st) {
  if (a.L.head_dim * 2 > kCombThreads * 2 || a.L.head_dim % 4) return fail(TADA_ERR_CONFIG, "combine needs head_dim % 4 == 0");
  if (a.L.head_dim == 128 && TADA_K3_KV) {  // any residual length: the rows stream through 8 warps per KV head
    const int G = a.Hq / a.L.heads;
    const dim3 grid(a.L.heads, batch);
    // staged residual chunk: up to 128 rows (the default residual_length) of K and V, padded rows
    const int rch = int(a.res_seq_stride < 128 ? (a.res_seq_stride + 31) / 32 * 32 : 128);
    const size_t dsm = size_t(rch > 0 ? rch : 32) * 2 * (128 + 4) * 4;
    cudaError_t e = cudaErrorInvalidValue;
    auto go = [&](auto kern, int warps, std::atomic<uint64_t>& done) {
      if (ensure_smem(kern, 128 * 2 * (128 + 4) * 4, done, "combine_kv") != TADA_OK) return cudaErrorInvalidValue;
      return launch_maybe_pdl(kern, grid, dim3(warps * 32), dsm, st, a, rch > 0 ? rch : 32);
    };
    static std::atomic<uint64_t> d1{0}, d2{0}, d4{0}, d8{0};
    switch (G) {
      case 1: e = go(combine_kv_kernel<1>, 9, d1); break;
      case 2: e = go(combine_kv_kernel<2>, 10, d2); break;
      case 4: e = go(combine_kv_kernel<4>, 12, d4); break;
      case 8: e = go(combine_kv_kernel<8>, 16, d8); break;
      default: break;
    }
    if (G == 1 || G == 2 || G == 4 || G == 8) {
      if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("decode_attn_combine: ") + cudaGetErrorString(e));
      return check_launch("decode_attn_combine_residual");
    }
  }
  if (a.L.head_dim == 128) {  // any residual length: the pair kernel streams the rows
    const int rows = a.Hq * batch;
    const cudaError_t e = launch_maybe_pdl(combine_pair_kernel, dim3((rows + 1) / 2), dim3(256), 0, st, a, rows);
    if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("decode_attn_combine: ") + cudaGetErrorString(e));
    return check_launch("decode_attn_combine_residual");
  }
  const size_t smem = (size_t(a.L.head_dim) * 3 + size_t(a.res_seq_stride) + size_t(a.splits) + 8) * 4;
  if (smem > 220 * 1024) return fail(TADA_ERR_CONFIG, "residual_length too large for the combine kernel");
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(combine_residual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("combine smem: ") + cudaGetErrorString(e));
  }
  combine_residual_kernel<<<dim3(a.Hq, batch), kCombThreads, smem, st>>>(a);
  return check_launch("decode_attn_combine_residual");
}

template <typename QT>
static int launch_generic(const AttnArgs& a, int batch, cudaStream_t st) {
  const int Hq = a.Hq, D = a.L.head_dim;
  const size_t smem = (size_t(2) * Hq * D + size_t(Hq) * kGenTile + 3 * Hq) * 4;
  void (*kern)(AttnArgs) = nullptr;
  switch (a.L.bits) {
    case 2: kern = attn_generic_kernel<QT, 2>; break;
    case 4: kern = attn_generic_kernel<QT, 4>; break;
    case 8: kern = attn_generic_kernel<QT, 8>; break;
    default: kern = attn_generic_kernel<QT, 16>; break;
  }
  if (smem > 48 * 1024) {
    if (smem > 220 * 1024) return fail(TADA_ERR_CONFIG, "num_q_heads*head_dim too large for decode attention");
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("attn smem: ") + cudaGetErrorString(e));
  }
  kern<<<dim3(a.splits, batch), 256, smem, st>>>(a);
  return check_launch("decode_attn_generic");
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TADA_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace tada

namespace tada {

// ---------------------------------------------------------------- group-size and head-count remapping of the
// tensor-core path.  The tensor-core kernels are instantiated for 8 KV heads and q-head groups G in {1, 2, 4, 8}
// (G <= 4 at 8-bit, whose stages leave no room for 64 q heads).
//  * Any other G runs in `passes` passes of up to gc q heads per KV head: pass p takes q heads p*gc .. p*gc + n - 1
//    of every group, zero-padded to gp = 2^ceil(log2 n) rows (a zero query row attends harmlessly and is dropped).
//  * A layout with 16, 24, 32, ... KV heads (e.g. Llama-2's multi-head attention) runs one view per group of 8 KV
//    heads (head_group_view: the code / meta rows are read at an offset with the full row pitch, the residual and
//    step rows likewise through AttnArgs::kv_rh / kv_h0).  Every view re-reads the f32 mean rows, so the bytes
//    moved grow by 512 B per token and side for each extra group.
// Each (head group, pass) stages its q rows, runs K2 + K3 into staging buffers, and puts the output rows back.
constexpr int kMaxUnits = 8;  // concurrent (view, pass) launches (launch_fast_mapped)
tada_page_layout head_group_view(const tada_page_layout& L, int j) {
  tada_page_layout v = L;
  v.heads = 8;
  for (int side = 0; side < 2; ++side) {
    v.off_codes[side] += int64_t(8) * j * L.group_bytes;
    v.off_meta[side] += int64_t(8) * j * 8;
  }
  return v;
}

bool fast_map(const tada_page_layout& L, int Hq, FastMap* m) {
  if (L.heads <= 0 || Hq <= 0 || Hq % L.heads) return false;
  const int G = Hq / L.heads;
  if (fast_supported(L, Hq)) {
    *m = FastMap{1, G, G, G};
    return true;
  }
  if (L.head_dim != 128 || !(L.bits == 2 || L.bits == 4 || L.bits == 8)) return false;
  // multiples of 8 KV heads: one view per 8; fewer than 8: one view whose missing heads read as zeros (TMA: the
  // code rows must be whole 128-byte bands and the meta row pitch a multiple of 16 bytes, so an even head count)
  if (L.heads % 8 && (L.heads > 8 || (int64_t(L.heads) * L.group_bytes) % 128 || L.heads % 2)) return false;
  const tada_page_layout v = head_group_view(L, 0);
  const int gc = L.bits == 8 ? 4 : 8;
  const int n0 = G < gc ? G : gc;
  int gp = 1;
  while (gp < n0) gp *= 2;
  if (!fast_supported(v, 8 * gp)) return false;
  *m = FastMap{(G + gc - 1) / gc, gc, gp, G};
  m->hg = L.heads < 8 ? 1 : L.heads / 8;
  m->view = L.heads != 8;
  return true;
}

// qp[b][h][j] = q[b][hb + h][j0 + j] for j < n (q heads grouped by KV head: row (b * H + hb + h) * G + j0 + j),
// zero otherwise; qp is [B][8][gp]
template <typename T>
__global__ void pad_q_kernel(const T* __restrict__ q, T* __restrict__ qp, int H, int hb, int G, int j0, int n, int gp,
                             int D, int64_t total) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int d = int(i % D);
    const int64_t r = i / D;
    const int j = int(r % gp);
    const int64_t bh = r / gp;  // b * 8 + h
    const int hh = hb + int(bh % 8);  // KV head in the layout; >= H: a view's missing head
    const int64_t src = ((bh / 8) * H + hh) * G + j0 + j;
    qp[i] = (j < n && hh < H) ? q[src * D + d] : T(0.f);
  }
}

template <typename T>
__global__ void unpad_out_kernel(const T* __restrict__ op, const float* __restrict__ lp, T* __restrict__ out,
                                 float* __restrict__ lse, int H, int hb, int G, int j0, int n, int gp, int D,
                                 int64_t total) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int d = int(i % D);
    const int64_t r = i / D;  // (b, h, j) row of the output, j < n
    const int j = int(r % n);
    const int64_t bh = r / n;
    const int hh = hb + int(bh % 8);
    if (hh >= H) continue;  // a view's missing head
    const int64_t src = bh * gp + j, dst = ((bh / 8) * H + hh) * G + j0 + j;
    out[dst * D + d] = op[src * D + d];
    if (lse && d == 0) lse[dst] = lp[src];
  }
}

// Auxiliary streams of the current device for concurrent (view, pass) launches (created once, never freed).
struct AuxStreams {
  cudaStream_t s[kMaxUnits];
  cudaEvent_t fork, join[kMaxUnits];
  bool ok = false;
};
static AuxStreams* aux_streams() {
  static std::mutex mu;
  static AuxStreams per_dev[16];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  AuxStreams& x = per_dev[dev];
  if (!x.ok) {
    bool good = cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; good && i < kMaxUnits; ++i)
      good = cudaStreamCreateWithFlags(&x.s[i], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&x.join[i], cudaEventDisableTiming) == cudaSuccess;
    if (!good) {
      cudaGetLastError();
      return nullptr;
    }
    x.ok = true;
  }
  return &x;
}

int launch_fast_mapped(const AttnArgs& a0, int batch, const FastMap& fm, int mode, void* workspace, cudaStream_t st) {
  const int D = a0.L.head_dim, hq = 8 * fm.gp, H = a0.L.heads;
  const int64_t rows = int64_t(batch) * hq;
  const bool qbf = a0.q_dtype == TADA_BF16, obf = a0.out_dtype == TADA_BF16;
  auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  // one (view, pass) unit: pad its q rows, K2 + K3 into its staging buffers, put its output rows back
  auto run_unit = [&](int jg, int p, uint8_t* ws, int splits, int commit_units, bool commit,
                      cudaStream_t s) {
    const int j0 = p * fm.gc, n = fm.g - j0 < fm.gc ? fm.g - j0 : fm.gc, hb = 8 * jg;
    const int64_t part_bytes = rows * splits * (int64_t(D) + 2) * 4;
    void* qp = ws + al(part_bytes);
    void* op = reinterpret_cast<uint8_t*>(qp) + rows * D * 4;
    float* lp = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(op) + rows * D * 4);
    AttnArgs a = a0;
    if (fm.view) {
      a.L = head_group_view(a0.L, jg);
      a.kv_rh = H;
      a.kv_h0 = hb;
    }
    a.Hq = hq;
    a.q = qp;
    a.out = op;
    a.splits = a.slots = splits;
    a.step_commit = commit;
    a.commit_units = commit_units;
    a.lse_out = a0.lse_out ? lp : nullptr;
    a.part_acc = reinterpret_cast<float*>(ws);
    a.part_ml = a.part_acc + rows * a.slots * D;
    int rc = TADA_OK;
    {
      const int64_t tq = rows * D;
      const int grid = int((tq + 255) / 256 < 148 * 16 ? (tq + 255) / 256 : 148 * 16);
      if (qbf)
        pad_q_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(a0.q),
                                          reinterpret_cast<__nv_bfloat16*>(qp), H, hb, fm.g, j0, n, fm.gp, D, tq);
      else
        pad_q_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const float*>(a0.q), reinterpret_cast<float*>(qp), H, hb,
                                          fm.g, j0, n, fm.gp, D, tq);
      rc = check_launch("decode_attn_pad_q");
      if (rc != TADA_OK) return rc;
    }
    rc = (mode != 3 && v8_supported(a.L, hq)) ? launch_v8(a, batch, s) : launch_fast(a, batch, s);
    if (rc == TADA_OK) rc = launch_combine_residual(a, batch, s);
    if (rc != TADA_OK) return rc;
    {
      const int64_t to = int64_t(batch) * 8 * n * D;
      const int g2 = int((to + 255) / 256 < 148 * 16 ? (to + 255) / 256 : 148 * 16);
      if (obf)
        unpad_out_kernel<<<g2, 256, 0, s>>>(reinterpret_cast<const __nv_bfloat16*>(op), lp,
                                            reinterpret_cast<__nv_bfloat16*>(a0.out), a0.lse_out, H, hb, fm.g, j0, n,
                                            fm.gp, D, to);
      else
        unpad_out_kernel<<<g2, 256, 0, s>>>(reinterpret_cast<const float*>(op), lp, reinterpret_cast<float*>(a0.out),
                                            a0.lse_out, H, hb, fm.g, j0, n, fm.gp, D, to);
      rc = check_launch("decode_attn_unpad");
    }
    return rc;
  };
  const int units = fm.hg * fm.passes;
  // Concurrent units: every (view, pass) re-reads the f32 mean rows (views) or the whole tile (q-head passes),
  // and each unit's K3, q padding and output copy leave the GPU partly idle between K2s.  The units run on
  // auxiliary streams, so one unit's K2 overlaps the previous one's tail and K3, and units reading the same
  // token ranges at nearly the same time share bytes through L2.  Measured (tools/attn_bench.py, mode 0):
  // two units with half the splits each, MHA 16 KV heads 4-bit 4015 -> 4543 GB/s, 8-bit 4412 -> 4846;
  // more units keep the full split count (divided, their start skew left one unit running alone at the end:
  // 32 KV heads B=16 3728 -> 2180; undivided 3937, and 2708 -> 3281 at B=4).  Needs the units' buffers to
  // fit the documented workspace and the auxiliary streams to exist before a graph capture.
  static const int conc_env = getenv("TADA_MAPPED_CONCURRENT") ? atoi(getenv("TADA_MAPPED_CONCURRENT")) : 1;
  const int splits_u = units == 2 ? a0.splits / 2 : a0.splits;
  const int64_t unit_bytes = al(rows * splits_u * (int64_t(D) + 2) * 4) + 2 * rows * D * 4 + al(rows * 4);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  static std::atomic<bool> made{false};
  AuxStreams* aux = nullptr;
  if (conc_env && units > 1 && units <= kMaxUnits && splits_u >= 1 &&
      units * unit_bytes <= tada_decode_attn_workspace_bytes(batch, a0.Hq, D, a0.splits) &&
      (cap == cudaStreamCaptureStatusNone || made.load())) {
    aux = aux_streams();
    if (aux) made.store(true);
  }
  uint8_t* ws = reinterpret_cast<uint8_t*>(workspace);
  if (!aux) {  // one unit after another on the caller's stream; only the last one advances a step's lengths
    for (int jg = 0; jg < fm.hg; ++jg)
      for (int p = 0; p < fm.passes; ++p) {
        const int rc = run_unit(jg, p, ws, a0.splits, 1, jg == fm.hg - 1 && p == fm.passes - 1, st);
        if (rc != TADA_OK) return rc;
      }
    return TADA_OK;
  }
  // the fork / join events and streams are shared by every caller on this device: issue under a lock so that
  // two host threads cannot interleave their records and waits
  static std::mutex issue_mu;
  std::lock_guard<std::mutex> lock(issue_mu);
  if (cudaEventRecord(aux->fork, st) != cudaSuccess) return fail(TADA_ERR_CUDA, "decode_attn: fork event");
  for (int u = 0; u < units; ++u) {
    if (cudaStreamWaitEvent(aux->s[u], aux->fork, 0) != cudaSuccess) return fail(TADA_ERR_CUDA, "decode_attn: fork");
    // every unit's K3 counts towards the step's arrivals: the last CTA of all units advances the lengths
    const int rc = run_unit(u / fm.passes, u % fm.passes, ws + u * unit_bytes, splits_u, units, true, aux->s[u]);
    if (rc != TADA_OK) return rc;
    if (cudaEventRecord(aux->join[u], aux->s[u]) != cudaSuccess || cudaStreamWaitEvent(st, aux->join[u], 0) != cudaSuccess)
      return fail(TADA_ERR_CUDA, "decode_attn: join");
  }
  return TADA_OK;
}

}  // namespace tada

using namespace tada;

extern "C" {

int64_t tada_decode_attn_workspace_bytes(int32_t batch, int32_t num_q_heads, int32_t head_dim, int32_t num_splits) {
  // slots = splits + 1 (the tensor-core path puts the residual rows in an extra slot); a remapped layout or
  // group size (FastMap) runs views of 8 KV heads x gp <= 8 padded q heads, i.e. <= 64 q rows per sequence, and
  // stages their q, outputs and lse here too
  const int64_t rows = int64_t(batch) * (num_q_heads > 64 ? num_q_heads : 64);
  return rows * (num_splits + 1) * (int64_t(head_dim) + 2) * 4 + int64_t(batch) * 64 * (2 * int64_t(head_dim) + 1) * 4 +
         256;
}

// Split count for `slots` concurrently resident CTAs: the fewest whole waves whose last wave is
// >= 90% full, keeping >= 256 tokens per split (fewer, longer splits amortise the per-CTA q setup).
static int32_t plan_splits(int64_t slots, int32_t batch, int64_t max_tokens, bool short_ok = false) {
  if (batch <= 0 || max_tokens <= 0) return 1;
  // >= 256 tokens per split amortise the per-CTA q setup; for the exact kernel (short_ok), when that leaves SMs
  // idle (small batches, short caches), splits go down to 64 tokens (the tensor-core path's K3 merges the
  // splits of a head on one CTA, so more splits cost it more than they gain at small batches)
  int64_t max_s = (max_tokens + 255) / 256;
  if (short_ok && max_s * batch < slots) max_s = (max_tokens + 63) / 64;
  int64_t best = 1;
  for (int64_t waves = 1; waves <= 8; ++waves) {
    const int64_t s = waves * slots / batch;
    if (s < 1) continue;
    const int64_t ctas = s * batch;
    const int64_t used = (ctas + slots - 1) / slots * slots;
    best = s;
    if (ctas * 10 >= used * 9) break;
  }
  if (best > max_s) best = max_s;
  return int32_t(best < 1 ? 1 : best);
}

int32_t tada_decode_attn_suggest_splits(int32_t batch, int64_t max_tokens, int32_t page_tokens) {
  (void)page_tokens;
  return plan_splits(148, batch, max_tokens);
}

int32_t tada_decode_attn_plan_splits_mode(const tada_page_layout* layout, int32_t num_q_heads, int32_t batch,
                                          int64_t max_tokens, int32_t mode) {
  if (!layout || num_q_heads <= 0) return 1;
  int per_sm = 1;
  FastMap fm;
  const bool mapped = mode != 1 && fast_map(*layout, num_q_heads, &fm);  // else the exact kernels run
  const int hq = mapped ? 8 * fm.gp : num_q_heads;  // the instantiation that runs
  const tada_page_layout lv = mapped && fm.view ? head_group_view(*layout, 0) : *layout;
  if (mapped && v8_supported(lv, hq)) per_sm = 2;  // attn_v8_kernel: two CTAs per SM
  else if (mapped && fast_supported(lv, hq)) per_sm = fast_tile_tokens(lv, hq) == 16 ? 2 : 1;
  else per_sm = exact_ctas_per_sm(*layout, num_q_heads);
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return plan_splits(int64_t(sms) * per_sm, batch, max_tokens, !mapped);
}

int32_t tada_decode_attn_plan_splits(const tada_page_layout* layout, int32_t num_q_heads, int32_t batch,
                                     int64_t max_tokens) {
  return tada_decode_attn_plan_splits_mode(layout, num_q_heads, batch, max_tokens, 0);
}

static int decode_attn_impl(const tada_page_layout* layout, const uint8_t* pool, const void* q, int32_t q_dtype,
                            int32_t batch, int32_t num_q_heads, const int32_t* page_table, int32_t pt_stride,
                            const int32_t* comp_len, const int32_t* res_len, const float* res_k, const float* res_v,
                            int64_t res_seq_stride, float scale, int32_t num_splits, void* workspace, void* out,
                            int32_t out_dtype, int32_t mode, float* lse_out, void* stream,
                            const void* new_k = nullptr, const void* new_v = nullptr, int32_t new_dtype = 0,
                            int32_t step_R = -1, int32_t* step_sync = nullptr, const int32_t* range_word = nullptr) {
  if (!layout) return fail(TADA_ERR_CONFIG, "null layout");
  if (q_dtype != TADA_F32 && q_dtype != TADA_BF16) return fail(TADA_ERR_CONFIG, "q dtype must be f32 or bf16");
  if (out_dtype != TADA_F32 && out_dtype != TADA_BF16) return fail(TADA_ERR_CONFIG, "out dtype must be f32 or bf16");
  if (batch < 0 || num_q_heads <= 0 || num_q_heads % layout->heads != 0)
    return fail(TADA_ERR_CONFIG, "num_q_heads must be a positive multiple of num_kv_heads");
  if (num_splits < 1 || num_splits > 4096) return fail(TADA_ERR_CONFIG, "num_splits out of range");
  if (batch == 0) return TADA_OK;
  if (!q || !out || !comp_len || !res_len) return fail(TADA_ERR_SHAPE, "null buffer");
  if (mode < 0 || mode > 3)
    return fail(TADA_ERR_CONFIG, "mode must be 0 (auto), 1 (exact), 2 (fast) or 3 (fast, two-barrier kernel)");
  FastMap fm{};
  const bool mapped = fast_map(*layout, num_q_heads, &fm);
  const bool fast = mode >= 2 || (mode == 0 && mapped);
  if (mode >= 2 && !mapped)
    return fail(TADA_ERR_CONFIG, "fast decode attention needs a multiple of 8 KV heads, head_dim 128, bits 2/4/8 and page_tokens % 32 == 0");
  if (!workspace && (num_splits > 1 || fast || exact_smem_bytes(*layout, num_q_heads)))
    return fail(TADA_ERR_SHAPE, "workspace required");
  AttnArgs a{};
  a.L = *layout;
  a.pool = pool;
  a.q = q;
  a.Hq = num_q_heads;
  a.page_table = page_table;
  a.pt_stride = pt_stride;
  a.comp_len = comp_len;
  a.res_len = res_len;
  a.res_k = res_k;
  a.res_v = res_v;
  a.res_seq_stride = res_seq_stride;
  a.scale = scale;
  a.splits = num_splits;
  a.slots = num_splits;
  a.part_acc = reinterpret_cast<float*>(workspace);
  a.part_ml = a.part_acc + int64_t(batch) * num_q_heads * a.slots * layout->head_dim;
  a.out = out;
  a.out_dtype = out_dtype;
  a.q_dtype = q_dtype;
  a.lse_out = lse_out;
  a.new_k = new_k;
  a.new_v = new_v;
  a.new_dtype = new_dtype;
  a.step = step_R >= 0;
  a.step_R = step_R;
  a.step_sync = step_sync;
  a.range = range_word;
  a.kv_rh = layout->heads;
  a.kv_h0 = 0;
  a.step_commit = true;
  {
    static const int diag = getenv("TADA_ATTN_DIAG") ? atoi(getenv("TADA_ATTN_DIAG")) : 0;
    a.diag = diag;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int rc;
  if (fast && !fm.direct()) return launch_fast_mapped(a, batch, fm, mode, workspace, st);
  if (fast) {
    rc = (mode != 3 && v8_supported(*layout, num_q_heads)) ? launch_v8(a, batch, st) : launch_fast(a, batch, st);
    if (rc == TADA_OK && a.diag != 3) rc = launch_combine_residual(a, batch, st);  // diag 3: K2 alone (timing only)
    return rc;
  } else if (exact_smem_bytes(*layout, num_q_heads) && combine_residual_ok(a)) {
    rc = launch_exact(a, batch, st);  // staged f32 kernel over the compressed tokens; K3 the residual + merge
    if (rc == TADA_OK) rc = launch_combine_residual(a, batch, st);
    return rc;
  } else {
    rc = q_dtype == TADA_F32 ? launch_generic<float>(a, batch, st) : launch_generic<__nv_bfloat16>(a, batch, st);
    if (rc != TADA_OK || num_splits == 1) return rc;
  }
  if (rc != TADA_OK) return rc;
  combine_kernel<<<unsigned(int64_t(batch) * num_q_heads), 128, 0, st>>>(a.part_acc, a.part_ml, a.slots,
                                                                          layout->head_dim, out, out_dtype, a.lse_out);
  return check_launch("decode_attn_combine");
}

int tada_decode_attn(const tada_page_layout* layout, const uint8_t* pool, const void* q, int32_t q_dtype, int32_t batch,
                     int32_t num_q_heads, const int32_t* page_table, int32_t pt_stride, const int32_t* comp_len,
                     const int32_t* res_len, const float* res_k, const float* res_v, int64_t res_seq_stride,
                     float scale, int32_t num_splits, void* workspace, void* out, int32_t out_dtype, int32_t mode,
                     const int32_t* range_word, void* stream) {
  return decode_attn_impl(layout, pool, q, q_dtype, batch, num_q_heads, page_table, pt_stride, comp_len, res_len, res_k,
                          res_v, res_seq_stride, scale, num_splits, workspace, out, out_dtype, mode, nullptr, stream,
                          nullptr, nullptr, 0, -1, nullptr, range_word);
}

int tada_decode_attn_lse(const tada_page_layout* layout, const uint8_t* pool, const void* q, int32_t q_dtype,
                         int32_t batch, int32_t num_q_heads, const int32_t* page_table, int32_t pt_stride,
                         const int32_t* comp_len, const int32_t* res_len, const float* res_k, const float* res_v,
                         int64_t res_seq_stride, float scale, int32_t num_splits, void* workspace, void* out,
                         int32_t out_dtype, int32_t mode, float* lse_out, const int32_t* range_word, void* stream) {
  if (!lse_out) return fail(TADA_ERR_SHAPE, "null lse buffer");
  return decode_attn_impl(layout, pool, q, q_dtype, batch, num_q_heads, page_table, pt_stride, comp_len, res_len, res_k,
                          res_v, res_seq_stride, scale, num_splits, workspace, out, out_dtype, mode, lse_out, stream,
                          nullptr, nullptr, 0, -1, nullptr, range_word);
}

int tada_decode_step(const tada_page_layout* layout, uint8_t* pool, const void* q, int32_t q_dtype, int32_t batch,
                     int32_t num_q_heads, const int32_t* page_table, int32_t pt_stride, int32_t* comp_len,
                     int32_t* res_len, float* res_k, float* res_v, int64_t res_seq_stride, int32_t residual_length,
                     const void* new_k, const void* new_v, int32_t new_dtype, int32_t k1_rows, int32_t* step_sync,
                     float scale, int32_t num_splits, void* workspace, void* out, int32_t out_dtype, int32_t mode,
                     int32_t* err_flag, int32_t* range_word, void* stream) {
  if (!layout) return fail(TADA_ERR_CONFIG, "null layout");
  FastMap fm;
  if (mode == 1 || !fast_map(*layout, num_q_heads, &fm) || layout->head_dim != 128)
    return fail(TADA_ERR_CONFIG, "the fused decode step needs the tensor-core attention path (head_dim 128)");
  if (!new_k || !new_v || !res_k || !res_v || !step_sync || !comp_len || !res_len) return fail(TADA_ERR_SHAPE, "null buffer");
  if (new_dtype != TADA_F32 && new_dtype != TADA_BF16) return fail(TADA_ERR_CONFIG, "new row dtype must be f32 or bf16");
  if (residual_length < 0 || (residual_length > 0 && residual_length > res_seq_stride) ||
      k1_rows > (residual_length > 0 ? residual_length - 1 : 0))
    return fail(TADA_ERR_CONFIG, "residual buffer / flush rows out of range");
  if (batch == 0) return TADA_OK;
  // K1 for the sequences whose residual fills this step (each decides on the device): its residual rows,
  // then the new row; k1_rows < 0 means the caller knows no sequence compresses a token this step
  if (k1_rows > 0) {
    const int rc = tada_quant_append_plan(layout, pool, res_k, res_v, TADA_F32, batch, k1_rows, res_seq_stride,
                                          page_table, pt_stride, comp_len, res_len, residual_length, 1, nullptr, 1,
                                          nullptr, 0, nullptr, 0, err_flag, range_word, stream);
    if (rc != TADA_OK) return rc;
  }
  if (k1_rows >= 0) {
    const int rc = tada_quant_append_plan(layout, pool, new_k, new_v, new_dtype, batch, 1, 1, page_table, pt_stride,
                                          comp_len, res_len, residual_length, 1, nullptr, 2, nullptr, 0, nullptr, 0,
                                          err_flag, range_word, stream);
    if (rc != TADA_OK) return rc;
  }
  return decode_attn_impl(layout, pool, q, q_dtype, batch, num_q_heads, page_table, pt_stride, comp_len, res_len, res_k,
                          res_v, res_seq_stride, scale, num_splits, workspace, out, out_dtype, mode == 0 ? 2 : mode,
                          nullptr, stream, new_k, new_v, new_dtype, residual_length, step_sync, range_word);
}

int tada_combine_lse(const float* o_parts, const float* lse_parts, int32_t n_parts, int64_t rows, int32_t head_dim,
                     void* out, int32_t out_dtype, float* lse_out, void* stream) {
  if (n_parts < 1 || rows < 0 || head_dim <= 0) return fail(TADA_ERR_CONFIG, "bad combine geometry");
  if (out_dtype != TADA_F32 && out_dtype != TADA_BF16) return fail(TADA_ERR_CONFIG, "out dtype must be f32 or bf16");
  if (rows == 0) return TADA_OK;
  if (!o_parts || !lse_parts || !out) return fail(TADA_ERR_SHAPE, "null buffer");
  combine_lse_kernel<<<unsigned(rows), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      o_parts, lse_parts, n_parts, rows, head_dim, out, out_dtype, lse_out);
  return check_launch("combine_lse");
}

}  // extern "C"
