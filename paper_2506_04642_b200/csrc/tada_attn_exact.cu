// K2-exact: split-K decode attention over the compressed paged cache in f32 on the CUDA cores, for ANY
// geometry the reference accepts (heads, q heads, head_dim, widths 2/4/8/16) — the kernel behind
// attend_streaming / attend_naive (attention.py:66-151) and mode 1.
//
// Arithmetic: K̂ = mean - fmaf(code, scale, min), bit-identical to the reference's reconstruct_slice
// (cache.py:190-213, quant.py:177-180; width 16: mean - raw deviation); logits = f32 dot * F32(1/sqrt(D))
// (attention.py:118-136); online softmax and P·V̂ in f32.  Only the summation order differs from numpy's
// sgemv, so outputs sit within the reference's own streaming-vs-naive bar (1e-5, test_acceptance.py:150-178).
//
// CTA = (split, sequence), 8 warps.  Per 32-token tile the CTA stages both sides' mean rows (padded to
// D + 1 floats), the code rows of all heads and the (scale, min) metas into shared memory with coalesced
// loads (the f32 mean row is shared by every head: read once per tile).  Warp w then takes KV heads
// w, w + 8, ...; for each, up to four of its q heads at a time:
//   phase 1, lane = token: the lane dequantises its token's K̂ row once and forms the dots with the q rows
//            (broadcast from shared memory), then a warp-wide online-softmax update;
//   phase 2, lane = column: V̂ entries dequantised once per (token, column) and accumulated for the q heads
//            with the tile's weights (broadcast from shared memory).
// The running (max, sum, output) rows of each q head live in shared memory, owned by one warp.  The residual
// rows and the split merge are K3's (tada_attn.cu), exactly as for the tensor-core kernels.
#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "tada_attn.cuh"
#include "tada_attn_exact2.cuh"

namespace tada {
namespace exact {

constexpr int TT = 32, NW = 8, NTHR = 256, GC = 4;  // tokens per tile (lane = token), warps, q heads per pass
constexpr int kMaxSmem = 200 * 1024;

struct Plan {
  int mrow;  // floats per staged mean row
  int crow;  // bytes per staged code row (all heads of one token)
  int off_km, off_vm, off_kc, off_vc, off_kmeta, off_vmeta, off_q, off_acc, off_ml, off_p, off_pg, off_row, total;
};

inline Plan make_plan(int H, int D, int gb, int Hq) {
  Plan p{};
  p.mrow = D + 1;  // lane-per-token reads of column d hit 32 distinct banks
  p.crow = (H * gb + 3) / 4 * 4 + 4;
  int off = 0;
  auto take = [&](int bytes) {
    const int o = off;
    off = (off + bytes + 15) / 16 * 16;
    return o;
  };
  p.off_km = take(TT * p.mrow * 4);
  p.off_vm = take(TT * p.mrow * 4);
  p.off_kc = take(TT * p.crow);
  p.off_vc = take(TT * p.crow);
  p.off_kmeta = take(TT * H * 8);
  p.off_vmeta = take(TT * H * 8);
  p.off_q = take(Hq * D * 4);
  p.off_acc = take(Hq * D * 4);
  p.off_ml = take(Hq * 2 * 4);
  p.off_p = take(NW * GC * TT * 4);
  p.off_pg = take(TT * 8);
  p.off_row = take(TT * 4);
  p.total = off;
  return p;
}

template <int BITS>
__device__ __forceinline__ float dequant_dev(const uint8_t* grp, int d, float2 sm) {
  if (BITS == 16) return reinterpret_cast<const float*>(grp)[d];
  return __fmaf_rn(float(get_code(grp, d, BITS)), sm.x, sm.y);
}

template <int BITS, typename QT>
__global__ void __launch_bounds__(NTHR) attn_exact_kernel(AttnArgs a, Plan pl) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int H = a.L.heads, D = a.L.head_dim, Hq = a.Hq, G = Hq / H, P = a.L.page_tokens, gb = a.L.group_bytes;
  const int cb = H * gb;
  const int b = blockIdx.y, split = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* km = reinterpret_cast<float*>(smem + pl.off_km);
  float* vm = reinterpret_cast<float*>(smem + pl.off_vm);
  uint8_t* kc = smem + pl.off_kc;
  uint8_t* vc = smem + pl.off_vc;
  float2* kmeta = reinterpret_cast<float2*>(smem + pl.off_kmeta);
  float2* vmeta = reinterpret_cast<float2*>(smem + pl.off_vmeta);
  float* qs = reinterpret_cast<float*>(smem + pl.off_q);
  float* acc = reinterpret_cast<float*>(smem + pl.off_acc);
  float* ml = reinterpret_cast<float*>(smem + pl.off_ml);
  float* pbuf = reinterpret_cast<float*>(smem + pl.off_p) + warp * GC * TT;
  const uint8_t** pg = reinterpret_cast<const uint8_t**>(smem + pl.off_pg);
  int* prow = reinterpret_cast<int*>(smem + pl.off_row);
  const float NEG_INF = -__int_as_float(0x7f800000);

  pdl_enter();  // no global reads above this line
  const int C = comp_tokens(a, b);
  int t_begin, t_end;
  split_range(C, a.splits, split, TT, t_begin, t_end);
  const QT* q = reinterpret_cast<const QT*>(a.q) + int64_t(b) * Hq * D;
  for (int i = tid; i < Hq * D; i += NTHR) {
    qs[i] = to_f32(q[i]);
    acc[i] = 0.f;
  }
  for (int g = tid; g < Hq; g += NTHR) {
    ml[2 * g] = NEG_INF;
    ml[2 * g + 1] = 0.f;
  }
  const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
  const bool words = (cb & 3) == 0;

  for (int t0 = t_begin; t0 < t_end; t0 += TT) {
    const int nv = min(TT, t_end - t0);
    __syncthreads();  // the previous tile is consumed (first tile: q / acc / ml initialised)
    if (tid < nv) {
      const int t = t0 + tid;
      pg[tid] = a.pool + int64_t(pt[t / P]) * a.L.page_bytes;
      prow[tid] = t % P;
    }
    __syncthreads();
    // ---- stage the tile: mean rows, code rows of all heads, metas (coalesced global reads)
    for (int i = tid; i < nv * D; i += NTHR) {
      const int t = i / D, d = i - t * D;
      const uint8_t* page = pg[t];
      const int64_t e = int64_t(prow[t]) * D + d;
      km[t * pl.mrow + d] = reinterpret_cast<const float*>(page + a.L.off_mean[0])[e];
      vm[t * pl.mrow + d] = reinterpret_cast<const float*>(page + a.L.off_mean[1])[e];
    }
    if (words) {
      const int cw = cb >> 2;
      for (int i = tid; i < nv * cw; i += NTHR) {
        const int t = i / cw, w = i - t * cw;
        const uint8_t* page = pg[t];
        const int64_t e = int64_t(prow[t]) * cw + w;
        reinterpret_cast<uint32_t*>(kc + t * pl.crow)[w] = reinterpret_cast<const uint32_t*>(page + a.L.off_codes[0])[e];
        reinterpret_cast<uint32_t*>(vc + t * pl.crow)[w] = reinterpret_cast<const uint32_t*>(page + a.L.off_codes[1])[e];
      }
    } else {
      for (int i = tid; i < nv * cb; i += NTHR) {
        const int t = i / cb, w = i - t * cb;
        const uint8_t* page = pg[t];
        const int64_t e = int64_t(prow[t]) * cb + w;
        kc[t * pl.crow + w] = page[a.L.off_codes[0] + e];
        vc[t * pl.crow + w] = page[a.L.off_codes[1] + e];
      }
    }
    for (int i = tid; i < nv * H; i += NTHR) {
      const int t = i / H, h = i - t * H;
      const uint8_t* page = pg[t];
      const int64_t e = int64_t(prow[t]) * H + h;
      kmeta[i] = reinterpret_cast<const float2*>(page + a.L.off_meta[0])[e];
      vmeta[i] = reinterpret_cast<const float2*>(page + a.L.off_meta[1])[e];
    }
    __syncthreads();

    for (int h = warp; h < H; h += NW) {
      for (int g0 = 0; g0 < G; g0 += GC) {
        const int gn = min(GC, G - g0);
        const int row0 = h * G + g0;
        // ---- phase 1 (lane = token): K̂ row once, dots with up to GC q rows
        float z[GC] = {0.f, 0.f, 0.f, 0.f};
        if (lane < nv) {
          const float* kr = km + lane * pl.mrow;
          const uint8_t* grp = kc + lane * pl.crow + h * gb;
          const float2 sm = kmeta[lane * H + h];
          for (int d = 0; d < D; ++d) {
            const float kh = __fsub_rn(kr[d], dequant_dev<BITS>(grp, d, sm));
#pragma unroll
            for (int gg = 0; gg < GC; ++gg)
              if (gg < gn) z[gg] = __fmaf_rn(qs[(row0 + gg) * D + d], kh, z[gg]);
          }
        }
        // ---- online softmax over the tile (natural-log units, attention.py:139-147)
        float corr[GC];
#pragma unroll
        for (int gg = 0; gg < GC; ++gg) {
          corr[gg] = 1.f;
          if (gg < gn) {
            const float zz = lane < nv ? __fmul_rn(z[gg], a.scale) : NEG_INF;
            const float m_old = ml[2 * (row0 + gg)];
            const float m_new = fmaxf(m_old, warp_max(zz));
            corr[gg] = expf(m_old - m_new);
            const float p = lane < nv ? expf(zz - m_new) : 0.f;
            const float lsum = warp_sum(p);
            pbuf[gg * TT + lane] = p;
            if (lane == 0) {
              ml[2 * (row0 + gg)] = m_new;
              ml[2 * (row0 + gg) + 1] = ml[2 * (row0 + gg) + 1] * corr[gg] + lsum;
            }
          }
        }
        __syncwarp();
        // ---- phase 2 (lane = column): V̂ entries once per (token, column), weights broadcast
        for (int d = lane; d < D; d += 32) {
          float ac[GC];
#pragma unroll
          for (int gg = 0; gg < GC; ++gg) ac[gg] = gg < gn ? acc[(row0 + gg) * D + d] * corr[gg] : 0.f;
          for (int t = 0; t < nv; ++t) {
            const float vh = __fsub_rn(vm[t * pl.mrow + d], dequant_dev<BITS>(vc + t * pl.crow + h * gb, d, vmeta[t * H + h]));
#pragma unroll
            for (int gg = 0; gg < GC; ++gg) ac[gg] = __fmaf_rn(pbuf[gg * TT + t], vh, ac[gg]);
          }
#pragma unroll
          for (int gg = 0; gg < GC; ++gg)
            if (gg < gn) acc[(row0 + gg) * D + d] = ac[gg];
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < Hq * D; i += NTHR) {
    const int g = i / D, d = i - g * D;
    const int64_t slot = (int64_t(b) * Hq + g) * a.slots + split;
    a.part_acc[slot * D + d] = acc[i];
    if (d == 0) {
      const float l = ml[2 * g + 1];
      a.part_ml[slot * 2] = l > 0.f ? ml[2 * g] : NEG_INF;
      a.part_ml[slot * 2 + 1] = l;
    }
  }
}

}  // namespace exact

namespace exact2 {
template <int BITS>
static int launch_b(const AttnArgs& a, int batch, const Plan& pl, cudaStream_t st) {
  return a.L.head_dim == 128 ? launch_g<BITS, 128>(a, batch, pl, st) : exact2_launch_other_d(a, batch, pl, st);
}
static int launch(const AttnArgs& a, int batch, const Plan& pl, cudaStream_t st) {
  switch (a.L.bits) {
    case 2: return launch_b<2>(a, batch, pl, st);
    case 4: return launch_b<4>(a, batch, pl, st);
    case 8: return launch_b<8>(a, batch, pl, st);
    default: return launch_b<16>(a, batch, pl, st);
  }
}
}  // namespace exact2

int exact_smem_bytes(const tada_page_layout& L, int Hq) {
  exact2::Plan p2;
  if (exact2::plan(L, Hq, &p2)) return p2.total;
  const exact::Plan p = exact::make_plan(L.heads, L.head_dim, L.group_bytes, Hq);
  return p.total <= exact::kMaxSmem && L.head_dim % 4 == 0 ? p.total : 0;
}

int exact_ctas_per_sm(const tada_page_layout& L, int Hq) {
  exact2::Plan p2;
  if (exact2::plan(L, Hq, &p2)) return (227 * 1024) / (p2.total + 1024) >= 2 ? 2 : 1;
  const int bytes = exact_smem_bytes(L, Hq);
  if (!bytes) return 1;
  const int by_smem = (227 * 1024) / (bytes + 1024);
  return by_smem < 1 ? 1 : (by_smem > 8 ? 8 : by_smem);
}

template <int BITS, typename QT>
static int launch_exact_t(const AttnArgs& a, int batch, const exact::Plan& pl, cudaStream_t st) {
  auto kern = exact::attn_exact_kernel<BITS, QT>;
  static std::atomic<uint64_t> done{0};
  if (const int rc = ensure_smem(kern, exact::kMaxSmem, done, "attn_exact"); rc != TADA_OK) return rc;
  const cudaError_t e = launch_maybe_pdl(kern, dim3(a.splits, batch), dim3(exact::NTHR), size_t(pl.total), st, a, pl);
  if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("decode_attn_exact: ") + cudaGetErrorString(e));
  return check_launch("decode_attn_exact");
}

template <typename QT>
static int launch_exact_q(const AttnArgs& a, int batch, const exact::Plan& pl, cudaStream_t st) {
  switch (a.L.bits) {
    case 2: return launch_exact_t<2, QT>(a, batch, pl, st);
    case 4: return launch_exact_t<4, QT>(a, batch, pl, st);
    case 8: return launch_exact_t<8, QT>(a, batch, pl, st);
    default: return launch_exact_t<16, QT>(a, batch, pl, st);
  }
}

int launch_exact(const AttnArgs& a, int batch, cudaStream_t st) {
  exact2::Plan p2;
  static const bool v1 = getenv("TADA_EXACT_V1") != nullptr;  // A/B: the previous staged kernel
  if (!v1 && exact2::plan(a.L, a.Hq, &p2)) return exact2::launch(a, batch, p2, st);
  if (!exact_smem_bytes(a.L, a.Hq)) return fail(TADA_ERR_CONFIG, "geometry too large for the staged exact kernel");
  const exact::Plan pl = exact::make_plan(a.L.heads, a.L.head_dim, a.L.group_bytes, a.Hq);
  return a.q_dtype == TADA_F32 ? launch_exact_q<float>(a, batch, pl, st) : launch_exact_q<__nv_bfloat16>(a, batch, pl, st);
}

}  // namespace tada
