// K2-fast: split-K flash-decoding over the compressed paged cache with the grouped-head
// contraction on tensor cores (mma.sync m16n8k16, f16 in / f32 accumulate), sm_100a.
//
// Reference semantics: attend_streaming (pkg/src/tadakv/attention.py:103-151) with
// K̂ = mean - (min + scale*code) (cache.py:193-200, quant.py:177-180).  The kernel uses
// the algebraically identical factored form (SURVEY §7 hard part 2):
//   q·k̂      = q·mean − min·Σq − scale·(q·code)
//   Σ p·v̂    = p·vmean − Σ(p·vmin) − (p∘vscale)·vcode
// Codes (≤255) are exact in f16, so q·code is exact per product; the f32 means enter
// as an f16 hi + lo pair (≈22-bit); accumulation is f32.  Residual (uncompressed) rows
// are handled by attn_residual_kernel into an extra split slot; K3 merges the slots.
//
// CTA = (split, sequence): 8 consumer warps + 1 producer warp.  The producer streams
// 32-token tiles (K/V means, packed codes, scale/min) with cp.async.bulk (TMA bulk
// copies, UBLKCP) into a 2-stage mbarrier ring; each tile the consumers
//   1. convert the f32 means to f16 hi/lo in place (swizzled for ldmatrix),
//   2. QK: S[tok, head] = mean-term + per-kv-head code-term MMAs, fold min/scale,
//   3. online softmax (running max / normaliser per q head), P and P' = -p*vscale to smem,
//   4. PV: O^T[d, head] += vmean^T·P^T + vcode^T·P'^T (one f32 accumulator).
#include <cuda_runtime.h>

#include <string>

#include "tada_attn.cuh"

namespace tada {
namespace fast {

constexpr int D = 128;
constexpr int TT = 32;    // tokens per tile
constexpr int NCW = 8;    // consumer warps
constexpr int NTHR = (NCW + 1) * 32;
constexpr int SROW = TT + 4;  // logits row stride (floats): conflict-free fragment stores
constexpr int PROW = TT + 8;  // P row stride (halves): conflict-free B-fragment loads
constexpr int STAGES = 2;

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "TADA_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TADA_WAIT_%=;\n}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory"); }

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// Masked integer pair (v in the low bits of each 16-bit half) -> exact f16x2 (v0, v1):
// (0x6400 | v) is the f16 1024 + v; subtracting 1024 is exact.
__device__ __forceinline__ uint32_t ints_to_h2(uint32_t x) {
  uint32_t r;
  asm("sub.f16x2 %0, %1, %2;" : "=r"(r) : "r"(x | 0x64006400u), "r"(0x64006400u));
  return r;
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void split_h2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 back = __half22float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack_h2(x0 - back.x, x1 - back.y);
}

// ------------------------------------------------------------------ k-slot <-> d maps (QK)
// Thread quad-index i owns d in [32i, 32i+32) of every token; within k-step s its slots
// (2i, 2i+1, 2i+8, 2i+9) map to d = 32i + base(s) + off[which] so that each f16x2
// operand is one masked shift of a packed code word (see file header).
template <int BITS>
__device__ __forceinline__ int slot_base(int s) {
  return BITS == 4 ? 8 * (s >> 1) + 2 * (s & 1) : (BITS == 2 ? 16 * (s >> 2) + 2 * (s & 3) : 4 * s);
}
template <int BITS>
__device__ __forceinline__ int slot_off1() {
  return BITS == 4 ? 4 : (BITS == 2 ? 8 : 2);
}
// slot 'which' (0: 2i, 1: 2i+1, 2: 2i+8, 3: 2i+9) -> d offset within the thread's 32-d block
template <int BITS>
__device__ __forceinline__ int slot_d(int s, int which) {
  const int o1 = slot_off1<BITS>();
  const int off = which == 0 ? 0 : (which == 1 ? o1 : (which == 2 ? 1 : o1 + 1));
  return slot_base<BITS>(s) + off;
}

// Code A-fragment regs for one token row (QK): from the thread's packed words of that row.
template <int BITS>
__device__ __forceinline__ void qk_code_pair(const uint32_t* w, int s, uint32_t& lo, uint32_t& hi) {
  if (BITS == 4) {
    const uint32_t x = w[s >> 1] >> (8 * (s & 1));
    lo = ints_to_h2(x & 0x000F000Fu);
    hi = ints_to_h2((x >> 4) & 0x000F000Fu);
  } else if (BITS == 2) {
    const uint32_t x = w[s >> 2] >> (4 * (s & 3));
    lo = ints_to_h2(x & 0x00030003u);
    hi = ints_to_h2((x >> 2) & 0x00030003u);
  } else {
    lo = ints_to_h2(prmt(w[s], 0, 0x4240u) & 0x00FF00FFu);
    hi = ints_to_h2(prmt(w[s], 0, 0x4341u) & 0x00FF00FFu);
  }
}

// ------------------------------------------------------------------ shared memory plan
struct Plan {
  int H, gb;
  int mean_bytes, codes_bytes, meta_bytes, side_bytes, stage_bytes;
  int off_sbuf, off_pbuf, off_p2buf, off_qsum, off_corr, off_stats, off_bar, total;
};

__host__ __device__ inline int up128(int x) { return (x + 127) / 128 * 128; }

__host__ __device__ inline Plan make_plan(int H, int gb, int HQ) {
  Plan p{};
  p.H = H;
  p.gb = gb;
  p.mean_bytes = TT * D * 4;
  p.codes_bytes = up128(TT * H * gb);
  p.meta_bytes = up128(TT * H * 8);
  p.side_bytes = p.mean_bytes + p.codes_bytes + p.meta_bytes;
  p.stage_bytes = 2 * p.side_bytes;
  int off = STAGES * p.stage_bytes;
  p.off_sbuf = off;
  off += up128(HQ * SROW * 4);
  p.off_pbuf = off;
  off += up128(HQ * PROW * 2);
  p.off_p2buf = off;
  off += up128(HQ * PROW * 2);
  p.off_qsum = off;
  off += up128(HQ * 4);
  p.off_corr = off;
  off += up128(HQ * 4);
  p.off_stats = off;
  off += up128(HQ * 4 * 4);
  p.off_bar = off;
  off += 128;
  p.total = off;
  return p;
}

// ------------------------------------------------------------------ the kernel
template <int BITS, int HQ>
__global__ void __launch_bounds__(NTHR, 1) attn_fast_kernel(AttnArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int NT = HQ / 8;  // n-tiles of 8 q heads
  constexpr int NQK = 2 * NT;  // QK work items (m-tile x n-tile)
  constexpr int IPW = (NQK + NCW - 1) / NCW;  // items per warp (QK and PV alike)
  constexpr int TPH = (NCW * 32) / HQ;  // softmax threads per q head
  constexpr int TPT = TT / TPH;         // tokens per softmax thread
  const int H = a.L.heads, G = HQ / H, gb = a.L.group_bytes, P = a.L.page_tokens;
  const Plan pl = make_plan(H, gb, HQ);
  const int b = blockIdx.y, split = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, qi = lane & 3;

  float* sbuf = reinterpret_cast<float*>(smem + pl.off_sbuf);
  __half* pbuf = reinterpret_cast<__half*>(smem + pl.off_pbuf);
  __half* p2buf = reinterpret_cast<__half*>(smem + pl.off_p2buf);
  float* qsum = reinterpret_cast<float*>(smem + pl.off_qsum);
  float* corr_s = reinterpret_cast<float*>(smem + pl.off_corr);
  float* stats = reinterpret_cast<float*>(smem + pl.off_stats);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + pl.off_bar);
  uint64_t* empty = full + STAGES;

  const int C = a.comp_len[b];
  int t_begin, t_end;
  split_range(C, a.splits, split, TT, t_begin, t_end);
  const int ntiles = (t_end - t_begin + TT - 1) / TT;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // q row sums (f32, for the min term)
  const float* qf = reinterpret_cast<const float*>(a.q) + int64_t(b) * HQ * D;
  const __nv_bfloat16* qb = reinterpret_cast<const __nv_bfloat16*>(a.q) + int64_t(b) * HQ * D;
  auto qload = [&](int g, int d) -> float { return a.q_dtype == TADA_F32 ? qf[g * D + d] : __bfloat162float(qb[g * D + d]); };
  for (int g = warp; g < HQ; g += NCW + 1) {
    float sacc = 0.f;
    for (int d = lane; d < D; d += 32) sacc += qload(g, d);
    sacc = warp_sum(sacc);
    if (lane == 0) qsum[g] = sacc;
  }
  __syncthreads();

  if (warp == NCW) {
    // ================================================================ producer
    if (lane == 0) {
      const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
      const uint32_t row_bytes_mean = D * 4, row_bytes_codes = H * gb, row_bytes_meta = H * 8;
      for (int it = 0; it < ntiles; ++it) {
        const int stg = it % STAGES;
        if (it >= STAGES) mbar_wait(&empty[stg], ((it / STAGES) - 1) & 1);
        const int t0 = t_begin + it * TT;
        const int nv = min(TT, t_end - t0);
        const uint8_t* page = a.pool + int64_t(pt[t0 / P]) * a.L.page_bytes;
        const int row = t0 % P;
        uint8_t* dst = smem + stg * pl.stage_bytes;
        const uint32_t bm = nv * row_bytes_mean;
        const uint32_t bc = (nv * row_bytes_codes + 15) & ~15u;
        const uint32_t bt = (nv * row_bytes_meta + 15) & ~15u;
        mbar_expect_tx(&full[stg], 2 * (bm + bc + bt));
        for (int side = 0; side < 2; ++side) {
          uint8_t* d0 = dst + side * pl.side_bytes;
          bulk_g2s(d0, page + a.L.off_mean[side] + int64_t(row) * row_bytes_mean, bm, &full[stg]);
          bulk_g2s(d0 + pl.mean_bytes, page + a.L.off_codes[side] + int64_t(row) * row_bytes_codes, bc, &full[stg]);
          bulk_g2s(d0 + pl.mean_bytes + pl.codes_bytes, page + a.L.off_meta[side] + int64_t(row) * row_bytes_meta, bt,
                   &full[stg]);
        }
      }
    }
    return;
  }

  // ================================================================== consumers
  // Q B-fragments (k = d slot, n = q head) for this warp's QK n-tiles, f16.
  uint32_t bq[IPW][8][2];
  int qk_mt[IPW], qk_nt[IPW];
#pragma unroll
  for (int j = 0; j < IPW; ++j) {
    const int item = warp + j * NCW;
    qk_mt[j] = item % 2;
    qk_nt[j] = item / 2;
    if (item < NQK) {
      const int g = 8 * qk_nt[j] + r;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        const int dbase = 32 * qi;
        bq[j][s][0] = pack_h2(qload(g, dbase + slot_d<BITS>(s, 0)), qload(g, dbase + slot_d<BITS>(s, 1)));
        bq[j][s][1] = pack_h2(qload(g, dbase + slot_d<BITS>(s, 2)), qload(g, dbase + slot_d<BITS>(s, 3)));
      }
    }
  }
  // PV accumulators O^T[d, head]: item -> (d-half dh, n-tile nt), 4 m-tiles of 16 d-rows.
  float oacc[IPW][4][4];
#pragma unroll
  for (int j = 0; j < IPW; ++j)
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int e = 0; e < 4; ++e) oacc[j][k][e] = 0.f;

  // softmax ownership: thread -> (q head sg, token part)
  const int sg = tid / TPH, spart = tid % TPH;
  const int sh = sg / G;  // its kv head
  float m_run = -__int_as_float(0x7f800000), l_part = 0.f, bp_part = 0.f;
  const float scale = a.scale;
  const float LOG2E = 1.4426950408889634f;

  for (int it = 0; it < ntiles; ++it) {
    const int stg = it % STAGES;
    const int t0 = t_begin + it * TT;
    const int nv = min(TT, t_end - t0);
    mbar_wait(&full[stg], (it / STAGES) & 1);
    uint8_t* base = smem + stg * pl.stage_bytes;
    float* kmean = reinterpret_cast<float*>(base);
    const uint8_t* kcodes = base + pl.mean_bytes;
    const float2* kmeta = reinterpret_cast<const float2*>(base + pl.mean_bytes + pl.codes_bytes);
    float* vmean = reinterpret_cast<float*>(base + pl.side_bytes);
    const uint8_t* vcodes = base + pl.side_bytes + pl.mean_bytes;
    const float2* vmeta = reinterpret_cast<const float2*>(base + pl.side_bytes + pl.mean_bytes + pl.codes_bytes);

    // ---------------------------------------------------------------- 1. mean f32 -> f16 hi/lo, in place
    {
      // K: item (t, s, i): slots (2i,2i+1) -> chunk 2s word i, slots (2i+8,2i+9) -> chunk 2s+1 word i
      float2 ka[4], kb[4];
      float va[2][8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int item = tid + u * NCW * 32;  // 0..1023
        const int t = item >> 5, s = (item >> 2) & 7, i = item & 3;
        const float* row = kmean + t * D + 32 * i + slot_base<BITS>(s);
        ka[u] = *reinterpret_cast<const float2*>(row);
        kb[u] = *reinterpret_cast<const float2*>(row + slot_off1<BITS>());
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int item = tid + u * NCW * 32;  // 0..511: (t, q8)
        const int t = item >> 4, q8 = item & 15;
        const float4 x0 = *reinterpret_cast<const float4*>(vmean + t * D + 8 * q8);
        const float4 x1 = *reinterpret_cast<const float4*>(vmean + t * D + 8 * q8 + 4);
        const bool ok = t < nv;
        va[u][0] = ok ? x0.x : 0.f; va[u][1] = ok ? x0.y : 0.f; va[u][2] = ok ? x0.z : 0.f; va[u][3] = ok ? x0.w : 0.f;
        va[u][4] = ok ? x1.x : 0.f; va[u][5] = ok ? x1.y : 0.f; va[u][6] = ok ? x1.z : 0.f; va[u][7] = ok ? x1.w : 0.f;
      }
      consumer_sync();
      uint32_t* khi = reinterpret_cast<uint32_t*>(kmean);          // [TT][64 words] swizzled chunks
      uint32_t* klo = reinterpret_cast<uint32_t*>(kmean) + TT * 64;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int item = tid + u * NCW * 32;
        const int t = item >> 5, s = (item >> 2) & 7, i = item & 3;
        uint32_t h0, l0, h1, l1;
        split_h2(ka[u].x, kb[u].x, h0, l0);
        split_h2(ka[u].y, kb[u].y, h1, l1);
        const int c0 = (2 * s) ^ (t & 7), c1 = (2 * s + 1) ^ (t & 7);
        khi[t * 64 + c0 * 4 + i] = h0;
        klo[t * 64 + c0 * 4 + i] = l0;
        khi[t * 64 + c1 * 4 + i] = h1;
        klo[t * 64 + c1 * 4 + i] = l1;
      }
      __half* vhi = reinterpret_cast<__half*>(vmean);  // [TT][16 chunks][8]
      __half* vlo = vhi + TT * D;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int item = tid + u * NCW * 32;
        const int t = item >> 4, q8 = item & 15, dh = q8 >> 3, rr = q8 & 7;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = (8 * dh + j) ^ (t & 7);
          const __half h = __float2half_rn(va[u][j]);
          vhi[t * D + c * 8 + rr] = h;
          vlo[t * D + c * 8 + rr] = __float2half_rn(va[u][j] - __half2float(h));
        }
      }
      consumer_sync();
    }

    // ---------------------------------------------------------------- 2. QK
#pragma unroll
    for (int j = 0; j < IPW; ++j) {
      const int item = warp + j * NCW;
      if (item >= NQK) break;
      const int mt = qk_mt[j], nt = qk_nt[j];
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      {
        const int tok = 16 * mt + (lane & 7) + 8 * ((lane >> 3) & 1);
        const int sub = lane >> 4;
        const uint32_t rowhi = su32(kmean) + tok * 256, rowlo = rowhi + TT * 256;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const int c = (2 * s + sub) ^ (tok & 7);
          uint32_t ah[4], al[4];
          ldsm_x4(ah, rowhi + c * 16);
          ldsm_x4(al, rowlo + c * 16);
          mma(acc, ah, bq[j][s][0], bq[j][s][1]);
          mma(acc, al, bq[j][s][0], bq[j][s][1]);
        }
      }
      const int t_r = 16 * mt + r, t_r8 = t_r + 8;
      const int g0 = 8 * nt + 2 * qi, g1 = g0 + 1;
      const int h0 = g0 / G, h1 = g1 / G;
      const float qs0 = qsum[g0], qs1 = qsum[g1];
      const int hfirst = (8 * nt) / G, hlast = (8 * nt + 7) / G;
      constexpr int WPR = BITS == 8 ? 8 : (BITS == 4 ? 4 : 2);  // code words per (token, head) per thread
      for (int h = hfirst; h <= hlast; ++h) {
        uint32_t wr[WPR], wr8[WPR];
        const uint8_t* cr = kcodes + (t_r * H + h) * gb + (32 * qi * BITS) / 8;
        const uint8_t* cr8 = kcodes + (t_r8 * H + h) * gb + (32 * qi * BITS) / 8;
#pragma unroll
        for (int w = 0; w < WPR; w += 2) {
          const uint2 x = *reinterpret_cast<const uint2*>(cr + 4 * w);
          const uint2 y = *reinterpret_cast<const uint2*>(cr8 + 4 * w);
          wr[w] = x.x; wr[w + 1] = x.y; wr8[w] = y.x; wr8[w + 1] = y.y;
        }
        float cacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          uint32_t af[4];
          qk_code_pair<BITS>(wr, s, af[0], af[2]);
          qk_code_pair<BITS>(wr8, s, af[1], af[3]);
          mma(cacc, af, bq[j][s][0], bq[j][s][1]);
        }
        const float2 m_r = kmeta[t_r * H + h], m_r8 = kmeta[t_r8 * H + h];
        if (h0 == h) {
          acc[0] = fmaf(-m_r.x, cacc[0], fmaf(-m_r.y, qs0, acc[0]));
          acc[2] = fmaf(-m_r8.x, cacc[2], fmaf(-m_r8.y, qs0, acc[2]));
        }
        if (h1 == h) {
          acc[1] = fmaf(-m_r.x, cacc[1], fmaf(-m_r.y, qs1, acc[1]));
          acc[3] = fmaf(-m_r8.x, cacc[3], fmaf(-m_r8.y, qs1, acc[3]));
        }
      }
      const float ninf = -__int_as_float(0x7f800000);
      sbuf[g0 * SROW + t_r] = t_r < nv ? acc[0] * scale : ninf;
      sbuf[g1 * SROW + t_r] = t_r < nv ? acc[1] * scale : ninf;
      sbuf[g0 * SROW + t_r8] = t_r8 < nv ? acc[2] * scale : ninf;
      sbuf[g1 * SROW + t_r8] = t_r8 < nv ? acc[3] * scale : ninf;
    }
    consumer_sync();

    // ---------------------------------------------------------------- 3. online softmax
    {
      float x[TPT];
      float tmax = -__int_as_float(0x7f800000);
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        x[u] = sbuf[sg * SROW + spart * TPT + u];
        tmax = fmaxf(tmax, x[u]);
      }
#pragma unroll
      for (int o = TPH / 2; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
      const float m_new = fmaxf(m_run, tmax);
      const float corr = exp2f((m_run - m_new) * LOG2E);
      m_run = m_new;
      float lsum = 0.f, bsum = 0.f;
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const int t = spart * TPT + u;
        const float p = exp2f((x[u] - m_new) * LOG2E);
        const float2 vm = t < nv ? vmeta[t * H + sh] : make_float2(0.f, 0.f);
        lsum += p;
        bsum = fmaf(p, vm.y, bsum);
        pbuf[sg * PROW + t] = __float2half_rn(p);
        p2buf[sg * PROW + t] = __float2half_rn(-p * vm.x);
      }
      l_part = l_part * corr + lsum;
      bp_part = bp_part * corr + bsum;
      if (spart == 0) corr_s[sg] = corr;
    }
    consumer_sync();

    // ---------------------------------------------------------------- 4. PV
#pragma unroll
    for (int j = 0; j < IPW; ++j) {
      const int item = warp + j * NCW;
      if (item >= NQK) break;
      const int dh = item % 2, nt = item / 2;
      const int gc0 = 8 * nt + 2 * qi;
      const float c0 = corr_s[gc0], c1 = corr_s[gc0 + 1];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        oacc[j][k][0] *= c0;
        oacc[j][k][1] *= c1;
        oacc[j][k][2] *= c0;
        oacc[j][k][3] *= c1;
      }
      const int gb_row = 8 * nt + r;  // B column (q head) of this thread
      const int hcol = gb_row / G;
      const int hfirst = (8 * nt) / G, hlast = (8 * nt + 7) / G;
#pragma unroll
      for (int ks = 0; ks < TT / 16; ++ks) {
        const uint32_t bp0 = *reinterpret_cast<const uint32_t*>(pbuf + gb_row * PROW + 16 * ks + 2 * qi);
        const uint32_t bp1 = *reinterpret_cast<const uint32_t*>(pbuf + gb_row * PROW + 16 * ks + 2 * qi + 8);
        const uint32_t bq0 = *reinterpret_cast<const uint32_t*>(p2buf + gb_row * PROW + 16 * ks + 2 * qi);
        const uint32_t bq1 = *reinterpret_cast<const uint32_t*>(p2buf + gb_row * PROW + 16 * ks + 2 * qi + 8);
        // mean term: ldmatrix.trans of the converted vmean (rows = d, cols = tokens)
        {
          const int mat = lane >> 3;
          const int tok = 16 * ks + (lane & 7) + 8 * (mat >> 1);
          const uint32_t rowhi = su32(vmean) + tok * 256, rowlo = rowhi + TT * 256;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int c = (8 * dh + 2 * k + (mat & 1)) ^ (tok & 7);
            uint32_t ah[4], al[4];
            ldsm_x4_t(ah, rowhi + c * 16);
            ldsm_x4_t(al, rowlo + c * 16);
            mma(oacc[j][k], ah, bp0, bp1);
            mma(oacc[j][k], al, bp0, bp1);
          }
        }
        // code term, one kv head at a time, B = -p*vscale masked to that head's columns
        const int ta = 16 * ks + 2 * qi, tb = ta + 1, tc = ta + 8, td = ta + 9;
        for (int h = hfirst; h <= hlast; ++h) {
          const uint32_t m0 = hcol == h ? bq0 : 0u, m1 = hcol == h ? bq1 : 0u;
          uint32_t af[4][4];
          if (BITS == 4) {
            const int off = 32 * dh + 4 * r;
            const uint32_t wa = *reinterpret_cast<const uint32_t*>(vcodes + (ta * H + h) * gb + off);
            const uint32_t wb = *reinterpret_cast<const uint32_t*>(vcodes + (tb * H + h) * gb + off);
            const uint32_t wc = *reinterpret_cast<const uint32_t*>(vcodes + (tc * H + h) * gb + off);
            const uint32_t wd = *reinterpret_cast<const uint32_t*>(vcodes + (td * H + h) * gb + off);
            const uint32_t x01 = prmt(wa, wb, 0x5410u), y01 = prmt(wa, wb, 0x7632u);
            const uint32_t x23 = prmt(wc, wd, 0x5410u), y23 = prmt(wc, wd, 0x7632u);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t u01 = k < 2 ? x01 : y01, u23 = k < 2 ? x23 : y23;
              const int shf = 8 * (k & 1);
              af[k][0] = ints_to_h2((u01 >> shf) & 0x000F000Fu);
              af[k][1] = ints_to_h2((u01 >> (shf + 4)) & 0x000F000Fu);
              af[k][2] = ints_to_h2((u23 >> shf) & 0x000F000Fu);
              af[k][3] = ints_to_h2((u23 >> (shf + 4)) & 0x000F000Fu);
            }
          } else if (BITS == 2) {
            const int off = 16 * dh + 2 * r;
            const uint32_t wa = *reinterpret_cast<const uint16_t*>(vcodes + (ta * H + h) * gb + off);
            const uint32_t wb = *reinterpret_cast<const uint16_t*>(vcodes + (tb * H + h) * gb + off);
            const uint32_t wc = *reinterpret_cast<const uint16_t*>(vcodes + (tc * H + h) * gb + off);
            const uint32_t wd = *reinterpret_cast<const uint16_t*>(vcodes + (td * H + h) * gb + off);
            const uint32_t x01 = wa | (wb << 16), x23 = wc | (wd << 16);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              af[k][0] = ints_to_h2((x01 >> (4 * k)) & 0x00030003u);
              af[k][1] = ints_to_h2((x01 >> (4 * k + 2)) & 0x00030003u);
              af[k][2] = ints_to_h2((x23 >> (4 * k)) & 0x00030003u);
              af[k][3] = ints_to_h2((x23 >> (4 * k + 2)) & 0x00030003u);
            }
          } else {
            const int off = 64 * dh + 8 * r;
            const uint2 wa = *reinterpret_cast<const uint2*>(vcodes + (ta * H + h) * gb + off);
            const uint2 wb = *reinterpret_cast<const uint2*>(vcodes + (tb * H + h) * gb + off);
            const uint2 wc = *reinterpret_cast<const uint2*>(vcodes + (tc * H + h) * gb + off);
            const uint2 wd = *reinterpret_cast<const uint2*>(vcodes + (td * H + h) * gb + off);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              // offsets 2k (row r) and 2k+1 (row r+8) live in word k/2, bytes (2k)%4 and (2k+1)%4
              const uint32_t a01 = k < 2 ? wa.x : wa.y, b01 = k < 2 ? wb.x : wb.y;
              const uint32_t a23 = k < 2 ? wc.x : wc.y, b23 = k < 2 ? wd.x : wd.y;
              const uint32_t n0 = (2 * k) & 3, n1 = n0 + 1;
              const uint32_t s0 = n0 | (n0 << 4) | ((4 + n0) << 8) | ((4 + n0) << 12);
              const uint32_t s1 = n1 | (n1 << 4) | ((4 + n1) << 8) | ((4 + n1) << 12);
              af[k][0] = ints_to_h2(prmt(a01, b01, s0) & 0x00FF00FFu);
              af[k][1] = ints_to_h2(prmt(a01, b01, s1) & 0x00FF00FFu);
              af[k][2] = ints_to_h2(prmt(a23, b23, s0) & 0x00FF00FFu);
              af[k][3] = ints_to_h2(prmt(a23, b23, s1) & 0x00FF00FFu);
            }
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) mma(oacc[j][k], af[k], m0, m1);
        }
      }
    }
    // release the stage: generic-proxy writes (in-place conversion) must be ordered
    // before the next async-proxy bulk copy into this buffer.
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stg]);
  }

  // ------------------------------------------------------------------ epilogue
  {
#pragma unroll
    for (int o = TPH / 2; o > 0; o >>= 1) {
      l_part += __shfl_xor_sync(0xffffffffu, l_part, o);
      bp_part += __shfl_xor_sync(0xffffffffu, bp_part, o);
    }
    if (spart == 0) {
      stats[4 * sg + 0] = m_run;
      stats[4 * sg + 1] = l_part;
      stats[4 * sg + 2] = bp_part;
    }
  }
  consumer_sync();
#pragma unroll
  for (int j = 0; j < IPW; ++j) {
    const int item = warp + j * NCW;
    if (item >= NQK) break;
    const int dh = item % 2, nt = item / 2;
    const int g0 = 8 * nt + 2 * qi;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int g = g0 + e;
      const float m = stats[4 * g], l = stats[4 * g + 1], bp = stats[4 * g + 2];
      float* pa = a.part_acc + ((int64_t(b) * HQ + g) * a.slots + split) * D;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int d = 64 * dh + 8 * r + 2 * k;
        // rows r (d) and r+8 (d+1): elements e and e+2 of the accumulator
        *reinterpret_cast<float2*>(pa + d) = make_float2(oacc[j][k][e] - bp, oacc[j][k][e + 2] - bp);
      }
      if (dh == 0 && r == 0) {
        float* ml = a.part_ml + ((int64_t(b) * HQ + g) * a.slots + split) * 2;
        ml[0] = l > 0.f ? m : -__int_as_float(0x7f800000);
        ml[1] = l;
      }
    }
  }
}

}  // namespace fast

// ------------------------------------------------------------------ residual rows -> extra split slot
// The raw f32 residual tokens (cache.py:174-180) of each sequence, attended exactly like
// the reference's residual tiles (attention.py:94-100); result goes to slot `splits`.
__global__ void __launch_bounds__(256) attn_residual_kernel(AttnArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int H = a.L.heads, D = a.L.head_dim, Hq = a.Hq, G = Hq / H;
  const int b = blockIdx.x, tid = threadIdx.x, bd = blockDim.x;
  const int R = a.res_len[b];
  constexpr int TILE = 32;
  float* qs = sm;                 // [Hq][D]
  float* acc = qs + Hq * D;       // [Hq][D]
  float* lg = acc + Hq * D;       // [Hq][TILE]
  float* mrow = lg + Hq * TILE;
  float* lrow = mrow + Hq;
  float* crow = lrow + Hq;
  for (int i = tid; i < Hq * D; i += bd) {
    qs[i] = a.q_dtype == TADA_F32 ? reinterpret_cast<const float*>(a.q)[int64_t(b) * Hq * D + i]
                                  : __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.q)[int64_t(b) * Hq * D + i]);
    acc[i] = 0.f;
  }
  for (int g = tid; g < Hq; g += bd) {
    mrow[g] = -__int_as_float(0x7f800000);
    lrow[g] = 0.f;
  }
  __syncthreads();
  const int64_t base = int64_t(b) * a.res_seq_stride;
  for (int t0 = 0; t0 < R; t0 += TILE) {
    const int nt = min(TILE, R - t0);
    for (int pair = tid; pair < Hq * nt; pair += bd) {
      const int g = pair / nt, j = pair - g * nt, h = g / G;
      const float* kr = a.res_k + ((base + t0 + j) * H + h) * D;
      const float* qg = qs + g * D;
      float dot = 0.f;
      for (int d = 0; d < D; ++d) dot = __fmaf_rn(qg[d], kr[d], dot);
      lg[g * TILE + j] = __fmul_rn(dot, a.scale);
    }
    __syncthreads();
    for (int g = tid; g < Hq; g += bd) {
      float tmax = lg[g * TILE];
      for (int j = 1; j < nt; ++j) tmax = fmaxf(tmax, lg[g * TILE + j]);
      const float m_new = fmaxf(mrow[g], tmax);
      const float corr = expf(mrow[g] - m_new);
      float sum = 0.f;
      for (int j = 0; j < nt; ++j) {
        const float p = expf(lg[g * TILE + j] - m_new);
        lg[g * TILE + j] = p;
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
      for (int j = 0; j < nt; ++j) av = __fmaf_rn(lg[g * TILE + j], a.res_v[((base + t0 + j) * H + h) * D + d], av);
      acc[pair] = av;
    }
    __syncthreads();
  }
  for (int pair = tid; pair < Hq * D; pair += bd) {
    const int g = pair / D, d = pair - g * D;
    a.part_acc[((int64_t(b) * Hq + g) * a.slots + a.splits) * D + d] = acc[pair];
  }
  for (int g = tid; g < Hq; g += bd) {
    float* ml = a.part_ml + ((int64_t(b) * Hq + g) * a.slots + a.splits) * 2;
    ml[0] = mrow[g];
    ml[1] = lrow[g];
  }
}

bool fast_supported(const tada_page_layout& L, int Hq) {
  if (L.head_dim != 128 || !(L.bits == 2 || L.bits == 4 || L.bits == 8)) return false;
  if (!(Hq == 8 || Hq == 16 || Hq == 32 || Hq == 64) || Hq % L.heads) return false;
  const int G = Hq / L.heads;
  if (!(G == 1 || G == 2 || G == 4 || G == 8)) return false;
  if (L.page_tokens % fast::TT) return false;
  return fast::make_plan(L.heads, L.group_bytes, Hq).total <= 227 * 1024;
}

template <int BITS, int HQ>
static int launch_fast_t(const AttnArgs& a, int batch, cudaStream_t st) {
  const fast::Plan pl = fast::make_plan(a.L.heads, a.L.group_bytes, HQ);
  auto kern = fast::attn_fast_kernel<BITS, HQ>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("attn_fast smem: ") + cudaGetErrorString(e));
    attr_set = true;
  }
  kern<<<dim3(a.splits, batch), fast::NTHR, pl.total, st>>>(a);
  return check_launch("decode_attn_fast");
}

template <int BITS>
static int launch_fast_b(const AttnArgs& a, int batch, cudaStream_t st) {
  switch (a.Hq) {
    case 8: return launch_fast_t<BITS, 8>(a, batch, st);
    case 16: return launch_fast_t<BITS, 16>(a, batch, st);
    case 32: return launch_fast_t<BITS, 32>(a, batch, st);
    default: return launch_fast_t<BITS, 64>(a, batch, st);
  }
}

int launch_fast(const AttnArgs& a, int batch, cudaStream_t st) {
  switch (a.L.bits) {
    case 2: return launch_fast_b<2>(a, batch, st);
    case 4: return launch_fast_b<4>(a, batch, st);
    default: return launch_fast_b<8>(a, batch, st);
  }
}

int launch_residual(const AttnArgs& a, int batch, cudaStream_t st) {
  const size_t smem = (size_t(2) * a.Hq * a.L.head_dim + size_t(a.Hq) * 32 + 3 * a.Hq) * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(attn_residual_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("attn_residual smem: ") + cudaGetErrorString(e));
  }
  attn_residual_kernel<<<batch, 256, smem, st>>>(a);
  return check_launch("decode_attn_residual");
}

}  // namespace tada
