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
// CTA = (split, sequence): 8 consumer warps + 1 producer warp.  The producer warp streams
// 32-token tiles with cp.async.bulk (TMA bulk copies, UBLKCP), one copy per token row into
// bank-shifted padded rows, through a 2-3 stage mbarrier ring.  Per tile the consumers
//   1. QK (warp = 8 tokens x half of head_dim): S[g, t] = Q·mean (f16 hi/lo, converted in
//      registers) - min*sum(q) - scale*(Q·codes), q heads on the MMA M dimension;
//   2. online softmax per q head (exp2 domain); P and P' = -p*vscale to smem (f16);
//   3. PV (warp = 16 of head_dim): O[g, d] += P·vmean + P'_h·vcode_h, one f32 accumulator.
#include <cuda_runtime.h>

#include <cudaTypedefs.h>

#include <mutex>
#include <string>
#include <unordered_map>

#include "tada_attn.cuh"

namespace tada {
namespace fast {

constexpr int D = 128;
constexpr int TT = 32;    // tokens per tile
constexpr int NCW = 8;    // consumer warps
constexpr int NTHR = NCW * 32;  // no dedicated producer warp: thread 0 issues the TMA copies
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
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory"); }  // all warps

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
// A stage holds one 32-token tile of both sides, loaded with 3-D TMA tensor copies
// (cp.async.bulk.tensor, UTMALDG) from the paged pool:
//   mean  : 4 bands of [32 rows x 128 B], 128B-swizzled  (D*4 = 512 B per row)
//   codes : H*gb/128 bands of [32 rows x 128 B], 128B-swizzled
//   meta  : one box [32 rows x TROW B] (TROW = H*8 + 16: the 16 B past the row are the
//           TMA's out-of-bounds zero fill, which shifts banks by 4 per row)
constexpr int BAND = TT * 128;  // bytes per 128-byte-wide band of a tile

struct Plan {
  int H, gb, trow, nbands_c;
  int mean_bytes, codes_bytes, meta_bytes, side_bytes, stage_bytes, stages;
  int off_sbuf, off_pbuf, off_p2m, off_qsum, off_corr, off_stats, off_bar, total;
};

__host__ __device__ inline int up128(int x) { return (x + 127) / 128 * 128; }
__host__ __device__ inline int up1k(int x) { return (x + 1023) / 1024 * 1024; }

__host__ __device__ inline Plan make_plan(int H, int gb, int HQ) {
  Plan p{};
  const int MT = (HQ + 15) / 16;
  p.H = H;
  p.gb = gb;
  p.trow = H * 8 + 16;
  p.nbands_c = (H * gb) / 128;
  p.mean_bytes = (D * 4 / 128) * BAND;
  p.codes_bytes = p.nbands_c * BAND;
  // stage = [K mean][K codes][V mean][V codes][K meta][V meta]: the swizzled regions stay 1 KB
  // aligned while the two small meta boxes share the tail (8-bit then fits two stages)
  p.meta_bytes = up128(TT * p.trow);
  p.side_bytes = p.mean_bytes + p.codes_bytes;
  p.stage_bytes = up1k(2 * p.side_bytes + 2 * p.meta_bytes);
  // sbuf doubles as the f16 q staging area (prologue) and the PV partial-sum area (epilogue)
  const int sbuf = up128(2 * HQ * SROW * 4);
  const int stage_q = MT * 16 * D * 2;
  const int sb = sbuf > stage_q ? sbuf : stage_q;
  const int tail = sb + up128(MT * 16 * PROW * 2) + up128(H * 16 * PROW * 2) + 2 * up128(HQ * 4) + up128(HQ * 16) +
                   128 + 1024;
  const int budget = 227 * 1024;
  p.stages = (3 * p.stage_bytes + tail <= budget) ? 3 : ((2 * p.stage_bytes + tail <= budget) ? 2 : 1);
  int off = p.stages * p.stage_bytes;
  p.off_sbuf = off;
  off += sb;
  p.off_pbuf = off;
  off += up128(MT * 16 * PROW * 2);
  p.off_p2m = off;
  off += up128(H * 16 * PROW * 2);
  p.off_qsum = off;
  off += up128(HQ * 4);
  p.off_corr = off;
  off += up128(HQ * 4);
  p.off_stats = off;
  off += up128(HQ * 16);
  p.off_bar = off;
  off += 128;
  p.total = off + 1024;
  return p;
}

// byte offset of (row t, byte o) inside a 128B-swizzled [TT x 128 B] band
__device__ __forceinline__ int swz(int t, int o) { return t * 128 + ((((o >> 4) ^ t) & 7) << 4) + (o & 15); }

__device__ __forceinline__ void tma_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
// Wait with a suspend-time hint: the thread sleeps in hardware instead of spinning.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "TADA_WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra TADA_WAITS_%=;\n}\n" ::"r"(su32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// ------------------------------------------------------------------ the kernel
// Fragment orientation: q heads on M for both products.
//   QK: S[g, t] = Q[g, d] · K̂^T[d, t]    A = Q (registers, f16), B = K-mean / K-codes tiles
//       warp = (token octet, half of head_dim)
//   PV: O[g, d] = P[g, t] · V̂[t, d]      A = P, P'_h (smem, ldmatrix), B = V-mean / V-codes tiles
//       warp = (32-wide d slice, 16-token half of the tile)
// so every mean and code byte of a tile is read from smem by exactly one warp.
template <int BITS, int HQ, int H>
__global__ void __launch_bounds__(NTHR, 1) attn_fast_kernel(AttnArgs a, const __grid_constant__ TmaMaps maps) {
  extern __shared__ uint8_t smem_raw[];
  // 1 KB alignment (128B-swizzle atoms) by pointer arithmetic on the __shared__ array, so the
  // compiler keeps the shared state space (LDS, 32-bit addressing) for every access below
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  constexpr int G = HQ / H;
  constexpr int MT = (HQ + 15) / 16;    // m-tiles of 16 q heads
  constexpr int HPM = 16 / G < H ? 16 / G : H;  // kv heads per m-tile
  constexpr int TPH = (NCW * 32) / HQ;  // softmax threads per q head
  constexpr int TPT = TT / TPH;         // tokens per softmax thread
  constexpr int GB = BITS * D / 8;      // code bytes per (token, head)
  const int P = a.L.page_tokens;
  const Plan pl = make_plan(H, GB, HQ);
  const int b = blockIdx.y, split = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, qi = lane & 3;

  float* sbuf = reinterpret_cast<float*>(smem + pl.off_sbuf);  // [2][HQ][SROW]
  __half* pbuf = reinterpret_cast<__half*>(smem + pl.off_pbuf);  // [MT*16][PROW]
  __half* p2m = reinterpret_cast<__half*>(smem + pl.off_p2m);    // [H][16][PROW]: -p*vscale, rows of kv head h only
  float* qsum = reinterpret_cast<float*>(smem + pl.off_qsum);
  float* corr_s = reinterpret_cast<float*>(smem + pl.off_corr);
  float* stats = reinterpret_cast<float*>(smem + pl.off_stats);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + pl.off_bar);
  const int S = pl.stages;

  const int C = a.comp_len[b];
  int t_begin, t_end;
  split_range(C, a.splits, split, TT, t_begin, t_end);
  const int ntiles = (t_end - t_begin + TT - 1) / TT;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // zero P'_h (rows not belonging to head h stay zero forever) and the padded P rows
  for (int i = tid; i < (H * 16 * PROW) / 2; i += NTHR) reinterpret_cast<uint32_t*>(p2m)[i] = 0u;
  for (int i = tid; i < (MT * 16 * PROW) / 2; i += NTHR) reinterpret_cast<uint32_t*>(pbuf)[i] = 0u;
  __syncthreads();

  // TMA producer (thread 0): tile `it` -> stage it % S.  A stage is refilled only after a
  // consumer barrier that every warp reaches after finishing the stage's previous tile.
  const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
  const uint32_t tx = 2u * uint32_t(pl.mean_bytes + pl.codes_bytes + TT * pl.trow);
  auto issue = [&](int it) {
    const int stg = it % S;
    const int t0 = t_begin + it * TT;
    const int page = pt[t0 / P];
    const int row0 = t0 % P;
    uint8_t* dst = smem + stg * pl.stage_bytes;
    mbar_expect_tx(&full[stg], tx);
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      uint8_t* d0 = dst + side * pl.side_bytes;
#pragma unroll
      for (int j = 0; j < 4; ++j) tma_3d(d0 + j * BAND, &maps.m[side][0], 128 * j, row0, page, &full[stg]);
#pragma unroll
      for (int j = 0; j < (H * GB) / 128; ++j)
        tma_3d(d0 + pl.mean_bytes + j * BAND, &maps.m[side][1], 128 * j, row0, page, &full[stg]);
      tma_3d(dst + 2 * pl.side_bytes + side * pl.meta_bytes, &maps.m[side][2], 0, row0, page, &full[stg]);
    }
  };
  if (tid == 0) {
    for (int s2 = 0; s2 < 2; ++s2)
      for (int k = 0; k < 3; ++k)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[s2][k])) : "memory");
    for (int it = 0; it < S - 1 && it < ntiles; ++it) issue(it);
  }

  // ================================================================== consumers
  // prologue: q rows -> f32 row sums (min term) + f16 copy (staged in sbuf)
  {
    __half* q16 = reinterpret_cast<__half*>(sbuf);
    for (int g = warp; g < MT * 16; g += NCW) {
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (g < HQ) {
        if (a.q_dtype == TADA_F32) load4(reinterpret_cast<const float*>(a.q) + (int64_t(b) * HQ + g) * D + 4 * lane, v);
        else load4(reinterpret_cast<const __nv_bfloat16*>(a.q) + (int64_t(b) * HQ + g) * D + 4 * lane, v);
      }
      const float ssum = warp_sum(v[0] + v[1] + v[2] + v[3]);
      if (lane == 0 && g < HQ) qsum[g] = ssum;
      *reinterpret_cast<uint2*>(q16 + g * D + 4 * lane) = make_uint2(pack_h2(v[0], v[1]), pack_h2(v[2], v[3]));
    }
  }
  consumer_sync();
  const int kh = warp & 1, tq = 8 * (warp >> 1) + r;  // QK: k-half and this thread's B column (token)
  const int tc0 = 8 * (warp >> 1) + 2 * qi;           // QK accumulator columns (tokens) tc0, tc0+1
  uint32_t qa[MT][4][4];
  {
    const __half* q16 = reinterpret_cast<const __half*>(sbuf);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const int s = 4 * kh + k4, dq = 32 * qi;
        const int g0 = 16 * mt + r, g1 = g0 + 8;
        auto q2 = [&](int g, int w0, int w1) -> uint32_t {
          const __half2 h = __halves2half2(q16[g * D + dq + slot_d<BITS>(s, w0)], q16[g * D + dq + slot_d<BITS>(s, w1)]);
          return *reinterpret_cast<const uint32_t*>(&h);
        };
        qa[mt][k4][0] = q2(g0, 0, 1);
        qa[mt][k4][1] = q2(g1, 0, 1);
        qa[mt][k4][2] = q2(g0, 2, 3);
        qa[mt][k4][3] = q2(g1, 2, 3);
      }
  }
  // kv head of this thread's accumulator rows (16mt + r, 16mt + r + 8); -1 = padding row
  int kvr[MT][2];
  float qsr[MT][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int g = 16 * mt + r + 8 * e;
      kvr[mt][e] = g < HQ ? g / G : -1;
      qsr[mt][e] = g < HQ ? qsum[g] : 0.f;
    }
  // QK code addresses: (row tq, byte h*GB + off) with off = (32qi + 16kh)*BITS/8 < 128
  constexpr int CW = BITS == 8 ? 4 : (BITS == 4 ? 2 : 1);  // code words per (token, head) per thread
  const int qk_c0 = swz(tq, ((32 * qi + 16 * kh) * BITS) / 8);
  // PV: warp = (d slice dq of 32, token half kk); B column r <-> d = 32dq + 4r + n (n-tile n = 0..3)
  const int dq = warp & 3, kk = warp >> 2;
  float oacc[MT][4][4];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int e = 0; e < 4; ++e) oacc[mt][n][e] = 0.f;
  const int sg = tid / TPH, spart = tid % TPH, sh = sg / G;  // softmax ownership
  float m_run = -__int_as_float(0x7f800000), l_part = 0.f, bp_part = 0.f;
  const float scale_log2 = a.scale * 1.4426950408889634f;
  consumer_sync();  // q16 staging area is dead from here on

  for (int it = 0; it < ntiles; ++it) {
    const int stg = it % S;
    const int t0 = t_begin + it * TT;
    const int nv = min(TT, t_end - t0);
    mbar_wait(&full[stg], (it / S) & 1);
    const uint8_t* base = smem + stg * pl.stage_bytes;
    const uint8_t* kmean = base;
    const uint8_t* kcodes = base + pl.mean_bytes;
    const uint8_t* kmeta = base + 2 * pl.side_bytes;
    const uint8_t* vmean = base + pl.side_bytes;
    const uint8_t* vcodes = vmean + pl.mean_bytes;
    const uint8_t* vmeta = kmeta + pl.meta_bytes;

    // ---------------------------------------------------------------- QK (warp = token octet x k-half)
    {
      float acc[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
      // mean term: d = 32qi + 16kh + [0,16) of token tq = band qi, bytes 64kh + [0,64)
      float x[16];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 v = *reinterpret_cast<const float4*>(kmean + qi * BAND + swz(tq, 64 * kh + 16 * u));
        x[4 * u] = v.x; x[4 * u + 1] = v.y; x[4 * u + 2] = v.z; x[4 * u + 3] = v.w;
      }
#pragma unroll
      for (int k4 = 0; k4 < 4; ++k4) {
        const int rb = slot_base<BITS>(k4), o1 = slot_off1<BITS>();  // == slot_base(4kh+k4) - 16kh
        uint32_t h0, l0, h1, l1;
        split_h2(x[rb], x[rb + o1], h0, l0);
        split_h2(x[rb + 1], x[rb + o1 + 1], h1, l1);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          mma(acc[mt], qa[mt][k4], h0, h1);
          mma(acc[mt], qa[mt][k4], l0, l1);
        }
      }
      // code term: per m-tile, its HPM kv heads as independent accumulation chains
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        uint32_t w[HPM][CW];
        float cacc[HPM][4];
#pragma unroll
        for (int j = 0; j < HPM; ++j) {
          const int h = mt * HPM + j;
          const int hb = h * GB;
          const uint8_t* cp = kcodes + (hb >> 7) * BAND + (qk_c0 ^ (hb & 127));
          if (CW == 4) {
            const uint4 v = *reinterpret_cast<const uint4*>(cp);
            w[j][0] = v.x; w[j][1 % CW] = v.y; w[j][2 % CW] = v.z; w[j][3 % CW] = v.w;
          } else if (CW == 2) {
            const uint2 v = *reinterpret_cast<const uint2*>(cp);
            w[j][0] = v.x; w[j][1 % CW] = v.y;
          } else {
            w[j][0] = *reinterpret_cast<const uint32_t*>(cp);
          }
          cacc[j][0] = cacc[j][1] = cacc[j][2] = cacc[j][3] = 0.f;
        }
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4)
#pragma unroll
          for (int j = 0; j < HPM; ++j) {
            uint32_t b0, b1;
            qk_code_pair<BITS>(w[j], k4, b0, b1);
            mma(cacc[j], qa[mt][k4], b0, b1);
          }
#pragma unroll
        for (int j = 0; j < HPM; ++j) {
          const int h = mt * HPM + j;
          const float2 ma = *reinterpret_cast<const float2*>(kmeta + tc0 * pl.trow + h * 8);
          const float2 mb = *reinterpret_cast<const float2*>(kmeta + (tc0 + 1) * pl.trow + h * 8);
          const float mna = kh == 0 ? ma.y : 0.f, mnb = kh == 0 ? mb.y : 0.f;
          if (kvr[mt][0] == h) {
            acc[mt][0] = fmaf(-ma.x, cacc[j][0], fmaf(-mna, qsr[mt][0], acc[mt][0]));
            acc[mt][1] = fmaf(-mb.x, cacc[j][1], fmaf(-mnb, qsr[mt][0], acc[mt][1]));
          }
          if (kvr[mt][1] == h) {
            acc[mt][2] = fmaf(-ma.x, cacc[j][2], fmaf(-mna, qsr[mt][1], acc[mt][2]));
            acc[mt][3] = fmaf(-mb.x, cacc[j][3], fmaf(-mnb, qsr[mt][1], acc[mt][3]));
          }
        }
      }
      float* sb = sbuf + kh * HQ * SROW;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int g0 = 16 * mt + r, g1 = g0 + 8;
        if (g0 < HQ) *reinterpret_cast<float2*>(sb + g0 * SROW + tc0) = make_float2(acc[mt][0], acc[mt][1]);
        if (g1 < HQ) *reinterpret_cast<float2*>(sb + g1 * SROW + tc0) = make_float2(acc[mt][2], acc[mt][3]);
      }
    }
    consumer_sync();

    // every warp has finished tile it-1 (its PV) -> refill that stage with tile it+S-1
    if (tid == 0 && it + S - 1 < ntiles) issue(it + S - 1);
    // ---------------------------------------------------------------- online softmax
    {
      float x[TPT];
      float tmax = -__int_as_float(0x7f800000);
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const int t = spart + TPH * u;
        x[u] = t < nv ? (sbuf[sg * SROW + t] + sbuf[(HQ + sg) * SROW + t]) * scale_log2 : -__int_as_float(0x7f800000);
        tmax = fmaxf(tmax, x[u]);
      }
#pragma unroll
      for (int o = TPH / 2; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
      const float m_new = fmaxf(m_run, tmax);  // in log2 units
      const float corr = exp2f(m_run - m_new);
      m_run = m_new;
      float lsum = 0.f, bsum = 0.f;
      __half* p2row = p2m + (sh * 16 + (sg & 15)) * PROW;
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const int t = spart + TPH * u;
        const float p = exp2f(x[u] - m_new);
        const float2 vm = t < nv ? *reinterpret_cast<const float2*>(vmeta + t * pl.trow + sh * 8) : make_float2(0.f, 0.f);
        lsum += p;
        bsum = fmaf(p, vm.y, bsum);
        pbuf[sg * PROW + t] = __float2half_rn(p);
        p2row[t] = __float2half_rn(-p * vm.x);
      }
      l_part = l_part * corr + lsum;
      bp_part = bp_part * corr + bsum;
      if (spart == 0) corr_s[sg] = corr;
    }
    consumer_sync();

    // ---------------------------------------------------------------- PV (warp = 32-wide d slice x 16 tokens)
    {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const float c0 = kvr[mt][0] >= 0 ? corr_s[16 * mt + r] : 0.f;
        const float c1 = kvr[mt][1] >= 0 ? corr_s[16 * mt + r + 8] : 0.f;
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          oacc[mt][n][0] *= c0;
          oacc[mt][n][1] *= c0;
          oacc[mt][n][2] *= c1;
          oacc[mt][n][3] *= c1;
        }
      }
      const int ta = 16 * kk + 2 * qi;  // this thread's B rows: tokens ta, ta+1, ta+8, ta+9
      // mean term: float4 of d = 32dq + 4r .. +3 for each of the 4 tokens
      uint32_t bh[4][2], bl[4][2];
      {
        const uint8_t* vb = vmean + dq * BAND;
        const float4 xa = *reinterpret_cast<const float4*>(vb + swz(ta, 16 * r));
        const float4 xb = *reinterpret_cast<const float4*>(vb + swz(ta + 1, 16 * r));
        const float4 xc = *reinterpret_cast<const float4*>(vb + swz(ta + 8, 16 * r));
        const float4 xd = *reinterpret_cast<const float4*>(vb + swz(ta + 9, 16 * r));
        split_h2(xa.x, xb.x, bh[0][0], bl[0][0]);
        split_h2(xc.x, xd.x, bh[0][1], bl[0][1]);
        split_h2(xa.y, xb.y, bh[1][0], bl[1][0]);
        split_h2(xc.y, xd.y, bh[1][1], bl[1][1]);
        split_h2(xa.z, xb.z, bh[2][0], bl[2][0]);
        split_h2(xc.z, xd.z, bh[2][1], bl[2][1]);
        split_h2(xa.w, xb.w, bh[3][0], bl[3][0]);
        split_h2(xc.w, xd.w, bh[3][1], bl[3][1]);
      }
      const int mrow = (lane & 7) + 8 * ((lane >> 3) & 1), tcol = 16 * kk + 8 * (lane >> 4);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        uint32_t pa[4];
        ldsm_x4(pa, su32(pbuf + (16 * mt + mrow) * PROW + tcol));
#pragma unroll
        for (int n = 0; n < 4; ++n) {
          mma(oacc[mt][n], pa, bh[n][0], bh[n][1]);
          mma(oacc[mt][n], pa, bl[n][0], bl[n][1]);
        }
      }
      // code term: per kv head, A = P'_h (pre-masked rows), B = its codes of d = 32dq + 4r .. +3
      constexpr int CB = BITS * 4 / 8;  // code bytes per token for the thread's 4 d
      const int pv_c = (32 * dq + 4 * r) * BITS / 8;
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int hb = h * GB + pv_c;
        const uint8_t* cband = vcodes + (hb >> 7) * BAND;
        const int co = hb & 127;
        uint32_t xa, xb, xc, xd;
        if (CB == 4) {
          xa = *reinterpret_cast<const uint32_t*>(cband + swz(ta, co));
          xb = *reinterpret_cast<const uint32_t*>(cband + swz(ta + 1, co));
          xc = *reinterpret_cast<const uint32_t*>(cband + swz(ta + 8, co));
          xd = *reinterpret_cast<const uint32_t*>(cband + swz(ta + 9, co));
        } else if (CB == 2) {
          xa = *reinterpret_cast<const uint16_t*>(cband + swz(ta, co));
          xb = *reinterpret_cast<const uint16_t*>(cband + swz(ta + 1, co));
          xc = *reinterpret_cast<const uint16_t*>(cband + swz(ta + 8, co));
          xd = *reinterpret_cast<const uint16_t*>(cband + swz(ta + 9, co));
        } else {
          xa = cband[swz(ta, co)];
          xb = cband[swz(ta + 1, co)];
          xc = cband[swz(ta + 8, co)];
          xd = cband[swz(ta + 9, co)];
        }
        uint32_t bc[4][2];
        if (BITS == 8) {
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            const uint32_t sel = n | (n << 4) | ((4 + n) << 8) | ((4 + n) << 12);
            bc[n][0] = ints_to_h2(prmt(xa, xb, sel) & 0x00FF00FFu);
            bc[n][1] = ints_to_h2(prmt(xc, xd, sel) & 0x00FF00FFu);
          }
        } else {
          constexpr uint32_t M = BITS == 4 ? 0x000F000Fu : 0x00030003u;
          const uint32_t u = xa | (xb << 16), v = xc | (xd << 16);
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            bc[n][0] = ints_to_h2((u >> (BITS * n)) & M);
            bc[n][1] = ints_to_h2((v >> (BITS * n)) & M);
          }
        }
        constexpr int mth_div = 16 / G;
        const int mth = h / (mth_div < 1 ? 1 : mth_div);
        uint32_t am[4];
        ldsm_x4(am, su32(p2m + (h * 16 + mrow) * PROW + tcol));
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          if (mt != mth) continue;
#pragma unroll
          for (int n = 0; n < 4; ++n) mma(oacc[mt][n], am, bc[n][0], bc[n][1]);
        }
      }
    }
  }

  // ------------------------------------------------------------------ epilogue
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
  // the two token halves (kk) hold partial O: kk = 1 parks its half in smem, kk = 0 adds it
  float* park = reinterpret_cast<float*>(smem);  // stages are idle now: [MT*16][D] floats
  consumer_sync();
  // thread rows g = 16mt + r (+8); cols: n-tile n, col 2qi / 2qi+1 <-> d = 32dq + 8qi + n / + 4 + n
  if (kk == 1) {
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        float* row = park + (16 * mt + r + 8 * e) * D + 32 * dq + 8 * qi;
        *reinterpret_cast<float4*>(row) =
            make_float4(oacc[mt][0][2 * e], oacc[mt][1][2 * e], oacc[mt][2][2 * e], oacc[mt][3][2 * e]);
        *reinterpret_cast<float4*>(row + 4) =
            make_float4(oacc[mt][0][2 * e + 1], oacc[mt][1][2 * e + 1], oacc[mt][2][2 * e + 1], oacc[mt][3][2 * e + 1]);
      }
  }
  consumer_sync();
  if (kk == 0) {
    const float LN2 = 0.6931471805599453f;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int g = 16 * mt + r + 8 * e;
        if (g >= HQ) continue;
        const float m = stats[4 * g], l = stats[4 * g + 1], bp = stats[4 * g + 2];
        const float* row = park + g * D + 32 * dq + 8 * qi;
        const float4 p0 = *reinterpret_cast<const float4*>(row);
        const float4 p1 = *reinterpret_cast<const float4*>(row + 4);
        float* pa = a.part_acc + ((int64_t(b) * HQ + g) * a.slots + split) * D + 32 * dq + 8 * qi;
        *reinterpret_cast<float4*>(pa) =
            make_float4(oacc[mt][0][2 * e] + p0.x - bp, oacc[mt][1][2 * e] + p0.y - bp, oacc[mt][2][2 * e] + p0.z - bp,
                        oacc[mt][3][2 * e] + p0.w - bp);
        *reinterpret_cast<float4*>(pa + 4) =
            make_float4(oacc[mt][0][2 * e + 1] + p1.x - bp, oacc[mt][1][2 * e + 1] + p1.y - bp,
                        oacc[mt][2][2 * e + 1] + p1.z - bp, oacc[mt][3][2 * e + 1] + p1.w - bp);
        if (dq == 0 && qi == 0) {
          float* ml = a.part_ml + ((int64_t(b) * HQ + g) * a.slots + split) * 2;
          ml[0] = l > 0.f ? m * LN2 : -__int_as_float(0x7f800000);  // back to natural-log units for K3
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
  // compiled geometries: 8 KV heads (the Llama-3 family) with 8/16/32/64 q heads
  if (L.head_dim != 128 || !(L.bits == 2 || L.bits == 4 || L.bits == 8) || L.heads != 8) return false;
  if (!(Hq == 8 || Hq == 16 || Hq == 32 || Hq == 64)) return false;
  if (L.page_tokens % fast::TT) return false;
  const fast::Plan pl = fast::make_plan(L.heads, L.group_bytes, Hq);
  return pl.stages >= 2 && pl.total <= 227 * 1024;  // one stage cannot overlap load and compute
}

// ---------------------------------------------------------------- TMA descriptors
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3-D byte tensor over the pool: (byte in row, row in page, page); box = [box0 B, 32 rows, 1 page].
static bool encode_region(CUtensorMap* m, const uint8_t* base, uint64_t row_bytes, uint64_t rows, uint64_t page_bytes,
                          uint32_t box0, bool swizzle) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[3] = {row_bytes, rows, uint64_t(1) << 20};
  const cuuint64_t strides[2] = {row_bytes, page_bytes};
  const cuuint32_t box[3] = {box0, uint32_t(fast::TT), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int get_maps(const AttnArgs& a, TmaMaps* out) {
  struct Key {
    const uint8_t* pool;
    int64_t page_bytes;
    int bits, heads, page_tokens;
    bool operator==(const Key& o) const {
      return pool == o.pool && page_bytes == o.page_bytes && bits == o.bits && heads == o.heads &&
             page_tokens == o.page_tokens;
    }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.pool) ^ (std::hash<int64_t>()(k.page_bytes) << 1) ^ size_t(k.bits * 131 + k.heads);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, TmaMaps, Hash> cache;
  const Key key{a.pool, a.L.page_bytes, a.L.bits, a.L.heads, a.L.page_tokens};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return TADA_OK;
  }
  TmaMaps m{};
  const tada_page_layout& L = a.L;
  const uint32_t trow = uint32_t(L.heads * 8 + 16);
  for (int side = 0; side < 2; ++side) {
    if (!encode_region(&m.m[side][0], a.pool + L.off_mean[side], uint64_t(L.head_dim) * 4, L.page_tokens, L.page_bytes,
                       128, true) ||
        !encode_region(&m.m[side][1], a.pool + L.off_codes[side], uint64_t(L.heads) * L.group_bytes, L.page_tokens,
                       L.page_bytes, 128, true) ||
        !encode_region(&m.m[side][2], a.pool + L.off_meta[side], uint64_t(L.heads) * 8, L.page_tokens, L.page_bytes,
                       trow, false))
      return fail(TADA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the decode-attention pool");
  }
  if (cache.size() > 256) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return TADA_OK;
}

template <int BITS, int HQ>
static int launch_fast_t(const AttnArgs& a, int batch, cudaStream_t st) {
  const fast::Plan pl = fast::make_plan(a.L.heads, a.L.group_bytes, HQ);
  auto kern = fast::attn_fast_kernel<BITS, HQ, 8>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("attn_fast smem: ") + cudaGetErrorString(e));
    attr_set = true;
  }
  TmaMaps maps;
  const int rc = get_maps(a, &maps);
  if (rc != TADA_OK) return rc;
  kern<<<dim3(a.splits, batch), fast::NTHR, pl.total, st>>>(a, maps);
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
