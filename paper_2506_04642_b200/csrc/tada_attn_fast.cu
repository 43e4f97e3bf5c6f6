// K2-fast: split-K flash-decoding over the compressed paged cache, sm_100a.
//
// Reference semantics: attend_streaming (pkg/src/tadakv/attention.py:103-151) with
// K̂ = mean - (min + scale*code) (cache.py:193-200, quant.py:177-180).  The kernel uses the
// algebraically identical factored form (SURVEY §7 hard part 2):
//   q·k̂   = q·mean − min·Σq − scale·(q·code)
//   Σ p·v̂ = p·vmean − Σ(p·vmin) + p'·vcode,      p' = −p·vscale
// and runs both contractions on tensor cores (mma.sync m16n8k16, f16 × f16 → f32).  Codes
// (≤ 255) are exact in f16; the f32 means enter as an f16 hi + lo pair (≈ 22-bit).
//
// Why mma.sync and not tcgen05: every operand here is produced in registers (packed codes
// → f16 by a LOP3 + HSUB2 per pair, means split hi/lo), N is the GQA group (≤ 8), and the
// kernel is HBM-bound.  tcgen05 would need the dequantised operands written back to shared
// memory in the UMMA layout first (an extra 64 KB of STS per 32-token tile per side).
//
// CTA = (split, sequence), 16 warps.  Warp w owns KV head h = w & 7 and token half
// hf = w >> 3 of every 32-token tile:
//   * QK code term, token-on-M: S_h^T[tok, n] = codes_h[tok, d] · Q_h^T[d, n], n = the G q
//     heads of h (N = 8 columns, G used);
//   * its own online softmax over its 16 tokens (m, l per q head and half);
//   * PV code term, d-on-M: O_h^T[d, n] += codes_h^T[d, tok] · P'_h^T[tok, n].
// The mean terms are shared by all KV heads and are split across the 16 warps as pieces:
//   * QK: S_mean[q, tok] = Q[q, d] · mean^T[d, tok]     (q-tile, token octet, d half)
//   * PV: O_mean[q, d]  += P_hf[q, tok] · vmean[tok, d]  (token half, q-tile, 32-wide d block)
// Tiles stream in with 3-D TMA tensor copies (cp.async.bulk.tensor, 128B swizzle) through a
// 2-3 stage mbarrier ring; two CTA barriers per tile.
#include <cuda_runtime.h>

#include <cudaTypedefs.h>

#include <mutex>
#include <string>
#include <unordered_map>

#include "tada_attn.cuh"
#include "tada_mma.cuh"

namespace tada {
namespace fast {
using namespace mmaops;

constexpr int D = 128;
constexpr int HT = 16;  // tokens per warp (one m16 tile of the token-on-M QK code term)
// Tile geometry: TT tokens per tile, TT/2 warps (warp = KV head x 16-token half), so TT = 32 runs
// one 512-thread CTA per SM and TT = 16 runs two 256-thread CTAs per SM (their barriers interleave).
__host__ __device__ constexpr int nw_of(int tt) { return tt / 2; }
__host__ __device__ constexpr int sr_of(int tt) { return tt + 4; }   // S row stride (floats)
__host__ __device__ constexpr int pr_of(int tt) { return tt + 8; }   // P / P' row stride (halves): conflict-free
__host__ __device__ constexpr int band_of(int tt) { return tt * 128; }  // bytes of one 128-B-wide swizzled band

// ------------------------------------------------------------------ shared memory plan
struct Plan {
  int mean_bytes, codes_bytes, meta_bytes, side_bytes, stage_bytes, stages;
  int trow;
  int off_sbuf, off_q16, off_qa, qa_bytes, off_pbuf, off_p2, off_corr, off_red, off_qsum, off_bar, total;
};

__host__ __device__ constexpr int up128(int x) { return (x + 127) / 128 * 128; }
__host__ __device__ constexpr int up1k(int x) { return (x + 1023) / 1024 * 1024; }
// QK mean-term partial planes (d splits): 4 (16 warps x 2 k-steps), or 2 (8 warps x 4 k-steps) where
// shared memory is tight (8-bit); plus one plane for the code term
__host__ __device__ constexpr int nkq_for(int gb) { return gb >= 128 ? 2 : 4; }

__host__ __device__ constexpr Plan make_plan(int H, int gb, int HQ, int TT) {
  Plan p{};
  const int NSP = nkq_for(gb) + 1;
  const int BAND = band_of(TT), SROW = sr_of(TT), PROW2 = pr_of(TT);
  const int mrows = HQ >= 16 ? HQ : 16;
  p.trow = H * 8 + 16;  // meta box row: the 16 B past the row are TMA zero fill (shifts banks by 4 per row)
  p.mean_bytes = (D * 4 / 128) * BAND;
  p.codes_bytes = (H * gb / 128) * BAND;
  // stage = [means K, V][codes K, V][metas K, V] (one TMA copy each); swizzled regions 1 KB aligned
  p.meta_bytes = TT * p.trow;
  p.side_bytes = p.mean_bytes + p.codes_bytes;
  p.stage_bytes = up1k(2 * p.side_bytes + 2 * p.meta_bytes);
  const int sb = up128(NSP * mrows * SROW * 4);
  const int pb = up128(mrows * PROW2 * 2);
  const int p2 = up128(H * 8 * PROW2 * 2);
  // TT = 16 keeps the QK mean-term Q fragments in shared memory (registers are the limit at 128)
  p.qa_bytes = TT == 16 ? up128(mrows * D * 2) : 0;
  const int tail = sb + p.qa_bytes + pb + p2 + up128(mrows * 4) + up128(3 * HQ * 4) + up128(HQ * 4) + 128;
  const int budget = TT == 16 ? 113 * 1024 : 227 * 1024;  // TT = 16: two CTAs per SM
  p.stages = (3 * p.stage_bytes + tail <= budget) ? 3 : ((2 * p.stage_bytes + tail <= budget) ? 2 : 1);
  int off = p.stages * p.stage_bytes;
  // the epilogue parks the partial output [HQ][D] f32 in the (idle) stages
  if (off < HQ * D * 4) p.stages = 0;
  p.off_sbuf = off;
  off += sb;
  p.off_q16 = (p.stages - 1) * p.stage_bytes;  // prologue-only q staging: the last stage is loaded after it
  p.off_qa = off;
  off += p.qa_bytes;
  p.off_pbuf = off;
  off += pb;
  p.off_p2 = off;
  off += p2;
  p.off_corr = off;
  off += up128(mrows * 4);
  p.off_red = off;
  off += up128(3 * HQ * 4);
  p.off_qsum = off;
  off += up128(HQ * 4);
  p.off_bar = off;
  off += 128;
  p.total = off;
  return p;
}

// ------------------------------------------------------------------ the kernel
// Per 32-token tile (phases separated by the two CTA barriers):
//  A  QK mean piece  (warp w: token octet w&3, d quarter w>>2, all q tiles) -> S [q][tok] (red.shared.add)
//     QK code term   (warp (h, half))                                        -> S [q][tok] (red.shared.add)
//  B  softmax, dense: thread = (q head, TT/TPQ tokens); P [q][tok], P'_h^T [n][tok], corr [q]
//  C  PV code term   (warp (h, half): its 16 tokens, all d)       -> O_h^T in registers
//     PV mean piece  (warp w: d octet w, all q tiles, all tokens) -> O_mean in registers
template <int BITS, int HQ, int TT>
__global__ void __launch_bounds__(TT * 16, TT == 16 ? 2 : 1) attn_fast_kernel(AttnArgs a,
                                                                              const __grid_constant__ TmaMaps maps) {
  constexpr int NW = nw_of(TT), NTHR = NW * 32, SROW = sr_of(TT), PROW2 = pr_of(TT), BAND = band_of(TT);
  // The dynamic shared window of a CTA without static shared memory starts 1 KB aligned (the TMA
  // 128B-swizzle atom); with the base a link-time constant every shared address below is an
  // immediate offset.  Checked once, loudly.
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0 && (su32(smem) & 1023u) != 0) __trap();
  constexpr int H = 8;
  constexpr int G = HQ / H;                     // q heads per KV head (N columns used)
  constexpr int MT = HQ >= 16 ? HQ / 16 : 1;    // 16-row q tiles
  constexpr int MROWS = MT * 16;
  constexpr int GB = BITS * D / 8;              // code bytes per (token, head)
  constexpr Plan pl = make_plan(H, GB, HQ, TT);
  constexpr int S = pl.stages < 2 ? 2 : pl.stages;  // geometries with < 2 stages are never launched
  constexpr int NKQ = nkq_for(GB), NSP = NKQ + 1, KS = 8 / NKQ;  // mean-term d splits, planes, k-steps each
  constexpr int TPQ0 = (NTHR / HQ) < 32 ? (NTHR / HQ) : 32;
  constexpr int TPQ = TPQ0 < TT ? TPQ0 : TT;                // softmax threads per q head
  constexpr int TPT = TT / TPQ;                             // tokens per softmax thread
  constexpr int NSM = HQ * TPQ;                             // active softmax threads
  const int P = a.L.page_tokens;
  const int b = blockIdx.y, split = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, c = lane & 3;
  const int h = warp & 7, half = warp >> 3;

  float* sbuf = reinterpret_cast<float*>(smem + pl.off_sbuf);    // [NSP][MROWS][SROW]: logit partials
  __half* q16s = reinterpret_cast<__half*>(smem + pl.off_q16);   // [MROWS][D] f16 q
  __half* pbuf = reinterpret_cast<__half*>(smem + pl.off_pbuf);  // [MROWS][PROW2]
  __half* p2all = reinterpret_cast<__half*>(smem + pl.off_p2);   // [H][8 n][PROW2]: P'_h^T
  float* corrb = reinterpret_cast<float*>(smem + pl.off_corr);   // [MROWS]
  float* red = reinterpret_cast<float*>(smem + pl.off_red);      // [3][HQ] epilogue (l, Σp·vmin, m)
  float* qsum = reinterpret_cast<float*>(smem + pl.off_qsum);    // [HQ]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + pl.off_bar);

  const int C = comp_tokens(a, b);
  int t_begin, t_end;
  split_range(C, a.splits, split, TT, t_begin, t_end);
  const int ntiles = t_end > t_begin ? (t_end - t_begin + TT - 1) / TT : 0;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // P rows of padding q heads and P' rows of unused columns n >= G stay zero forever
  for (int i = tid; i < (MROWS * PROW2) / 2; i += NTHR) reinterpret_cast<uint32_t*>(pbuf)[i] = 0u;
  for (int i = tid; i < (H * 8 * PROW2) / 2; i += NTHR) reinterpret_cast<uint32_t*>(p2all)[i] = 0u;
  for (int i = tid; i < MROWS; i += NTHR) corrb[i] = 1.f;
  int* exact_flag = reinterpret_cast<int*>(red);  // prologue only: a query element beyond the f16 range
  if (tid == 0) *exact_flag = 0;
  __syncthreads();

  // TMA producer (thread 0): tile `it` -> stage it % S.  A stage is refilled only after the CTA
  // barrier that every warp reaches once it has finished the stage's previous tile.
  const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
  constexpr uint32_t tx = 2u * uint32_t(pl.mean_bytes + pl.codes_bytes + TT * pl.trow);
  auto page_of = [&](int it) { return it < ntiles ? pt[(t_begin + it * TT) / P] : 0; };
  auto issue = [&](int it, int page) {  // one thread: three copies per tile
    const int stg = it % S;
    const int row0 = (t_begin + it * TT) % P;
    uint8_t* dst = smem + stg * pl.stage_bytes;
    mbar_expect_tx(&full[stg], tx);
    tma_5d(dst, &maps.m[0][0], row0, page, &full[stg]);
    tma_5d(dst + 2 * pl.mean_bytes, &maps.m[0][1], row0, page, &full[stg]);
    tma_4d(dst + 2 * pl.side_bytes, &maps.m[0][2], row0, page, &full[stg]);
  };
  if (tid == 0) {
    for (int k = 0; k < 3; ++k)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[0][k])) : "memory");
    for (int it = 0; it < S - 1 && it < ntiles; ++it) issue(it, page_of(it));
  }

  // ---------------------------------------------------------------- prologue: q -> f16 fragments
  {
    __half* q16 = q16s;
    for (int g = warp; g < MROWS; g += NW) {
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (g < HQ) {
        if (a.q_dtype == TADA_F32) load4(reinterpret_cast<const float*>(a.q) + (int64_t(b) * HQ + g) * D + 4 * lane, v);
        else load4(reinterpret_cast<const __nv_bfloat16*>(a.q) + (int64_t(b) * HQ + g) * D + 4 * lane, v);
      }
      const bool big = !(fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3]))) < 32768.f);
      if (__any_sync(0xffffffffu, big) && lane == 0) *exact_flag = 1;
      const uint32_t lo = pack_h2(v[0], v[1]), hi = pack_h2(v[2], v[3]);
      *reinterpret_cast<uint2*>(q16 + g * D + 4 * lane) = make_uint2(lo, hi);
      // max |q| of the f16-rounded row: the fixed-point scale of the integer code term
      const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&lo));
      const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&hi));
      float amax = fmaxf(fmaxf(fabsf(f0.x), fabsf(f0.y)), fmaxf(fabsf(f1.x), fabsf(f1.y)));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (lane == 0 && g < HQ) qsum[g] = amax;
    }
  }
  __syncthreads();
  const bool to_exact = *exact_flag || beyond_f16(a, kFastScaleExp);
  __syncthreads();  // every warp has read the flag: red[] (which it aliases) is written by the epilogue, which an
                    // empty split reaches without another barrier
  if (to_exact) {  // CTA-uniform, rare: operands beyond f16 -> exact f32 path
    for (int it = 0; it < S - 1 && it < ntiles; ++it) mbar_wait(&full[it % S], 0u);  // no copy lands after exit
    exact_split_partials<BITS, HQ / H>(a, b, split, t_begin, t_end, warp, lane);
    return;
  }
  // QK code B operand: Q_h^T as 16-bit fixed point (scale sq per KV head) split into two s8 pieces
  // (q = sq * (256 * hi + lo)), k laid out by dk(); column n = r <-> q head h*G + r.  The integer
  // products and sums are exact, so the code term is q_fx . code with no rounding at all.
  uint32_t qbh[4][2], qbl[4][2];
  float sq, qs[2];  // qs: Σ q_fx of this thread's two code columns n = 2c, 2c+1
  {
    const __half* q16 = q16s;
    float mx = 0.f;
    for (int e = 0; e < G; ++e) mx = fmaxf(mx, qsum[h * G + e]);
    constexpr float QMAX = 32639.f;  // 127 * 256 + 127: both pieces stay in s8
    sq = mx > 0.f ? mx / QMAX : 1.f;
    const float inv = mx > 0.f ? QMAX / mx : 0.f;
    const __half* qr = q16 + (h * G + (r < G ? r : 0)) * D;
    int isum = 0;
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        uint32_t ph = 0u, pl8 = 0u;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int qi = __float2int_rn(__half2float(qr[dk<BITS>(c, s, which, i)]) * inv);
          qi = r < G ? max(-32639, min(32639, qi)) : 0;
          isum += qi;
          const int qh = (qi + 128) >> 8, ql = qi - qh * 256;
          ph |= uint32_t(qh & 0xFF) << (8 * i);
          pl8 |= uint32_t(ql & 0xFF) << (8 * i);
        }
        qbh[s][which] = ph;
        qbl[s][which] = pl8;
      }
    isum += __shfl_xor_sync(0xffffffffu, isum, 1);
    isum += __shfl_xor_sync(0xffffffffu, isum, 2);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int v = __shfl_sync(0xffffffffu, isum, ((2 * c + e) & 7) * 4);
      qs[e] = (2 * c + e < G) ? sq * float(v) : 0.f;
    }
  }
  // QK mean A operand: q tile mt, k-step s = 2*kq + ks; slots (2c,2c+1 | 2c+8,2c+9) <-> d = 16s+4c+(0,1 | 2,3)
  constexpr int NT8 = TT / 8;  // token octets per tile
  const int nt = warp % NT8, kq = warp / NT8;  // QK mean piece of warps with kq < NKQ
  constexpr bool QA_SMEM = pl.qa_bytes > 0;
  uint32_t qa[QA_SMEM ? 1 : MT][QA_SMEM ? 1 : KS][4];
  uint4* qa_s = reinterpret_cast<uint4*>(smem + pl.off_qa);  // [kq][mt][ks][lane] fragments
  {
    const __half* q16 = q16s;
    if (QA_SMEM) {  // pack every piece's fragments once: (kq, mt, ks) by the warps, lane-major
      for (int f = warp; f < NKQ * MT * KS; f += NW) {
        const int kq2 = f / (MT * KS), mt = (f / KS) % MT, ks = f % KS;
        const __half* r0 = q16 + (16 * mt + r) * D + 16 * ((KS * kq2 + ks) ^ (c & 1)) + 4 * c;  // see the kmean load
        const __half* r1 = r0 + 8 * D;
        qa_s[f * 32 + lane] = make_uint4(*reinterpret_cast<const uint32_t*>(r0), *reinterpret_cast<const uint32_t*>(r1),
                                         *reinterpret_cast<const uint32_t*>(r0 + 2),
                                         *reinterpret_cast<const uint32_t*>(r1 + 2));
      }
    } else {
#pragma unroll
      for (int mt = 0; mt < (QA_SMEM ? 1 : MT); ++mt)
#pragma unroll
        for (int ks = 0; ks < (QA_SMEM ? 1 : KS); ++ks) {
          const __half* r0 = q16 + (16 * mt + r) * D + 16 * (((KS * kq + ks) & 7) ^ (c & 1)) + 4 * c;
          const __half* r1 = r0 + 8 * D;
          qa[mt][ks][0] = *reinterpret_cast<const uint32_t*>(r0);
          qa[mt][ks][1] = *reinterpret_cast<const uint32_t*>(r1);
          qa[mt][ks][2] = *reinterpret_cast<const uint32_t*>(r0 + 2);
          qa[mt][ks][3] = *reinterpret_cast<const uint32_t*>(r1 + 2);
        }
    }
  }
  fence_proxy_async();  // q staging lives in the last stage, which TMA fills after the next barrier

  // accumulators
  float oc[8][4];    // PV code term, O_h^T: m-tile of 16 d (rows) x 8 n (cols), this warp's tokens
  constexpr int NDT = 16 / NW;  // d octets per warp in the PV mean term
  float om[NDT][MT][4];  // PV mean term: q tile rows x this warp's d octets
#pragma unroll
  for (int i = 0; i < 8; ++i) oc[i][0] = oc[i][1] = oc[i][2] = oc[i][3] = 0.f;
#pragma unroll
  for (int j = 0; j < NDT; ++j)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) om[j][mt][0] = om[j][mt][1] = om[j][mt][2] = om[j][mt][3] = 0.f;
  // softmax ownership: q head sg, tokens sj + TPQ*u
  const int sg = tid / TPQ, sj = tid % TPQ, sh = sg / G;
  const bool s_active = tid < NSM;
  float m_run = -__int_as_float(0x7f800000), l_part = 0.f, bp_part = 0.f;
  const float scale_log2 = a.scale * 1.4426950408889634f;
  const float NEG_INF = -__int_as_float(0x7f800000);
  __half* p2 = p2all + h * 8 * PROW2;

  // warp 0 issues the refills right after barrier A; a late page-table load there would hold up
  // barrier B for every warp, so the page of the next refill is fetched one tile ahead
  int next_page = tid == 0 ? page_of(S - 1) : 0;
  for (int it = 0; it < ntiles; ++it) {
    const int stg = it % S;
    const int t0 = t_begin + it * TT;
    const int nv = min(TT, t_end - t0);
    mbar_wait(&full[stg], (it / S) & 1);
    const uint8_t* base = smem + stg * pl.stage_bytes;
    const uint8_t* kmean = base;
    const uint8_t* vmean = base + pl.mean_bytes;
    const uint8_t* kcodes = base + 2 * pl.mean_bytes;
    const uint8_t* vcodes = kcodes + pl.codes_bytes;
    const uint8_t* kmeta = base + 2 * pl.side_bytes;
    const uint8_t* vmeta = kmeta + pl.meta_bytes;
    if (nv < TT) {  // tail tile: rows past the sequence may hold anything; P·vmean needs them finite
      uint8_t* vm = const_cast<uint8_t*>(vmean);
      for (int i = tid; i < (TT - nv) * 32; i += NTHR) {
        const int t = nv + (i >> 5), j = i & 31;
        *reinterpret_cast<uint4*>(vm + (j >> 3) * BAND + t * 128 + (j & 7) * 16) = make_uint4(0u, 0u, 0u, 0u);
      }
      fence_proxy_async();  // generic writes before the next async (TMA) refill of this stage
    }

    // ------------------------------------------------------------ A1: QK mean piece -> S_mean[kq]
    if (kq < NKQ) {
      const int tok = 8 * nt + r;
      float acc[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int s = KS * kq + ks;
        // odd thread quads take chunk s ^ 1: an 8-lane phase (rows r, r + 1) then reads 8 distinct 16-B chunks
        const float4 x = *reinterpret_cast<const float4*>(kmean + (s >> 1) * BAND + swz(tok, 64 * ((s ^ c) & 1) + 16 * c));
        uint32_t h0, l0, h1, l1;
        split_h2(x.x, x.y, h0, l0);
        split_h2(x.z, x.w, h1, l1);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          uint32_t af[4];
          if (QA_SMEM) {
            const uint4 f = qa_s[((kq * MT + mt) * KS + ks) * 32 + lane];
            af[0] = f.x;
            af[1] = f.y;
            af[2] = f.z;
            af[3] = f.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) af[e] = qa[QA_SMEM ? 0 : mt][QA_SMEM ? 0 : ks][e];
          }
          mma(acc[mt], af, h0, h1);
          mma(acc[mt], af, l0, l1);
        }
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        float* sm = sbuf + (kq * MROWS + 16 * mt + r) * SROW + 8 * nt + 2 * c;
        *reinterpret_cast<float2*>(sm) = make_float2(acc[mt][0], acc[mt][1]);
        *reinterpret_cast<float2*>(sm + 8 * SROW) = make_float2(acc[mt][2], acc[mt][3]);
      }
    }
    // ------------------------------------------------------------ A2: QK code term (head h, token half) -> S_code
    {
      const int ta = HT * half + r, tb = ta + 8;  // accumulator rows (tokens)
      constexpr int NWD = BITS == 8 ? 8 : (BITS == 4 ? 4 : 2);  // code words per row segment
      uint32_t wa[NWD], wb[NWD];
      constexpr int SEG = GB / 4;
      const int hb = h * GB + c * SEG;
      const uint8_t* cb = kcodes + (hb >> 7) * BAND;
      const int o = hb & 127;
      if (BITS == 4) {
        const uint4 x = *reinterpret_cast<const uint4*>(cb + swz(ta, o));
        const uint4 y = *reinterpret_cast<const uint4*>(cb + swz(tb, o));
        wa[0] = x.x; wa[1 % NWD] = x.y; wa[2 % NWD] = x.z; wa[3 % NWD] = x.w;
        wb[0] = y.x; wb[1 % NWD] = y.y; wb[2 % NWD] = y.z; wb[3 % NWD] = y.w;
      } else if (BITS == 2) {
        const uint2 x = *reinterpret_cast<const uint2*>(cb + swz(ta, o));
        const uint2 y = *reinterpret_cast<const uint2*>(cb + swz(tb, o));
        wa[0] = x.x; wa[1] = x.y;
        wb[0] = y.x; wb[1] = y.y;
      } else {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const uint4 x = *reinterpret_cast<const uint4*>(cb + swz(ta, o + 16 * u));
          const uint4 y = *reinterpret_cast<const uint4*>(cb + swz(tb, o + 16 * u));
          wa[(4 * u) % NWD] = x.x; wa[(4 * u + 1) % NWD] = x.y; wa[(4 * u + 2) % NWD] = x.z; wa[(4 * u + 3) % NWD] = x.w;
          wb[(4 * u) % NWD] = y.x; wb[(4 * u + 1) % NWD] = y.y; wb[(4 * u + 2) % NWD] = y.z; wb[(4 * u + 3) % NWD] = y.w;
        }
      }
      int ch[4] = {0, 0, 0, 0}, cl[4] = {0, 0, 0, 0};  // hi / lo q-piece accumulators
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        uint32_t af[4];
        af[0] = qk_quad<BITS>(wa, s, 0);
        af[1] = qk_quad<BITS>(wb, s, 0);
        af[2] = qk_quad<BITS>(wa, s, 1);
        af[3] = qk_quad<BITS>(wb, s, 1);
        imma(ch, af, qbh[s][0], qbh[s][1]);
        imma(cl, af, qbl[s][0], qbl[s][1]);
      }
      float cs[4];  // q_fx . code / sq  (|.| <= 2^30: exact in int32)
#pragma unroll
      for (int e = 0; e < 4; ++e) cs[e] = float(ch[e] * 256 + cl[e]);
      // − scale·(q·code) − min·Σq, for the G real columns
      if (2 * c < G) {
        const float2 ka = *reinterpret_cast<const float2*>(kmeta + ta * pl.trow + 8 * h);
        const float2 kb = *reinterpret_cast<const float2*>(kmeta + tb * pl.trow + 8 * h);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (2 * c + e < G) {
            float* row = sbuf + (NKQ * MROWS + h * G + 2 * c + e) * SROW;
            row[ta] = -fmaf(ka.x * sq, cs[e], ka.y * qs[e]);
            row[tb] = -fmaf(kb.x * sq, cs[2 + e], kb.y * qs[e]);
          }
        }
      }
    }
    __syncthreads();  // ---- BARRIER A: S complete; every warp is done with the previous tile
    if (tid == 0 && it + S - 1 < ntiles) {
      issue(it + S - 1, next_page);
      next_page = page_of(it + S);
    }

    // ------------------------------------------------------------ B: online softmax, dense over (q, token)
    if (s_active) {  // thread = (q head sg, tokens TPT*sj .. +TPT-1)
      float x[TPT];
#pragma unroll
      for (int u = 0; u < TPT; ++u) x[u] = 0.f;
#pragma unroll
      for (int k = 0; k < NSP; ++k) {
        const float* srow = sbuf + (k * MROWS + sg) * SROW + TPT * sj;
        if (TPT == 4) {
          const float4 v = *reinterpret_cast<const float4*>(srow);
          x[0] += v.x; x[TPT > 1 ? 1 : 0] += v.y; x[TPT > 2 ? 2 : 0] += v.z; x[TPT > 3 ? 3 : 0] += v.w;
        } else if (TPT == 2) {
          const float2 v = *reinterpret_cast<const float2*>(srow);
          x[0] += v.x; x[TPT > 1 ? 1 : 0] += v.y;
        } else {
          x[0] += srow[0];
        }
      }
      float tmax = NEG_INF;
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        x[u] = (TPT * sj + u < nv) ? x[u] * scale_log2 : NEG_INF;
        tmax = fmaxf(tmax, x[u]);
      }
      // Lazy rescaling: the reference max only moves when a logit exceeds it by more than
      // 2^LAZY (p <= 256 stays exact enough in f16/f32), so most tiles skip the row reduction
      // and the O rescale.  A q row's TPQ threads are lanes of one warp, so the vote is uniform.
      constexpr float LAZY = 8.f;
      float corr = 1.f;
      if (__any_sync(0xffffffffu, tmax > m_run + LAZY)) {
#pragma unroll
        for (int o = TPQ / 2; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        const float m_new = fmaxf(m_run, tmax);  // finite: every tile has >= 1 valid token
        corr = ex2(m_run - m_new);
        m_run = m_new;
      }
      const float m_new = m_run;
      float lsum = 0.f, bsum = 0.f;
      __half pv[TPT], p2v[TPT];
#pragma unroll
      for (int u = 0; u < TPT; ++u) {
        const int t = TPT * sj + u;
        const float p = ex2(x[u] - m_new);
        const float2 vm = *reinterpret_cast<const float2*>(vmeta + t * pl.trow + 8 * sh);
        const bool ok = t < nv;
        lsum += p;
        bsum = fmaf(p, ok ? vm.y : 0.f, bsum);
        pv[u] = __float2half_rn(p);
        // P' in f16 unscaled: with p <= 2^8 (lazy max) it holds group scales below 2^8; layers with larger
        // scales (a deviation range above ~65k at 8 bits) are attended on the exact path (kFastScaleExp).
        // A 2^-8 pre-scale as in attn_v8_kernel would push 8-bit P' (scales ~range/255) into f16 subnormals.
        p2v[u] = __float2half_rn(ok ? -p * vm.x : 0.f);
      }
      __half* prow = pbuf + sg * PROW2 + TPT * sj;
      __half* p2r = p2all + (sh * 8 + (sg - sh * G)) * PROW2 + TPT * sj;
      if (TPT == 4) {
        *reinterpret_cast<uint2*>(prow) = *reinterpret_cast<const uint2*>(pv);
        *reinterpret_cast<uint2*>(p2r) = *reinterpret_cast<const uint2*>(p2v);
      } else if (TPT == 2) {
        *reinterpret_cast<uint32_t*>(prow) = *reinterpret_cast<const uint32_t*>(pv);
        *reinterpret_cast<uint32_t*>(p2r) = *reinterpret_cast<const uint32_t*>(p2v);
      } else {
        prow[0] = pv[0];
        p2r[0] = p2v[0];
      }
      l_part = fmaf(l_part, corr, lsum);
      bp_part = fmaf(bp_part, corr, bsum);
      if (sj == 0) corrb[sg] = corr;
    }
    __syncthreads();  // ---- BARRIER B: P, P', corr visible
    // ------------------------------------------------------------ C1: PV code term (head h, token half), d-on-M
    {
      const float c0 = (2 * c < G) ? corrb[h * G + 2 * c] : 1.f;
      const float c1 = (2 * c + 1 < G) ? corrb[h * G + 2 * c + 1] : 1.f;
      if (__any_sync(0xffffffffu, c0 != 1.f || c1 != 1.f)) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          oc[i][0] *= c0;
          oc[i][1] *= c1;
          oc[i][2] *= c0;
          oc[i][3] *= c1;
        }
      }
      const uint32_t b0 = *reinterpret_cast<const uint32_t*>(p2 + r * PROW2 + HT * half + 2 * c);
      const uint32_t b1 = *reinterpret_cast<const uint32_t*>(p2 + r * PROW2 + HT * half + 2 * c + 8);
      // rows: m-tile mt, row r <-> d = 16r + 2mt, row r+8 <-> d = 16r + 2mt + 1
      const int hb = h * GB + 2 * r * BITS;  // byte of d = 16r within head h's group
      const uint8_t* cb = vcodes + (hb >> 7) * BAND;
      const int o = hb & 127;
      const int t0a = HT * half + 2 * c;  // tokens t0a, t0a+1 (k slots 2c, 2c+1) and t0a+8, t0a+9
      if (BITS == 4) {
        uint2 w[4];
        w[0] = *reinterpret_cast<const uint2*>(cb + swz(t0a, o));
        w[1] = *reinterpret_cast<const uint2*>(cb + swz(t0a + 1, o));
        w[2] = *reinterpret_cast<const uint2*>(cb + swz(t0a + 8, o));
        w[3] = *reinterpret_cast<const uint2*>(cb + swz(t0a + 9, o));
#pragma unroll
        for (int wi = 0; wi < 2; ++wi) {
          const uint32_t xa = wi ? w[0].y : w[0].x, xb = wi ? w[1].y : w[1].x;
          const uint32_t xc = wi ? w[2].y : w[2].x, xd = wi ? w[3].y : w[3].x;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {  // d + 8wi + 4hh + (0..3)
            const uint32_t sel = hh ? 0x7632u : 0x5410u;
            const uint32_t u = prmt(xa, xb, sel), v = prmt(xc, xd, sel);
#pragma unroll
            for (int sh2 = 0; sh2 < 2; ++sh2) {  // d + 8wi + 4hh + 2sh2 + (0, 1)
              const uint32_t uu = sh2 ? (u >> 8) : u, vv = sh2 ? (v >> 8) : v;
              uint32_t af[4];
              af[0] = field_h2<0>(uu, 0x000F000Fu);
              af[1] = field_h2<4>(uu, 0x000F000Fu);
              af[2] = field_h2<0>(vv, 0x000F000Fu);
              af[3] = field_h2<4>(vv, 0x000F000Fu);
              mma(oc[4 * wi + 2 * hh + sh2], af, b0, b1);
            }
          }
        }
      } else if (BITS == 2) {
        const uint32_t xa = *reinterpret_cast<const uint32_t*>(cb + swz(t0a, o));
        const uint32_t xb = *reinterpret_cast<const uint32_t*>(cb + swz(t0a + 1, o));
        const uint32_t xc = *reinterpret_cast<const uint32_t*>(cb + swz(t0a + 8, o));
        const uint32_t xd = *reinterpret_cast<const uint32_t*>(cb + swz(t0a + 9, o));
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // codes 8hh .. 8hh+7 of the thread's 16
          const uint32_t sel = hh ? 0x7632u : 0x5410u;
          const uint32_t u = prmt(xa, xb, sel), v = prmt(xc, xd, sel);
#pragma unroll
          for (int sh2 = 0; sh2 < 2; ++sh2) {
            const uint32_t uu = sh2 ? (u >> 8) : u, vv = sh2 ? (v >> 8) : v;
            uint32_t af[4];
            af[0] = field_h2<0>(uu, 0x00030003u);
            af[1] = field_h2<2>(uu, 0x00030003u);
            af[2] = field_h2<0>(vv, 0x00030003u);
            af[3] = field_h2<2>(vv, 0x00030003u);
            mma(oc[4 * hh + 2 * sh2], af, b0, b1);
            af[0] = field_h2<4>(uu, 0x00030003u);
            af[1] = field_h2<6>(uu, 0x00030003u);
            af[2] = field_h2<4>(vv, 0x00030003u);
            af[3] = field_h2<6>(vv, 0x00030003u);
            mma(oc[4 * hh + 2 * sh2 + 1], af, b0, b1);
          }
        }
      } else {
        const uint4 xa = *reinterpret_cast<const uint4*>(cb + swz(t0a, o));
        const uint4 xb = *reinterpret_cast<const uint4*>(cb + swz(t0a + 1, o));
        const uint4 xc = *reinterpret_cast<const uint4*>(cb + swz(t0a + 8, o));
        const uint4 xd = *reinterpret_cast<const uint4*>(cb + swz(t0a + 9, o));
        const uint32_t A[4] = {xa.x, xa.y, xa.z, xa.w}, B[4] = {xb.x, xb.y, xb.z, xb.w};
        const uint32_t Cc[4] = {xc.x, xc.y, xc.z, xc.w}, Dd[4] = {xd.x, xd.y, xd.z, xd.w};
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {  // d = 16r + 2mt (+1): bytes j, j+1 (j = 2(mt&1)) of word mt/2
          const uint32_t sel = (mt & 1) ? 0x7632u : 0x5410u;  // [x.b(j), x.b(j+1), y.b(j), y.b(j+1)]
          const uint32_t u = prmt(A[mt >> 1], B[mt >> 1], sel), v = prmt(Cc[mt >> 1], Dd[mt >> 1], sel);
          uint32_t af[4];
          af[0] = hsub2(lop_and_or(u, 0x00FF00FFu, 0x64006400u), 0x64006400u);
          af[1] = hsub2(lop_and_or(u >> 8, 0x00FF00FFu, 0x64006400u), 0x64006400u);
          af[2] = hsub2(lop_and_or(v, 0x00FF00FFu, 0x64006400u), 0x64006400u);
          af[3] = hsub2(lop_and_or(v >> 8, 0x00FF00FFu, 0x64006400u), 0x64006400u);
          mma(oc[mt], af, b0, b1);
        }
      }
    }
    // ------------------------------------------------------------ C2: PV mean piece (d octet = warp)
    {
      float cr[MT][2];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        cr[mt][0] = corrb[16 * mt + r];
        cr[mt][1] = corrb[16 * mt + r + 8];
      }
      bool any = false;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) any |= (cr[mt][0] != 1.f) || (cr[mt][1] != 1.f);
      if (any) {
#pragma unroll
        for (int j = 0; j < NDT; ++j)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            om[j][mt][0] *= cr[mt][0];
            om[j][mt][1] *= cr[mt][0];
            om[j][mt][2] *= cr[mt][1];
            om[j][mt][3] *= cr[mt][1];
          }
      }
      const int mrow = (lane & 7) + 8 * ((lane >> 3) & 1), tcol = 8 * (lane >> 4);
#pragma unroll
      for (int ks = 0; ks < TT / 16; ++ks) {
        uint32_t pa[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) ldsm_x4(pa[mt], su32(pbuf + (16 * mt + mrow) * PROW2 + 16 * ks + tcol));
        const int t = 16 * ks + 2 * c;
#pragma unroll
        for (int j = 0; j < NDT; ++j) {
          const int d = 8 * (warp + NW * j) + r;  // this thread's B column
          const uint8_t* vb = vmean + (d >> 5) * BAND;
          const int ob = 4 * (d & 31);
          const float e0 = *reinterpret_cast<const float*>(vb + swz(t, ob));
          const float e1 = *reinterpret_cast<const float*>(vb + swz(t + 1, ob));
          const float e2 = *reinterpret_cast<const float*>(vb + swz(t + 8, ob));
          const float e3 = *reinterpret_cast<const float*>(vb + swz(t + 9, ob));
          uint32_t bh0, bl0, bh1, bl1;
          split_h2(e0, e1, bh0, bl0);
          split_h2(e2, e3, bh1, bl1);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            mma(om[j][mt], pa[mt], bh0, bh1);
            mma(om[j][mt], pa[mt], bl0, bl1);
          }
        }
      }
    }
  }

  // ------------------------------------------------------------------ epilogue
  // per-thread partial l and Σp·vmin -> per q head
  if (s_active) {
#pragma unroll
    for (int o = TPQ / 2; o > 0; o >>= 1) {
      l_part += __shfl_xor_sync(0xffffffffu, l_part, o);
      bp_part += __shfl_xor_sync(0xffffffffu, bp_part, o);
    }
    if (sj == 0) {
      red[sg] = l_part;
      red[HQ + sg] = bp_part;
      red[2 * HQ + sg] = m_run;
    }
  }
  float* park = reinterpret_cast<float*>(smem);  // [HQ][D]: the stages are idle now
  __syncthreads();
  // 1) mean term: rows q = 16mt + r (+8), cols d = 8*warp + 2c (+1)
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int g = 16 * mt + r + 8 * e;
      if (g < HQ)
#pragma unroll
        for (int j = 0; j < NDT; ++j)
          *reinterpret_cast<float2*>(park + g * D + 8 * (warp + NW * j) + 2 * c) =
              make_float2(om[j][mt][2 * e], om[j][mt][2 * e + 1]);
    }
  __syncthreads();
  // 2) code term, half 0 then half 1 (same softmax reference): rows d = 16r + 2mt (+1), cols n = 2c (+1)
#pragma unroll
  for (int hp = 0; hp < 2; ++hp) {
    if (half == hp) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 2 * c + e;
        if (n < G) {
          float* row = park + (h * G + n) * D + 16 * r;
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            row[2 * mt] += oc[mt][e];
            row[2 * mt + 1] += oc[mt][2 + e];
          }
        }
      }
    }
    __syncthreads();
  }
  // 3) write the split slot (natural-log LSE units for K3)
  const float LN2 = 0.6931471805599453f;
  for (int i = tid; i < HQ * D; i += NTHR) {
    const int g = i / D, d = i - g * D;
    const float l = red[g], bp = red[HQ + g], m = red[2 * HQ + g];
    const int64_t slot = (int64_t(b) * HQ + g) * a.slots + split;
    a.part_acc[slot * D + d] = l > 0.f ? park[g * D + d] - bp : 0.f;
    if (d == 0) {
      a.part_ml[slot * 2] = l > 0.f ? m * LN2 : NEG_INF;
      a.part_ml[slot * 2 + 1] = l;
    }
  }
}

}  // namespace fast

bool fast_supported(const tada_page_layout& L, int Hq) {
  // compiled geometries: 8 KV heads (the Llama-3 family) with 8/16/32/64 q heads
  if (L.head_dim != 128 || !(L.bits == 2 || L.bits == 4 || L.bits == 8) || L.heads != 8) return false;
  if (!(Hq == 8 || Hq == 16 || Hq == 32 || Hq == 64)) return false;
  const int tt = fast::make_plan(8, L.group_bytes, Hq, 16).stages >= 2
                     ? 16
                     : (fast::make_plan(8, L.group_bytes, Hq, 32).stages >= 2 ? 32 : 0);
  return tt != 0 && L.page_tokens % tt == 0;  // one stage cannot overlap load and compute
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

// One tensor map per region (means, codes, metas) covering BOTH sides, so a 32-token tile is three
// TMA copies.  Byte tensor dims (innermost first): byte within a 128-byte band, row (token) in the
// page, band, side, page.  The box [128 | 32 | bands | 2 | 1] lands in shared memory as
// [side][band][row][128 B]: every 128-byte line is one (band, row), so the 128B swizzle XORs the
// 16-byte chunk index with (row & 7) exactly like swz().
static bool encode_region5(CUtensorMap* m, const uint8_t* base, uint64_t row_bytes, uint64_t rows, uint64_t side_stride,
                           uint64_t page_bytes, uint32_t tt, uint64_t row_stride = 0, uint64_t row_extent = 0) {
  auto enc = get_encode();
  if (!enc) return false;
  // row_bytes: the bytes read per row; row_stride: the row pitch; row_extent: the bytes that exist from the base
  // (a view of fewer than 8 KV heads reads the missing ones as zeros: the box exceeds the tensor)
  const uint64_t nband = row_bytes / 128, nreal = (row_extent ? row_extent : row_bytes) / 128;
  const cuuint64_t dims[5] = {128, rows, nreal, 2, uint64_t(1) << 20};
  const cuuint64_t strides[4] = {row_stride ? row_stride : row_bytes, 128, side_stride, page_bytes};
  const cuuint32_t box[5] = {128, tt, uint32_t(nband), 2, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, const_cast<uint8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// metas: (byte in row, row, side, page); the box is 16 bytes wider than a row (zero fill) so that
// smem rows are trow = H*8 + 16 bytes apart (bank spread for the per-token loads)
static bool encode_meta(CUtensorMap* m, const uint8_t* base, uint64_t row_bytes, uint64_t rows, uint64_t side_stride,
                        uint64_t page_bytes, uint32_t box0, uint32_t tt, uint64_t row_stride = 0) {
  auto enc = get_encode();
  if (!enc) return false;
  const cuuint64_t dims[4] = {row_bytes, rows, 2, uint64_t(1) << 20};
  const cuuint64_t strides[3] = {row_stride ? row_stride : row_bytes, side_stride, page_bytes};
  const cuuint32_t box[4] = {box0, tt, 2, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int get_tma_maps(const AttnArgs& a, TmaMaps* out, int tt) {
  struct Key {
    const uint8_t* pool;
    int64_t page_bytes, off_codes;
    int bits, heads, page_tokens, tt, rh;
    bool operator==(const Key& o) const {
      return pool == o.pool && page_bytes == o.page_bytes && off_codes == o.off_codes && bits == o.bits &&
             heads == o.heads && page_tokens == o.page_tokens && tt == o.tt && rh == o.rh;
    }
  };
  struct Hash {
    size_t operator()(const Key& k) const {
      return std::hash<const void*>()(k.pool) ^ (std::hash<int64_t>()(k.page_bytes) << 1) ^ size_t(k.bits * 131 + k.heads);
    }
  };
  static std::mutex mu;
  static std::unordered_map<Key, TmaMaps, Hash> cache;
  const Key key{a.pool, a.L.page_bytes, a.L.off_codes[0], a.L.bits, a.L.heads, a.L.page_tokens, tt, a.kv_rh};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return TADA_OK;
  }
  TmaMaps m{};
  const tada_page_layout& L = a.L;
  const int real_heads = a.kv_rh - a.kv_h0 < L.heads ? a.kv_rh - a.kv_h0 : L.heads;  // < 8: zero-filled view
  const uint64_t side_stride = uint64_t(L.off_mean[1] - L.off_mean[0]);
  if (uint64_t(L.off_codes[1] - L.off_codes[0]) != side_stride || uint64_t(L.off_meta[1] - L.off_meta[0]) != side_stride)
    return fail(TADA_ERR_CONFIG, "page layout sides are not uniformly strided");
  if (!encode_region5(&m.m[0][0], a.pool + L.off_mean[0], uint64_t(L.head_dim) * 4, L.page_tokens, side_stride,
                      L.page_bytes, uint32_t(tt)) ||
      !encode_region5(&m.m[0][1], a.pool + L.off_codes[0], uint64_t(L.heads) * L.group_bytes, L.page_tokens,
                      side_stride, L.page_bytes, uint32_t(tt), uint64_t(a.kv_rh) * L.group_bytes,
                      uint64_t(real_heads) * L.group_bytes) ||
      !encode_meta(&m.m[0][2], a.pool + L.off_meta[0], uint64_t(real_heads) * 8, L.page_tokens, side_stride,
                   L.page_bytes, uint32_t(L.heads * 8 + 16), uint32_t(tt), uint64_t(a.kv_rh) * 8))
    return fail(TADA_ERR_CUDA, "cuTensorMapEncodeTiled failed for the decode-attention pool");
  if (cache.size() > 256) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return TADA_OK;
}

// Tile size per geometry: 16-token tiles (two CTAs per SM) where two stages fit in half the
// shared memory, else 32-token tiles (one CTA per SM).
static int tile_tokens(int bits, int hq) {
  const int gb = bits * 128 / 8;
  if (fast::make_plan(8, gb, hq, 16).stages >= 2) return 16;
  if (fast::make_plan(8, gb, hq, 32).stages >= 2) return 32;
  return 0;
}

template <int BITS, int HQ, int TT>
static int launch_fast_tt(const AttnArgs& a, int batch, cudaStream_t st) {
  constexpr fast::Plan pl = fast::make_plan(8, BITS * 128 / 8, HQ, TT);
  auto kern = fast::attn_fast_kernel<BITS, HQ, TT>;
  static std::atomic<uint64_t> smem_set{0};  // per instantiation, per device
  if (const int rc0 = ensure_smem(kern, pl.total, smem_set, "attn_fast"); rc0 != TADA_OK) return rc0;
  TmaMaps maps;
  const int rc = get_tma_maps(a, &maps, TT);
  if (rc != TADA_OK) return rc;
  kern<<<dim3(a.splits, batch), TT * 16, pl.total, st>>>(a, maps);
  return check_launch("decode_attn_fast");
}

template <int BITS, int HQ>
static int launch_fast_t(const AttnArgs& a, int batch, cudaStream_t st) {
  return tile_tokens(BITS, HQ) == 16 ? launch_fast_tt<BITS, HQ, 16>(a, batch, st)
                                     : launch_fast_tt<BITS, HQ, 32>(a, batch, st);
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

int fast_tile_tokens(const tada_page_layout& L, int Hq) { return tile_tokens(L.bits, Hq); }

}  // namespace tada
