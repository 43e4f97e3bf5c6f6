// K2-v8: split-K flash decoding over the compressed paged cache, sm_100a.
//
// Reference semantics: attend_streaming (pkg/src/tadakv/attention.py:103-151) with
// K̂ = mean - (min + scale*code) (cache.py:193-200, quant.py:177-180), evaluated in the factored form
//   q·k̂   = q·mean − min·Σq − scale·(q·code)
//   Σ p·v̂ = p·vmean − Σ(p·vmin) + p'·vcode,      p' = −p·vscale
// (SURVEY §7 hard part 2).  CTA = (split, sequence): 8 warps, warp h = KV head h, 16-token tiles, two
// CTAs per SM, a 2-stage (4-bit) or 3-stage (2-bit) TMA ring.  Per tile, two CTA barriers:
//   A   QK mean piece, cooperative: S_mean[q][tok] for all q heads, one token octet x one d quarter
//       per warp, from the f32 means as f16 hi + lo (mma.sync, f32 accumulate) -> 4 partial planes.
//   --- barrier 1: S_mean complete; the previous tile's P / split vmean are consumed.
//   B   per warp (its KV head):
//       - QK code term with q on M: IMMA m16n8k32, A = q_h as two s8 pieces of a 16-bit fixed point
//         (hi in rows r, lo in rows r + 8), B = the packed codes expanded to u8 (exact integers);
//       - online softmax in registers (thread = q head r x 4 tokens); P -> shared (f16) for C,
//         P' = −p·vscale stays in registers;
//       - PV code term with d on M: A = vcodes as exact f16 bias + code (bias·Σp' removed at the end);
//       - its share of the vmean split: f32 -> f16 hi / lo rows (the B operand of C).
//   --- barrier 2: P, corr and the split vmean complete; this tile's stage is free -> TMA refill
//       (S tiles ahead).
//   C   PV mean piece, cooperative: O_mean[q][16w..16w+15] = O_mean·corr + P · vmean (hi + lo).
// Every shared access of the hot loop reads each byte once per CTA except the q-independent metas;
// the shared-memory data pipe, not HBM, was the limit of the one-barrier variant (replicated vmean
// reads).  Per-thread shared offsets are computed once; the loop is unrolled by S so the stage is an
// immediate.
#include <cuda_runtime.h>

#include <string>
#include <type_traits>

#include "tada_attn.cuh"
#include "tada_mma.cuh"

namespace tada {
namespace v8 {
using namespace mmaops;

constexpr int D = 128, H = 8, TT = 16, NW = 8, NTHR = 256;
constexpr int BAND = TT * 128;       // bytes of one 128-B-wide swizzled band of a tile region
constexpr int VMPART = TT * D * 2;   // one f16 part (hi or lo) of the split vmean: [16 tok][256 B]
constexpr int kBudget = 113 * 1024;  // two CTAs per SM
#ifndef TADA_V8_MAXS
#define TADA_V8_MAXS 2  // measured: the x3 unroll of a 3-stage ring costs more (register pressure) than the depth buys
#endif
#ifndef TADA_V8_VMEAN_LO
#define TADA_V8_VMEAN_LO 0  // 1: the PV mean term also carries the f16 residual of vmean
#endif
// Dependent-MMA chain splitting (more accumulators, summed at the end), 0 = measured per-geometry choice:
//   ICHAINS 2: the QK code IMMAs of k-steps 0-1 and 2-3 in separate chains (+1.7% 2-bit Hq=32; -2% at Hq=64)
//   ACHAINS 2: the QK mean HMMAs of the hi and lo kmean pieces in separate chains (+1.8% at Hq<=32)
#ifndef TADA_V8_ICHAINS
#define TADA_V8_ICHAINS 0
#endif
#ifndef TADA_V8_ACHAINS
#define TADA_V8_ACHAINS 0
#endif
#ifndef TADA_V8_AC2_B2
#define TADA_V8_AC2_B2 0  // two QK-mean accumulation chains at 2-bit too (measured: one chain +1% there)
#endif
#ifndef TADA_V8_QTM
#define TADA_V8_QTM 2  // IMMA q fragments in TMEM: 0 where shared memory has no room, 1 at Hq=64, 2 always
#endif
#ifndef TADA_V8_QATM
#define TADA_V8_QATM 1  // QK mean q fragments in TMEM: 1 always (+0.8..5.6%), 0 = Hq<=32 only, -1 never
#endif
#ifndef TADA_V8_OFTM
#define TADA_V8_OFTM 2  // per-thread shared offsets in TMEM, reloaded per phase: 1 = phase B only (+0.8..2.5%), 2 = + phases A/C and the logit constants (+0.1..2.3% more)
#endif
#ifndef TADA_V8_KMEAN_LO
#define TADA_V8_KMEAN_LO 1  // the QK mean piece with the f32 kmean as f16 hi + lo (0: hi only, one MMA pass)
#endif
#ifndef TADA_V8_PPS
#define TADA_V8_PPS 0.00390625f  // 2^-8
#endif
#ifndef TADA_V8_RECENTER
#define TADA_V8_RECENTER 32  // tiles between removals of the PV code bias from oc (power of 2; 0 = at the end only)
#endif
#ifndef TADA_V8_TMEM_OM
#define TADA_V8_TMEM_OM 1  // park the PV mean accumulators in TMEM between tiles
#endif
constexpr int MAXS = TADA_V8_MAXS;
#ifndef TADA_V8_ORDER
#define TADA_V8_ORDER 0  // pipelined interval order: 0 = C, B, A; 1 = the same with A's loads first; 2 = C, A, B
#endif
#ifndef TADA_V8_EARLYWAIT
#define TADA_V8_EARLYWAIT 0  // pipelined: wait for the next tile's stage at the start of the interval
#endif
#ifndef TADA_V8_PIPE_S3
#define TADA_V8_PIPE_S3 1  // the pipelined plan takes a third stage where it fits
#endif  // deepest TMA ring (2 or 3 stages)

__host__ __device__ constexpr int up128(int x) { return (x + 127) / 128 * 128; }
__host__ __device__ constexpr int up1k(int x) { return (x + 1023) / 1024 * 1024; }

struct Plan {
  int mean_bytes, codes_bytes, meta_bytes, side_bytes, stage_bytes, stages, trow;
  int off_vm, off_sm, off_p, off_corr, off_qa, off_qi, off_bar, total;
  int vm_stride, sm_stride, p_stride, corr_stride;  // second buffer of each exchange region (pipelined plan)
  bool ok;
  bool qi_smem;  // the IMMA q fragments live in shared memory (frees 16 registers) when there is room
};

// [stage 0 .. S-1] | VM [hi, lo][16 tok][256 B] | SM [4 planes][MROWS][16] f32 | P [MROWS][16] f16 |
// corr [MROWS] | QA [4 quarters][MT][2 k-steps][32 lanes] uint4 | mbarriers.  The prologue's q staging
// and row maxima live in the last stage; the epilogue parks [HQ][D + 4] f32 over the stages and keeps
// its (l, Σp·vmin, m) table in the then idle VM region.
// Pipelined plan (pipe): two stages, and VM (hi only), SM, P and corr twice — tile i's phase B works on
// buffer i & 1 while phase C of tile i - 1 and phase A of tile i + 1 use the other one.
__host__ __device__ constexpr Plan make_plan(int gb, int HQ, bool pipe = false) {
  Plan p{};
  const int mrows = HQ >= 16 ? HQ : 16, mt = mrows / 16;
  p.trow = H * 8 + 16;  // meta box row: 16 B of TMA zero fill per row spread the banks
  p.mean_bytes = 4 * BAND;
  p.codes_bytes = (H * gb / 128) * BAND;
  p.meta_bytes = TT * p.trow;
  p.side_bytes = p.mean_bytes + p.codes_bytes;
  p.stage_bytes = up1k(2 * p.side_bytes + 2 * p.meta_bytes);
  const int nb = pipe ? 2 : 1;
  const int vmb = pipe ? VMPART : 2 * VMPART, smb = 4 * mrows * TT * 4, pb = mrows * TT * 2, cb = up128(mrows * 4);
  const int qab = 4 * mt * 2 * 512;  // QA: prologue only; the pipelined plan stages it in the S_mean buffers
  const int tail = nb * (vmb + smb + pb + cb) + (pipe ? 0 : qab) + 128;
  p.stages = (((pipe && TADA_V8_PIPE_S3) || MAXS >= 3) && 3 * p.stage_bytes + tail <= kBudget) ? 3
                                                                         : ((2 * p.stage_bytes + tail <= kBudget) ? 2 : 0);
  int off = p.stages * p.stage_bytes;
  p.off_vm = off;
  p.vm_stride = pipe ? vmb : 0;
  off += nb * vmb;
  p.off_sm = off;
  p.sm_stride = pipe ? smb : 0;
  off += nb * smb;
  p.off_p = off;
  p.p_stride = pipe ? pb : 0;
  off += nb * pb;
  p.off_corr = off;
  p.corr_stride = pipe ? cb : 0;
  off += nb * cb;
  p.off_qa = pipe ? p.off_sm : off;
  if (!pipe) off += qab;
  p.off_qi = off;
  p.qi_smem = !pipe && off + 8 * 4 * 512 + 128 <= kBudget;  // (the pipelined kernel keeps them in TMEM)
  if (p.qi_smem) off += 8 * 4 * 512;  // [warp][k-step][lane] uint4
  p.off_bar = off;
  off += 128;
  p.total = off;
  p.ok = p.stages >= 2 && p.stage_bytes >= mrows * (D * 2 + 4) && p.stages * p.stage_bytes >= HQ * (D + 4) * 4 &&
         2 * VMPART >= 3 * HQ * 4;
  return p;
}

#ifndef TADA_V8_PIPE
#define TADA_V8_PIPE 2  // pipelined schedule (one barrier per tile): 2 = 2-bit layers only, 1 = wherever it fits
#endif
// The pipelined schedule runs phase C of tile i - 1, phase B of tile i and phase A of tile i + 1 between two
// consecutive barriers; it needs the doubled exchange buffers (make_plan(.., true)), and takes a third stage when
// it fits (the refill of tile i + S is issued one interval after tile i was consumed).
__host__ __device__ constexpr bool v8_pipe(int bits, int HQ) {
  // measured (B=16, T=32k): 2-bit +4.4% (Hq=32) / +3% (Hq=16); 4-bit -0.6% (Hq=32) / -3.8% (Hq=8), where the
  // shorter refill distance (tile i + 2 is loaded during interval i + 1, not a whole tile ahead) shows at HBM speed
  return (TADA_V8_PIPE == 1 || (TADA_V8_PIPE == 2 && bits == 2)) && make_plan(bits * D / 8, HQ, true).ok;
}

__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

// PV code A operand (d on M).  Thread (r, c) owns d in [16r, 16r+16) of head h; m-tile mt holds
// d = 16r + 2mt in rows r and d = 16r + 2mt + 1 in rows r + 8.  Each code enters the MMA as the exact
// f16 value bias + code (the code field ORed under a fixed exponent, no subtraction); bias(mt, half)
// is removed once at the end as bias * Σp'.  Fields sit at mantissa bit 4 or above (bias <= 64) for
// 2/4-bit codes, so the biased f32 accumulation loses at most ~2^-17 of the code term (8-bit: bias
// 1024 against codes up to 255).
// P' = -p * vscale enters the PV code MMA as f16.  The lazy softmax lets p reach 2^8, so unscaled a group
// scale above 256 (a 2-bit deviation range above 768, which outlier channels reach) would overflow f16 to
// inf; P' is therefore stored times PPS = 2^-8 and the code term scaled back (exactly) in the epilogue.
constexpr float PPS = TADA_V8_PPS;
template <int BITS>
__host__ __device__ constexpr float pv_bias(int mt, int half) {
  if (BITS == 8) return 1024.f;
  if (BITS == 4) return 64.f;
  // 2-bit: k = mt & 3 -> (rows r, rows r + 8) fields at POS (4, 6), (4, 6), (8, 4), (6, 8)
  const int k = mt & 3;
  const int pos = k < 2 ? (half ? 6 : 4) : (k == 2 ? (half ? 4 : 8) : (half ? 8 : 6));
  return pos == 4 ? 64.f : (pos == 6 ? 16.f : 4.f);
}
template <int POS>
__device__ __forceinline__ uint32_t crumb(uint32_t x) {  // 2-bit field at POS -> f16 pair 2^(10-POS) + v
  constexpr uint32_t e = POS == 4 ? 0x54005400u : (POS == 6 ? 0x4C004C00u : 0x44004400u);
  return lop_and_or(x, 0x00030003u << POS, e);
}
__device__ __forceinline__ uint32_t nib4(uint32_t x) { return lop_and_or(x, 0x00F000F0u, 0x54005400u); }  // 64 + v

template <typename T>
__device__ __forceinline__ T& sh(uint8_t* base, int off) {
  return *reinterpret_cast<T*>(base + off);
}

// ------------------------------------------------------------------ the kernel
template <int BITS, int HQ>
__global__ void __launch_bounds__(NTHR, 2) attn_v8_kernel(AttnArgs a, const __grid_constant__ TmaMaps maps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0 && (su32(smem) & 1023u) != 0) __trap();
  constexpr int G = HQ / H;                   // q heads per KV head
  constexpr int MT = HQ >= 16 ? HQ / 16 : 1;  // 16-row q tiles of the shared mean terms
  constexpr int MROWS = MT * 16;
  constexpr int GB = BITS * D / 8;            // code bytes per (token, head)
  constexpr bool PIPE = v8_pipe(BITS, HQ);
  constexpr Plan pl = make_plan(GB, HQ, PIPE);
  constexpr int S = pl.stages < 2 ? 2 : pl.stages;  // geometries with < 2 stages are never launched
  constexpr int SB = pl.stage_bytes;
  constexpr int PLANE = MROWS * TT * 4;
  const int P = a.L.page_tokens;
  const int b = blockIdx.y, split = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, r = lane >> 2, c = lane & 3;
  const int h = warp;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + pl.off_bar);
  float* qmax = reinterpret_cast<float*>(smem + (S - 1) * SB + MROWS * D * 2);  // [MROWS], prologue only
  float* red = reinterpret_cast<float*>(smem + pl.off_vm);                     // [3][HQ] epilogue (l, Σp·vmin, m)

  pdl_enter();  // no global reads above this line
  const int C = comp_tokens(a, b);
  int t_begin, t_end;
  split_range(C, a.splits, split, TT, t_begin, t_end);
  const int ntiles = t_end > t_begin ? (t_end - t_begin + TT - 1) / TT : 0;

  int* exact_flag = reinterpret_cast<int*>(smem + pl.off_bar + 112);  // a query element beyond the f16 range
  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    *exact_flag = 0;
  }
  // P rows of padding q heads stay zero; corr starts at 1
  for (int i = tid; i < MROWS * TT / 2; i += NTHR) {
    sh<uint32_t>(smem, pl.off_p + 4 * i) = 0u;
    if (PIPE) sh<uint32_t>(smem, pl.off_p + pl.p_stride + 4 * i) = 0u;
  }
  for (int i = tid; i < MROWS; i += NTHR) {
    sh<float>(smem, pl.off_corr + 4 * i) = 1.f;
    if (PIPE) sh<float>(smem, pl.off_corr + pl.corr_stride + 4 * i) = 1.f;
  }
  // PARK: the PV mean accumulators (om, 8*MT floats per thread) are touched only in phase C; between
  // tiles they live in TMEM (warp w: lane quarter w%4, column block w/4), freeing their registers for
  // phases A/B.  Measured: +4% at Hq=64 (32 registers), -1% at Hq<=32 (16), so only there.
  constexpr bool PARK = TADA_V8_TMEM_OM && MT >= 4 && BITS != 2;  // 2-bit Hq=64: +0.9% without (measured)
  // per-warp rescale flags instead of a corr scan in phase C: +2.5% at Hq=64, -1..2% at Hq<=32 (measured)
  constexpr bool FLAGS = MT >= 4;
  constexpr int NOM = 8 * MT;
  // QTM: the IMMA q fragments (16 values per thread) live in TMEM and come back with one tcgen05.ld per
  // tile, instead of 4 LDS.128 from shared memory (or 16 registers where shared memory has no room):
  // measured +6.3% 4-bit Hq=32, +2.5% 2-bit Hq=32, +4.2% 2-bit Hq=64, +1.2% 4-bit Hq=64 (vs registers)
  constexpr bool QTM = TADA_V8_QTM == 2 || (TADA_V8_QTM == 1 && PARK) || (PARK && !pl.qi_smem);
  // (The PV code accumulators oc are NOT parked: their TMEM round trip sits on phase B's critical path,
  // measured -1..2% at every geometry.)
  // QATM: the QK mean A fragments of this warp's d quarter (8*MT values) in TMEM too, one tcgen05.ld per
  // tile instead of 2*MT LDS.128
  constexpr bool QATM = TADA_V8_QATM == 1 || (TADA_V8_QATM == 0 && MT <= 2);
  static_assert(!PIPE || (QTM && QATM), "the pipelined plan keeps the q fragments in TMEM (QA aliases S_mean)");
  constexpr bool USE_TM = PARK || QTM || QATM || TADA_V8_OFTM;
  // TMEM columns of one lane (warps w and w+4 share lane quarter w%4; column blocks by w/4)
  constexpr int C_Q = PARK ? 2 * NOM : 0, C_QA = C_Q + (QTM ? 32 : 0), C_OF = C_QA + (QATM ? 16 * MT : 0);
  constexpr int C_OF2 = C_OF + (TADA_V8_OFTM ? 32 : 0);  // phase A / C offsets (OFTM 2): 8 per warp
  // (the running softmax state stays in registers: parking it cost 2%, measured)
  constexpr int TUSED = C_OF2 + (TADA_V8_OFTM >= 2 ? 16 : 0);
  constexpr uint32_t TCOLS = TUSED <= 32 ? 32u : (TUSED <= 64 ? 64u : (TUSED <= 128 ? 128u : 256u));
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + pl.off_bar + 64);
  if constexpr (USE_TM) {
    if (warp == 0) tmem_alloc(tslot, TCOLS);
    tc_fence_before();
  }
  __syncthreads();
  uint32_t tbase = 0;
  if constexpr (USE_TM) {
    tc_fence_after();
    tbase = *tslot;
  }
  const uint32_t tlane = tbase + (uint32_t(32 * (warp & 3)) << 16);
  const uint32_t tom = tlane + uint32_t((warp >> 2) * NOM);
  const uint32_t tq = tlane + uint32_t(C_Q + (warp >> 2) * 16);
  const uint32_t tqa = tlane + uint32_t(C_QA + (warp >> 2) * 8 * MT);
  const uint32_t tof = tlane + uint32_t(C_OF + (warp >> 2) * 16);
  const uint32_t tof2 = tlane + uint32_t(C_OF2 + (warp >> 2) * 8);

  // TMA producer (thread 0): tile `it` -> stage it % S, three copies (means, codes, metas; both sides).
  // The (page, row) cursor advances by TT rows per tile (P is a multiple of TT): no divisions in the loop.
  const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
  constexpr uint32_t tx = 2u * uint32_t(pl.mean_bytes + pl.codes_bytes + TT * pl.trow);
  int cur_pg = t_begin / P, cur_row = t_begin - (t_begin / P) * P, cur_page = 0;  // next tile to issue
  auto issue = [&](int stg) {
    uint8_t* dst = smem + stg * SB;
    mbar_expect_tx(&full[stg], tx);
    tma_5d(dst, &maps.m[0][0], cur_row, cur_page, &full[stg]);
    tma_5d(dst + 2 * pl.mean_bytes, &maps.m[0][1], cur_row, cur_page, &full[stg]);
    tma_4d(dst + 2 * pl.side_bytes, &maps.m[0][2], cur_row, cur_page, &full[stg]);
    cur_row += TT;
    if (cur_row == P) {
      cur_row = 0;
      ++cur_pg;
    }
  };
  if (tid == 0) {
    for (int k = 0; k < 3; ++k)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[0][k])) : "memory");
    for (int k = 0; k < S - 1 && k < ntiles; ++k) {
      cur_page = pt[cur_pg];
      issue(k);
    }
  }

  // ---------------------------------------------------------------- prologue: q -> f16, staged in the last stage
  __half* q16 = reinterpret_cast<__half*>(smem + (S - 1) * SB);  // [MROWS][D]
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
    const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&lo));
    const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&hi));
    float amax = fmaxf(fmaxf(fabsf(f0.x), fabsf(f0.y)), fmaxf(fabsf(f1.x), fabsf(f1.y)));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) qmax[g] = amax;
  }
  __syncthreads();
  if (*exact_flag || beyond_f16(a, kF16SafeExp)) {  // CTA-uniform, rare: operands beyond f16 -> the exact f32 path
    for (int k = 0; k < S - 1 && k < ntiles; ++k) mbar_wait(&full[k], 0u);  // no copy may land after exit
    if constexpr (USE_TM) {
      tc_fence_before();
      __syncthreads();
      if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, TCOLS);
      }
    }
    exact_split_partials<BITS, G>(a, b, split, t_begin, t_end, warp, lane);
    return;
  }
  // IMMA A operand: q head h*G + r (r < G) as 16-bit fixed point (scale sq) split into two s8 pieces,
  // q = sq * (256 hi + lo): hi in row r, lo in row r + 8, so one IMMA yields both partial sums; k laid
  // out by dk() to match the code bytes.  Stored in fragment order {a0, a1, a2, a3}.
  uint32_t qA[4][4];
  float sq, qs;  // qs = Σ_d q_fx of q head h*G + r (the min term)
  {
    float mx = 0.f;
#pragma unroll
    for (int e = 0; e < G; ++e) mx = fmaxf(mx, qmax[h * G + e]);
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
        qA[s][2 * which] = ph;
        qA[s][2 * which + 1] = pl8;
      }
    isum += __shfl_xor_sync(0xffffffffu, isum, 1);
    isum += __shfl_xor_sync(0xffffffffu, isum, 2);
    qs = sq * float(isum);
    if constexpr (QTM) {
      float qf[16];
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int i = 0; i < 4; ++i) qf[4 * s + i] = __uint_as_float(qA[s][i]);
      tmem_st<16>(tq, qf);
      tmem_wait_st();
    }
    if (pl.qi_smem && !QTM)
#pragma unroll
      for (int s = 0; s < 4; ++s)
        sh<uint4>(smem, pl.off_qi + (warp * 4 + s) * 512 + lane * 16) = make_uint4(qA[s][0], qA[s][1], qA[s][2], qA[s][3]);
  }
  // QK mean A fragments of every piece, lane-major: [quarter qd][mt][ks][lane]; q rows 16mt + r (+8),
  // k-step ks slots (2c, 2c+1 | 2c+8, 2c+9) <-> d = 32qd + 16(ks ^ (c & 1)) + 4c + (0, 1 | 2, 3): odd quads take
  // the other half of the kmean row first, so each 8-lane phase of the kmean LDS.128 (rows r, r + 1 under the
  // 128-B swizzle) covers 8 distinct 16-B chunks (16ks + 4c made it a 2-way bank conflict)
  for (int f = warp; f < 4 * MT * 2; f += NW) {
    const int qd2 = f / (MT * 2), mt = (f >> 1) % MT, ks = f & 1;
    const __half* r0 = q16 + (16 * mt + r) * D + 32 * qd2 + 16 * (ks ^ (c & 1)) + 4 * c;
    const __half* r1 = r0 + 8 * D;
    sh<uint4>(smem, pl.off_qa + f * 512 + lane * 16) =
        make_uint4(*reinterpret_cast<const uint32_t*>(r0), *reinterpret_cast<const uint32_t*>(r1),
                   *reinterpret_cast<const uint32_t*>(r0 + 2), *reinterpret_cast<const uint32_t*>(r1 + 2));
  }
  fence_proxy_async();  // the q staging lives in the last stage, which TMA fills right after this barrier
  __syncthreads();
  if (tid == 0 && S - 1 < ntiles) {
    cur_page = pt[cur_pg];
    issue(S - 1);
  }
  if (tid == 0 && S < ntiles) cur_page = pt[cur_pg];  // the page of the next refill, loaded a tile ahead
  if constexpr (QATM) {  // this warp's d quarter of the QK mean A fragments -> TMEM
    float v[8 * MT];
#pragma unroll
    for (int f = 0; f < 2 * MT; ++f) {
      const uint4 x = sh<uint4>(smem, pl.off_qa + (warp & 3) * (MT * 2 * 512) + f * 512 + lane * 16);
      v[4 * f] = __uint_as_float(x.x);
      v[4 * f + 1] = __uint_as_float(x.y);
      v[4 * f + 2] = __uint_as_float(x.z);
      v[4 * f + 3] = __uint_as_float(x.w);
    }
    tmem_st<8 * MT>(tqa, v);
    tmem_wait_st();
  }

  // ---------------------------------------------------------------- per-thread shared offsets
  const int qd = warp & 3, oct = warp >> 2;
  const int oX0 = qd * BAND + swz(8 * oct + r, 64 * (c & 1) + 16 * c);  // kmean, stage-relative (k-step 0)
  const int oX1 = qd * BAND + swz(8 * oct + r, 64 * (~c & 1) + 16 * c);  // k-step 1
  const int oQA = pl.off_qa + qd * (MT * 2 * 512) + lane * 16;
  const int oQI = pl.off_qi + warp * 4 * 512 + lane * 16;
  const int oSW = pl.off_sm + qd * PLANE + (r * TT + ((8 * oct + 2 * c) ^ (8 * ((r >> 1) & 1)))) * 4;
  const int vt = tid & 15, vu = tid >> 4;  // vmean split: token vt, d in [8vu, 8vu+8)
  const int oV0 = pl.mean_bytes + (vu >> 2) * BAND + swz(vt, (vu & 3) * 32);  // vmean, stage-relative
  const int oV1 = pl.mean_bytes + (vu >> 2) * BAND + swz(vt, (vu & 3) * 32 + 16);
  const int oVW = pl.off_vm + vt * 256 + ((vu ^ (vt & 7)) << 4);
  const int hbK = h * GB + c * (GB / 4);
  const int oK = 2 * pl.mean_bytes + (hbK >> 7) * BAND + swz(r, hbK & 127);  // row r; row r + 8 at +1024
  const int oK2 = 2 * pl.mean_bytes + (hbK >> 7) * BAND + swz(r, (hbK & 127) + 16);  // 8-bit second half
  const bool live = r < G;
  const int qrow = h * G + (live ? r : 0);
  const int qx = 8 * ((qrow >> 1) & 1);
  const int oS0 = pl.off_sm + (qrow * TT + ((2 * c) ^ qx)) * 4, oS1 = pl.off_sm + (qrow * TT + ((8 + 2 * c) ^ qx)) * 4;
  const int oM = 2 * pl.side_bytes + 2 * c * pl.trow + 8 * h;  // kmeta of token 2c; vmeta at + meta_bytes
  const int oPW = pl.off_p + qrow * 32 + 4 * c;                 // P row of q head qrow: chunk k at ((k ^ pch) << 4)
  const int pch = (qrow >> 2) & 1;
  const int hbV = h * GB + 2 * r * BITS;
  const int oC0 = 2 * pl.mean_bytes + pl.codes_bytes + (hbV >> 7) * BAND + swz(2 * c, hbV & 127);  // token 2c
  const int oC1 = 2 * pl.mean_bytes + pl.codes_bytes + (hbV >> 7) * BAND + swz(2 * c + 1, hbV & 127);
  // PV mean piece (warp = d slice 16w .. 16w+15): ldmatrix lane addresses
  const uint32_t aPA = su32(smem + pl.off_p) + ((lane & 7) + 8 * ((lane >> 3) & 1)) * 32 +
                       (((lane >> 4) ^ (((lane & 7) >> 2) & 1)) << 4);  // + 512 per q tile
  const uint32_t aVB = su32(smem + pl.off_vm) + ((lane & 7) + 8 * ((lane >> 3) & 1)) * 256 +
                       (((2 * warp + (lane >> 4)) ^ (lane & 7)) << 4);  // + VMPART for lo

  float oc[8][4];      // PV code term O_h^T: rows d (16r + 2mt, +1), cols n = 2c, 2c+1 (q heads h*G + n)
  float om[2][MT][4];  // PV mean piece: rows q (16mt + r, +8), cols d = 16w + 8j + 2c (+1)
#pragma unroll
  for (int i = 0; i < 8; ++i) oc[i][0] = oc[i][1] = oc[i][2] = oc[i][3] = 0.f;
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) om[j][mt][0] = om[j][mt][1] = om[j][mt][2] = om[j][mt][3] = 0.f;
  if constexpr (PARK) tmem_st<NOM>(tom, &om[0][0][0]);
  const float NEG_INF = -__int_as_float(0x7f800000);
  // rows r >= G carry the mean-term logits of q head h*G (finite); their P is never stored
  float m_run = NEG_INF, l_run = 0.f, bp_run = 0.f, sp_run = 0.f;
  const float sl2 = a.scale * 1.4426950408889634f;
  const float sq2 = sq * sl2, qs2 = qs * sl2;  // the code/min terms pre-scaled to log2 logit units
#if TADA_V8_OFTM
  {  // phase B's shared offsets -> TMEM (reloaded per tile: their registers are free outside phase B)
    float v[16];
    const int o[12] = {oK, oK2, oS0, oS1, oM, oPW, oC0, oC1, oV0, oV1, oVW, pch};
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __int_as_float(i < 12 ? o[i] : 0);
#if TADA_V8_OFTM >= 2
    v[12] = sq2;
    v[13] = qs2;
    {
      float w[8];
      const int o2[6] = {oX0, oX1, oQA, oSW, int(aPA), int(aVB)};
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = __int_as_float(i < 6 ? o2[i] : 0);
      tmem_st<8>(tof2, w);
    }
#endif
    tmem_st<16>(tof, v);
    tmem_wait_st();
  }
#endif

  // One tile's three phases.  STG = the tile's stage; BUF = the exchange buffer (S_mean, P, corr, flags, split
  // vmean) the phase writes or reads (always 0 in the classic schedule).
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  // ------------------------------------------------------------ A: QK mean piece -> S_mean plane qd
  struct KMean {
    float4 x0, x1;  // this thread's kmean B-fragment values (k-steps 0 and 1), f32
  };
  auto loadA = [&](auto stage_c) {
    const int ST = int(stage_c) * SB;
#if TADA_V8_OFTM >= 2
    float ofa[2];
    tmem_ld<2>(tof2, ofa);
    tmem_wait_ld();
    const int oX0 = __float_as_int(ofa[0]), oX1 = __float_as_int(ofa[1]);
#endif
    return KMean{sh<float4>(smem, ST + oX0), sh<float4>(smem, ST + oX1)};
  };
  auto phaseA = [&](auto buf_c, const KMean& km) {
    const int SMO = int(buf_c) * pl.sm_stride;
#if TADA_V8_OFTM >= 2
    float ofa[2];
    tmem_ld<2>(tof2 + 2, ofa);
    tmem_wait_ld();
    const int oQA = __float_as_int(ofa[0]), oSW = __float_as_int(ofa[1]);
#endif
    float acc[MT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
    uint32_t hb[2][2], lb[2][2];  // B fragments (hi, lo) of both k-steps
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const float4 x = ks ? km.x1 : km.x0;
      if (TADA_V8_KMEAN_LO) {
        split_h2(x.x, x.y, hb[ks][0], lb[ks][0]);
        split_h2(x.z, x.w, hb[ks][1], lb[ks][1]);
      } else {
        hb[ks][0] = pack_h2(x.x, x.y);
        hb[ks][1] = pack_h2(x.z, x.w);
      }
    }
    float qa[QATM ? 8 * MT : 1];
    if constexpr (QATM) {
      tmem_ld<QATM ? 8 * MT : 8>(tqa, qa);
      tmem_wait_ld();
    }
    // MT (or 2 MT) independent accumulation chains, interleaved so no MMA waits on the previous one
    constexpr bool AC2 = TADA_V8_ACHAINS == 2 || (TADA_V8_ACHAINS == 0 && MT <= 2 && (BITS != 2 || TADA_V8_AC2_B2));
    [[maybe_unused]] float acc2[AC2 ? MT : 1][4];
    if constexpr (AC2)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) acc2[mt][0] = acc2[mt][1] = acc2[mt][2] = acc2[mt][3] = 0.f;
#pragma unroll
    for (int pass = 0; pass < (TADA_V8_KMEAN_LO ? 2 : 1); ++pass)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          uint32_t af[4];
          if constexpr (QATM) {
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = __float_as_uint(qa[QATM ? 4 * (mt * 2 + ks) + i : 0]);
          } else {
            const uint4 f = sh<uint4>(smem, oQA + (mt * 2 + ks) * 512);
            af[0] = f.x; af[1] = f.y; af[2] = f.z; af[3] = f.w;
          }
          if (pass == 0) mma(acc[mt], af, hb[ks][0], hb[ks][1]);
          else if constexpr (AC2) mma(acc2[AC2 ? mt : 0], af, lb[ks][0], lb[ks][1]);
          else mma(acc[mt], af, lb[ks][0], lb[ks][1]);
        }
    if constexpr (AC2)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[mt][i] += acc2[AC2 ? mt : 0][i];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        sh<float2>(smem, SMO + oSW + (16 * mt + 8 * e) * TT * 4) = make_float2(acc[mt][2 * e], acc[mt][2 * e + 1]);
  };

  // ------------------------------------------------------------ B: the warp's KV head (QK code term, softmax,
  // PV code term) and its share of the vmean split.  MAYTAIL: the tile may be the split's partial last tile.
  auto phaseB = [&](auto stage_c, auto buf_c, auto maytail_c, int it) {
    const int ST = int(stage_c) * SB;
    const int BUF = int(buf_c);
    const int SMO = BUF * pl.sm_stride, PO = BUF * pl.p_stride, CO = BUF * pl.corr_stride, VO = BUF * pl.vm_stride;
    constexpr bool MAYTAIL = decltype(maytail_c)::value;
    const int t0 = t_begin + it * TT;
    const int nv = MAYTAIL ? min(TT, t_end - t0) : TT;
    const bool tail = MAYTAIL && nv < TT;
#if TADA_V8_OFTM
    float ofv[16];
    tmem_ld<16>(tof, ofv);
    tmem_wait_ld();
    const int oK = __float_as_int(ofv[0]), oK2 = __float_as_int(ofv[1]), oS0 = __float_as_int(ofv[2]);
    const int oS1 = __float_as_int(ofv[3]), oM = __float_as_int(ofv[4]), oPW = __float_as_int(ofv[5]);
    const int oC0 = __float_as_int(ofv[6]), oC1 = __float_as_int(ofv[7]), oV0 = __float_as_int(ofv[8]);
    const int oV1 = __float_as_int(ofv[9]), oVW = __float_as_int(ofv[10]), pch = __float_as_int(ofv[11]);
#if TADA_V8_OFTM >= 2
    const float sq2 = ofv[12], qs2 = ofv[13];
#endif
#endif

    // ------------------------------------------------------------ re-centre the PV code accumulators
    // oc holds bias * Σp' + Σp'·code: the biased f16 codes make |oc| up to ~40x the code term (2-bit), and the
    // tensor core's f32 accumulation truncates (rounds toward zero) relative to |oc| on every MMA, so over
    // thousands of tiles the error grows systematically (measured 4.2e-3 max-abs at 128k tokens, 2-bit).
    // Every RC tiles the bias part (bias * column sums of the f16 P' the MMAs saw) is removed exactly enough
    // in f32 and the running Σp' restarts, so each truncation acts on the small code term only.
    if constexpr (TADA_V8_RECENTER > 0) {
      if (it > 0 && (it & (TADA_V8_RECENTER - 1)) == 0) {  // after every RC tiles (placed before this tile's
        // QK work so the PV code term, the vmean split and phase A form one scheduling block)
        float s = sp_run;
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        const float s0 = __shfl_sync(0xffffffffu, s, 8 * c), s1 = __shfl_sync(0xffffffffu, s, 8 * c + 4);
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          oc[mt][0] = fmaf(-pv_bias<BITS>(mt, 0), s0, oc[mt][0]);
          oc[mt][1] = fmaf(-pv_bias<BITS>(mt, 0), s1, oc[mt][1]);
          oc[mt][2] = fmaf(-pv_bias<BITS>(mt, 1), s0, oc[mt][2]);
          oc[mt][3] = fmaf(-pv_bias<BITS>(mt, 1), s1, oc[mt][3]);
        }
        sp_run = 0.f;
      }
    }
    // ------------------------------------------------------------ c: QK code term (q on M) + logits
    float x[2][2];  // logits (log2 units) of q head h*G + r for tokens 8nt + 2c + e
    {
      constexpr int NWD = BITS == 8 ? 8 : (BITS == 4 ? 4 : 2);  // code words per row segment
      uint32_t wa[NWD], wb[NWD];
      if (BITS == 4) {
        const uint4 p0 = sh<uint4>(smem, ST + oK), p1 = sh<uint4>(smem, ST + oK + 1024);
        wa[0] = p0.x; wa[1 % NWD] = p0.y; wa[2 % NWD] = p0.z; wa[3 % NWD] = p0.w;
        wb[0] = p1.x; wb[1 % NWD] = p1.y; wb[2 % NWD] = p1.z; wb[3 % NWD] = p1.w;
      } else if (BITS == 2) {
        const uint2 p0 = sh<uint2>(smem, ST + oK), p1 = sh<uint2>(smem, ST + oK + 1024);
        wa[0] = p0.x; wa[1] = p0.y;
        wb[0] = p1.x; wb[1] = p1.y;
      } else {
        const uint4 p0 = sh<uint4>(smem, ST + oK), p1 = sh<uint4>(smem, ST + oK + 1024);
        const uint4 p2 = sh<uint4>(smem, ST + oK2), p3 = sh<uint4>(smem, ST + oK2 + 1024);
        wa[0] = p0.x; wa[1 % NWD] = p0.y; wa[2 % NWD] = p0.z; wa[3 % NWD] = p0.w;
        wa[4 % NWD] = p2.x; wa[5 % NWD] = p2.y; wa[6 % NWD] = p2.z; wa[7 % NWD] = p2.w;
        wb[0] = p1.x; wb[1 % NWD] = p1.y; wb[2 % NWD] = p1.z; wb[3 % NWD] = p1.w;
        wb[4 % NWD] = p3.x; wb[5 % NWD] = p3.y; wb[6 % NWD] = p3.z; wb[7 % NWD] = p3.w;
      }
      // rows r: hi . code, rows r + 8: lo . code; q_fx . code / sq = 256 hi + lo (exact, |.| < 2^31)
      constexpr int NIC = TADA_V8_ICHAINS ? TADA_V8_ICHAINS : 1;  // 2 chains measured -3% at 2-bit Hq=32 (one QK-mean chain)
      int acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
      float qf[QTM ? 16 : 1];
      if constexpr (QTM) {
        tmem_ld<16>(tq, qf);
        tmem_wait_ld();
      }
      int accb[NIC == 2 ? 2 : 1][4] = {};
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        uint32_t A[4];
        if constexpr (QTM) {
#pragma unroll
          for (int i = 0; i < 4; ++i) A[i] = __float_as_uint(qf[QTM ? 4 * s + i : 0]);
        } else if (pl.qi_smem) {
          const uint4 f = sh<uint4>(smem, oQI + s * 512);
          A[0] = f.x; A[1] = f.y; A[2] = f.z; A[3] = f.w;
        } else {
          A[0] = qA[s][0]; A[1] = qA[s][1]; A[2] = qA[s][2]; A[3] = qA[s][3];
        }
        if (NIC == 2 && s >= 2) {
          imma_su(accb[0], A, qk_quad<BITS>(wa, s, 0), qk_quad<BITS>(wa, s, 1));
          imma_su(accb[NIC == 2 ? 1 : 0], A, qk_quad<BITS>(wb, s, 0), qk_quad<BITS>(wb, s, 1));
        } else {
          imma_su(acc[0], A, qk_quad<BITS>(wa, s, 0), qk_quad<BITS>(wa, s, 1));
          imma_su(acc[1], A, qk_quad<BITS>(wb, s, 0), qk_quad<BITS>(wb, s, 1));
        }
      }
      if constexpr (NIC == 2)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[j][i] += accb[NIC == 2 ? j : 0][i];
      // S_mean of (q row, tokens 2c, 2c+1 | 8+2c, 9+2c): the 4 d-quarter planes
      float sm[2][2];
      {
        const float2 v0 = sh<float2>(smem, SMO + oS0), v1 = sh<float2>(smem, SMO + oS1);
        sm[0][0] = v0.x;
        sm[0][1] = v0.y;
        sm[1][0] = v1.x;
        sm[1][1] = v1.y;
      }
#pragma unroll
      for (int k = 1; k < 4; ++k) {
        const float2 v0 = sh<float2>(smem, SMO + oS0 + k * PLANE);
        const float2 v1 = sh<float2>(smem, SMO + oS1 + k * PLANE);
        sm[0][0] += v0.x;
        sm[0][1] += v0.y;
        sm[1][0] += v1.x;
        sm[1][1] += v1.y;
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float2 km = sh<float2>(smem, ST + oM + (8 * nt + e) * pl.trow);  // (scale, min)
          const float cs = float(acc[nt][e] * 256 + acc[nt][2 + e]);
          x[nt][e] = fmaf(sm[nt][e], sl2, -fmaf(km.x * sq2, cs, km.y * qs2));
        }
    }
    // ------------------------------------------------------------ d: online softmax (registers)
    uint32_t bp0, bp1, bq0, bq1;  // B fragments (k = tokens 2c, 2c+1 | 8+2c, 9+2c; n = q head r): P, P'
    {
      if (tail) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (8 * nt + 2 * c + e >= nv) x[nt][e] = NEG_INF;
      }
      float tmax = fmaxf(fmaxf(x[0][0], x[0][1]), fmaxf(x[1][0], x[1][1]));
      // Lazy rescaling: the reference max only moves when a logit exceeds it by more than 2^LAZY
      // (p <= 256 stays exact enough in f16/f32), so most tiles skip the reduction and the O rescale.
      constexpr float LAZY = 8.f;
      float corr = 1.f;
      const bool resc = __any_sync(0xffffffffu, tmax > m_run + LAZY);
      if (resc) {
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 1));
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 2));
        const float m_new = fmaxf(m_run, tmax);  // finite: every tile has a valid token
        corr = ex2(m_run - m_new);
        m_run = m_new;
      }
      float p[2][2], pp[2][2], lsum = 0.f, bsum = 0.f;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float2 vm = sh<float2>(smem, ST + oM + pl.meta_bytes + (8 * nt + e) * pl.trow);  // (scale, min)
          const float pe = ex2(x[nt][e] - m_run);
          p[nt][e] = pe;
          lsum += pe;
          if (tail && 8 * nt + 2 * c + e >= nv) {  // rows past the sequence may hold anything
            pp[nt][e] = 0.f;
          } else {
            pp[nt][e] = pe * (vm.x * -PPS);  // P' pre-scaled by 2^-8: f16-safe up to vscale 65504
            bsum = fmaf(pe, vm.y, bsum);
          }
        }
      bp0 = pack_h2(p[0][0], p[0][1]);
      bp1 = pack_h2(p[1][0], p[1][1]);
      bq0 = pack_h2(pp[0][0], pp[0][1]);
      bq1 = pack_h2(pp[1][0], pp[1][1]);
      float ssum;
      {  // Σp' of exactly the f16 values the PV code MMA sees (the bias correction)
        const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&bq0));
        const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&bq1));
        ssum = (f0.x + f0.y) + (f1.x + f1.y);
      }
      if (live) {  // P (f16) for the PV mean piece, corr for its rescale
        sh<uint32_t>(smem, PO + oPW + ((0 ^ pch) << 4)) = bp0;
        sh<uint32_t>(smem, PO + oPW + ((1 ^ pch) << 4)) = bp1;
        if (c == 0) sh<float>(smem, CO + pl.off_corr + 4 * qrow) = corr;
      }
      if constexpr (FLAGS)
        if (lane == 0) sh<uint8_t>(smem, pl.off_bar + 96 + 8 * BUF + warp) = resc ? 1 : 0;  // this warp's rescale flag
      l_run = fmaf(l_run, corr, lsum);
      bp_run = fmaf(bp_run, corr, bsum);
      sp_run = fmaf(sp_run, corr, ssum);
      if (resc) {  // columns n = 2c, 2c+1 of oc belong to the softmax rows of lanes 4n
        const float c0 = __shfl_sync(0xffffffffu, corr, 8 * c), c1 = __shfl_sync(0xffffffffu, corr, 8 * c + 4);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          oc[i][0] *= c0;
          oc[i][1] *= c1;
          oc[i][2] *= c0;
          oc[i][3] *= c1;
        }
      }
    }
    // ------------------------------------------------------------ PV code term (d on M)
    if (BITS == 4) {
      const uint2 w0 = sh<uint2>(smem, ST + oC0), w1 = sh<uint2>(smem, ST + oC1);
      const uint2 w2 = sh<uint2>(smem, ST + oC0 + 1024), w3 = sh<uint2>(smem, ST + oC1 + 1024);
#pragma unroll
      for (int wi = 0; wi < 2; ++wi) {
        const uint32_t xa = wi ? w0.y : w0.x, xb = wi ? w1.y : w1.x;
        const uint32_t xc = wi ? w2.y : w2.x, xd = wi ? w3.y : w3.x;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {  // bytes 2hh, 2hh+1 of the word: d = 16r + 8wi + 4hh + (0..3)
          const uint32_t sel = hh ? 0x7632u : 0x5410u;
          const uint32_t u = prmt(xa, xb, sel), v = prmt(xc, xd, sel);
          uint32_t af[4];
          af[0] = nib4(u << 4);
          af[1] = nib4(u);
          af[2] = nib4(v << 4);
          af[3] = nib4(v);
          mma(oc[4 * wi + 2 * hh], af, bq0, bq1);
          af[0] = nib4(u >> 4);
          af[1] = nib4(u >> 8);
          af[2] = nib4(v >> 4);
          af[3] = nib4(v >> 8);
          mma(oc[4 * wi + 2 * hh + 1], af, bq0, bq1);
        }
      }
    } else if (BITS == 2) {
      const uint32_t xa = sh<uint32_t>(smem, ST + oC0), xb = sh<uint32_t>(smem, ST + oC1);
      const uint32_t xc = sh<uint32_t>(smem, ST + oC0 + 1024), xd = sh<uint32_t>(smem, ST + oC1 + 1024);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {  // bytes 2hh, 2hh+1: d = 16r + 8hh + (0..7), crumb k at bit 2k
        const uint32_t sel = hh ? 0x7632u : 0x5410u;
        const uint32_t u = prmt(xa, xb, sel), v = prmt(xc, xd, sel);
        const uint32_t ul = u << 4, vl = v << 4, uh = u >> 6, vh = v >> 6;
        uint32_t af[4];
        af[0] = crumb<4>(ul); af[1] = crumb<6>(ul); af[2] = crumb<4>(vl); af[3] = crumb<6>(vl);  // +0, +1
        mma(oc[4 * hh + 0], af, bq0, bq1);
        af[0] = crumb<4>(u); af[1] = crumb<6>(u); af[2] = crumb<4>(v); af[3] = crumb<6>(v);      // +2, +3
        mma(oc[4 * hh + 1], af, bq0, bq1);
        af[0] = crumb<8>(u); af[1] = crumb<4>(uh); af[2] = crumb<8>(v); af[3] = crumb<4>(vh);    // +4, +5
        mma(oc[4 * hh + 2], af, bq0, bq1);
        af[0] = crumb<6>(uh); af[1] = crumb<8>(uh); af[2] = crumb<6>(vh); af[3] = crumb<8>(vh);  // +6, +7
        mma(oc[4 * hh + 3], af, bq0, bq1);
      }
    } else {
      const uint4 xa = sh<uint4>(smem, ST + oC0), xb = sh<uint4>(smem, ST + oC1);
      const uint4 xc = sh<uint4>(smem, ST + oC0 + 1024), xd = sh<uint4>(smem, ST + oC1 + 1024);
      const uint32_t A[4] = {xa.x, xa.y, xa.z, xa.w}, B[4] = {xb.x, xb.y, xb.z, xb.w};
      const uint32_t Cc[4] = {xc.x, xc.y, xc.z, xc.w}, Dd[4] = {xd.x, xd.y, xd.z, xd.w};
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {  // d = 16r + 2mt (+1): bytes j, j+1 (j = 2(mt&1)) of word mt/2
        const uint32_t sel = (mt & 1) ? 0x7632u : 0x5410u;
        const uint32_t u = prmt(A[mt >> 1], B[mt >> 1], sel), v = prmt(Cc[mt >> 1], Dd[mt >> 1], sel);
        uint32_t af[4];
        af[0] = lop_and_or(u, 0x00FF00FFu, 0x64006400u);  // 1024 + code
        af[1] = lop_and_or(u >> 8, 0x00FF00FFu, 0x64006400u);
        af[2] = lop_and_or(v, 0x00FF00FFu, 0x64006400u);
        af[3] = lop_and_or(v >> 8, 0x00FF00FFu, 0x64006400u);
        mma(oc[mt], af, bq0, bq1);
      }
    }
    // ------------------------------------------------------------ this warp's share of the vmean split
    {  // token vt, d = 8vu .. 8vu+7 -> f16 hi / lo rows [tok][d] (16-B chunk vu at vu ^ (vt & 7))
      const float4 x0 = sh<float4>(smem, ST + oV0), x1 = sh<float4>(smem, ST + oV1);
      uint4 hi;
#if TADA_V8_VMEAN_LO
      static_assert(!PIPE, "the pipelined plan holds the hi part of the split vmean only");
      uint4 lo;
      split_h2(x0.x, x0.y, hi.x, lo.x);
      split_h2(x0.z, x0.w, hi.y, lo.y);
      split_h2(x1.x, x1.y, hi.z, lo.z);
      split_h2(x1.z, x1.w, hi.w, lo.w);
      if (tail && vt >= nv) lo = make_uint4(0u, 0u, 0u, 0u);
      sh<uint4>(smem, oVW + VMPART) = lo;
#else
      // vmean enters the PV mean MMA as f16 (RN): |error| <= 2^-12 |vmean|, the same relative
      // precision as the f16 P it multiplies (the logit side keeps hi + lo: errors there exponentiate)
      hi = make_uint4(pack_h2(x0.x, x0.y), pack_h2(x0.z, x0.w), pack_h2(x1.x, x1.y), pack_h2(x1.z, x1.w));
#endif
      if (tail && vt >= nv) hi = make_uint4(0u, 0u, 0u, 0u);  // rows past the sequence may hold anything
      sh<uint4>(smem, VO + oVW) = hi;
    }
  };

  // ------------------------------------------------------------ C: PV mean piece (d slice of this warp)
  auto phaseC = [&](auto buf_c) {
    const int BUF = int(buf_c);
    const int PO = BUF * pl.p_stride, CO = BUF * pl.corr_stride, VO = BUF * pl.vm_stride;
#if TADA_V8_OFTM >= 2
    float ofc[2];
    tmem_ld<2>(tof2 + 4, ofc);
    tmem_wait_ld();
    const uint32_t aPA = __float_as_uint(ofc[0]), aVB = __float_as_uint(ofc[1]);
#endif
    // FLAGS: one 8-byte read of the per-warp rescale flags (rare after the first tiles) decides whether
    // to touch corr at all; otherwise every thread reads its rows' corr and the warp votes
    float cr[MT][2];
    bool any = false;
    if constexpr (FLAGS) {
      const uint2 fl = sh<uint2>(smem, pl.off_bar + 96 + 8 * BUF);
      any = (fl.x | fl.y) != 0u;  // CTA-uniform
    } else {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        cr[mt][0] = sh<float>(smem, CO + pl.off_corr + 4 * (16 * mt + r));
        cr[mt][1] = sh<float>(smem, CO + pl.off_corr + 4 * (16 * mt + r + 8));
        any |= (cr[mt][0] != 1.f) || (cr[mt][1] != 1.f);
      }
      any = __any_sync(0xffffffffu, any);
    }
    if constexpr (PARK) {
      tmem_wait_st();
      tmem_ld<NOM>(tom, &om[0][0][0]);
      tmem_wait_ld();
    }
    if (any) {
      if constexpr (FLAGS) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          cr[mt][0] = sh<float>(smem, CO + pl.off_corr + 4 * (16 * mt + r));
          cr[mt][1] = sh<float>(smem, CO + pl.off_corr + 4 * (16 * mt + r + 8));
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          om[j][mt][0] *= cr[mt][0];
          om[j][mt][1] *= cr[mt][0];
          om[j][mt][2] *= cr[mt][1];
          om[j][mt][3] *= cr[mt][1];
        }
    }
    uint32_t bh[4];
    ldsm_x4_t(bh, aVB + VO);
#if TADA_V8_VMEAN_LO
    uint32_t bl[4];
    ldsm_x4_t(bl, aVB + VMPART);
#endif
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      uint32_t pa[4];
      ldsm_x4(pa, aPA + PO + mt * 512);
#pragma unroll
      for (int j = 0; j < 2; ++j) mma(om[j][mt], pa, bh[2 * j], bh[2 * j + 1]);
#if TADA_V8_VMEAN_LO
#pragma unroll
      for (int j = 0; j < 2; ++j) mma(om[j][mt], pa, bl[2 * j], bl[2 * j + 1]);
#endif
    }
    if constexpr (PARK) tmem_st<NOM>(tom, &om[0][0][0]);
  };

  if constexpr (!PIPE) {
    // classic schedule: A | barrier | B | barrier, refill | C
    auto body = [&](auto stage_c, int it) {
      constexpr int STG = decltype(stage_c)::value;
      mbar_wait(&full[STG], uint32_t(it / S) & 1u);
      if (a.diag == 1) {  // diagnostics: pipeline only
        __syncthreads();
        __syncthreads();
        if (tid == 0 && it + S < ntiles) {
          issue(STG);
          if (it + S + 1 < ntiles && a.diag != 2) cur_page = pt[cur_pg];
        }
        return;
      }
      phaseA(I0{}, loadA(stage_c));
      __syncthreads();  // ---- barrier 1: S_mean complete; the previous tile's P and split vmean are consumed
      phaseB(stage_c, I0{}, std::true_type{}, it);
      __syncthreads();  // ---- barrier 2: P, corr and the split vmean complete; this tile's stage is free
      if (tid == 0 && it + S < ntiles) {
        issue(STG);
        // (a late page-table load here would stall the next barrier; diag 2 re-reads one L2-resident page)
        if (it + S + 1 < ntiles && a.diag != 2) cur_page = pt[cur_pg];
      }
      phaseC(I0{});
    };
    for (int it = 0; it < ntiles; it += S) {
      body(std::integral_constant<int, 0>{}, it);
      if (it + 1 < ntiles) body(std::integral_constant<int, 1>{}, it + 1);
      if constexpr (S == 3)
        if (it + 2 < ntiles) body(std::integral_constant<int, 2>{}, it + 2);
    }
  } else {
    // pipelined schedule (tile i in stage i % S, exchange buffer i & 1):
    //   A(0) | barrier | { C(i-1), B(i), A(i+1) | barrier, refill stage i % S with tile i + S } for each i | C(last)
    // One barrier per tile; the three phases are independent dependency chains the scheduler interleaves.  The
    // loop is unrolled by U = 2S so stage, buffer and mbarrier parity are immediates (J = i mod U: stage J % S,
    // buffer J & 1, parity (J / S) & 1 since U / S is even); the < U leftover tiles run one runtime-indexed copy.
    constexpr int U = 2 * S;
    auto step = [&](auto stg, auto buf, auto st1, auto buf1, uint32_t par1, auto maytail_c, int it) {
#if TADA_V8_ORDER == 1  // the next tile's kmean loads issued first, consumed after phase B
      KMean km{};
      if (it + 1 < ntiles) {
        mbar_wait(&full[int(st1)], par1);
        km = loadA(st1);
      }
      if (it > 0) phaseC(buf1);  // tile i - 1 used buffer (i - 1) & 1 = buf ^ 1
      phaseB(stg, buf, maytail_c, it);
      if (it + 1 < ntiles) phaseA(buf1, km);
#elif TADA_V8_ORDER == 2  // C, A, B
      if (it > 0) phaseC(buf1);
      if (it + 1 < ntiles) {
        mbar_wait(&full[int(st1)], par1);
        phaseA(buf1, loadA(st1));
      }
      phaseB(stg, buf, maytail_c, it);
#else
      if (TADA_V8_EARLYWAIT && it + 1 < ntiles) mbar_wait(&full[int(st1)], par1);
      if (it > 0) phaseC(buf1);  // tile i - 1 used buffer (i - 1) & 1 = buf ^ 1
      phaseB(stg, buf, maytail_c, it);
      if (it + 1 < ntiles) {
        if (!TADA_V8_EARLYWAIT) mbar_wait(&full[int(st1)], par1);
        phaseA(buf1, loadA(st1));
      }
#endif
      __syncthreads();  // ---- S_mean(i+1), P(i) and the split vmean(i) complete; stage i % S is free
      if (tid == 0 && it + S < ntiles) {
        issue(int(stg));
        if (it + S + 1 < ntiles) cur_page = pt[cur_pg];
      }
    };
    auto stepJ = [&](auto j_c, int it) {
      constexpr int J = decltype(j_c)::value;
      step(std::integral_constant<int, J % S>{}, std::integral_constant<int, J & 1>{},
           std::integral_constant<int, (J + 1) % S>{}, std::integral_constant<int, (J + 1) & 1>{},
           uint32_t(((J + 1) / S) & 1), std::false_type{}, it);
    };
    __syncthreads();  // the QA staging (aliased onto the S_mean buffers) is in TMEM in every warp
    if (ntiles > 0) {
      mbar_wait(&full[0], 0u);
      phaseA(I0{}, loadA(I0{}));
    }
    __syncthreads();
    const int nfull = (t_end - t_begin) / TT;  // tiles with TT valid tokens (only the last may be partial)
    int it = 0;
    for (; it + U <= nfull; it += U) {
      stepJ(std::integral_constant<int, 0>{}, it);
      stepJ(std::integral_constant<int, 1>{}, it + 1);
      stepJ(std::integral_constant<int, 2>{}, it + 2);
      stepJ(std::integral_constant<int, 3>{}, it + 3);
      if constexpr (U == 6) {
        stepJ(std::integral_constant<int, U == 6 ? 4 : 0>{}, it + 4);
        stepJ(std::integral_constant<int, U == 6 ? 5 : 0>{}, it + 5);
      }
    }
    int st = 0;  // leftover tiles: it is a multiple of U here, so tile it sits in stage 0 at parity 0
    uint32_t par = 0u;
    auto step_rt = [&](auto maytail_c, int it) {
      const int st1 = st + 1 == S ? 0 : st + 1;
      const uint32_t par1 = st + 1 == S ? par ^ 1u : par;
      step(st, it & 1, st1, (it & 1) ^ 1, par1, maytail_c, it);
      st = st1;
      par = par1;
    };
    for (; it < nfull; ++it) step_rt(std::false_type{}, it);
    if (it < ntiles) step_rt(std::true_type{}, it);
    if (ntiles > 0) phaseC((ntiles - 1) & 1);
  }

  // ------------------------------------------------------------------ epilogue
  // per q head: l, Σp·vmin and Σp' over the row's four c lanes
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    l_run += __shfl_xor_sync(0xffffffffu, l_run, o);
    bp_run += __shfl_xor_sync(0xffffffffu, bp_run, o);
    sp_run += __shfl_xor_sync(0xffffffffu, sp_run, o);
  }
  const float sp0 = __shfl_sync(0xffffffffu, sp_run, 8 * c), sp1 = __shfl_sync(0xffffffffu, sp_run, 8 * c + 4);
  __syncthreads();  // every tile consumed: the stages and the split vmean are idle
  if (live && c == 0) {
    red[qrow] = l_run;
    red[HQ + qrow] = bp_run;
    red[2 * HQ + qrow] = m_run;
  }
  constexpr int PR = D + 4;  // park row (padded)
  float* park = reinterpret_cast<float*>(smem);  // [HQ][PR]
  if constexpr (USE_TM) {
    tmem_wait_st();
    if constexpr (PARK) tmem_ld<NOM>(tom, &om[0][0][0]);
    tmem_wait_ld();
    tc_fence_before();  // the __syncthreads below orders every warp's last TMEM read before the dealloc
  }
  // 1) mean term: rows q = 16mt + r (+8), cols d = 16w + 8j + 2c (+1)
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int q = 16 * mt + r + 8 * e;
      if (q < HQ)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          *reinterpret_cast<float2*>(park + q * PR + 16 * warp + 8 * j + 2 * c) =
              make_float2(om[j][mt][2 * e], om[j][mt][2 * e + 1]);
    }
  __syncthreads();
  if constexpr (USE_TM) {
    if (warp == 0) {
      tc_fence_after();
      tmem_dealloc(tbase, TCOLS);
    }
  }
  // 2) code term minus its bias: rows d = 16r + 2mt (+1), cols n = 2c (+1)
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int n = 2 * c + e;
    if (n < G) {
      const float sp = e ? sp1 : sp0;
      float* row = park + (h * G + n) * PR + 16 * r;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        row[2 * mt] += (oc[mt][e] - pv_bias<BITS>(mt, 0) * sp) * (1.f / PPS);
        row[2 * mt + 1] += (oc[mt][2 + e] - pv_bias<BITS>(mt, 1) * sp) * (1.f / PPS);
      }
    }
  }
  __syncthreads();
  // 3) write the split slot (natural-log LSE units for K3)
  const float LN2 = 0.6931471805599453f;
  for (int i = tid; i < HQ * D; i += NTHR) {
    const int g = i / D, d = i - g * D;
    const float l = red[g], bp = red[HQ + g], m = red[2 * HQ + g];
    const int64_t slot = (int64_t(b) * HQ + g) * a.slots + split;
    a.part_acc[slot * D + d] = l > 0.f ? park[g * PR + d] - bp : 0.f;
    if (d == 0) {
      a.part_ml[slot * 2] = l > 0.f ? m * LN2 : NEG_INF;
      a.part_ml[slot * 2 + 1] = l;
    }
  }
}

}  // namespace v8

bool v8_supported(const tada_page_layout& L, int Hq) {
  if (L.head_dim != 128 || L.heads != 8 || !(L.bits == 2 || L.bits == 4 || L.bits == 8)) return false;
  if (!(Hq == 8 || Hq == 16 || Hq == 32 || Hq == 64)) return false;
  if (L.page_tokens % v8::TT != 0) return false;
  return v8::make_plan(L.group_bytes, Hq).ok;
}

template <int BITS, int HQ>
static int launch_v8_t(const AttnArgs& a, int batch, cudaStream_t st) {
  constexpr v8::Plan pl = v8::make_plan(BITS * 128 / 8, HQ, v8::v8_pipe(BITS, HQ));  // the kernel's own plan
  if constexpr (!pl.ok) {
    return fail(TADA_ERR_CONFIG, "decode_attn_v8: geometry does not fit two stages");
  } else {
    auto kern = v8::attn_v8_kernel<BITS, HQ>;
    static std::atomic<uint64_t> smem_set{0};  // per instantiation, per device
    if (const int rc0 = ensure_smem(kern, pl.total, smem_set, "attn_v8"); rc0 != TADA_OK) return rc0;
    TmaMaps maps;
    const int rc = get_tma_maps(a, &maps, v8::TT);
    if (rc != TADA_OK) return rc;
    const cudaError_t e = launch_maybe_pdl(kern, dim3(a.splits, batch), dim3(v8::NTHR), size_t(pl.total), st, a, maps);
    if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("decode_attn_v8: ") + cudaGetErrorString(e));
    return check_launch("decode_attn_v8");
  }
}

template <int BITS>
static int launch_v8_b(const AttnArgs& a, int batch, cudaStream_t st) {
  switch (a.Hq) {
    case 8: return launch_v8_t<BITS, 8>(a, batch, st);
    case 16: return launch_v8_t<BITS, 16>(a, batch, st);
    case 32: return launch_v8_t<BITS, 32>(a, batch, st);
    default: return launch_v8_t<BITS, 64>(a, batch, st);
  }
}

int launch_v8(const AttnArgs& a, int batch, cudaStream_t st) {
  switch (a.L.bits) {
    case 2: return launch_v8_b<2>(a, batch, st);
    case 4: return launch_v8_b<4>(a, batch, st);
    default: return launch_v8_b<8>(a, batch, st);
  }
}

}  // namespace tada
