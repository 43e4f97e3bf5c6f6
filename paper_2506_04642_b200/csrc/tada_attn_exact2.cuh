// K2-exact v2 (attn_exact2_kernel), shared by tada_attn_exact.cu (head_dim 128) and tada_attn_exact_d.cu
// (head_dim 32 / 64 / 256): the instantiations are split over two translation units so they compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <string>

#include "tada_attn.cuh"
#include "tada_mma.cuh"

namespace tada {
// ---------------------------------------------------------------------------------------------------------------
// K2-exact v2 (attn_exact2_kernel): the same arithmetic for head_dim 32 / 64 / 128 / 256, widths 2/4/8/16 and any KV head count
// and group size whose phase-2 accumulators fit (see plan()), with the element-wise f32 work on the packed FP32x2
// pipe (FADD2 / FFMA2: two elements per issue).
//
// CTA = (split, sequence), 256 threads, 32-token tiles in a two-stage cp.async ring (both sides' mean rows, the code
// rows of all heads, the metas; rows padded so the per-lane row reads below are bank-conflict free).
//   phase 1 (scores), lane = token, warp = (KV head, GT of its q heads): the lane expands its token's codes for the
//     head (PRMT into 2^23-biased floats), forms K̂ = mean - fma(code, scale, min) in pairs and the dots with the GT
//     q rows (broadcast from shared memory) in FFMA2 pairs — no cross-lane reduction;
//   softmax, warp per q head, lane = token: online max / sum in f32 (attention.py:139-147);
//   phase 2 (P·V̂), thread = (KV head, 4 columns, GT q heads): V̂ expanded once per (token, column) and accumulated
//     for the GT q heads in registers (FFMA2 with the weight broadcast).
// Partials leave in the tensor-core kernels' slot format; K3 adds the residual rows and merges the splits.
#ifndef TADA_EX2_UNROLL
#define TADA_EX2_UNROLL 4  // phase-1 column loop unroll (A/B switch; 4 measured +3-5% over 2)
#endif
namespace exact2 {
constexpr int kEx2Unroll = TADA_EX2_UNROLL;

constexpr int NTHR = 256;

struct Plan {
  int tt;  // tokens per tile (16)
  int H, G, Hq, gb, gt, nqc, upt, RS, CRS, QS, PS;
  int gs;  // q rows per KV head in shared memory: G, or G padded to gt (G in 3, 5, 6, 7) with zero rows
  int cshift;  // log2 of the 16-byte chunks per code row when a power of two, else -1 (tile staging, below)
  int sb;  // bytes per stage; stage st starts at st * sb
  int off_km, off_vm, off_kc, off_vc, off_kx, off_vx;  // within a stage
  int off_q, off_s, off_p, off_corr, off_ml, total;
};

inline bool plan(const tada_page_layout& L, int Hq, Plan* out) {
  Plan p{};
  const int D = L.head_dim;
  p.H = L.heads;
  if (!(D == 32 || D == 64 || D == 128 || D == 256) || p.H <= 0 || Hq % p.H) return false;
  if (!(L.bits == 2 || L.bits == 4 || L.bits == 8 || L.bits == 16)) return false;
  p.G = Hq / p.H;
  p.Hq = Hq;
  p.gb = int(L.group_bytes);
  if ((p.H * p.gb) % 16) return false;
  p.gt = 1;  // q heads per unit: the largest power of two <= 8 dividing G
  while (p.gt < 8 && p.G % (2 * p.gt) == 0) p.gt *= 2;
  p.nqc = p.G / p.gt;
  p.gs = p.G;
  if (p.G < 8 && p.gt != p.G) {  // G in 3, 5, 6, 7: one unit of gt = 4 / 8 rows per KV head, the extra rows zero
    p.gt = p.G <= 4 ? 4 : 8;
    p.nqc = 1;
    p.gs = p.gt;
  }
  const int units = p.H * p.nqc * (D / 4);
  p.upt = (units + NTHR - 1) / NTHR;
  if (p.upt == 3) p.upt = 4;
  if (p.upt > 4 || p.upt * p.gt > 8) return false;
  p.RS = D + 4;                 // lane-per-row float4 reads: 8 lanes hit 8 distinct 16-byte bank groups
  p.CRS = p.H * p.gb + 16;      // ... and the code rows likewise
  p.cshift = -1;
  for (int c = (p.H * p.gb) / 16, k = 0; k < 16; ++k)
    if (c == (1 << k)) p.cshift = k;
  p.QS = D + 4;  // the upper half of a q row sits 4 floats further: the two column halves of phase 1 differ in bank
  for (int tt = 16; tt >= 16; tt /= 2) {
    const int TT = tt;
    p.tt = tt;
    p.PS = TT + 4;  // 16-byte rows: four tokens' weights per load
    int off = 0;
    auto take = [&](int bytes) {
      const int o = off;
      off = (off + bytes + 127) / 128 * 128;
      return o;
    };
    p.off_km = take(TT * p.RS * 4);
    p.off_vm = take(TT * p.RS * 4);
    p.off_kc = take(TT * p.CRS);
    p.off_vc = take(TT * p.CRS);
    p.off_kx = take(TT * p.H * 8);
    p.off_vx = take(TT * p.H * 8);
    p.sb = off;
    off = 2 * p.sb;
    const int hqs = p.H * p.gs;  // q rows in shared memory
    p.off_q = take(hqs * p.QS * 4);
    p.off_s = take(hqs * p.PS * 4);  // scores, then the weights P in place
    p.off_p = p.off_s;
    p.off_corr = take(hqs * 4);
    p.off_ml = take(hqs * 8);
    p.total = off;
    if (p.total <= 220 * 1024) {
      *out = p;
      return true;
    }
  }
  return false;
}

__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// 4 consecutive codes (BITS 2/4/8) held in the low bits of w (LSB-first) as exact floats: (2^23 | code) - 2^23
template <int BITS>
__device__ __forceinline__ void codes4(uint32_t w, float2& c01, float2& c23) {
  constexpr uint32_t M = 0x4B000000u;
  uint32_t t0, t1, t2, t3;
  if (BITS == 8) {
    t0 = prmt(w, M, 0x7650u);
    t1 = prmt(w, M, 0x7651u);
    t2 = prmt(w, M, 0x7652u);
    t3 = prmt(w, M, 0x7653u);
  } else if (BITS == 4) {
    const uint32_t lo = w & 0x0F0Fu, hi = (w >> 4) & 0x0F0Fu;
    t0 = prmt(lo, M, 0x7650u);
    t1 = prmt(hi, M, 0x7650u);
    t2 = prmt(lo, M, 0x7651u);
    t3 = prmt(hi, M, 0x7651u);
  } else {
    t0 = M | (w & 3u);
    t1 = M | ((w >> 2) & 3u);
    t2 = M | ((w >> 4) & 3u);
    t3 = M | ((w >> 6) & 3u);
  }
  c01 = __fadd2_rn(make_float2(__uint_as_float(t0), __uint_as_float(t1)), make_float2(-8388608.f, -8388608.f));
  c23 = __fadd2_rn(make_float2(__uint_as_float(t2), __uint_as_float(t3)), make_float2(-8388608.f, -8388608.f));
}

// 4 reconstructed elements mean - fma(code, scale, min) (cache.py:190-213, quant.py:177-180) from the codes in w;
// width 16: mean - raw deviation (dev4)
template <int BITS>
__device__ __forceinline__ void recon4(float4 m, uint32_t w, float4 dev4, float2 sm, float2& r01, float2& r23) {
  if (BITS == 16) {
    r01 = __fadd2_rn(make_float2(m.x, m.y), make_float2(-dev4.x, -dev4.y));
    r23 = __fadd2_rn(make_float2(m.z, m.w), make_float2(-dev4.z, -dev4.w));
    return;
  }
  float2 c01, c23;
  codes4<BITS>(w, c01, c23);
  const float2 d01 = __ffma2_rn(c01, make_float2(sm.x, sm.x), make_float2(sm.y, sm.y));
  const float2 d23 = __ffma2_rn(c23, make_float2(sm.x, sm.x), make_float2(sm.y, sm.y));
  r01 = __fadd2_rn(make_float2(m.x, m.y), make_float2(-d01.x, -d01.y));
  r23 = __fadd2_rn(make_float2(m.z, m.w), make_float2(-d23.x, -d23.y));
}

template <int BITS, int D, int GT, int UPT, int TT>
__global__ void __launch_bounds__(NTHR, 2) attn_exact2_kernel(AttnArgs a, Plan pl) {
  constexpr int CPW = BITS == 16 ? 1 : 32 / BITS;  // codes per 32-bit word
  constexpr int RS = D + 4, QS = D + 4, PS = TT + 4;  // = plan()'s row strides, as immediates
  extern __shared__ __align__(128) uint8_t smem[];
  const int H = pl.H, G = pl.G, Hq = pl.Hq, gb = pl.gb, P = a.L.page_tokens, nqc = pl.nqc;
  const int b = blockIdx.y, split = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* qs = reinterpret_cast<float*>(smem + pl.off_q);
  float* S = reinterpret_cast<float*>(smem + pl.off_s);
  float* corr = reinterpret_cast<float*>(smem + pl.off_corr);
  float2* ml = reinterpret_cast<float2*>(smem + pl.off_ml);
  const float NEG_INF = -__int_as_float(0x7f800000);

  pdl_enter();  // no global reads above this line
  const int C = comp_tokens(a, b);
  int t_begin, t_end;
  split_range(C, a.splits, split, TT, t_begin, t_end);
  const int gs = pl.gs, hqs = H * gs;  // shared-memory q rows: row h * gs + j is q head h * G + j (j < G), else 0
  for (int i = tid; i < hqs * D; i += NTHR) {
    const int r = i / D, dd = i - r * D, j = r % gs;
    if (j >= G) {
      qs[r * QS + dd + (dd >= D / 2 ? 4 : 0)] = 0.f;
      continue;
    }
    const int64_t qi = (int64_t(b) * Hq + (r / gs) * G + j) * D + dd;
    const int g = i / D, d = i - g * D;
    qs[g * QS + d + (d >= D / 2 ? 4 : 0)] = a.q_dtype == TADA_F32 ? reinterpret_cast<const float*>(a.q)[qi]
                                                                    : to_f32(reinterpret_cast<const __nv_bfloat16*>(a.q)[qi]);
  }
  for (int g = tid; g < hqs; g += NTHR) ml[g] = make_float2(NEG_INF, 0.f);
  const int32_t* pt = a.page_table + int64_t(b) * a.pt_stride;
  const int pshift = (P & (P - 1)) == 0 ? __ffs(P) - 1 : -1;

  // ---- staging of tile [t0, t0 + TT) into stage st (cp.async; tokens past t_end are not loaded).
  // Tiles start at multiples of TT (split_range), so with page_tokens a multiple of TT a tile's rows are
  // consecutive rows of one page and each block (means, codes, metas) is one contiguous run: the CTA copies
  // it as a flat range of 16-byte chunks, one page-table read per tile (`tile_page`, read one tile ahead).
  // Otherwise: warp per (side, token row), lanes over the row's 16-byte chunks.
  const bool flat = pshift >= 0 && P % TT == 0 && pl.cshift >= 0;
  auto stage_flat = [&](int t0, int st, int32_t page_id) {
    const int nv = min(TT, t_end - t0);
    uint8_t* sb = smem + st * pl.sb;
    const int row0 = t0 & (P - 1);
    const uint8_t* page = a.pool + int64_t(page_id) * a.L.page_bytes;
    constexpr int MC = D / 4, MS = MC == 8 ? 3 : MC == 16 ? 4 : MC == 32 ? 5 : 6;  // 16-byte chunks per mean row
    const int cs = pl.cshift, nm = nv * H / 2;  // metas: H * 8 bytes per row
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const float* msrc = reinterpret_cast<const float*>(page + a.L.off_mean[side]) + int64_t(row0) * D;
      float* mdst = reinterpret_cast<float*>(sb + (side ? pl.off_vm : pl.off_km));
      const uint8_t* csrc = page + a.L.off_codes[side] + int64_t(row0) * H * gb;
      uint8_t* cdst = sb + (side ? pl.off_vc : pl.off_kc);
      if (nv == TT && (TT << MS) % NTHR == 0) {  // full tile: constant trip counts
#pragma unroll
        for (int k = 0; k < (TT << MS) / NTHR; ++k) {
          const int j = tid + k * NTHR;
          cp16(mdst + (j >> MS) * RS + 4 * (j & (MC - 1)), msrc + 4 * j);
        }
      } else {
        for (int j = tid; j < (nv << MS); j += NTHR) cp16(mdst + (j >> MS) * RS + 4 * (j & (MC - 1)), msrc + 4 * j);
      }
      for (int j = tid; j < (nv << cs); j += NTHR)
        cp16(cdst + (j >> cs) * pl.CRS + 16 * (j & ((1 << cs) - 1)), csrc + 16 * j);
      const uint8_t* xsrc = page + a.L.off_meta[side] + int64_t(row0) * H * 8;
      uint8_t* xdst = sb + (side ? pl.off_vx : pl.off_kx);
      if (side == 0) {  // key metas transposed to [head][token]: phase 1's 16 token lanes read 128 contiguous bytes
        for (int j = tid; j < H * TT; j += NTHR) {
          const int h = j / TT, t = j - h * TT;
          if (t < nv) cp8(xdst + 8 * j, xsrc + 8 * (t * H + h));
        }
      } else {  // value metas stay [token][head] (phase 2 broadcasts one per warp)
        for (int j = tid; j < nm; j += NTHR) cp16(xdst + 16 * j, xsrc + 16 * j);
        if ((nv * H) & 1 && tid == NTHR - 1) cp8(xdst + 16 * nm, xsrc + 16 * nm);  // odd H, partial tile
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto tile_page = [&](int t0) { return t0 < t_end ? pt[t0 >> pshift] : 0; };
  auto stage = [&](int t0, int st) {
    const int nv = min(TT, t_end - t0);
    uint8_t* sb = smem + st * pl.sb;
    for (int r = warp; r < 2 * nv; r += NTHR / 32) {
      const int side = r & 1, t = r >> 1, tok = t0 + t;
      const int pg = pshift >= 0 ? tok >> pshift : tok / P;  // page_tokens is a power of two in practice
      const uint8_t* page = a.pool + int64_t(pt[pg]) * a.L.page_bytes;
      const int row = tok - pg * P;
      const float* msrc = reinterpret_cast<const float*>(page + a.L.off_mean[side]) + int64_t(row) * D;
      float* mdst = reinterpret_cast<float*>(sb + (side ? pl.off_vm : pl.off_km)) + t * RS;
      for (int c = lane; c < D / 4; c += 32) cp16(mdst + 4 * c, msrc + 4 * c);
      const uint8_t* csrc = page + a.L.off_codes[side] + int64_t(row) * H * gb;
      uint8_t* cdst = sb + (side ? pl.off_vc : pl.off_kc) + t * pl.CRS;
      for (int c = lane; c < H * gb / 16; c += 32) cp16(cdst + 16 * c, csrc + 16 * c);
      const uint8_t* xsrc = page + a.L.off_meta[side] + int64_t(row) * H * 8;
      if (side == 0)  // key metas [head][token] (see stage_flat)
        for (int h = lane; h < H; h += 32) cp8(sb + pl.off_kx + 8 * (h * TT + t), xsrc + 8 * h);
      else
        for (int h = lane; h < H; h += 32) cp8(sb + pl.off_vx + 8 * (t * H + h), xsrc + 8 * h);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // phase-2 accumulators: unit i = (KV head, q chunk, 4-column chunk), GT q heads, two column pairs
  float2 acc[UPT][GT][2];
#pragma unroll
  for (int i = 0; i < UPT; ++i)
#pragma unroll
    for (int g = 0; g < GT; ++g) acc[i][g][0] = acc[i][g][1] = make_float2(0.f, 0.f);

  int32_t next_page = 0;  // page of the tile after the one being staged (flat staging)
  if (t_begin < t_end) {
    if (flat) {
      stage_flat(t_begin, 0, tile_page(t_begin));
      next_page = tile_page(t_begin + TT);
    } else {
      stage(t_begin, 0);
    }
  }
  int st = 0;
  for (int t0 = t_begin; t0 < t_end; t0 += TT, st ^= 1) {
    const int nv = min(TT, t_end - t0);
    if (t0 + TT < t_end) {
      if (flat) {
        stage_flat(t0 + TT, st ^ 1, next_page);
        next_page = tile_page(t0 + 2 * TT);
      } else {
        stage(t0 + TT, st ^ 1);
      }
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const uint8_t* sbase = smem + st * pl.sb;
    const float* km = reinterpret_cast<const float*>(sbase + pl.off_km);
    const float* vm = reinterpret_cast<const float*>(sbase + pl.off_vm);
    const uint8_t* kc = sbase + pl.off_kc;
    const uint8_t* vc = sbase + pl.off_vc;
    const float2* kx = reinterpret_cast<const float2*>(sbase + pl.off_kx);
    const float2* vx = reinterpret_cast<const float2*>(sbase + pl.off_vx);

    // ---- phase 1: lane = (token, column half), warp = (KV head, q chunk); the halves meet by one shuffle.
    // 2/4-bit (ILV): lane = 2 token + half and the halves interleave 16-column blocks (half hf takes blocks
    // hf, hf + 2, ...), so the code loads of one phase hit distinct banks (the contiguous halves, lane = token +
    // 16 half, put rows t and t + 8 of a 16-byte-padded code row on the same bank: 2-way at 4-bit, 4-way at 2-bit).
    constexpr bool ILV = BITS == 2 || BITS == 4;
    constexpr int HX = ILV ? 1 : TT;  // lane distance between the two halves of a token
    for (int u = warp; u < H * nqc; u += NTHR / 32) {
      const int h = u / nqc, g0 = h * gs + (u - h * nqc) * GT;  // shared-memory row of the unit's first q head
      const int t = ILV ? lane >> 1 : lane & (TT - 1), hf = ILV ? lane & 1 : lane / TT;
      const float* mrow = km + t * RS;
      const uint8_t* crow = kc + t * pl.CRS + h * gb;
      const float2 sm = kx[h * TT + t];
      float2 z2[GT];
#pragma unroll
      for (int g = 0; g < GT; ++g) z2[g] = make_float2(0.f, 0.f);
#pragma unroll kEx2Unroll
      for (int i = 0; i < D / 32; ++i) {
        const int d = ILV ? 16 * hf + 32 * i : hf * (D / 2) + 16 * i;
        // q columns >= D/2 sit 4 floats further in their row (staging above)
        const float* qrow = qs + (d >= D / 2 ? 4 : 0);
        uint4 w4 = make_uint4(0, 0, 0, 0);  // the 16 codes of columns d .. d + 15 (BITS < 16)
        if (BITS == 2) w4.x = *reinterpret_cast<const uint32_t*>(crow + d / 4);
        if (BITS == 4) *reinterpret_cast<uint2*>(&w4) = *reinterpret_cast<const uint2*>(crow + d / 2);
        if (BITS == 8) w4 = *reinterpret_cast<const uint4*>(crow + d);
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          const float4 m = *reinterpret_cast<const float4*>(mrow + d + e);
          float4 dev4 = make_float4(0.f, 0.f, 0.f, 0.f);
          uint32_t w = 0;
          if (BITS == 16) dev4 = *reinterpret_cast<const float4*>(crow + 4 * (d + e));
          else {
            const uint32_t words[4] = {w4.x, w4.y, w4.z, w4.w};
            w = words[e / CPW] >> (BITS * (e % CPW));
          }
          float2 k01, k23;
          recon4<BITS>(m, w, dev4, sm, k01, k23);
#pragma unroll
          for (int g = 0; g < GT; ++g) {
            const float4 q4 = *reinterpret_cast<const float4*>(qrow + (g0 + g) * QS + d + e);
            z2[g] = __ffma2_rn(make_float2(q4.x, q4.y), k01, z2[g]);
            z2[g] = __ffma2_rn(make_float2(q4.z, q4.w), k23, z2[g]);
          }
        }
      }
      // online softmax of the unit's q heads over the tile, in the same warp (attention.py:139-147): the two
      // column halves hold the same sums after the shuffle, so both lanes of a token agree; P goes to shared memory
      // (the GT reductions interleaved: independent shuffle chains; 16-lane butterflies, the halves being equal)
      float zz[GT], mx[GT], pe[GT], ls[GT];
#pragma unroll
      for (int g = 0; g < GT; ++g) {
        float z = z2[g].x + z2[g].y;
        z += __shfl_xor_sync(0xffffffffu, z, HX);
        zz[g] = t < nv ? __fmul_rn(z, a.scale) : NEG_INF;
        mx[g] = zz[g];
      }
#pragma unroll
      for (int o = TT / 2; o > 0; o >>= 1)
#pragma unroll
        for (int g = 0; g < GT; ++g) mx[g] = fmaxf(mx[g], __shfl_xor_sync(0xffffffffu, mx[g], ILV ? 2 * o : o));
#pragma unroll
      for (int g = 0; g < GT; ++g) {
        mx[g] = fmaxf(ml[g0 + g].x, mx[g]);
        pe[g] = t < nv ? expf(zz[g] - mx[g]) : 0.f;
        ls[g] = pe[g];
      }
#pragma unroll
      for (int o = TT / 2; o > 0; o >>= 1)
#pragma unroll
        for (int g = 0; g < GT; ++g) ls[g] += __shfl_xor_sync(0xffffffffu, ls[g], ILV ? 2 * o : o);
#pragma unroll
      for (int g = 0; g < GT; ++g) {
        if (hf == 0) S[(g0 + g) * PS + t] = pe[g];
        if (lane == 0) {
          const float2 m0 = ml[g0 + g];
          const float cf = expf(m0.x - mx[g]);
          ml[g0 + g] = make_float2(mx[g], m0.y * cf + ls[g]);
          corr[g0 + g] = cf;
        }
      }
    }
    __syncthreads();  // P and the rescale factors of every q head are in shared memory
    // ---- phase 2: acc = acc * corr + P · V̂ per (KV head, q chunk, 4 columns)
#pragma unroll
    for (int i = 0; i < UPT; ++i) {
      const int u = tid + NTHR * i;
      if (u >= H * nqc * (D / 4)) continue;
      const int hq = u / (D / 4), c = u - hq * (D / 4);
      const int h = hq / nqc, g0 = h * gs + (hq - h * nqc) * GT, d0 = 4 * c;
#pragma unroll
      for (int g = 0; g < GT; ++g) {
        const float cf = corr[g0 + g];
        acc[i][g][0] = __fmul2_rn(acc[i][g][0], make_float2(cf, cf));
        acc[i][g][1] = __fmul2_rn(acc[i][g][1], make_float2(cf, cf));
      }
      const uint8_t* ccol = vc + h * gb + (BITS == 16 ? 16 * c : c * BITS / 2);
      const float* mcol = vm + d0;
      const float2* xcol = vx + h;
      const float* srow = S + g0 * PS;
      auto token = [&](int t, const float (&pw)[GT]) {
        const float4 m = *reinterpret_cast<const float4*>(mcol + t * RS);
        float4 dev4 = make_float4(0.f, 0.f, 0.f, 0.f);
        uint32_t w = 0;
        const uint8_t* cp = ccol + t * pl.CRS;
        if (BITS == 16) dev4 = *reinterpret_cast<const float4*>(cp);
        else if (BITS == 8) w = *reinterpret_cast<const uint32_t*>(cp);
        else if (BITS == 4) w = *reinterpret_cast<const uint16_t*>(cp);
        else w = *cp;
        float2 v01, v23;
        recon4<BITS>(m, w, dev4, xcol[t * H], v01, v23);
#pragma unroll
        for (int g = 0; g < GT; ++g) {
          acc[i][g][0] = __ffma2_rn(v01, make_float2(pw[g], pw[g]), acc[i][g][0]);
          acc[i][g][1] = __ffma2_rn(v23, make_float2(pw[g], pw[g]), acc[i][g][1]);
        }
      };
      if (nv == TT) {  // full tile: weights of 4 tokens per load
#pragma unroll
        for (int t = 0; t < TT; t += 4) {
          float4 w4[GT];
#pragma unroll
          for (int g = 0; g < GT; ++g) w4[g] = *reinterpret_cast<const float4*>(srow + g * PS + t);
          float pw[GT];
#pragma unroll
          for (int g = 0; g < GT; ++g) pw[g] = w4[g].x;
          token(t, pw);
#pragma unroll
          for (int g = 0; g < GT; ++g) pw[g] = w4[g].y;
          token(t + 1, pw);
#pragma unroll
          for (int g = 0; g < GT; ++g) pw[g] = w4[g].z;
          token(t + 2, pw);
#pragma unroll
          for (int g = 0; g < GT; ++g) pw[g] = w4[g].w;
          token(t + 3, pw);
        }
      } else {
        for (int t = 0; t < nv; ++t) {
          float pw[GT];
#pragma unroll
          for (int g = 0; g < GT; ++g) pw[g] = srow[g * PS + t];
          token(t, pw);
        }
      }
    }
    __syncthreads();  // this stage and S are consumed before the next tile's loads land in it
  }
  // ---- partials in the slot format K3 merges
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    const int u = tid + NTHR * i;
    if (u >= H * nqc * (D / 4)) continue;
    const int hq = u / (D / 4), c = u - hq * (D / 4);
    const int h = hq / nqc, qc0 = (hq - h * nqc) * GT;
#pragma unroll
    for (int g = 0; g < GT; ++g) {
      if (qc0 + g >= G) continue;  // a zero padding row
      const int64_t slot = (int64_t(b) * Hq + h * G + qc0 + g) * a.slots + split;
      *reinterpret_cast<float4*>(a.part_acc + slot * D + 4 * c) =
          make_float4(acc[i][g][0].x, acc[i][g][0].y, acc[i][g][1].x, acc[i][g][1].y);
    }
  }
  for (int r = tid; r < hqs; r += NTHR) {
    if (r % gs >= G) continue;  // a zero padding row
    const int64_t slot = (int64_t(b) * Hq + (r / gs) * G + r % gs) * a.slots + split;
    const float2 m = ml[r];
    a.part_ml[slot * 2] = m.y > 0.f ? m.x : NEG_INF;
    a.part_ml[slot * 2 + 1] = m.y;
  }
}

template <int BITS, int D, int GT, int UPT>
inline int launch_t(const AttnArgs& a, int batch, const Plan& pl, cudaStream_t st) {
  if constexpr (GT * UPT > 8) {
    return fail(TADA_ERR_CONFIG, "attn_exact2: accumulators do not fit");
  } else {
    auto kern = attn_exact2_kernel<BITS, D, GT, UPT, 16>;
    static std::atomic<uint64_t> done{0};
    if (const int rc = ensure_smem(kern, 220 * 1024, done, "attn_exact2"); rc != TADA_OK) return rc;
    const cudaError_t e = launch_maybe_pdl(kern, dim3(a.splits, batch), dim3(NTHR), size_t(pl.total), st, a, pl);
    if (e != cudaSuccess) return fail(TADA_ERR_CUDA, std::string("decode_attn_exact2: ") + cudaGetErrorString(e));
    return check_launch("decode_attn_exact2");
  }
}
template <int BITS, int D, int GT>
inline int launch_u(const AttnArgs& a, int batch, const Plan& pl, cudaStream_t st) {
  switch (pl.upt) {
    case 1: return launch_t<BITS, D, GT, 1>(a, batch, pl, st);
    case 2: return launch_t<BITS, D, GT, 2>(a, batch, pl, st);
    default: return launch_t<BITS, D, GT, 4>(a, batch, pl, st);
  }
}
template <int BITS, int D>
inline int launch_g(const AttnArgs& a, int batch, const Plan& pl, cudaStream_t st) {
  switch (pl.gt) {
    case 1: return launch_u<BITS, D, 1>(a, batch, pl, st);
    case 2: return launch_u<BITS, D, 2>(a, batch, pl, st);
    case 4: return launch_u<BITS, D, 4>(a, batch, pl, st);
    default: return launch_u<BITS, D, 8>(a, batch, pl, st);
  }
}
}  // namespace exact2
// head_dim 32 / 64 / 256 instantiations (tada_attn_exact_d.cu)
int exact2_launch_other_d(const AttnArgs& a, int batch, const exact2::Plan& pl, cudaStream_t st);
}  // namespace tada
