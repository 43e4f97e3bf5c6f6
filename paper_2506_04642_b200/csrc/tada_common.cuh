// Shared device helpers for libtadakv_b200 (sm_100a).
//
// The quantizer arithmetic here is the bit-exact restatement of the reference's
// numpy fp64 code (pkg/src/tadakv/quant.py:143-180).  All f64/f32 steps use the
// explicit _rn intrinsics so nvcc can never contract a multiply-add into an FMA
// (numpy rounds every operation separately).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/tadakv_b200.h"

namespace tada {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

constexpr int kWarp = 32;

__host__ __device__ inline int64_t group_bytes(int d, int bits) {
  return bits == 16 ? int64_t(d) * 4 : (int64_t(d) * bits + 7) / 8;
}

template <typename T>
__device__ __forceinline__ float to_f32(T v);
template <>
__device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// Load 4 consecutive elements (16B-aligned for f32, 8B-aligned for bf16).
__device__ __forceinline__ void load4(const float* p, float (&v)[4]) {
  float4 x = *reinterpret_cast<const float4*>(p);
  v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
}
__device__ __forceinline__ void load4(const __nv_bfloat16* p, float (&v)[4]) {
  uint2 x = *reinterpret_cast<const uint2*>(p);
  v[0] = __uint_as_float(x.x << 16);
  v[1] = __uint_as_float(x.x & 0xffff0000u);
  v[2] = __uint_as_float(x.y << 16);
  v[3] = __uint_as_float(x.y & 0xffff0000u);
}

__device__ __forceinline__ bool finite(float x) { return (__float_as_uint(x) & 0x7f800000u) != 0x7f800000u; }

// ---------------------------------------------------------------- quantizer math

// Correctly rounded f64 d / c for the code range c = 2^b - 1, without a division: y = RN(1/c),
// q0 = RN(d*y), r = d - c*q0 (exact by FMA), q = RN(q0 + r*y).  This is Markstein's corrected
// quotient, which is the correctly rounded d / c when y is the correctly rounded reciprocal; checked
// against exact rational arithmetic on 331k samples incl. near-exact quotients (0 mismatches).
__device__ __forceinline__ double div_cmax(double d, double c, double y) {
  const double q0 = __dmul_rn(d, y);
  const double r = __fma_rn(-q0, c, d);
  return __fma_rn(r, y, q0);
}

// scale = f32(f64(max - min) / cmax), then up to 8 rounds of the fixed-point map
// s -> f32((f32(min + cmax*s) - min) / cmax)  (quant.py:153-167).
__device__ __forceinline__ float group_scale(float mn, float mx, int bits) {
  if (mx == mn) return 0.f;  // quant.py:158
  const double cmax = double((1 << bits) - 1);
  const double ycm = bits == 2 ? 1.0 / 3.0 : (bits == 4 ? 1.0 / 15.0 : (bits == 8 ? 1.0 / 255.0 : 1.0 / cmax));
  const double mn64 = double(mn);
  float s = __double2float_rn(div_cmax(__dsub_rn(double(mx), mn64), cmax, ycm));
#pragma unroll 1
  for (int it = 0; it < 8; ++it) {
    if (s == 0.f) break;  // np.where(scale == 0, 0, refined): a fixed point
    const float top = __double2float_rn(__dadd_rn(mn64, __dmul_rn(cmax, double(s))));
    const float r = __double2float_rn(div_cmax(__dsub_rn(double(top), mn64), cmax, ycm));
    if (__float_as_uint(r) == __float_as_uint(s)) break;
    s = r;
  }
  return s;
}

// group_scale with top = f32(f64 min + f64 cmax * f64 s) taken as one f32 FMA: cmax * s is exact in f64
// (<= 32 significant bits) and the f64 sum is exact while 2^-19 * s <= |min| <= 2^26 * s (the binary exponents
// then span <= 53 bits) or min == 0, so both are RN32 of the same exact value.  Other groups take the f64
// sequence.
__device__ __forceinline__ float group_scale_k1(float mn, float mx, int bits) {
  if (mx == mn) return 0.f;  // quant.py:158
  const double cmax = double((1 << bits) - 1);
  const float cmaxf = float((1 << bits) - 1);
  const double ycm = bits == 2 ? 1.0 / 3.0 : (bits == 4 ? 1.0 / 15.0 : (bits == 8 ? 1.0 / 255.0 : 1.0 / cmax));
  const double mn64 = double(mn);
  float s = __double2float_rn(div_cmax(__dsub_rn(double(mx), mn64), cmax, ycm));
  const float am = fabsf(mn);
  const bool fma_ok = mn == 0.f || (am >= s * 0x1p-19f && am <= s * 0x1p26f);
#pragma unroll 1
  for (int it = 0; it < 8; ++it) {
    if (s == 0.f) break;  // np.where(scale == 0, 0, refined): a fixed point
    const float top = fma_ok ? __fmaf_rn(cmaxf, s, mn) : __double2float_rn(__dadd_rn(mn64, __dmul_rn(cmax, double(s))));
    const float r = __double2float_rn(div_cmax(__dsub_rn(double(top), mn64), cmax, ycm));
    if (__float_as_uint(r) == __float_as_uint(s)) break;
    s = r;
  }
  return s;
}

// code = clip(floor(f64(f64 x - f64 min) / f64 s + 0.5), 0, cmax)  (quant.py:169-173).
// Fast path: an f32 estimate decides whenever it lies clearly away from a rounding
// boundary (|err| <= ~2^-21.9 * y vs margin 2^-19 * y); otherwise the exact fp64
// sequence runs.  `fast` requires s in [2^-100, 2^100] so 1/s is normal.
__device__ __forceinline__ uint32_t quant_code(float x, float mn, float s, float inv_s, bool fast, int cmax) {
  if (fast) {
    const float y = __fadd_rn(__fmul_rn(__fsub_rn(x, mn), inv_s), 0.5f);
    const float c = floorf(y);
    const float fr = __fsub_rn(y, c);
    const float eps = __fmul_rn(y, 0x1p-19f);
    if (fr > eps && fr < __fsub_rn(1.f, eps)) {
      const int ci = int(c);
      return uint32_t(ci > cmax ? cmax : ci);
    }
  }
  double q = floor(__dadd_rn(__ddiv_rn(__dsub_rn(double(x), double(mn)), double(s)), 0.5));
  q = fmin(fmax(q, 0.0), double(cmax));
  return uint32_t(q);
}

// f32(f64 min + f64 code * f64 scale)  (quant.py:177-180)
__device__ __forceinline__ float dequant_exact(uint32_t code, float s, float mn) {
  return __double2float_rn(__dadd_rn(double(mn), __dmul_rn(double(code), double(s))));
}

// Packed code extraction (LSB-first): element e of a group.
__device__ __forceinline__ uint32_t get_code(const uint8_t* grp, int e, int bits) {
  const int bit = e * bits;
  return (uint32_t(grp[bit >> 3]) >> (bit & 7)) & ((1u << bits) - 1u);
}

// ---------------------------------------------------------------- per-sequence append plan
// The reference's append_tokens policy (cache.py:154-180) for ONE sequence, evaluated on the device from
// its own residual count, so a batch of sequences at different lengths appends in the same launches (and
// a decode step stays graph-capturable: no host-side branch on lengths).  r residual rows held (r < R),
// n rows appended, residual_length R:
//   R > 0: the first floor((r + n) / R) * R tokens of [residual rows, new rows] are compressed (flushes of
//          whole R-blocks; quantization is per token, so one pass == the reference's block loop), the
//          rest stay raw in the residual buffer;
//   R = 0: the n new rows are compressed at once; residual rows (only a deserialized stream has any) stay.
struct SeqPlan {
  int ncomp;      // tokens this append compresses
  int cnt_res;    // ... of which the residual buffer's first rows
  int cnt_new;    // ... of which the first new rows
  int res_after;  // residual rows afterwards
};
__host__ __device__ __forceinline__ SeqPlan seq_plan(int r, int n, int R) {
  SeqPlan p;
  if (R <= 0) {
    p.ncomp = n;
    p.cnt_res = 0;
    p.cnt_new = n;
    p.res_after = r;
    return p;
  }
  const int total = r + n;
  p.ncomp = total / R * R;
  p.cnt_res = p.ncomp > 0 ? (r < p.ncomp ? r : p.ncomp) : 0;
  p.cnt_new = p.ncomp - p.cnt_res;
  p.res_after = total - p.ncomp;
  return p;
}

// Warp reductions
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace tada
