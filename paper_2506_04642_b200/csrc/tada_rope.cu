// RoPE for the compressed-cache append path.
//
// Reference: tensor.py:63-89 apply_rope / 92-105 rotate_heads.  Each adjacent (2j, 2j+1) pair of a
// head row is rotated by angle pos * base^(-2j/D).  The angles and their cos/sin are computed by the
// host in f64 exactly as the reference does (np.cos(angles).astype(f32)) and handed over as a table
// rope_cs[pos][j] = (cos, sin) f32, so the device never evaluates a transcendental and the rotation
// is bit-identical to numpy:
//   out[2j]   = f32(f32(e * c) - f32(o * s))
//   out[2j+1] = f32(f32(e * s) + f32(o * c))
// (separately rounded products, no FMA contraction: numpy materialises every temporary in f32).
#include <cuda_runtime.h>

#include "tada_common.cuh"

namespace tada {

__device__ __forceinline__ void rope_pair(float e, float o, float c, float s, float& oe, float& oo) {
  oe = __fsub_rn(__fmul_rn(e, c), __fmul_rn(o, s));
  oo = __fadd_rn(__fmul_rn(e, s), __fmul_rn(o, c));
}

// one thread per (row, pair); row = (token, head), token = row / heads
template <typename T>
__global__ void rope_kernel(const T* __restrict__ x, int64_t rows, int heads, int D, const int32_t* __restrict__ pos,
                            const float2* __restrict__ cs, int rope_rows, float* __restrict__ out,
                            int32_t* __restrict__ err) {
  const int half = D >> 1;
  const int64_t n = rows * half;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = i / half;
    const int j = int(i - row * half);
    const int p = pos[row / heads];
    if (p < 0 || p >= rope_rows) {  // the host validates positions; this guards device-side ones
      if (err) atomicOr(err, 2);
      continue;
    }
    const float2 c = cs[int64_t(p) * half + j];
    const float e = to_f32(x[row * D + 2 * j]), o = to_f32(x[row * D + 2 * j + 1]);
    float oe, oo;
    rope_pair(e, o, c.x, c.y, oe, oo);
    out[row * D + 2 * j] = oe;
    out[row * D + 2 * j + 1] = oo;
  }
}

}  // namespace tada

using namespace tada;

extern "C" int tada_apply_rope(const void* x, int32_t dtype, int64_t n_tok, int32_t heads, int32_t head_dim,
                               const int32_t* positions, const float* rope_cs, int32_t rope_rows, float* out,
                               int32_t* err_flag, void* stream) {
  if (dtype != TADA_F32 && dtype != TADA_BF16) return fail(TADA_ERR_CONFIG, "dtype must be f32 or bf16");
  if (head_dim <= 0 || head_dim % 2 != 0) return fail(TADA_ERR_CONFIG, "rotary head_dim must be a positive even integer");
  if (n_tok < 0 || heads <= 0 || rope_rows < 0) return fail(TADA_ERR_SHAPE, "bad rope geometry");
  if (n_tok == 0) return TADA_OK;
  if (!x || !positions || !rope_cs || !out) return fail(TADA_ERR_SHAPE, "null buffer");
  const int64_t rows = n_tok * heads, n = rows * (head_dim / 2);
  const int64_t blocks = (n + 255) / 256;
  const int grid = int(blocks < 148 * 16 ? blocks : 148 * 16);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const float2* cs = reinterpret_cast<const float2*>(rope_cs);
  if (dtype == TADA_F32)
    rope_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(x), rows, heads, head_dim, positions, cs,
                                            rope_rows, out, err_flag);
  else
    rope_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), rows, heads, head_dim,
                                                    positions, cs, rope_rows, out, err_flag);
  return check_launch("apply_rope");
}
