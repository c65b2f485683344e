// Positional encoding helpers shared by the tensor-core MLP (per sample
// position) and the ray setup (per ray view direction, computed once and
// reused by every sample of the ray).
//
// Reference: core.py:132-152 positional_encode: [v, sin(fl32(v*fl32(2^k pi))),
// cos(...)] per octave k, layout raw(3) then for each k: sin(xyz), cos(xyz).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace gf {

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  uint32_t r;  // one F2FP.F16.F32.PACK_AB; low half = a
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

// relu(fp16(a)), relu(fp16(b)) == fp16(relu(a)), fp16(relu(b)) in one F2FP.RELU
__device__ __forceinline__ uint32_t pack_h2_relu(float a, float b) {
  uint32_t r;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

// two IEEE float32 adds in one FADD2 (sm_100)
__device__ __forceinline__ void fadd2(float& x0, float& x1, float b0, float b1) {
  asm("{\n\t.reg .b64 a, b;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 b, {%2, %3};\n\t"
      "add.rn.f32x2 a, a, b;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(x0), "+f"(x1)
      : "f"(b0), "f"(b1));
}

// sin / cos of x * 2^k * pi: the angle is formed exactly as numpy forms it
// (fl32(x * fl32(2^k pi)) == 2^k fl32(x*pi)), reduced by 2pi with a two-term
// Cody-Waite split, then MUFU sin/cos (~5e-7 abs).
__device__ __forceinline__ void sincos_scaled(float x, int k, float* s, float* c) {
  const float a = __fmul_rn(x, __int_as_float(0x40490FDB + (k << 23)));
  const float n = rintf(a * 0.15915494309189535f);
  float r = fmaf(-n, 6.28125f, a);          // 2pi_hi (exact times n <= 2^9)
  r = fmaf(-n, 1.9353071795864769e-3f, r);  // 2pi_lo
  __sincosf(r, s, c);
}

// octaves k < L: MUFU anchors every third octave, double-angle steps in
// between (max abs error 2.6e-6 vs 4.9e-4 fp16 operand rounding)
template <int L>
__device__ __forceinline__ void encode_octaves(float x, float* s, float* c) {
#pragma unroll
  for (int k = 0; k < L; ++k) {
    if (k % 3 == 0) {
      sincos_scaled(x, k, &s[k], &c[k]);
    } else {
      const float sp = s[k - 1], cp = c[k - 1];
      s[k] = 2.0f * sp * cp;
      c[k] = (cp - sp) * (cp + sp);
    }
  }
}

// gamma(d) for the direction layer as 32 fp16 values (27 used, zero padded):
// the exact K-chunk image (4 x 8 features) the MLP stores next to the
// feature vector in its direction-layer operand.
__device__ __forceinline__ void encode_direction_h(const float* d, uint4* out) {
  float e[32];
  e[0] = d[0]; e[1] = d[1]; e[2] = d[2];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float s[4], c[4];
    encode_octaves<4>(d[a], s, c);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      e[3 + 6 * k + a] = s[k];
      e[6 + 6 * k + a] = c[k];
    }
  }
#pragma unroll
  for (int j = 27; j < 32; ++j) e[j] = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    out[q] = make_uint4(pack_h2(e[8 * q + 0], e[8 * q + 1]), pack_h2(e[8 * q + 2], e[8 * q + 3]),
                        pack_h2(e[8 * q + 4], e[8 * q + 5]), pack_h2(e[8 * q + 6], e[8 * q + 7]));
}

}  // namespace gf
