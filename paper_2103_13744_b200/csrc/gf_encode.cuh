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

// ---- packed float32 pairs (FMUL2 / FADD2 / FFMA2 on sm_100): each lane of
// the pair is the same IEEE round-to-nearest operation as the scalar form
struct F2 {
  unsigned long long v;
};
__device__ __forceinline__ F2 f2(float a, float b) {
  F2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2_split(F2 p, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(p.v)); }
__device__ __forceinline__ F2 f2_mul(F2 a, F2 b) {
  F2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 f2_add(F2 a, F2 b) {
  F2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 f2_sub(F2 a, F2 b) {
  F2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
__device__ __forceinline__ F2 f2_fma(F2 a, F2 b, F2 c) {
  F2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}

// sincos_scaled for two independent (value, octave) pairs at once: the
// angle products and the 2pi reduction run as f32x2 (identical roundings:
// rint(-t) == -rint(t) and fma(n', hi, a) with n' = -n is fmaf(-n, hi, a))
__device__ __forceinline__ void sincos_scaled2(float x0, int k0, float x1, int k1, float* s0, float* c0, float* s1,
                                               float* c1) {
  const F2 a = f2_mul(f2(x0, x1), f2(__int_as_float(0x40490FDB + (k0 << 23)), __int_as_float(0x40490FDB + (k1 << 23))));
  // n = -rint(a / 2pi): round to nearest even by the 1.5 * 2^23 shifter
  // (|a / 2pi| <= 2^9 here), on the FMA pipe instead of two FRND on XU
  const F2 M = f2(12582912.0f, 12582912.0f);
  const F2 n = f2_sub(f2_add(f2_mul(a, f2(-0.15915494309189535f, -0.15915494309189535f)), M), M);
  F2 r = f2_fma(n, f2(6.28125f, 6.28125f), a);
  r = f2_fma(n, f2(1.9353071795864769e-3f, 1.9353071795864769e-3f), r);
  float r0, r1;
  f2_split(r, r0, r1);
  __sincosf(r0, s0, c0);
  __sincosf(r1, s1, c1);
}

// one double-angle step for two independent chains: s' = (s + s) c,
// c' = (c - s)(c + s)
__device__ __forceinline__ void double_angle2(F2& s, F2& c) {
  const F2 s2 = f2_mul(f2_add(s, s), c);
  c = f2_mul(f2_sub(c, s), f2_add(c, s));
  s = s2;
}

// the same step in 4 paired ops: s' = (s + s) c, c' = fma(c, c, -s s).  An
// error delta in (s, c) grows to at most ~2 delta per step, as above.
__device__ __forceinline__ void double_angle2_fma(F2& s, F2& c) {
  const F2 s2 = f2_mul(f2_add(s, s), c);
  const F2 ss = f2_mul(s, s);
  F2 nss;
  asm("{\n\t.reg .b64 t;\n\tmov.b64 t, %1;\n\txor.b64 %0, t, 0x8000000080000000;\n\t}" : "=l"(nss.v) : "l"(ss.v));
  c = f2_fma(c, c, nss);
  s = s2;
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
