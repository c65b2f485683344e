// Device form of gf_analytic_t (include/gridfield_b200.h): float32 constants
// exactly as numpy's float32 evaluation sees them (scene.py, NEP 50).
#pragma once
#include <algorithm>

#include "gf_common.cuh"

namespace gf {

struct AnalyticPrim {
  int kind;          // 0 sphere, 1 box
  float a[3], b[3];  // sphere: centre; box: lo, hi
  float color[3];
  float radius, r2, density, feather;
};

struct AnalyticDev {
  int n_prims;
  AnalyticPrim prims[GF_MAX_PRIMS];
  float texture_freq, texture_amp, one_minus_amp, view_tint, half_tint;
  float tint_axis[3];
};

// scene.py:21-24 (_smoothstep), 40-53 (Sphere.density_at), 65-74 (Box.density_at)
__device__ __forceinline__ float smoothstep32(float u) {
  u = fminf(fmaxf(u, 0.f), 1.f);  // np.clip(u, 0.0, 1.0)
  return __fmul_rn(__fmul_rn(u, u), __fsub_rn(3.0f, __fmul_rn(2.0f, u)));
}

__device__ __forceinline__ float prim_density(const AnalyticPrim& p, float x, float y, float z) {
  if (p.kind == 0) {  // Sphere.density_at (scene.py:40-53)
    const float tx = __fsub_rn(x, p.a[0]), ty = __fsub_rn(y, p.a[1]), tz = __fsub_rn(z, p.a[2]);
    float d2 = __fmul_rn(tx, tx);
    d2 = __fadd_rn(d2, __fmul_rn(ty, ty));
    d2 = __fadd_rn(d2, __fmul_rn(tz, tz));
    if (!(d2 < p.r2)) return 0.f;
    if (!(p.feather > 0.f)) return p.density;
    const float dist = __fsqrt_rn(d2);
    return __fmul_rn(p.density, smoothstep32(__fdiv_rn(__fsub_rn(p.radius, dist), p.feather)));
  }
  // Box.density_at (scene.py:65-74)
  const float dx = fminf(__fsub_rn(x, p.a[0]), __fsub_rn(p.b[0], x));
  const float dy = fminf(__fsub_rn(y, p.a[1]), __fsub_rn(p.b[1], y));
  const float dz = fminf(__fsub_rn(z, p.a[2]), __fsub_rn(p.b[2], z));
  const float depth = fminf(fminf(dx, dy), dz);
  if (!(depth > 0.f)) return 0.f;
  if (!(p.feather > 0.f)) return p.density;
  return __fmul_rn(p.density, smoothstep32(__fdiv_rn(depth, p.feather)));
}

// AnalyticScene.density_at (scene.py:107-113): max over the primitives
__device__ __forceinline__ float analytic_density(const AnalyticDev& A, float x, float y, float z) {
  float s = 0.f;
  for (int k = 0; k < A.n_prims; ++k) s = fmaxf(s, prim_density(A.prims[k], x, y, z));
  return s;
}

int num_sms();
bool make_analytic(const gf_analytic_t* s, AnalyticDev* A);
void launch_composite(const float* c, const float* a, int64_t nr, int64_t ns, float* rgb, float* tr, cudaStream_t st);
void launch_brute_force(const AnalyticDev& A, const gf_camera_t& cam, const double* lo, const double* hi, int64_t ray0,
                        int64_t n_rays, int n, const float* bg, float* alpha, float* color, float* rgb, float* trans,
                        float* out, cudaStream_t st);
void launch_empty_cells(const gf_analytic_t& S, const int* res, uint8_t* out, cudaStream_t st);
void launch_field_analytic(const AnalyticDev& A, const uint32_t* offsets, const float4* srec, const float4* ray_dir,
                           int stride_shift, uint32_t stride, float4* res, int64_t max_rows, cudaStream_t st);
void launch_query_analytic(const AnalyticDev& A, const float* pos, const float* dir, int64_t n, float* rgb,
                           float* sigma, cudaStream_t st);

}  // namespace gf
