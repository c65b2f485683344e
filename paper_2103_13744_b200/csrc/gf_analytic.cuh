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

int num_sms();
bool make_analytic(const gf_analytic_t* s, AnalyticDev* A);
void launch_field_analytic(const AnalyticDev& A, const uint32_t* offsets, const float4* srec, const float4* ray_dir,
                           int stride_shift, uint32_t stride, float4* res, int64_t max_rows, cudaStream_t st);
void launch_query_analytic(const AnalyticDev& A, const float* pos, const float* dir, int64_t n, float* rgb,
                           float* sigma, cudaStream_t st);

}  // namespace gf
