// Analytic test scenes on the device: the closed-form
// density / colour field of scene.py AnalyticScene evaluated per sample in
// place of the per-cell MLPs, so the reference's own ERT-bound and
// ESS-exactness acceptance checks run through the B200 marcher.
//
// Reference: scene.py:21-24 (_smoothstep), 27-53 (Sphere.density_at),
// 56-74 (Box.density_at), 77-135 (AnalyticScene.density_at / query_points).
// numpy evaluates these in the positions' dtype (float32) with NEP 50 weak
// Python scalars (cast to float32 before the operation); the device repeats
// that operation order with explicitly rounded intrinsics, so densities are
// bit-exact.  Colours use sinf (texture) and a 3-term dot (view tint), which
// numpy evaluates with its own SIMD sin / BLAS order: equal to ~1 ulp.
#include "gf_analytic.cuh"

namespace gf {

// AnalyticScene.query_points (scene.py:115-135) for one point
__device__ __forceinline__ void analytic_eval(const AnalyticDev& A, float x, float y, float z, float dx, float dy,
                                              float dz, float* rgb, float* sigma) {
  float s = 0.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
  for (int k = 0; k < A.n_prims; ++k) {
    const AnalyticPrim& p = A.prims[k];
    const float d = prim_density(p, x, y, z);
    if (d > 0.f && d >= s) {  // densest primitive colours the point
      c0 = p.color[0];
      c1 = p.color[1];
      c2 = p.color[2];
    }
    s = fmaxf(s, d);
  }
  if (A.texture_freq > 0.f) {
    const float f = A.texture_freq;
    const float s0 = sinf(__fmul_rn(f, x));
    const float s1 = sinf(__fadd_rn(__fmul_rn(f, y), 1.3f));
    const float s2 = sinf(__fadd_rn(__fmul_rn(f, z), 2.1f));
    const float inner = __fadd_rn(0.5f, __fmul_rn(__fmul_rn(__fmul_rn(0.5f, s0), s1), s2));
    const float mod = __fadd_rn(A.one_minus_amp, __fmul_rn(A.texture_amp, inner));
    c0 = __fmul_rn(c0, mod);
    c1 = __fmul_rn(c1, mod);
    c2 = __fmul_rn(c2, mod);
  }
  if (A.view_tint != 0.f) {
    const float dot = __fadd_rn(__fadd_rn(__fmul_rn(dx, A.tint_axis[0]), __fmul_rn(dy, A.tint_axis[1])),
                                __fmul_rn(dz, A.tint_axis[2]));
    const float shift = __fmul_rn(A.half_tint, dot);
    const float m = s > 0.f ? shift : 0.f;
    c0 = fminf(fmaxf(__fadd_rn(c0, m), 0.f), 1.f);
    c1 = fminf(fmaxf(__fadd_rn(c1, m), 0.f), 1.f);
    c2 = fminf(fmaxf(__fadd_rn(c2, m), 0.f), 1.f);
  }
  rgb[0] = c0;
  rgb[1] = c1;
  rgb[2] = c2;
  *sigma = s;
}

// render path: the marcher's kept samples of this round, all in one bucket
// (the analytic field has no cells): rows [0, offsets[1]) of the sorted records
__global__ void __launch_bounds__(256) k_field_analytic(AnalyticDev A, const uint32_t* __restrict__ offsets,
                                                        const float4* __restrict__ srec, const float4* __restrict__ ray_dir,
                                                        int stride_shift, uint32_t stride, float4* res) {
  const uint32_t n = offsets[1];
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    const float4 q = srec[r];
    const uint32_t idx = __float_as_uint(q.w);
    const uint32_t ray = stride_shift >= 0 ? idx >> stride_shift : idx / stride;
    const float4 d = ray_dir[ray];
    float rgb[3], s;
    analytic_eval(A, q.x, q.y, q.z, d.x, d.y, d.z, rgb, &s);
    res[idx] = make_float4(rgb[0], rgb[1], rgb[2], s);
  }
}

__global__ void __launch_bounds__(256) k_query_analytic(AnalyticDev A, const float* __restrict__ pos,
                                                        const float* __restrict__ dir, int64_t n, float* rgb,
                                                        float* sigma) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float c[3], s;
    analytic_eval(A, pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], dir[3 * i], dir[3 * i + 1], dir[3 * i + 2], c, &s);
    rgb[3 * i + 0] = c[0];
    rgb[3 * i + 1] = c[1];
    rgb[3 * i + 2] = c[2];
    sigma[i] = s;
  }
}

bool make_analytic(const gf_analytic_t* s, AnalyticDev* A) {
  if (!s || s->n_prims < 0 || s->n_prims > GF_MAX_PRIMS) return false;
  A->n_prims = s->n_prims;
  for (int k = 0; k < s->n_prims; ++k) {
    const gf_prim_t& p = s->prims[k];
    AnalyticPrim& q = A->prims[k];
    if (p.kind != 0 && p.kind != 1) return false;
    q.kind = p.kind;
    for (int a = 0; a < 3; ++a) {
      q.a[a] = (float)p.a[a];  // x.dtype.type(c) / np.asarray(lo, dtype=x.dtype)
      q.b[a] = (float)p.b[a];
      q.color[a] = (float)p.color[a];
    }
    q.radius = (float)p.radius;
    q.r2 = (float)(p.radius * p.radius);  // Python float product, compared as float32 (NEP 50)
    q.density = (float)p.density;
    q.feather = (float)p.feather;
  }
  A->texture_freq = (float)s->texture_freq;
  A->texture_amp = (float)s->texture_amp;
  A->one_minus_amp = (float)(1.0 - s->texture_amp);
  A->view_tint = (float)s->view_tint;
  A->half_tint = (float)(s->view_tint * 0.5);
  for (int a = 0; a < 3; ++a) A->tint_axis[a] = (float)s->tint_axis[a];
  return true;
}

void launch_field_analytic(const AnalyticDev& A, const uint32_t* offsets, const float4* srec, const float4* ray_dir,
                           int stride_shift, uint32_t stride, float4* res, int64_t max_rows, cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(max_rows > 0 ? max_rows : 1, 256),
                                                    (int64_t)num_sms() * 8);
  k_field_analytic<<<grid, 256, 0, st>>>(A, offsets, srec, ray_dir, stride_shift, stride, res);
}

void launch_query_analytic(const AnalyticDev& A, const float* pos, const float* dir, int64_t n, float* rgb,
                           float* sigma, cudaStream_t st) {
  if (n == 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(n, 256), (int64_t)num_sms() * 16);
  k_query_analytic<<<grid, 256, 0, st>>>(A, pos, dir, n, rgb, sigma);
}

}  // namespace gf
