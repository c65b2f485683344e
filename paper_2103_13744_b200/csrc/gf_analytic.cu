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
#include <algorithm>

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

// scene.py:214-252 render_brute_force, segment stage: ray r's segment i of
// n (Simpson optical depth from the half-step lattice ends 2i, 2i+2 and
// midpoint 2i+1, colour at the midpoint), float64 placement, float32 field
__global__ void __launch_bounds__(256) k_brute_segments(AnalyticDev A, gf_camera_t cam, double lx, double ly,
                                                        double lz, double hx, double hy, double hz, int64_t ray0,
                                                        int64_t n_rays, int n, float* alpha, float* color) {
  const double lo[3] = {lx, ly, lz}, hi[3] = {hx, hy, hz};
  const int64_t total = n_rays * (int64_t)n;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rl = q / n, g = ray0 + rl;
    const int i = (int)(q % n);
    // render.py:139-148 generate_rays (float32 rays), then .astype(float64)
    const int64_t px = g % cam.width, py = g / cam.width;
    const double u = __ddiv_rn(__dsub_rn(__dadd_rn((double)px, 0.5), cam.cx), cam.fx);
    const double v = __ddiv_rn(__dsub_rn(__dadd_rn((double)py, 0.5), cam.cy), cam.fy);
    double dv[3];
    for (int a = 0; a < 3; ++a)
      dv[a] = __dadd_rn(__dadd_rn(__dmul_rn(u, cam.c2w[4 * a + 0]), __dmul_rn(v, cam.c2w[4 * a + 1])), cam.c2w[4 * a + 2]);
    const double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dv[0], dv[0]), __dmul_rn(dv[1], dv[1])),
                                           __dmul_rn(dv[2], dv[2])));
    float d32[3];
    double o[3], d[3];
    for (int a = 0; a < 3; ++a) {
      d32[a] = __double2float_rn(__ddiv_rn(dv[a], nn));
      d[a] = (double)d32[a];
      o[a] = (double)__double2float_rn(cam.c2w[4 * a + 3]);
    }
    // render.py:151-171 slab test
    double near = -INFINITY, far = INFINITY;
    for (int a = 0; a < 3; ++a) {
      double nl, fr;
      if (d[a] == 0.0) {
        const bool inside = o[a] >= lo[a] && o[a] <= hi[a];
        nl = inside ? -INFINITY : INFINITY;
        fr = inside ? INFINITY : -INFINITY;
      } else {
        const double ta = __ddiv_rn(__dsub_rn(lo[a], o[a]), d[a]), tb = __ddiv_rn(__dsub_rn(hi[a], o[a]), d[a]);
        nl = fmin(ta, tb);
        fr = fmax(ta, tb);
      }
      near = a == 0 ? nl : fmax(near, nl);
      far = a == 0 ? fr : fmin(far, fr);
    }
    const double t0 = fmax(near, 0.0), t1 = far;
    float al = 0.f, c[3] = {0.f, 0.f, 0.f};
    if (t1 > t0) {  // a miss blends nothing: its composite is exactly the background
      const double seg = __ddiv_rn(__dsub_rn(t1, t0), (double)n), hs = __dmul_rn(0.5, seg);
      float sg[3];
      for (int m = 0; m < 3; ++m) {
        const double t = __dadd_rn(t0, __dmul_rn((double)(2 * i + m), hs));
        float p[3];
        for (int a = 0; a < 3; ++a) {  // .astype(float32), then np.clip against the float64 box
          const double pa = (double)__double2float_rn(__dadd_rn(o[a], __dmul_rn(t, d[a])));
          p[a] = __double2float_rn(fmin(fmax(pa, lo[a]), hi[a]));
        }
        float cc[3];
        analytic_eval(A, p[0], p[1], p[2], d32[0], d32[1], d32[2], cc, &sg[m]);
        if (m == 1) { c[0] = cc[0]; c[1] = cc[1]; c[2] = cc[2]; }
      }
      // depth = (seg32 / 6) * (s_2i + 4 s_2i+1 + s_2i+2), alpha = -expm1(-depth)
      const float depth = __fmul_rn(__fdiv_rn(__double2float_rn(seg), 6.0f),
                                    __fadd_rn(__fadd_rn(sg[0], __fmul_rn(4.0f, sg[1])), sg[2]));
      al = -expm1f(-depth);
    }
    alpha[q] = al;
    color[3 * q + 0] = c[0];
    color[3 * q + 1] = c[1];
    color[3 * q + 2] = c[2];
  }
}

// out = clip(rgb + T * bg, 0, 1) (scene.py:249-252)
__global__ void k_brute_finish(const float* rgb, const float* trans, int64_t n, float b0, float b1, float b2,
                               float* out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float bg[3] = {b0, b1, b2};
  for (int a = 0; a < 3; ++a)
    out[3 * r + a] = fminf(fmaxf(__fadd_rn(rgb[3 * r + a], __fmul_rn(trans[r], bg[a])), 0.f), 1.f);
}

void launch_brute_force(const AnalyticDev& A, const gf_camera_t& cam, const double* lo, const double* hi, int64_t ray0,
                        int64_t n_rays, int n, const float* bg, float* alpha, float* color, float* rgb, float* trans,
                        float* out, cudaStream_t st) {
  if (n_rays <= 0) return;
  const int64_t total = n_rays * (int64_t)n;
  const unsigned grid = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(total, 256), (int64_t)num_sms() * 16);
  k_brute_segments<<<grid, 256, 0, st>>>(A, cam, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], ray0, n_rays, n, alpha,
                                         color);
  launch_composite(color, alpha, n_rays, n, rgb, trans, st);  // render.py:269-284, sequential in sample order
  k_brute_finish<<<(unsigned)gf_div_up<int64_t>(n_rays, 128), 128, 0, st>>>(rgb, trans, n_rays, bg[0], bg[1], bg[2],
                                                                           out);
}

// scene.py:186-211 analytically_empty_cells: a cell is touched by a sphere
// if the clamped distance from the centre is within the radius, by a box on
// interval overlap (float64); out[c] = 1 for untouched cells
__global__ void k_empty_cells(gf_analytic_t S, int rx, int ry, int rz, uint8_t* out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)rx * ry * rz;
  if (c >= n) return;
  const int64_t ix = c % rx, iy = (c / rx) % ry, iz = c / ((int64_t)rx * ry);
  const int64_t id[3] = {ix, iy, iz};
  const int res[3] = {rx, ry, rz};
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    const double cell = __ddiv_rn(__dsub_rn(S.b_max[a], S.b_min[a]), (double)res[a]);
    lo[a] = __dadd_rn(S.b_min[a], __dmul_rn((double)id[a], cell));
    hi[a] = __dadd_rn(lo[a], cell);
  }
  bool touched = false;
  for (int k = 0; k < S.n_prims && !touched; ++k) {
    const gf_prim_t& p = S.prims[k];
    if (p.kind == 0) {
      double d2 = 0.0;
      for (int a = 0; a < 3; ++a) {
        const double q = __dsub_rn(fmin(fmax(p.a[a], lo[a]), hi[a]), p.a[a]);
        d2 = __dadd_rn(d2, __dmul_rn(q, q));
      }
      touched = __dsqrt_rn(d2) <= p.radius;
    } else {
      touched = hi[0] >= p.a[0] && lo[0] <= p.b[0] && hi[1] >= p.a[1] && lo[1] <= p.b[1] && hi[2] >= p.a[2] &&
                lo[2] <= p.b[2];
    }
  }
  out[c] = touched ? 0 : 1;
}

void launch_empty_cells(const gf_analytic_t& S, const int* res, uint8_t* out, cudaStream_t st) {
  const int64_t n = (int64_t)res[0] * res[1] * res[2];
  if (n > 0) k_empty_cells<<<(unsigned)gf_div_up<int64_t>(n, 256), 256, 0, st>>>(S, res[0], res[1], res[2], out);
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
