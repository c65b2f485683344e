// Standalone device versions of the reference's pointwise primitives, so the
// public functions of the drop-in (core.*, occupancy.occupied_at,
// render.composite / generate_rays) run on the GPU like the fused path does.
#include "gf_common.cuh"

namespace gf {

// core.py:79-112 bin_point + flatten_cell_index
template <typename T>
__global__ void k_bin_points(GfGrid g, const T* __restrict__ x, int64_t n, int64_t* flat, int64_t* err) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T p[3];
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    p[a] = x[3 * i + a];
    if (!((double)p[a] >= g.b_min[a] && (double)p[a] <= g.b_max[a])) {
      atomicMin((unsigned long long*)err, (unsigned long long)(3 * i + a));
      ok = false;
    }
  }
  flat[i] = ok ? (int64_t)gf_flat_cell(g, p[0], p[1], p[2]) : -1;
}

// occupancy.py:76-79 occupied_at
template <typename T>
__global__ void k_occupied_at(GfGrid g, const uint8_t* __restrict__ bits, const T* __restrict__ x, int64_t n,
                              uint8_t* out, int64_t* err) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T p[3];
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    p[a] = x[3 * i + a];
    if (!((double)p[a] >= g.b_min[a] && (double)p[a] <= g.b_max[a])) {
      atomicMin((unsigned long long*)err, (unsigned long long)(3 * i + a));
      ok = false;
    }
  }
  uint8_t v = 0;
  if (ok) {
    uint32_t f = gf_flat_cell(g, p[0], p[1], p[2]);
    v = (bits[f >> 3] >> (f & 7)) & 1;
  }
  out[i] = v;
}

// core.py:52-68 clip_into
__global__ void k_clip(double lx, double ly, double lz, double hx, double hy, double hz, const float* __restrict__ x,
                       int64_t n, float* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[3 * i + 0] = gf_clip_component(x[3 * i + 0], lx, hx);
  out[3 * i + 1] = gf_clip_component(x[3 * i + 1], ly, hy);
  out[3 * i + 2] = gf_clip_component(x[3 * i + 2], lz, hz);
}

// core.py:132-152 positional_encode: angle = x * (2^k pi rounded to the
// input dtype), computed in the input dtype.
__device__ __forceinline__ float pi_scaled(float, int k) { return ldexpf(__int_as_float(0x40490FDB), k); }
__device__ __forceinline__ double pi_scaled(double, int k) { return ldexp(3.141592653589793, k); }
__device__ __forceinline__ void sincos_(float a, float* s, float* c) { sincosf(a, s, c); }
__device__ __forceinline__ void sincos_(double a, double* s, double* c) { sincos(a, s, c); }
__device__ __forceinline__ float expm1_(float a) { return expm1f(a); }
__device__ __forceinline__ double expm1_(double a) { return expm1(a); }

template <typename T>
__global__ void k_encode(const T* __restrict__ v, int64_t n, int dim, int L, int raw, T* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int width = dim * ((raw ? 1 : 0) + 2 * L);
  T* o = out + i * width;
  const T* x = v + i * dim;
  int c = 0;
  if (raw)
    for (int a = 0; a < dim; ++a) o[c++] = x[a];
  for (int k = 0; k < L; ++k) {
    const T f = pi_scaled(T(0), k);
    for (int a = 0; a < dim; ++a) {
      T s, cc;
      sincos_(x[a] * f, &s, &cc);
      o[c + a] = s;
      o[c + dim + a] = cc;
    }
    c += 2 * dim;
  }
}

// core.py:187-194 density_to_alpha
template <typename T>
__global__ void k_alpha(const T* __restrict__ s, const T* __restrict__ d, int64_t n, T* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = -expm1_((-s[i]) * d[i]);
}

// render.py:269-284 composite (one thread per ray): sum_j (T_j * a_j) * c_j
// accumulated in sample order, T by running product; float32 or float64 like
// the numpy original (which computes in the input dtype).
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }

template <typename T>
__global__ void k_composite(const T* __restrict__ col, const T* __restrict__ alpha, int64_t n_rays, int64_t n_s,
                            T* rgb, T* trans) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rays) return;
  T t = 1, a0 = 0, a1 = 0, a2 = 0;
  for (int64_t j = 0; j < n_s; ++j) {
    T a = alpha[r * n_s + j];
    T w = mul_(t, a);
    const T* c = col + (r * n_s + j) * 3;
    a0 = add_(a0, mul_(w, c[0]));
    a1 = add_(a1, mul_(w, c[1]));
    a2 = add_(a2, mul_(w, c[2]));
    t = mul_(t, sub_((T)1, a));
  }
  rgb[3 * r + 0] = a0;
  rgb[3 * r + 1] = a1;
  rgb[3 * r + 2] = a2;
  trans[r] = t;
}

// render.py:139-148 generate_rays
__global__ void k_gen_rays(gf_camera_t c, float* o, float* dir) {
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)c.width * c.height) return;
  int64_t px = g % c.width, py = g / c.width;
  double u = __ddiv_rn(__dsub_rn(__dadd_rn((double)px, 0.5), c.cx), c.fx);
  double v = __ddiv_rn(__dsub_rn(__dadd_rn((double)py, 0.5), c.cy), c.fy);
  double d[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    d[a] = __dadd_rn(__dadd_rn(__dmul_rn(u, c.c2w[4 * a + 0]), __dmul_rn(v, c.c2w[4 * a + 1])), c.c2w[4 * a + 2]);
  double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    dir[3 * g + a] = __double2float_rn(__ddiv_rn(d[a], nn));
    o[3 * g + a] = __double2float_rn(c.c2w[4 * a + 3]);
  }
}

static unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// out[j] = float32(x[idx[j]]) for (n, 3) rows; x float32 or float64 (the
// grouped layout of a query batch, batched.py:73-78, straight on the device)
template <typename T>
__global__ void k_gather_rows3(const T* __restrict__ x, const int64_t* __restrict__ idx, int64_t n, float* out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = idx[j];
#pragma unroll
    for (int a = 0; a < 3; ++a) out[3 * j + a] = (float)x[3 * s + a];
  }
}

void launch_gather_rows3(const void* x, int f64, const int64_t* idx, int64_t n, float* out, cudaStream_t st) {
  if (n <= 0) return;
  if (f64) k_gather_rows3<double><<<blocks(n, 256), 256, 0, st>>>((const double*)x, idx, n, out);
  else k_gather_rows3<float><<<blocks(n, 256), 256, 0, st>>>((const float*)x, idx, n, out);
}

void launch_bin_points(const GfGrid& g, const void* x, int f64, int64_t n, int64_t* flat, int64_t* err,
                       cudaStream_t st) {
  if (n <= 0) return;
  if (f64) k_bin_points<double><<<blocks(n, 256), 256, 0, st>>>(g, (const double*)x, n, flat, err);
  else k_bin_points<float><<<blocks(n, 256), 256, 0, st>>>(g, (const float*)x, n, flat, err);
}
void launch_occupied_at(const GfGrid& g, const uint8_t* bits, const void* x, int f64, int64_t n, uint8_t* out,
                        int64_t* err, cudaStream_t st) {
  if (n <= 0) return;
  if (f64) k_occupied_at<double><<<blocks(n, 256), 256, 0, st>>>(g, bits, (const double*)x, n, out, err);
  else k_occupied_at<float><<<blocks(n, 256), 256, 0, st>>>(g, bits, (const float*)x, n, out, err);
}
void launch_clip(const double* lo, const double* hi, const float* x, int64_t n, float* out, cudaStream_t st) {
  if (n > 0) k_clip<<<blocks(n, 256), 256, 0, st>>>(lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], x, n, out);
}
void launch_encode(const void* v, int f64, int64_t n, int dim, int L, int raw, void* out, cudaStream_t st) {
  if (n <= 0) return;
  if (f64) k_encode<double><<<blocks(n, 128), 128, 0, st>>>((const double*)v, n, dim, L, raw, (double*)out);
  else k_encode<float><<<blocks(n, 128), 128, 0, st>>>((const float*)v, n, dim, L, raw, (float*)out);
}
void launch_alpha(const void* s, const void* d, int f64, int64_t n, void* out, cudaStream_t st) {
  if (n <= 0) return;
  if (f64) k_alpha<double><<<blocks(n, 256), 256, 0, st>>>((const double*)s, (const double*)d, n, (double*)out);
  else k_alpha<float><<<blocks(n, 256), 256, 0, st>>>((const float*)s, (const float*)d, n, (float*)out);
}
void launch_composite(const float* c, const float* a, int64_t nr, int64_t ns, float* rgb, float* tr, cudaStream_t st) {
  if (nr > 0) k_composite<float><<<blocks(nr, 128), 128, 0, st>>>(c, a, nr, ns, rgb, tr);
}
void launch_composite_f64(const double* c, const double* a, int64_t nr, int64_t ns, double* rgb, double* tr,
                          cudaStream_t st) {
  if (nr > 0) k_composite<double><<<blocks(nr, 128), 128, 0, st>>>(c, a, nr, ns, rgb, tr);
}
// render.py:151-171 intersect_aabb: float64 slab test (division, parallel
// axes by the inside test), t0 = max(near, 0), t1 = min(far)
__global__ void k_intersect_aabb(const double* __restrict__ o, const double* __restrict__ d, int64_t n, double lx,
                                 double ly, double lz, double hx, double hy, double hz, double* t0, double* t1) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double lo[3] = {lx, ly, lz}, hi[3] = {hx, hy, hz};
  double near = -INFINITY, far = INFINITY;
  for (int a = 0; a < 3; ++a) {
    const double oa = o[3 * i + a], da = d[3 * i + a];
    double nl, fr;
    if (da == 0.0) {
      const bool inside = oa >= lo[a] && oa <= hi[a];
      nl = inside ? -INFINITY : INFINITY;
      fr = inside ? INFINITY : -INFINITY;
    } else {
      const double ta = __ddiv_rn(__dsub_rn(lo[a], oa), da), tb = __ddiv_rn(__dsub_rn(hi[a], oa), da);
      nl = fmin(ta, tb);
      fr = fmax(ta, tb);
    }
    near = a == 0 ? nl : fmax(near, nl);
    far = a == 0 ? fr : fmin(far, fr);
  }
  t0[i] = fmax(near, 0.0);
  t1[i] = far;
}

// render.py:256-258 sample_ray positions: f32(o + (t0 + (j + jit_j) seg) d), float64 arithmetic in numpy's order
__global__ void k_ray_samples(double ox, double oy, double oz, double dx, double dy, double dz, double t0, double seg,
                              const double* __restrict__ jit, int64_t k, float* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= k) return;
  const double t = __dadd_rn(t0, __dmul_rn(__dadd_rn((double)j, jit[j]), seg));
  out[3 * j + 0] = __double2float_rn(__dadd_rn(ox, __dmul_rn(t, dx)));
  out[3 * j + 1] = __double2float_rn(__dadd_rn(oy, __dmul_rn(t, dy)));
  out[3 * j + 2] = __double2float_rn(__dadd_rn(oz, __dmul_rn(t, dz)));
}

void launch_intersect_aabb(const double* o, const double* d, int64_t n, const double* lo, const double* hi, double* t0,
                           double* t1, cudaStream_t st) {
  if (n > 0) k_intersect_aabb<<<blocks(n, 256), 256, 0, st>>>(o, d, n, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2], t0, t1);
}

void launch_ray_samples(const double* o, const double* d, double t0, double seg, const double* jit, int64_t k,
                        float* out, cudaStream_t st) {
  if (k > 0)
    k_ray_samples<<<blocks(k, 256), 256, 0, st>>>(o[0], o[1], o[2], d[0], d[1], d[2], t0, seg, jit, k, out);
}

void launch_gen_rays(const gf_camera_t& c, float* o, float* d, cudaStream_t st) {
  int64_t n = (int64_t)c.width * c.height;
  if (n > 0) k_gen_rays<<<blocks(n, 256), 256, 0, st>>>(c, o, d);
}

}  // namespace gf
