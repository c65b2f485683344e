// mlp.forward / mlp.backward (mlp.py:222-316) on the device for ANY manifest
// and a stack of networks, in float32 or float64: the reference's plain
// (non-grouped) network API, which takes already-encoded inputs
// x_enc (*lead, B, pos_dim) / d_enc (*lead, B, dir_dim) with the stacked
// parameters (*lead, out, in) (mlp.py:112-174).
//
// forward: one CTA per 32 rows of one network, activations in shared memory
// transposed ([feature][row]); every layer is a sequential FMA chain over its
// inputs from 0, the bias added after the dot product -- the same arithmetic
// as the fused SIMT kernel (gf_mlp_simt.cuh), so grouped_forward and
// mlp.forward agree bit for bit on the same network (test_batched.py:61-70).
// The activations backward needs (mlp.py:252-256: hs, sigma, feat, g, color)
// are written out on request.
//
// backward (mlp.py:269-316), two phases:
//  1. row-parallel: per 32 rows, dz of every layer (sigmoid', ReLU masks from
//     the cached activations, dh = dz . W as transposed products), stored to
//     a workspace (rows x out per layer);
//  2. per layer, gw = dz^T . input and gb = sum_rows dz, summed over the rows
//     in a fixed order (deterministic), input being the cached activation
//     or the concatenation the forward pass used ([x_enc, h] at the skip
//     layer, [feat, d_enc] at the direction layer).
#include <cuda_runtime.h>

#include <cstdio>

#include "gf_mlp.cuh"

namespace gf {

namespace {

constexpr int DSUB = 32;     // rows per CTA
constexpr int DKC = 16;      // reduction chunk staged in shared memory
constexpr int DTHREADS = 256;

struct DenseNet {  // one manifest, stacked weights (n_net, out, in)
  int n_layers, trunk, width, view, pos_dim, dir_dim, skip;
  int in[GF_MAX_LAYERS], out[GF_MAX_LAYERS];
  const void* w[GF_MAX_LAYERS];
  const void* b[GF_MAX_LAYERS];
};

template <typename T>
__device__ __forceinline__ T fma_(T a, T b, T c);
template <>
__device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
template <>
__device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ float sigmoid_split_t(float z) {  // mlp.py:228-235
  if (z >= 0.f) return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
  const float e = expf(z);
  return __fdiv_rn(e, __fadd_rn(1.0f, e));
}
__device__ __forceinline__ double sigmoid_split_t(double z) {
  if (z >= 0.0) return __ddiv_rn(1.0, __dadd_rn(1.0, exp(-z)));
  const double e = exp(z);
  return __ddiv_rn(e, __dadd_rn(1.0, e));
}

// out[o][row] = b[o] + sum_k in[k][row] W[o][k] (sequential FMA over k from 0)
// for this CTA's 32 rows; the input is the concatenation of up to two
// transposed segments.  W row-major (out, in).
template <typename T, int OPT>
__device__ void dense_fw(const T* __restrict__ W, const T* __restrict__ bias, int in_dim, int out_dim, const T* s1,
                         int n1, const T* s2, T* ws, T* dst, bool relu) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  T acc[4][OPT];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < OPT; ++j) acc[r][j] = T(0);
  for (int k0 = 0; k0 < in_dim; k0 += DKC) {
    __syncthreads();
    const int kc = min(DKC, in_dim - k0);
    for (int idx = tid; idx < out_dim * DKC; idx += DTHREADS) {
      const int o = idx / DKC, kk = idx % DKC;
      ws[kk * out_dim + o] = kk < kc ? W[(size_t)o * in_dim + k0 + kk] : T(0);
    }
    __syncthreads();
    for (int kk = 0; kk < kc; ++kk) {
      const int k = k0 + kk;
      const T* src = (k < n1 ? s1 + k * DSUB : s2 + (k - n1) * DSUB) + 4 * warp;
      const T a0 = src[0], a1 = src[1], a2 = src[2], a3 = src[3];
      const T* wk = ws + kk * out_dim;
#pragma unroll
      for (int j = 0; j < OPT; ++j) {
        const int o = lane + 32 * j;
        if (o < out_dim) {
          const T w = wk[o];
          acc[0][j] = fma_(a0, w, acc[0][j]);
          acc[1][j] = fma_(a1, w, acc[1][j]);
          acc[2][j] = fma_(a2, w, acc[2][j]);
          acc[3][j] = fma_(a3, w, acc[3][j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < OPT; ++j) {
    const int o = lane + 32 * j;
    if (o < out_dim) {
      const T b = bias[o];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        T z = add_rn(acc[r][j], b);
        if (relu) z = z > T(0) ? z : T(0);
        dst[o * DSUB + 4 * warp + r] = z;
      }
    }
  }
}

// out[i][row] = sum_o dz[o][row] W[o][col0 + i] for i < n_cols (the
// transposed product dz . W of mlp.py:261), sequential over o
template <typename T, int OPT>
__device__ void dense_bw(const T* __restrict__ W, int w_in, int col0, int n_out, int n_cols, const T* dz, T* ws,
                         T* dst) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  T acc[4][OPT];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < OPT; ++j) acc[r][j] = T(0);
  for (int o0 = 0; o0 < n_out; o0 += DKC) {
    __syncthreads();
    const int oc = min(DKC, n_out - o0);
    for (int idx = tid; idx < n_cols * DKC; idx += DTHREADS) {
      const int oo = idx / n_cols, i = idx % n_cols;
      ws[oo * n_cols + i] = oo < oc ? W[(size_t)(o0 + oo) * w_in + col0 + i] : T(0);
    }
    __syncthreads();
    for (int oo = 0; oo < oc; ++oo) {
      const T* src = dz + (o0 + oo) * DSUB + 4 * warp;
      const T a0 = src[0], a1 = src[1], a2 = src[2], a3 = src[3];
      const T* wk = ws + oo * n_cols;
#pragma unroll
      for (int j = 0; j < OPT; ++j) {
        const int i = lane + 32 * j;
        if (i < n_cols) {
          const T w = wk[i];
          acc[0][j] = fma_(a0, w, acc[0][j]);
          acc[1][j] = fma_(a1, w, acc[1][j]);
          acc[2][j] = fma_(a2, w, acc[2][j]);
          acc[3][j] = fma_(a3, w, acc[3][j]);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < OPT; ++j) {
    const int i = lane + 32 * j;
    if (i < n_cols)
#pragma unroll
      for (int r = 0; r < 4; ++r) dst[i * DSUB + 4 * warp + r] = acc[r][j];
  }
}

struct FwOut {
  void* color;
  void* sigma;
  void* hs[GF_MAX_LAYERS];  // per trunk layer (n_net, rows, width), optional
  void* feat;                // (n_net, rows, width), optional
  void* g;                   // (n_net, rows, view), optional
};

template <typename T>
__device__ __forceinline__ const T* wl(const DenseNet& N, int l, int64_t c) {
  return reinterpret_cast<const T*>(N.w[l]) + (size_t)c * N.out[l] * N.in[l];
}
template <typename T>
__device__ __forceinline__ const T* bl(const DenseNet& N, int l, int64_t c) {
  return reinterpret_cast<const T*>(N.b[l]) + (size_t)c * N.out[l];
}

// transposed [feature][row] buffer <-> row-major (rows, n) global array
template <typename T>
__device__ void load_T(const T* src, int64_t row0, int64_t rows, int n, T* dst) {
  for (int idx = threadIdx.x; idx < n * DSUB; idx += DTHREADS) {
    const int f = idx / DSUB, r = idx % DSUB;
    dst[f * DSUB + r] = row0 + r < rows ? src[(row0 + r) * n + f] : T(0);
  }
}
template <typename T>
__device__ void store_T(const T* src, int64_t row0, int64_t rows, int n, T* dst) {
  for (int idx = threadIdx.x; idx < n * DSUB; idx += DTHREADS) {
    const int f = idx % n, r = idx / n;
    if (row0 + r < rows) dst[(row0 + r) * n + f] = src[f * DSUB + r];
  }
}

struct DSmem {  // element offsets into dynamic shared memory (computed on the host)
  int xe, de, ha, hb, ws, small, total;
};
inline DSmem dsmem(int pos_dim, int dir_dim, int wmax, int cmax) {
  DSmem s;
  s.xe = 0;
  s.de = s.xe + pos_dim * DSUB;
  s.ha = s.de + dir_dim * DSUB;
  s.hb = s.ha + wmax * DSUB;
  s.ws = s.hb + wmax * DSUB;
  s.small = s.ws + DKC * cmax;
  s.total = s.small + 4 * DSUB;
  return s;
}

template <typename T, int OPT>
__global__ void __launch_bounds__(DTHREADS) k_dense_forward(DenseNet N, int64_t rows, const T* __restrict__ x_enc,
                                                            const T* __restrict__ d_enc, FwOut out, DSmem M) {
  extern __shared__ double dsm_d[];
  T* sm = reinterpret_cast<T*>(dsm_d);
  T *xe = sm + M.xe, *de = sm + M.de, *ha = sm + M.ha, *hb = sm + M.hb, *ws = sm + M.ws, *sm4 = sm + M.small;
  const int64_t c = blockIdx.y, row0 = (int64_t)blockIdx.x * DSUB, base = c * rows;
  const int T_ = N.trunk;
  load_T(x_enc + base * N.pos_dim, row0, rows, N.pos_dim, xe);
  load_T(d_enc + base * N.dir_dim, row0, rows, N.dir_dim, de);
  auto save = [&](void* dst, const T* src, int n) {
    if (dst) {
      __syncthreads();
      store_T(src, row0, rows, n, reinterpret_cast<T*>(dst) + base * n);
    }
  };
  dense_fw<T, OPT>(wl<T>(N, 0, c), bl<T>(N, 0, c), N.in[0], N.out[0], xe, N.in[0], nullptr, ws, ha, true);
  save(out.hs[0], ha, N.width);
  T *h = ha, *o = hb;
  for (int k = 1; k < T_; ++k) {
    if (k == N.skip)
      dense_fw<T, OPT>(wl<T>(N, k, c), bl<T>(N, k, c), N.in[k], N.out[k], xe, N.pos_dim, h, ws, o, true);
    else
      dense_fw<T, OPT>(wl<T>(N, k, c), bl<T>(N, k, c), N.in[k], N.out[k], h, N.in[k], nullptr, ws, o, true);
    T* s = h; h = o; o = s;
    save(out.hs[k], h, N.width);
  }
  T* sig = sm4;           // density (1 x 32)
  T* col = sm4 + DSUB;    // color (3 x 32)
  dense_fw<T, OPT>(wl<T>(N, T_, c), bl<T>(N, T_, c), N.in[T_], 1, h, N.in[T_], nullptr, ws, sig, true);
  dense_fw<T, OPT>(wl<T>(N, T_ + 1, c), bl<T>(N, T_ + 1, c), N.in[T_ + 1], N.out[T_ + 1], h, N.in[T_ + 1], nullptr,
                   ws, o, false);
  save(out.feat, o, N.width);
  dense_fw<T, OPT>(wl<T>(N, T_ + 2, c), bl<T>(N, T_ + 2, c), N.in[T_ + 2], N.out[T_ + 2], o, N.width, de, ws, h,
                   true);
  save(out.g, h, N.view);
  dense_fw<T, OPT>(wl<T>(N, T_ + 3, c), bl<T>(N, T_ + 3, c), N.in[T_ + 3], 3, h, N.in[T_ + 3], nullptr, ws, col,
                   false);
  __syncthreads();
  if (threadIdx.x < DSUB && row0 + threadIdx.x < rows) {
    const int64_t r = base + row0 + threadIdx.x;
    T* cl = reinterpret_cast<T*>(out.color) + r * 3;
#pragma unroll
    for (int q = 0; q < 3; ++q) cl[q] = sigmoid_split_t(col[q * DSUB + threadIdx.x]);
    reinterpret_cast<T*>(out.sigma)[r] = sig[threadIdx.x];
  }
}

struct BwIn {
  const void* hs[GF_MAX_LAYERS];
  const void *feat, *g, *color, *sigma, *d_color, *d_sigma;
  void* dz[GF_MAX_LAYERS];  // workspace: (n_net, rows, out_l) per manifest layer
};

// phase 1: dz of every layer for this CTA's 32 rows (mlp.py:277-296)
template <typename T, int OPT>
__global__ void __launch_bounds__(DTHREADS) k_dense_backward_dz(DenseNet N, int64_t rows, BwIn B, DSmem M) {
  extern __shared__ double dsm_d[];
  T* sm = reinterpret_cast<T*>(dsm_d);
  T *za = sm + M.ha, *zb = sm + M.hb, *ws = sm + M.ws;
  T* s4 = sm + M.small;
  const int64_t c = blockIdx.y, row0 = (int64_t)blockIdx.x * DSUB, base = c * rows;
  const int T_ = N.trunk, L_den = T_, L_feat = T_ + 1, L_dir = T_ + 2, L_col = T_ + 3;
  auto dz_out = [&](int l, const T* src, int n) {
    __syncthreads();
    store_T(src, row0, rows, n, reinterpret_cast<T*>(B.dz[l]) + base * n);
  };
  // dz_color = d_color * color * (1 - color)
  for (int idx = threadIdx.x; idx < 3 * DSUB; idx += DTHREADS) {
    const int q = idx / DSUB, r = idx % DSUB;
    T v = T(0);
    if (row0 + r < rows) {
      const int64_t i = (base + row0 + r) * 3 + q;
      const T col = reinterpret_cast<const T*>(B.color)[i];
      v = mul_rn(mul_rn(reinterpret_cast<const T*>(B.d_color)[i], col), sub_rn(T(1), col));
    }
    s4[q * DSUB + r] = v;
  }
  dz_out(L_col, s4, 3);
  // dg = dz_color . W_col ; dz_dir = dg * (g > 0)
  dense_bw<T, OPT>(wl<T>(N, L_col, c), N.in[L_col], 0, 3, N.view, s4, ws, za);
  __syncthreads();
  {
    const T* gg = reinterpret_cast<const T*>(B.g) + base * N.view;
    for (int idx = threadIdx.x; idx < N.view * DSUB; idx += DTHREADS) {
      const int i = idx / DSUB, r = idx % DSUB;
      if (row0 + r >= rows || !(gg[(row0 + r) * N.view + i] > T(0))) za[idx] = T(0);
    }
  }
  dz_out(L_dir, za, N.view);
  // dfeat = (dz_dir . W_dir)[:, :width] (feature is unactivated: its dz)
  dense_bw<T, OPT>(wl<T>(N, L_dir, c), N.in[L_dir], 0, N.view, N.width, za, ws, zb);
  dz_out(L_feat, zb, N.width);
  // dh = dfeat . W_feat + dz_density . W_density, dz_density = d_sigma * (sigma > 0)
  dense_bw<T, OPT>(wl<T>(N, L_feat, c), N.in[L_feat], 0, N.width, N.width, zb, ws, za);
  __syncthreads();
  if (threadIdx.x < DSUB) {
    const int r = threadIdx.x;
    T v = T(0);
    if (row0 + r < rows) {
      const int64_t i = base + row0 + r;
      v = reinterpret_cast<const T*>(B.sigma)[i] > T(0) ? reinterpret_cast<const T*>(B.d_sigma)[i] : T(0);
    }
    s4[r] = v;
  }
  dz_out(L_den, s4, 1);
  __syncthreads();
  {
    const T* wden = wl<T>(N, L_den, c);
    for (int idx = threadIdx.x; idx < N.width * DSUB; idx += DTHREADS) {
      const int i = idx / DSUB, r = idx % DSUB;
      za[idx] = add_rn(za[idx], mul_rn(s4[r], wden[i]));
    }
  }
  // trunk k = T-1 .. 1: dz = dh * (hs[k] > 0); dh = dz . W_k (skip: the h part)
  T *dh = za, *o = zb;
  for (int k = T_ - 1; k >= 0; --k) {
    __syncthreads();
    {  // ReLU mask straight from the cached activation (global, row-major)
      const T* hk = reinterpret_cast<const T*>(B.hs[k]) + base * N.width;
      for (int idx = threadIdx.x; idx < N.width * DSUB; idx += DTHREADS) {
        const int i = idx / DSUB, r = idx % DSUB;
        if (row0 + r >= rows || !(hk[(row0 + r) * N.width + i] > T(0))) dh[idx] = T(0);
      }
    }
    dz_out(k, dh, N.width);
    if (k == 0) break;
    const int col0 = k == N.skip ? N.pos_dim : 0;
    dense_bw<T, OPT>(wl<T>(N, k, c), N.in[k], col0, N.width, N.width, dh, ws, o);
    T* s = dh; dh = o; o = s;
  }
}

// phase 2: gw[c][o][i] = sum_r dz[r][o] X[r][i] (fixed r order), X = [X1 | X2]
template <typename T>
__global__ void __launch_bounds__(256) k_wgrad(const T* __restrict__ dz, int n_out, const T* __restrict__ x1, int n1,
                                               const T* __restrict__ x2, int n2, int64_t rows, T* __restrict__ gw,
                                               T* __restrict__ gb) {
  __shared__ T sz[32][33];
  __shared__ T sx[32][33];
  const int n_in = n1 + n2;
  const int64_t c = blockIdx.z;
  const int o0 = blockIdx.y * 32, i0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 2 x 2 outputs each
  T acc[2][2] = {{T(0), T(0)}, {T(0), T(0)}};
  T accb[2] = {T(0), T(0)};
  const T* dzc = dz + c * rows * n_out;
  const T* x1c = x1 + c * rows * n1;
  const T* x2c = x2 ? x2 + c * rows * n2 : nullptr;
  for (int64_t r0 = 0; r0 < rows; r0 += 32) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < 32 * 32; idx += 256) {
      const int rr = idx / 32, q = idx % 32;
      const int64_t r = r0 + rr;
      sz[rr][q] = (r < rows && o0 + q < n_out) ? dzc[r * n_out + o0 + q] : T(0);
      const int i = i0 + q;
      T xv = T(0);
      if (r < rows && i < n_in) xv = i < n1 ? x1c[r * n1 + i] : x2c[r * n2 + (i - n1)];
      sx[rr][q] = xv;
    }
    __syncthreads();
    const int nr = rows - r0 < 32 ? (int)(rows - r0) : 32;
    for (int rr = 0; rr < nr; ++rr) {
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const T z = sz[rr][ty + 16 * a];
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b] = fma_(z, sx[rr][tx + 16 * b], acc[a][b]);
        if (blockIdx.x == 0 && tx == 0) accb[a] = add_rn(accb[a], z);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int o = o0 + ty + 16 * a;
    if (o >= n_out) continue;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int i = i0 + tx + 16 * b;
      if (i < n_in) gw[((size_t)c * n_out + o) * n_in + i] = acc[a][b];
    }
    if (blockIdx.x == 0 && tx == 0) gb[(size_t)c * n_out + o] = accb[a];
  }
}

bool make_net(const gf_manifest_t* m, DenseNet* N) {
  if (!m || m->hidden_layers < 3 || m->width < 1 || m->pos_dim < 1 || m->dir_dim < 0) return false;
  const int T_ = m->hidden_layers - 2;
  if (T_ + 4 > GF_MAX_LAYERS) return false;
  if (m->skip_layer > 0 && m->skip_layer >= T_) return false;
  N->trunk = T_;
  N->width = m->width;
  N->view = m->view_width > 0 ? m->view_width : m->width;
  N->pos_dim = m->pos_dim;
  N->dir_dim = m->dir_dim;
  N->skip = m->skip_layer > 0 ? m->skip_layer : -1;
  int l = 0;
  N->in[l] = N->pos_dim; N->out[l++] = N->width;
  for (int k = 1; k < T_; ++k) {
    N->in[l] = k == N->skip ? N->width + N->pos_dim : N->width;
    N->out[l++] = N->width;
  }
  N->in[l] = N->width; N->out[l++] = 1;
  N->in[l] = N->width; N->out[l++] = N->width;
  N->in[l] = N->width + N->dir_dim; N->out[l++] = N->view;
  N->in[l] = N->view; N->out[l++] = 3;
  N->n_layers = l;
  return true;
}

template <typename T>
DSmem dense_layout(const DenseNet& N) {
  const int wmax = N.width > N.view ? N.width : N.view;
  return dsmem(N.pos_dim, N.dir_dim, wmax, wmax > 4 ? wmax : 4);
}

int opt_of(const DenseNet& N) {
  const int w = N.width > N.view ? N.width : N.view;
  return w <= 64 ? 2 : (w <= 256 ? 8 : (w <= 512 ? 16 : 0));
}

template <typename T, int OPT>
bool forward_t(const DenseNet& N, int64_t n_net, int64_t rows, const void* x, const void* d, const FwOut& out,
               cudaStream_t st) {
  const DSmem M = dense_layout<T>(N);
  const size_t smem = (size_t)M.total * sizeof(T);
  if (smem > 227 * 1024) return false;
  auto k = k_dense_forward<T, OPT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (rows > 0 && n_net > 0)
    k<<<dim3((unsigned)((rows + DSUB - 1) / DSUB), (unsigned)n_net), DTHREADS, smem, st>>>(N, rows, (const T*)x,
                                                                                        (const T*)d, out, M);
  return true;
}

template <typename T, int OPT>
bool backward_t(const DenseNet& N, int64_t n_net, int64_t rows, const void* x, const void* d, const BwIn& B,
                void* const* gw, void* const* gb, cudaStream_t st) {
  const DSmem M = dense_layout<T>(N);
  const size_t smem = (size_t)M.total * sizeof(T);
  if (smem > 227 * 1024) return false;
  auto k = k_dense_backward_dz<T, OPT>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (rows > 0 && n_net > 0)
    k<<<dim3((unsigned)((rows + DSUB - 1) / DSUB), (unsigned)n_net), DTHREADS, smem, st>>>(N, rows, B, M);
  // phase 2, layer by layer: the input each layer saw in the forward pass
  const int T_ = N.trunk;
  for (int l = 0; l < N.n_layers; ++l) {
    const T *x1 = nullptr, *x2 = nullptr;
    int n1 = 0, n2 = 0;
    if (l == 0) { x1 = (const T*)x; n1 = N.pos_dim; }
    else if (l < T_) {
      if (l == N.skip) { x1 = (const T*)x; n1 = N.pos_dim; x2 = (const T*)B.hs[l - 1]; n2 = N.width; }
      else { x1 = (const T*)B.hs[l - 1]; n1 = N.width; }
    } else if (l == T_ || l == T_ + 1) { x1 = (const T*)B.hs[T_ - 1]; n1 = N.width; }
    else if (l == T_ + 2) { x1 = (const T*)B.feat; n1 = N.width; x2 = (const T*)d; n2 = N.dir_dim; }
    else { x1 = (const T*)B.g; n1 = N.view; }
    const dim3 grid((unsigned)((N.in[l] + 31) / 32), (unsigned)((N.out[l] + 31) / 32), (unsigned)n_net);
    if (n_net > 0)
      k_wgrad<T><<<grid, 256, 0, st>>>((const T*)B.dz[l], N.out[l], x1, n1, x2, n2, rows, (T*)gw[l], (T*)gb[l]);
  }
  return true;
}

}  // namespace

bool dense_mlp_supported(const gf_manifest_t* m) {
  DenseNet N;
  return make_net(m, &N) && opt_of(N) > 0 && N.pos_dim <= 1024 && N.dir_dim <= 1024;
}

size_t dense_backward_workspace(const gf_manifest_t* m, int f64, int64_t n_net, int64_t rows) {
  DenseNet N;
  if (!make_net(m, &N)) return 0;
  size_t bytes = 0;
  for (int l = 0; l < N.n_layers; ++l) bytes += gf_align((size_t)n_net * rows * N.out[l] * (f64 ? 8 : 4));
  return bytes;
}

bool launch_dense_forward(const gf_manifest_t* m, int f64, int64_t n_net, int64_t rows, const void* const* w,
                          const void* const* b, const void* x, const void* d, void* color, void* sigma,
                          void* const* hs, void* feat, void* g, cudaStream_t st) {
  DenseNet N;
  if (!make_net(m, &N)) return false;
  for (int l = 0; l < N.n_layers; ++l) { N.w[l] = w[l]; N.b[l] = b[l]; }
  FwOut out;
  out.color = color;
  out.sigma = sigma;
  for (int k = 0; k < GF_MAX_LAYERS; ++k) out.hs[k] = (hs && k < N.trunk) ? hs[k] : nullptr;
  out.feat = feat;
  out.g = g;
  const int opt = opt_of(N);
  if (f64) {
    if (opt == 2) return forward_t<double, 2>(N, n_net, rows, x, d, out, st);
    if (opt == 8) return forward_t<double, 8>(N, n_net, rows, x, d, out, st);
    if (opt == 16) return forward_t<double, 16>(N, n_net, rows, x, d, out, st);
  } else {
    if (opt == 2) return forward_t<float, 2>(N, n_net, rows, x, d, out, st);
    if (opt == 8) return forward_t<float, 8>(N, n_net, rows, x, d, out, st);
    if (opt == 16) return forward_t<float, 16>(N, n_net, rows, x, d, out, st);
  }
  return false;
}

bool launch_dense_backward(const gf_manifest_t* m, int f64, int64_t n_net, int64_t rows, const void* const* w,
                           const void* x, const void* d, const void* const* hs, const void* feat, const void* g,
                           const void* color, const void* sigma, const void* d_color, const void* d_sigma,
                           void* const* gw, void* const* gb, void* ws, cudaStream_t st) {
  DenseNet N;
  if (!make_net(m, &N)) return false;
  for (int l = 0; l < N.n_layers; ++l) { N.w[l] = w[l]; N.b[l] = nullptr; }
  BwIn B;
  for (int k = 0; k < GF_MAX_LAYERS; ++k) B.hs[k] = k < N.trunk ? hs[k] : nullptr;
  B.feat = feat;
  B.g = g;
  B.color = color;
  B.sigma = sigma;
  B.d_color = d_color;
  B.d_sigma = d_sigma;
  uint8_t* p = (uint8_t*)ws;
  for (int l = 0; l < GF_MAX_LAYERS; ++l) {
    B.dz[l] = nullptr;
    if (l < N.n_layers) {
      B.dz[l] = p;
      p += gf_align((size_t)n_net * rows * N.out[l] * (f64 ? 8 : 4));
    }
  }
  const int opt = opt_of(N);
  if (f64) {
    if (opt == 2) return backward_t<double, 2>(N, n_net, rows, x, d, B, gw, gb, st);
    if (opt == 8) return backward_t<double, 8>(N, n_net, rows, x, d, B, gw, gb, st);
    if (opt == 16) return backward_t<double, 16>(N, n_net, rows, x, d, B, gw, gb, st);
  } else {
    if (opt == 2) return backward_t<float, 2>(N, n_net, rows, x, d, B, gw, gb, st);
    if (opt == 8) return backward_t<float, 8>(N, n_net, rows, x, d, B, gw, gb, st);
    if (opt == 16) return backward_t<float, 16>(N, n_net, rows, x, d, B, gw, gb, st);
  }
  return false;
}


}  // namespace gf
