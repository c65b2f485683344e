// fp32 SIMT evaluation of per-cell MLPs of ANY manifest (mlp.py:30-87): any
// depth and hidden width, a separate direction-layer width, the skip layer
// that re-concatenates gamma(x) onto a trunk layer's input (mlp.py:79-81,
// 241-243), any number of encoding octaves.  This is the path of the
// teacher network (train.py:93-101, mlp.py:90-109: 10 x 256, skip 5, view
// 128) and of any NetworkGrid whose architecture the fused tiny-MLP kernels
// (gf_mlp_simt.cuh, gf_mlp_tc.cu) do not cover.
//
// One CTA (256 threads) walks the 128-row tiles of its range, 32 rows at a
// time.  Activations stay in shared memory, transposed ([feature][row], so a
// warp reads its 4 rows of one feature with one broadcast 16-byte load);
// each layer streams its weights from global memory (L2) in chunks of KC
// inputs into shared memory as [k][out]; warp w owns rows 4w..4w+3 and lane
// l accumulates outputs l, l+32, ... in registers (fp32 FMA, bias added after
// the dot product as matmul(x, W^T) + b does, mlp.py:222-225).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "gf_mlp.cuh"

namespace gf {

namespace {

constexpr int GSUB = 32;   // rows per pass
constexpr int GKC = 16;    // inputs per staged weight chunk
constexpr int GTHREADS = 256;

struct GenericArgs {
  LayerTable t;
  Fp32Layout L;
  int pos_freqs, dir_freqs, raw;
  int pp, dp, wmax, omax;  // padded feature counts / buffer widths (floats)
};

struct GSmem {  // float offsets into dynamic shared memory
  int xe, de, ha, hb, ws, sig, col, total;
};

__host__ __device__ inline GSmem gsmem_layout(const GenericArgs& A) {
  GSmem s;
  s.xe = 0;
  s.de = s.xe + A.pp * GSUB;
  s.ha = s.de + A.dp * GSUB;
  s.hb = s.ha + A.wmax * GSUB;
  s.ws = s.hb + A.wmax * GSUB;
  s.sig = s.ws + GKC * A.omax;
  s.col = s.sig + GSUB;
  s.total = s.col + 4 * GSUB;
  return s;
}

// gamma(v) in the core.py:132-152 layout ([v,] then per octave k: sin xyz,
// cos xyz; angle = fl32(v * fl32(2^k pi)), accurate sincosf), written to a
// transposed [feature][row] buffer
__device__ inline void encode_T(const float* v, int freqs, int raw, float* dst, int row) {
  int c = 0;
  if (raw) {
    for (int a = 0; a < 3; ++a) dst[(c + a) * GSUB + row] = v[a];
    c = 3;
  }
  for (int k = 0; k < freqs; ++k) {
    const float f = __int_as_float(0x40490FDB + (k << 23));  // fl32(pi) * 2^k == fl32(2^k pi)
    for (int a = 0; a < 3; ++a) {
      float s, co;
      sincosf(__fmul_rn(v[a], f), &s, &co);
      dst[(c + a) * GSUB + row] = s;
      dst[(c + 3 + a) * GSUB + row] = co;
    }
    c += 6;
  }
}

// out[row][o] = b[o] + sum_k in[row][k] W[o][k] for this CTA's 32 rows, the
// input being the concatenation of up to two transposed segments; the result
// (ReLU optional) goes to dst ([o][row]).  W is the cell's fp32 packed layer:
// row-major [out][in_pad], then the bias.
template <int OPT>
__device__ void dense_T(const float* __restrict__ W, const float* __restrict__ bias, int in_dim, int in_pad,
                        int out_dim, const float* s1, int n1, const float* s2, float* ws, float* dst, bool relu) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float acc[4][OPT];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int j = 0; j < OPT; ++j) acc[r][j] = 0.f;
  for (int k0 = 0; k0 < in_dim; k0 += GKC) {
    __syncthreads();  // previous chunk consumed (and the previous layer's output written)
    const int kc = min(GKC, in_dim - k0);
    for (int idx = tid; idx < out_dim * GKC; idx += GTHREADS) {
      const int o = idx / GKC, kk = idx % GKC;
      ws[kk * out_dim + o] = kk < kc ? __ldg(W + (size_t)o * in_pad + k0 + kk) : 0.f;
    }
    __syncthreads();
    for (int kk = 0; kk < kc; ++kk) {
      const int k = k0 + kk;
      const float* src = k < n1 ? s1 + k * GSUB : s2 + (k - n1) * GSUB;
      const float4 a = *reinterpret_cast<const float4*>(src + 4 * warp);
      const float* wk = ws + kk * out_dim;
#pragma unroll
      for (int j = 0; j < OPT; ++j) {
        const int o = lane + 32 * j;
        if (o < out_dim) {
          const float w = wk[o];
          acc[0][j] = fmaf(a.x, w, acc[0][j]);
          acc[1][j] = fmaf(a.y, w, acc[1][j]);
          acc[2][j] = fmaf(a.z, w, acc[2][j]);
          acc[3][j] = fmaf(a.w, w, acc[3][j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < OPT; ++j) {
    const int o = lane + 32 * j;
    if (o < out_dim) {
      const float b = __ldg(bias + o);
      float4 z;
      z.x = __fadd_rn(acc[0][j], b);
      z.y = __fadd_rn(acc[1][j], b);
      z.z = __fadd_rn(acc[2][j], b);
      z.w = __fadd_rn(acc[3][j], b);
      if (relu) {
        z.x = fmaxf(z.x, 0.f); z.y = fmaxf(z.y, 0.f); z.z = fmaxf(z.z, 0.f); z.w = fmaxf(z.w, 0.f);
      }
      *reinterpret_cast<float4*>(dst + o * GSUB + 4 * warp) = z;
    }
  }
}

__device__ __forceinline__ float sigmoid_split_g(float z) {  // mlp.py:228-235
  if (z >= 0.f) return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
  const float e = expf(z);
  return __fdiv_rn(e, __fadd_rn(1.0f, e));
}

template <int OPT, class IO>
__global__ void __launch_bounds__(GTHREADS) k_mlp_generic(const float* __restrict__ packed, GenericArgs A, TileSched S,
                                                          IO io) {
  extern __shared__ float4 gsm4[];
  float* sm = reinterpret_cast<float*>(gsm4);
  const GSmem M = gsmem_layout(A);
  float *xe = sm + M.xe, *de = sm + M.de, *ha = sm + M.ha, *hb = sm + M.hb, *ws = sm + M.ws, *sig = sm + M.sig,
        *col = sm + M.col;
  const LayerTable& t = A.t;
  const int T = t.trunk;
  const uint32_t nt = *S.n_tiles;
  const uint32_t per = (nt + gridDim.x - 1) / gridDim.x;
  const uint32_t t_begin = min(nt, blockIdx.x * per), t_end = min(nt, t_begin + per);
  for (uint32_t tt = t_begin; tt < t_end; ++tt) {
    const uint2 tl = S.tiles[tt];
    const uint32_t cell = gf_tile_cell(tl), rows = gf_tile_rows(tl);
    const float* cw = packed + (size_t)cell * A.L.cell_floats;
    auto Wl = [&](int l) { return cw + A.L.w_off[l]; };
    auto Bl = [&](int l) { return cw + A.L.b_off[l]; };
    for (uint32_t sub = 0; sub < rows; sub += GSUB) {
      __syncthreads();  // the previous pass's outputs were read
      uint32_t idx = 0;
      bool valid = false;
      if (threadIdx.x < GSUB) {
        const uint32_t r = sub + threadIdx.x;
        float x[3] = {0.f, 0.f, 0.f}, d[3] = {0.f, 0.f, 0.f};
        valid = r < rows;
        if (valid) io.template fetch<true>(S, tl.y + r, idx, x, d);
        encode_T(x, A.pos_freqs, A.raw, xe, threadIdx.x);
        encode_T(d, A.dir_freqs, A.raw, de, threadIdx.x);
      }
      // trunk (mlp.py:239-244): trunk0 on gamma(x); trunk k on [gamma(x), h] at the skip layer
      dense_T<OPT>(Wl(0), Bl(0), t.in[0], A.L.in_pad[0], t.out[0], xe, t.in[0], nullptr, ws, ha, true);
      float *h = ha, *o = hb;
      for (int k = 1; k < T; ++k) {
        if (k == t.skip)
          dense_T<OPT>(Wl(k), Bl(k), t.in[k], A.L.in_pad[k], t.out[k], xe, t.pos_dim, h, ws, o, true);
        else
          dense_T<OPT>(Wl(k), Bl(k), t.in[k], A.L.in_pad[k], t.out[k], h, t.in[k], nullptr, ws, o, true);
        float* s = h; h = o; o = s;
      }
      // density (ReLU), feature (unactivated), direction on [feat, gamma(d)], color
      dense_T<OPT>(Wl(T), Bl(T), t.in[T], A.L.in_pad[T], 1, h, t.in[T], nullptr, ws, sig, true);
      dense_T<OPT>(Wl(T + 1), Bl(T + 1), t.in[T + 1], A.L.in_pad[T + 1], t.out[T + 1], h, t.in[T + 1], nullptr, ws, o,
                   false);
      dense_T<OPT>(Wl(T + 2), Bl(T + 2), t.in[T + 2], A.L.in_pad[T + 2], t.out[T + 2], o, t.width, de, ws, h, true);
      dense_T<OPT>(Wl(T + 3), Bl(T + 3), t.in[T + 3], A.L.in_pad[T + 3], 3, h, t.in[T + 3], nullptr, ws, col, false);
      __syncthreads();
      if (threadIdx.x < GSUB && valid) {
        const int r = threadIdx.x;
        io.store(idx, tl.y + sub + r, sigmoid_split_g(col[0 * GSUB + r]), sigmoid_split_g(col[1 * GSUB + r]),
                 sigmoid_split_g(col[2 * GSUB + r]), sig[r]);
      }
    }
  }
}

GenericArgs make_args(const LayerTable& t, const gf_arch_t* arch) {
  GenericArgs A;
  A.t = t;
  A.L = make_fp32_layout(t);
  A.pos_freqs = arch->pos_freqs;
  A.dir_freqs = arch->dir_freqs;
  A.raw = arch->include_raw ? 1 : 0;
  A.pp = gf_pad4(t.pos_dim);
  A.dp = gf_pad4(t.dir_dim);
  A.wmax = gf_pad4(t.width > t.view ? t.width : t.view);
  A.omax = A.wmax > 4 ? A.wmax : 4;
  return A;
}

template <int OPT, class IO>
bool launch_generic_opt(const GenericArgs& A, const float* packed, const TileSched& S, const IO& io, cudaStream_t st,
                        bool launch) {
  const size_t smem = (size_t)gsmem_layout(A).total * sizeof(float);
  if (smem > 227 * 1024) return false;
  auto k = k_mlp_generic<OPT, IO>;
  static thread_local size_t smem_set = 0;  // attribute set once per size (outside graph capture via prepare)
  if (smem_set < smem) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set = smem;
  }
  if (launch) {
    const int per_sm = smem <= 100 * 1024 ? 2 : 1;
    k<<<num_sms() * per_sm, GTHREADS, smem, st>>>(packed, A, S, io);
  }
  return true;
}

template <class IO>
bool launch_generic(const LayerTable& t, const gf_arch_t* arch, const float* packed, const TileSched& S, const IO& io,
                    cudaStream_t st, bool launch) {
  const GenericArgs A = make_args(t, arch);
  const int w = A.wmax;
  if (w <= 64) return launch_generic_opt<2>(A, packed, S, io, st, launch);
  if (w <= 256) return launch_generic_opt<8>(A, packed, S, io, st, launch);
  if (w <= 512) return launch_generic_opt<16>(A, packed, S, io, st, launch);
  return false;
}

}  // namespace

bool generic_mlp_supported(const LayerTable& t) {
  const int w = t.width > t.view ? t.width : t.view;
  return t.n_layers <= GF_MAX_LAYERS && w <= 512 && t.pos_dim <= 3 * 21 * 2 && t.dir_dim <= 3 * 21 * 2;
}

bool launch_mlp_generic_render(const LayerTable& t, const gf_arch_t* arch, const float* packed, const TileSched& S,
                               const RenderIO& io, cudaStream_t st) {
  return generic_mlp_supported(t) && launch_generic(t, arch, packed, S, io, st, true);
}

bool launch_mlp_generic_query(const LayerTable& t, const gf_arch_t* arch, const float* packed, const TileSched& S,
                              const QueryIO& io, cudaStream_t st) {
  return generic_mlp_supported(t) && launch_generic(t, arch, packed, S, io, st, true);
}

bool prepare_mlp_generic(const LayerTable& t, const gf_arch_t* arch) {
  if (!generic_mlp_supported(t)) return false;
  TileSched S{};
  RenderIO rio{};
  QueryIO qio{};
  return launch_generic(t, arch, nullptr, S, rio, 0, false) && launch_generic(t, arch, nullptr, S, qio, 0, false);
}

}  // namespace gf
