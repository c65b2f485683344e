// fp32 SIMT evaluation of the per-cell tiny MLPs (reference-faithful mode).
//
// One CTA walks a contiguous range of 128-row tiles; each tile belongs to one
// cell, whose packed fp32 parameters sit in shared memory (reloaded only when
// the cell changes).  One thread evaluates one row: float32 positional
// encoding (core.py:132-152: angle = fl32(x * fl32(2^k pi)), accurate
// sincosf), then the six affine layers with fp32 FMA accumulation and the
// bias added after the dot product, as matmul(x, W^T) + b does (mlp.py:222-225),
// ReLU / unactivated feature / sign-split sigmoid (mlp.py:228-266).
#pragma once
#include "gf_mlp.cuh"

namespace gf {

template <int IN, int INP, int OUT, bool RELU>
__device__ __forceinline__ void dense_f32(const float* __restrict__ w, const float* __restrict__ b, const float* in,
                                          float* out) {
#pragma unroll
  for (int o = 0; o < OUT; ++o) {
    const float4* wr = reinterpret_cast<const float4*>(w + o * INP);
    float acc = 0.f;
#pragma unroll
    for (int i4 = 0; i4 < INP / 4; ++i4) {
      float4 q = wr[i4];
      if (4 * i4 + 0 < IN) acc = fmaf(in[4 * i4 + 0], q.x, acc);
      if (4 * i4 + 1 < IN) acc = fmaf(in[4 * i4 + 1], q.y, acc);
      if (4 * i4 + 2 < IN) acc = fmaf(in[4 * i4 + 2], q.z, acc);
      if (4 * i4 + 3 < IN) acc = fmaf(in[4 * i4 + 3], q.w, acc);
    }
    float z = __fadd_rn(acc, b[o]);
    out[o] = RELU ? fmaxf(z, 0.f) : z;
  }
}

__device__ __forceinline__ float sigmoid_split(float z) {
  if (z >= 0.f) return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
  float e = expf(z);
  return __fdiv_rn(e, __fadd_rn(1.0f, e));
}

template <int L>
__device__ __forceinline__ void encode_f32(const float* v, float* out) {
  out[0] = v[0]; out[1] = v[1]; out[2] = v[2];
#pragma unroll
  for (int k = 0; k < L; ++k) {
    const float f = __int_as_float(0x40490FDB + (k << 23));  // fl32(pi) * 2^k == fl32(2^k pi)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      float s, c;
      sincosf(__fmul_rn(v[a], f), &s, &c);
      out[3 + 6 * k + a] = s;
      out[3 + 6 * k + 3 + a] = c;
    }
  }
}

template <int W, int T, int LX, int LD, class IO>
__global__ void __launch_bounds__(128) k_mlp_fp32(const float* __restrict__ packed, Fp32Layout L, TileSched S, IO io) {
  constexpr int P = 3 * (1 + 2 * LX), D = 3 * (1 + 2 * LD);
  constexpr int PP = (P + 3) & ~3, WP = (W + 3) & ~3, DP = (W + D + 3) & ~3;
  extern __shared__ float4 smem4[];
  float* sw = reinterpret_cast<float*>(smem4);
  const uint32_t nt = *S.n_tiles;
  const uint32_t per = (nt + gridDim.x - 1) / gridDim.x;
  const uint32_t t_begin = blockIdx.x * per, t_end = min(nt, t_begin + per);
  int cur = -1;
  for (uint32_t t = t_begin; t < t_end; ++t) {
    const uint2 tl = S.tiles[t];
    const uint32_t cell = gf_tile_cell(tl);
    if ((int)cell != cur) {
      __syncthreads();
      const float4* src = reinterpret_cast<const float4*>(packed + (size_t)cell * L.cell_floats);
      for (int j = threadIdx.x; j < L.cell_floats / 4; j += blockDim.x) smem4[j] = __ldg(src + j);
      __syncthreads();
      cur = (int)cell;
    }
    if (threadIdx.x >= gf_tile_rows(tl)) continue;
    uint32_t idx;
    float x[3], d[3];
    io.template fetch<true>(S, tl.y + threadIdx.x, idx, x, d);
    float xe[P];
    encode_f32<LX>(x, xe);
    float h[W], h2[W];
    dense_f32<P, PP, W, true>(sw + L.w_off[0], sw + L.b_off[0], xe, h);
    float4* act = nullptr;
    if constexpr (IO::kHasAct && W == 32 && T == 2)
      if (io.act) act = reinterpret_cast<float4*>(io.act + (size_t)(tl.y + threadIdx.x) * GF_ACT_FLOATS);
    auto put = [&](int at, const float* v, int nv) {  // nv a multiple of 4
      for (int q = 0; q < nv; q += 4) act[at / 4 + q / 4] = make_float4(v[q], v[q + 1], v[q + 2], v[q + 3]);
    };
    if (act) put(0, h, W);
#pragma unroll
    for (int k = 1; k < T; ++k) {
      dense_f32<W, WP, W, true>(sw + L.w_off[k], sw + L.b_off[k], h, h2);
#pragma unroll
      for (int q = 0; q < W; ++q) h[q] = h2[q];
    }
    if (act) put(W, h, W);
    float sig[1];
    dense_f32<W, WP, 1, true>(sw + L.w_off[T], sw + L.b_off[T], h, sig);
    float cat[W + D];
    dense_f32<W, WP, W, false>(sw + L.w_off[T + 1], sw + L.b_off[T + 1], h, cat);
    encode_f32<LD>(d, cat + W);
    dense_f32<W + D, DP, W, true>(sw + L.w_off[T + 2], sw + L.b_off[T + 2], cat, h2);
    float z[3];
    dense_f32<W, WP, 3, false>(sw + L.w_off[T + 3], sw + L.b_off[T + 3], h2, z);
    if (act) {
      put(2 * W, cat, W);
      put(3 * W, h2, W);
      act[W] = make_float4(sig[0], z[0], z[1], z[2]);
    }
    io.store(idx, tl.y + threadIdx.x, sigmoid_split(z[0]), sigmoid_split(z[1]), sigmoid_split(z[2]), sig[0]);
  }
}

template <int W, class IO>
void launch_fp32_width(const float* packed, const Fp32Layout& L, const TileSched& S, const IO& io, cudaStream_t st) {
  size_t smem = (size_t)L.cell_floats * sizeof(float);
  auto k = k_mlp_fp32<W, 2, 10, 4, IO>;
  static thread_local size_t smem_set = 0;  // attribute set once per thread (outside graph capture)
  if (smem_set < smem) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set = smem;
  }
  k<<<num_sms() * 4, 128, smem, st>>>(packed, L, S, io);
}

void launch_fp32_w32(const float* packed, const Fp32Layout& L, const TileSched& S, const RenderIO& io, cudaStream_t st);
void launch_fp32_w32(const float* packed, const Fp32Layout& L, const TileSched& S, const QueryIO& io, cudaStream_t st);
void launch_fp32_w64(const float* packed, const Fp32Layout& L, const TileSched& S, const RenderIO& io, cudaStream_t st);
void launch_fp32_w64(const float* packed, const Fp32Layout& L, const TileSched& S, const QueryIO& io, cudaStream_t st);

}  // namespace gf
