// Per-cell tiny-MLP evaluation: shared declarations.
//
// Reference: mlp.py:73-84 (layer manifest), mlp.py:222-266 (forward),
// core.py:132-152 (positional encoding), batched.py:120-151 (grouped eval).
#pragma once
#include "gf_bucket.cuh"

namespace gf {

#define GF_MAX_LAYERS 16

// Layer table for one architecture; manifest order trunk0..trunk{T-1},
// density, feature, direction, color (mlp.py:73-84).
struct LayerTable {
  int n_layers, trunk, width, view, pos_dim, dir_dim;
  int skip;  // trunk layer whose input is [gamma(x), h] (mlp.py:79-81), -1: none
  int in[GF_MAX_LAYERS], out[GF_MAX_LAYERS];
};

__host__ inline bool make_layer_table(const gf_arch_t* a, LayerTable* t) {
  if (a->hidden_layers < 3 || a->width < 1 || a->hidden_layers - 2 + 4 > GF_MAX_LAYERS) return false;
  t->trunk = a->hidden_layers - 2;
  t->width = a->width;
  t->view = a->view_width > 0 ? a->view_width : a->width;
  t->pos_dim = 3 * ((a->include_raw ? 1 : 0) + 2 * a->pos_freqs);
  t->dir_dim = 3 * ((a->include_raw ? 1 : 0) + 2 * a->dir_freqs);
  t->skip = a->skip_layer > 0 ? a->skip_layer : -1;
  if (t->skip >= t->trunk) return false;  // mlp.py:63-64: 1 <= skip_layer < trunk layers
  int l = 0;
  t->in[l] = t->pos_dim; t->out[l++] = t->width;
  for (int k = 1; k < t->trunk; ++k) {
    t->in[l] = k == t->skip ? t->width + t->pos_dim : t->width;
    t->out[l++] = t->width;
  }
  t->in[l] = t->width; t->out[l++] = 1;                      // density
  t->in[l] = t->width; t->out[l++] = t->width;               // feature
  t->in[l] = t->width + t->dir_dim; t->out[l++] = t->view;   // direction
  t->in[l] = t->view; t->out[l++] = 3;                       // color
  t->n_layers = l;
  return true;
}

// fp32 packed layout: per cell, per layer, W rows padded to a multiple of 4
// floats (16-byte aligned rows for LDS.128), then the bias padded to 4.
struct Fp32Layout {
  int w_off[GF_MAX_LAYERS], b_off[GF_MAX_LAYERS], in_pad[GF_MAX_LAYERS];
  int cell_floats;
};

__host__ __device__ inline int gf_pad4(int x) { return (x + 3) & ~3; }

__host__ inline Fp32Layout make_fp32_layout(const LayerTable& t) {
  Fp32Layout L;
  int off = 0;
  for (int l = 0; l < t.n_layers; ++l) {
    L.in_pad[l] = gf_pad4(t.in[l]);
    L.w_off[l] = off;
    off += t.out[l] * L.in_pad[l];
    L.b_off[l] = off;
    off += gf_pad4(t.out[l]);
  }
  L.cell_floats = off;
  return L;
}

// Sources / sinks of MLP rows ------------------------------------------------
// Render: rows are kept samples in the ray-major staging buffer; the view
// direction is the ray's (render.py:326).
struct TileSched {
  const uint2* tiles;       // gf_make_tile entries
  const uint32_t* n_tiles;
  const uint32_t* sorted;   // query paths without moved records: caller row per sorted row (NULL: identity)
  const float4* srec;       // sorted records (x, y, z, index bits): render path and bulk queries
  const float4* sdir;       // bulk queries: sorted directions (x, y, z, 0)
};

struct RenderIO {
  static constexpr bool kDirEnc = true;  // tensor-core path reads the ray's pre-encoded gamma(d)
  static constexpr bool kHasAct = false;
  float4* res;
  const float4* ray_dir;
  uint32_t stride;
  const uint4* denc;  // 4 x uint4 per ray (gf_encode.cuh encode_direction_h), from k_ray_init
  int stride_shift;   // log2(stride) when stride is a power of two, else -1
  __device__ __forceinline__ uint32_t ray_of(uint32_t idx) const {
    return stride_shift >= 0 ? idx >> stride_shift : idx / stride;
  }
  // sorted row -> (staging index, position[, direction])
  template <bool DIR>
  __device__ __forceinline__ void fetch(const TileSched& S, uint32_t row, uint32_t& idx, float* x, float* d) const {
    const float4 r = gf_ld_hint(S.srec + row, gf_pol_first());
    idx = __float_as_uint(r.w);
    x[0] = r.x; x[1] = r.y; x[2] = r.z;
    if (DIR) {
      const float4 dd = ray_dir[ray_of(idx)];
      d[0] = dd.x; d[1] = dd.y; d[2] = dd.z;
    }
  }
  __device__ __forceinline__ void load_denc(uint32_t idx, uint32_t, uint4* de) const {
    const uint4* q = denc + 4ull * ray_of(idx);
#pragma unroll
    for (int c = 0; c < 4; ++c) de[c] = q[c];
  }
  __device__ __forceinline__ void store(uint32_t idx, uint32_t, float r, float g, float b, float s) const {
    gf_st_hint(res + idx, make_float4(r, g, b, s), gf_pol_last());  // read by the next march pass
  }
};

// Bulk query: caller's float32 (N,3) arrays, results in caller order.
struct QueryIO {
  static constexpr bool kDirEnc = true;  // direction gathered + encoded one layer ahead of its use (load_denc)
  static constexpr bool kHasAct = true;
  const float* pos;
  const float* dir;
  float* rgb;
  float* sigma;
  const int64_t* store_idx;  // optional: row idx is written to store_idx[idx] (grouped_forward)
  const float4* sdir;        // bulk path: directions in sorted order (read by sorted row)
  template <bool DIR>
  __device__ __forceinline__ void fetch(const TileSched& S, uint32_t row, uint32_t& idx, float* x, float* d) const {
    if (S.srec) {  // records moved into sorted order by the bucketing pass
      const float4 r = S.srec[row];
      idx = __float_as_uint(r.w);
      x[0] = r.x; x[1] = r.y; x[2] = r.z;
      if (DIR) {
        const float4 q = S.sdir[row];
        d[0] = q.x; d[1] = q.y; d[2] = q.z;
      }
      return;
    }
    idx = S.sorted ? S.sorted[row] : row;
    const float* p = pos + 3ull * idx;
    x[0] = p[0]; x[1] = p[1]; x[2] = p[2];
    if (DIR) {
      const float* q = dir + 3ull * idx;
      d[0] = q[0]; d[1] = q[1]; d[2] = q[2];
    }
  }
  float4* sorted_out;        // bulk path: results in sorted-row order (un-permuted by a coalesced gather pass)
  __device__ __forceinline__ void store(uint32_t row, uint32_t srow, float r, float g, float b, float s) const {
    if (sorted_out) {
      sorted_out[srow] = make_float4(r, g, b, s);
      return;
    }
    const uint64_t idx = store_idx ? (uint64_t)store_idx[row] : (uint64_t)row;
    rgb[3ull * idx + 0] = r;
    rgb[3ull * idx + 1] = g;
    rgb[3ull * idx + 2] = b;
    sigma[idx] = s;
  }
  __device__ __forceinline__ void load_denc(uint32_t idx, uint32_t row, uint4* de) const;  // gf_mlp_tc.cu
  // training forward (fp32 SIMT kernel, 32-wide tiny manifest): per grouped
  // row the activations the backward needs, GF_ACT_FLOATS floats:
  // [h0 | h1 | feature | g | sigma | color logits]
  float* act;
};
#define GF_ACT_FLOATS 132

// launchers (gf_mlp_simt.cu / gf_mlp_tc.cu); return false if the architecture
// has no compiled variant
bool launch_mlp_fp32_render(const LayerTable& t, const float* packed, const TileSched& S, const RenderIO& io,
                            cudaStream_t st);
bool launch_mlp_fp32_query(const LayerTable& t, const float* packed, const TileSched& S, const QueryIO& io,
                           cudaStream_t st);
bool launch_pack_fp32(const LayerTable& t, int64_t n_cells, const float* const* w, const float* const* b,
                      float* packed, cudaStream_t st);

// fp16 tcgen05 path
size_t fp16_cell_bytes(const LayerTable& t);
bool launch_pack_fp16(const LayerTable& t, int64_t n_cells, const float* const* w, const float* const* b,
                      void* packed, cudaStream_t st);
bool launch_mlp_tc_render(const LayerTable& t, const void* packed, const TileSched& S, const RenderIO& io,
                          cudaStream_t st);
bool launch_mlp_tc_query(const LayerTable& t, const void* packed, const TileSched& S, const QueryIO& io,
                         cudaStream_t st);

// any manifest (depth, widths, skip layer, octaves): fp32 SIMT, gf_mlp_generic.cu
bool generic_mlp_supported(const LayerTable& t);
bool launch_mlp_generic_render(const LayerTable& t, const gf_arch_t* arch, const float* packed, const TileSched& S,
                               const RenderIO& io, cudaStream_t st);
bool launch_mlp_generic_query(const LayerTable& t, const gf_arch_t* arch, const float* packed, const TileSched& S,
                              const QueryIO& io, cudaStream_t st);
bool prepare_mlp_generic(const LayerTable& t, const gf_arch_t* arch);

// mlp.forward / mlp.backward on encoded inputs, any manifest, f32 / f64:
// gf_mlp_dense.cu
bool dense_mlp_supported(const gf_manifest_t* m);
size_t dense_backward_workspace(const gf_manifest_t* m, int f64, int64_t n_net, int64_t rows);
bool launch_dense_forward(const gf_manifest_t* m, int f64, int64_t n_net, int64_t rows, const void* const* w,
                          const void* const* b, const void* x, const void* d, void* color, void* sigma,
                          void* const* hs, void* feat, void* g, cudaStream_t st);
bool launch_dense_backward(const gf_manifest_t* m, int f64, int64_t n_net, int64_t rows, const void* const* w,
                           const void* x, const void* d, const void* const* hs, const void* feat, const void* g,
                           const void* color, const void* sigma, const void* d_color, const void* d_sigma,
                           void* const* gw, void* const* gb, void* ws, cudaStream_t st);

int num_sms();

// one-time per-process launch setup (smem attribute, residency) done outside
// graph capture; return false if the architecture has no compiled variant
bool prepare_mlp_fp32(const LayerTable& t);
bool prepare_mlp_tc(const LayerTable& t);

}  // namespace gf
