// fp32 SIMT tiny-MLP: launch glue and weight packing (kernel template in
// gf_mlp_simt.cuh; widths 32 / 64 are instantiated in gf_mlp_simt32.cu /
// gf_mlp_simt64.cu so they compile in parallel).
#include "gf_mlp_simt.cuh"

namespace gf {

template <class IO>
static bool launch_fp32(const LayerTable& t, const float* packed, const TileSched& S, const IO& io, cudaStream_t st) {
  Fp32Layout L = make_fp32_layout(t);
  const bool tiny = t.pos_dim == 63 && t.dir_dim == 27 && t.view == t.width && t.trunk == 2 && t.skip < 0;
  if (!tiny) return false;
  if (t.width == 32) { launch_fp32_w32(packed, L, S, io, st); return true; }
  if (t.width == 64) { launch_fp32_w64(packed, L, S, io, st); return true; }
  return false;
}

bool prepare_mlp_fp32(const LayerTable& t) {
  return t.pos_dim == 63 && t.dir_dim == 27 && t.view == t.width && t.trunk == 2 && t.skip < 0 &&
         (t.width == 32 || t.width == 64);
}

bool launch_mlp_fp32_render(const LayerTable& t, const float* packed, const TileSched& S, const RenderIO& io,
                            cudaStream_t st) {
  return launch_fp32(t, packed, S, io, st);
}

bool launch_mlp_fp32_query(const LayerTable& t, const float* packed, const TileSched& S, const QueryIO& io,
                           cudaStream_t st) {
  return launch_fp32(t, packed, S, io, st);
}

// ---------------------------------------------------------------------------
// packing: layer-major (n_cells, out, in) -> per-cell padded blob
// (replaces MlpParams.at(cells) gathers, mlp.py:148-154)
// ---------------------------------------------------------------------------
struct PackArgs {
  const float* w[GF_MAX_LAYERS];
  const float* b[GF_MAX_LAYERS];
};

__global__ void k_pack_fp32(LayerTable t, Fp32Layout L, PackArgs A, int64_t n_cells, float* packed) {
  int64_t cell = blockIdx.x;
  if (cell >= n_cells) return;
  float* dst = packed + cell * L.cell_floats;
  for (int l = 0; l < t.n_layers; ++l) {
    const int in = t.in[l], out = t.out[l], ip = L.in_pad[l];
    const float* w = A.w[l] + cell * (int64_t)in * out;
    for (int j = threadIdx.x; j < out * ip; j += blockDim.x) {
      int o = j / ip, i = j % ip;
      dst[L.w_off[l] + j] = i < in ? w[o * in + i] : 0.f;
    }
    for (int j = threadIdx.x; j < gf_pad4(out); j += blockDim.x)
      dst[L.b_off[l] + j] = j < out ? A.b[l][cell * out + j] : 0.f;
  }
}

bool launch_pack_fp32(const LayerTable& t, int64_t n_cells, const float* const* w, const float* const* b,
                      float* packed, cudaStream_t st) {
  Fp32Layout L = make_fp32_layout(t);
  PackArgs A;
  for (int l = 0; l < t.n_layers; ++l) { A.w[l] = w[l]; A.b[l] = b[l]; }
  if (n_cells > 0) k_pack_fp32<<<(unsigned)n_cells, 256, 0, st>>>(t, L, A, n_cells, packed);
  return true;
}

}  // namespace gf
