// tcgen05 fp16 tiny-MLP kernel (placeholder until the tensor-core path lands).
#include "gf_mlp.cuh"

namespace gf {
size_t fp16_cell_bytes(const LayerTable& t) { (void)t; return 0; }
bool launch_pack_fp16(const LayerTable&, int64_t, const float* const*, const float* const*, void*, cudaStream_t) {
  return false;
}
bool launch_mlp_tc_render(const LayerTable&, const void*, const TileSched&, const RenderIO&, cudaStream_t) {
  return false;
}
bool launch_mlp_tc_query(const LayerTable&, const void*, const TileSched&, const QueryIO&, cudaStream_t) {
  return false;
}
}  // namespace gf
