// Instantiation of the fp32 SIMT MLP kernel for hidden width 32.
#include "gf_mlp_simt.cuh"

namespace gf {
void launch_fp32_w32(const float* packed, const Fp32Layout& L, const TileSched& S, const RenderIO& io, cudaStream_t st) {
  launch_fp32_width<32>(packed, L, S, io, st);
}
void launch_fp32_w32(const float* packed, const Fp32Layout& L, const TileSched& S, const QueryIO& io, cudaStream_t st) {
  launch_fp32_width<32>(packed, L, S, io, st);
}
}  // namespace gf
