// train.prepare_ray_samples on the device (gf_samples.cu).
#pragma once
#include "gf_common.cuh"

namespace gf {

struct PrepArgs {
  const float* origins;  // (n, 3) float32
  const float* dirs;     // (n, 3) float32
  int64_t n;
  int k, stratified;
  double b_min[3], b_max[3];
  u128 state, inc;       // the caller Generator's PCG64 state
  int has_uint32;
  uint32_t uinteger;
  GfGrid occ;
  const uint8_t* occ_bits;  // NULL: no empty-space skipping
  int64_t* offsets;      // (n + 1): per-ray counts, then exclusive offsets (offsets[n] = total)
  float* deltas;         // (n,) seg32
  double* pos;           // (Q, 3) float64 positions
  float* dir_out;        // (Q, 3) the ray's float32 direction
  int64_t* ray_index;    // (Q,)
  int64_t* slot;         // (Q,)
};

void launch_prepare_count(const PrepArgs& A, cudaStream_t st);
void launch_prepare_write(const PrepArgs& A, cudaStream_t st);

}  // namespace gf
