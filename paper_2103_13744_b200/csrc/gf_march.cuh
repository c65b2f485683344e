// Marcher data structures shared by gf_march.cu and gf_api.cu.
#pragma once
#include "gf_common.cuh"

#define GF_RAY_ALIVE 1
#define GF_RAY_HIT 2
#define GF_RAY_TERMINATED 4

namespace gf {

struct MarchParams {
  GfGrid grid;        // network lattice geometry (cell keys)
  GfGrid occ;         // occupancy geometry
  const uint8_t* occ_bits;
  gf_camera_t cam;
  int use_cam;
  const float* origins;
  const float* dirs;
  int64_t ray_offset, n_rays, first_block;
  const u128* block_seeds;  // [2*b] state, [2*b+1] inc
  int k, chunk, n_rounds, stride, stratified, ert, eps_f64;
  double epsilon;
  float bg[3];
  float* rgb_out;
  int64_t* stats;
  gf_trace_rec_t* trace;
  int64_t trace_capacity;
  int64_t* trace_count;
};

// Per-ray state for the whole frame (SoA, 16-byte aligned).
struct RayState {
  float4* org;    // ox, oy, oz, t0_32
  float4* dir;    // dx, dy, dz, seg_32
  float4* acc;    // r, g, b, transmittance
  u128* rng;      // PCG64 state positioned at the ray's next float32 draw
  uint32_t* run;  // queried samples of the ray in the last marched round
  uint8_t* flags;
};

// Per-round buffers.  Staging is ray-major with a fixed stride (= chunk): the
// kept samples of ray i in this round are rec[i*stride .. i*stride+run[i]),
// in slot order, which is the order compositing consumes them.
struct RoundBufs {
  float4* rec;        // x, y, z, cell(bits)
  float4* res;        // r, g, b, sigma written by the MLP
  uint32_t* counts;   // per-cell histogram of this round
};

__global__ void k_seed_blocks(uint64_t seed, int64_t first_block, int64_t n_blocks, u128* seeds);
__global__ void k_ray_init(MarchParams P, RayState R);
__global__ void k_march(MarchParams P, RayState R, RoundBufs B, int round);

}  // namespace gf
