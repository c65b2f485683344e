// Marcher data structures shared by gf_march.cu and gf_api.cu.
#pragma once
#include "gf_bucket.cuh"

#define GF_RAY_ALIVE 1
#define GF_RAY_HIT 2
#define GF_RAY_TERMINATED 4
#define GF_RAY_HAD 8         // queried samples in the last marched round (composite them next pass)
#define GF_RAY_ALLROUNDS 16  // no per-round candidate mask: every round is a candidate round
#define GF_RAY_HAD_ALL (8u | 32u | 64u | 128u)  // grouped rounds: round p of the group queried samples
// flag bit of round p of a group (p = 0 is GF_RAY_HAD), and of rounds < p
__host__ __device__ __forceinline__ uint32_t gf_had_bit(int p) { return p == 0 ? 8u : (16u << p); }
__host__ __device__ __forceinline__ uint32_t gf_had_below(int p) {
  return p <= 0 ? 0u : (p == 1 ? 8u : (p == 2 ? 40u : 104u));
}

namespace gf {

#define GF_STAT_SLOTS 1024  // warps flush their counters into slot (warp id mod 1024)

struct MarchParams {
  GfGrid grid;        // network lattice geometry (cell keys)
  GfGrid occ;         // occupancy geometry
  const uint8_t* occ_bits;
  GfGrid coarse;      // dilated coarse occupancy mip (empty-space pre-test)
  const uint32_t* coarse_bits;  // NULL: every candidate takes the exact path
  float ivl_pad;      // world-distance padding of the DDA intervals (float32 error)
  unsigned long long* stats_part;  // GF_STAT_SLOTS x GF_STAT_COUNT partial counters (spread: no hot address)
  const uint32_t* fine_bits;  // occupancy dilated by >= seg/2 + margin (occupancy geometry): per-candidate
                              // pre-test at the segment midpoint, before the jitter and the exact placement
  const uint64_t* occ_brick;  // the occupancy bits regrouped per 4^3 brick (one u64 per coarse cell, bit
                              // x + 4y + 16z): a ray's consecutive samples share a word (k_march<true>)
  int brick_cx, brick_cy;     // bricks per row / per column
  const uint32_t* occ_bbox;   // set cells of the dilated coarse mip: x,y,z min then max (coarse cells);
                              // the ray's DDA runs only inside this box (min > max: no set cell)
  gf_camera_t cam;
  int use_cam;
  const float* origins;   // (n, 3) float32, or double when rays_f64
  const float* dirs;
  int rays_f64;
  int64_t ray_offset, n_rays, first_block, block_stride;
  const u128* block_seeds;  // [2*b] state, [2*b+1] inc
  const u128* jump;         // [2*d] A^d, [2*d+1] sum_{k<d} A^k  (d <= GF_JUMP_MAX)
  const u128* start;        // [2*r], [2*r+1]: the same pair for the jump to block row r's first draw
  const u128* round_jump;   // [2*(2*round+parity)], +1: jump from a ray's slot-0 word to round's first word
  const u128* block_ci;     // [b*GF_CI_N + d] = (sum_{k<d} A^k) * inc_b: the increment part of a d-word jump
  int net_from_occ;         // network cell = occupancy cell >> net_shift per axis (see gf_api.cu)
  int net_shift[3];
  int k, chunk, n_rounds, stride, stratified, ert, eps_f64;
  int group;          // rounds per group (1, 2 or 4): placed by G passes, evaluated together, composited in order
  int fuse;           // one marcher launch places all of a group's rounds
  int tile2d, tiles_x;  // k_march thread -> ray map: 8x4 pixel tiles per warp, 2x2 of them per CTA (whole-image calls)
  int64_t n_cells;
  int64_t march_threads;
  int count_candidates;  // diagnostics (GF_COUNT_CANDIDATES=1): exact-path candidates added to stats[N_RAYS]
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
  u128* rng;      // PCG64 state of the word holding the ray's slot-0 float32 draw
  uint32_t* run;  // queried samples of the ray in the last marched round (groups: one byte per round)
  uint32_t* pend; // groups: [4] per ray, round p's (queries | ess_skipped << 16), committed if the ray survives rounds < p
  uint32_t* flags;  // GF_RAY_* bits | (rounds with candidate slots, bit r) << 8
  uint32_t* ivl;  // GF_MAX_IVL candidate slot ranges per ray (lo | hi << 16), from the coarse DDA
  uint4* denc;    // NULL, or 4 x uint4 per ray: gamma(d) as fp16 for the tensor-core MLP
};

#define GF_MAX_IVL 8
#define GF_IVL_ALL 0xFFFFFFFFu  // sentinel in ivl[0]: every slot is a candidate

// Per-round buffers.  Staging is ray-major with a fixed stride (= chunk): the
// kept samples of ray i in this round are rec[i*stride .. i*stride+run[i]),
// in slot order, which is the order compositing consumes them.
struct RoundBufs {
  float4* rec;        // x, y, z, rank of the sample inside its cell's segment (bits)
  float4* res;        // r, g, b, sigma written by the MLP
  uint32_t* counts;   // [2][n_cells] per-cell histograms, by round parity
  uint32_t* emit_list;   // rays that queried samples this round (for the scatter)
  uint32_t* emit_count;  // [2], indexed by round parity
};

// Global index (within the render_rays call) of the call's local ray i.
// block_stride S > 1 interleaves 4096-ray blocks across shards: local block
// lb is global block ray_offset/4096 + lb*S (ray_offset is block-aligned).
__device__ __forceinline__ int64_t global_ray(const MarchParams& P, int64_t i) {
  if (P.block_stride == 1) return P.ray_offset + i;
  return P.ray_offset + (i / GF_RAY_BLOCK) * P.block_stride * GF_RAY_BLOCK + i % GF_RAY_BLOCK;
}
// k_march thread -> call-local ray index; with tile2d a warp covers an 8x4
// pixel tile so its rays cross the same cells at the same rounds (coherent
// branches); out-of-image lanes get n_rays (inactive).
__device__ __forceinline__ int64_t march_ray(const MarchParams& P, int64_t t) {
  if (!P.tile2d) return t;
  const uint32_t warp = (uint32_t)(t >> 5), lane = (uint32_t)t & 31u;  // < 2^32 warps per call
  uint32_t ty, tx;
  if (P.tile2d == 2) {  // a CTA's 4 warps cover 2x2 tiles (16x8 pixels): P.tiles_x counts CTA columns
    const uint32_t cta = warp >> 2, wib = warp & 3u;
    const uint32_t cy = cta / (uint32_t)P.tiles_x, cx = cta - cy * (uint32_t)P.tiles_x;
    tx = 2 * cx + (wib & 1u);
    ty = 2 * cy + (wib >> 1);
  } else {
    ty = warp / (uint32_t)P.tiles_x;
    tx = warp - ty * (uint32_t)P.tiles_x;
  }
  const int64_t x = (int64_t)(tx * 8u + (lane & 7u)), y = (int64_t)(ty * 4u + (lane >> 3));
  return (x < P.cam.width && y < P.cam.height) ? y * P.cam.width + x : P.n_rays;
}
// slot of the ray's block in the per-call seed table
__device__ __forceinline__ int64_t seed_slot(const MarchParams& P, int64_t g) {
  const int64_t b = g / GF_RAY_BLOCK - P.first_block;
  return P.block_stride == 1 ? b : b / P.block_stride;  // no 64-bit division on the unsharded path
}

#define GF_JUMP_MAX 32  // largest PCG64 jump inside one round (chunk <= 32 -> <= 16 outputs)
#define GF_CI_N 17      // per-block increment terms for jumps of 0..16 words

// K2 for the render path (fused scan + tile list + rank-based placement);
// returns the number of launches it made
void launch_stats_fold(const unsigned long long* part, int64_t* stats, cudaStream_t st);
int launch_place(const GfGrid& grid, const RoundBufs& RB, const uint32_t* run, const BucketBufs& Bk, int64_t n_cells,
                 int stride, int half, int round, int64_t max_rows, cudaStream_t st);

__global__ void k_seed_blocks(uint64_t seed, int64_t first_block, int64_t block_stride, int64_t n_blocks,
                              int k, int chunk, int n_rounds, u128* seeds, u128* jump, u128* start,
                              u128* round_jump, u128* block_ci);
__global__ void k_ray_init(MarchParams P, RayState R);
__global__ void k_coarse_reduce(const uint8_t* occ_bits, int3 occ_res, int factor, int3 cres, uint8_t* coarse);
__global__ void k_coarse_dilate(const uint8_t* coarse, int3 cres, int radius, uint32_t* bits);
__global__ void k_coarse_reduce_w(const uint32_t* fine, int3 ores, int f, int3 cres, uint32_t* out, uint64_t* brick,
                                  uint32_t* bbox);
__global__ void k_dilate_x(const uint32_t* in, uint32_t* out, int3 cres, int r);
__global__ void k_dilate_yz(const uint32_t* in, uint32_t* out, int3 cres, int r, int axis, uint32_t* bbox);

// Approximate (clamped) coarse cell of a float32 point; exactness is not
// needed because the mip is dilated past the evaluation error.
__device__ __forceinline__ uint32_t gf_coarse_cell(const GfGrid& g, float x, float y, float z) {
  float v[3] = {x, y, z};
  int idx[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float q = (v[a] - g.b_min_f[a]) * g.inv_cell_f[a];
    q = fminf(fmaxf(q, 0.f), (float)(g.res[a] - 1));
    idx[a] = __float_as_int(__fadd_rz(q, 8388608.0f)) - 0x4B000000;
  }
  return (uint32_t)(idx[0] + g.res[0] * (idx[1] + g.res[1] * idx[2]));
}
template <bool FAST>
__global__ void k_march(MarchParams P, RayState R, RoundBufs B, int round, int phase);

}  // namespace gf
