// Shared device helpers for the gridfield B200 kernels.
//
// Exactness contract: everything that decides *which* samples exist and which
// cell they land in (ray directions, slab test, sample distance, clip, binning)
// is computed with explicitly rounded IEEE intrinsics (__dadd_rn, __dmul_rn,
// __ddiv_rn, ...) so nvcc cannot contract to FMA; the same operation order as
// the numpy reference gives bit-identical sample positions and cell indices.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gridfield_b200.h"

#define GF_RAY_BLOCK 4096  // render.py:22 RAY_BLOCK
#define GF_TILE_ROWS 128   // MLP rows per tile (one TMEM lane per row)

typedef unsigned __int128 u128;

// ---------------------------------------------------------------------------
// numpy PCG64 (XSL-RR 128/64) and SeedSequence, host + device
// ---------------------------------------------------------------------------
#define GF_PCG_MULT ((((u128)0x2360ED051FC65DA4ull) << 64) | (u128)0x4385DF649FCCF645ull)

__host__ __device__ __forceinline__ uint64_t gf_pcg_output(u128 s) {
  uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  uint64_t x = hi ^ lo;
  unsigned rot = (unsigned)(hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

// one 32-bit half of gf_pcg_output(s) (the float32 draw numpy takes from
// it): the 64-bit rotate collapses to one funnel shift of the xor'd halves
__device__ __forceinline__ uint32_t gf_pcg_output_half(u128 s, uint32_t hi_half) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const uint64_t x = hi ^ lo;
  const uint32_t rot = (uint32_t)(hi >> 58);
  const uint32_t xl = (uint32_t)x, xh = (uint32_t)(x >> 32);
  const bool sw = (((rot >> 5) ^ hi_half) & 1u) != 0;
  return __funnelshift_r(sw ? xh : xl, sw ? xl : xh, rot);
}

__host__ __device__ __forceinline__ u128 gf_pcg_step(u128 s, u128 inc) { return s * GF_PCG_MULT + inc; }

// LCG jump-ahead by `delta` steps (Brown, "Random number generation with
// arbitrary strides").
__host__ __device__ inline u128 gf_pcg_advance(u128 s, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = GF_PCG_MULT, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * s + acc_plus;
}

struct GfHash {
  uint32_t c, m;
  __host__ __device__ uint32_t operator()(uint32_t v) {
    v ^= c;
    c *= m;
    v *= c;
    return v ^ (v >> 16);
  }
};

__host__ __device__ __forceinline__ uint32_t gf_ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
  return r ^ (r >> 16);
}

// PCG64(SeedSequence([seed, block_start])) -> (state, inc).  Entropy words are
// the little-endian uint32 limbs of each integer (0 -> one zero word).
__host__ __device__ inline void gf_seed_block(uint64_t seed, uint64_t block_start, u128* state, u128* inc) {
  uint32_t w[4];
  int nw = 0;
  uint64_t v = seed;
  if (v == 0) w[nw++] = 0;
  while (v) { w[nw++] = (uint32_t)v; v >>= 32; }
  v = block_start;
  if (v == 0) w[nw++] = 0;
  while (v) { w[nw++] = (uint32_t)v; v >>= 32; }
  GfHash ha{0x43B0D7E5u, 0x931E8875u};
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = ha(i < nw ? w[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = gf_ss_mix(pool[d], ha(pool[s]));
  for (int s = 4; s < nw; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = gf_ss_mix(pool[d], ha(w[s]));
  GfHash hb{0x8B51F9DDu, 0x58F38DEDu};
  uint64_t g[4];
  for (int i = 0; i < 4; ++i) {
    uint32_t lo = hb(pool[(2 * i) & 3]);
    uint32_t hi = hb(pool[(2 * i + 1) & 3]);
    g[i] = (uint64_t)lo | ((uint64_t)hi << 32);
  }
  u128 initstate = ((u128)g[0] << 64) | g[1];
  u128 initseq = ((u128)g[2] << 64) | g[3];
  u128 c = (initseq << 1) | 1;
  u128 s = c;  // step from state 0
  s += initstate;
  s = gf_pcg_step(s, c);
  *state = s;
  *inc = c;
}

__device__ __forceinline__ float gf_u32_to_unit_float(uint32_t u) {
  return (float)(u >> 8) * (1.0f / 16777216.0f);
}

// ---------------------------------------------------------------------------
// exact binning (core.py:79-112)
// ---------------------------------------------------------------------------
struct GfGrid {
  double b_min[3], b_max[3], cell[3], inv_cell[3];
  float b_min_f[3], b_max_f[3], inv_cell_f[3];
  int32_t res[3];
  int32_t pow2;    // all cell sizes are powers of two: x*inv is exact == x/cell
  int32_t fast;    // pow2 && bounds exactly representable in float32 (see gf_bin_axis_fast)
};

__host__ inline GfGrid gf_make_grid(const gf_grid_geom_t* g) {
  GfGrid o;
  bool p2 = true, f32 = true;
  for (int a = 0; a < 3; ++a) {
    o.b_min[a] = g->b_min[a];
    o.b_max[a] = g->b_max[a];
    o.res[a] = g->res[a];
    o.cell[a] = (g->b_max[a] - g->b_min[a]) / (double)g->res[a];
    o.inv_cell[a] = 1.0 / o.cell[a];
    o.b_min_f[a] = (float)g->b_min[a];
    o.b_max_f[a] = (float)g->b_max[a];
    o.inv_cell_f[a] = (float)o.inv_cell[a];
    int e;
    double m = frexp(o.cell[a], &e);
    if (m != 0.5) p2 = false;
    if ((double)o.b_min_f[a] != g->b_min[a] || (double)o.b_max_f[a] != g->b_max[a] || g->res[a] > (1 << 22) ||
        (double)o.inv_cell_f[a] != o.inv_cell[a])
      f32 = false;
  }
  o.pow2 = p2 ? 1 : 0;
  o.fast = (p2 && f32) ? 1 : 0;
  return o;
}

// Exact float32 route to floor((f64(x) - b_min) / cell) for x >= b_min, valid
// when b_min is float32-exact and cell is a power of two (grid.fast):
// y = RZ(x - b_min) is the largest float <= the exact difference v, and every
// cell boundary n*cell is a float, so y >= n*cell <=> v >= n*cell; y*inv is an
// exact power-of-two scaling; adding 2^23 with round-toward-zero leaves
// floor(q) in the mantissa.  No FP64 and no F2I conversions.
__device__ __forceinline__ int gf_bin_axis_fast(const GfGrid& g, int a, float x) {
  const float q = __fmul_rn(__fsub_rz(x, g.b_min_f[a]), g.inv_cell_f[a]);
  int i = __float_as_int(__fadd_rz(q, 8388608.0f)) - 0x4B000000;
  i = i < 0 ? 0 : i;
  return i < g.res[a] - 1 ? i : g.res[a] - 1;
}

// gf_bin_axis_fast for x already clipped into [b_min_f, b_max_f]: q >= 0,
// so only the upper clamp (x == b_max) remains
__device__ __forceinline__ int gf_bin_axis_clipped(const GfGrid& g, int a, float x) {
  const float q = __fmul_rn(__fsub_rz(x, g.b_min_f[a]), g.inv_cell_f[a]);
  const int i = __float_as_int(__fadd_rz(q, 8388608.0f)) - 0x4B000000;
  return i < g.res[a] - 1 ? i : g.res[a] - 1;
}

__device__ __forceinline__ uint32_t gf_flat_cell_fast(const GfGrid& g, float x, float y, float z) {
  int ix = gf_bin_axis_fast(g, 0, x), iy = gf_bin_axis_fast(g, 1, y), iz = gf_bin_axis_fast(g, 2, z);
  return (uint32_t)(ix + g.res[0] * (iy + g.res[1] * iz));
}

// floor((f64(x) - b_min) / cell) clamped to res-1; caller guarantees in-bounds.
__device__ __forceinline__ int gf_bin_axis(const GfGrid& g, int a, float x) {
  double r = __dsub_rn((double)x, g.b_min[a]);
  double q = g.pow2 ? __dmul_rn(r, g.inv_cell[a]) : __ddiv_rn(r, g.cell[a]);
  int i = (int)floor(q);
  return i < g.res[a] - 1 ? i : g.res[a] - 1;
}

__device__ __forceinline__ int gf_bin_axis(const GfGrid& g, int a, double x) {
  double r = __dsub_rn(x, g.b_min[a]);
  double q = g.pow2 ? __dmul_rn(r, g.inv_cell[a]) : __ddiv_rn(r, g.cell[a]);
  int i = (int)floor(q);
  return i < g.res[a] - 1 ? i : g.res[a] - 1;
}

__device__ __forceinline__ uint32_t gf_flat_cell(const GfGrid& g, double x, double y, double z) {
  int ix = gf_bin_axis(g, 0, x), iy = gf_bin_axis(g, 1, y), iz = gf_bin_axis(g, 2, z);
  return (uint32_t)(ix + g.res[0] * (iy + g.res[1] * iz));
}

__device__ __forceinline__ uint32_t gf_flat_cell(const GfGrid& g, float x, float y, float z) {
  if (g.fast) return gf_flat_cell_fast(g, x, y, z);
  int ix = gf_bin_axis(g, 0, x), iy = gf_bin_axis(g, 1, y), iz = gf_bin_axis(g, 2, z);
  return (uint32_t)(ix + g.res[0] * (iy + g.res[1] * iz));
}

// core.py:52-68 clip_into for one float32 component against f64 bounds.
__device__ __forceinline__ float gf_clip_component(float p, double lo, double hi) {
  double v = (double)p;
  v = v < lo ? lo : v;   // np.clip == minimum(maximum(x, lo), hi)
  v = v > hi ? hi : v;
  float c = __double2float_rn(v);
  if ((double)c > hi) c = nextafterf(c, -INFINITY);
  if ((double)c < lo) c = nextafterf(c, INFINITY);
  return c;
}

// clip_into when the bounds are float32-exact (grid.fast): clamping in f64 and
// casting back can then never leave the box, so it is a float32 clamp.
__device__ __forceinline__ float gf_clip_fast(float p, float lo, float hi) { return fminf(fmaxf(p, lo), hi); }

// ---------------------------------------------------------------------------
// L2 residency hints for the per-round staging buffers: records written by
// one kernel and read once by the next are stored evict_last and loaded
// evict_first, so they survive the streaming traffic in between.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t gf_pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));  // pure: hoisted out of loops
  return p;
}
__device__ __forceinline__ uint64_t gf_pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ float4 gf_ld_hint(const float4* a, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void gf_st_hint(float4* a, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w), "l"(pol)
               : "memory");
}

// ---------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned gf_lane() { return threadIdx.x & 31u; }

template <typename T>
__host__ __device__ __forceinline__ T gf_div_up(T a, T b) { return (a + b - 1) / b; }

__host__ __device__ __forceinline__ size_t gf_align(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL) between the frame's kernels: the next
// kernel of the round chain is launched early and its CTAs run their
// independent setup while the previous kernel drains; gf_pdl_wait() (before
// any read of the previous kernel's results) blocks until that kernel has
// completed and its writes are visible.  Outside a PDL launch both are no-ops.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void gf_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void gf_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool gf_pdl_enabled();  // gf_api.cu: on unless GF_NO_PDL=1

template <typename... KArgs, typename... Args>
inline cudaError_t gf_launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = gf_pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}
