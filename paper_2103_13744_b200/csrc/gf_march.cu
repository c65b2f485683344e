// Ray marcher: ray generation, slab test, stratified PCG64 jitter, sample
// placement, clip, empty-space skipping, per-round emission, compositing and
// early ray termination.
//
// Reference: render.py:139-171 (rays, slab), render.py:287-348 (_march_block),
// render.py:351-384 (4096-ray blocks + SeedSequence jitter streams),
// core.py:52-112 (clip / bin), occupancy.py:65-79 (bit lookup),
// core.py:187-194 (alpha).
//
// One thread owns one ray for the whole frame.  Rounds (ert_chunk samples)
// are separate launches because the next round's live set depends on the
// MLP results of this round (chunk-granular ERT, render.py:338-343).
#include "gf_encode.cuh"
#include "gf_march.cuh"

namespace gf {

// -------------------------------------------------------------------------
// per-block PCG64 seeds: SeedSequence([seed, 4096*b])   (render.py:375)
// -------------------------------------------------------------------------
__global__ void k_seed_blocks(uint64_t seed, int64_t first_block, int64_t block_stride, int64_t n_blocks,
                              int k, int chunk, int n_rounds, u128* seeds, u128* jump, u128* start,
                              u128* round_jump, u128* block_ci) {
  gf_pdl_wait();
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) {
    // LCG jump table: S_{n+d} = A^d S_n + (sum_{k<d} A^k) inc, d = 0..GF_JUMP_MAX
    u128 a = 1, c = 0;
    for (int d = 0; d <= GF_JUMP_MAX; ++d) {
      jump[2 * d] = a;
      jump[2 * d + 1] = c;
      c = c * GF_PCG_MULT + 1;
      a = a * GF_PCG_MULT;
    }
  }
  if (b < GF_RAY_BLOCK) {
    // row r of a block starts at float32 draw r*k, i.e. after (r*k >> 1) + 1
    // PCG64 steps (each step yields two float32 draws): the same jump for
    // every block, so it is tabulated once per call instead of per ray
    const uint64_t d = (((uint64_t)b * (uint64_t)k) >> 1) + 1;
    start[2 * b] = gf_pcg_advance(1, 0, d);      // A^d
    start[2 * b + 1] = gf_pcg_advance(0, 1, d);  // sum_{j<d} A^j
  }
  if (b < 2 * n_rounds) {
    // round r of a ray whose slot-0 draw has parity p starts (p + r*chunk) >> 1
    // PCG64 words after the ray's slot-0 word
    const uint64_t d = ((uint64_t)(b & 1) + (uint64_t)(b >> 1) * (uint64_t)chunk) >> 1;
    round_jump[2 * b] = gf_pcg_advance(1, 0, d);
    round_jump[2 * b + 1] = gf_pcg_advance(0, 1, d);
  }
  if (b >= n_blocks) return;
  u128 s, inc;
  gf_seed_block(seed, (uint64_t)((first_block + b * block_stride) * GF_RAY_BLOCK), &s, &inc);
  seeds[2 * b] = s;
  seeds[2 * b + 1] = inc;
  u128 c = 0;  // sum_{k<d} A^k
  for (int d = 0; d < GF_CI_N; ++d) {
    block_ci[b * GF_CI_N + d] = c * inc;
    c = c * GF_PCG_MULT + 1;
  }
}

// -------------------------------------------------------------------------
// Candidate slot ranges of one ray: a 3-D DDA (Amanatides-Woo) through the
// dilated coarse mip collects the distance intervals [s_in, s_out] (from the
// entry point) where the ray is inside a set coarse cell; slot j is a
// candidate iff its nominal midpoint (j + 0.5) * seg lies in one (padded for
// float32 error).  Because the mip is dilated by >= seg/2 + margin, a
// non-candidate slot's sample provably lands in an empty fine cell.
// -------------------------------------------------------------------------
__device__ void coarse_intervals(const MarchParams& P, uint32_t* out, float ex, float ey, float ez, const float* d,
                                 float smax, float seg, float s_lo, float s_hi) {
  const GfGrid& g = P.coarse;
  // the walk runs over [s_lo, s_hi] of the ray (distances from its entry):
  // outside that range every coarse cell is clear (k_ray_init)
  const float pos[3] = {fmaf(d[0], s_lo, ex), fmaf(d[1], s_lo, ey), fmaf(d[2], s_lo, ez)};
  int cell[3], step[3];
  float snext[3], sdelta[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float q = (pos[a] - g.b_min_f[a]) * g.inv_cell_f[a];
    q = fminf(fmaxf(q, 0.f), (float)g.res[a] - 1e-3f);
    cell[a] = (int)floorf(q);
    cell[a] = cell[a] < g.res[a] - 1 ? cell[a] : g.res[a] - 1;
    const float v = d[a] * g.inv_cell_f[a];  // cells per unit distance
    if (v > 0.f) {
      step[a] = 1;
      snext[a] = ((float)(cell[a] + 1) - q) / v;
      sdelta[a] = 1.f / v;
    } else if (v < 0.f) {
      step[a] = -1;
      snext[a] = ((float)cell[a] - q) / v;
      sdelta[a] = -1.f / v;
    } else {
      step[a] = 0;
      snext[a] = INFINITY;
      sdelta[a] = INFINITY;
    }
  }
  const float inv_seg = 1.f / seg;
  const float kmax = (float)(P.k - 1);
  int n = 0;
  auto emit = [&](float sa, float sb) {
    float lo = floorf((sa - P.ivl_pad) * inv_seg - 0.5f), hi = ceilf((sb + P.ivl_pad) * inv_seg - 0.5f);
    lo = fmaxf(lo, 0.f);
    hi = fminf(hi, kmax);
    if (lo > hi) return;
    const uint32_t v = (uint32_t)lo | ((uint32_t)hi << 16);
    if (n < GF_MAX_IVL) {
      out[n++] = v;
    } else {  // out of room: widen the last range (conservative)
      out[GF_MAX_IVL - 1] = (out[GF_MAX_IVL - 1] & 0xFFFFu) | ((uint32_t)hi << 16);
    }
  };
  // per-axis state in scalars (no local-memory arrays): next crossing
  // distance, crossing spacing, flat-index delta and steps left in the grid
  const int rx = g.res[0], rxy = g.res[0] * g.res[1];
  float n0 = s_lo + snext[0], n1 = s_lo + snext[1], n2 = s_lo + snext[2];
  const float e0 = sdelta[0], e1 = sdelta[1], e2 = sdelta[2];
  const int f0 = step[0], f1 = step[1] * rx, f2 = step[2] * rxy;
  int l0 = step[0] > 0 ? g.res[0] - 1 - cell[0] : cell[0];
  int l1 = step[1] > 0 ? g.res[1] - 1 - cell[1] : cell[1];
  int l2 = step[2] > 0 ? g.res[2] - 1 - cell[2] : cell[2];
  int c = cell[0] + rx * cell[1] + rxy * cell[2];
  float s = s_lo, s_open = s_lo;
  bool open = false;
  for (int it = 0; it < 4096; ++it) {
    const bool occ = (__ldg(P.coarse_bits + (c >> 5)) >> (c & 31)) & 1;
    if (occ != open) {
      if (occ) s_open = s;
      else emit(s_open, s);
      open = occ;
    }
    const bool a0 = n0 < n1 && n0 < n2;
    const bool a1 = !a0 && n1 < n2;
    const float sn = a0 ? n0 : (a1 ? n1 : n2);
    if (!(sn < s_hi)) break;
    const int left = a0 ? l0 : (a1 ? l1 : l2);
    if (left == 0) break;  // the next crossing leaves the grid
    s = sn;
    c += a0 ? f0 : (a1 ? f1 : f2);
    if (a0) { n0 += e0; --l0; }
    else if (a1) { n1 += e1; --l1; }
    else { n2 += e2; --l2; }
  }
  if (open) emit(s_open, s_hi);
  for (int k = n; k < GF_MAX_IVL; ++k) out[k] = 0x0000FFFFu;  // empty (lo > hi)
}

// -------------------------------------------------------------------------
// ray setup: render.py:139-148 generate_rays (if camera), 368-369 f64 upcast,
// 486-500 slab test / seg / t0 in float32, and the ray's jitter stream
// position.
// -------------------------------------------------------------------------
__global__ void k_ray_init(MarchParams P, RayState R) {
  gf_pdl_wait();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n_rays) return;
  const int64_t g = global_ray(P, i);  // ray index within the render_rays call
  float o32[3], d32[3];
  double o64[3], d64[3];
  if (P.use_cam) {
    const gf_camera_t& c = P.cam;
    int64_t px = g % c.width, py = g / c.width;
    double u = __ddiv_rn(__dsub_rn(__dadd_rn((double)px, 0.5), c.cx), c.fx);
    double v = __ddiv_rn(__dsub_rn(__dadd_rn((double)py, 0.5), c.cy), c.fy);
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
      d[a] = __dadd_rn(__dadd_rn(__dmul_rn(u, c.c2w[4 * a + 0]), __dmul_rn(v, c.c2w[4 * a + 1])), c.c2w[4 * a + 2]);
    double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      d32[a] = __double2float_rn(__ddiv_rn(d[a], nn));
      o32[a] = __double2float_rn(c.c2w[4 * a + 3]);
    }
  } else if (P.rays_f64) {  // render.py:368: the slab test on the caller's float64 rays
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      o64[a] = reinterpret_cast<const double*>(P.origins)[3 * i + a];
      d64[a] = reinterpret_cast<const double*>(P.dirs)[3 * i + a];
      o32[a] = __double2float_rn(o64[a]);  // render.py:304-305: samples use the float32 roundings
      d32[a] = __double2float_rn(d64[a]);
    }
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      o32[a] = P.origins[3 * i + a];
      d32[a] = P.dirs[3 * i + a];
    }
  }
  if (!P.rays_f64 || P.use_cam) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      o64[a] = (double)o32[a];
      d64[a] = (double)d32[a];
    }
  }
  // slab test in f64 (render.py:151-171)
  double lo_max = -INFINITY, hi_min = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double o = o64[a], d = d64[a];
    double lo, hi;
    if (d == 0.0) {
      bool inside = (o >= P.grid.b_min[a]) && (o <= P.grid.b_max[a]);
      lo = inside ? -INFINITY : INFINITY;
      hi = inside ? INFINITY : -INFINITY;
    } else {
      double ta = __ddiv_rn(__dsub_rn(P.grid.b_min[a], o), d);
      double tb = __ddiv_rn(__dsub_rn(P.grid.b_max[a], o), d);
      lo = fmin(ta, tb);
      hi = fmax(ta, tb);
    }
    lo_max = fmax(lo_max, lo);
    hi_min = fmin(hi_min, hi);
  }
  double t0 = fmax(lo_max, 0.0), t1 = hi_min;
  bool hit = t1 > t0;
  float seg = hit ? __double2float_rn(__ddiv_rn(__dsub_rn(t1, t0), (double)P.k)) : 0.0f;
  R.org[i] = make_float4(o32[0], o32[1], o32[2], __double2float_rn(t0));
  R.dir[i] = make_float4(d32[0], d32[1], d32[2], seg);
  R.acc[i] = make_float4(0.f, 0.f, 0.f, 1.f);
  R.run[i] = 0;
  uint32_t fw = hit ? (uint32_t)(GF_RAY_ALIVE | GF_RAY_HIT) : 0u;
  if (R.denc && hit) {  // gamma(d) once per ray for every sample's direction layer (render.py:326)
    uint4 de[4];
    encode_direction_h(d32, de);
#pragma unroll
    for (int q = 0; q < 4; ++q) R.denc[4 * i + q] = de[q];
  }
  if (P.coarse_bits && hit) {
    const float ex = __double2float_rn(__dadd_rn((double)o32[0], __dmul_rn(t0, (double)d32[0])));
    const float ey = __double2float_rn(__dadd_rn((double)o32[1], __dmul_rn(t0, (double)d32[1])));
    const float ez = __double2float_rn(__dadd_rn((double)o32[2], __dmul_rn(t0, (double)d32[2])));
    const float smax = (float)(t1 - t0);
    // clip the walk to the set cells' bounding box, enlarged by one coarse
    // cell on every side (float32 slab test; a miss leaves no candidate)
    float s_lo = 0.f, s_hi = smax;
    if (P.occ_bbox) {
      const uint32_t* bb = P.occ_bbox;
      const float e[3] = {ex, ey, ez};
      if (bb[0] > bb[3]) s_hi = -1.f;  // no set coarse cell
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const float cs = 1.f / P.coarse.inv_cell_f[a];
        const float lo_w = fmaf((float)bb[a] - 1.f, cs, P.coarse.b_min_f[a]);
        const float hi_w = fmaf((float)bb[3 + a] + 2.f, cs, P.coarse.b_min_f[a]);
        if (d32[a] != 0.f) {
          const float ta = (lo_w - e[a]) / d32[a], tb = (hi_w - e[a]) / d32[a];
          s_lo = fmaxf(s_lo, fminf(ta, tb));
          s_hi = fminf(s_hi, fmaxf(ta, tb));
        } else if (e[a] < lo_w || e[a] > hi_w) {
          s_hi = -1.f;
        }
      }
    }
    if (s_lo < s_hi) {
      coarse_intervals(P, R.ivl + i * GF_MAX_IVL, ex, ey, ez, d32, smax, seg, s_lo, s_hi);
    } else {
#pragma unroll
      for (int k = 0; k < GF_MAX_IVL; ++k) R.ivl[i * GF_MAX_IVL + k] = 0x0000FFFFu;  // no candidate slot
    }
    if (P.n_rounds <= 24) {  // rounds holding at least one candidate slot
      const uint4* iv = reinterpret_cast<const uint4*>(R.ivl + i * GF_MAX_IVL);
      const uint4 q0 = iv[0], q1 = iv[1];
      const uint32_t v[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      uint32_t rm = 0;
#pragma unroll
      for (int k = 0; k < GF_MAX_IVL; ++k) {
        const int lo = (int)(v[k] & 0xFFFFu), hi = (int)(v[k] >> 16);
        if (lo <= hi) {
          const int r0 = lo / P.chunk, r1 = hi / P.chunk;
          rm |= (r1 - r0 >= 31 ? 0xFFFFFFFFu : ((2u << (r1 - r0)) - 1u)) << r0;
        }
      }
      fw |= (rm & 0xFFFFFFu) << 8;
    } else {
      fw |= GF_RAY_ALLROUNDS;
    }
  } else if (hit) {
    fw |= GF_RAY_ALLROUNDS;
  }
  R.flags[i] = fw;
  if (P.stratified) {
    const int64_t b = seed_slot(P, g);
    const int r = (int)(g % GF_RAY_BLOCK);  // the ray's row in its block: slot 0 is float32 draw r*k
    R.rng[i] = P.start[2 * r] * P.block_seeds[2 * b] + P.start[2 * r + 1] * P.block_seeds[2 * b + 1];
  }
  if (i == 0) atomicAdd((unsigned long long*)&P.stats[GF_STAT_N_RAYS], (unsigned long long)P.n_rays);
}

// -------------------------------------------------------------------------
// coarse occupancy mip: OR over factor^3 fine cells, then dilation by
// `radius` coarse cells (Chebyshev), stored as bits.
// -------------------------------------------------------------------------
__global__ void k_coarse_reduce(const uint8_t* __restrict__ occ_bits, int3 ores, int f, int3 cres, uint8_t* coarse) {
  gf_pdl_wait();
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)cres.x * cres.y * cres.z;
  if (c >= n) return;
  const int cx = (int)(c % cres.x), cy = (int)((c / cres.x) % cres.y), cz = (int)(c / ((int64_t)cres.x * cres.y));
  uint8_t any = 0;
  for (int z = cz * f; z < cz * f + f && !any; ++z)
    for (int y = cy * f; y < cy * f + f && !any; ++y)
      for (int x = cx * f; x < cx * f + f; ++x) {
        const int64_t fi = x + (int64_t)ores.x * (y + (int64_t)ores.y * z);
        if ((occ_bits[fi >> 3] >> (fi & 7)) & 1) { any = 1; break; }
      }
  coarse[c] = any;
}

__global__ void k_coarse_dilate(const uint8_t* __restrict__ coarse, int3 cres, int r, uint32_t* bits) {
  gf_pdl_wait();
  int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 32-bit word per thread
  const int64_t n = (int64_t)cres.x * cres.y * cres.z;
  if (w * 32 >= n) return;
  uint32_t word = 0;
  for (int b = 0; b < 32; ++b) {
    const int64_t c = w * 32 + b;
    if (c >= n) break;
    const int cx = (int)(c % cres.x), cy = (int)((c / cres.x) % cres.y), cz = (int)(c / ((int64_t)cres.x * cres.y));
    bool any = false;
    for (int z = max(cz - r, 0); z <= min(cz + r, cres.z - 1) && !any; ++z)
      for (int y = max(cy - r, 0); y <= min(cy + r, cres.y - 1) && !any; ++y)
        for (int x = max(cx - r, 0); x <= min(cx + r, cres.x - 1); ++x)
          if (coarse[x + (int64_t)cres.x * (y + (int64_t)cres.y * z)]) { any = true; break; }
    if (any) word |= 1u << b;
  }
  bits[w] = word;
}

// Word-parallel variants (fine rows 32-bit aligned: occ res.x % (32*factor) == 0).
// One thread = 32 coarse cells along x.
__global__ void k_coarse_reduce_w(const uint32_t* __restrict__ fine, int3 ores, int f, int3 cres, uint32_t* out,
                                  uint64_t* brick, uint32_t* bbox) {
  gf_pdl_wait();
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (bbox && w < 6) bbox[w] = w < 3 ? 0xFFFFFFFFu : 0u;  // reduced by the last dilation pass
  const int wpr = cres.x / 32;
  if (w >= (int64_t)wpr * cres.y * cres.z) return;
  const int wx = (int)(w % wpr), cy = (int)((w / wpr) % cres.y), cz = (int)(w / ((int64_t)wpr * cres.y));
  if (brick && f == 4) {
    // this word's 32 coarse cells as 4^3 bricks (bit dx + 4 dy + 16 dz) and
    // their OR (the coarse bit): 16 fine rows of 4 words each
    uint64_t br[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) br[b] = 0;
#pragma unroll
    for (int dz = 0; dz < 4; ++dz)
#pragma unroll
      for (int dy = 0; dy < 4; ++dy) {
        const int64_t row = ((int64_t)ores.x * (4 * cy + dy + (int64_t)ores.y * (4 * cz + dz))) / 32 + (int64_t)wx * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t v = __ldg(fine + row + q);
#pragma unroll
          for (int bb = 0; bb < 8; ++bb) br[8 * q + bb] |= (uint64_t)((v >> (4 * bb)) & 0xFu) << (4 * dy + 16 * dz);
        }
      }
    uint32_t res = 0;
    uint64_t* dst = brick + ((int64_t)cz * cres.y + cy) * cres.x + 32 * wx;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      dst[b] = br[b];
      res |= (br[b] != 0 ? 1u : 0u) << b;
    }
    out[w] = res;
    return;
  }
  uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int fz = cz * f; fz < cz * f + f; ++fz)
    for (int fy = cy * f; fy < cy * f + f; ++fy) {
      const int64_t row = ((int64_t)ores.x * (fy + (int64_t)ores.y * fz)) / 32 + (int64_t)wx * f;
      for (int q = 0; q < f; ++q) acc[q] |= __ldg(fine + row + q);
    }
  const uint32_t lowf = (1u << f) - 1u;
  uint32_t res = 0;
  for (int b = 0; b < 32; ++b) {
    const int bit = b * f;
    if ((acc[bit >> 5] >> (bit & 31)) & lowf) res |= 1u << b;
  }
  out[w] = res;
}

__global__ void k_dilate_x(const uint32_t* __restrict__ in, uint32_t* out, int3 cres, int r) {
  gf_pdl_wait();
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int wpr = cres.x / 32;
  if (w >= (int64_t)wpr * cres.y * cres.z) return;
  const int wx = (int)(w % wpr);
  const uint32_t v = in[w], prev = wx > 0 ? in[w - 1] : 0u, next = wx + 1 < wpr ? in[w + 1] : 0u;
  uint32_t res = v;
  for (int s = 1; s <= r; ++s) res |= (v << s) | (v >> s) | (prev >> (32 - s)) | (next << (32 - s));
  out[w] = res;
}

// axis 1: y (stride = words per row), axis 2: z (stride = words per plane)
__global__ void k_dilate_yz(const uint32_t* __restrict__ in, uint32_t* out, int3 cres, int r, int axis,
                            uint32_t* bbox) {
  gf_pdl_wait();
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int wpr = cres.x / 32;
  const bool valid = w < (int64_t)wpr * cres.y * cres.z;
  uint32_t res = 0;
  if (valid) {
    const int64_t stride = axis == 1 ? wpr : (int64_t)wpr * cres.y;
    const int n = axis == 1 ? cres.y : cres.z;
    const int c = axis == 1 ? (int)((w / wpr) % cres.y) : (int)(w / ((int64_t)wpr * cres.y));
    for (int o = max(c - r, 0); o <= min(c + r, n - 1); ++o) res |= in[w + (int64_t)(o - c) * stride];
    out[w] = res;
  }
  if (bbox) {  // the final pass: bounding box of the set cells (warp-reduced, then 6 atomics per warp)
    uint32_t lo[3] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu}, hi[3] = {0u, 0u, 0u};
    if (res) {
      const uint32_t wx = (uint32_t)(w % wpr), y = (uint32_t)((w / wpr) % cres.y),
                     z = (uint32_t)(w / ((int64_t)wpr * cres.y));
      lo[0] = 32u * wx + (uint32_t)(__ffs(res) - 1);
      hi[0] = 32u * wx + 31u - (uint32_t)__clz(res);
      lo[1] = hi[1] = y;
      lo[2] = hi[2] = z;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const uint32_t l = __reduce_min_sync(0xffffffffu, lo[a]), h = __reduce_max_sync(0xffffffffu, hi[a]);
      if (gf_lane() == 0 && l <= h) {
        atomicMin(bbox + a, l);
        atomicMax(bbox + 3 + a, h);
      }
    }
  }
}

// -------------------------------------------------------------------------
// K2 placement (batched.py:60-85 group_by_network, as the MLP consumes it):
// every record already carries its rank inside its cell (from the marcher's
// histogram atomics), so its sorted slot is offsets[cell] + rank with no
// atomics here; the record itself (with its staging index in .w) moves to
// its sorted slot, so the MLP streams its rows with no gather.  SMEM: each CTA scans the per-cell counts into shared memory
// itself (no separate scan launch); block 0 publishes offsets / n_tiles and
// every thread writes part of the tile list.  !SMEM (very large grids):
// offsets and tiles come from k_scan_cells.
// -------------------------------------------------------------------------
template <bool SMEM, int GR>
__global__ void __launch_bounds__(512) k_place(GfGrid grid, RoundBufs RB, const uint32_t* __restrict__ run,
                                               BucketBufs Bk, int64_t n_cells, int stride, int half, int round) {
  extern __shared__ uint32_t s_scan[];  // [n_cells+1] row offsets, [n_cells+1] tile offsets
  gf_pdl_wait();     // the marcher's histogram and records
  const uint32_t* counts = RB.counts + (size_t)(round & 1) * (size_t)n_cells;
  const uint32_t* off = Bk.offsets;
  const int tid = threadIdx.x;
  const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + tid, gthreads = (uint64_t)gridDim.x * blockDim.x;
  if (SMEM) {
    __shared__ uint32_t wsum[2][16];
    uint32_t* s_off = s_scan;
    uint32_t* s_toff = s_scan + n_cells + 1;
    const int per = (int)((n_cells + 511) / 512);  // <= 16 (n_cells <= 8192 on this path)
    const int64_t c0 = (int64_t)tid * per;
    uint32_t a = 0, b = 0, cv[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {  // all loads in flight at once, kept for the second pass
      const int64_t c = c0 + q;
      cv[q] = (q < per && c < n_cells) ? counts[c] : 0u;
    }
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      a += cv[q];
      b += (cv[q] + GF_TILE_ROWS - 1) / GF_TILE_ROWS;
    }
    // block exclusive scan of (a, b)
    const int lane = tid & 31, wid = tid >> 5;
    uint32_t xa = a, xb = b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ya = __shfl_up_sync(0xffffffffu, xa, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
      if (lane >= o) { xa += ya; xb += yb; }
    }
    if (lane == 31) { wsum[0][wid] = xa; wsum[1][wid] = xb; }
    __syncthreads();
    if (wid == 0) {
      uint32_t ta = lane < 16 ? wsum[0][lane] : 0, tb = lane < 16 ? wsum[1][lane] : 0;
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        const uint32_t ya = __shfl_up_sync(0xffffffffu, ta, o), yb = __shfl_up_sync(0xffffffffu, tb, o);
        if (lane >= o) { ta += ya; tb += yb; }
      }
      if (lane < 16) { wsum[0][lane] = ta; wsum[1][lane] = tb; }
    }
    __syncthreads();
    uint32_t ea = (wid ? wsum[0][wid - 1] : 0) + xa - a, eb = (wid ? wsum[1][wid - 1] : 0) + xb - b;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int64_t c = c0 + q;
      if (q < per && c < n_cells) {
        const uint32_t v = cv[q];
        s_off[c] = ea;
        s_toff[c] = eb;
        ea += v;
        eb += (v + GF_TILE_ROWS - 1) / GF_TILE_ROWS;
      }
    }
    if (tid == 511) {
      s_off[n_cells] = ea;
      s_toff[n_cells] = eb;
    }
    __syncthreads();
    const uint32_t n_tiles = s_toff[n_cells];
    if (blockIdx.x == 0) {
      for (int64_t c = tid; c <= n_cells; c += 512) Bk.offsets[c] = s_off[c];
      if (tid == 0) {
        *Bk.n_tiles = n_tiles;
        RB.emit_count[(round + 1) & 1] = 0;
      }
    }
    uint32_t* other = RB.counts + (size_t)((round + 1) & 1) * (size_t)n_cells;  // next round's histogram
    for (uint64_t c = gtid; c < (uint64_t)n_cells; c += gthreads) other[c] = 0;
    // one thread per tile (a large cell's tiles would serialise one thread):
    // the tile's cell is the last c with s_toff[c] <= u (binary search)
    for (uint64_t u = gtid; u < (uint64_t)n_tiles; u += gthreads) {
      uint32_t lo = 0, hi = (uint32_t)n_cells;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_toff[mid] <= (uint32_t)u) lo = mid;
        else hi = mid;
      }
      const uint32_t n_seg = s_off[lo + 1] - s_off[lo], r0 = ((uint32_t)u - s_toff[lo]) * GF_TILE_ROWS;
      Bk.tiles[u] = gf_make_tile(lo, s_off[lo] + r0, min(n_seg - r0, (uint32_t)GF_TILE_ROWS));
    }
    off = s_off;
  } else if (gtid == 0) {
    RB.emit_count[(round + 1) & 1] = 0;
  }
  // warp-cooperative record walk: a warp takes 32 listed rays, prefix-sums
  // their runs and moves their records 32 at a time (one per lane), so every
  // lane has an independent load -> cell -> store chain in flight
  const uint32_t n_list = RB.emit_count[round & 1];
  const unsigned lane = gf_lane();
  const uint64_t pol_first = gf_pol_first(), pol_last = gf_pol_last();
  const uint64_t warp_g = gtid >> 5, n_warps = gthreads >> 5;
  for (uint64_t k0 = warp_g * 32; k0 < n_list; k0 += n_warps * 32) {
    const uint64_t k = k0 + lane;
    const uint32_t i = k < n_list ? RB.emit_list[k] : 0u;
    const uint32_t rv = k < n_list ? run[i] : 0u;
    // grouped rounds: one count byte per round of the group, records of round
    // p at staging offset p * half
    // GR rounds per group (one count byte each); cum = prefix counts after
    // rounds 0, 1, 2 of the group, one byte each
    const uint32_t c1 = rv & 0xFFu, c2 = c1 + ((rv >> 8) & 0xFFu), c3 = c2 + ((rv >> 16) & 0xFFu);
    const uint32_t nr = GR == 1 ? rv : (GR == 2 ? c2 : (GR == 3 ? c3 : c3 + (rv >> 24)));
    const uint32_t cum = GR == 2 ? c1 : (c1 | (c2 << 8) | (c3 << 16));
    uint32_t incl = nr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)lane >= o) incl += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31), excl = incl - nr;
    // U records per lane per pass: U independent loads in flight per lane
    constexpr int U = 4;
    for (uint32_t b0 = 0; b0 < total; b0 += 32 * U) {
      float4 r[U];
      uint32_t src[U];
      bool ok[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t q = b0 + 32 * u + lane;
        int own = 0;  // smallest lane whose inclusive count exceeds q
#pragma unroll
        for (int st = 16; st; st >>= 1) {
          const uint32_t v = __shfl_sync(0xffffffffu, incl, own + st - 1);
          if (v <= q) own += st;
        }
        const uint32_t j = q - __shfl_sync(0xffffffffu, excl, own);
        const uint32_t i_o = __shfl_sync(0xffffffffu, i, own);
        ok[u] = q < total;
        // staging index (< 2^32, checked on the host): j-th record of the ray
        // over its group's rounds, round p's records `p * half` further
        uint32_t off = j;
        if (GR == 2) {
          const uint32_t a1 = __shfl_sync(0xffffffffu, cum, own);
          off = j < a1 ? j : (uint32_t)half + j - a1;
        } else if (GR >= 3) {
          const uint32_t cu = __shfl_sync(0xffffffffu, cum, own);
          const uint32_t a1 = cu & 0xFFu, a2 = (cu >> 8) & 0xFFu, a3 = cu >> 16;
          off = j < a1 ? j
                       : (j < a2 ? (uint32_t)half + j - a1 : (j < a3 ? 2u * half + j - a2 : 3u * half + j - a3));
        }
        src[u] = i_o * (uint32_t)stride + off;
        if (ok[u]) r[u] = gf_ld_hint(RB.rec + src[u], pol_first);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (ok[u]) {
          const uint32_t cell = gf_flat_cell(grid, r[u].x, r[u].y, r[u].z);
          gf_st_hint(Bk.srec + off[cell] + __float_as_uint(r[u].w),
                     make_float4(r[u].x, r[u].y, r[u].z, __uint_as_float(src[u])), pol_last);
        }
      }
    }
  }
}

template <int GR>
static int launch_place_g(const GfGrid& grid, const RoundBufs& RB, const uint32_t* run, const BucketBufs& Bk,
                          int64_t n_cells, int stride, int half, int round, int64_t max_rows, cudaStream_t st) {
  const size_t smem = (size_t)2 * (n_cells + 1) * 4;
  if (n_cells <= 8192) {
    static thread_local bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_place<true, GR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 8193 * 4);
      attr = true;
    }
    gf_launch_pdl(k_place<true, GR>, dim3(num_sms() * 2), dim3(512), smem, st, grid, RB, run, Bk, n_cells, stride, half,
                  round);
    return 1;
  }
  BucketBufs b = Bk;
  b.counts = RB.counts + (size_t)(round & 1) * (size_t)n_cells;
  const int n = launch_scan_cells(b, n_cells, st, max_rows);  // offsets + tiles; clears this round's counts
  gf_launch_pdl(k_place<false, GR>, dim3(num_sms() * 2), dim3(512), 0, st, grid, RB, run, Bk, n_cells, stride, half,
                round);
  return n + 1;
}

int launch_place(const GfGrid& grid, const RoundBufs& RB, const uint32_t* run, const BucketBufs& Bk, int64_t n_cells,
                 int stride, int half, int round, int64_t max_rows, cudaStream_t st) {
  const int group = half > 0 ? stride / half : 1;  // rounds per group (1 to 4)
  if (group == 4) return launch_place_g<4>(grid, RB, run, Bk, n_cells, stride, half, round, max_rows, st);
  if (group == 3) return launch_place_g<3>(grid, RB, run, Bk, n_cells, stride, half, round, max_rows, st);
  if (group == 2) return launch_place_g<2>(grid, RB, run, Bk, n_cells, stride, half, round, max_rows, st);
  return launch_place_g<1>(grid, RB, run, Bk, n_cells, stride, 0, round, max_rows, st);
}

__device__ __forceinline__ u128 ldg_u128(const u128* p) {
  const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
  return ((u128)v.y << 64) | v.x;
}

// warp-aggregated histogram increment: lanes with `pred` add 1 to hist[key]
// and receive their rank among all samples of that key this round (the
// atomic's return value), i.e. their final row inside the cell's segment.
__device__ __forceinline__ uint32_t hist_rank(uint32_t* hist, bool pred, uint32_t key) {
  unsigned act = __ballot_sync(0xffffffffu, pred);
  uint32_t rank = 0;
  if (pred) {
    unsigned peers = __match_any_sync(act, key);
    const int leader = __ffs(peers) - 1;
    uint32_t b = 0;
    if ((int)gf_lane() == leader) b = atomicAdd(&hist[key], (uint32_t)__popc(peers));
    rank = __shfl_sync(peers, b, leader) + __popc(peers & ((1u << gf_lane()) - 1u));
  }
  return rank;
}

__device__ __forceinline__ void warp_add_u64(int64_t* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (gf_lane() == 0 && v) atomicAdd((unsigned long long*)dst, v);
}

// RenderStats counters of one marcher thread, flushed once per warp per pass
// into a spread slot (one global counter per stat serialised ~10^5 atomics
// per pass); k_stats_fold sums the slots into the caller's stats at the end
struct MarchStats {
  unsigned long long v[GF_STAT_COUNT] = {0ull, 0ull, 0ull, 0ull};
};

__device__ __forceinline__ void flush_stats(const MarchParams& P, MarchStats& S) {  // warp-uniform
  const uint32_t slot = ((blockIdx.x * (blockDim.x >> 5)) + (threadIdx.x >> 5)) & (GF_STAT_SLOTS - 1);
  if (P.k < (1 << 24)) {
    // a thread's counts in one pass are below 2k: the warp sum fits 32 bits,
    // one REDUX per counter
#pragma unroll
    for (int c = 0; c < GF_STAT_COUNT; ++c) {
      const unsigned v = __reduce_add_sync(0xffffffffu, (unsigned)S.v[c]);
      if (gf_lane() == 0 && v) atomicAdd(P.stats_part + slot * GF_STAT_COUNT + c, (unsigned long long)v);
    }
    return;
  }
#pragma unroll
  for (int c = 0; c < GF_STAT_COUNT; ++c) {
    unsigned long long v = S.v[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (gf_lane() == 0 && v) atomicAdd(P.stats_part + slot * GF_STAT_COUNT + c, v);
  }
}

__global__ void k_stats_fold(const unsigned long long* __restrict__ part, int64_t* stats) {
  gf_pdl_wait();
  __shared__ unsigned long long acc[GF_STAT_COUNT];
  if (threadIdx.x < GF_STAT_COUNT) acc[threadIdx.x] = 0ull;
  __syncthreads();
  unsigned long long v[GF_STAT_COUNT] = {0ull, 0ull, 0ull, 0ull};
  for (int s = threadIdx.x; s < GF_STAT_SLOTS; s += blockDim.x)
#pragma unroll
    for (int c = 0; c < GF_STAT_COUNT; ++c) v[c] += part[s * GF_STAT_COUNT + c];
#pragma unroll
  for (int c = 0; c < GF_STAT_COUNT; ++c) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&acc[c], v[c]);
  }
  __syncthreads();
  if (threadIdx.x < GF_STAT_COUNT && acc[threadIdx.x])
    atomicAdd((unsigned long long*)&stats[threadIdx.x], acc[threadIdx.x]);
}

void launch_stats_fold(const unsigned long long* part, int64_t* stats, cudaStream_t st) {
  gf_launch_pdl(k_stats_fold, dim3(1), dim3(256), 0, st, part, stats);
}

// -------------------------------------------------------------------------
// march pass r: composite round r-1 (+ERT), then place / skip / emit round r.
// At r == n_rounds: composite the last round and write the final colours.
// -------------------------------------------------------------------------
// one round's sampling for the marcher's ray i (render.py:311-330): placement,
// ESS, histogram ranks, staging records, counters; `fw` is the ray's flag word
// FAST: the benchmarked configuration fixed at compile time -- stratified,
// float32-exact clip, network cell from the occupancy cell, no trace, no fine
// pre-test -- so the candidate loop carries no flag tests or their constants.
template <bool FAST>
__device__ __forceinline__ void march_sample(const MarchParams& P, const RayState& R, const RoundBufs& B, int64_t i,
                                             uint32_t& fw, int round, int phase, MarchStats& ST) {
  const bool stratified = FAST || P.stratified;
  const bool from_occ = FAST || P.net_from_occ;
  const bool tracing = !FAST && P.trace;
  const uint32_t* fine_bits = FAST ? nullptr : P.fine_bits;
  // ---- sample round r (render.py:311-330)
  const int s0 = round * P.chunk;
  const int m = min(P.chunk, P.k - s0);
  const bool alive = (fw & GF_RAY_ALIVE) != 0;
  // rays whose coarse intervals have no slot in this round only add to ess_skipped
  const bool active = alive && ((fw & GF_RAY_ALLROUNDS) || (round < 24 && ((fw >> (8 + round)) & 1u)));
  // later round of a group: a ray whose earlier rounds in the group queried
  // samples may still die at their ERT checks, so its counters wait in R.pend
  const bool earlier = phase > 0 && (fw & gf_had_below(phase));
  const bool defer = alive && earlier;
  const int par = ((round - phase) / P.group) & 1;             // histogram / emit-list parity (group-uniform)
  const uint32_t half = (uint32_t)phase * (uint32_t)P.chunk;   // staging offset of the group's round
  ST.v[GF_STAT_ESS_SKIPPED] += (alive && !active && !defer) ? (unsigned long long)m : 0ull;
  if (defer && !active) R.pend[4 * (uint64_t)i + phase] = (uint32_t)m << 16;
  if (!__any_sync(0xffffffffu, active)) return;
  float4 o = active ? R.org[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 d = active ? R.dir[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  u128 S = 0, inc = 0;
  uint64_t outw = 0;
  uint64_t draw = 0;
  uint32_t blk = 0;
  if (stratified && active) {
    // state of the word holding this round's first draw: a tabulated jump
    // from the ray's slot-0 state (R.rng stays read-only)
    const int64_t g = global_ray(P, i);
    blk = (uint32_t)seed_slot(P, g);
    inc = P.block_seeds[2 * blk + 1];
    const uint64_t draw0 = (uint64_t)(g % GF_RAY_BLOCK) * (uint64_t)P.k;
    const int jr = 2 * (2 * round + (int)(draw0 & 1));
    S = ldg_u128(&P.round_jump[jr]) * R.rng[i] + ldg_u128(&P.round_jump[jr + 1]) * inc;
    outw = gf_pcg_output(S);
    draw = draw0 + (uint64_t)s0;
  }
  const double t0 = (double)o.w, sg64 = (double)d.w;
  const double ox = (double)o.x, oy = (double)o.y, oz = (double)o.z;
  const double dx = (double)d.x, dy = (double)d.y, dz = (double)d.z;
  const uint64_t base = (uint64_t)i * (uint64_t)P.stride;
  // candidate slots of this round from the ray's coarse-DDA ranges
  uint32_t cmask = m >= 32 ? 0xFFFFFFFFu : ((1u << m) - 1u);
  if (P.coarse_bits && active) {
    const uint4* iv = reinterpret_cast<const uint4*>(R.ivl + i * GF_MAX_IVL);
    const uint4 q0 = iv[0], q1 = iv[1];
    const uint32_t v[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
    uint32_t msk = 0;
#pragma unroll
    for (int k = 0; k < GF_MAX_IVL; ++k) {
      const int lo = max((int)(v[k] & 0xFFFFu), s0), hi = min((int)(v[k] >> 16), s0 + m - 1);
      if (lo <= hi) {
        const int nb = hi - lo + 1;
        msk |= (nb >= 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u)) << (lo - s0);
      }
    }
    cmask &= msk;
  }
  const bool fast_clip = FAST || P.grid.fast != 0;
  uint32_t* counts_r = B.counts + (size_t)par * (size_t)P.n_cells;  // this round's histogram
  uint32_t kept = 0;
  if (m <= 32) {
    // ---- warp-cooperative path: the warp's candidate (ray, slot) pairs are
    // compacted into a shared-memory list in (lane, slot) order and processed
    // 32 at a time, one per lane, so the exact float64 placement never runs
    // on idle lanes.  Each candidate lane reads its ray's parameters from
    // shared memory (broadcast when several lanes share a ray).
    struct RayPar {
      double t0, seg, ox, oy, oz, dx, dy, dz;  // the float32 ray, widened once per round
      uint4 S;          // PCG64 state at draw d0 (rounded down to a word)
      uint64_t rec;     // record index of the ray's first sample of this round
      const u128* ci;   // the ray's block row of (sum_{k<d} A^k) * inc
      uint32_t i, d0;   // call-local ray index, float32 draw index of slot s0
      uint32_t carry;   // kept samples so far this round
      uint32_t span;    // the ray's candidates in the list: [span & 0xFFFF, span >> 16)
    };
    __shared__ RayPar s_ray[4][32];
    __shared__ uint16_t s_list[4][32 * 32];
    const int wib = threadIdx.x >> 5;
    const unsigned lane = gf_lane();
    if (!active) cmask = 0;
    const uint32_t cnt = __popc(cmask);
    if (P.count_candidates) ST.v[GF_STAT_N_RAYS] += cnt;
    uint32_t incl = cnt;
#pragma unroll
    for (int o2 = 1; o2 < 32; o2 <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o2);
      if ((int)lane >= o2) incl += v;
    }
    const uint32_t total_c = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t d0 = (uint32_t)draw;  // float32 draw index of slot s0 in the ray's block stream
    {
      RayPar& rp = s_ray[wib][lane];
      rp.t0 = t0;
      rp.seg = sg64;
      rp.ox = ox;
      rp.oy = oy;
      rp.oz = oz;
      rp.dx = dx;
      rp.dy = dy;
      rp.dz = dz;
      rp.S = make_uint4((uint32_t)S, (uint32_t)(S >> 32), (uint32_t)(S >> 64), (uint32_t)(S >> 96));
      rp.rec = base + half;
      rp.ci = P.block_ci + (size_t)blk * GF_CI_N;
      rp.i = (uint32_t)i;
      rp.d0 = d0;
      rp.carry = 0;
      rp.span = (incl - cnt) | (incl << 16);
      uint32_t msk = cmask, pos = incl - cnt;  // candidate list in (lane, slot) order
      while (msk) {  // this lane's candidate slots, ascending
        const int j = __ffs(msk) - 1;
        s_list[wib][pos++] = (uint16_t)((lane << 5) | (uint32_t)j);
        msk &= msk - 1u;
      }
    }
    __syncwarp();
    uint32_t total = total_c;
    if (fine_bits) {
      // pre-test at the segment midpoint against the dilated fine bitmap:
      // the exact sample lies within seg/2 (+ float32 margin) of it, so a
      // clear bit proves an ESS skip; survivors are compacted in place
      // (writes never pass the batch being read)
      constexpr int FU = 4;  // batches in flight: FU bitmap loads per lane before the first ballot
      uint32_t kept_n = 0;
      for (uint32_t b0 = 0; b0 < total_c; b0 += 32 * FU) {
        uint32_t e[FU], word[FU], bit[FU];
#pragma unroll
        for (int u = 0; u < FU; ++u) {
          const uint32_t k = b0 + 32 * u + lane;
          e[u] = k < total_c ? (uint32_t)s_list[wib][k] : 0xFFFFFFFFu;
          word[u] = 0u;
          bit[u] = 0u;
          if (e[u] != 0xFFFFFFFFu) {
            const RayPar& rp = s_ray[wib][e[u] >> 5];
            const float tm = fmaf((float)(s0 + (int)(e[u] & 31u)) + 0.5f, (float)rp.seg, (float)rp.t0);
            const float px = fmaf(tm, (float)rp.dx, (float)rp.ox), py = fmaf(tm, (float)rp.dy, (float)rp.oy),
                        pz = fmaf(tm, (float)rp.dz, (float)rp.oz);
            const uint32_t f = (uint32_t)(gf_bin_axis_fast(P.occ, 0, px) +
                                          P.occ.res[0] * (gf_bin_axis_fast(P.occ, 1, py) +
                                                          P.occ.res[1] * gf_bin_axis_fast(P.occ, 2, pz)));
            word[u] = __ldg(fine_bits + (f >> 5));
            bit[u] = f & 31u;
          }
        }
        __syncwarp();  // every lane has read its FU entries before any is overwritten
#pragma unroll
        for (int u = 0; u < FU; ++u) {
          const bool pass = e[u] != 0xFFFFFFFFu && ((word[u] >> bit[u]) & 1u);
          const unsigned pm = __ballot_sync(0xffffffffu, pass);
          if (pass) s_list[wib][kept_n + __popc(pm & ((1u << lane) - 1u))] = (uint16_t)e[u];
          kept_n += __popc(pm);
        }
        __syncwarp();
      }
      total = kept_n;
    }
    // the record of the previous batch waiting for its cell rank
    bool pend_ok = false;
    uint32_t pend_raw = 0, pend_peers = 0;
    int pend_leader = (int)lane;
    uint64_t pend_addr = 0;
    float pend_x = 0.f, pend_y = 0.f, pend_z = 0.f;
    const uint64_t pol_last = gf_pol_last();
    auto resolve = [&]() {  // warp-uniform
      const uint32_t b = __shfl_sync(0xffffffffu, pend_raw, pend_leader);
      if (pend_ok) {
        const uint32_t crank = b + __popc(pend_peers & ((1u << lane) - 1u));
        gf_st_hint(B.rec + pend_addr, make_float4(pend_x, pend_y, pend_z, __uint_as_float(crank)), pol_last);
      }
    };
    for (uint32_t b0 = 0; b0 < total; b0 += 32) {
      const uint32_t k = b0 + lane;
      const bool has = k < total;
      // idle lanes of a partial batch redo the list's last candidate (valid
      // addresses, no divergent branches) and keep nothing
      const uint32_t e = (uint32_t)s_list[wib][has ? k : total - 1u];
      const int own = (int)(e >> 5);
      const int j = (int)(e & 31u);
      const RayPar& rp = s_ray[wib][own];
      const uint64_t rec = rp.rec;
      // slot + jitter: f64(slot) + (u >> 8) * 2^-24 is exact (< 2^52 in
      // units of 2^-24), so it is built as one integer and scaled
      uint64_t v = ((uint64_t)(uint32_t)(s0 + j) << 24) | (1ull << 23);  // unstratified: slot + 0.5
      if (stratified) {
        const uint32_t d0_o = rp.d0;
        const uint4 sv = rp.S;
        const u128 So = ((u128)(((uint64_t)sv.w << 32) | sv.z) << 64) | (((uint64_t)sv.y << 32) | sv.x);
        const uint32_t dd = d0_o + (uint32_t)j;
        const uint32_t delta = (dd >> 1) - (d0_o >> 1);
        // S_delta = A^delta S + (sum_{k<delta} A^k) inc; the second term is tabulated per block
        const u128 Sj = ldg_u128(&P.jump[2 * delta]) * So + ldg_u128(rp.ci + delta);
        const uint32_t u = gf_pcg_output_half(Sj, dd & 1);
        v = ((uint64_t)(uint32_t)(s0 + j) << 24) | (uint64_t)(u >> 8);
      }
      const double x = __dmul_rn(__dsub_rn(__hiloint2double(0x43300000 | (int)(v >> 32), (int)(uint32_t)v),
                                           4503599627370496.0),
                                 5.9604644775390625e-8);
      // t = f64(t0_32) + (f64(slot) + f64(jit)) * f64(seg_32); p = f32(f64(o32) + t*f64(d32))
      const double t = __dadd_rn(rp.t0, __dmul_rn(x, rp.seg));
      float px = __double2float_rn(__dadd_rn(rp.ox, __dmul_rn(t, rp.dx)));
      float py = __double2float_rn(__dadd_rn(rp.oy, __dmul_rn(t, rp.dy)));
      float pz = __double2float_rn(__dadd_rn(rp.oz, __dmul_rn(t, rp.dz)));
      if (fast_clip) {
        px = gf_clip_fast(px, P.grid.b_min_f[0], P.grid.b_max_f[0]);
        py = gf_clip_fast(py, P.grid.b_min_f[1], P.grid.b_max_f[1]);
        pz = gf_clip_fast(pz, P.grid.b_min_f[2], P.grid.b_max_f[2]);
      } else {
        px = gf_clip_component(px, P.grid.b_min[0], P.grid.b_max[0]);
        py = gf_clip_component(py, P.grid.b_min[1], P.grid.b_max[1]);
        pz = gf_clip_component(pz, P.grid.b_min[2], P.grid.b_max[2]);
      }
      bool keep;
      uint32_t cell;
      if (from_occ) {  // both grids fast, same box, occupancy cells nest 2^s per network cell
        const int ox = gf_bin_axis_clipped(P.occ, 0, px), oy = gf_bin_axis_clipped(P.occ, 1, py),
                  oz = gf_bin_axis_clipped(P.occ, 2, pz);
        if (FAST) {  // brick word of the sample's 4^3 block (k_coarse_reduce_w)
          const uint32_t bi = (uint32_t)((ox >> 2) + P.brick_cx * ((oy >> 2) + P.brick_cy * (oz >> 2)));
          const uint32_t bit = (uint32_t)((ox & 3) | ((oy & 3) << 2) | ((oz & 3) << 4));
          keep = has && ((__ldg(P.occ_brick + bi) >> bit) & 1ull);
        } else {
          const uint32_t f = (uint32_t)(ox + P.occ.res[0] * (oy + P.occ.res[1] * oz));
          keep = has && ((__ldg(P.occ_bits + (f >> 3)) >> (f & 7)) & 1);
        }
        cell = (uint32_t)((ox >> P.net_shift[0]) +
                          P.grid.res[0] * ((oy >> P.net_shift[1]) + P.grid.res[1] * (oz >> P.net_shift[2])));
      } else {
        keep = has;
        if (P.occ_bits) {
          const uint32_t f = gf_flat_cell(P.occ, px, py, pz);
          keep = keep && ((__ldg(P.occ_bits + (f >> 3)) >> (f & 7)) & 1);
        }
        cell = keep ? gf_flat_cell(P.grid, px, py, pz) : 0u;
      }
      // position of this sample in its ray's run: kept items of the same ray
      // earlier in this batch + kept items of earlier batches
      const unsigned kb = __ballot_sync(0xffffffffu, keep);
      // lanes of this lane's ray in the batch up to and including it, and
      // whether it is the ray's last lane here: a ray's candidates are
      // contiguous in the list, unless the fine pre-test compacted it
      unsigned run_le;
      bool run_last;
      if (fine_bits) {
        const unsigned same = __match_any_sync(0xffffffffu, has ? own : 32 + (int)lane);
        run_le = same & ((2u << lane) - 1u);
        run_last = (int)lane == 31 - __clz(same);
      } else {
        const uint32_t span = rp.span;
        const int lo = max((int)(span & 0xFFFFu) - (int)b0, 0);
        run_le = ((2u << lane) - 1u) & ~((1u << lo) - 1u);
        run_last = lane == 31u || k + 1u >= (span >> 16);
      }
      // issue this batch's warp-aggregated rank atomic now, consume it one
      // batch later: the previous batch's records are stored meanwhile
      uint32_t peers = 0, raw = 0;
      int leader = (int)lane;
      if (keep) {
        peers = __match_any_sync(kb, cell);
        leader = __ffs(peers) - 1;
        if ((int)lane == leader) raw = atomicAdd(&counts_r[cell], (uint32_t)__popc(peers));
      }
      resolve();
      pend_ok = keep;
      pend_raw = raw;
      pend_peers = peers;
      pend_leader = leader;
      if (keep) {
        const uint32_t pos = s_ray[wib][own].carry + __popc(kb & run_le & ((1u << lane) - 1u));
        pend_addr = rec + pos;
        pend_x = px;
        pend_y = py;
        pend_z = pz;
        if (tracing) {
          unsigned long long slotpos = atomicAdd((unsigned long long*)P.trace_count, 1ull);
          if ((int64_t)slotpos < P.trace_capacity)
            P.trace[slotpos] = gf_trace_rec_t{px, py, pz, (uint32_t)global_ray(P, (int64_t)rp.i), (uint32_t)(s0 + j), cell};
        }
      }
      __syncwarp();
      if (has && run_last) s_ray[wib][own].carry += __popc(kb & run_le);
      __syncwarp();
    }
    resolve();  // the last batch's records
    kept = s_ray[wib][lane].carry;
  } else {
  double jd = (double)s0;
  for (int j = 0; j < m; ++j, jd += 1.0) {
    double jit = 0.5;
    if (P.stratified && active) {
      const uint32_t u = (draw & 1) ? (uint32_t)(outw >> 32) : (uint32_t)outw;
      // (u >> 8) * 2^-24 exactly, built in f64 without an I2F conversion
      jit = __dmul_rn(__dsub_rn(__hiloint2double(0x43300000, (int)(u >> 8)), 4503599627370496.0),
                      5.9604644775390625e-8);
      ++draw;
      if (!(draw & 1)) {
        S = gf_pcg_step(S, inc);
        outw = gf_pcg_output(S);
      }
    }
    // coarse test: the sample lies within seg/2 (+margin) of the segment
    // midpoint; the mip is dilated by that radius, so a clear bit proves the
    // exact sample is in an empty fine cell (skipped, counted in ess_skipped)
    const bool cand = active && (j >= 32 || ((cmask >> j) & 1u));
    bool keep = false;
    uint32_t cell = 0;
    float px = 0.f, py = 0.f, pz = 0.f;
    if (__any_sync(0xffffffffu, cand) && cand) {
      // t = f64(t0_32) + (f64(slot) + f64(jit)) * f64(seg_32); p = f32(f64(o32) + t*f64(d32))
      const double t = __dadd_rn(t0, __dmul_rn(__dadd_rn(jd, jit), sg64));
      px = __double2float_rn(__dadd_rn(ox, __dmul_rn(t, dx)));
      py = __double2float_rn(__dadd_rn(oy, __dmul_rn(t, dy)));
      pz = __double2float_rn(__dadd_rn(oz, __dmul_rn(t, dz)));
      if (fast_clip) {
        px = gf_clip_fast(px, P.grid.b_min_f[0], P.grid.b_max_f[0]);
        py = gf_clip_fast(py, P.grid.b_min_f[1], P.grid.b_max_f[1]);
        pz = gf_clip_fast(pz, P.grid.b_min_f[2], P.grid.b_max_f[2]);
      } else {
        px = gf_clip_component(px, P.grid.b_min[0], P.grid.b_max[0]);
        py = gf_clip_component(py, P.grid.b_min[1], P.grid.b_max[1]);
        pz = gf_clip_component(pz, P.grid.b_min[2], P.grid.b_max[2]);
      }
      keep = true;
      if (P.occ_bits) {
        const uint32_t f = gf_flat_cell(P.occ, px, py, pz);
        keep = (__ldg(P.occ_bits + (f >> 3)) >> (f & 7)) & 1;
      }
      if (keep) cell = gf_flat_cell(P.grid, px, py, pz);
    }
    const uint32_t rank = hist_rank(counts_r, keep, cell);
    if (keep) {
      B.rec[base + kept] = make_float4(px, py, pz, __uint_as_float(rank));
      if (P.trace) {
        unsigned long long slotpos = atomicAdd((unsigned long long*)P.trace_count, 1ull);
        if ((int64_t)slotpos < P.trace_capacity)
          P.trace[slotpos] = gf_trace_rec_t{px, py, pz, (uint32_t)global_ray(P, i), (uint32_t)(s0 + j), cell};
      }
      ++kept;
    }
  }
  }  // sequential path (ert_chunk > 32)
  if (active && kept > 0) {
    // groups: one byte per round of the group (the first writer of a group
    // clears the others); single rounds: the whole word
    R.run[i] = P.group == 1 ? kept : ((earlier ? R.run[i] : 0u) | (kept << (8 * phase)));
    fw |= gf_had_bit(phase);
  }
  if (defer && active) R.pend[4 * (uint64_t)i + phase] = kept | ((uint32_t)(m - (int)kept) << 16);
  {  // compact list of rays with queried samples (once per group), for the scatter kernel
    const bool emit = active && kept > 0 && !earlier;
    const unsigned em = __ballot_sync(0xffffffffu, emit);
    if (em) {
      uint32_t b = 0;
      if (gf_lane() == 0) b = atomicAdd(&B.emit_count[par], (uint32_t)__popc(em));
      b = __shfl_sync(0xffffffffu, b, 0);
      if (emit) B.emit_list[b + __popc(em & ((1u << gf_lane()) - 1u))] = (uint32_t)i;
    }
  }
  ST.v[GF_STAT_TOTAL_QUERIES] += defer ? 0ull : (unsigned long long)kept;
  ST.v[GF_STAT_ESS_SKIPPED] += (active && !defer) ? (unsigned long long)(m - (int)kept) : 0ull;
}

// 7 CTAs/SM (<= 72 registers): measured faster than the unconstrained 85
// registers despite a few spilled bytes
#ifndef GF_MARCH_MINB
#define GF_MARCH_MINB 7
#endif
template <bool FAST>
__global__ void __launch_bounds__(128, GF_MARCH_MINB) k_march(MarchParams P, RayState R, RoundBufs B, int round, int phase) {
  gf_pdl_wait();     // the previous MLP / marcher pass
  const int64_t i = march_ray(P, (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  const bool in_range = i < P.n_rays;
  uint32_t fw = in_range ? R.flags[i] : 0u;  // flags | candidate-round mask << 8
  const uint32_t fw0 = fw;
  const bool final_pass = round >= P.n_rounds;
  if (!final_pass && !__any_sync(0xffffffffu, fw & GF_RAY_ALIVE)) return;

  // ---- composite the previous round (render.py:333-337), float32, no
  // contraction; only rays that queried samples then have anything to blend.
  // Grouped rounds (P.group = G > 1): rounds G*s .. G*s+G-1 are placed by G
  // marcher passes and evaluated by one K2 + MLP pass, then composited here
  // in order with the ERT check after each; a ray that dies inside the group
  // drops the later rounds' samples and their deferred counters, exactly as
  // if those rounds had never run.
  float4 acc = make_float4(0.f, 0.f, 0.f, 1.f);
  const uint32_t had_bits = (fw & GF_RAY_ALIVE) ? (fw & GF_RAY_HAD_ALL) : 0u;
  const bool had = phase == 0 && had_bits != 0;
  unsigned long long commit_q = 0, commit_s = 0;
  if (had) {
    acc = R.acc[i];
    const float seg = R.dir[i].w;
    const uint64_t base = (uint64_t)i * (uint64_t)P.stride;
    const uint32_t run = R.run[i];
    const uint64_t pol_first = gf_pol_first();
    auto blend = [&](uint64_t b0, uint32_t n) {
      float tr = 1.0f, sr = 0.f, sg = 0.f, sb = 0.f;
      for (uint32_t j = 0; j < n; ++j) {
        float4 q = gf_ld_hint(B.res + b0 + j, pol_first);
        float a = -expm1f(__fmul_rn(-q.w, seg));
        float w = __fmul_rn(tr, a);
        tr = __fmul_rn(tr, __fsub_rn(1.0f, a));
        sr = __fadd_rn(sr, __fmul_rn(w, q.x));
        sg = __fadd_rn(sg, __fmul_rn(w, q.y));
        sb = __fadd_rn(sb, __fmul_rn(w, q.z));
      }
      acc.x = __fadd_rn(acc.x, __fmul_rn(acc.w, sr));
      acc.y = __fadd_rn(acc.y, __fmul_rn(acc.w, sg));
      acc.z = __fadd_rn(acc.z, __fmul_rn(acc.w, sb));
      acc.w = __fmul_rn(acc.w, tr);
    };
    // one blend site (keeps the marcher's registers down).  Part p is round
    // round - G + p; the ERT check after it counts a termination if round
    // p + 1 exists (render.py:338-343).  Transmittance only moves in rounds
    // with samples, so other rays cannot cross epsilon.
    const int G = P.group;
    bool dead = false;
#pragma unroll 1
    for (int part = 0; part < G && !dead; ++part) {
      const int c = round - G + part;  // the composited round
      if (part > 0 && c < P.n_rounds && (had_bits & gf_had_below(part))) {
        // the round really ran for this ray: its deferred counters stand
        const uint32_t pend = R.pend[4 * (uint64_t)i + part];
        commit_q += pend & 0xFFFFu;
        commit_s += pend >> 16;
      }
      if (!(had_bits & gf_had_bit(part))) continue;
      blend(base + (uint64_t)part * (uint64_t)P.chunk, G == 1 ? run : ((run >> (8 * part)) & 0xFFu));
      if (P.ert) {
        dead = P.eps_f64 ? ((double)acc.w < P.epsilon) : (acc.w < (float)P.epsilon);
        if (dead) {
          fw &= ~(uint32_t)GF_RAY_ALIVE;
          if ((int64_t)(c + 1) * P.chunk < P.k) fw |= GF_RAY_TERMINATED;  // rounds remained
        }
      }
    }
    R.acc[i] = acc;
  }
  MarchStats ST;
  ST.v[GF_STAT_TOTAL_QUERIES] = commit_q;
  ST.v[GF_STAT_ESS_SKIPPED] = commit_s;
  if (phase == 0) fw &= ~(uint32_t)GF_RAY_HAD_ALL;

  if (final_pass) {
    if (in_range) {
      if (!had) acc = R.acc[i];
      // render.py:345-348: acc + trans*bg, clip to [0,1]
      float c0 = __fadd_rn(acc.x, __fmul_rn(acc.w, P.bg[0]));
      float c1 = __fadd_rn(acc.y, __fmul_rn(acc.w, P.bg[1]));
      float c2 = __fadd_rn(acc.z, __fmul_rn(acc.w, P.bg[2]));
      P.rgb_out[3 * i + 0] = fminf(fmaxf(c0, 0.f), 1.f);
      P.rgb_out[3 * i + 1] = fminf(fmaxf(c1, 0.f), 1.f);
      P.rgb_out[3 * i + 2] = fminf(fmaxf(c2, 0.f), 1.f);
    }
    ST.v[GF_STAT_ERT_TERMINATED] += (fw & GF_RAY_TERMINATED) ? 1ull : 0ull;
    flush_stats(P, ST);
    return;
  }

  // ---- sample this pass's round(s): with P.fuse the whole group of rounds
  // is placed by this one pass, else one round per launch (phase)
  const int nsub = P.fuse ? min(P.group, P.n_rounds - round) : 1;
#pragma unroll 1
  for (int sub = 0; sub < nsub; ++sub) march_sample<FAST>(P, R, B, i, fw, round + sub, phase + sub, ST);
  if (in_range && fw != fw0) R.flags[i] = fw;
  flush_stats(P, ST);
}

template __global__ void k_march<false>(MarchParams, RayState, RoundBufs, int, int);
template __global__ void k_march<true>(MarchParams, RayState, RoundBufs, int, int);

}  // namespace gf
