// Ray marcher: ray generation, slab test, stratified PCG64 jitter, sample
// placement, clip, empty-space skipping, per-round emission, compositing and
// early ray termination.
//
// Reference: render.py:333-365 (rays, slab), render.py:481-542 (_march_block),
// render.py:545-578 (4096-ray blocks + SeedSequence jitter streams),
// core.py:52-112 (clip / bin), occupancy.py:65-79 (bit lookup),
// core.py:187-194 (alpha).
//
// One thread owns one ray for the whole frame.  Rounds (ert_chunk samples)
// are separate launches because the next round's live set depends on the
// MLP results of this round (chunk-granular ERT, render.py:532-537).
#include "gf_march.cuh"

namespace gf {

// -------------------------------------------------------------------------
// per-block PCG64 seeds: SeedSequence([seed, 4096*b])   (render.py:569)
// -------------------------------------------------------------------------
__global__ void k_seed_blocks(uint64_t seed, int64_t first_block, int64_t block_stride, int64_t n_blocks,
                              u128* seeds) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  u128 s, inc;
  gf_seed_block(seed, (uint64_t)((first_block + b * block_stride) * GF_RAY_BLOCK), &s, &inc);
  seeds[2 * b] = s;
  seeds[2 * b + 1] = inc;
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
                                 float smax, float seg) {
  const GfGrid& g = P.coarse;
  const float pos[3] = {ex, ey, ez};
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
  float s = 0.f, s_open = 0.f;
  bool open = false;
  for (int it = 0; it < 4096; ++it) {
    const uint32_t c = (uint32_t)(cell[0] + g.res[0] * (cell[1] + g.res[1] * cell[2]));
    const bool occ = (__ldg(P.coarse_bits + (c >> 5)) >> (c & 31)) & 1;
    if (occ && !open) {
      open = true;
      s_open = s;
    } else if (!occ && open) {
      emit(s_open, s);
      open = false;
    }
    const int ax = snext[0] < snext[1] ? (snext[0] < snext[2] ? 0 : 2) : (snext[1] < snext[2] ? 1 : 2);
    const float sn = snext[ax];
    if (!(sn < smax)) break;
    s = sn;
    cell[ax] += step[ax];
    if (cell[ax] < 0 || cell[ax] >= g.res[ax]) break;
    snext[ax] += sdelta[ax];
  }
  if (open) emit(s_open, smax);
  for (int k = n; k < GF_MAX_IVL; ++k) out[k] = 0x0000FFFFu;  // empty (lo > hi)
}

// -------------------------------------------------------------------------
// ray setup: render.py:333-342 generate_rays (if camera), 368-369 f64 upcast,
// 486-500 slab test / seg / t0 in float32, and the ray's jitter stream
// position.
// -------------------------------------------------------------------------
__global__ void k_ray_init(MarchParams P, RayState R) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n_rays) return;
  const int64_t g = global_ray(P, i);  // ray index within the render_rays call
  float o32[3], d32[3];
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
  } else {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      o32[a] = P.origins[3 * i + a];
      d32[a] = P.dirs[3 * i + a];
    }
  }
  // slab test in f64 (render.py:345-365)
  double lo_max = -INFINITY, hi_min = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double o = (double)o32[a], d = (double)d32[a];
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
  R.flags[i] = hit ? (uint8_t)(GF_RAY_ALIVE | GF_RAY_HIT) : (uint8_t)0;
  if (P.coarse_bits && hit) {
    const float ex = __double2float_rn(__dadd_rn((double)o32[0], __dmul_rn(t0, (double)d32[0])));
    const float ey = __double2float_rn(__dadd_rn((double)o32[1], __dmul_rn(t0, (double)d32[1])));
    const float ez = __double2float_rn(__dadd_rn((double)o32[2], __dmul_rn(t0, (double)d32[2])));
    coarse_intervals(P, R.ivl + i * GF_MAX_IVL, ex, ey, ez, d32, (float)(t1 - t0), seg);
  }
  if (P.stratified) {
    const int64_t b = seed_slot(P, g);
    uint64_t draw0 = (uint64_t)(g % GF_RAY_BLOCK) * (uint64_t)P.k;  // float32 draw index of slot 0
    u128 s = gf_pcg_advance(P.block_seeds[2 * b], P.block_seeds[2 * b + 1], (draw0 >> 1) + 1);
    R.rng[i] = s;
  }
  if (i == 0) atomicAdd((unsigned long long*)&P.stats[GF_STAT_N_RAYS], (unsigned long long)P.n_rays);
}

// -------------------------------------------------------------------------
// coarse occupancy mip: OR over factor^3 fine cells, then dilation by
// `radius` coarse cells (Chebyshev), stored as bits.
// -------------------------------------------------------------------------
__global__ void k_coarse_reduce(const uint8_t* __restrict__ occ_bits, int3 ores, int f, int3 cres, uint8_t* coarse) {
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

// warp-aggregated histogram increment: lanes with `pred` add 1 to hist[key]
__device__ __forceinline__ void hist_add(uint32_t* hist, bool pred, uint32_t key) {
  unsigned act = __ballot_sync(0xffffffffu, pred);
  if (pred) {
    unsigned peers = __match_any_sync(act, key);
    if ((unsigned)__ffs(peers) - 1 == gf_lane()) atomicAdd(&hist[key], (uint32_t)__popc(peers));
  }
}

__device__ __forceinline__ void warp_add_u64(int64_t* dst, unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (gf_lane() == 0 && v) atomicAdd((unsigned long long*)dst, v);
}

// -------------------------------------------------------------------------
// march pass r: composite round r-1 (+ERT), then place / skip / emit round r.
// At r == n_rounds: composite the last round and write the final colours.
// -------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_march(MarchParams P, RayState R, RoundBufs B, int round) {
  const int64_t i = march_ray(P, (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  bool in_range = i < P.n_rays;
  uint8_t flags = in_range ? R.flags[i] : 0;
  bool final_pass = round == P.n_rounds;
  if (!final_pass && !__any_sync(0xffffffffu, flags & GF_RAY_ALIVE)) return;

  float4 acc = make_float4(0.f, 0.f, 0.f, 1.f);
  float seg = 0.f;
  uint64_t base = (uint64_t)i * (uint64_t)P.stride;
  if (flags & GF_RAY_ALIVE) {
    acc = R.acc[i];
    seg = R.dir[i].w;
    if (round > 0) {
      // ---- composite round r-1 (render.py:527-531), float32, no contraction
      uint32_t n = R.run[i];
      float tr = 1.0f, sr = 0.f, sg = 0.f, sb = 0.f;
      for (uint32_t j = 0; j < n; ++j) {
        float4 q = B.res[base + j];
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
      // ---- ERT after the round (render.py:532-537)
      if (P.ert) {
        bool dead = P.eps_f64 ? ((double)acc.w < P.epsilon) : (acc.w < (float)P.epsilon);
        if (dead) {
          flags &= (uint8_t)~GF_RAY_ALIVE;
          if ((int64_t)round * P.chunk < P.k) flags |= GF_RAY_TERMINATED;  // rounds remained
        }
      }
      R.acc[i] = acc;
    }
  } else if (final_pass && in_range) {
    acc = R.acc[i];
  }

  if (final_pass) {
    if (in_range) {
      // render.py:539-542: acc + trans*bg, clip to [0,1]
      float c0 = __fadd_rn(acc.x, __fmul_rn(acc.w, P.bg[0]));
      float c1 = __fadd_rn(acc.y, __fmul_rn(acc.w, P.bg[1]));
      float c2 = __fadd_rn(acc.z, __fmul_rn(acc.w, P.bg[2]));
      P.rgb_out[3 * i + 0] = fminf(fmaxf(c0, 0.f), 1.f);
      P.rgb_out[3 * i + 1] = fminf(fmaxf(c1, 0.f), 1.f);
      P.rgb_out[3 * i + 2] = fminf(fmaxf(c2, 0.f), 1.f);
    }
    warp_add_u64(&P.stats[GF_STAT_ERT_TERMINATED], (flags & GF_RAY_TERMINATED) ? 1ull : 0ull);
    return;
  }

  bool active = (flags & GF_RAY_ALIVE) != 0;
  if (in_range) {
    R.flags[i] = flags;
    if (!active) R.run[i] = 0;  // a ray that stops here must not re-emit last round's samples
  }
  if (!__any_sync(0xffffffffu, active)) return;

  // ---- sample round r (render.py:505-524)
  int s0 = round * P.chunk;
  int m = min(P.chunk, P.k - s0);
  float4 o = active ? R.org[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  float4 d = active ? R.dir[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  u128 S = 0, inc = 0;
  uint64_t outw = 0;
  uint64_t draw = 0;
  if (P.stratified && active) {
    const int64_t g = global_ray(P, i);
    inc = P.block_seeds[2 * seed_slot(P, g) + 1];
    S = R.rng[i];
    outw = gf_pcg_output(S);
    draw = (uint64_t)(g % GF_RAY_BLOCK) * (uint64_t)P.k + (uint64_t)s0;
  }
  const double t0 = (double)o.w, sg64 = (double)d.w;
  const double ox = (double)o.x, oy = (double)o.y, oz = (double)o.z;
  const double dx = (double)d.x, dy = (double)d.y, dz = (double)d.z;
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
  const bool fast_clip = P.grid.fast != 0;
  uint32_t kept = 0;
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
    if (__any_sync(0xffffffffu, cand) && cand) {
      // t = f64(t0_32) + (f64(slot) + f64(jit)) * f64(seg_32); p = f32(f64(o32) + t*f64(d32))
      const double t = __dadd_rn(t0, __dmul_rn(__dadd_rn(jd, jit), sg64));
      float px = __double2float_rn(__dadd_rn(ox, __dmul_rn(t, dx)));
      float py = __double2float_rn(__dadd_rn(oy, __dmul_rn(t, dy)));
      float pz = __double2float_rn(__dadd_rn(oz, __dmul_rn(t, dz)));
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
      if (keep) {
        cell = gf_flat_cell(P.grid, px, py, pz);
        B.rec[base + kept] = make_float4(px, py, pz, __uint_as_float(cell));
        if (P.trace) {
          unsigned long long slotpos = atomicAdd((unsigned long long*)P.trace_count, 1ull);
          if ((int64_t)slotpos < P.trace_capacity)
            P.trace[slotpos] = gf_trace_rec_t{px, py, pz, (uint32_t)global_ray(P, i), (uint32_t)(s0 + j), cell};
        }
        ++kept;
      }
    }
    hist_add(B.counts, keep, cell);
  }
  if (active) {
    R.run[i] = kept;
    if (P.stratified) R.rng[i] = S;
  }
  warp_add_u64(&P.stats[GF_STAT_TOTAL_QUERIES], kept);
  warp_add_u64(&P.stats[GF_STAT_ESS_SKIPPED], active ? (unsigned long long)(m - (int)kept) : 0ull);
}

}  // namespace gf
