// Occupancy extraction on the device.
//
// Reference: occupancy.py:94-128 extract_occupancy.  Every occupancy cell is
// probed on its 3x3x3 lattice {0, 0.5, 1}^3 (occupancy.py:18-19
// _PROBE_OFFSETS, ij order: probe p = 9a + 3b + c has offsets (o[a], o[b], o[c]));
// a cell is occupied iff any probe density is > tau.  Probe positions follow
// the reference's float64 arithmetic exactly:
//   lo  = b_min + f64(i) * cell                     (occupancy.py:118)
//   p32 = f32(lo + offset * cell)                   (occupancy.py:122)
//   x   = clip_into(p32, aabb)                      (occupancy.py:123, core.py:52-68)
// The threshold compare is done as f64(sigma) > tau_eff: the host passes
// tau_eff = f32(tau) for a Python scalar (NEP 50 weak scalar -> float32
// comparison) and tau itself for a float64 scalar, which is numpy's semantics.
//
// Bits are written as the reference packs them (np.packbits little-endian):
// a warp covers 32 consecutive cells, one ballot, four byte stores.
#include "gf_analytic.cuh"
#include "gf_extract.cuh"

namespace gf {

__device__ __forceinline__ float probe_axis(const GfGrid& g, int a, int64_t i, int o) {
  const double lo = __dadd_rn(g.b_min[a], __dmul_rn((double)i, g.cell[a]));
  const double off = o == 0 ? 0.0 : (o == 1 ? 0.5 : 1.0);
  const float p = __double2float_rn(__dadd_rn(lo, __dmul_rn(off, g.cell[a])));
  return gf_clip_component(p, g.b_min[a], g.b_max[a]);
}

struct CellIdx {
  int64_t ix, iy, iz;
};

__device__ __forceinline__ CellIdx cell_of(const GfGrid& g, int64_t c) {
  CellIdx r;
  r.ix = c % g.res[0];
  r.iy = (c / g.res[0]) % g.res[1];
  r.iz = c / ((int64_t)g.res[0] * g.res[1]);
  return r;
}

// one warp stores the packed bits of its 32 consecutive cells (c = warp base + lane)
__device__ __forceinline__ void store_bits(bool occ, int64_t c, uint8_t* bits, int64_t nbytes) {
  const unsigned m = __ballot_sync(0xffffffffu, occ);
  const int lane = threadIdx.x & 31;
  if ((lane & 7) == 0) {
    const int64_t byte = c >> 3;
    if (byte < nbytes) bits[byte] = (uint8_t)(m >> lane);
  }
}

// analytic field: probes, density and threshold fused per cell (no HBM traffic
// but the bitmap); the first probe above tau ends the cell's loop.
__global__ void __launch_bounds__(256) k_extract_analytic(AnalyticDev A, GfGrid g, int64_t n, double tau,
                                                          uint8_t* bits, int64_t nbytes) {
  const int64_t n_pad = (n + 31) & ~(int64_t)31;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_pad; c += (int64_t)gridDim.x * blockDim.x) {
    bool occ = false;
    if (c < n) {
      const CellIdx ci = cell_of(g, c);
      float px[3], py[3], pz[3];
#pragma unroll
      for (int o = 0; o < 3; ++o) {
        px[o] = probe_axis(g, 0, ci.ix, o);
        py[o] = probe_axis(g, 1, ci.iy, o);
        pz[o] = probe_axis(g, 2, ci.iz, o);
      }
      for (int p = 0; p < 27 && !occ; ++p)
        occ = (double)analytic_density(A, px[p / 9], py[(p / 3) % 3], pz[p % 3]) > tau;
    }
    store_bits(occ, c, bits, nbytes);
  }
}

// network field: the probes of cells [first, first + count) as query points
// (27 per cell, in the reference's order) with the probe's fixed direction
__global__ void __launch_bounds__(256) k_probe_points(GfGrid g, int64_t first, int64_t count, float dx, float dy,
                                                      float dz, float* __restrict__ pos, float* __restrict__ dir) {
  const int64_t n = count * 27;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = first + q / 27;
    const int p = (int)(q % 27);
    const CellIdx ci = cell_of(g, c);
    pos[3 * q + 0] = probe_axis(g, 0, ci.ix, p / 9);
    pos[3 * q + 1] = probe_axis(g, 1, ci.iy, (p / 3) % 3);
    pos[3 * q + 2] = probe_axis(g, 2, ci.iz, p % 3);
    dir[3 * q + 0] = dx;
    dir[3 * q + 1] = dy;
    dir[3 * q + 2] = dz;
  }
}

// (sigma.reshape(len(lo), 27) > tau).any(axis=1) for one chunk; first % 32 == 0
__global__ void __launch_bounds__(256) k_probe_any(const float* __restrict__ sigma, int64_t first, int64_t count,
                                                   double tau, uint8_t* bits, int64_t nbytes) {
  const int64_t n_pad = (count + 31) & ~(int64_t)31;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_pad; c += (int64_t)gridDim.x * blockDim.x) {
    bool occ = false;
    if (c < count)
      for (int p = 0; p < 27 && !occ; ++p) occ = (double)sigma[c * 27 + p] > tau;
    store_bits(occ, first + c, bits, nbytes);
  }
}

// first out-of-bounds probe component against the field's box, flat index
// (probe * 3 + axis) over the whole probe array (core.py:92-101 reports the
// first offending component of the first failing chunk == the global first).
__global__ void __launch_bounds__(256) k_probe_oob(GfGrid g, GfGrid field, int64_t n_cells, int64_t* err) {
  const int64_t n = n_cells * 27;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const CellIdx ci = cell_of(g, q / 27);
    const int p = (int)(q % 27);
    const int64_t idx[3] = {ci.ix, ci.iy, ci.iz};
    const int o[3] = {p / 9, (p / 3) % 3, p % 3};
    for (int a = 0; a < 3; ++a) {
      const double v = (double)probe_axis(g, a, idx[a], o[a]);
      if (v < field.b_min[a] || v > field.b_max[a]) {
        atomicMin((unsigned long long*)err, (unsigned long long)(q * 3 + a));
        break;
      }
    }
  }
}

static unsigned grid_for(int64_t n, int per_sm) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(gf_div_up<int64_t>(n, 256), (int64_t)num_sms() * per_sm));
}

void launch_extract_analytic(const AnalyticDev& A, const GfGrid& g, int64_t n, double tau, uint8_t* bits,
                             cudaStream_t st) {
  if (n == 0) return;
  k_extract_analytic<<<grid_for((n + 31) & ~31ll, 8), 256, 0, st>>>(A, g, n, tau, bits, (n + 7) / 8);
}

void launch_probe_points(const GfGrid& g, int64_t first, int64_t count, const float d[3], float* pos, float* dir,
                         cudaStream_t st) {
  if (count == 0) return;
  k_probe_points<<<grid_for(count * 27, 16), 256, 0, st>>>(g, first, count, d[0], d[1], d[2], pos, dir);
}

void launch_probe_any(const float* sigma, int64_t first, int64_t count, int64_t n_cells, double tau, uint8_t* bits,
                      cudaStream_t st) {
  if (count == 0) return;
  k_probe_any<<<grid_for((count + 31) & ~31ll, 16), 256, 0, st>>>(sigma, first, count, tau, bits, (n_cells + 7) / 8);
}

void launch_probe_oob(const GfGrid& g, const GfGrid& field, int64_t n_cells, int64_t* err, cudaStream_t st) {
  if (n_cells == 0) return;
  k_probe_oob<<<grid_for(n_cells * 27, 16), 256, 0, st>>>(g, field, n_cells, err);
}

}  // namespace gf
