// train.prepare_ray_samples (train.py:175-209) on the device.
//
// For each ray (float32 origin / direction): the float64 slab test
// (render.py:151-171), seg32 = f32((t1 - t0) / k), and k samples
//   t = f64(f32(t0)) + (f64(j) + f64(jit)) * f64(seg32)      (train.py:196)
//   p = f64(o32) + t * f64(d32), clamped into the box in f64  (train.py:197-198)
// kept iff the ray hits the box and (with an occupancy grid) p's cell is set
// (train.py:199-201).  Positions stay float64, as numpy promotes them there
// (int64 arange + float32 jitter -> float64).
//
// The jitter is the caller's numpy Generator: rng.random((n, k), float32) is
// draw g = i*k + j of its PCG64 stream, where each float32 consumes one 32-bit
// half of a 64-bit output (low half first) after an optional buffered half
// (has_uint32 / uinteger).  Thread i jumps straight to its first word
// (gf_pcg_advance) and steps from there; the host advances the Generator by
// the same number of draws afterwards.
//
// One warp per ray: lane l takes the contiguous slot slice [l*S, (l+1)*S),
// S = ceil(k / 32), jumping straight to the slice's first draw.  Output order
// is np.nonzero's (ray-major, slot ascending): a count pass (lane counts summed
// per ray), a single-CTA exclusive scan over rays, and a write pass that
// recounts, places each lane's slice after the lower lanes' samples, and
// recomputes the samples.
#include "gf_common.cuh"
#include "gf_samples.cuh"

namespace gf {

struct RaySetup {
  double o[3], d[3];
  float o32[3], d32[3];
  double t0_32;  // f64(f32(t0))
  float seg;
  bool hit;
};

__device__ __forceinline__ RaySetup ray_setup(const PrepArgs& A, int64_t i) {
  RaySetup r;
  double lo_max = -INFINITY, hi_min = INFINITY;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    r.o32[a] = A.origins[3 * i + a];
    r.d32[a] = A.dirs[3 * i + a];
    const double o = (double)r.o32[a], d = (double)r.d32[a];
    r.o[a] = o;
    r.d[a] = d;
    double lo, hi;
    if (d == 0.0) {
      const bool inside = (o >= A.b_min[a]) && (o <= A.b_max[a]);
      lo = inside ? -INFINITY : INFINITY;
      hi = inside ? INFINITY : -INFINITY;
    } else {
      const double ta = __ddiv_rn(__dsub_rn(A.b_min[a], o), d);
      const double tb = __ddiv_rn(__dsub_rn(A.b_max[a], o), d);
      lo = fmin(ta, tb);
      hi = fmax(ta, tb);
    }
    lo_max = fmax(lo_max, lo);
    hi_min = fmin(hi_min, hi);
  }
  const double t0 = fmax(lo_max, 0.0), t1 = hi_min;
  r.hit = t1 > t0;
  r.seg = r.hit ? __double2float_rn(__ddiv_rn(__dsub_rn(t1, t0), (double)A.k)) : 0.0f;
  r.t0_32 = (double)__double2float_rn(t0);
  return r;
}

// the caller Generator's float32 draws g0, g0+1, ... in order
struct DrawStream {
  u128 s, inc;
  uint64_t word;
  int half;       // next half of `word` to use (0 low, 1 high); 2: fetch a new word
  int buffered;   // the Generator's buffered uint32 is the next draw
  uint32_t uinteger;

  __device__ __forceinline__ void init(const PrepArgs& A, uint64_t g0) {
    inc = A.inc;
    uinteger = A.uinteger;
    buffered = (A.has_uint32 && g0 == 0) ? 1 : 0;
    const uint64_t gg = g0 - (uint64_t)(A.has_uint32 && g0 > 0 ? 1 : 0);  // draws past the buffered half
    const uint64_t w = gg >> 1;                                           // words fully before draw gg
    s = gf_pcg_advance(A.state, inc, w);  // state after w outputs
    half = 2;
    if (!buffered && (gg & 1)) {  // draw gg is the high half of output w+1
      s = gf_pcg_step(s, inc);
      word = gf_pcg_output(s);
      half = 1;
    }
  }
  __device__ __forceinline__ uint32_t next() {
    if (buffered) {
      buffered = 0;
      return uinteger;
    }
    if (half == 2) {
      s = gf_pcg_step(s, inc);
      word = gf_pcg_output(s);
      half = 0;
    }
    const uint32_t u = half == 0 ? (uint32_t)word : (uint32_t)(word >> 32);
    half = half == 0 ? 1 : 2;
    return u;
  }
};

// samples of ray i in slots [j0, j1): count them, or write them from row `out0`
template <bool WRITE>
__device__ __forceinline__ uint32_t ray_samples(const PrepArgs& A, const RaySetup& r, int64_t i, int j0, int j1,
                                                int64_t out0) {
  if (!r.hit) return 0;  // a miss keeps nothing (its draws are accounted for by the host's Generator advance)
  DrawStream ds;
  if (A.stratified && j0 < j1) ds.init(A, (uint64_t)i * (uint64_t)A.k + (uint64_t)j0);
  uint32_t c = 0;
  for (int j = j0; j < j1; ++j) {
    float jit = 0.5f;
    if (A.stratified) jit = (float)(ds.next() >> 8) * (1.0f / 16777216.0f);
    const double t = __dadd_rn(r.t0_32, __dmul_rn(__dadd_rn((double)j, (double)jit), (double)r.seg));
    double p[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double v = __dadd_rn(r.o[a], __dmul_rn(t, r.d[a]));
      p[a] = fmin(fmax(v, A.b_min[a]), A.b_max[a]);  // np.clip against the f64 box
    }
    bool keep = true;
    if (A.occ_bits) {
      const uint32_t f = (uint32_t)(gf_bin_axis(A.occ, 0, p[0]) +
                                    A.occ.res[0] * (gf_bin_axis(A.occ, 1, p[1]) +
                                                    A.occ.res[1] * gf_bin_axis(A.occ, 2, p[2])));
      keep = (A.occ_bits[f >> 3] >> (f & 7)) & 1;
    }
    if (!keep) continue;
    if (WRITE) {
      const int64_t q = out0 + c;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        A.pos[3 * q + a] = p[a];
        A.dir_out[3 * q + a] = r.d32[a];
      }
      A.ray_index[q] = i;
      A.slot[q] = j;
    }
    ++c;
  }
  return c;
}

__global__ void __launch_bounds__(128) k_prep_count(PrepArgs A) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= A.n) return;  // warp-uniform
  const int S = (A.k + 31) / 32, j0 = min(A.k, lane * S), j1 = min(A.k, j0 + S);
  const RaySetup r = ray_setup(A, i);
  const uint32_t c = __reduce_add_sync(0xffffffffu, ray_samples<false>(A, r, i, j0, j1, 0));
  if (lane == 0) A.offsets[i] = c;
}

// exclusive scan of the per-ray counts (one CTA, fixed order); offsets[n] = total
__global__ void __launch_bounds__(1024) k_prep_scan(PrepArgs A) {
  __shared__ int64_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t per = (A.n + 1023) / 1024, c0 = (int64_t)tid * per;
  int64_t local = 0;
  for (int64_t c = c0; c < c0 + per && c < A.n; ++c) local += A.offsets[c];
  int64_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int64_t t = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  int64_t base = (wid ? wsum[wid - 1] : 0) + x - local;
  for (int64_t c = c0; c < c0 + per && c < A.n; ++c) {
    const int64_t v = A.offsets[c];
    A.offsets[c] = base;
    base += v;
  }
  if (tid == 1023) A.offsets[A.n] = base;
}

__global__ void __launch_bounds__(128) k_prep_write(PrepArgs A) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= A.n) return;  // warp-uniform
  const int S = (A.k + 31) / 32, j0 = min(A.k, lane * S), j1 = min(A.k, j0 + S);
  const RaySetup r = ray_setup(A, i);
  if (lane == 0) A.deltas[i] = r.seg;
  if (!r.hit) return;  // no samples (the draws only matter for the host-side Generator advance)
  const uint32_t c = ray_samples<false>(A, r, i, j0, j1, 0);
  uint32_t x = c;  // inclusive scan of the lane counts
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (c) ray_samples<true>(A, r, i, j0, j1, A.offsets[i] + (x - c));
}

void launch_prepare_count(const PrepArgs& A, cudaStream_t st) {
  if (A.n <= 0) return;
  const unsigned g = (unsigned)gf_div_up<int64_t>(A.n * 32, 128);
  k_prep_count<<<g, 128, 0, st>>>(A);
  k_prep_scan<<<1, 1024, 0, st>>>(A);
}

void launch_prepare_write(const PrepArgs& A, cudaStream_t st) {
  if (A.n <= 0) return;
  k_prep_write<<<(unsigned)gf_div_up<int64_t>(A.n * 32, 128), 128, 0, st>>>(A);
}

}  // namespace gf
