// Bucketing of samples by network cell: counting sort with a device scan.
//
// Reference: batched.py:60-85 group_by_network (stable argsort + bincount +
// cumsum offsets) and grid.py:44-45 cell_index.  The render and query paths do
// not observe the order inside a segment (each query's result depends only on
// its own inputs and its cell's weights), so they use a warp-aggregated
// atomic scatter; the public group_by_network entry point uses the stable
// variant in gf_group.cu.
#include "gf_bucket.cuh"

namespace gf {

// ---------------------------------------------------------------------------
// single-CTA scan over the per-cell histogram -> segment offsets, scatter
// cursors and the MLP tile list (one tile = up to GF_TILE_ROWS rows of one
// cell).  Also clears the histogram for the next round.
// ---------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ uint2 block_exclusive_scan2(uint2 v, uint2* warp_tot, uint2& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint2 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t a = __shfl_up_sync(0xffffffffu, x.x, o), b = __shfl_up_sync(0xffffffffu, x.y, o);
    if (lane >= o) { x.x += a; x.y += b; }
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint2 t = lane < NT / 32 ? warp_tot[lane] : make_uint2(0, 0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t a = __shfl_up_sync(0xffffffffu, t.x, o), b = __shfl_up_sync(0xffffffffu, t.y, o);
      if (lane >= o) { t.x += a; t.y += b; }
    }
    if (lane < NT / 32) warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  uint2 before = wid ? warp_tot[wid - 1] : make_uint2(0, 0);
  total = warp_tot[NT / 32 - 1];
  __syncthreads();
  return make_uint2(before.x + x.x - v.x, before.y + x.y - v.y);
}

template <int NT, int ITEMS>
__global__ void __launch_bounds__(NT) k_scan_cells(BucketBufs B, int64_t n_cells) {
  __shared__ uint2 warp_tot[NT / 32];
  extern __shared__ uint32_t s_toff[];  // per-cell first tile (n_cells + 1), when it fits
  const bool in_smem = B.scan_smem_cells >= n_cells;
  uint32_t* toff = in_smem ? s_toff : B.tile_off;
  uint2 carry = make_uint2(0, 0);
  for (int64_t chunk = 0; chunk < n_cells; chunk += (int64_t)NT * ITEMS) {
    uint32_t cnt[ITEMS];
    uint2 loc = make_uint2(0, 0);
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      int64_t c = chunk + (int64_t)threadIdx.x * ITEMS + j;
      cnt[j] = c < n_cells ? B.counts[c] : 0u;
      loc.x += cnt[j];
      loc.y += gf_div_up<uint32_t>(cnt[j], GF_TILE_ROWS);
    }
    uint2 tot;
    uint2 ex = block_exclusive_scan2<NT>(loc, warp_tot, tot);
    ex.x += carry.x;
    ex.y += carry.y;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      int64_t c = chunk + (int64_t)threadIdx.x * ITEMS + j;
      if (c < n_cells) {
        B.offsets[c] = ex.x;
        B.cursor[c] = ex.x;
        toff[c] = ex.y;
        B.counts[c] = 0;
        ex.x += cnt[j];
        ex.y += gf_div_up<uint32_t>(cnt[j], GF_TILE_ROWS);
      }
    }
    carry.x += tot.x;
    carry.y += tot.y;
  }
  if (threadIdx.x == 0) {
    B.offsets[n_cells] = carry.x;
    *B.n_tiles = carry.y;
    toff[n_cells] = carry.y;
  }
  __syncthreads();
  // tile list, all threads in parallel: tile t belongs to the last cell whose
  // first tile is <= t (binary search; empty cells share their successor's start)
  const uint32_t nt = carry.y;
  for (uint32_t t = threadIdx.x; t < nt; t += NT) {
    int64_t lo = 0, hi = n_cells;  // invariant: toff[lo] <= t < toff[hi]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (toff[mid] <= t) lo = mid;
      else hi = mid;
    }
    const uint32_t r0 = (t - toff[lo]) * GF_TILE_ROWS, n_seg = B.offsets[lo + 1] - B.offsets[lo];
    B.tiles[t] = gf_make_tile((uint32_t)lo, B.offsets[lo] + r0, min(n_seg - r0, (uint32_t)GF_TILE_ROWS));
  }
}

void launch_scan_cells(const BucketBufs& B, int64_t n_cells, cudaStream_t st) {
  BucketBufs b = B;
  const int64_t smem_cells = 48 * 1024 / 4 - 1;  // default dynamic smem budget
  b.scan_smem_cells = n_cells <= smem_cells ? n_cells : 0;
  const size_t smem = b.scan_smem_cells ? (size_t)(n_cells + 1) * 4 : 0;
  k_scan_cells<1024, 4><<<1, 1024, smem, st>>>(b, n_cells);
}

// warp-aggregated cursor claim
__device__ __forceinline__ uint32_t claim_slot(uint32_t* cursor, bool pred, uint32_t key) {
  unsigned act = __ballot_sync(0xffffffffu, pred);
  uint32_t pos = 0;
  if (pred) {
    unsigned peers = __match_any_sync(act, key);
    int leader = __ffs(peers) - 1;
    uint32_t b = 0;
    if ((int)gf_lane() == leader) b = atomicAdd(&cursor[key], (uint32_t)__popc(peers));
    b = __shfl_sync(peers, b, leader);
    pos = b + __popc(peers & ((1u << gf_lane()) - 1u));
  }
  return pos;
}

// render path: records of ray i live at rec[i*stride .. +run[i]); only the
// rays the marcher listed (run > 0) are visited.  Persistent grid-stride;
// also clears the other parity's list counter for the next round.
__global__ void __launch_bounds__(256) k_scatter_render(const float4* __restrict__ rec, const uint32_t* __restrict__ run,
                                                        const uint32_t* __restrict__ list, uint32_t* counts2,
                                                        int round, int stride, BucketBufs B) {
  const uint32_t n = counts2[round & 1];
  if (blockIdx.x == 0 && threadIdx.x == 0) counts2[(round + 1) & 1] = 0;
  const uint32_t step = gridDim.x * blockDim.x;
  for (uint32_t base_k = blockIdx.x * blockDim.x; base_k < n; base_k += step) {
    const uint32_t k = base_k + threadIdx.x;
    const bool ok = k < n;
    const uint32_t i = ok ? list[k] : 0u;
    const uint32_t cnt = ok ? run[i] : 0u;
    const uint32_t nmax = __reduce_max_sync(0xffffffffu, cnt);
    const uint64_t base = (uint64_t)i * (uint64_t)stride;
    for (uint32_t j = 0; j < nmax; ++j) {
      const bool p = j < cnt;
      const uint32_t key = p ? __float_as_uint(rec[base + j].w) : 0u;
      const uint32_t pos = claim_slot(B.cursor, p, key);
      if (p) B.sorted[pos] = (uint32_t)(base + j);
    }
  }
}

void launch_scatter_render(const float4* rec, const uint32_t* run, const uint32_t* list, uint32_t* counts2, int round,
                           int stride, const BucketBufs& B, cudaStream_t st) {
  k_scatter_render<<<num_sms() * 8, 256, 0, st>>>(rec, run, list, counts2, round, stride, B);
}

// query path, pass 1: bounds check (core.py:92-101), network cell, histogram
__global__ void __launch_bounds__(256) k_query_keys(GfGrid g, const float* __restrict__ pos, int64_t n,
                                                    uint32_t* keys, uint32_t* counts, int64_t* err) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool p = i < n;
  uint32_t key = 0;
  if (p) {
    float x[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      x[a] = pos[3 * i + a];
      // core.py:92-101 (NaN is rejected too: it has no cell)
      if (!((double)x[a] >= g.b_min[a] && (double)x[a] <= g.b_max[a])) {
        atomicMin((unsigned long long*)err, (unsigned long long)(3 * i + a));
        p = false;
      }
    }
    if (p) key = gf_flat_cell(g, x[0], x[1], x[2]);
    keys[i] = p ? key : 0xFFFFFFFFu;
  }
  unsigned act = __ballot_sync(0xffffffffu, p);
  if (p) {
    unsigned peers = __match_any_sync(act, key);
    if ((unsigned)__ffs(peers) - 1 == gf_lane()) atomicAdd(&counts[key], (uint32_t)__popc(peers));
  }
}

__global__ void __launch_bounds__(256) k_scatter_query(const uint32_t* __restrict__ keys, int64_t n, BucketBufs B) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t key = i < n ? keys[i] : 0xFFFFFFFFu;
  bool p = key != 0xFFFFFFFFu;
  uint32_t pos = claim_slot(B.cursor, p, key);
  if (p) B.sorted[pos] = (uint32_t)i;
}

// grouped_forward: segments given by offsets; rows are already in order
__global__ void k_counts_from_offsets(const int64_t* __restrict__ offsets, int64_t n_cells, uint32_t* counts) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_cells) counts[c] = (uint32_t)(offsets[c + 1] - offsets[c]);
}

__global__ void k_iota(uint32_t* out, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (uint32_t)i;
}

void launch_segments_from_offsets(const int64_t* offsets, int64_t n_cells, int64_t n, const BucketBufs& B,
                                  cudaStream_t st) {
  k_counts_from_offsets<<<(unsigned)gf_div_up<int64_t>(n_cells, 256), 256, 0, st>>>(offsets, n_cells, B.counts);
  launch_scan_cells(B, n_cells, st);
  if (n > 0) k_iota<<<(unsigned)gf_div_up<int64_t>(n, 256), 256, 0, st>>>(B.sorted, n);
}

void launch_query_keys(const GfGrid& g, const float* pos, int64_t n, uint32_t* keys, uint32_t* counts, int64_t* err,
                       cudaStream_t st) {
  if (n == 0) return;
  k_query_keys<<<(unsigned)gf_div_up<int64_t>(n, 256), 256, 0, st>>>(g, pos, n, keys, counts, err);
}

void launch_scatter_query(const uint32_t* keys, int64_t n, const BucketBufs& B, cudaStream_t st) {
  if (n == 0) return;
  k_scatter_query<<<(unsigned)gf_div_up<int64_t>(n, 256), 256, 0, st>>>(keys, n, B);
}

}  // namespace gf
