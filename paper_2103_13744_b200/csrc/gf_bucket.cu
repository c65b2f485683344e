// Bucketing of samples by network cell: counting sort with a device scan.
//
// Reference: batched.py:60-85 group_by_network (stable argsort + bincount +
// cumsum offsets) and grid.py:44-45 cell_index.  The render and query paths do
// not observe the order inside a segment (each query's result depends only on
// its own inputs and its cell's weights), so they use a warp-aggregated
// atomic scatter; the public group_by_network entry point uses the stable
// variant in gf_group.cu.
#include <algorithm>
#include <cstdlib>

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
  gf_pdl_wait();  // counts from the preceding pass (no-op outside a PDL launch)
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
  if (!in_smem) return;  // tile list built by k_fill_tiles from B.tile_off
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

// tile list from the per-cell first-tile table, one thread per tile (binary
// search over tile_off; empty cells share their successor's start)
__global__ void __launch_bounds__(256) k_fill_tiles(BucketBufs B, int64_t n_cells) {
  gf_pdl_wait();  // counts from the preceding pass (no-op outside a PDL launch)
  const uint32_t nt = *B.n_tiles;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n_cells;  // invariant: tile_off[lo] <= t < tile_off[hi]
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (B.tile_off[mid] <= t) lo = mid;
      else hi = mid;
    }
    const uint32_t r0 = (t - B.tile_off[lo]) * GF_TILE_ROWS, n_seg = B.offsets[lo + 1] - B.offsets[lo];
    B.tiles[t] = gf_make_tile((uint32_t)lo, B.offsets[lo] + r0, min(n_seg - r0, (uint32_t)GF_TILE_ROWS));
  }
}

// large grids: a two-kernel multi-CTA scan, 1024 cells per CTA, coalesced.
// (a) every CTA's (rows, tiles) total into B.tile_off (as uint2 pairs)
__global__ void __launch_bounds__(1024) k_scan_tot(BucketBufs B, int64_t n_cells) {
  gf_pdl_wait();  // counts from the preceding pass
  __shared__ uint2 warp_tot[32];
  const int64_t c = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const uint32_t cnt = c < n_cells ? B.counts[c] : 0u;
  uint2 tot;
  block_exclusive_scan2<1024>(make_uint2(cnt, gf_div_up<uint32_t>(cnt, GF_TILE_ROWS)), warp_tot, tot);
  if (threadIdx.x == 0) reinterpret_cast<uint2*>(B.tile_off)[blockIdx.x] = tot;
}

// (b) the predecessors' totals + this CTA's cells: offsets, cursors, cleared
// counts, and the tiles of this CTA's cells (binary search in shared memory;
// empty cells share their successor's first tile)
__global__ void __launch_bounds__(1024) k_scan_apply(BucketBufs B, int64_t n_cells) {
  gf_pdl_wait();
  __shared__ uint2 warp_tot[32];
  __shared__ uint32_t s_off[1025], s_toff[1025];
  const int tid = threadIdx.x;
  const uint2* tot = reinterpret_cast<const uint2*>(B.tile_off);
  uint2 p = make_uint2(0, 0);
  for (uint32_t k = tid; k < blockIdx.x; k += 1024) {
    const uint2 v = tot[k];
    p.x += v.x;
    p.y += v.y;
  }
  uint2 pre;
  block_exclusive_scan2<1024>(p, warp_tot, pre);
  const int64_t cell0 = (int64_t)blockIdx.x * 1024, c = cell0 + tid;
  const uint32_t cnt = c < n_cells ? B.counts[c] : 0u, nt = gf_div_up<uint32_t>(cnt, GF_TILE_ROWS);
  uint2 mine;
  uint2 ex = block_exclusive_scan2<1024>(make_uint2(cnt, nt), warp_tot, mine);
  ex.x += pre.x;
  ex.y += pre.y;
  if (c < n_cells) {
    B.offsets[c] = ex.x;
    B.cursor[c] = ex.x;
    B.counts[c] = 0;
  }
  s_off[tid] = ex.x;
  s_toff[tid] = ex.y;
  if (tid == 1023) {
    s_off[1024] = ex.x + cnt;
    s_toff[1024] = ex.y + nt;
    if (blockIdx.x == gridDim.x - 1) {
      B.offsets[n_cells] = ex.x + cnt;
      *B.n_tiles = ex.y + nt;
    }
  }
  __syncthreads();
  for (uint32_t t = s_toff[0] + tid; t < s_toff[1024]; t += 1024) {
    int lo = 0, hi = 1024;  // invariant: s_toff[lo] <= t < s_toff[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s_toff[mid] <= t) lo = mid;
      else hi = mid;
    }
    const uint32_t r0 = (t - s_toff[lo]) * GF_TILE_ROWS, n_seg = s_off[lo + 1] - s_off[lo];
    B.tiles[t] = gf_make_tile((uint32_t)(cell0 + lo), s_off[lo] + r0, min(n_seg - r0, (uint32_t)GF_TILE_ROWS));
  }
}

// offsets + tile list.  Small grids: one CTA does both with the tile table in
// shared memory.  Large grids / many tiles: the scan CTA writes the table to
// global memory and a grid-wide kernel fills the tiles.
int launch_scan_cells(const BucketBufs& B, int64_t n_cells, cudaStream_t st, int64_t max_rows) {
  BucketBufs b = B;
  const int64_t smem_cells = 48 * 1024 / 4 - 1;  // default dynamic smem budget
  const bool one_cta = n_cells <= smem_cells && max_rows <= (int64_t)1 << 20;
  b.scan_smem_cells = one_cta ? n_cells : 0;
  const size_t smem = one_cta ? (size_t)(n_cells + 1) * 4 : 0;
  if (n_cells > smem_cells && !getenv("GF_SCAN_ONE_CTA")) {
    // grids too large for one CTA's shared memory (C4: 32768 cells):
    // per-CTA totals, then offsets + tiles (one CTA scanning 4096 cells at a
    // time took 45 us + 9 us for the tiles; C4 frame 2.50 -> 2.24 ms).  Few
    // cells with very many rows (C5) keep the grid-wide tile fill below.
    const unsigned g = (unsigned)gf_div_up<int64_t>(n_cells, 1024);
    gf_launch_pdl(k_scan_tot, dim3(g), dim3(1024), 0, st, b, n_cells);
    gf_launch_pdl(k_scan_apply, dim3(g), dim3(1024), 0, st, b, n_cells);
    return 2;
  }
  gf_launch_pdl(k_scan_cells<1024, 4>, dim3(1), dim3(1024), smem, st, b, n_cells);
  if (!one_cta) {
    const int64_t max_tiles = max_rows / GF_TILE_ROWS + n_cells + 1;
    gf_launch_pdl(k_fill_tiles, dim3((unsigned)std::min<int64_t>(gf_div_up<int64_t>(max_tiles, 256), (int64_t)num_sms() * 8)),
                  dim3(256), 0, st, b, n_cells);
    return 2;
  }
  return 1;
}

// ---------------------------------------------------------------------------
// bulk query bucketing (NetworkGrid.query_points at scale, grid.py:50-56):
// a two-level counting sort that MOVES the (position, index) and
// (direction, key) records so the MLP streams its rows.
//   pass 1: bin each point (bounds check core.py:92-101) -> key, per-cell
//           counts (shared-memory histogram, one global atomic per bin);
//   scan:   segment offsets; cursors start at them;
//   pass 2: records -> super-cell order (key >> sb, <= 64 buckets);
//   pass 3: super-cell order -> cell order (a chunk spans few super-cells).
// Passes 2 and 3 stage GF_QB_TILE records per iteration in shared memory,
// grouped by bucket (local counting sort), reserve each bucket's run with one
// global atomic and write the runs out contiguously: scattering 16-byte
// records one by one leaves partially written lines that cost DRAM
// read-modify-writes.  Order inside a cell is arbitrary: each query's result
// depends only on its own inputs and its cell's weights.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(GF_QB_THREADS) k_query_keys_hist(GfGrid g, const float* __restrict__ pos,
                                                                   int64_t n, int64_t n_cells, uint32_t* keys,
                                                                   uint32_t* counts, int64_t* err) {
  extern __shared__ uint32_t hist[];
  for (int64_t c = threadIdx.x; c < n_cells; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float x[3];
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      x[a] = pos[3 * i + a];
      if (!((double)x[a] >= g.b_min[a] && (double)x[a] <= g.b_max[a])) {  // core.py:92-101 (NaN rejected)
        atomicMin((unsigned long long*)err, (unsigned long long)(3 * i + a));
        ok = false;
      }
    }
    uint32_t key = 0xFFFFFFFFu;
    if (ok) {
      key = gf_flat_cell(g, x[0], x[1], x[2]);
      atomicAdd(&hist[key], 1u);
    }
    keys[i] = key;
  }
  __syncthreads();
  for (int64_t c = threadIdx.x; c < n_cells; c += blockDim.x)
    if (hist[c]) atomicAdd(&counts[c], hist[c]);
}

// one staged scatter step: the block's GF_QB_TILE items (bucket bk[k] in
// [0, nb), or nb for none) are grouped by bucket in shared memory and written
// as contiguous runs at cursor[bucket] (+= run length).
struct QbStage {
  float4 rec[GF_QB_TILE];
  float4 dir[GF_QB_TILE];
  uint16_t bucket[GF_QB_TILE];
};

// dest_of (optional): dest_of[item0 + k] = the item's output row, written in
// item order (coalesced); composing the two levels' maps un-permutes results.
template <class Load>
__device__ __forceinline__ void qb_stage_scatter(QbStage& st, uint32_t* hist, uint32_t* lbase, uint32_t* gbase,
                                                 int nb, uint32_t* cursor, int cursor_shift, float4* orec,
                                                 float4* odir, uint32_t* dest_of, int64_t item0, Load load) {
  constexpr int PER = GF_QB_TILE / GF_QB_THREADS;
  for (int c = threadIdx.x; c < nb; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  float4 r[PER], d[PER];
  int bk[PER];
  uint32_t rank[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    bk[q] = load(q * GF_QB_THREADS + threadIdx.x, r[q], d[q]);  // < 0: no item
    if (bk[q] >= 0) rank[q] = atomicAdd(&hist[bk[q]], 1u);
  }
  __syncthreads();
  // exclusive scan of the bucket counts (nb <= blockDim) and global run reservation
  if (threadIdx.x < nb) {
    const uint32_t h = hist[threadIdx.x];
    gbase[threadIdx.x] = h ? atomicAdd(&cursor[(uint32_t)threadIdx.x << cursor_shift], h) : 0u;
  }
  {
    __shared__ uint32_t wsum[GF_QB_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t v = threadIdx.x < nb ? hist[threadIdx.x] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t t = lane < GF_QB_THREADS / 32 ? wsum[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      if (lane < GF_QB_THREADS / 32) wsum[lane] = t;
    }
    __syncthreads();
    if (threadIdx.x < nb) lbase[threadIdx.x] = (wid ? wsum[wid - 1] : 0u) + x - v;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (bk[q] >= 0) {
      const uint32_t k = lbase[bk[q]] + rank[q];
      st.rec[k] = r[q];
      st.dir[k] = d[q];
      st.bucket[k] = (uint16_t)bk[q];
      if (dest_of) dest_of[item0 + q * GF_QB_THREADS + threadIdx.x] = gbase[bk[q]] + rank[q];
    }
  }
  __syncthreads();
  const uint32_t total = lbase[nb - 1] + hist[nb - 1];
  for (uint32_t k = threadIdx.x; k < total; k += blockDim.x) {  // consecutive k -> consecutive run slots
    const int b = st.bucket[k];
    const uint32_t dst = gbase[b] + (k - lbase[b]);
    orec[dst] = st.rec[k];
    odir[dst] = st.dir[k];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(GF_QB_THREADS, 2) k_query_move_super(const float* __restrict__ pos,
                                                                       const float* __restrict__ dir, int64_t n,
                                                                       int sb, const uint32_t* __restrict__ keys,
                                                                       uint32_t* cursor, float4* trec, float4* tdir,
                                                                       uint32_t* dest2) {
  extern __shared__ __align__(16) uint8_t qsm[];
  QbStage& st = *reinterpret_cast<QbStage*>(qsm);
  uint32_t* hist = reinterpret_cast<uint32_t*>(qsm + sizeof(QbStage));
  uint32_t* lbase = hist + GF_QB_SUPER;
  uint32_t* gbase = lbase + GF_QB_SUPER;
  for (int64_t t0 = (int64_t)blockIdx.x * GF_QB_TILE; t0 < n; t0 += (int64_t)gridDim.x * GF_QB_TILE) {
    qb_stage_scatter(st, hist, lbase, gbase, GF_QB_SUPER, cursor, sb, trec, tdir, dest2, t0,
                     [&](int k, float4& r, float4& d) -> int {
                       const int64_t i = t0 + k;
                       if (i >= n) return -1;
                       const uint32_t key = keys[i];
                       if (key == 0xFFFFFFFFu) return -1;
                       r = make_float4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], __uint_as_float((uint32_t)i));
                       d = make_float4(dir[3 * i], dir[3 * i + 1], dir[3 * i + 2], __uint_as_float(key));
                       return (int)(key >> sb);
                     });
  }
}

// pass 3: a CTA walks a contiguous range of the super-cell order; every tile
// of it lies within one super-cell (tiles never straddle: ranges are cut at
// super-cell starts), so its buckets are the <= 2^sb cells of that super-cell
__global__ void __launch_bounds__(GF_QB_THREADS, 2) k_query_move_cell(const uint32_t* __restrict__ offsets,
                                                                      int64_t n_cells, int sb,
                                                                      const float4* __restrict__ trec,
                                                                      const float4* __restrict__ tdir,
                                                                      uint32_t* cursor, float4* srec, float4* sdir,
                                                                      uint32_t* dest3) {
  extern __shared__ __align__(16) uint8_t qsm[];
  QbStage& st = *reinterpret_cast<QbStage*>(qsm);
  uint32_t* hist = reinterpret_cast<uint32_t*>(qsm + sizeof(QbStage));
  uint32_t* lbase = hist + (1 << GF_QB_SUB_BITS);
  uint32_t* gbase = lbase + (1 << GF_QB_SUB_BITS);
  const int s = blockIdx.y;                       // super-cell
  const uint32_t s0 = offsets[(uint32_t)s << sb], s1 = offsets[min((uint32_t)(s + 1) << sb, (uint32_t)n_cells)];
  const uint32_t nb = 1u << sb;
  for (uint32_t t0 = s0 + blockIdx.x * GF_QB_TILE; t0 < s1; t0 += gridDim.x * GF_QB_TILE) {
    qb_stage_scatter(st, hist, lbase, gbase, (int)nb, cursor + ((uint32_t)s << sb), 0, srec, sdir, dest3, t0,
                     [&](int k, float4& r, float4& d) -> int {
                       const uint32_t row = t0 + (uint32_t)k;
                       if (row >= s1) return -1;
                       r = trec[row];
                       d = tdir[row];
                       return (int)(__float_as_uint(d.w) & (nb - 1u));
                     });
  }
}

// results back to caller order in two gathers that mirror the two sort
// levels (each reads from <= 64 advancing runs, so the gathers stay local;
// scattering results from the MLP would cost DRAM read-modify-writes):
//   super order: so[t] = sorted_out[dest3[t]];   caller order: out[i] = so[dest2[i]]
__global__ void __launch_bounds__(256) k_query_unperm_super(const uint32_t* __restrict__ n_valid,
                                                            const uint32_t* __restrict__ dest3,
                                                            const float4* __restrict__ sorted_out, float4* so) {
  const uint32_t nv = *n_valid;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nv; t += gridDim.x * blockDim.x)
    so[t] = sorted_out[dest3[t]];
}

__global__ void __launch_bounds__(256) k_query_unperm_caller(int64_t n, const uint32_t* __restrict__ keys,
                                                             const uint32_t* __restrict__ dest2,
                                                             const float4* __restrict__ so, float* rgb, float* sigma) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (keys[i] == 0xFFFFFFFFu) continue;  // out of bounds: the call reports an error
    const float4 v = so[dest2[i]];
    rgb[3 * i + 0] = v.x;
    rgb[3 * i + 1] = v.y;
    rgb[3 * i + 2] = v.z;
    sigma[i] = v.w;
  }
}

int launch_query_unpermute(int64_t n, const uint32_t* n_valid, const uint32_t* keys, const uint32_t* dest2,
                           const uint32_t* dest3, const float4* sorted_out, float4* so, float* rgb, float* sigma,
                           cudaStream_t st) {
  if (n == 0) return 0;
  const unsigned grid = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(n, 256), (int64_t)num_sms() * 16);
  k_query_unperm_super<<<grid, 256, 0, st>>>(n_valid, dest3, sorted_out, so);
  k_query_unperm_caller<<<grid, 256, 0, st>>>(n, keys, dest2, so, rgb, sigma);
  return 2;
}

bool query_bucket_fast_ok(int64_t n, int64_t n_cells) {
  // super-cells x sub-cells must cover the grid; offsets[n_cells] is read at the last super-cell end
  return n_cells <= ((int64_t)GF_QB_SUPER << GF_QB_SUB_BITS) && n < 0xFFFFFFF0ll && n_cells >= 1;
}

int query_super_shift(int64_t n_cells) {
  int sb = 0;
  while ((n_cells - 1) >> sb >= GF_QB_SUPER) ++sb;
  return sb;
}

size_t query_stage_smem() { return sizeof(QbStage) + 3 * (size_t)(1 << GF_QB_SUB_BITS) * 4; }

int launch_query_bucket(const GfGrid& g, const float* pos, const float* dir, int64_t n, int64_t n_cells,
                        uint32_t* keys, const BucketBufs& B, float4* trec, float4* tdir, uint32_t* cursor2,
                        uint32_t* dest2, uint32_t* dest3, int64_t* err, cudaStream_t st, int pass) {
  if (n == 0) return 0;
  const int sb = query_super_shift(n_cells);
  if (pass == 1) {
    const size_t smem = (size_t)n_cells * 4;
    static thread_local size_t smem_set = 0;
    if (smem > 48 * 1024 && smem_set < smem) {
      cudaFuncSetAttribute(k_query_keys_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      smem_set = smem;
    }
    const int64_t ctas = std::min<int64_t>(gf_div_up<int64_t>(n, GF_QB_THREADS), (int64_t)num_sms() * 2);
    k_query_keys_hist<<<(unsigned)ctas, GF_QB_THREADS, smem, st>>>(g, pos, n, n_cells, keys, B.counts, err);
    return 1;
  }
  const size_t smem = query_stage_smem();
  static thread_local bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_query_move_super, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_query_move_cell, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  // cursors: B.cursor = offsets (set by k_scan_cells) serves pass 3; pass 2
  // uses a copy (its super-cell runs start at the same offsets)
  cudaMemcpyAsync(cursor2, B.cursor, (size_t)n_cells * 4, cudaMemcpyDeviceToDevice, st);
  k_query_move_super<<<num_sms() * 2, GF_QB_THREADS, smem, st>>>(pos, dir, n, sb, keys, cursor2, trec, tdir, dest2);
  const int n_super = (int)((n_cells - 1) >> sb) + 1;
  // about 8 waves of CTAs (2 per SM): with one wave and a bit the last few
  // CTAs ran alone (C5 move_cell 1.56 ms; 8 waves: scatter 4.13 -> 3.50 ms)
  const char* pse = getenv("GF_QB_PER_SUPER");
  const unsigned per_super =
      pse ? (unsigned)atoi(pse) : (unsigned)std::max<int64_t>(1, gf_div_up<int64_t>((int64_t)num_sms() * 2 * 8, n_super));
  k_query_move_cell<<<dim3(per_super, (unsigned)n_super), GF_QB_THREADS, smem, st>>>(B.offsets, n_cells, sb, trec, tdir,
                                                                                      B.cursor, B.srec, B.sdir, dest3);
  return 2;
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
  launch_scan_cells(B, n_cells, st, n);  // rows are already in order: TileSched.sorted = NULL (identity)
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
