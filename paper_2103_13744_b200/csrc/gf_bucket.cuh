#pragma once
#include "gf_common.cuh"

namespace gf {

// MLP work unit: up to GF_TILE_ROWS consecutive sorted rows of one cell.
// x = cell | (rows - 1) << 25, y = absolute first sorted row.
#define GF_TILE_CELL_BITS 25
#define GF_MAX_CELLS (1ll << GF_TILE_CELL_BITS)
__host__ __device__ __forceinline__ uint2 gf_make_tile(uint32_t cell, uint32_t row0, uint32_t rows) {
  return make_uint2(cell | ((rows - 1u) << GF_TILE_CELL_BITS), row0);
}
__host__ __device__ __forceinline__ uint32_t gf_tile_cell(uint2 t) { return t.x & ((1u << GF_TILE_CELL_BITS) - 1u); }
__host__ __device__ __forceinline__ uint32_t gf_tile_rows(uint2 t) { return (t.x >> GF_TILE_CELL_BITS) + 1u; }

struct BucketBufs {
  uint32_t* counts;   // [n_cells]   histogram (zeroed by the scan)
  uint32_t* offsets;  // [n_cells+1] segment starts in `sorted`
  uint32_t* cursor;   // [n_cells]   scatter cursors
  uint2* tiles;       // [max_tiles] gf_make_tile(cell, first row, rows)
  uint32_t* n_tiles;  // [1]
  uint32_t* sorted;   // [capacity]  item index per sorted slot (query paths)
  float4* srec;       // [capacity]  sorted records (x, y, z, staging / caller index): render and bulk query
  float4* sdir;       // [capacity]  bulk query: sorted directions (x, y, z, cell bits)
  uint32_t* tile_off; // [n_cells+1] first tile of each cell (global fallback for large grids)
  int64_t scan_smem_cells;  // set by launch_scan_cells
};

// max_rows: upper bound on the rows to tile (sizes the tile-fill grid)
int launch_scan_cells(const BucketBufs& B, int64_t n_cells, cudaStream_t st, int64_t max_rows);  // -> launches

// bulk-query bucketing (gf_bucket.cu): two-level record-moving counting sort
#define GF_QB_THREADS 512
#define GF_QB_TILE 2048        // records staged in shared memory per step (2 x 16 B + 2 B each)
#define GF_QB_SUPER 64         // first-level buckets (super-cell = key >> shift)
#define GF_QB_SUB_BITS 9       // second level: <= 512 cells per super-cell (grids <= 32768 cells)
bool query_bucket_fast_ok(int64_t n, int64_t n_cells);
// pass 1 -> 1 launch; pass 2 -> 2 launches (returned)
int launch_query_bucket(const GfGrid& g, const float* pos, const float* dir, int64_t n, int64_t n_cells,
                        uint32_t* keys, const BucketBufs& B, float4* trec, float4* tdir, uint32_t* cursor2,
                        uint32_t* dest2, uint32_t* dest3, int64_t* err, cudaStream_t st, int pass);
int launch_query_unpermute(int64_t n, const uint32_t* n_valid, const uint32_t* keys, const uint32_t* dest2,
                           const uint32_t* dest3, const float4* sorted_out, float4* so, float* rgb, float* sigma,
                           cudaStream_t st);
int num_sms();
void launch_query_keys(const GfGrid& g, const float* pos, int64_t n, uint32_t* keys, uint32_t* counts, int64_t* err,
                       cudaStream_t st);
void launch_segments_from_offsets(const int64_t* offsets, int64_t n_cells, int64_t n, const BucketBufs& B,
                                  cudaStream_t st);
void launch_scatter_query(const uint32_t* keys, int64_t n, const BucketBufs& B, cudaStream_t st);

}  // namespace gf
