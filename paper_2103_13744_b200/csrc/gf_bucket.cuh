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
  float4* srec;       // [capacity]  render path: the sorted sample records themselves (x, y, z, staging index)
  uint32_t* tile_off; // [n_cells+1] first tile of each cell (global fallback for large grids)
  int64_t scan_smem_cells;  // set by launch_scan_cells
};

void launch_scan_cells(const BucketBufs& B, int64_t n_cells, cudaStream_t st);
void launch_scatter_render(const float4* rec, const uint32_t* run, const uint32_t* list, uint32_t* counts2, int round,
                           int stride, const BucketBufs& B, cudaStream_t st);
int num_sms();
void launch_query_keys(const GfGrid& g, const float* pos, int64_t n, uint32_t* keys, uint32_t* counts, int64_t* err,
                       cudaStream_t st);
void launch_segments_from_offsets(const int64_t* offsets, int64_t n_cells, int64_t n, const BucketBufs& B,
                                  cudaStream_t st);
void launch_scatter_query(const uint32_t* keys, int64_t n, const BucketBufs& B, cudaStream_t st);

}  // namespace gf
