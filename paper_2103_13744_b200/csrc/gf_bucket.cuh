#pragma once
#include "gf_common.cuh"

namespace gf {

struct BucketBufs {
  uint32_t* counts;   // [n_cells]   histogram (zeroed by the scan)
  uint32_t* offsets;  // [n_cells+1] segment starts in `sorted`
  uint32_t* cursor;   // [n_cells]   scatter cursors
  uint2* tiles;       // [max_tiles] (cell, first row)
  uint32_t* n_tiles;  // [1]
  uint32_t* sorted;   // [capacity]  item index per sorted slot
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
