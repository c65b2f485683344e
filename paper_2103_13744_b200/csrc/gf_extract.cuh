// Occupancy extraction kernels (gf_extract.cu, occupancy.py:94-128).
#pragma once
#include "gf_analytic.cuh"

namespace gf {
void launch_extract_analytic(const AnalyticDev& A, const GfGrid& g, int64_t n, double tau, uint8_t* bits,
                             cudaStream_t st);
void launch_probe_points(const GfGrid& g, int64_t first, int64_t count, const float d[3], float* pos, float* dir,
                         cudaStream_t st);
void launch_probe_any(const float* sigma, int64_t first, int64_t count, int64_t n_cells, double tau, uint8_t* bits,
                      cudaStream_t st);
void launch_probe_oob(const GfGrid& g, const GfGrid& field, int64_t n_cells, int64_t* err, cudaStream_t st);
}  // namespace gf
