// Training kernels (gf_train.cu).
#pragma once
#include "gf_mlp.cuh"

namespace gf {

struct BwdArgs {
  const float* pos;         // (n, 3) rows in grouped (cell-sorted) order
  const float* dir;         // (n, 3)
  const int64_t* offsets;   // (n_cells + 1) segment starts
  const int64_t* order;     // sorted row -> index of its upstream gradient (NULL: identity)
  const float* d_color;     // (n, 3) upstream, original query order
  const float* d_sigma;     // (n,)
  float* gw[GF_MAX_LAYERS]; // reference layout (n_cells, out, in)
  float* gb[GF_MAX_LAYERS]; // (n_cells, out)
  const float* act;         // NULL, or the training forward's activations per grouped row (GF_ACT_FLOATS, W = 32)
};

struct PhotoArgs {
  int64_t n_rays, n_queries;
  int k;
  const int64_t* ray_index;  // (Q,)
  const int64_t* slot;       // (Q,)
  const float* color;        // (Q, 3) query colours
  const float* sigma;        // (Q,)
  const float* noise;        // (Q,) or NULL
  const float* deltas;       // (B,) per-ray nominal segment
  const float* gt;           // (B, 3)
  float bg[3];
  float two_over_b;          // float32(2.0 / B)
  float* d_color_q;          // (Q, 3) out, NULL: loss only
  float* d_sigma_q;          // (Q,) out
};

struct AdamCoef {
  float b1, one_minus_b1, b2, one_minus_b2, bc1, bc2, lr, eps;
};

struct DistillArgs {
  int64_t n;                // n_cells * points_per_cell queries
  const float* s_color;     // (n, 3) student
  const float* s_sigma;     // (n,)
  const float* t_color;     // (n, 3) teacher
  const float* t_sigma;     // (n,)
  float delta;              // float32(delta_ref)
  float c_sigma;            // float32(2 * w_a / m)
  float c_color;            // float32(2 / m)
  float* d_color;           // (n, 3) out
  float* d_sigma;           // (n,) out
};

size_t bwd_workspace(const LayerTable& t, int64_t n_cells, int64_t n);
bool launch_grouped_backward(const LayerTable& t, const float* packed, const BwdArgs& A, int64_t n_cells, int64_t n,
                             void* ws, cudaStream_t st);
size_t photo_workspace(int64_t n_rays, int k, int64_t n_queries);
void launch_photometric(const PhotoArgs& A, void* ws, double* loss_sum, cudaStream_t st);
void launch_adam(float* p, const float* g, float* m, float* v, int64_t n, const AdamCoef& c, cudaStream_t st);
void launch_sumsq(const float* x, int64_t n, double* parts, int n_parts, double* out, cudaStream_t st);
void launch_axpy(const float* x, const float* y, int64_t n, float f, float* out, cudaStream_t st);
void launch_distill(const DistillArgs& A, double* parts, double* sums, cudaStream_t st);

}  // namespace gf
