/*
 * gridfield_b200.h — C ABI of the B200-native KiloNeRF render / network-query
 * hot path (libgridfield_b200.so).
 *
 * Plain pointers and sizes only.  Every pointer named *_dev is device memory
 * on the current CUDA device; `stream` is a cudaStream_t passed as void*.
 * All calls are asynchronous on `stream` unless stated otherwise and return a
 * gf_status_t; on failure gf_last_error() holds a thread-local message.
 *
 * The reference (gridfield, pure numpy: /root/reference/pkg/src/gridfield) has
 * no FFI; each entry point below replaces the Python function cited beside it,
 * and the Python host mirror (paper_2103_13744_b200/) binds them with ctypes
 * (see INTEGRATION.md).
 */
#ifndef GRIDFIELD_B200_H
#define GRIDFIELD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GF_ABI_VERSION 2

#if defined(__GNUC__)
#define GF_API __attribute__((visibility("default")))
#else
#define GF_API
#endif

typedef enum {
  GF_OK = 0,
  GF_ERR_INVALID = 1,      /* bad argument (host-side validation)            */
  GF_ERR_CUDA = 2,         /* CUDA launch / runtime error                    */
  GF_ERR_WORKSPACE = 3,    /* workspace smaller than *_workspace_bytes()     */
  GF_ERR_UNSUPPORTED = 4,  /* architecture / precision not compiled in       */
} gf_status_t;

/* Arithmetic used for the per-cell MLP layers. */
typedef enum {
  GF_PRECISION_FP32 = 0,   /* SIMT fp32 FMA (reference-faithful, slow)        */
  GF_PRECISION_FP16 = 1,   /* tcgen05.mma kind::f16, fp16 operands, fp32 acc  */
} gf_precision_t;

/* mlp.py:30-87 MlpArchitecture + core.py:155-184 PositionalEncoding. */
typedef struct {
  int32_t hidden_layers;   /* >= 3; trunk layers = hidden_layers - 2          */
  int32_t width;           /* hidden width (32 tiny, 64 for config 4)         */
  int32_t view_width;      /* direction-layer width (== width for tiny nets)  */
  int32_t pos_freqs;       /* 10 -> 63-wide position encoding                 */
  int32_t dir_freqs;       /* 4  -> 27-wide direction encoding                */
  int32_t include_raw;     /* 1: raw coordinates prepended                    */
  int32_t skip_layer;      /* trunk layer fed [gamma(x), h] (mlp.py:79-81); 0: none */
} gf_arch_t;

/* grid.py:19-45 NetworkGrid geometry, occupancy.py:29-79 OccupancyGrid. */
typedef struct {
  double b_min[3];
  double b_max[3];
  int32_t res[3];
} gf_grid_geom_t;

/* render.py:174-196 RenderConfig plus the call's seed. */
typedef struct {
  int32_t k;               /* nominal samples per ray                         */
  int32_t ert_chunk;       /* samples per marching round                      */
  int32_t stratified;      /* 1: PCG64 jitter per 4096-ray block              */
  int32_t eps_compare_f64; /* 0: transmittance < float32(eps) (Python float, NEP 50); 1: float64 compare */
  double epsilon;          /* ERT threshold, 0 disables                       */
  float background[3];
  int32_t rays_f64;        /* 1: origins / dirs are double (n, 3): the slab test runs on them,
                              samples on their float32 roundings (render.py:292-306) */
  uint64_t seed;           /* render_rays(seed=...)                           */
} gf_march_cfg_t;

/* render.py:25-57 Camera (pinhole, c2w row-major 3x4). */
typedef struct {
  int32_t width, height;
  double fx, fy, cx, cy;
  double c2w[12];
} gf_camera_t;

/* RenderStats counters (render.py:210-222), int64 on device, in this order. */
enum { GF_STAT_TOTAL_QUERIES = 0, GF_STAT_ESS_SKIPPED = 1, GF_STAT_ERT_TERMINATED = 2, GF_STAT_N_RAYS = 3, GF_STAT_COUNT = 4 };

/* Optional per-sample trace of the marcher (test / debug only). */
typedef struct {
  float x, y, z;            /* clipped float32 sample position                */
  uint32_t ray;             /* ray index within the call                      */
  uint32_t slot;            /* sample index along the ray (0..k-1)            */
  uint32_t cell;            /* network cell (flat, x-major)                   */
} gf_trace_rec_t;

GF_API int gf_abi_version(void);
GF_API const char* gf_last_error(void);

/* Number of float parameters per cell in manifest order (mlp.py:86-87). */
GF_API int64_t gf_param_count(const gf_arch_t* arch);

/* --- weight packing ------------------------------------------------------
 * Replaces the per-bucket gather MlpParams.at(cells) (mlp.py:148-154,
 * batched.py:140): the reference stores weights layer-major (n_cells,out,in);
 * the device wants one contiguous blob per cell in the layout the MLP kernel
 * stages into shared memory.  layer_w_dev[l] / layer_b_dev[l] are the
 * (n_cells,out,in) / (n_cells,out) float32 arrays of manifest layer l.      */
GF_API size_t gf_packed_bytes(const gf_arch_t* arch, int64_t n_cells, int precision);
GF_API int gf_pack_weights(const gf_arch_t* arch, int64_t n_cells, const float* const* layer_w_dev,
                    const float* const* layer_b_dev, void* packed_dev, int precision, void* stream);

/* The same from a checkpoint payload (io.py:162-175 / 204-214): flat_dev is
 * the float32 parameter block of a gridfield checkpoint, layer by layer in
 * manifest order, each layer's weights (n_cells,out,in) then biases
 * (n_cells,out) -- one host-to-device copy of the file's payload feeds K3. */
GF_API int gf_pack_weights_flat(const gf_arch_t* arch, int64_t n_cells, const float* flat_dev, void* packed_dev,
                                int precision, void* stream);

/* --- NetworkGrid.query_points (grid.py:50-56) -----------------------------
 * Bin at network resolution, bucket by cell, fused encode + tiny MLP,
 * results written in the caller's query order.  err_dev (int64, device) must
 * be initialised to INT64_MAX; out-of-bounds inputs leave the first offending
 * flat component index (point*3 + axis) there (core.py:92-101).           */
GF_API size_t gf_query_workspace_bytes(const gf_arch_t* arch, const gf_grid_geom_t* grid, int64_t n);
GF_API int gf_query_points(const gf_arch_t* arch, const gf_grid_geom_t* grid, const void* packed_dev, int precision,
                    const float* pos_dev, const float* dir_dev, int64_t n, float* rgb_dev, float* sigma_dev,
                    int64_t* err_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* --- batched.grouped_forward (batched.py:120-151) -------------------------
 * Rows pos/dir are already grouped: cell c owns rows offsets[c]..offsets[c+1]
 * (int64, n_cells+1).  Row j's result is written to index order[j] (int64;
 * NULL = j), i.e. back in the original query order.                        */
GF_API size_t gf_grouped_workspace_bytes(int64_t n_cells, int64_t n);
GF_API int gf_grouped_forward(const gf_arch_t* arch, int64_t n_cells, const void* packed_dev, int precision,
                              const float* pos_dev, const float* dir_dev, int64_t n, const int64_t* offsets_dev,
                              const int64_t* order_dev, float* rgb_dev, float* sigma_dev, void* ws_dev,
                              size_t ws_bytes, void* stream);
/* The training forward (batched.py:141-150 with caches): gf_grouped_forward
 * in fp32 that also keeps, per grouped row j, the activations the backward
 * needs in act_dev[j * 132 ...] = [h0 | h1 | feature | g | sigma | 3 colour
 * logits] (the reference's per-bucket caches).  Only the 32-wide tiny
 * manifest (GF_ERR_UNSUPPORTED otherwise).  Pass act_dev to
 * gf_grouped_backward_act: the backward then reads them instead of
 * recomputing the forward (identical values: same fp32 operation order). */
GF_API int gf_grouped_forward_act(const gf_arch_t* arch, int64_t n_cells, const void* packed_dev,
                                  const float* pos_dev, const float* dir_dev, int64_t n, const int64_t* offsets_dev,
                                  const int64_t* order_dev, float* rgb_dev, float* sigma_dev, float* act_dev,
                                  void* ws_dev, size_t ws_bytes, void* stream);

/* --- render.render_rays / render_image (render.py:351-400) ---------------
 * Rays come either from `cam` (pixel index = ray_offset + i, row-major) or
 * from float32 origins/directions (ray i of the call is global ray
 * ray_offset + i).  ray_offset selects the 4096-ray jitter blocks so shards of
 * one image reproduce the single-device image bit for bit.  With
 * ray_block_stride S > 1 (block-aligned ray_offset) the call's rays are the
 * interleaved blocks ray_offset/4096 + k*S (k = 0, 1, ...) — the balanced
 * multi-GPU partition; origins/dirs/rgb stay compact (n_rays rows).  occ_bits_dev may
 * be NULL (no empty-space skipping).  stats_dev: int64[GF_STAT_COUNT],
 * accumulated (caller zeroes).  trace_dev / trace_count_dev may be NULL.   */
GF_API size_t gf_render_workspace_bytes(const gf_arch_t* arch, const gf_grid_geom_t* grid, const gf_march_cfg_t* cfg,
                                 int64_t n_rays);
GF_API int gf_render_rays(const gf_arch_t* arch, const gf_grid_geom_t* grid, const void* packed_dev, int precision,
                   const gf_grid_geom_t* occ, const uint8_t* occ_bits_dev, const gf_march_cfg_t* cfg,
                   const gf_camera_t* cam, const float* origins_dev, const float* dirs_dev, int64_t ray_offset,
                   int64_t ray_block_stride, int64_t n_rays, float* rgb_dev, int64_t* stats_dev, gf_trace_rec_t* trace_dev,
                   int64_t trace_capacity, int64_t* trace_count_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* --- batched.group_by_network (batched.py:60-85) --------------------------
 * Stable counting sort of keys (< n_keys).  order/inverse: int64[n];
 * offsets: int64[n_keys+1].  err_dev as above (bad key index).             */
GF_API size_t gf_group_workspace_bytes(int64_t n, int64_t n_keys);
GF_API int gf_group_by_key(const int64_t* keys_dev, int64_t n, int64_t n_keys, int64_t* order_dev, int64_t* inverse_dev,
                    int64_t* offsets_dev, int64_t* err_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* --- pointwise primitives (core.py, occupancy.py, render.py) ------------- */
/* Points are (n,3) float32 (x_f64 = 0) or float64 (x_f64 = 1); arithmetic
 * follows numpy's promotion (binning is always float64).                    */
/* core.py:79-112 bin_point + flatten_cell_index -> flat cell per point.    */
GF_API int gf_bin_points(const gf_grid_geom_t* grid, const void* x_dev, int32_t x_f64, int64_t n, int64_t* flat_dev,
                         int64_t* err_dev, void* stream);
/* occupancy.py:76-79 occupied_at.                                          */
GF_API int gf_occupied_at(const gf_grid_geom_t* occ, const uint8_t* bits_dev, const void* x_dev, int32_t x_f64,
                          int64_t n, uint8_t* out_dev, int64_t* err_dev, void* stream);
/* render.py:151-171 intersect_aabb: float64 rays (n, 3) -> t0, t1 (n,).   */
GF_API int gf_intersect_aabb(const double* o_dev, const double* d_dev, int64_t n, const double* b_min,
                             const double* b_max, double* t0_dev, double* t1_dev, void* stream);
/* render.py:256-258 sample_ray positions: out[j] = float32(o + (t0 + (j +
 * jitter[j]) * seg) * d) in float64, for the caller's k jitter values.   */
GF_API int gf_ray_samples(const double* origin3, const double* direction3, double t0, double seg,
                          const double* jitter_dev, int64_t k, float* out_dev, void* stream);
/* core.py:52-68 clip_into (float32 points).                                */
GF_API int gf_clip_into(const double* b_min, const double* b_max, const float* x_dev, int64_t n, float* out_dev,
                 void* stream);
/* core.py:132-152 positional_encode in the input dtype, width dim*(raw+2L). */
GF_API int gf_positional_encode(const void* v_dev, int32_t v_f64, int64_t n, int32_t dim, int32_t n_freqs,
                                int32_t include_raw, void* out_dev, void* stream);
/* core.py:187-194 density_to_alpha (elementwise, same length, same dtype). */
GF_API int gf_density_to_alpha(const void* sigma_dev, const void* delta_dev, int32_t f64, int64_t n, void* out_dev,
                               void* stream);
/* render.py:269-284 composite: n_rays x n_samples, float32.                */
GF_API int gf_composite(const float* colors_dev, const float* alphas_dev, int64_t n_rays, int64_t n_samples,
                 float* rgb_dev, float* trans_dev, void* stream);
GF_API int gf_composite_f64(const double* colors_dev, const double* alphas_dev, int64_t n_rays, int64_t n_samples,
                     double* rgb_dev, double* trans_dev, void* stream);
/* render.py:139-148 generate_rays for a camera (float32 origins, dirs).    */
GF_API int gf_generate_rays(const gf_camera_t* cam, float* origins_dev, float* dirs_dev, void* stream);

/* --- analytic test scenes (scene.py:27-135) ---------------
 * The closed-form AnalyticScene field (spheres, then boxes, in the
 * reference's iteration order) evaluated on the device in place of the MLPs,
 * so scene renders (the reference's ERT-bound / ESS-exactness acceptance
 * checks, render_image(scene, ...)) run through the same marcher.          */
#define GF_MAX_PRIMS 16
typedef struct {
  int32_t kind;            /* 0 Sphere(center=a, radius), 1 Box(lo=a, hi=b)  */
  int32_t _pad;
  double a[3], b[3];
  double color[3];
  double radius, density, feather;
} gf_prim_t;

typedef struct {
  double b_min[3], b_max[3];  /* scene.aabb                                  */
  int32_t n_prims;
  int32_t _pad;
  gf_prim_t prims[GF_MAX_PRIMS];
  double texture_freq, texture_amp, view_tint;
  double tint_axis[3];
} gf_analytic_t;

/* AnalyticScene.query_points (scene.py:115-135) for n float32 points.      */
GF_API int gf_query_analytic(const gf_analytic_t* scene, const float* pos_dev, const float* dir_dev, int64_t n,
                             float* rgb_dev, float* sigma_dev, void* stream);
/* scene.py:214-252 render_brute_force: dense Simpson quadrature (n_samples
 * segments per ray over the box interval, no occupancy, no termination) of
 * the camera's rays [ray0, ray0 + n_rays) -> out (n_rays, 3) in [0, 1].   */
GF_API size_t gf_brute_force_workspace_bytes(int32_t n_samples, int64_t n_rays);
GF_API int gf_render_brute_force(const gf_analytic_t* scene, const gf_camera_t* cam, int32_t n_samples,
                                 const float* background3, int64_t ray0, int64_t n_rays, float* out_dev, void* ws_dev,
                                 size_t ws_bytes, void* stream);
/* scene.py:186-211 analytically_empty_cells: out[c] = 1 when no primitive
 * touches cell c of a res[0] x res[1] x res[2] grid over the scene box.   */
GF_API int gf_analytic_empty_cells(const gf_analytic_t* scene, const int32_t* res3, uint8_t* out_dev, void* stream);
/* render.render_rays / render_image with an AnalyticScene field: arguments as
 * gf_render_rays minus the network (the scene box is the march box).       */
GF_API size_t gf_render_analytic_workspace_bytes(const gf_analytic_t* scene, const gf_march_cfg_t* cfg,
                                                 int64_t n_rays);
GF_API int gf_render_rays_analytic(const gf_analytic_t* scene, const gf_grid_geom_t* occ, const uint8_t* occ_bits_dev,
                                   const gf_march_cfg_t* cfg, const gf_camera_t* cam, const float* origins_dev,
                                   const float* dirs_dev, int64_t ray_offset, int64_t ray_block_stride, int64_t n_rays,
                                   float* rgb_dev, int64_t* stats_dev, gf_trace_rec_t* trace_dev,
                                   int64_t trace_capacity, int64_t* trace_count_dev, void* ws_dev, size_t ws_bytes,
                                   void* stream);

/* --- caller-evaluated fields (render.py:361-364 field protocol) -----------
 * Any field object with aabb + query_points: the device marches, places and
 * composites as for the built-in fields, and once per round group hands the
 * caller the group's queried samples.  The callback gets the sorted sample
 * records (float4 x, y, z, staging index bits), their count n, the per-ray
 * direction records (float4, ray = index >> stride_shift, or index / stride
 * when stride_shift < 0) and the result buffer (float4 r, g, b, sigma by
 * staging index); gf_field_gather / gf_field_scatter convert between those
 * and plain (n, 3) / (n,) arrays.  Nonzero return aborts the render.  No
 * CUDA graph: the stream is synchronised before each callback.            */
typedef int (*gf_field_fn)(void* user, const void* srec_dev, int64_t n, const void* ray_dir_dev,
                           int32_t stride_shift, uint32_t stride, void* res_dev, void* stream);
GF_API size_t gf_render_field_workspace_bytes(const gf_grid_geom_t* box, const gf_march_cfg_t* cfg, int64_t n_rays);
GF_API int gf_render_rays_field(gf_field_fn fn, void* user, const gf_grid_geom_t* box, const gf_grid_geom_t* occ,
                                const uint8_t* occ_bits_dev, const gf_march_cfg_t* cfg, const gf_camera_t* cam,
                                const float* origins_dev, const float* dirs_dev, int64_t ray_offset,
                                int64_t ray_block_stride, int64_t n_rays, float* rgb_dev, int64_t* stats_dev,
                                gf_trace_rec_t* trace_dev, int64_t trace_capacity, int64_t* trace_count_dev,
                                void* ws_dev, size_t ws_bytes, void* stream);
GF_API int gf_field_gather(const void* srec_dev, int64_t n, const void* ray_dir_dev, int32_t stride_shift,
                           uint32_t stride, float* pos_dev, float* dir_dev, void* stream);
GF_API int gf_field_scatter(const void* srec_dev, int64_t n, const float* rgb_dev, const float* sigma_dev,
                            void* res_dev, void* stream);

/* Grouped-order rows of a query batch (batched.py:73-78 positions[order]):
 * out[j] = float32(x[idx[j]]) for (n, 3) rows, x float32 or float64.       */
GF_API int gf_gather_rows3(const void* x_dev, int32_t x_f64, const int64_t* idx_dev, int64_t n, float* out_dev,
                           void* stream);

/* --- occupancy.extract_occupancy (occupancy.py:94-128) ---------------------
 * Probe every cell of `occ` (box + resolution of the extraction) on its 3x3x3
 * lattice, clip into the box, threshold f64(density) > tau, and write the
 * packed little-endian bitmap (ceil(n_cells/8) bytes) to bits_dev.  `tau` is
 * the effective threshold: float32(tau) for a Python scalar (numpy's NEP 50
 * float32 compare), tau itself for a float64 scalar.
 * _analytic: field = AnalyticScene.density_at (scene.py:107-113), bit-exact.
 * _network:  field = train.density_probe(model, direction) (train.py:577-586),
 *   i.e. NetworkGrid.query_points at a fixed direction; probes are queried in
 *   chunks of chunk_cells cells (0 = default) through gf_query_points.  err_dev
 *   (init INT64_MAX) receives the first out-of-bounds probe component
 *   (probe*3 + axis) when the extraction box leaves the network's box, and no
 *   bit is written then.                                                    */
GF_API int gf_extract_occupancy_analytic(const gf_analytic_t* scene, const gf_grid_geom_t* occ, double tau,
                                         uint8_t* bits_dev, void* stream);
GF_API size_t gf_extract_workspace_bytes(const gf_arch_t* arch, const gf_grid_geom_t* net, const gf_grid_geom_t* occ,
                                         int64_t chunk_cells);
GF_API int gf_extract_occupancy_network(const gf_arch_t* arch, const gf_grid_geom_t* net, const void* packed_dev,
                                        int precision, const float* direction, const gf_grid_geom_t* occ, double tau,
                                        int64_t chunk_cells, uint8_t* bits_dev, int64_t* err_dev, void* ws_dev,
                                        size_t ws_bytes, void* stream);

/* --- mlp.forward / mlp.backward (mlp.py:222-316) ---------------------------
 * The reference's plain network API on ALREADY-ENCODED inputs, for any
 * manifest (depth, widths, skip layer) and a stack of n_net networks, in
 * float32 (f64 = 0) or float64 (f64 = 1).  w[l] / b[l]: layer l of the
 * manifest, (n_net, out, in) / (n_net, out); x_enc (n_net, rows, pos_dim),
 * d_enc (n_net, rows, dir_dim); color (n_net, rows, 3), sigma (n_net, rows).
 * forward optionally writes the activations backward consumes (mlp.py:252-
 * 256): hs[k] (n_net, rows, width) per trunk layer, feat (.., width), g (..,
 * view); NULL skips them.  backward takes those activations plus color /
 * sigma and the upstream d_color / d_sigma and writes gw[l] / gb[l] (same
 * shapes as w / b), summed over the rows in a fixed order.                 */
typedef struct {
  int32_t hidden_layers;   /* >= 3 (mlp.py:30-64)                              */
  int32_t width;
  int32_t view_width;      /* direction-layer width; 0: width                 */
  int32_t pos_dim;         /* position_input_dim                              */
  int32_t dir_dim;         /* direction_input_dim                             */
  int32_t skip_layer;      /* 0: none                                         */
} gf_manifest_t;

GF_API int gf_mlp_forward(const gf_manifest_t* m, int32_t f64, int64_t n_net, int64_t rows,
                          const void* const* w_dev, const void* const* b_dev, const void* x_enc_dev,
                          const void* d_enc_dev, void* color_dev, void* sigma_dev, void* const* hs_dev,
                          void* feat_dev, void* g_dev, void* stream);
GF_API size_t gf_mlp_backward_workspace_bytes(const gf_manifest_t* m, int32_t f64, int64_t n_net, int64_t rows);
GF_API int gf_mlp_backward(const gf_manifest_t* m, int32_t f64, int64_t n_net, int64_t rows,
                           const void* const* w_dev, const void* x_enc_dev, const void* d_enc_dev,
                           const void* const* hs_dev, const void* feat_dev, const void* g_dev, const void* color_dev,
                           const void* sigma_dev, const void* d_color_dev, const void* d_sigma_dev,
                           void* const* gw_dev, void* const* gb_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* --- training ----------------------------------------------
 * batched.grouped_backward (batched.py:154-187) + mlp.backward (mlp.py:269-316):
 * parameter gradients of sum(d_color*color + d_sigma*sigma) per cell.  Rows
 * pos/dir are grouped (cell c owns rows offsets[c]..offsets[c+1]); row j's
 * upstream gradient is d_color[order[j]] / d_sigma[order[j]] (order NULL =
 * identity).  packed_dev is the GF_PRECISION_FP32 packing.  gw[l] / gb[l]
 * receive layer l's gradients in the reference layout (n_cells, out, in) /
 * (n_cells, out), manifest order; cells without rows get zeros.  For the
 * 32-wide tiny manifest the wide layers' weight gradients run on tcgen05
 * (bf16 3-piece split operands, float32-level sums; GF_BWD_TC=0: CUDA
 * cores), and the workspace then also holds the operand tiles (~2 KB per
 * row).  Results are deterministic run to run.                          */
GF_API size_t gf_grouped_backward_workspace_bytes(const gf_arch_t* arch, int64_t n_cells, int64_t n);
GF_API int gf_grouped_backward(const gf_arch_t* arch, int64_t n_cells, const void* packed_dev, const float* pos_dev,
                               const float* dir_dev, int64_t n, const int64_t* offsets_dev, const int64_t* order_dev,
                               const float* d_color_dev, const float* d_sigma_dev, float* const* gw_dev,
                               float* const* gb_dev, void* ws_dev, size_t ws_bytes, void* stream);
/* gf_grouped_backward reading the training forward's activations
 * (gf_grouped_forward_act on the same grouped rows); act_dev is ignored for
 * manifests other than the 32-wide tiny one.                              */
GF_API int gf_grouped_backward_act(const gf_arch_t* arch, int64_t n_cells, const void* packed_dev,
                                   const float* pos_dev, const float* dir_dev, int64_t n, const int64_t* offsets_dev,
                                   const int64_t* order_dev, const float* d_color_dev, const float* d_sigma_dev,
                                   const float* act_dev, float* const* gw_dev, float* const* gb_dev, void* ws_dev,
                                   size_t ws_bytes, void* stream);
/* train.photometric_loss_and_grads compositing (train.py:243-288): queries
 * (ray_index, slot) of B rays x k slots with colours and densities (noise:
 * optional density perturbation, train.py:245-249), per-ray deltas, ground
 * truth gt (B,3), host background[3], two_over_b = float32(2/B).  Writes the
 * float64 sum over rays of ||pred - gt||^2 to loss_sum_dev and, when
 * d_color_q_dev is not NULL, the per-query upstream gradients.            */
GF_API size_t gf_photometric_workspace_bytes(int64_t n_rays, int32_t k, int64_t n_queries);
GF_API int gf_photometric_loss(int64_t n_rays, int32_t k, int64_t n_queries, const int64_t* ray_index_dev,
                               const int64_t* slot_dev, const float* color_dev, const float* sigma_dev,
                               const float* noise_dev, const float* deltas_dev, const float* gt_dev,
                               const float* background, float two_over_b, float* d_color_q_dev, float* d_sigma_q_dev,
                               double* loss_sum_dev, void* ws_dev, size_t ws_bytes, void* stream);
/* train.adam_update (train.py:130-143) over one flat float32 array, in place.
 * coef (host) = float32 {b1, 1-b1, b2, 1-b2, 1-b1^t, 1-b2^t, lr, eps}.    */
GF_API int gf_adam_update(float* p_dev, const float* g_dev, float* m_dev, float* v_dev, int64_t n, const float* coef,
                          void* stream);
/* train.regularization_term (train.py:146-160) helpers: float64 sum of
 * squares (fixed order), and out = y + float32(f) * x (y NULL: f * x).      */
GF_API size_t gf_sum_squares_workspace_bytes(void);
GF_API int gf_sum_squares(const float* x_dev, int64_t n, double* out_dev, void* ws_dev, size_t ws_bytes, void* stream);
GF_API int gf_axpy(const float* x_dev, const float* y_dev, int64_t n, float f, float* out_dev, void* stream);
/* train.distill_step loss terms (train.py:369-385): student / teacher colours
 * and densities of n queries, delta = float32(delta_ref), c_sigma =
 * float32(2*w_a/m), c_color = float32(2/m).  sums_dev[0] = sum(d_alpha^2),
 * sums_dev[1] = sum(d_color^2) in float64; d_color / d_sigma = upstream.   */
GF_API size_t gf_distill_workspace_bytes(int64_t n);
GF_API int gf_distill_loss(int64_t n, const float* s_color_dev, const float* s_sigma_dev, const float* t_color_dev,
                           const float* t_sigma_dev, float delta, float c_sigma, float c_color, float* d_color_dev,
                           float* d_sigma_dev, double* sums_dev, void* ws_dev, size_t ws_bytes, void* stream);

/* train.prepare_ray_samples (train.py:175-209): n float32 rays, k slots,
 * box = {b_min[3], b_max[3]}, the caller Generator's PCG64 state pcg =
 * {state_hi, state_lo, inc_hi, inc_lo} with its buffered half (has_uint32,
 * uinteger) -- only read when stratified.  _count writes per-ray kept counts
 * turned into exclusive offsets (offsets_dev[n] = Q); _write fills deltas
 * (n,), float64 positions (Q,3), float32 directions (Q,3), ray_index and
 * slot (Q,) in np.nonzero order.  The caller advances its Generator by n*k
 * float32 draws afterwards.                                               */
GF_API int gf_prepare_samples_count(const float* origins_dev, const float* dirs_dev, int64_t n, int32_t k,
                                    int32_t stratified, const double* box, const uint64_t* pcg, int32_t has_uint32,
                                    uint32_t uinteger, const gf_grid_geom_t* occ, const uint8_t* occ_bits_dev,
                                    int64_t* offsets_dev, void* stream);
GF_API int gf_prepare_samples_write(const float* origins_dev, const float* dirs_dev, int64_t n, int32_t k,
                                    int32_t stratified, const double* box, const uint64_t* pcg, int32_t has_uint32,
                                    uint32_t uinteger, const gf_grid_geom_t* occ, const uint8_t* occ_bits_dev,
                                    const int64_t* offsets_dev, float* deltas_dev, double* pos_dev, float* dirs_out_dev,
                                    int64_t* ray_index_dev, int64_t* slot_dev, void* stream);

/* --- instrumentation ------------------------------------------------------
 * Stage timing: while enabled, gf_render_rays / gf_query_points record CUDA
 * events on their stream between stages; gf_stage_times() synchronises and
 * returns accumulated milliseconds per stage (GF_STAGE_*) and launches per
 * stage, then clears.  gf_launch_count() counts every kernel this library
 * has launched in the process.                                             */
enum { GF_STAGE_SETUP = 0, GF_STAGE_MARCH = 1, GF_STAGE_SCAN = 2, GF_STAGE_SCATTER = 3, GF_STAGE_MLP = 4,
       GF_STAGE_COUNT = 5 };
GF_API int gf_stage_timing(int32_t enable);
GF_API int gf_stage_times(double* ms_out, int64_t* launches_out);
GF_API int64_t gf_launch_count(void);
/* CUDA-graph activity of gf_render_rays since process start: {replays of a
 * cached graph, in-place exec updates (new camera/seed/buffers), fresh
 * instantiations, eager runs because the stream could not be captured}.
 * Calls on the legacy default stream (0) run their graph on a per-thread
 * side stream ordered by events.                                           */
GF_API int gf_graph_counters(int64_t out4[4]);

/* --- host-side helpers (no device work) ---------------------------------- */
/* PCG64(SeedSequence([seed, block_start])).state as {state_hi, state_lo,
 * inc_hi, inc_lo} (numpy semantics; render.py:375).                          */
GF_API int gf_pcg64_block_state(uint64_t seed, uint64_t block_start, uint64_t out4[4]);

#ifdef __cplusplus
}
#endif
#endif /* GRIDFIELD_B200_H */
