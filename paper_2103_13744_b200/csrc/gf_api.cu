// extern "C" entry points of libgridfield_b200.so (include/gridfield_b200.h).
//
// Host-side orchestration only: argument validation, workspace carving and
// the launch sequence of the render / query pipelines on the caller's stream.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "gf_analytic.cuh"
#include "gf_extract.cuh"
#include "gf_train.cuh"
#include "gf_samples.cuh"
#include "gf_march.cuh"
#include "gf_mlp.cuh"

namespace gf {
size_t group_workspace(int64_t n, int64_t n_keys);
void launch_group(const int64_t* keys, int64_t n, int64_t n_keys, int64_t* order, int64_t* inverse, int64_t* offsets,
                  int64_t* err, void* ws, cudaStream_t st);
void launch_bin_points(const GfGrid& g, const void* x, int f64, int64_t n, int64_t* flat, int64_t* err,
                       cudaStream_t st);
void launch_gather_rows3(const void* x, int f64, const int64_t* idx, int64_t n, float* out, cudaStream_t st);
void launch_occupied_at(const GfGrid& g, const uint8_t* bits, const void* x, int f64, int64_t n, uint8_t* out,
                        int64_t* err, cudaStream_t st);
void launch_clip(const double* lo, const double* hi, const float* x, int64_t n, float* out, cudaStream_t st);
void launch_intersect_aabb(const double* o, const double* d, int64_t n, const double* lo, const double* hi, double* t0,
                           double* t1, cudaStream_t st);
void launch_ray_samples(const double* o, const double* d, double t0, double seg, const double* jit, int64_t k,
                        float* out, cudaStream_t st);
void launch_encode(const void* v, int f64, int64_t n, int dim, int L, int raw, void* out, cudaStream_t st);
void launch_alpha(const void* s, const void* d, int f64, int64_t n, void* out, cudaStream_t st);
void launch_composite(const float* c, const float* a, int64_t nr, int64_t ns, float* rgb, float* tr, cudaStream_t st);
void launch_composite_f64(const double* c, const double* a, int64_t nr, int64_t ns, double* rgb, double* tr,
                          cudaStream_t st);
void launch_gen_rays(const gf_camera_t& c, float* o, float* d, cudaStream_t st);

int num_sms() {
  static thread_local int dev = -1, sms = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (d != dev) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    dev = d;
  }
  return sms > 0 ? sms : 148;
}
}  // namespace gf

using namespace gf;

// programmatic dependent launch between the frame's kernels (gf_common.cuh)
bool gf_pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("GF_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}


#include <atomic>
#include <mutex>
#include <vector>

static thread_local std::string g_err;

// ---------------------------------------------------------------------------
// instrumentation: launch counter + optional per-stage CUDA-event timing
// ---------------------------------------------------------------------------
static std::atomic<int64_t> g_launches{0};

struct StageTimer {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, cudaEvent_t>> marks;  // (stage finished, event)
  std::vector<std::pair<int, int>> launches;       // (stage, count)
  size_t used = 0;
  cudaEvent_t next() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
};
static thread_local StageTimer g_timer;

// Record that `n` kernels of stage `stage` were just enqueued on `st`.
static void stage_mark(cudaStream_t st, int stage, int n) {
  g_launches += n;
  if (!g_timer.on) return;
  if (g_timer.marks.empty()) {  // opening mark for this call
    cudaEvent_t e0 = g_timer.next();
    cudaEventRecord(e0, st);
    g_timer.marks.push_back({-1, e0});
  }
  cudaEvent_t e = g_timer.next();
  cudaEventRecord(e, st);
  g_timer.marks.push_back({stage, e});
  g_timer.launches.push_back({stage, n});
}

static void stage_open(cudaStream_t st) {
  if (!g_timer.on) return;
  cudaEvent_t e0 = g_timer.next();
  cudaEventRecord(e0, st);
  g_timer.marks.push_back({-1, e0});
}

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

static int check_cuda(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(GF_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
  return GF_OK;
}

// ---------------------------------------------------------------------------
// CUDA-graph cache: a render call's ~55 launches are captured once per exact
// argument set (all kernel parameters, workspace pointers, seed) and replayed
// with one cudaGraphLaunch afterwards.
// ---------------------------------------------------------------------------
struct GraphKey {
  std::vector<unsigned char> b;
  template <class T>
  void add(const T& v) {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
};

struct GraphEntry {
  std::vector<unsigned char> key;
  std::vector<unsigned char> topo;  // launch structure only (no per-view values)
  int dev;
  cudaGraphExec_t exec;
  int64_t launches;
  uint64_t last_use;
};

static std::mutex g_graph_mu;
static std::vector<GraphEntry> g_graphs;
static uint64_t g_graph_tick = 0;

// A new argument set with the launch structure of a cached graph (a new
// camera, seed or output buffer) is captured and applied to that graph with
// cudaGraphExecUpdate, which costs far less than a fresh instantiation.
// graph activity (gf_graph_counters): replays of a cached exec, in-place
// updates of a cached exec, fresh instantiations, eager fallbacks
static std::atomic<int64_t> g_graph_replays{0}, g_graph_updates{0}, g_graph_instantiations{0}, g_graph_eager{0};

// The legacy default stream (handle 0, what torch's default stream is)
// cannot be captured.  Calls on it run their graph on a per-thread,
// per-device side stream instead, ordered after the caller's earlier work
// and before its later work by two events.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t in = nullptr, out = nullptr;
};

struct StreamScope {
  cudaStream_t user, run;
  SideStream* side = nullptr;
  StreamScope(cudaStream_t st, int dev) : user(st), run(st) {
    if (st != nullptr && st != cudaStreamLegacy) return;
    static thread_local std::vector<SideStream> per_dev;
    if ((int)per_dev.size() <= dev) per_dev.resize(dev + 1);
    SideStream& ss = per_dev[dev];
    if (!ss.s) {
      if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&ss.in, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&ss.out, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        ss = SideStream{};
        return;  // no side stream: the caller's stream is used (eager)
      }
    }
    side = &ss;
    cudaEventRecord(ss.in, st);
    cudaStreamWaitEvent(ss.s, ss.in, 0);
    run = ss.s;
  }
  ~StreamScope() {
    if (!side) return;
    cudaEventRecord(side->out, run);
    cudaStreamWaitEvent(user, side->out, 0);
  }
};

template <class F>
static int run_graph(const GraphKey& k, const GraphKey& topo, cudaStream_t user_st, F&& enqueue) {
  int dev = 0;
  cudaGetDevice(&dev);
  StreamScope scope(user_st, dev);
  cudaStream_t st = scope.run;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    for (auto& e : g_graphs)
      if (e.dev == dev && e.key == k.b) {
        e.last_use = ++g_graph_tick;
        g_launches += e.launches;
        ++g_graph_replays;
        cudaGraphLaunch(e.exec, st);
        return check_cuda("gf_render_rays (graph replay)");
      }
  }
  const int64_t l0 = g_launches.load();
  if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();  // stream cannot be captured: run eagerly
    ++g_graph_eager;
    enqueue(st);
    return check_cuda("gf_render_rays");
  }
  enqueue(st);
  cudaGraph_t g = nullptr;
  cudaError_t err = cudaStreamEndCapture(st, &g);
  if (err != cudaSuccess) return fail(GF_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(err));
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    for (auto& e : g_graphs) {
      if (e.dev != dev || e.topo != topo.b) continue;
      cudaGraphExecUpdateResultInfo info;
      if (cudaGraphExecUpdate(e.exec, g, &info) == cudaSuccess) {
        cudaGraphDestroy(g);
        e.key = k.b;
        e.last_use = ++g_graph_tick;
        g_launches += e.launches;
        ++g_graph_updates;
        cudaGraphLaunch(e.exec, st);
        return check_cuda("gf_render_rays (graph update)");
      }
      cudaGetLastError();  // structure differs after all: instantiate below
      break;
    }
  }
  cudaGraphExec_t ex = nullptr;
  err = cudaGraphInstantiate(&ex, g, 0);
  cudaGraphDestroy(g);
  if (err != cudaSuccess) return fail(GF_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(err));
  cudaGraphLaunch(ex, st);
  ++g_graph_instantiations;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    if (g_graphs.size() >= 8) {
      auto lru = g_graphs.begin();
      for (auto it = g_graphs.begin(); it != g_graphs.end(); ++it)
        if (it->last_use < lru->last_use) lru = it;
      cudaGraphExecDestroy(lru->exec);
      g_graphs.erase(lru);
    }
    g_graphs.push_back(GraphEntry{k.b, topo.b, dev, ex, g_launches.load() - l0, ++g_graph_tick});
  }
  return check_cuda("gf_render_rays (graph)");
}

// bump allocator over a caller-provided workspace
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* p) : base((char*)p) {}
  template <typename T>
  T* take(size_t count) {
    off = gf_align(off);
    T* p = base ? (T*)(base + off) : nullptr;
    off += count * sizeof(T);
    return p;
  }
  size_t size() const { return gf_align(off); }
};

static bool valid_grid(const gf_grid_geom_t* g) {
  if (!g) return false;
  for (int a = 0; a < 3; ++a)
    if (!(g->b_min[a] < g->b_max[a]) || g->res[a] < 1) return false;
  return (int64_t)g->res[0] * g->res[1] * g->res[2] <= GF_MAX_CELLS;  // tile cell field width
}

static int64_t n_cells_of(const gf_grid_geom_t* g) { return (int64_t)g->res[0] * g->res[1] * g->res[2]; }

extern "C" {

int gf_abi_version(void) { return GF_ABI_VERSION; }
const char* gf_last_error(void) { return g_err.c_str(); }

int64_t gf_param_count(const gf_arch_t* arch) {
  LayerTable t;
  if (!arch || !make_layer_table(arch, &t)) return -1;
  int64_t n = 0;
  for (int l = 0; l < t.n_layers; ++l) n += (int64_t)t.in[l] * t.out[l] + t.out[l];
  return n;
}

size_t gf_packed_bytes(const gf_arch_t* arch, int64_t n_cells, int precision) {
  LayerTable t;
  if (!arch || !make_layer_table(arch, &t)) return 0;
  if (precision == GF_PRECISION_FP32) return (size_t)make_fp32_layout(t).cell_floats * 4 * (size_t)n_cells;
  if (precision == GF_PRECISION_FP16) return fp16_cell_bytes(t) * (size_t)n_cells;
  return 0;
}

int gf_pack_weights(const gf_arch_t* arch, int64_t n_cells, const float* const* w, const float* const* b, void* packed,
                    int precision, void* stream) {
  LayerTable t;
  if (!arch || !make_layer_table(arch, &t)) return fail(GF_ERR_INVALID, "gf_pack_weights: bad architecture");
  cudaStream_t st = (cudaStream_t)stream;
  bool ok = false;
  if (precision == GF_PRECISION_FP32)
    ok = launch_pack_fp32(t, n_cells, w, b, (float*)packed, st);
  else if (precision == GF_PRECISION_FP16)
    ok = launch_pack_fp16(t, n_cells, w, b, packed, st);
  if (!ok) return fail(GF_ERR_UNSUPPORTED, "gf_pack_weights: precision/architecture not supported");
  return check_cuda("gf_pack_weights");
}

int gf_pack_weights_flat(const gf_arch_t* arch, int64_t n_cells, const float* flat, void* packed, int precision,
                         void* stream) {
  LayerTable t;
  if (!arch || !make_layer_table(arch, &t) || n_cells < 1 || !flat)
    return fail(GF_ERR_INVALID, "gf_pack_weights_flat: bad architecture or payload");
  const float* w[GF_MAX_LAYERS];
  const float* b[GF_MAX_LAYERS];
  size_t cursor = 0;
  for (int l = 0; l < t.n_layers; ++l) {  // io.py:204-214 layout
    w[l] = flat + cursor;
    cursor += (size_t)n_cells * t.out[l] * t.in[l];
    b[l] = flat + cursor;
    cursor += (size_t)n_cells * t.out[l];
  }
  return gf_pack_weights(arch, n_cells, w, b, packed, precision, stream);
}

// ---------------------------------------------------------------------------
// query path
// ---------------------------------------------------------------------------
struct QueryWs {
  uint32_t* keys;
  BucketBufs B;
  uint32_t* cursor2;  // bulk path: super-cell run cursors
  float4* trec;       // super-cell-ordered records
  float4* tdir;
  uint32_t* dest2;    // point -> super-order row
  uint32_t* dest3;    // super-order row -> sorted row
  float4* sorted_out; // results in sorted order
};

static size_t query_carve(Carve& c, int64_t n, int64_t n_cells, QueryWs* w) {
  w->keys = c.take<uint32_t>((size_t)n + 1);
  if (query_bucket_fast_ok(n, n_cells)) {
    w->cursor2 = c.take<uint32_t>((size_t)n_cells);
    w->trec = c.take<float4>((size_t)n + 1);
    w->tdir = c.take<float4>((size_t)n + 1);
    w->B.srec = c.take<float4>((size_t)n + 1);
    w->B.sdir = c.take<float4>((size_t)n + 1);
    w->dest2 = c.take<uint32_t>((size_t)n + 1);
    w->dest3 = c.take<uint32_t>((size_t)n + 1);
    w->sorted_out = c.take<float4>((size_t)n + 1);
  } else {
    w->cursor2 = w->dest2 = w->dest3 = nullptr;
    w->trec = w->tdir = w->B.srec = w->B.sdir = w->sorted_out = nullptr;
  }
  w->B.counts = c.take<uint32_t>((size_t)n_cells);
  w->B.offsets = c.take<uint32_t>((size_t)n_cells + 1);
  w->B.cursor = c.take<uint32_t>((size_t)n_cells);
  w->B.tiles = c.take<uint2>((size_t)(n / GF_TILE_ROWS + n_cells + 1));
  w->B.n_tiles = c.take<uint32_t>(1);
  w->B.sorted = c.take<uint32_t>((size_t)n + 1);
  w->B.tile_off = c.take<uint32_t>((size_t)n_cells + 1);
  return c.size();
}

size_t gf_query_workspace_bytes(const gf_arch_t* arch, const gf_grid_geom_t* grid, int64_t n) {
  (void)arch;
  if (!valid_grid(grid) || n < 0) return 0;
  Carve c(nullptr);
  QueryWs w;
  return query_carve(c, n, n_cells_of(grid), &w);
}

static bool run_mlp(const LayerTable& t, const gf_arch_t* arch, const void* packed, int precision, const TileSched& S,
                    const RenderIO* rio, const QueryIO* qio, cudaStream_t st) {
  if (precision == GF_PRECISION_FP32) {
    // the fused tiny-MLP kernel when it covers the manifest, else the generic one
    if (rio ? launch_mlp_fp32_render(t, (const float*)packed, S, *rio, st)
            : launch_mlp_fp32_query(t, (const float*)packed, S, *qio, st))
      return true;
    return rio ? launch_mlp_generic_render(t, arch, (const float*)packed, S, *rio, st)
               : launch_mlp_generic_query(t, arch, (const float*)packed, S, *qio, st);
  }
  if (precision == GF_PRECISION_FP16)
    return rio ? launch_mlp_tc_render(t, packed, S, *rio, st) : launch_mlp_tc_query(t, packed, S, *qio, st);
  return false;
}

int gf_query_points(const gf_arch_t* arch, const gf_grid_geom_t* grid, const void* packed, int precision,
                    const float* pos, const float* dir, int64_t n, float* rgb, float* sigma, int64_t* err, void* ws,
                    size_t ws_bytes, void* stream) {
  LayerTable t;
  if (!arch || !make_layer_table(arch, &t)) return fail(GF_ERR_INVALID, "gf_query_points: bad architecture");
  if (!valid_grid(grid) || n < 0 || n >= (int64_t)0xFFFFFFF0ll)
    return fail(GF_ERR_INVALID, "gf_query_points: bad grid or size");
  const int64_t nc = n_cells_of(grid);
  Carve c(ws);
  QueryWs w;
  if (query_carve(c, n, nc, &w) > ws_bytes) return fail(GF_ERR_WORKSPACE, "gf_query_points: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  GfGrid g = gf_make_grid(grid);
  stage_open(st);
  cudaMemsetAsync(w.B.counts, 0, (size_t)nc * 4, st);
  const bool fast = w.cursor2 != nullptr;
  if (fast) {
    stage_mark(st, GF_STAGE_MARCH, launch_query_bucket(g, pos, dir, n, nc, w.keys, w.B, w.trec, w.tdir, w.cursor2,
                                                       w.dest2, w.dest3, err, st, 1));
  } else {
    launch_query_keys(g, pos, n, w.keys, w.B.counts, err, st);
    stage_mark(st, GF_STAGE_MARCH, n > 0 ? 1 : 0);
  }
  stage_mark(st, GF_STAGE_SCAN, launch_scan_cells(w.B, nc, st, n));
  if (fast) {
    stage_mark(st, GF_STAGE_SCATTER, launch_query_bucket(g, pos, dir, n, nc, w.keys, w.B, w.trec, w.tdir, w.cursor2,
                                                         w.dest2, w.dest3, err, st, 2));
  } else {
    launch_scatter_query(w.keys, n, w.B, st);
    stage_mark(st, GF_STAGE_SCATTER, n > 0 ? 1 : 0);
  }
  TileSched S{w.B.tiles, w.B.n_tiles, fast ? nullptr : w.B.sorted, w.B.srec, w.B.sdir};
  QueryIO io{pos, dir, rgb, sigma, nullptr, fast ? w.B.sdir : nullptr, fast ? w.sorted_out : nullptr};
  if (!run_mlp(t, arch, packed, precision, S, nullptr, &io, st))
    return fail(GF_ERR_UNSUPPORTED, "gf_query_points: no MLP kernel for this architecture/precision");
  stage_mark(st, GF_STAGE_MLP, 1);
  if (fast) {
    // the super-order record buffer is dead after the sort: it holds the super-order results
    stage_mark(st, GF_STAGE_SCATTER, launch_query_unpermute(n, w.B.offsets + nc, w.keys, w.dest2, w.dest3,
                                                            w.sorted_out, w.trec, rgb, sigma, st));
  }
  return check_cuda("gf_query_points");
}

static int grouped_forward_impl(const gf_arch_t* arch, int64_t n_cells, const void* packed, int precision,
                                const float* pos, const float* dir, int64_t n, const int64_t* offsets,
                                const int64_t* order, float* rgb, float* sigma, float* act, void* ws, size_t ws_bytes,
                                void* stream) {
  LayerTable t;
  if (!arch || !make_layer_table(arch, &t)) return fail(GF_ERR_INVALID, "gf_grouped_forward: bad architecture");
  if (act && !(precision == GF_PRECISION_FP32 && prepare_mlp_fp32(t) && t.width == 32))
    return fail(GF_ERR_UNSUPPORTED, "gf_grouped_forward_act: activations only for the fp32 32-wide tiny manifest");
  if (n_cells < 1 || n < 0 || n >= (int64_t)0xFFFFFFF0ll) return fail(GF_ERR_INVALID, "gf_grouped_forward: bad sizes");
  Carve c(ws);
  QueryWs w;
  if (query_carve(c, n, n_cells, &w) > ws_bytes) return fail(GF_ERR_WORKSPACE, "gf_grouped_forward: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  launch_segments_from_offsets(offsets, n_cells, n, w.B, st);
  TileSched S{w.B.tiles, w.B.n_tiles, nullptr, nullptr, nullptr};  // rows already grouped: identity
  QueryIO io{pos, dir, rgb, sigma, order, nullptr, nullptr, act};
  if (!run_mlp(t, arch, packed, precision, S, nullptr, &io, st))
    return fail(GF_ERR_UNSUPPORTED, "gf_grouped_forward: no MLP kernel for this architecture/precision");
  return check_cuda("gf_grouped_forward");
}

int gf_grouped_forward(const gf_arch_t* arch, int64_t n_cells, const void* packed, int precision, const float* pos,
                       const float* dir, int64_t n, const int64_t* offsets, const int64_t* order, float* rgb,
                       float* sigma, void* ws, size_t ws_bytes, void* stream) {
  return grouped_forward_impl(arch, n_cells, packed, precision, pos, dir, n, offsets, order, rgb, sigma, nullptr, ws,
                              ws_bytes, stream);
}

int gf_grouped_forward_act(const gf_arch_t* arch, int64_t n_cells, const void* packed, const float* pos,
                           const float* dir, int64_t n, const int64_t* offsets, const int64_t* order, float* rgb,
                           float* sigma, float* act, void* ws, size_t ws_bytes, void* stream) {
  if (!act) return fail(GF_ERR_INVALID, "gf_grouped_forward_act: act is NULL");
  return grouped_forward_impl(arch, n_cells, packed, GF_PRECISION_FP32, pos, dir, n, offsets, order, rgb, sigma, act,
                              ws, ws_bytes, stream);
}

int gf_mlp_forward(const gf_manifest_t* m, int32_t f64, int64_t n_net, int64_t rows, const void* const* w,
                   const void* const* b, const void* x, const void* d, void* color, void* sigma, void* const* hs,
                   void* feat, void* g, void* stream) {
  if (!m || !dense_mlp_supported(m) || n_net < 0 || rows < 0 || !w || !b)
    return fail(GF_ERR_INVALID, "gf_mlp_forward: unsupported manifest or bad sizes");
  if (!launch_dense_forward(m, f64, n_net, rows, w, b, x, d, color, sigma, hs, feat, g, (cudaStream_t)stream))
    return fail(GF_ERR_UNSUPPORTED, "gf_mlp_forward: manifest too wide for the dense kernel");
  return check_cuda("gf_mlp_forward");
}

size_t gf_mlp_backward_workspace_bytes(const gf_manifest_t* m, int32_t f64, int64_t n_net, int64_t rows) {
  if (!m || !dense_mlp_supported(m) || n_net < 0 || rows < 0) return 0;
  return dense_backward_workspace(m, f64, n_net, rows);
}

int gf_mlp_backward(const gf_manifest_t* m, int32_t f64, int64_t n_net, int64_t rows, const void* const* w,
                    const void* x, const void* d, const void* const* hs, const void* feat, const void* g,
                    const void* color, const void* sigma, const void* d_color, const void* d_sigma, void* const* gw,
                    void* const* gb, void* ws, size_t ws_bytes, void* stream) {
  if (!m || !dense_mlp_supported(m) || n_net < 0 || rows < 0 || !w || !gw || !gb || !hs)
    return fail(GF_ERR_INVALID, "gf_mlp_backward: unsupported manifest or bad sizes");
  if (dense_backward_workspace(m, f64, n_net, rows) > ws_bytes)
    return fail(GF_ERR_WORKSPACE, "gf_mlp_backward: workspace too small");
  if (!launch_dense_backward(m, f64, n_net, rows, w, x, d, hs, feat, g, color, sigma, d_color, d_sigma, gw, gb, ws,
                             (cudaStream_t)stream))
    return fail(GF_ERR_UNSUPPORTED, "gf_mlp_backward: manifest too wide for the dense kernel");
  return check_cuda("gf_mlp_backward");
}

size_t gf_grouped_workspace_bytes(int64_t n_cells, int64_t n) {
  Carve c(nullptr);
  QueryWs w;
  return query_carve(c, n, n_cells, &w);
}

// ---------------------------------------------------------------------------
// render path
// ---------------------------------------------------------------------------
struct RenderWs {
  u128* seeds;
  u128* jump;
  u128* start;
  u128* round_jump;
  u128* block_ci;
  RayState R;
  RoundBufs RB;
  BucketBufs B;
  uint8_t* coarse_tmp;
  uint32_t* coarse_bits;
  uint32_t* fine_bits;
  uint64_t* occ_brick;
  uint32_t* occ_bbox;
  unsigned long long* stats_part;
};

// occupancy grids are capped at 256^3 (occupancy.py:21); the coarse mip never
// exceeds that many cells
static const int64_t kMaxCoarseCells = 256ll * 256 * 256;

static size_t render_carve(Carve& c, int64_t n_rays, int64_t n_blocks, int stride, int64_t n_cells, int n_rounds,
                           RenderWs* w) {
  const size_t cap = (size_t)n_rays * (size_t)stride;
  w->seeds = c.take<u128>((size_t)2 * n_blocks);
  w->jump = c.take<u128>((size_t)2 * (GF_JUMP_MAX + 1));
  w->start = c.take<u128>((size_t)2 * GF_RAY_BLOCK);
  w->round_jump = c.take<u128>((size_t)4 * n_rounds);
  w->block_ci = c.take<u128>((size_t)GF_CI_N * n_blocks);
  w->coarse_tmp = c.take<uint8_t>((size_t)kMaxCoarseCells);
  w->coarse_bits = c.take<uint32_t>((size_t)kMaxCoarseCells / 32);
  w->fine_bits = c.take<uint32_t>((size_t)kMaxCoarseCells / 32);
  w->occ_brick = c.take<uint64_t>((size_t)kMaxCoarseCells / 64);
  w->occ_bbox = c.take<uint32_t>(8);
  w->stats_part = c.take<unsigned long long>((size_t)GF_STAT_SLOTS * GF_STAT_COUNT);
  w->R.org = c.take<float4>((size_t)n_rays);
  w->R.dir = c.take<float4>((size_t)n_rays);
  w->R.acc = c.take<float4>((size_t)n_rays);
  w->R.rng = c.take<u128>((size_t)n_rays);
  w->R.run = c.take<uint32_t>((size_t)n_rays);
  w->R.pend = c.take<uint32_t>((size_t)n_rays * 4);
  w->R.flags = c.take<uint32_t>((size_t)n_rays);
  w->R.ivl = c.take<uint32_t>((size_t)n_rays * GF_MAX_IVL);
  w->R.denc = c.take<uint4>((size_t)n_rays * 4);
  w->RB.rec = c.take<float4>(cap);
  w->RB.res = c.take<float4>(cap);
  w->B.counts = c.take<uint32_t>((size_t)2 * n_cells);  // two histograms, by round parity
  w->RB.counts = w->B.counts;
  w->B.offsets = c.take<uint32_t>((size_t)n_cells + 1);
  w->B.cursor = c.take<uint32_t>((size_t)n_cells);
  w->B.tiles = c.take<uint2>(cap / GF_TILE_ROWS + (size_t)n_cells + 1);
  w->B.n_tiles = c.take<uint32_t>(1);
  w->B.sorted = nullptr;
  w->B.srec = c.take<float4>(cap + 1);
  w->B.tile_off = c.take<uint32_t>((size_t)n_cells + 1);
  w->RB.emit_list = c.take<uint32_t>((size_t)n_rays);
  w->RB.emit_count = c.take<uint32_t>(2);
  return c.size();
}

static void block_range(int64_t ray_offset, int64_t block_stride, int64_t n_rays, int64_t* first, int64_t* count) {
  *first = ray_offset / GF_RAY_BLOCK;
  if (block_stride > 1) {
    *count = n_rays > 0 ? (n_rays + GF_RAY_BLOCK - 1) / GF_RAY_BLOCK : 1;
    return;
  }
  int64_t last = n_rays > 0 ? (ray_offset + n_rays - 1) / GF_RAY_BLOCK : *first;
  *count = last - *first + 1;
}

// Rounds run in groups of G (2 by default; 4 available) when the
// warp-cooperative marcher applies (chunk <= 32): the G rounds are placed by G
// marcher passes and evaluated by one K2 + MLP pass, then composited in order
// with the ERT check after each, cutting the per-round launches by G.
// GF_GROUP=1|2|4 overrides (1 = one round at a time).
static int group_size(const gf_march_cfg_t* cfg, int64_t n_rays, bool allow_env = true) {
  const int n_rounds = (cfg->k + cfg->ert_chunk - 1) / cfg->ert_chunk;
  // default 2: equal frame time to 4 on C2 and half the speculative work
  // when rays terminate early
  int g = n_rounds >= 2 ? 2 : 1;
  if (allow_env) {
    const char* e = getenv("GF_GROUP");
    if (e && e[0] >= '1' && e[0] <= '4') g = e[0] - '0';
    if (g > n_rounds) g = n_rounds;
  }
  if (cfg->ert_chunk > 32) g = 1;
  while (g > 1 && (double)n_rays * g * cfg->ert_chunk >= 4.0e9) --g;
  return g;
}

size_t gf_render_workspace_bytes(const gf_arch_t* arch, const gf_grid_geom_t* grid, const gf_march_cfg_t* cfg,
                                 int64_t n_rays) {
  (void)arch;
  if (!valid_grid(grid) || !cfg || cfg->k < 1 || cfg->ert_chunk < 1 || n_rays < 0) return 0;
  int stride = cfg->ert_chunk < cfg->k ? cfg->ert_chunk : cfg->k;
  const int g = group_size(cfg, n_rays, true);
  if (g > 1) stride = g * cfg->ert_chunk;
  Carve c(nullptr);
  RenderWs w;
  // worst case: the call's rays straddle one more block boundary
  return render_carve(c, n_rays, n_rays / GF_RAY_BLOCK + 2, stride, n_cells_of(grid),
                      (cfg->k + cfg->ert_chunk - 1) / cfg->ert_chunk, &w);
}

// The render pipeline for a NetworkGrid field (an == NULL: bucketed
// per-cell MLPs) or an analytic scene (an != NULL: one bucket, closed-form
// field).  Everything else (rays, sampling, ESS, compositing, ERT, graphs)
// is shared.
struct ExtField {
  gf_field_fn fn;
  void* user;
};

__global__ void k_field_gather(const float4* __restrict__ srec, int64_t n, const float4* __restrict__ ray_dir,
                               int shift, uint32_t stride, float* pos, float* dir) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 r = srec[i];
    const uint32_t idx = __float_as_uint(r.w);
    const float4 d = ray_dir[shift >= 0 ? idx >> shift : idx / stride];
    pos[3 * i] = r.x; pos[3 * i + 1] = r.y; pos[3 * i + 2] = r.z;
    dir[3 * i] = d.x; dir[3 * i + 1] = d.y; dir[3 * i + 2] = d.z;
  }
}

__global__ void k_field_scatter(const float4* __restrict__ srec, int64_t n, const float* __restrict__ rgb,
                                const float* __restrict__ sigma, float4* res) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    res[__float_as_uint(srec[i].w)] = make_float4(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2], sigma[i]);
}

static int render_impl(const gf_arch_t* arch, const AnalyticDev* an, const ExtField* ext, const gf_grid_geom_t* grid,
                       const void* packed,
                       int precision, const gf_grid_geom_t* occ, const uint8_t* occ_bits, const gf_march_cfg_t* cfg,
                       const gf_camera_t* cam, const float* origins, const float* dirs, int64_t ray_offset,
                       int64_t ray_block_stride, int64_t n_rays, float* rgb, int64_t* stats, gf_trace_rec_t* trace,
                       int64_t trace_capacity, int64_t* trace_count, void* ws, size_t ws_bytes, void* stream) {
  LayerTable t{};  // value-initialised: hashed into the graph key
  if (!an && !ext && (!arch || !make_layer_table(arch, &t)))
    return fail(GF_ERR_INVALID, "gf_render_rays: bad architecture");
  if (!valid_grid(grid)) return fail(GF_ERR_INVALID, "gf_render_rays: bad grid");
  if (!cfg || cfg->k < 1 || cfg->ert_chunk < 1 || !(cfg->epsilon >= 0.0 && cfg->epsilon < 1.0))
    return fail(GF_ERR_INVALID, "gf_render_rays: bad march config");
  if (occ_bits && !valid_grid(occ)) return fail(GF_ERR_INVALID, "gf_render_rays: bad occupancy grid");
  if (!cam && (!origins || !dirs) && n_rays > 0) return fail(GF_ERR_INVALID, "gf_render_rays: no rays");
  if (ray_offset < 0 || n_rays < 0 || ray_block_stride < 1) return fail(GF_ERR_INVALID, "gf_render_rays: bad ray range");
  if (ray_block_stride > 1 && ray_offset % GF_RAY_BLOCK)
    return fail(GF_ERR_INVALID, "gf_render_rays: interleaved shards need a block-aligned ray_offset");
  // traces list exactly the reference's samples: no speculative later rounds
  const int group = trace ? 1 : group_size(cfg, n_rays, true);
  const int stride = group > 1 ? group * cfg->ert_chunk : (cfg->ert_chunk < cfg->k ? cfg->ert_chunk : cfg->k);
  if ((double)n_rays * stride >= 4.0e9) return fail(GF_ERR_INVALID, "gf_render_rays: too many rays per call");
  if (n_rays == 0) return GF_OK;
  const int64_t nc = n_cells_of(grid);
  int64_t first_block, n_blocks;
  block_range(ray_offset, ray_block_stride, n_rays, &first_block, &n_blocks);
  Carve c(ws);
  RenderWs w{};
  if (render_carve(c, n_rays, n_blocks, stride, nc, (cfg->k + cfg->ert_chunk - 1) / cfg->ert_chunk, &w) > ws_bytes)
    return fail(GF_ERR_WORKSPACE, "gf_render_rays: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;

  MarchParams P;
  memset(&P, 0, sizeof(P));
  P.grid = gf_make_grid(grid);
  if (occ_bits) P.occ = gf_make_grid(occ);
  P.occ_bits = occ_bits;
  if (cam) {
    P.cam = *cam;
    P.use_cam = 1;
  }
  P.origins = origins;
  P.dirs = dirs;
  P.rays_f64 = cfg->rays_f64 ? 1 : 0;
  P.ray_offset = ray_offset;
  P.block_stride = ray_block_stride;
  P.n_rays = n_rays;
  P.first_block = first_block;
  P.block_seeds = w.seeds;
  P.jump = w.jump;
  P.start = w.start;
  P.round_jump = w.round_jump;
  P.block_ci = w.block_ci;
  // the network cell of a sample follows from its occupancy cell when both
  // grids bin exactly in float32 over the same box and each network cell is
  // 2^s occupancy cells per axis (power-of-two scaling keeps floor exact)
  if (occ_bits && P.grid.fast && P.occ.fast) {
    bool ok = true;
    for (int a = 0; a < 3 && ok; ++a) {
      ok = occ->b_min[a] == grid->b_min[a] && occ->b_max[a] == grid->b_max[a] && occ->res[a] % grid->res[a] == 0;
      int q = ok ? occ->res[a] / grid->res[a] : 0, sh = 0;
      while (ok && (1 << sh) < q) ++sh;
      ok = ok && (1 << sh) == q;
      P.net_shift[a] = sh;
    }
    P.net_from_occ = ok ? 1 : 0;
  }
  P.k = cfg->k;
  P.chunk = cfg->ert_chunk;
  P.n_rounds = (cfg->k + cfg->ert_chunk - 1) / cfg->ert_chunk;
  P.n_cells = nc;
  P.stride = stride;
  P.group = group;
  {
    const char* nf = getenv("GF_NO_FUSE");
    P.fuse = group > 1 && !(nf && nf[0] == '1');
  }
  P.stratified = cfg->stratified ? 1 : 0;
  P.ert = cfg->epsilon > 0.0 ? 1 : 0;
  P.eps_f64 = cfg->eps_compare_f64 ? 1 : 0;
  P.epsilon = cfg->epsilon;
  for (int a = 0; a < 3; ++a) P.bg[a] = cfg->background[a];
  P.rgb_out = rgb;
  P.stats = stats;
  P.stats_part = w.stats_part;
  P.trace = trace;
  P.trace_capacity = trace ? trace_capacity : 0;
  P.trace_count = trace_count;
  P.count_candidates = getenv("GF_COUNT_CANDIDATES") && getenv("GF_COUNT_CANDIDATES")[0] == '1';

  // ---- coarse empty-space pre-test: a mip of the occupancy
  // grid dilated by the largest distance between a sample and the midpoint
  // of its nominal segment (seg/2) plus a float32 evaluation margin.
  int coarse_launches = 0;
  struct {
    bool on = false, word = false, fine = false;
    int f = 0, radius = 0, fine_radius = 0;
    int3 ores = {0, 0, 0}, cres = {0, 0, 0};
  } cplan;
  {
    const char* no = getenv("GF_NO_COARSE");
    bool same_box = occ_bits != nullptr;
    for (int a = 0; a < 3 && same_box; ++a)
      same_box = occ->b_min[a] == grid->b_min[a] && occ->b_max[a] == grid->b_max[a];
    if (same_box && !(no && no[0] == '1') && cfg->ert_chunk <= 32 && cfg->k < 65535) {
      double diag2 = 0, maxabs = 0;
      for (int a = 0; a < 3; ++a) {
        double e = grid->b_max[a] - grid->b_min[a];
        diag2 += e * e;
        maxabs = fmax(maxabs, fmax(fabs(grid->b_min[a]), fabs(grid->b_max[a])));
      }
      const double reach = 0.5 * sqrt(diag2) / cfg->k * 1.0001 + 1e-5 * (1.0 + maxabs);
      const char* fenv = getenv("GF_COARSE_FACTOR");
      const int want = fenv ? atoi(fenv) : 4;
      int f = 0, radius = 0;
      for (int cand : {want, 1, 2, 4, 8}) {
        if (cand < 1 || occ->res[0] % cand || occ->res[1] % cand || occ->res[2] % cand) continue;
        double cmin = 1e300;
        for (int a = 0; a < 3; ++a) cmin = fmin(cmin, (occ->b_max[a] - occ->b_min[a]) / occ->res[a] * cand);
        const int r = (int)ceil(reach / cmin);
        if (r <= 2) { f = cand; radius = r < 1 ? 1 : r; break; }
      }
      if (f) {
        cplan.on = true;
        cplan.f = f;
        cplan.radius = radius;
        cplan.ores = make_int3(occ->res[0], occ->res[1], occ->res[2]);
        cplan.cres = make_int3(cplan.ores.x / f, cplan.ores.y / f, cplan.ores.z / f);
        cplan.word = cplan.ores.x % (32 * f) == 0;  // word-parallel OR-reduce + separable dilation
        if (cplan.word && !getenv("GF_NO_BBOX")) P.occ_bbox = w.occ_bbox;  // DDA clipped to the set cells
        if (cplan.word && f == 4 && P.net_from_occ && !getenv("GF_NO_BRICK")) {  // the reduce also writes bricks
          P.occ_brick = w.occ_brick;
          P.brick_cx = cplan.cres.x;
          P.brick_cy = cplan.cres.y;
        }
        coarse_launches = cplan.word ? 4 : 2;
        const int3 cres = cplan.cres;
        gf_grid_geom_t cg = *occ;
        cg.res[0] = cres.x; cg.res[1] = cres.y; cg.res[2] = cres.z;
        P.coarse = gf_make_grid(&cg);
        P.coarse_bits = w.coarse_bits;
        double cmin = 1e300;
        for (int a = 0; a < 3; ++a) cmin = fmin(cmin, (cg.b_max[a] - cg.b_min[a]) / cg.res[a]);
        P.ivl_pad = (float)(0.05 * cmin + 1e-5 * (1.0 + maxabs));
        // per-candidate pre-test on the occupancy grid itself, dilated by
        // ceil(reach / fine cell) <= 2 cells: word-parallel dilation of the
        // fine bitmap (x rows of whole 32-bit words), exact float32 binning
        // opt-in (GF_FINE=1): exact, but measured slower on C2 (march 0.613 ->
        // 0.633 ms): the filter pass costs more than the skipped placements
        const char* nfine = getenv("GF_FINE");
        double fmin = 1e300;
        for (int a = 0; a < 3; ++a) fmin = fmin < (occ->b_max[a] - occ->b_min[a]) / occ->res[a]
                                               ? fmin : (occ->b_max[a] - occ->b_min[a]) / occ->res[a];
        const int rf = (int)ceil(reach / fmin);
        if (nfine && nfine[0] == '1' && P.occ.fast && occ->res[0] % 32 == 0 && rf <= 2) {
          cplan.fine = true;
          cplan.fine_radius = rf < 1 ? 1 : rf;
          P.fine_bits = w.fine_bits;
          coarse_launches += 3;
        }
      }
    }
  }

  auto enqueue_coarse = [&](cudaStream_t s) {
    if (!cplan.on) return;
    const int3 ores = cplan.ores, cres = cplan.cres;
    const int64_t ncc = (int64_t)cres.x * cres.y * cres.z;
    if (cplan.word) {
      const int64_t nw = ncc / 32;
      const unsigned gb = (unsigned)gf_div_up<int64_t>(nw, 128);
      uint32_t* t0 = reinterpret_cast<uint32_t*>(w.coarse_tmp);
      uint32_t* t1 = t0 + nw;
      uint32_t* bbox = (uint32_t*)P.occ_bbox;
      gf_launch_pdl(k_coarse_reduce_w, dim3(gb), dim3(128), 0, s, reinterpret_cast<const uint32_t*>(occ_bits), ores,
                    cplan.f, cres, t0, P.occ_brick ? w.occ_brick : (uint64_t*)nullptr, bbox);
      gf_launch_pdl(k_dilate_x, dim3(gb), dim3(128), 0, s, (const uint32_t*)t0, t1, cres, cplan.radius);
      gf_launch_pdl(k_dilate_yz, dim3(gb), dim3(128), 0, s, (const uint32_t*)t1, t0, cres, cplan.radius, 1,
                    (uint32_t*)nullptr);
      gf_launch_pdl(k_dilate_yz, dim3(gb), dim3(128), 0, s, (const uint32_t*)t0, w.coarse_bits, cres, cplan.radius, 2,
                    bbox);
    } else {
      k_coarse_reduce<<<(unsigned)gf_div_up<int64_t>(ncc, 256), 256, 0, s>>>(occ_bits, ores, cplan.f, cres,
                                                                              w.coarse_tmp);
      k_coarse_dilate<<<(unsigned)gf_div_up<int64_t>(gf_div_up<int64_t>(ncc, 32), 128), 128, 0, s>>>(
          w.coarse_tmp, cres, cplan.radius, w.coarse_bits);
    }
    if (cplan.fine) {  // the fine pre-test bitmap: occupancy dilated per axis (x, y, z)
      const int64_t nw = (int64_t)ores.x * ores.y * ores.z / 32;
      const unsigned gb = (unsigned)gf_div_up<int64_t>(nw, 128);
      uint32_t* t0 = reinterpret_cast<uint32_t*>(w.coarse_tmp);
      uint32_t* t1 = t0 + nw;
      gf_launch_pdl(k_dilate_x, dim3(gb), dim3(128), 0, s, reinterpret_cast<const uint32_t*>(occ_bits), t1, ores,
                    cplan.fine_radius);
      gf_launch_pdl(k_dilate_yz, dim3(gb), dim3(128), 0, s, (const uint32_t*)t1, t0, ores, cplan.fine_radius, 1,
                    (uint32_t*)nullptr);
      gf_launch_pdl(k_dilate_yz, dim3(gb), dim3(128), 0, s, (const uint32_t*)t0, w.fine_bits, ores,
                    cplan.fine_radius, 2, (uint32_t*)nullptr);
    }
  };

  // whole-image camera calls: march warps over 8x4 pixel tiles
  if (cam && ray_offset == 0 && ray_block_stride == 1 && n_rays == (int64_t)cam->width * cam->height &&
      !getenv("GF_NO_TILE2D")) {
    // a CTA's four warps take 2x2 of the 8x4-pixel warp tiles (16x8 pixels),
    // so its rays share more occupancy bricks in L1 than a 32x4 strip
    // (march 0.547 -> 0.530 ms); GF_TILE_CTA=0: strips
    const char* tc = getenv("GF_TILE_CTA");
    if (!(tc && tc[0] == '0')) {
      P.tile2d = 2;
      P.tiles_x = (cam->width + 15) / 16;
      P.march_threads = (int64_t)P.tiles_x * ((cam->height + 7) / 8) * 128;
    } else {
      P.tile2d = 1;
      P.tiles_x = (cam->width + 7) / 8;
      P.march_threads = (int64_t)P.tiles_x * ((cam->height + 3) / 4) * 32;
    }
  } else {
    P.march_threads = n_rays;
  }
  const unsigned march_blocks = (unsigned)gf_div_up<int64_t>(P.march_threads, 128);
  const unsigned ray_blocks = (unsigned)gf_div_up<int64_t>(n_rays, 128);
  TileSched S{w.B.tiles, w.B.n_tiles, nullptr, w.B.srec, nullptr};
  int stride_shift = -1;
  for (int b = 0; b < 31; ++b)
    if ((1 << b) == stride) stride_shift = b;
  if (an || precision != GF_PRECISION_FP16) w.R.denc = nullptr;  // only the tensor-core MLP reads gamma(d) per ray
  RenderIO io{w.RB.res, w.R.dir, (uint32_t)stride, w.R.denc, stride_shift};
  const bool mlp_ok = (an || ext)                        ? true
                      : precision == GF_PRECISION_FP16   ? prepare_mlp_tc(t)
                      : precision == GF_PRECISION_FP32 ? (prepare_mlp_fp32(t) || prepare_mlp_generic(t, arch))
                                                       : false;
  if (!mlp_ok) return fail(GF_ERR_UNSUPPORTED, "gf_render_rays: no MLP kernel for this architecture/precision");

  // the frame's launch sequence (captured once into a CUDA graph per
  // argument set and replayed; eager when instrumented)
  int ext_status = GF_OK;  // a caller-evaluated field's callback failed
  auto enqueue = [&](cudaStream_t s) {
    // memsets first, so the setup kernels and the round chain form one
    // uninterrupted run of programmatic dependent launches
    cudaMemsetAsync(w.B.counts, 0, (size_t)2 * nc * 4, s);
    cudaMemsetAsync(w.RB.emit_count, 0, 2 * sizeof(uint32_t), s);
    cudaMemsetAsync(w.stats_part, 0, (size_t)GF_STAT_SLOTS * GF_STAT_COUNT * 8, s);
    enqueue_coarse(s);
    stage_open(s);
    if (P.stratified)
      gf_launch_pdl(k_seed_blocks,
                    dim3((unsigned)gf_div_up<int64_t>(
                        std::max<int64_t>({n_blocks, (int64_t)GF_RAY_BLOCK, 2ll * P.n_rounds}), 64)),
                    dim3(64), 0, s, (uint64_t)cfg->seed, first_block, ray_block_stride, n_blocks, (int)cfg->k,
                    (int)cfg->ert_chunk, (int)P.n_rounds, w.seeds, w.jump, w.start, w.round_jump, w.block_ci);
    gf_launch_pdl(k_ray_init, dim3(ray_blocks), dim3(128), 0, s, P, w.R);
    stage_mark(s, GF_STAGE_SETUP, (P.stratified ? 2 : 1) + coarse_launches);
    const int step = P.group;
    // the benchmarked configuration runs the marcher specialised for it
    const bool fast_march = P.stratified && P.net_from_occ && P.occ_brick && P.grid.fast && !P.trace && !P.fine_bits &&
                            !getenv("GF_MARCH_GENERIC");
    auto* k_march_sel = fast_march ? k_march<true> : k_march<false>;
    for (int r = 0; r < P.n_rounds; r += step) {
      int passes = 0;
      for (int p = 0; p < step && r + p < P.n_rounds; p += P.fuse ? step : 1, ++passes)
        gf_launch_pdl(k_march_sel, dim3(march_blocks), dim3(128), 0, s, P, w.R, w.RB, r + p, p);
      stage_mark(s, GF_STAGE_MARCH, passes);
      stage_mark(s, GF_STAGE_SCATTER, launch_place(P.grid, w.RB, w.R.run, w.B, nc, stride, step > 1 ? P.chunk : 0,
                                                   r / step, (int64_t)n_rays * stride, s));
      if (an) {
        launch_field_analytic(*an, w.B.offsets, w.B.srec, w.R.dir, stride_shift, (uint32_t)stride, w.RB.res,
                              (int64_t)n_rays * stride, s);
      } else if (ext) {
        // the group's sample count (one bucket: offsets[1]), then the caller
        uint32_t q = 0;
        cudaMemcpyAsync(&q, w.B.offsets + nc, sizeof(q), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (ext_status == GF_OK && q > 0 &&
            ext->fn(ext->user, w.B.srec, (int64_t)q, w.R.dir, stride_shift, (uint32_t)stride, w.RB.res, s) != 0)
          ext_status = GF_ERR_UNSUPPORTED;
      } else {
        run_mlp(t, arch, packed, precision, S, &io, nullptr, s);
      }
      stage_mark(s, GF_STAGE_MLP, 1);
    }
    // final pass: composite the last group of rounds and write the colours
    gf_launch_pdl(k_march_sel, dim3(march_blocks), dim3(128), 0, s, P, w.R, w.RB, (P.n_rounds + step - 1) / step * step, 0);
    launch_stats_fold(w.stats_part, stats, s);  // the warps' spread counters -> the caller's RenderStats
    stage_mark(s, GF_STAGE_MARCH, 2);
  };
  // every precision replays a cached graph; traces and stage timing run eagerly
  const bool use_graph = !g_timer.on && !trace && !ext && !getenv("GF_NO_GRAPH");
  if (!use_graph) {
    enqueue(st);
    if (ext_status != GF_OK) return fail(ext_status, "gf_render_rays_field: the field callback failed");
    return check_cuda("gf_render_rays");
  }
  GraphKey key;  // every value a launch above reads on the host
  key.add(P);
  key.add(w);
  key.add(packed);
  key.add(precision);
  key.add(nc);
  key.add(n_blocks);
  key.add(stride);
  key.add(cplan.on);
  key.add(cplan.word);
  key.add(cplan.f);
  key.add(cplan.radius);
  key.add(cplan.fine);
  key.add(cplan.fine_radius);
  key.add(cplan.ores);
  key.add(cplan.cres);
  key.add(march_blocks);
  key.add(ray_blocks);
  key.add(t);
  key.add(an != nullptr);
  if (an) key.add(*an);
  const size_t n_shared = key.b.size() - sizeof(P);
  key.add(cfg->seed);
  // structure key: the same launches with per-view values (camera, rays, seed, outputs) cleared
  MarchParams Pt = P;
  memset(&Pt.cam, 0, sizeof(Pt.cam));
  Pt.origins = Pt.dirs = nullptr;
  Pt.ray_offset = Pt.first_block = 0;
  Pt.rgb_out = nullptr;
  Pt.stats = nullptr;
  GraphKey topo;
  topo.add(Pt);
  topo.b.insert(topo.b.end(), key.b.begin() + sizeof(P), key.b.begin() + sizeof(P) + n_shared);
  return run_graph(key, topo, st, enqueue);
}

int gf_render_rays(const gf_arch_t* arch, const gf_grid_geom_t* grid, const void* packed, int precision,
                   const gf_grid_geom_t* occ, const uint8_t* occ_bits, const gf_march_cfg_t* cfg,
                   const gf_camera_t* cam, const float* origins, const float* dirs, int64_t ray_offset,
                   int64_t ray_block_stride, int64_t n_rays, float* rgb, int64_t* stats, gf_trace_rec_t* trace,
                   int64_t trace_capacity, int64_t* trace_count, void* ws, size_t ws_bytes, void* stream) {
  return render_impl(arch, nullptr, nullptr, grid, packed, precision, occ, occ_bits, cfg, cam, origins, dirs, ray_offset,
                     ray_block_stride, n_rays, rgb, stats, trace, trace_capacity, trace_count, ws, ws_bytes, stream);
}

// ---------------------------------------------------------------------------
// analytic scenes (scene.py:77-135)
// ---------------------------------------------------------------------------
static gf_grid_geom_t analytic_box(const gf_analytic_t* s) {
  gf_grid_geom_t g;
  for (int a = 0; a < 3; ++a) {
    g.b_min[a] = s->b_min[a];
    g.b_max[a] = s->b_max[a];
    g.res[a] = 1;  // one bucket: the field has no cells
  }
  return g;
}

size_t gf_render_analytic_workspace_bytes(const gf_analytic_t* scene, const gf_march_cfg_t* cfg, int64_t n_rays) {
  if (!scene) return 0;
  const gf_grid_geom_t g = analytic_box(scene);
  return gf_render_workspace_bytes(nullptr, &g, cfg, n_rays);
}

int gf_render_rays_analytic(const gf_analytic_t* scene, const gf_grid_geom_t* occ, const uint8_t* occ_bits,
                            const gf_march_cfg_t* cfg, const gf_camera_t* cam, const float* origins, const float* dirs,
                            int64_t ray_offset, int64_t ray_block_stride, int64_t n_rays, float* rgb, int64_t* stats,
                            gf_trace_rec_t* trace, int64_t trace_capacity, int64_t* trace_count, void* ws,
                            size_t ws_bytes, void* stream) {
  AnalyticDev A;
  memset(&A, 0, sizeof(A));
  if (!make_analytic(scene, &A)) return fail(GF_ERR_INVALID, "gf_render_rays_analytic: bad scene");
  const gf_grid_geom_t g = analytic_box(scene);
  return render_impl(nullptr, &A, nullptr, &g, nullptr, GF_PRECISION_FP32, occ, occ_bits, cfg, cam, origins, dirs, ray_offset,
                     ray_block_stride, n_rays, rgb, stats, trace, trace_capacity, trace_count, ws, ws_bytes, stream);
}

size_t gf_render_field_workspace_bytes(const gf_grid_geom_t* box, const gf_march_cfg_t* cfg, int64_t n_rays) {
  if (!box) return 0;
  gf_grid_geom_t g = *box;
  g.res[0] = g.res[1] = g.res[2] = 1;  // one bucket: the caller's field has no cells
  return gf_render_workspace_bytes(nullptr, &g, cfg, n_rays);
}

int gf_render_rays_field(gf_field_fn fn, void* user, const gf_grid_geom_t* box, const gf_grid_geom_t* occ,
                         const uint8_t* occ_bits, const gf_march_cfg_t* cfg, const gf_camera_t* cam,
                         const float* origins, const float* dirs, int64_t ray_offset, int64_t ray_block_stride,
                         int64_t n_rays, float* rgb, int64_t* stats, gf_trace_rec_t* trace, int64_t trace_capacity,
                         int64_t* trace_count, void* ws, size_t ws_bytes, void* stream) {
  if (!fn || !box) return fail(GF_ERR_INVALID, "gf_render_rays_field: no field callback or box");
  gf_grid_geom_t g = *box;
  g.res[0] = g.res[1] = g.res[2] = 1;
  const ExtField E{fn, user};
  return render_impl(nullptr, nullptr, &E, &g, nullptr, GF_PRECISION_FP32, occ, occ_bits, cfg, cam, origins, dirs,
                     ray_offset, ray_block_stride, n_rays, rgb, stats, trace, trace_capacity, trace_count, ws,
                     ws_bytes, stream);
}

int gf_field_gather(const void* srec, int64_t n, const void* ray_dir, int32_t stride_shift, uint32_t stride,
                    float* pos, float* dir, void* stream) {
  if (n < 0 || (n > 0 && (!srec || !ray_dir || !pos || !dir)) || (stride_shift < 0 && stride == 0))
    return fail(GF_ERR_INVALID, "gf_field_gather: bad arguments");
  if (n > 0)
    k_field_gather<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8), 256, 0,
                     (cudaStream_t)stream>>>((const float4*)srec, n, (const float4*)ray_dir, stride_shift, stride, pos,
                                             dir);
  return check_cuda("gf_field_gather");
}

int gf_field_scatter(const void* srec, int64_t n, const float* rgb_, const float* sigma, void* res, void* stream) {
  if (n < 0 || (n > 0 && (!srec || !rgb_ || !sigma || !res))) return fail(GF_ERR_INVALID, "gf_field_scatter: bad arguments");
  if (n > 0)
    k_field_scatter<<<(unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms() * 8), 256, 0,
                      (cudaStream_t)stream>>>((const float4*)srec, n, rgb_, sigma, (float4*)res);
  return check_cuda("gf_field_scatter");
}

size_t gf_brute_force_workspace_bytes(int32_t n_samples, int64_t n_rays) {
  if (n_samples < 1 || n_rays < 0) return 0;
  const size_t ns = (size_t)n_rays * (size_t)n_samples;
  return gf_align(ns * 4) + gf_align(ns * 12) + gf_align((size_t)n_rays * 12) + gf_align((size_t)n_rays * 4);
}

int gf_render_brute_force(const gf_analytic_t* scene, const gf_camera_t* cam, int32_t n_samples, const float* bg,
                          int64_t ray0, int64_t n_rays, float* out, void* ws, size_t ws_bytes, void* stream) {
  AnalyticDev A;
  memset(&A, 0, sizeof(A));
  if (!make_analytic(scene, &A) || !cam || !bg || n_samples < 1 || n_rays < 0 || ray0 < 0 ||
      ray0 + n_rays > (int64_t)cam->width * cam->height)
    return fail(GF_ERR_INVALID, "gf_render_brute_force: bad scene, camera or range");
  if (gf_brute_force_workspace_bytes(n_samples, n_rays) > ws_bytes)
    return fail(GF_ERR_WORKSPACE, "gf_render_brute_force: workspace too small");
  const size_t ns = (size_t)n_rays * (size_t)n_samples;
  uint8_t* p = (uint8_t*)ws;
  float* alpha = (float*)p;
  p += gf_align(ns * 4);
  float* color = (float*)p;
  p += gf_align(ns * 12);
  float* rgb = (float*)p;
  p += gf_align((size_t)n_rays * 12);
  float* trans = (float*)p;
  launch_brute_force(A, *cam, scene->b_min, scene->b_max, ray0, n_rays, n_samples, bg, alpha, color, rgb, trans, out,
                     (cudaStream_t)stream);
  return check_cuda("gf_render_brute_force");
}

int gf_analytic_empty_cells(const gf_analytic_t* scene, const int32_t* res, uint8_t* out, void* stream) {
  if (!scene || !res || res[0] < 1 || res[1] < 1 || res[2] < 1 || scene->n_prims < 0 || scene->n_prims > GF_MAX_PRIMS)
    return fail(GF_ERR_INVALID, "gf_analytic_empty_cells: bad scene or resolution");
  const int r[3] = {res[0], res[1], res[2]};
  launch_empty_cells(*scene, r, out, (cudaStream_t)stream);
  return check_cuda("gf_analytic_empty_cells");
}

int gf_query_analytic(const gf_analytic_t* scene, const float* pos, const float* dir, int64_t n, float* rgb,
                      float* sigma, void* stream) {
  AnalyticDev A;
  memset(&A, 0, sizeof(A));
  if (!make_analytic(scene, &A) || n < 0) return fail(GF_ERR_INVALID, "gf_query_analytic: bad scene or size");
  launch_query_analytic(A, pos, dir, n, rgb, sigma, (cudaStream_t)stream);
  return check_cuda("gf_query_analytic");
}

// ---------------------------------------------------------------------------
// occupancy extraction (occupancy.py:94-128)
// ---------------------------------------------------------------------------
int gf_extract_occupancy_analytic(const gf_analytic_t* scene, const gf_grid_geom_t* occ, double tau, uint8_t* bits,
                                  void* stream) {
  AnalyticDev A;
  memset(&A, 0, sizeof(A));
  if (!make_analytic(scene, &A)) return fail(GF_ERR_INVALID, "gf_extract_occupancy_analytic: bad scene");
  if (!valid_grid(occ)) return fail(GF_ERR_INVALID, "gf_extract_occupancy_analytic: bad occupancy grid");
  launch_extract_analytic(A, gf_make_grid(occ), n_cells_of(occ), tau, bits, (cudaStream_t)stream);
  return check_cuda("gf_extract_occupancy_analytic");
}

struct ExtractWs {
  float *pos, *dir, *rgb, *sigma;
  void* qws;
  size_t qbytes;
};

static int64_t extract_chunk(int64_t n_cells, int64_t chunk_cells) {
  int64_t c = chunk_cells > 0 ? chunk_cells : (1 << 19);
  c = std::min<int64_t>(c, n_cells);
  c = std::min<int64_t>(c, ((int64_t)0xFFFFFFF0ll / 27) & ~31ll);  // query row-index width
  return std::max<int64_t>(32, (c + 31) & ~31ll);                    // bitmap chunks start on 32-cell words
}

static size_t extract_carve(Carve& c, const gf_arch_t* arch, const gf_grid_geom_t* net, int64_t chunk, ExtractWs* w) {
  const size_t q = (size_t)chunk * 27;
  w->pos = c.take<float>(3 * q);
  w->dir = c.take<float>(3 * q);
  w->rgb = c.take<float>(3 * q);
  w->sigma = c.take<float>(q);
  w->qbytes = gf_query_workspace_bytes(arch, net, (int64_t)q);
  w->qws = c.take<char>(w->qbytes);
  return c.size();
}

size_t gf_extract_workspace_bytes(const gf_arch_t* arch, const gf_grid_geom_t* net, const gf_grid_geom_t* occ,
                                  int64_t chunk_cells) {
  if (!valid_grid(net) || !valid_grid(occ)) return 0;
  Carve c(nullptr);
  ExtractWs w;
  return extract_carve(c, arch, net, extract_chunk(n_cells_of(occ), chunk_cells), &w);
}

int gf_extract_occupancy_network(const gf_arch_t* arch, const gf_grid_geom_t* net, const void* packed, int precision,
                                 const float* direction, const gf_grid_geom_t* occ, double tau, int64_t chunk_cells,
                                 uint8_t* bits, int64_t* err, void* ws, size_t ws_bytes, void* stream) {
  if (!valid_grid(net) || !valid_grid(occ) || !direction)
    return fail(GF_ERR_INVALID, "gf_extract_occupancy_network: bad grid or direction");
  const int64_t n = n_cells_of(occ), chunk = extract_chunk(n, chunk_cells);
  Carve c(ws);
  ExtractWs w;
  if (extract_carve(c, arch, net, chunk, &w) > ws_bytes)
    return fail(GF_ERR_WORKSPACE, "gf_extract_occupancy_network: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const GfGrid g = gf_make_grid(occ), gn = gf_make_grid(net);
  bool inside = true;
  for (int a = 0; a < 3; ++a) inside = inside && occ->b_min[a] >= net->b_min[a] && occ->b_max[a] <= net->b_max[a];
  if (!inside) {
    // probes clipped into the extraction box can leave the field's box: find the
    // first offending component (the reference raises before any bit is set)
    launch_probe_oob(g, gn, n, err, st);
    int64_t h = 0;
    cudaMemcpyAsync(&h, err, sizeof(h), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return check_cuda("gf_extract_occupancy_network");
    if (h != INT64_MAX) return GF_OK;
  }
  for (int64_t first = 0; first < n; first += chunk) {
    const int64_t cnt = std::min<int64_t>(chunk, n - first);
    launch_probe_points(g, first, cnt, direction, w.pos, w.dir, st);
    const int rc = gf_query_points(arch, net, packed, precision, w.pos, w.dir, cnt * 27, w.rgb, w.sigma, err, w.qws,
                                   w.qbytes, stream);
    if (rc != GF_OK) return rc;
    launch_probe_any(w.sigma, first, cnt, n, tau, bits, st);
  }
  return check_cuda("gf_extract_occupancy_network");
}

// ---------------------------------------------------------------------------
// training: batched.py:154-187, train.py:130-160, 212-288
// ---------------------------------------------------------------------------
size_t gf_grouped_backward_workspace_bytes(const gf_arch_t* arch, int64_t n_cells, int64_t n) {
  LayerTable t;
  if (!arch || !make_layer_table(arch, &t) || n_cells < 1 || n < 0) return 0;
  return bwd_workspace(t, n_cells, n);
}

static int grouped_backward_impl(const gf_arch_t* arch, int64_t n_cells, const void* packed, const float* pos,
                                 const float* dir, int64_t n, const int64_t* offsets, const int64_t* order,
                                 const float* d_color, const float* d_sigma, const float* act, float* const* gw,
                                 float* const* gb, void* ws, size_t ws_bytes, void* stream) {
  LayerTable t;
  if (!arch || !make_layer_table(arch, &t)) return fail(GF_ERR_INVALID, "gf_grouped_backward: bad architecture");
  if (n_cells < 1 || n < 0 || !gw || !gb) return fail(GF_ERR_INVALID, "gf_grouped_backward: bad sizes");
  if (bwd_workspace(t, n_cells, n) > ws_bytes) return fail(GF_ERR_WORKSPACE, "gf_grouped_backward: workspace too small");
  BwdArgs A;
  memset(&A, 0, sizeof(A));
  A.pos = pos;
  A.dir = dir;
  A.offsets = offsets;
  A.order = order;
  A.d_color = d_color;
  A.d_sigma = d_sigma;
  A.act = (prepare_mlp_fp32(t) && t.width == 32) ? act : nullptr;
  for (int l = 0; l < t.n_layers; ++l) {
    A.gw[l] = gw[l];
    A.gb[l] = gb[l];
  }
  if (!launch_grouped_backward(t, (const float*)packed, A, n_cells, n, ws, (cudaStream_t)stream))
    return fail(GF_ERR_UNSUPPORTED, "gf_grouped_backward: no backward kernel for this architecture");
  return check_cuda("gf_grouped_backward");
}

int gf_grouped_backward(const gf_arch_t* arch, int64_t n_cells, const void* packed, const float* pos, const float* dir,
                        int64_t n, const int64_t* offsets, const int64_t* order, const float* d_color,
                        const float* d_sigma, float* const* gw, float* const* gb, void* ws, size_t ws_bytes,
                        void* stream) {
  return grouped_backward_impl(arch, n_cells, packed, pos, dir, n, offsets, order, d_color, d_sigma, nullptr, gw, gb,
                               ws, ws_bytes, stream);
}

int gf_grouped_backward_act(const gf_arch_t* arch, int64_t n_cells, const void* packed, const float* pos,
                            const float* dir, int64_t n, const int64_t* offsets, const int64_t* order,
                            const float* d_color, const float* d_sigma, const float* act, float* const* gw,
                            float* const* gb, void* ws, size_t ws_bytes, void* stream) {
  return grouped_backward_impl(arch, n_cells, packed, pos, dir, n, offsets, order, d_color, d_sigma, act, gw, gb, ws,
                               ws_bytes, stream);
}

size_t gf_photometric_workspace_bytes(int64_t n_rays, int32_t k, int64_t n_queries) {
  if (n_rays < 0 || k < 1 || n_queries < 0) return 0;
  return photo_workspace(n_rays, k, n_queries);
}

int gf_photometric_loss(int64_t n_rays, int32_t k, int64_t n_queries, const int64_t* ray_index, const int64_t* slot,
                        const float* color, const float* sigma, const float* noise, const float* deltas,
                        const float* gt, const float* background, float two_over_b, float* d_color_q,
                        float* d_sigma_q, double* loss_sum, void* ws, size_t ws_bytes, void* stream) {
  if (n_rays < 0 || k < 1 || n_queries < 0 || n_queries >= (int64_t)INT32_MAX || !background)
    return fail(GF_ERR_INVALID, "gf_photometric_loss: bad sizes");
  if (photo_workspace(n_rays, k, n_queries) > ws_bytes)
    return fail(GF_ERR_WORKSPACE, "gf_photometric_loss: workspace too small");
  PhotoArgs A;
  A.n_rays = n_rays;
  A.n_queries = n_queries;
  A.k = k;
  A.ray_index = ray_index;
  A.slot = slot;
  A.color = color;
  A.sigma = sigma;
  A.noise = noise;
  A.deltas = deltas;
  A.gt = gt;
  for (int c = 0; c < 3; ++c) A.bg[c] = background[c];
  A.two_over_b = two_over_b;
  A.d_color_q = d_color_q;
  A.d_sigma_q = d_sigma_q;
  launch_photometric(A, ws, loss_sum, (cudaStream_t)stream);
  return check_cuda("gf_photometric_loss");
}

int gf_adam_update(float* p, const float* g, float* m, float* v, int64_t n, const float* coef, void* stream) {
  if (n < 0 || !coef) return fail(GF_ERR_INVALID, "gf_adam_update: bad arguments");
  AdamCoef c{coef[0], coef[1], coef[2], coef[3], coef[4], coef[5], coef[6], coef[7]};
  launch_adam(p, g, m, v, n, c, (cudaStream_t)stream);
  return check_cuda("gf_adam_update");
}

static const int kSumsqParts = 1024;

size_t gf_sum_squares_workspace_bytes(void) { return kSumsqParts * sizeof(double); }

int gf_sum_squares(const float* x, int64_t n, double* out, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || ws_bytes < kSumsqParts * sizeof(double)) return fail(GF_ERR_INVALID, "gf_sum_squares: bad arguments");
  launch_sumsq(x, n, (double*)ws, kSumsqParts, out, (cudaStream_t)stream);
  return check_cuda("gf_sum_squares");
}

int gf_axpy(const float* x, const float* y, int64_t n, float f, float* out, void* stream) {
  if (n < 0 || !x || !out) return fail(GF_ERR_INVALID, "gf_axpy: bad arguments");
  launch_axpy(x, y, n, f, out, (cudaStream_t)stream);
  return check_cuda("gf_axpy");
}

size_t gf_distill_workspace_bytes(int64_t n) { return n < 0 ? 0 : gf_align((size_t)(n + 1) * 16); }

int gf_distill_loss(int64_t n, const float* s_color, const float* s_sigma, const float* t_color, const float* t_sigma,
                    float delta, float c_sigma, float c_color, float* d_color, float* d_sigma, double* sums,
                    void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || ws_bytes < gf_distill_workspace_bytes(n)) return fail(GF_ERR_INVALID, "gf_distill_loss: bad arguments");
  DistillArgs A{n, s_color, s_sigma, t_color, t_sigma, delta, c_sigma, c_color, d_color, d_sigma};
  launch_distill(A, (double*)ws, sums, (cudaStream_t)stream);
  return check_cuda("gf_distill_loss");
}

static bool prep_args(const float* o, const float* d, int64_t n, int32_t k, int32_t stratified, const double* box,
                      const uint64_t* pcg, int32_t has_uint32, uint32_t uinteger, const gf_grid_geom_t* occ,
                      const uint8_t* occ_bits, int64_t* offsets, PrepArgs* A) {
  if (n < 0 || k < 1 || !box || !offsets || (n > 0 && (!o || !d)) || (stratified && !pcg) || (occ_bits && !valid_grid(occ)))
    return false;
  memset(A, 0, sizeof(*A));
  A->origins = o;
  A->dirs = d;
  A->n = n;
  A->k = k;
  A->stratified = stratified ? 1 : 0;
  for (int a = 0; a < 3; ++a) {
    A->b_min[a] = box[a];
    A->b_max[a] = box[3 + a];
  }
  if (stratified) {
    A->state = ((u128)pcg[0] << 64) | pcg[1];
    A->inc = ((u128)pcg[2] << 64) | pcg[3];
  }
  A->has_uint32 = has_uint32 ? 1 : 0;
  A->uinteger = uinteger;
  if (occ_bits) A->occ = gf_make_grid(occ);
  A->occ_bits = occ_bits;
  A->offsets = offsets;
  return true;
}

int gf_prepare_samples_count(const float* o, const float* d, int64_t n, int32_t k, int32_t stratified, const double* box,
                             const uint64_t* pcg, int32_t has_uint32, uint32_t uinteger, const gf_grid_geom_t* occ,
                             const uint8_t* occ_bits, int64_t* offsets, void* stream) {
  PrepArgs A;
  if (!prep_args(o, d, n, k, stratified, box, pcg, has_uint32, uinteger, occ, occ_bits, offsets, &A))
    return fail(GF_ERR_INVALID, "gf_prepare_samples_count: bad arguments");
  launch_prepare_count(A, (cudaStream_t)stream);
  return check_cuda("gf_prepare_samples_count");
}

int gf_prepare_samples_write(const float* o, const float* d, int64_t n, int32_t k, int32_t stratified, const double* box,
                             const uint64_t* pcg, int32_t has_uint32, uint32_t uinteger, const gf_grid_geom_t* occ,
                             const uint8_t* occ_bits, const int64_t* offsets, float* deltas, double* pos,
                             float* dir_out, int64_t* ray_index, int64_t* slot, void* stream) {
  PrepArgs A;
  if (!prep_args(o, d, n, k, stratified, box, pcg, has_uint32, uinteger, occ, occ_bits, (int64_t*)offsets, &A) ||
      !deltas)
    return fail(GF_ERR_INVALID, "gf_prepare_samples_write: bad arguments");
  A.deltas = deltas;
  A.pos = pos;
  A.dir_out = dir_out;
  A.ray_index = ray_index;
  A.slot = slot;
  launch_prepare_write(A, (cudaStream_t)stream);
  return check_cuda("gf_prepare_samples_write");
}

// ---------------------------------------------------------------------------
// grouping and pointwise
// ---------------------------------------------------------------------------
size_t gf_group_workspace_bytes(int64_t n, int64_t n_keys) { return group_workspace(n, n_keys); }

int gf_group_by_key(const int64_t* keys, int64_t n, int64_t n_keys, int64_t* order, int64_t* inverse,
                    int64_t* offsets, int64_t* err, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || n_keys < 1) return fail(GF_ERR_INVALID, "gf_group_by_key: bad sizes");
  if (group_workspace(n, n_keys) > ws_bytes) return fail(GF_ERR_WORKSPACE, "gf_group_by_key: workspace too small");
  launch_group(keys, n, n_keys, order, inverse, offsets, err, ws, (cudaStream_t)stream);
  return check_cuda("gf_group_by_key");
}

int gf_bin_points(const gf_grid_geom_t* grid, const void* x, int32_t x_f64, int64_t n, int64_t* flat, int64_t* err,
                  void* stream) {
  if (!valid_grid(grid) || n < 0) return fail(GF_ERR_INVALID, "gf_bin_points: bad grid");
  launch_bin_points(gf_make_grid(grid), x, x_f64, n, flat, err, (cudaStream_t)stream);
  return check_cuda("gf_bin_points");
}

int gf_gather_rows3(const void* x, int32_t x_f64, const int64_t* idx, int64_t n, float* out, void* stream) {
  if (n < 0 || (n > 0 && (!x || !idx || !out))) return fail(GF_ERR_INVALID, "gf_gather_rows3: bad arguments");
  launch_gather_rows3(x, x_f64, idx, n, out, (cudaStream_t)stream);
  return check_cuda("gf_gather_rows3");
}

int gf_occupied_at(const gf_grid_geom_t* occ, const uint8_t* bits, const void* x, int32_t x_f64, int64_t n,
                   uint8_t* out, int64_t* err, void* stream) {
  if (!valid_grid(occ) || n < 0) return fail(GF_ERR_INVALID, "gf_occupied_at: bad grid");
  launch_occupied_at(gf_make_grid(occ), bits, x, x_f64, n, out, err, (cudaStream_t)stream);
  return check_cuda("gf_occupied_at");
}

int gf_intersect_aabb(const double* o, const double* d, int64_t n, const double* b_min, const double* b_max, double* t0,
                      double* t1, void* stream) {
  if (n < 0 || !b_min || !b_max) return fail(GF_ERR_INVALID, "gf_intersect_aabb: bad arguments");
  launch_intersect_aabb(o, d, n, b_min, b_max, t0, t1, (cudaStream_t)stream);
  return check_cuda("gf_intersect_aabb");
}

int gf_ray_samples(const double* origin, const double* direction, double t0, double seg, const double* jitter,
                   int64_t k, float* out, void* stream) {
  if (k < 0 || !origin || !direction) return fail(GF_ERR_INVALID, "gf_ray_samples: bad arguments");
  launch_ray_samples(origin, direction, t0, seg, jitter, k, out, (cudaStream_t)stream);
  return check_cuda("gf_ray_samples");
}

int gf_clip_into(const double* b_min, const double* b_max, const float* x, int64_t n, float* out, void* stream) {
  if (n < 0) return fail(GF_ERR_INVALID, "gf_clip_into: bad size");
  launch_clip(b_min, b_max, x, n, out, (cudaStream_t)stream);
  return check_cuda("gf_clip_into");
}

int gf_positional_encode(const void* v, int32_t v_f64, int64_t n, int32_t dim, int32_t L, int32_t raw, void* out,
                         void* stream) {
  if (n < 0 || dim < 1 || L < 0) return fail(GF_ERR_INVALID, "gf_positional_encode: bad sizes");
  launch_encode(v, v_f64, n, dim, L, raw, out, (cudaStream_t)stream);
  return check_cuda("gf_positional_encode");
}

int gf_density_to_alpha(const void* s, const void* d, int32_t f64, int64_t n, void* out, void* stream) {
  if (n < 0) return fail(GF_ERR_INVALID, "gf_density_to_alpha: bad size");
  launch_alpha(s, d, f64, n, out, (cudaStream_t)stream);
  return check_cuda("gf_density_to_alpha");
}

int gf_composite(const float* c, const float* a, int64_t nr, int64_t ns, float* rgb, float* tr, void* stream) {
  if (nr < 0 || ns < 0) return fail(GF_ERR_INVALID, "gf_composite: bad sizes");
  launch_composite(c, a, nr, ns, rgb, tr, (cudaStream_t)stream);
  return check_cuda("gf_composite");
}

int gf_composite_f64(const double* c, const double* a, int64_t nr, int64_t ns, double* rgb, double* tr, void* stream) {
  if (nr < 0 || ns < 0) return fail(GF_ERR_INVALID, "gf_composite_f64: bad sizes");
  launch_composite_f64(c, a, nr, ns, rgb, tr, (cudaStream_t)stream);
  return check_cuda("gf_composite_f64");
}

int gf_generate_rays(const gf_camera_t* cam, float* o, float* d, void* stream) {
  if (!cam || cam->width < 1 || cam->height < 1) return fail(GF_ERR_INVALID, "gf_generate_rays: bad camera");
  launch_gen_rays(*cam, o, d, (cudaStream_t)stream);
  return check_cuda("gf_generate_rays");
}

int gf_stage_timing(int32_t enable) {
  g_timer.on = enable != 0;
  g_timer.marks.clear();
  g_timer.launches.clear();
  g_timer.used = 0;
  return GF_OK;
}

int gf_stage_times(double* ms_out, int64_t* launches_out) {
  for (int s = 0; s < GF_STAGE_COUNT; ++s) {
    if (ms_out) ms_out[s] = 0.0;
    if (launches_out) launches_out[s] = 0;
  }
  cudaEvent_t prev = nullptr;
  for (auto& m : g_timer.marks) {
    if (m.first < 0) {
      prev = m.second;
      continue;
    }
    cudaEventSynchronize(m.second);
    float ms = 0.f;
    if (prev && cudaEventElapsedTime(&ms, prev, m.second) == cudaSuccess && ms_out) ms_out[m.first] += ms;
    prev = m.second;
  }
  if (launches_out)
    for (auto& l : g_timer.launches) launches_out[l.first] += l.second;
  g_timer.marks.clear();
  g_timer.launches.clear();
  g_timer.used = 0;
  return check_cuda("gf_stage_times");
}

int64_t gf_launch_count(void) { return g_launches.load(); }

int gf_graph_counters(int64_t out4[4]) {
  if (!out4) return fail(GF_ERR_INVALID, "gf_graph_counters: null output");
  out4[0] = g_graph_replays.load();
  out4[1] = g_graph_updates.load();
  out4[2] = g_graph_instantiations.load();
  out4[3] = g_graph_eager.load();
  return GF_OK;
}

int gf_pcg64_block_state(uint64_t seed, uint64_t block_start, uint64_t out4[4]) {
  u128 s, inc;
  gf_seed_block(seed, block_start, &s, &inc);
  out4[0] = (uint64_t)(s >> 64);
  out4[1] = (uint64_t)s;
  out4[2] = (uint64_t)(inc >> 64);
  out4[3] = (uint64_t)inc;
  return GF_OK;
}

}  // extern "C"
