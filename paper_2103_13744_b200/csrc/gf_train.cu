// Training kernels: the grouped backward pass of the
// per-cell tiny MLPs, the photometric loss with its compositing gradients,
// and the optimizer step.
//
// Reference:
//   batched.py:154-187  grouped_backward (per-cell parameter gradients)
//   mlp.py:269-316      backward (exact gradients of sum(dc*color + ds*sigma))
//   train.py:212-288    photometric_loss_and_grads (dense compositing, the
//                       rest-of-ray recurrence for d alpha, loss in float64)
//   train.py:130-143    adam_update;  train.py:146-160 regularization_term
//
// Everything is float32 SIMT (the reference's arithmetic type); results match
// the reference within a stated tolerance, not bit for bit, because numpy's
// sgemm and pairwise sums associate differently.  Every reduction here has a
// fixed order (one owner thread per parameter, one thread per ray), so the
// device results are deterministic run to run.
#include "gf_mlp_simt.cuh"
#include "gf_train.cuh"

namespace gf {

// ---------------------------------------------------------------------------
// grouped backward: one CTA per cell, TR rows per tile.  Phase A: four lanes
// per row (a row's lanes are adjacent in one warp and sync with __syncwarp)
// recompute the fp32 forward and run the backward data pass, each lane owning
// a quarter of every layer's outputs (or, for the transposed products, of the
// inputs); activations and deltas go to shared memory.  Phase B: every thread
// owns a fixed set of parameters and sums dz[o] * in[i] over the tile's rows
// in row order.  Each value is produced by one thread in a fixed order, so
// the result is deterministic.
// ---------------------------------------------------------------------------
template <int W>
struct BwdShape {
  static constexpr int P = 63, D = 27;
  // per-row shared-memory vectors (floats)
  static constexpr int X = 0;             // gamma(x)            P
  static constexpr int H0 = X + P;        // h0                  W
  static constexpr int H1 = H0 + W;       // h1                  W
  static constexpr int CAT = H1 + W;      // [feat, gamma(d)]    W + D
  static constexpr int G = CAT + W + D;   // g                   W
  static constexpr int DZ0 = G + W;       // dz trunk0           W
  static constexpr int DZ1 = DZ0 + W;     // dz trunk1           W
  static constexpr int DZS = DZ1 + W;     // dz density          1
  static constexpr int DZF = DZS + 1;     // dz feature          W
  static constexpr int DZD = DZF + W;     // dz direction        W
  static constexpr int DZC = DZD + W;     // dz color            3
  static constexpr int SIG = DZC + 3;     // sigma               1
  static constexpr int ZC = SIG + 1;      // color logits        3
  static constexpr int END = ZC + 3;
  static constexpr int LD = END | 1;      // odd row stride: conflict-free per-row access
  static constexpr int LANES = 4;         // threads per row in phase A
  static constexpr int TR = 32;           // rows per tile
  static constexpr int THREADS = TR * LANES;
  // W = 32: the four wide forward layers also staged transposed (wt[i][o],
  // row stride OS = W + 4: 16-byte rows, 4-way conflicts on the one-time fill)
  static constexpr bool WT = W == 32;
  static constexpr int OS = W + 4;
  static constexpr int T0 = 0, T1 = T0 + P * OS, T3 = T1 + W * OS, T4 = T3 + W * OS;
  static constexpr int WT_FLOATS = WT ? T4 + (W + D) * OS : 0;
  // ... and the rest of the cell's parameters (biases, density and colour
  // weights) in a small block; the natural copy of the wide layers is not kept
  static constexpr int WP = (W + 3) & ~3;
  static constexpr int SB0 = 0, SB1 = W, SB2 = 2 * W, SB3 = 2 * W + 4, SB4 = 3 * W + 4, SB5 = 4 * W + 4;
  static constexpr int SWD = 4 * W + 8, SWC = 5 * W + 8;
  static constexpr int SM_FLOATS = WT ? SWC + 3 * WP : 0;
  __host__ __device__ static constexpr int sb(int l) {
    return l == 0 ? SB0 : (l == 1 ? SB1 : (l == 2 ? SB2 : (l == 3 ? SB3 : (l == 4 ? SB4 : SB5))));
  }
  static constexpr int N_LAYERS = 6;
  // manifest order (mlp.py:73-84): trunk0, trunk1, density, feature, direction, color
  __host__ __device__ static constexpr int in_dim(int l) { return l == 0 ? P : (l == 4 ? W + D : W); }
  __host__ __device__ static constexpr int out_dim(int l) { return l == 2 ? 1 : (l == 5 ? 3 : W); }
  __host__ __device__ static constexpr int in_off(int l) {
    return l == 0 ? X : (l == 1 ? H0 : (l == 2 || l == 3 ? H1 : (l == 4 ? CAT : G)));
  }
  __host__ __device__ static constexpr int dz_off(int l) {
    return l == 0 ? DZ0 : (l == 1 ? DZ1 : (l == 2 ? DZS : (l == 3 ? DZF : (l == 4 ? DZD : DZC))));
  }
  __host__ __device__ static constexpr int count(int l) { return out_dim(l) * in_dim(l) + out_dim(l); }
  static constexpr int TOTAL = count(0) + count(1) + count(2) + count(3) + count(4) + count(5);
};

// outputs [o0, o0 + NO) of relu?(W in + b) for one row; input vector read
// from shared memory into registers once
template <int IN, int INP, int NO, bool RELU>
__device__ __forceinline__ void dense_part(const float* __restrict__ w, const float* __restrict__ b,
                                           const float* in_s, int o0, float* out_s) {
  float in[IN];
#pragma unroll
  for (int i = 0; i < IN; ++i) in[i] = in_s[i];
#pragma unroll 2
  for (int oo = 0; oo < NO; ++oo) {
    const int o = o0 + oo;
    const float4* wr = reinterpret_cast<const float4*>(w + o * INP);
    float acc = 0.f;
#pragma unroll
    for (int i4 = 0; i4 < INP / 4; ++i4) {
      const float4 q = wr[i4];
      if (4 * i4 + 0 < IN) acc = fmaf(in[4 * i4 + 0], q.x, acc);
      if (4 * i4 + 1 < IN) acc = fmaf(in[4 * i4 + 1], q.y, acc);
      if (4 * i4 + 2 < IN) acc = fmaf(in[4 * i4 + 2], q.z, acc);
      if (4 * i4 + 3 < IN) acc = fmaf(in[4 * i4 + 3], q.w, acc);
    }
    const float z = __fadd_rn(acc, b[o]);
    out_s[o] = RELU ? fmaxf(z, 0.f) : z;
  }
}

// dense_part with the layer's weights transposed in shared memory (wt[i][o],
// OUT floats per input): each lane keeps NO independent accumulators and
// streams the input once, instead of NO serial FMA chains over a register
// copy of the input.  Same per-output arithmetic (fmaf over i ascending from
// 0, then + b), so the values are identical.
template <int IN, int OS, int NO, bool RELU>
__device__ __forceinline__ void dense_part_t(const float* __restrict__ wt, const float* __restrict__ b,
                                             const float* in_s, int o0, float* out_s) {
  float acc[NO];
#pragma unroll
  for (int oo = 0; oo < NO; ++oo) acc[oo] = 0.f;
#pragma unroll 4
  for (int i = 0; i < IN; ++i) {
    const float x = in_s[i];
    const float4* wr = reinterpret_cast<const float4*>(wt + i * OS + o0);
#pragma unroll
    for (int v = 0; v < NO / 4; ++v) {
      const float4 q = wr[v];
      acc[4 * v + 0] = fmaf(x, q.x, acc[4 * v + 0]);
      acc[4 * v + 1] = fmaf(x, q.y, acc[4 * v + 1]);
      acc[4 * v + 2] = fmaf(x, q.z, acc[4 * v + 2]);
      acc[4 * v + 3] = fmaf(x, q.w, acc[4 * v + 3]);
    }
  }
#pragma unroll
  for (int oo = 0; oo < NO; ++oo) {
    const float z = __fadd_rn(acc[oo], b[o0 + oo]);
    out_s[o0 + oo] = RELU ? fmaxf(z, 0.f) : z;
  }
}

// dx[i] = sum_o dz[o] * W[o][i] for i in [i0, i0 + NI)  (matmul(dz, W), mlp.py:294-297)
template <int NI, int INP, int OUT>
__device__ __forceinline__ void dense_t_part(const float* __restrict__ w, const float* dz_s, int i0, float* dx) {
#pragma unroll
  for (int i = 0; i < NI; ++i) dx[i] = 0.f;
#pragma unroll 4
  for (int o = 0; o < OUT; ++o) {
    const float g = dz_s[o];
    const float* wr = w + o * INP + i0;
#pragma unroll
    for (int i = 0; i < NI; ++i) dx[i] = fmaf(g, wr[i], dx[i]);
  }
}

// dense_t_part over weights transposed in shared memory (wt[i][o], row
// stride OS): lane q owns inputs i = q + 4v (v < NI), so the four lanes of a
// row read four different bank groups; dx[v] = sum_o dz[o] * W[o][i] as an
// fmaf chain over o ascending from 0, like dense_t_part.
template <int NI, int OUT, int OS>
__device__ __forceinline__ void dense_t_part_t(const float* __restrict__ wt, const float* dz_s, int q, float* dx) {
#pragma unroll
  for (int v = 0; v < NI; ++v) dx[v] = 0.f;
#pragma unroll 2
  for (int o = 0; o < OUT; o += 4) {
    const float g0 = dz_s[o], g1 = dz_s[o + 1], g2 = dz_s[o + 2], g3 = dz_s[o + 3];
#pragma unroll
    for (int v = 0; v < NI; ++v) {
      const float4 w = *reinterpret_cast<const float4*>(wt + (q + 4 * v) * OS + o);
      dx[v] = fmaf(g0, w.x, dx[v]);
      dx[v] = fmaf(g1, w.y, dx[v]);
      dx[v] = fmaf(g2, w.z, dx[v]);
      dx[v] = fmaf(g3, w.w, dx[v]);
    }
  }
}

// work plan: every cell's rows split into chunks of GF_BWD_CHUNK rows (one CTA
// each, so a crowded cell does not serialise the kernel); chunk k's partial
// sums land in scratch row k and k_bwd_reduce adds a cell's chunks in order
#define GF_BWD_CHUNK 256

__global__ void __launch_bounds__(1024) k_bwd_plan(const int64_t* __restrict__ offsets, int64_t n_cells, uint2* chunks,
                                                   uint32_t* chunk_off, uint32_t* n_chunks) {
  __shared__ uint32_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t per = (n_cells + 1023) / 1024, c0 = (int64_t)tid * per;
  uint32_t local = 0;
  for (int64_t c = c0; c < c0 + per && c < n_cells; ++c)
    local += (uint32_t)((offsets[c + 1] - offsets[c] + GF_BWD_CHUNK - 1) / GF_BWD_CHUNK);
  uint32_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  uint32_t base = (wid ? wsum[wid - 1] : 0u) + x - local;
  for (int64_t c = c0; c < c0 + per && c < n_cells; ++c) {
    chunk_off[c] = base;
    const uint32_t nch = (uint32_t)((offsets[c + 1] - offsets[c] + GF_BWD_CHUNK - 1) / GF_BWD_CHUNK);
    for (uint32_t j = 0; j < nch; ++j) chunks[base + j] = make_uint2((uint32_t)c, j);
    base += nch;
  }
  if (tid == 1023) {
    chunk_off[n_cells] = base;
    *n_chunks = base;
  }
}

// chunk sums -> reference-layout gradients; cells without rows get zeros
template <int W>
__global__ void __launch_bounds__(256) k_bwd_reduce(const float* __restrict__ scratch,
                                                    const uint32_t* __restrict__ chunk_off, int64_t n_cells,
                                                    BwdArgs A) {
  using S = BwdShape<W>;
  const int64_t n = n_cells * S::TOTAL;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = e / S::TOTAL;
    const int p = (int)(e % S::TOTAL);
    float acc = 0.f;
    const uint32_t k0 = chunk_off[cell], k1 = chunk_off[cell + 1];
    for (uint32_t k = k0; k < k1; ++k) acc = k == k0 ? scratch[(size_t)k * S::TOTAL + p]
                                                    : __fadd_rn(acc, scratch[(size_t)k * S::TOTAL + p]);
    int l = 0, qq = p;
    while (qq >= S::count(l)) qq -= S::count(l++);
    const int in = S::in_dim(l), out = S::out_dim(l);
    if (qq >= out * in) A.gb[l][cell * out + (qq - out * in)] = acc;
    else A.gw[l][(cell * out + qq / in) * in + qq % in] = acc;
  }
}

// Phase B of one layer: gw[o][i] = sum_rows dz[o] * in[i] (fmaf chain in row
// order from 0) and gb[o] = sum_rows dz[o] (fadd chain), accumulated into the
// chunk's partial sums (first tile stores).  Threads own 4x4 (o, i) blocks:
// 8 shared loads per 16 FMAs instead of 2 per FMA, and no per-parameter index
// arithmetic; the per-parameter arithmetic sequence is unchanged.
template <class S, int OUT, int IN, int DZ, int INO, int NT>
__device__ __forceinline__ void bwd_layer_sums(const float* srow, int n_in, float* part, bool first, int tid, int& u) {
  constexpr int LD = S::LD, OB = (OUT + 3) / 4, IB = (IN + 3) / 4, NB = OB * IB;
  // units: NB weight blocks, then OB bias quads; unit u of the whole tile is
  // handled by thread u % NT (u runs over every layer's units in order)
  for (int b = (tid - u % NT + NT) % NT; b < NB + OB; b += NT) {
    if (b < NB) {
      const int o0 = (b / IB) * 4, i0 = (b % IB) * 4;
      float acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = 0.f;
      const float* dzp = srow + DZ + o0;
      const float* inp = srow + INO + i0;
      // later tiles add to the chunk's partial sums: their loads are issued
      // before the row loop so the global latency overlaps it
      float old[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          old[a][c] = (!first && o0 + a < OUT && i0 + c < IN) ? part[(o0 + a) * IN + i0 + c] : 0.f;
      for (int rr = 0; rr < n_in; ++rr) {
        float dz[4], in[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) dz[a] = (o0 + a < OUT) ? dzp[rr * LD + a] : 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) in[c] = (i0 + c < IN) ? inp[rr * LD + c] : 0.f;
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[a][c] = fmaf(dz[a], in[c], acc[a][c]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (o0 + a < OUT && i0 + c < IN) part[(o0 + a) * IN + i0 + c] = first ? acc[a][c] : __fadd_rn(old[a][c], acc[a][c]);
    } else {
      const int o0 = (b - NB) * 4;
      float acc[4] = {0.f, 0.f, 0.f, 0.f}, old[4];
      const float* dzp = srow + DZ + o0;
#pragma unroll
      for (int a = 0; a < 4; ++a) old[a] = (!first && o0 + a < OUT) ? part[OUT * IN + o0 + a] : 0.f;
      for (int rr = 0; rr < n_in; ++rr)
#pragma unroll
        for (int a = 0; a < 4; ++a)
          if (o0 + a < OUT) acc[a] = __fadd_rn(acc[a], dzp[rr * LD + a]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (o0 + a < OUT) part[OUT * IN + o0 + a] = first ? acc[a] : __fadd_rn(old[a], acc[a]);
    }
  }
  u += NB + OB;
}

template <class S, int NT>
__device__ __forceinline__ void bwd_param_sums(const float* srow, int n_in, float* part, bool first, int tid) {
  int u = 0;  // running unit count: spreads the layers' remainders over different threads
  bwd_layer_sums<S, S::out_dim(0), S::in_dim(0), S::dz_off(0), S::in_off(0), NT>(srow, n_in, part, first, tid, u);
  part += S::count(0);
  bwd_layer_sums<S, S::out_dim(1), S::in_dim(1), S::dz_off(1), S::in_off(1), NT>(srow, n_in, part, first, tid, u);
  part += S::count(1);
  bwd_layer_sums<S, S::out_dim(2), S::in_dim(2), S::dz_off(2), S::in_off(2), NT>(srow, n_in, part, first, tid, u);
  part += S::count(2);
  bwd_layer_sums<S, S::out_dim(3), S::in_dim(3), S::dz_off(3), S::in_off(3), NT>(srow, n_in, part, first, tid, u);
  part += S::count(3);
  bwd_layer_sums<S, S::out_dim(4), S::in_dim(4), S::dz_off(4), S::in_off(4), NT>(srow, n_in, part, first, tid, u);
  part += S::count(4);
  bwd_layer_sums<S, S::out_dim(5), S::in_dim(5), S::dz_off(5), S::in_off(5), NT>(srow, n_in, part, first, tid, u);
}

template <int W>
__global__ void __launch_bounds__(BwdShape<W>::THREADS) k_grouped_backward(const float* __restrict__ packed,
                                                                           Fp32Layout L, BwdArgs A,
                                                                           const uint2* __restrict__ chunks,
                                                                           const uint32_t* __restrict__ n_chunks,
                                                                           float* scratch) {
  using S = BwdShape<W>;
  constexpr int P = S::P, D = S::D, TR = S::TR, LD = S::LD, NT = S::THREADS, Q = W / S::LANES;
  constexpr int PP = (P + 3) & ~3, WP = (W + 3) & ~3, DP = (W + D + 3) & ~3;
  extern __shared__ float4 smem4[];
  // WT: [transposed wide layers | small block | rows]; else [packed cell | rows]
  float* sw = reinterpret_cast<float*>(smem4);
  float* swt = sw;
  float* ssm = sw + S::WT_FLOATS;
  float* srow = S::WT ? ssm + S::SM_FLOATS : sw + L.cell_floats;  // TR rows x LD floats
  if (blockIdx.x >= *n_chunks) return;
  const uint2 ch = chunks[blockIdx.x];
  const int64_t cell = ch.x;
  const int tid = threadIdx.x;
  const int r = tid / S::LANES, q = tid % S::LANES;  // row of the tile, lane within the row
  const float* gsrc = packed + (size_t)cell * L.cell_floats;
  if constexpr (S::WT) {
    // asynchronous 4-byte global -> shared copies (cp.async): every element
    // is in flight at once instead of one load -> store round trip each
    auto async4 = [&](float* dst, const float* src) {
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
    };
    auto transpose = [&](int l, int in, int t_off) {
      const float* w = gsrc + L.w_off[l];
      const int inp = (in + 3) & ~3;
      for (int e = tid; e < in * W; e += NT) {
        const int o = e / in, i = e - o * in;  // contiguous reads of w[o][*]
        async4(swt + t_off + i * S::OS + o, w + o * inp + i);
      }
    };
    transpose(0, P, S::T0);
    transpose(1, W, S::T1);
    transpose(3, W, S::T3);
    transpose(4, W + D, S::T4);
    auto copy = [&](int dst, int src, int n) {
      for (int j = tid; j < n; j += NT) async4(ssm + dst + j, gsrc + src + j);
    };
#pragma unroll
    for (int l = 0; l < 6; ++l) copy(S::sb(l), L.b_off[l], S::out_dim(l));
    copy(S::SWD, L.w_off[2], W);
    copy(S::SWC, L.w_off[5], 3 * WP);
    asm volatile("cp.async.wait_all;" ::: "memory");  // the tile loop's __syncthreads publishes them
  } else {
    const float4* src = reinterpret_cast<const float4*>(gsrc);
    for (int j = tid; j < L.cell_floats / 4; j += NT) smem4[j] = __ldg(src + j);
  }
  auto bias = [&](int l) -> const float* {
    if constexpr (S::WT) return ssm + S::sb(l);
    else return sw + L.b_off[l];
  };
  const float* w_den = S::WT ? ssm + S::SWD : sw + L.w_off[2];
  const float* w_col = S::WT ? ssm + S::SWC : sw + L.w_off[5];
  const int64_t r0 = A.offsets[cell] + (int64_t)ch.y * GF_BWD_CHUNK;
  const int64_t r1 = min(A.offsets[cell + 1], r0 + (int64_t)GF_BWD_CHUNK);
  const int n_tiles = (int)((r1 - r0 + TR - 1) / TR);  // >= 1: chunks hold rows
  float* part = scratch + (size_t)blockIdx.x * S::TOTAL;
  for (int t = 0; t < n_tiles; ++t) {
    const int64_t first = r0 + (int64_t)t * TR;
    const int n_in = (int)(r1 - first < (int64_t)TR ? r1 - first : (int64_t)TR);  // <= 0 for an empty cell
    __syncthreads();
    // ---------------- phase A (every lane reaches every __syncwarp)
    const bool on = r < n_in;
    float* s = srow + r * LD;
    const int64_t row = first + r;
    const int64_t src = on ? (A.order ? A.order[row] : row) : 0;  // upstream gradients arrive in query order
    if (on) {
      // gamma(x): lane q encodes octaves q, q+4, q+8; gamma(d): octave q (core.py:132-152)
      float x[3], d[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        x[a] = A.pos[3 * row + a];
        d[a] = A.dir[3 * row + a];
      }
      if (q == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          s[S::X + a] = x[a];
          s[S::CAT + W + a] = d[a];
        }
      }
      for (int k = q; k < 10; k += S::LANES) {
        const float f = __int_as_float(0x40490FDB + (k << 23));  // fl32(pi) * 2^k == fl32(2^k pi)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          float sv, cv;
          sincosf(__fmul_rn(x[a], f), &sv, &cv);
          s[S::X + 3 + 6 * k + a] = sv;
          s[S::X + 6 + 6 * k + a] = cv;
        }
      }
      {
        const int k = q;  // 4 direction octaves, one per lane
        const float f = __int_as_float(0x40490FDB + (k << 23));
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          float sv, cv;
          sincosf(__fmul_rn(d[a], f), &sv, &cv);
          s[S::CAT + W + 3 + 6 * k + a] = sv;
          s[S::CAT + W + 6 + 6 * k + a] = cv;
        }
      }
    }
    __syncwarp();
    // ---- forward (mlp.py:238-266)
    if constexpr (S::WT) {
      if (on) dense_part_t<P, S::OS, Q, true>(swt + S::T0, bias(0), s + S::X, q * Q, s + S::H0);
      __syncwarp();
      if (on) dense_part_t<W, S::OS, Q, true>(swt + S::T1, bias(1), s + S::H0, q * Q, s + S::H1);
      __syncwarp();
      if (on) {
        dense_part_t<W, S::OS, Q, false>(swt + S::T3, bias(3), s + S::H1, q * Q, s + S::CAT);  // feature
        if (q == 0) dense_part<W, WP, 1, true>(w_den, bias(2), s + S::H1, 0, s + S::SIG);
      }
      __syncwarp();
      if (on) dense_part_t<W + D, S::OS, Q, true>(swt + S::T4, bias(4), s + S::CAT, q * Q, s + S::G);
      __syncwarp();
    } else {
      if (on) dense_part<P, PP, Q, true>(sw + L.w_off[0], sw + L.b_off[0], s + S::X, q * Q, s + S::H0);
      __syncwarp();
      if (on) dense_part<W, WP, Q, true>(sw + L.w_off[1], sw + L.b_off[1], s + S::H0, q * Q, s + S::H1);
      __syncwarp();
      if (on) {
        dense_part<W, WP, Q, false>(sw + L.w_off[3], sw + L.b_off[3], s + S::H1, q * Q, s + S::CAT);  // feature
        if (q == 0) dense_part<W, WP, 1, true>(sw + L.w_off[2], sw + L.b_off[2], s + S::H1, 0, s + S::SIG);
      }
      __syncwarp();
      if (on) dense_part<W + D, DP, Q, true>(sw + L.w_off[4], sw + L.b_off[4], s + S::CAT, q * Q, s + S::G);
      __syncwarp();
    }
    // ---- backward (mlp.py:291-316)
    if (on && q < 3) {
      dense_part<W, WP, 1, false>(w_col, bias(5), s + S::G, q, s + S::ZC);  // logit q
      const float col = sigmoid_split(s[S::ZC + q]);
      s[S::DZC + q] = __fmul_rn(__fmul_rn(A.d_color[3 * src + q], col), __fsub_rn(1.0f, col));
    }
    if (on && q == 3) s[S::DZS] = s[S::SIG] > 0.f ? A.d_sigma[src] : 0.f;  // d_sigma * (sigma > 0)
    __syncwarp();
    if (on) {  // dz_dir = (dz_color W_color) * (g > 0)
      float dv[Q];
      dense_t_part<Q, WP, 3>(w_col, s + S::DZC, q * Q, dv);
#pragma unroll
      for (int i = 0; i < Q; ++i) s[S::DZD + q * Q + i] = s[S::G + q * Q + i] > 0.f ? dv[i] : 0.f;
    }
    __syncwarp();
    if constexpr (S::WT) {
      // transposed wide layers: lane q owns inputs q + 4v
      if (on) {  // dfeat = first W columns of dz_dir W_direction
        float dv[Q];
        dense_t_part_t<Q, W, S::OS>(swt + S::T4, s + S::DZD, q, dv);
#pragma unroll
        for (int v = 0; v < Q; ++v) s[S::DZF + q + 4 * v] = dv[v];
      }
      __syncwarp();
      if (on) {  // dz trunk1 = (dfeat W_feature + dz_density W_density) * (h1 > 0)
        float dv[Q];
        dense_t_part_t<Q, W, S::OS>(swt + S::T3, s + S::DZF, q, dv);
        const float dzs = s[S::DZS];
#pragma unroll
        for (int v = 0; v < Q; ++v) {
          const int i = q + 4 * v;
          const float h = __fadd_rn(dv[v], __fmul_rn(dzs, w_den[i]));
          s[S::DZ1 + i] = s[S::H1 + i] > 0.f ? h : 0.f;
        }
      }
      __syncwarp();
      if (on) {  // dz trunk0 = (dz1 W_trunk1) * (h0 > 0)
        float dv[Q];
        dense_t_part_t<Q, W, S::OS>(swt + S::T1, s + S::DZ1, q, dv);
#pragma unroll
        for (int v = 0; v < Q; ++v) {
          const int i = q + 4 * v;
          s[S::DZ0 + i] = s[S::H0 + i] > 0.f ? dv[v] : 0.f;
        }
      }
    } else {
      if (on) {  // dfeat = first W columns of dz_dir W_direction
        float dv[Q];
        dense_t_part<Q, DP, W>(sw + L.w_off[4], s + S::DZD, q * Q, dv);
#pragma unroll
        for (int i = 0; i < Q; ++i) s[S::DZF + q * Q + i] = dv[i];
      }
      __syncwarp();
      if (on) {  // dz trunk1 = (dfeat W_feature + dz_density W_density) * (h1 > 0)
        float dv[Q];
        dense_t_part<Q, WP, W>(sw + L.w_off[3], s + S::DZF, q * Q, dv);
        const float dzs = s[S::DZS];
        const float* wd = w_den + q * Q;
#pragma unroll
        for (int i = 0; i < Q; ++i) {
          const float h = __fadd_rn(dv[i], __fmul_rn(dzs, wd[i]));
          s[S::DZ1 + q * Q + i] = s[S::H1 + q * Q + i] > 0.f ? h : 0.f;
        }
      }
      __syncwarp();
      if (on) {  // dz trunk0 = (dz1 W_trunk1) * (h0 > 0)
        float dv[Q];
        dense_t_part<Q, WP, W>(sw + L.w_off[1], s + S::DZ1, q * Q, dv);
#pragma unroll
        for (int i = 0; i < Q; ++i) s[S::DZ0 + q * Q + i] = s[S::H0 + q * Q + i] > 0.f ? dv[i] : 0.f;
      }
    }
    __syncthreads();
    // ---------------- phase B: parameter sums over this tile's rows (gw = dz^T in, gb = sum dz)
    bwd_param_sums<S, NT>(srow, n_in, part, t == 0, tid);
  }
}

int64_t bwd_max_chunks(int64_t n_cells, int64_t n);

template <int W>
static bool launch_bwd_width(const float* packed, const Fp32Layout& L, const BwdArgs& A, int64_t n_cells, int64_t n,
                             void* ws, cudaStream_t st) {
  using S = BwdShape<W>;
  const size_t smem =
      (S::WT ? (size_t)(S::WT_FLOATS + S::SM_FLOATS) * 4 : (size_t)L.cell_floats * 4) + (size_t)S::TR * S::LD * 4;
  static thread_local size_t set = 0;
  if (set < smem) {
    if (cudaFuncSetAttribute(k_grouped_backward<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return false;
    set = smem;
  }
  if (n_cells <= 0) return true;
  const int64_t max_chunks = bwd_max_chunks(n_cells, n);
  char* p = (char*)ws;
  uint2* chunks = (uint2*)p;
  p += gf_align((size_t)max_chunks * 8);
  uint32_t* chunk_off = (uint32_t*)p;
  p += gf_align((size_t)(n_cells + 1) * 4);
  uint32_t* n_chunks = (uint32_t*)p;
  p += gf_align(4);
  float* scratch = (float*)p;
  k_bwd_plan<<<1, 1024, 0, st>>>(A.offsets, n_cells, chunks, chunk_off, n_chunks);
  if (max_chunks > 0)
    k_grouped_backward<W><<<(unsigned)max_chunks, S::THREADS, smem, st>>>(packed, L, A, chunks, n_chunks, scratch);
  const int64_t elems = n_cells * S::TOTAL;
  k_bwd_reduce<W><<<(unsigned)std::min<int64_t>(gf_div_up<int64_t>(elems, 256), (int64_t)num_sms() * 16), 256, 0, st>>>(
      scratch, chunk_off, n_cells, A);
  return true;
}

int64_t bwd_max_chunks(int64_t n_cells, int64_t n) { return n / GF_BWD_CHUNK + std::min<int64_t>(n_cells, n) + 1; }

size_t bwd_workspace(const LayerTable& t, int64_t n_cells, int64_t n) {
  if (!prepare_mlp_fp32(t)) return 0;
  const int total = t.width == 32 ? BwdShape<32>::TOTAL : BwdShape<64>::TOTAL;
  const int64_t mc = bwd_max_chunks(n_cells, n);
  return gf_align((size_t)mc * 8) + gf_align((size_t)(n_cells + 1) * 4) + gf_align(4) +
         gf_align((size_t)mc * total * 4);
}

bool launch_grouped_backward(const LayerTable& t, const float* packed, const BwdArgs& A, int64_t n_cells, int64_t n,
                             void* ws, cudaStream_t st) {
  if (!prepare_mlp_fp32(t)) return false;
  const Fp32Layout L = make_fp32_layout(t);
  return t.width == 32 ? launch_bwd_width<32>(packed, L, A, n_cells, n, ws, st)
                       : launch_bwd_width<64>(packed, L, A, n_cells, n, ws, st);
}

// ---------------------------------------------------------------------------
// photometric loss (train.py:243-288): dense (ray, slot) compositing of the
// queried samples, float64 loss, and the per-query upstream gradients.
// ---------------------------------------------------------------------------
// scatter queried samples into the dense (B, k) grid: (r, g, b, alpha) and the
// query index per slot; the density is perturbed / rectified first when a
// noise vector is given (train.py:245-249)
__global__ void k_photo_scatter(PhotoArgs A, float4* dense, int32_t* qidx, uint8_t* nmask) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < A.n_queries;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ray = A.ray_index[q], slot = A.slot[q];
    float s = A.sigma[q];
    if (A.noise) {
      const float sh = __fadd_rn(s, A.noise[q]);
      nmask[q] = sh > 0.f;
      s = fmaxf(sh, 0.f);
    }
    const float a = -expm1f(__fmul_rn(-s, A.deltas[ray]));  // density_to_alpha (core.py:187-194)
    const int64_t j = ray * A.k + slot;
    dense[j] = make_float4(A.color[3 * q], A.color[3 * q + 1], A.color[3 * q + 2], a);
    qidx[j] = (int32_t)q;
  }
}

// one thread per ray: forward composite (cumprod transmittance, weights,
// prediction + background), squared error in float64, then the backward
// rest-of-ray recurrence from the last slot down (no division by 1 - alpha)
__global__ void k_photo_ray(PhotoArgs A, const float4* __restrict__ dense, const int32_t* __restrict__ qidx,
                            const uint8_t* __restrict__ nmask, float* tb, double* loss_parts) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= A.n_rays) return;
  const int k = A.k;
  const float4* dr = dense + b * k;
  float* tbr = tb + b * k;
  float tr = 1.0f, p0 = 0.f, p1 = 0.f, p2 = 0.f;
  for (int i = 0; i < k; ++i) {
    const float4 v = dr[i];
    tbr[i] = tr;                          // t_before
    const float w = __fmul_rn(tr, v.w);   // weights = t_before * alpha
    p0 = __fadd_rn(p0, __fmul_rn(w, v.x));
    p1 = __fadd_rn(p1, __fmul_rn(w, v.y));
    p2 = __fadd_rn(p2, __fmul_rn(w, v.z));
    tr = __fmul_rn(tr, __fsub_rn(1.0f, v.w));  // cumprod(1 - alpha)
  }
  const float r0 = __fsub_rn(__fadd_rn(p0, __fmul_rn(tr, A.bg[0])), A.gt[3 * b + 0]);
  const float r1 = __fsub_rn(__fadd_rn(p1, __fmul_rn(tr, A.bg[1])), A.gt[3 * b + 1]);
  const float r2 = __fsub_rn(__fadd_rn(p2, __fmul_rn(tr, A.bg[2])), A.gt[3 * b + 2]);
  loss_parts[b] = __dadd_rn(__dadd_rn(__dmul_rn((double)r0, (double)r0), __dmul_rn((double)r1, (double)r1)),
                            __dmul_rn((double)r2, (double)r2));
  if (!A.d_color_q) return;
  const float d0 = __fmul_rn(A.two_over_b, r0), d1 = __fmul_rn(A.two_over_b, r1), d2 = __fmul_rn(A.two_over_b, r2);
  const float delta = A.deltas[b];
  float re0 = A.bg[0], re1 = A.bg[1], re2 = A.bg[2];  // rest[:, k-1] = bg
  for (int i = k - 1; i >= 0; --i) {
    const float4 v = dr[i];
    const int32_t q = qidx[b * k + i];
    if (q >= 0) {
      const float t = tbr[i];
      // d_alpha = sum_c (dpred_c * t_before) * (color_c - rest_c)
      const float e0 = __fmul_rn(__fmul_rn(d0, t), __fsub_rn(v.x, re0));
      const float e1 = __fmul_rn(__fmul_rn(d1, t), __fsub_rn(v.y, re1));
      const float e2 = __fmul_rn(__fmul_rn(d2, t), __fsub_rn(v.z, re2));
      const float da = __fadd_rn(__fadd_rn(e0, e1), e2);
      const float w = __fmul_rn(t, v.w);
      A.d_color_q[3 * q + 0] = __fmul_rn(w, d0);
      A.d_color_q[3 * q + 1] = __fmul_rn(w, d1);
      A.d_color_q[3 * q + 2] = __fmul_rn(w, d2);
      float ds = __fmul_rn(__fmul_rn(da, delta), __fsub_rn(1.0f, v.w));
      if (A.noise && !nmask[q]) ds = __fmul_rn(ds, 0.f);  // d_sigma_q * noise_mask
      A.d_sigma_q[q] = ds;
    }
    // rest[:, i-1] = alpha_i * color_i + (1 - alpha_i) * rest[:, i]
    const float om = __fsub_rn(1.0f, v.w);
    re0 = __fadd_rn(__fmul_rn(v.w, v.x), __fmul_rn(om, re0));
    re1 = __fadd_rn(__fmul_rn(v.w, v.y), __fmul_rn(om, re1));
    re2 = __fadd_rn(__fmul_rn(v.w, v.z), __fmul_rn(om, re2));
  }
}

// fixed-order float64 sum of n values (one CTA): deterministic loss reduction
__global__ void __launch_bounds__(1024) k_sum_f64(const double* v, int64_t n, double* out) {
  __shared__ double s[1024];
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += 1024) acc = __dadd_rn(acc, v[j]);
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 512; w; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] = __dadd_rn(s[threadIdx.x], s[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

size_t photo_workspace(int64_t n_rays, int k, int64_t n_queries) {
  const size_t cells = (size_t)n_rays * (size_t)k;
  return gf_align(cells * 16) + gf_align(cells * 4) * 2 + gf_align((size_t)n_queries + 1) +
         gf_align((size_t)n_rays * 8 + 8) + gf_align(8);
}

void launch_photometric(const PhotoArgs& A, void* ws, double* loss_sum, cudaStream_t st) {
  char* p = (char*)ws;
  const size_t cells = (size_t)A.n_rays * (size_t)A.k;
  float4* dense = (float4*)p;
  p += gf_align(cells * 16);
  int32_t* qidx = (int32_t*)p;
  p += gf_align(cells * 4);
  float* tb = (float*)p;
  p += gf_align(cells * 4);
  uint8_t* nmask = (uint8_t*)p;
  p += gf_align((size_t)A.n_queries + 1);
  double* parts = (double*)p;
  cudaMemsetAsync(dense, 0, cells * 16, st);
  cudaMemsetAsync(qidx, 0xFF, cells * 4, st);
  if (A.n_queries > 0) {
    const unsigned g = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(A.n_queries, 256), (int64_t)num_sms() * 8);
    k_photo_scatter<<<g, 256, 0, st>>>(A, dense, qidx, nmask);
  }
  if (A.n_rays > 0) k_photo_ray<<<(unsigned)gf_div_up<int64_t>(A.n_rays, 128), 128, 0, st>>>(A, dense, qidx, nmask, tb,
                                                                                            parts);
  k_sum_f64<<<1, 1024, 0, st>>>(parts, A.n_rays, loss_sum);
}

// ---------------------------------------------------------------------------
// optimizer (train.py:130-160): Adam in place over one flat parameter array,
// float32 with numpy's operation order (NEP 50: Python-float coefficients are
// rounded to float32 before use); L2 term sum(x^2) in float64.
// ---------------------------------------------------------------------------
__global__ void k_adam(float* p, const float* g, float* m, float* v, int64_t n, AdamCoef c) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const float gj = g[j];
    float mj = __fmul_rn(m[j], c.b1);                          // m *= b1
    mj = __fadd_rn(mj, __fmul_rn(c.one_minus_b1, gj));         // m += (1 - b1) * g
    float vj = __fmul_rn(v[j], c.b2);                          // v *= b2
    vj = __fadd_rn(vj, __fmul_rn(__fmul_rn(c.one_minus_b2, gj), gj));  // v += (1 - b2) * g * g
    // p -= lr * (m / bc1) / (sqrt(v / bc2) + eps)
    const float num = __fmul_rn(c.lr, __fdiv_rn(mj, c.bc1));
    const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(vj, c.bc2)), c.eps);
    p[j] = __fsub_rn(p[j], __fdiv_rn(num, den));
    m[j] = mj;
    v[j] = vj;
  }
}

void launch_adam(float* p, const float* g, float* m, float* v, int64_t n, const AdamCoef& c, cudaStream_t st) {
  if (n <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(n, 256), (int64_t)num_sms() * 16);
  k_adam<<<grid, 256, 0, st>>>(p, g, m, v, n, c);
}

// partial sums of squares in float64, then one fixed-order CTA sum
__global__ void __launch_bounds__(256) k_sumsq(const float* x, int64_t n, double* parts) {
  __shared__ double s[256];
  double acc = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x; j < n; j += (int64_t)gridDim.x * 256) {
    const double d = (double)x[j];
    acc = __dadd_rn(acc, __dmul_rn(d, d));
  }
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] = __dadd_rn(s[threadIdx.x], s[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) parts[blockIdx.x] = s[0];
}

// out = y + f * x (two roundings, as numpy's g + (2*weight) * w); y NULL: f * x
__global__ void k_axpy(const float* x, const float* y, int64_t n, float f, float* out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const float r = __fmul_rn(f, x[j]);
    out[j] = y ? __fadd_rn(y[j], r) : r;
  }
}

// distill_step's loss and upstream gradients (train.py:369-385) per query:
// alphas at the reference segment, L2 on alpha (weight w_a) and colour
__global__ void k_distill(DistillArgs A, double* parts) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < A.n; q += (int64_t)gridDim.x * blockDim.x) {
    const float ta = -expm1f(__fmul_rn(-A.t_sigma[q], A.delta));
    const float sa = -expm1f(__fmul_rn(-A.s_sigma[q], A.delta));
    const float da = __fsub_rn(sa, ta);
    double col = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float dc = __fsub_rn(A.s_color[3 * q + c], A.t_color[3 * q + c]);
      col = __dadd_rn(col, __dmul_rn((double)dc, (double)dc));
      A.d_color[3 * q + c] = __fmul_rn(A.c_color, dc);
    }
    // (2 w_a / m) * d_alpha * delta * (1 - s_alpha)
    A.d_sigma[q] = __fmul_rn(__fmul_rn(__fmul_rn(A.c_sigma, da), A.delta), __fsub_rn(1.0f, sa));
    parts[2 * q] = __dmul_rn((double)da, (double)da);
    parts[2 * q + 1] = col;
  }
}

// per-term fixed-order float64 sums of the (alpha, colour) parts
__global__ void __launch_bounds__(1024) k_sum_pairs_f64(const double* v, int64_t n, double* out) {
  __shared__ double s[2][1024];
  double a = 0.0, b = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += 1024) {
    a = __dadd_rn(a, v[2 * j]);
    b = __dadd_rn(b, v[2 * j + 1]);
  }
  s[0][threadIdx.x] = a;
  s[1][threadIdx.x] = b;
  __syncthreads();
  for (int w = 512; w; w >>= 1) {
    if ((int)threadIdx.x < w) {
      s[0][threadIdx.x] = __dadd_rn(s[0][threadIdx.x], s[0][threadIdx.x + w]);
      s[1][threadIdx.x] = __dadd_rn(s[1][threadIdx.x], s[1][threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s[0][0];
    out[1] = s[1][0];
  }
}

void launch_distill(const DistillArgs& A, double* parts, double* sums, cudaStream_t st) {
  if (A.n > 0) {
    const unsigned grid = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(A.n, 256), (int64_t)num_sms() * 16);
    k_distill<<<grid, 256, 0, st>>>(A, parts);
  }
  k_sum_pairs_f64<<<1, 1024, 0, st>>>(parts, A.n, sums);
}

void launch_sumsq(const float* x, int64_t n, double* parts, int n_parts, double* out, cudaStream_t st) {
  k_sumsq<<<n_parts, 256, 0, st>>>(x, n, parts);
  k_sum_f64<<<1, 1024, 0, st>>>(parts, n_parts, out);
}

void launch_axpy(const float* x, const float* y, int64_t n, float f, float* out, cudaStream_t st) {
  if (n <= 0) return;
  const unsigned grid = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(n, 256), (int64_t)num_sms() * 16);
  k_axpy<<<grid, 256, 0, st>>>(x, y, n, f, out);
}

}  // namespace gf
