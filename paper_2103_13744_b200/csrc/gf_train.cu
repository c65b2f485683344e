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
#include "gf_tc_ptx.cuh"

#include <cuda_bf16.h>

#include <cstdlib>

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

// 1024-thread exclusive scan of one value per thread (wsum: 32 words of shared memory)
__device__ __forceinline__ uint32_t block_excl_scan_1024(uint32_t local, uint32_t* wsum) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t x = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();  // wsum free (a previous scan's readers are done)
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
  return (wid ? wsum[wid - 1] : 0u) + x - local;
}

// chunk_tile (tensor-core path): index of the chunk's first 32-row operand
// tile; a cell's chunks are 256-row aligned, so chunk j of cell c starts at
// tile(c) + 8 j with tile(c) = sum over earlier cells of ceil(rows / 32)
__global__ void __launch_bounds__(1024) k_bwd_plan(const int64_t* __restrict__ offsets, int64_t n_cells, uint2* chunks,
                                                   uint32_t* chunk_off, uint32_t* n_chunks, uint32_t* chunk_tile,
                                                   uint4* red_cells, uint32_t* n_red, int red_blocks) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t s_red;
  const int tid = threadIdx.x;
  if (tid == 0) s_red = 0;
  const int64_t per = (n_cells + 1023) / 1024, c0 = (int64_t)tid * per;
  uint32_t local = 0, local_t = 0;
  for (int64_t c = c0; c < c0 + per && c < n_cells; ++c) {
    const int64_t rows = offsets[c + 1] - offsets[c];
    local += (uint32_t)((rows + GF_BWD_CHUNK - 1) / GF_BWD_CHUNK);
    local_t += (uint32_t)((rows + 31) / 32);
  }
  uint32_t base = block_excl_scan_1024(local, wsum);
  uint32_t tbase = chunk_tile ? block_excl_scan_1024(local_t, wsum) : 0u;
  for (int64_t c = c0; c < c0 + per && c < n_cells; ++c) {
    chunk_off[c] = base;
    const int64_t rows = offsets[c + 1] - offsets[c];
    const uint32_t nch = (uint32_t)((rows + GF_BWD_CHUNK - 1) / GF_BWD_CHUNK);
    // reduce work: cells without rows (zeros) or with 2..8 chunks as one
    // item; a cell with more chunks as one item per 256-parameter block
    if (nch == 0 || (nch > 1 && nch <= 8)) {
      red_cells[atomicAdd(&s_red, 1u)] = make_uint4((uint32_t)c, base, base + nch, 0xFFFFFFFFu);
    } else if (nch > 8) {
      const uint32_t nb = (uint32_t)red_blocks, at = atomicAdd(&s_red, nb);
      for (uint32_t j = 0; j < nb; ++j) red_cells[at + j] = make_uint4((uint32_t)c, base, base + nch, j);
    }
    for (uint32_t j = 0; j < nch; ++j) {
      chunks[base + j] = make_uint2((uint32_t)c, j);
      if (chunk_tile) chunk_tile[base + j] = tbase + j * (GF_BWD_CHUNK / 32);
    }
    base += nch;
    tbase += (uint32_t)((rows + 31) / 32);
  }
  if (tid == 1023) {
    chunk_off[n_cells] = base;
    *n_chunks = base;
  }
  __syncthreads();
  if (tid == 0) *n_red = s_red;
}

// chunk sums -> reference-layout gradients for the items k_bwd_plan listed
// (cell, first chunk, end chunk, parameter block or ALL): cells without rows
// (zeros) or with several chunks (added in chunk order); single-chunk cells
// were written in place.  One CTA per item (grid-stride); a crowded cell's
// parameters are split over 256-parameter items so its long chunk sums run
// on many SMs.
template <class S>
__device__ __forceinline__ void bwd_reduce_one(const float* __restrict__ scratch, const BwdArgs& A, size_t cell,
                                               uint32_t k0, uint32_t k1, int p) {
  float acc = 0.f;
  if (k1 > k0) {
    acc = scratch[(size_t)k0 * S::TOTAL + p];
#pragma unroll 8
    for (uint32_t k = k0 + 1; k < k1; ++k) acc = __fadd_rn(acc, scratch[(size_t)k * S::TOTAL + p]);
  }
  int l = 0, q = p;
#pragma unroll
  for (int j = 0; j < S::N_LAYERS - 1; ++j)
    if (l == j && q >= S::count(j)) {
      q -= S::count(j);
      l = j + 1;
    }
  const int in = S::in_dim(l), out = S::out_dim(l);
  if (q < out * in) A.gw[l][cell * (out * in) + q] = acc;
  else A.gb[l][cell * out + (q - out * in)] = acc;
}

template <int W>
__global__ void __launch_bounds__(256) k_bwd_reduce(const float* __restrict__ scratch,
                                                    const uint4* __restrict__ red_cells,
                                                    const uint32_t* __restrict__ n_red, BwdArgs A) {
  using S = BwdShape<W>;
  const uint32_t nr = *n_red;
  for (uint32_t ri = blockIdx.x; ri < nr; ri += gridDim.x) {
    const uint4 e = red_cells[ri];
    if (e.w != 0xFFFFFFFFu) {
      const int p = (int)e.w * 256 + threadIdx.x;
      if (p < S::TOTAL) bwd_reduce_one<S>(scratch, A, e.x, e.y, e.z, p);
      continue;
    }
    // whole cell, layer by layer (compile-time shapes, no per-parameter lookup)
    int base = 0;
#pragma unroll
    for (int l = 0; l < S::N_LAYERS; ++l) {
      const int in = S::in_dim(l), out = S::out_dim(l), cnt = S::count(l);
      float* gw = A.gw[l] + (size_t)e.x * (out * in);
      float* gb = A.gb[l] + (size_t)e.x * out;
      for (int q = threadIdx.x; q < cnt; q += 256) {
        // whole-cell items: no rows (zeros), or 2..8 chunks: all loads
        // issued, then added in chunk order
        float acc = 0.f;
        if (e.z > e.y) {
          const float* src = scratch + (size_t)e.y * S::TOTAL + base + q;
          const uint32_t nk = e.z - e.y;
          float vals[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) vals[u] = (uint32_t)u < nk ? src[(size_t)u * S::TOTAL] : 0.f;
          acc = vals[0];
#pragma unroll
          for (int u = 1; u < 8; ++u)
            if ((uint32_t)u < nk) acc = __fadd_rn(acc, vals[u]);
        }
        if (q < out * in) gw[q] = acc;
        else gb[q - out * in] = acc;
      }
      base += cnt;
    }
  }
}

// Phase B of one layer: gw[o][i] = sum_rows dz[o] * in[i] (fmaf chain in row
// order from 0) and gb[o] = sum_rows dz[o] (fadd chain), accumulated into the
// chunk's partial sums (first tile stores).  Threads own 4x4 (o, i) blocks:
// 8 shared loads per 16 FMAs instead of 2 per FMA, and no per-parameter index
// arithmetic; the per-parameter arithmetic sequence is unchanged.
template <class S, int OUT, int IN, int DZ, int INO, int NT>
__device__ __forceinline__ void bwd_layer_sums(const float* srow, int n_in, float* pw, float* pb, bool first, int tid,
                                               int& u) {
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
          old[a][c] = (!first && o0 + a < OUT && i0 + c < IN) ? pw[(o0 + a) * IN + i0 + c] : 0.f;
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
          if (o0 + a < OUT && i0 + c < IN) pw[(o0 + a) * IN + i0 + c] = first ? acc[a][c] : __fadd_rn(old[a][c], acc[a][c]);
    } else {
      const int o0 = (b - NB) * 4;
      float acc[4] = {0.f, 0.f, 0.f, 0.f}, old[4];
      const float* dzp = srow + DZ + o0;
#pragma unroll
      for (int a = 0; a < 4; ++a) old[a] = (!first && o0 + a < OUT) ? pb[o0 + a] : 0.f;
      for (int rr = 0; rr < n_in; ++rr)
#pragma unroll
        for (int a = 0; a < 4; ++a)
          if (o0 + a < OUT) acc[a] = __fadd_rn(acc[a], dzp[rr * LD + a]);
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (o0 + a < OUT) pb[o0 + a] = first ? acc[a] : __fadd_rn(old[a], acc[a]);
    }
  }
  u += NB + OB;
}

// where a chunk's parameter sums go: its scratch row (several chunks per
// cell, added by k_bwd_reduce in chunk order) or, for a cell with a single
// chunk, straight into the reference-layout gradients
struct GradDst {
  float* part;         // scratch row of the chunk, or NULL: direct
  const BwdArgs* A;
  int64_t cell;
  template <class S>
  __device__ __forceinline__ float* w(int l) const {
    if (part) {
      int off = 0;
      for (int k = 0; k < l; ++k) off += S::count(k);
      return part + off;
    }
    return A->gw[l] + cell * (S::out_dim(l) * S::in_dim(l));
  }
  template <class S>
  __device__ __forceinline__ float* b(int l) const {
    return part ? w<S>(l) + S::out_dim(l) * S::in_dim(l) : A->gb[l] + cell * S::out_dim(l);
  }
};

template <class S, int NT, int L>
__device__ __forceinline__ void bwd_sums_l(const float* srow, int n_in, const GradDst& g, bool first, int tid, int& u) {
  bwd_layer_sums<S, S::out_dim(L), S::in_dim(L), S::dz_off(L), S::in_off(L), NT>(srow, n_in, g.w<S>(L), g.b<S>(L),
                                                                                first, tid, u);
}

template <class S, int NT>
__device__ __forceinline__ void bwd_param_sums(const float* srow, int n_in, const GradDst& g, bool first, int tid) {
  int u = 0;  // running unit count: spreads the layers' remainders over different threads
  bwd_sums_l<S, NT, 0>(srow, n_in, g, first, tid, u);
  bwd_sums_l<S, NT, 1>(srow, n_in, g, first, tid, u);
  bwd_sums_l<S, NT, 2>(srow, n_in, g, first, tid, u);
  bwd_sums_l<S, NT, 3>(srow, n_in, g, first, tid, u);
  bwd_sums_l<S, NT, 4>(srow, n_in, g, first, tid, u);
  bwd_sums_l<S, NT, 5>(srow, n_in, g, first, tid, u);
}

// ---------------------------------------------------------------------------
// Tensor-core weight gradients (W = 32).  Phase A of k_grouped_backward
// writes every 32-row tile as bf16 operand pieces (x = hi + mid + lo, each
// the bf16 rounding of what the previous pieces leave: 24 significant bits,
// float32's precision) in the canonical K-major layout, K = the tile's rows,
// one 16-row sub-tile after the other:
//   A (M = 128): the stacked deltas  [dz0 | dz1 | dz_feature | dz_direction]
//   B (N = 192): the stacked inputs  [gamma(x) 63 | 1 | h0 | h1 | [feat, gamma(d)] 59 | 0 x5]
// k_bwd_tc accumulates D = A B^T over a chunk's tiles in TMEM, six MMAs per
// K step (the piece products down to 2^-16: lo.hi, hi.lo, mid.mid, mid.hi,
// hi.mid, hi.hi; the dropped ones are <= 2^-24 relative), so D[o][i] of the
// four diagonal blocks is gw = sum_rows dz[o] in[i] and column 63 (the ones
// row) is gb = sum_rows dz[o].  A tile with at most 16 rows has no second
// sub-tile (not written, not loaded).  The density and colour layers (33 + 99
// parameters) stay on the CUDA cores in phase B.
// ---------------------------------------------------------------------------
#ifndef GF_BWD_TC_PIECES
#define GF_BWD_TC_PIECES 3
#endif
#define GF_BWD_TC_A 4096                                         // one piece of A: 128 x 16 bf16
#define GF_BWD_TC_B 6144                                         // one piece of B: 192 x 16 bf16
#define GF_BWD_TC_SUB (GF_BWD_TC_PIECES * (GF_BWD_TC_A + GF_BWD_TC_B))  // one 16-row sub-tile
#define GF_BWD_TC_TILE (2 * GF_BWD_TC_SUB)

// bf16 pieces of two values (rows k, k+1: low half = even row)
__device__ __forceinline__ void bf16_pieces2(float a, float b, uint32_t (&out)[GF_BWD_TC_PIECES]) {
#pragma unroll
  for (int p = 0; p < GF_BWD_TC_PIECES; ++p) {
    const __nv_bfloat16 ha = __float2bfloat16_rn(a), hb = __float2bfloat16_rn(b);
    out[p] = (uint32_t)__bfloat16_as_ushort(ha) | ((uint32_t)__bfloat16_as_ushort(hb) << 16);
    a = __fsub_rn(a, __bfloat162float(ha));  // exact (Sterbenz / bf16 grid)
    b = __fsub_rn(b, __bfloat162float(hb));
  }
}

// one tile's operands: 16-byte units (8 consecutive rows of one feature),
// numbered so that consecutive threads store consecutive 16 bytes
template <class S>
__device__ __forceinline__ void bwd_tc_operands(const float* srow, int n_in, uint8_t* tile, int tid) {
  constexpr int LD = S::LD, W = 32, UNITS = 256 + 384;  // per 16-row sub-tile
  const int n_units = n_in > 16 ? 2 * UNITS : UNITS;
  for (int uu = tid; uu < n_units; uu += S::THREADS) {
    const int ks = uu >= UNITS, u = uu - ks * UNITS;
    const bool is_a = u < 256;
    const int v = is_a ? u : u - 256;
    const int f = ((v >> 4) << 3) | (v & 7), kg = (v >> 3) & 1;  // feature (M or N index), 8-row group
    int off = -1;  // srow offset; -1: zero; -2: the ones row
    if (is_a) {
      const int blk = f >> 5;
      off = (blk == 0 ? S::DZ0 : blk == 1 ? S::DZ1 : blk == 2 ? S::DZF : S::DZD) + (f & 31);
    } else if (f < 63) {
      off = S::X + f;
    } else if (f == 63) {
      off = -2;
    } else if (f < 64 + W) {
      off = S::H0 + f - 64;
    } else if (f < 64 + 2 * W) {
      off = S::H1 + f - 96;
    } else if (f < 128 + W + S::D) {
      off = S::CAT + f - 128;
    }
    uint32_t w[4][GF_BWD_TC_PIECES];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int r0 = ks * 16 + kg * 8 + 2 * p, r1 = r0 + 1;
      const float x0 = r0 < n_in ? (off >= 0 ? srow[r0 * LD + off] : (off == -2 ? 1.f : 0.f)) : 0.f;
      const float x1 = r1 < n_in ? (off >= 0 ? srow[r1 * LD + off] : (off == -2 ? 1.f : 0.f)) : 0.f;
      bf16_pieces2(x0, x1, w[p]);
    }
    uint8_t* d = tile + ks * GF_BWD_TC_SUB + (is_a ? 0 : GF_BWD_TC_PIECES * GF_BWD_TC_A) + v * 16;
#pragma unroll
    for (int p = 0; p < GF_BWD_TC_PIECES; ++p)
      *reinterpret_cast<uint4*>(d + p * (is_a ? GF_BWD_TC_A : GF_BWD_TC_B)) = make_uint4(w[0][p], w[1][p], w[2][p], w[3][p]);
  }
}

// phase B of the two narrow layers (density, colour) when the wide ones go to
// the tensor cores
template <class S, int NT>
__device__ __forceinline__ void bwd_narrow_sums(const float* srow, int n_in, const GradDst& g, bool first, int tid) {
  int u = 0;
  bwd_sums_l<S, NT, 2>(srow, n_in, g, first, tid, u);
  bwd_sums_l<S, NT, 5>(srow, n_in, g, first, tid, u);
}

// k_bwd_tc: persistent, one CTA per SM.  Warp 4 streams the chunk's operand
// tiles into a 4-stage shared-memory ring (one bulk copy per tile), warp 5
// issues the MMAs into one of two TMEM accumulators (192 columns each), and
// warps 0-3 drain the other accumulator: warp w owns TMEM lanes 32w..32w+31 =
// the outputs of one layer (trunk0, trunk1, feature, direction), staged in
// shared memory and written to the chunk's partial sums in reference order.
namespace bwdtc {
constexpr int NST = GF_BWD_TC_PIECES == 3 ? 3 : 4, THREADS = 192, N = 192, ACC_COLS = 256, EPI_LD = 65;
constexpr int EPI = NST * GF_BWD_TC_TILE;
constexpr int BAR = EPI + 128 * EPI_LD * 4;  // full[NST], empty[NST], tfull[2], tempty[2], tmem slot
constexpr int SMEM = BAR + 8 * (2 * NST + 4) + 16;
static_assert(SMEM <= 227 * 1024, "k_bwd_tc shared memory");
}  // namespace bwdtc

__global__ void __launch_bounds__(bwdtc::THREADS, 1)
    k_bwd_tc(const uint8_t* __restrict__ opbuf, const uint2* __restrict__ chunks,
             const uint32_t* __restrict__ chunk_tile, const uint32_t* __restrict__ n_chunks,
             const int64_t* __restrict__ offsets, const uint32_t* __restrict__ chunk_off, float* scratch,
             BwdArgs A) {
  using namespace tcx;
  using S = BwdShape<32>;
  using namespace bwdtc;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  const uint32_t full = sb + BAR, empty = full + 8 * NST, tfull = empty + 8 * NST, tempty = tfull + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + BAR + 8 * (2 * NST + 4));
  float* epi = reinterpret_cast<float*>(smem + EPI);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(2u * ACC_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      mbar_init(full + 8 * i, 1);
      mbar_init(empty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull + 8 * i, 1);
      mbar_init(tempty + 8 * i, 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t nch = *n_chunks;
  auto chunk_rows = [&](uint32_t ci) -> uint32_t {
    const uint2 ch = chunks[ci];
    return (uint32_t)min(offsets[ch.x + 1] - offsets[ch.x] - (int64_t)ch.y * GF_BWD_CHUNK, (int64_t)GF_BWD_CHUNK);
  };
  if (warp == 4) {  // ---- producer
    if (lane == 0) {
      uint32_t g = 0;
      for (uint32_t ci = blockIdx.x; ci < nch; ci += gridDim.x) {
        const uint32_t rows = chunk_rows(ci), nt = (rows + 31) / 32, t0 = chunk_tile[ci];
        for (uint32_t t = 0; t < nt; ++t, ++g) {
          const uint32_t s = g % NST, ph = (g / NST) & 1u;
          const uint32_t bytes = rows - 32 * t > 16 ? GF_BWD_TC_TILE : GF_BWD_TC_SUB;
          mbar_wait(empty + 8 * s, ph ^ 1u);
          bulk_load(sb + s * GF_BWD_TC_TILE, opbuf + (size_t)(t0 + t) * GF_BWD_TC_TILE, bytes, full + 8 * s);
        }
      }
    }
  } else if (warp == 5) {  // ---- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(128, N);
      uint32_t g = 0, it = 0;
      for (uint32_t ci = blockIdx.x; ci < nch; ci += gridDim.x, ++it) {
        const uint32_t acc = it & 1u, aph = (it >> 1) & 1u, rows = chunk_rows(ci), nt = (rows + 31) / 32;
        mbar_wait(tempty + 8 * acc, aph ^ 1u);
        fence_after();
        const uint32_t d = tmem + acc * ACC_COLS;
        for (uint32_t t = 0; t < nt; ++t, ++g) {
          const uint32_t s = g % NST, ph = (g / NST) & 1u, nks = rows - 32 * t > 16 ? 2u : 1u;
          mbar_wait(full + 8 * s, ph);
          fence_after();
          for (uint32_t ks = 0; ks < nks; ++ks) {
            const uint32_t base = sb + s * GF_BWD_TC_TILE + ks * GF_BWD_TC_SUB;
            uint64_t a[GF_BWD_TC_PIECES], b[GF_BWD_TC_PIECES];
#pragma unroll
            for (int p = 0; p < GF_BWD_TC_PIECES; ++p) {
              a[p] = desc_kmajor(base + p * GF_BWD_TC_A, 16);
              b[p] = desc_kmajor(base + GF_BWD_TC_PIECES * GF_BWD_TC_A + p * GF_BWD_TC_B, 16);
            }
            uint32_t accf = (t | ks) ? 1u : 0u;
#if GF_BWD_TC_PIECES == 3
            mma_ss(d, a[2], b[0], idesc, accf);  // small terms first
            mma_ss(d, a[0], b[2], idesc, 1u);
            mma_ss(d, a[1], b[1], idesc, 1u);
            accf = 1u;
#endif
            mma_ss(d, a[1], b[0], idesc, accf);
            mma_ss(d, a[0], b[1], idesc, 1u);
            mma_ss(d, a[0], b[0], idesc, 1u);
          }
          mma_commit(empty + 8 * s);  // the stage is free once these MMAs have read it
        }
        mma_commit(tfull + 8 * acc);
      }
    }
  } else {  // ---- epilogue: warp w = layer (trunk0, trunk1, feature, direction)
    const int layer = warp == 0 ? 0 : warp == 1 ? 1 : warp == 2 ? 3 : 4;
    const int in = S::in_dim(layer);
    const int col0 = warp == 0 ? 0 : warp == 1 ? 64 : warp == 2 ? 96 : 128;
    int base = 0;
    for (int l = 0; l < layer; ++l) base += S::count(l);
    float* er = epi + tid * EPI_LD;
    uint32_t it = 0;
    for (uint32_t ci = blockIdx.x; ci < nch; ci += gridDim.x, ++it) {
      const uint32_t acc = it & 1u, aph = (it >> 1) & 1u;
      mbar_wait(tfull + 8 * acc, aph);
      fence_after();
      const uint32_t ta = tmem + acc * ACC_COLS + ((uint32_t)(warp * 32) << 16);
      for (int c = 0; c < in; c += 16) {
        uint32_t r[16];
        tmem_ld16(ta + col0 + c, r);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (c + q < in) er[c + q] = __uint_as_float(r[q]);
      }
      const uint32_t b = tmem_ld1(ta + 63);
      tmem_wait_ld();
      er[64] = __uint_as_float(b);
      fence_before();
      mbar_arrive(tempty + 8 * acc);  // the accumulator may take the next chunk
      __syncwarp();
      const uint32_t cell = chunks[ci].x;
      const bool direct = chunk_off[cell + 1] - chunk_off[cell] == 1;
      float* dw = direct ? A.gw[layer] + (size_t)cell * (32 * in) : scratch + (size_t)ci * S::TOTAL + base;
      float* db = direct ? A.gb[layer] + (size_t)cell * 32 : dw + 32 * in;
      const float* ew = epi + warp * 32 * EPI_LD;
      for (int e = lane; e < 32 * in; e += 32) dw[e] = ew[(e / in) * EPI_LD + e % in];
      db[lane] = ew[lane * EPI_LD + 64];
      __syncwarp();
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2u * ACC_COLS));
}

template <int W, bool TCB>
__global__ void __launch_bounds__(BwdShape<W>::THREADS) k_grouped_backward(const float* __restrict__ packed,
                                                                           Fp32Layout L, BwdArgs A,
                                                                           const uint2* __restrict__ chunks,
                                                                           const uint32_t* __restrict__ n_chunks,
                                                                           const uint32_t* __restrict__ chunk_off,
                                                                           float* scratch, uint8_t* opbuf,
                                                                           const uint32_t* __restrict__ chunk_tile) {
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
    if (!A.act) transpose(0, P, S::T0);  // trunk0 is only needed to recompute the forward
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
  GradDst gd;
  gd.part = chunk_off[cell + 1] - chunk_off[cell] > 1 ? scratch + (size_t)blockIdx.x * S::TOTAL : nullptr;
  gd.A = &A;
  gd.cell = cell;
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
    // ---- forward (mlp.py:238-266): recomputed, or (W = 32) read from the
    // training forward's activations -- the same fp32 operation order, so
    // the same values
    const bool have_act = S::WT && A.act != nullptr;
    if (have_act) {
      if (on) {
        const float4* av = reinterpret_cast<const float4*>(A.act + (size_t)row * GF_ACT_FLOATS);
        for (int v = q; v < GF_ACT_FLOATS / 4; v += S::LANES) {
          const float4 x = av[v];
          const float e4[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int f = 4 * v + e;
            const int d = f < W ? S::H0 + f
                                : f < 2 * W ? S::H1 + f - W
                                            : f < 3 * W ? S::CAT + f - 2 * W
                                                        : f < 4 * W ? S::G + f - 3 * W
                                                                    : f == 4 * W ? S::SIG : S::ZC + f - 4 * W - 1;
            s[d] = e4[e];
          }
        }
      }
      __syncwarp();
    } else if constexpr (S::WT) {
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
      if (!have_act) dense_part<W, WP, 1, false>(w_col, bias(5), s + S::G, q, s + S::ZC);  // logit q
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
    if constexpr (TCB) {
      bwd_tc_operands<S>(srow, n_in, opbuf + ((size_t)chunk_tile[blockIdx.x] + t) * GF_BWD_TC_TILE, tid);
      bwd_narrow_sums<S, NT>(srow, n_in, gd, t == 0, tid);
    } else {
      bwd_param_sums<S, NT>(srow, n_in, gd, t == 0, tid);
    }
  }
}

int64_t bwd_max_chunks(int64_t n_cells, int64_t n) { return n / GF_BWD_CHUNK + std::min<int64_t>(n_cells, n) + 1; }
// reduce items: one per cell, plus (blocks - 1) per cell with more than 8 chunks
static size_t bwd_red_items(int64_t n_cells, int64_t n, int total) {
  return (size_t)n_cells + (size_t)(n / (8 * GF_BWD_CHUNK) + 1) * (size_t)((total + 255) / 256);
}
static int64_t bwd_max_tiles(int64_t n_cells, int64_t n) { return n / 32 + std::min<int64_t>(n_cells, n) + 1; }

// GF_BWD_TC=0: the wide layers' weight gradients on the CUDA cores too
static bool bwd_tc_enabled(int width) {
  static const bool on = [] {
    const char* e = std::getenv("GF_BWD_TC");
    return !(e && e[0] == '0');
  }();
  return on && width == 32;
}

template <int W>
static bool launch_bwd_width(const float* packed, const Fp32Layout& L, const BwdArgs& A, int64_t n_cells, int64_t n,
                             void* ws, cudaStream_t st) {
  using S = BwdShape<W>;
  constexpr bool TC_OK = W == 32;
  const bool tc = TC_OK && bwd_tc_enabled(W);
  const size_t smem =
      (S::WT ? (size_t)(S::WT_FLOATS + S::SM_FLOATS) * 4 : (size_t)L.cell_floats * 4) + (size_t)S::TR * S::LD * 4;
  static thread_local size_t set = 0;
  if (set < smem) {
    if (cudaFuncSetAttribute(k_grouped_backward<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return false;
    if (TC_OK && (cudaFuncSetAttribute(k_grouped_backward<W, TC_OK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem) != cudaSuccess ||
                  cudaFuncSetAttribute(k_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, bwdtc::SMEM) !=
                      cudaSuccess))
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
  p += gf_align((size_t)max_chunks * S::TOTAL * 4);
  uint4* red_cells = (uint4*)p;
  p += gf_align(bwd_red_items(n_cells, n, S::TOTAL) * 16);
  uint32_t* n_red = (uint32_t*)p;
  p += gf_align(4);
  uint32_t* chunk_tile = tc ? (uint32_t*)p : nullptr;
  p += gf_align((size_t)max_chunks * 4);
  uint8_t* opbuf = (uint8_t*)p;
  k_bwd_plan<<<1, 1024, 0, st>>>(A.offsets, n_cells, chunks, chunk_off, n_chunks, chunk_tile, red_cells, n_red,
                                 (S::TOTAL + 255) / 256);
  if (max_chunks > 0) {
    if (tc) {
      k_grouped_backward<W, TC_OK><<<(unsigned)max_chunks, S::THREADS, smem, st>>>(packed, L, A, chunks, n_chunks, chunk_off,
                                                                                  scratch, opbuf, chunk_tile);
      k_bwd_tc<<<(unsigned)std::min<int64_t>(max_chunks, (int64_t)num_sms()), bwdtc::THREADS, bwdtc::SMEM, st>>>(
          opbuf, chunks, chunk_tile, n_chunks, A.offsets, chunk_off, scratch, A);
    } else {
      k_grouped_backward<W, false><<<(unsigned)max_chunks, S::THREADS, smem, st>>>(packed, L, A, chunks, n_chunks, chunk_off,
                                                                                 scratch, nullptr, nullptr);
    }
  }
  k_bwd_reduce<W><<<(unsigned)std::min<int64_t>(n_cells, (int64_t)num_sms() * 8), 256, 0, st>>>(scratch, red_cells,
                                                                                                 n_red, A);
  return true;
}

size_t bwd_workspace(const LayerTable& t, int64_t n_cells, int64_t n) {
  if (!prepare_mlp_fp32(t)) return 0;
  const int total = t.width == 32 ? BwdShape<32>::TOTAL : BwdShape<64>::TOTAL;
  const int64_t mc = bwd_max_chunks(n_cells, n);
  size_t bytes = gf_align((size_t)mc * 8) + gf_align((size_t)(n_cells + 1) * 4) + gf_align(4) +
                 gf_align((size_t)mc * total * 4) + gf_align(bwd_red_items(n_cells, n, total) * 16) + gf_align(4);
  if (bwd_tc_enabled(t.width))
    bytes += gf_align((size_t)mc * 4) + (size_t)bwd_max_tiles(n_cells, n) * GF_BWD_TC_TILE;
  return bytes;
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
// rest-of-ray recurrence from the last slot down (no division by 1 - alpha).
// A warp owns 32 consecutive rays and stages PH_CS slots of all of them at a
// time through shared memory: the dense rows, t_before and the query indices
// move as whole 128-byte lines instead of one strided element per lane.
#define PH_CS 16
#define PH_WARPS 1  // one warp (32 rays) per CTA: 8192 rays -> 256 CTAs cover all 148 SMs
__global__ void __launch_bounds__(32 * PH_WARPS) k_photo_ray(PhotoArgs A, const float4* __restrict__ dense,
                                                             const int32_t* __restrict__ qidx,
                                                             const uint8_t* __restrict__ nmask, float* tb,
                                                             double* loss_parts) {
  __shared__ float4 s_v[PH_WARPS][32][PH_CS + 1];
  __shared__ float s_t[PH_WARPS][32][PH_CS + 1];
  __shared__ int32_t s_q[PH_WARPS][32][PH_CS + 1];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t b0 = ((int64_t)blockIdx.x * PH_WARPS + wp) * 32;
  if (b0 >= A.n_rays) return;  // warp-uniform
  const int64_t b = b0 + lane;
  const bool on = b < A.n_rays;
  const int nr = A.n_rays - b0 < 32 ? (int)(A.n_rays - b0) : 32;
  const int k = A.k;
  float4(*sv)[PH_CS + 1] = s_v[wp];
  float(*st)[PH_CS + 1] = s_t[wp];
  int32_t(*sq)[PH_CS + 1] = s_q[wp];
  // slots [i0, i0 + PH_CS) of the warp's rays, ray-major (lanes read
  // consecutive slots of a ray): element u of this lane is (e / PH_CS,
  // e % PH_CS), e = lane + 32 u.  The next chunk is fetched into registers
  // while the current one is composited (software pipelining).
  float4 pv[PH_CS];
  float pt[PH_CS];
  int32_t pq[PH_CS];
  auto fetch = [&](int i0, bool with_t) {
#pragma unroll
    for (int u = 0; u < PH_CS; ++u) {
      const int e = lane + 32 * u, r = e / PH_CS, j = e % PH_CS;
      if (i0 >= 0 && r < nr && i0 + j < k) {
        const size_t g = (size_t)(b0 + r) * k + i0 + j;
        pv[u] = dense[g];
        if (with_t) {
          pt[u] = tb[g];
          pq[u] = qidx[g];
        }
      }
    }
  };
  auto stage = [&](bool with_t) {
#pragma unroll
    for (int u = 0; u < PH_CS; ++u) {
      const int e = lane + 32 * u, r = e / PH_CS, j = e % PH_CS;
      sv[r][j] = pv[u];
      if (with_t) {
        st[r][j] = pt[u];
        sq[r][j] = pq[u];
      }
    }
    __syncwarp();
  };
  float tr = 1.0f, p0 = 0.f, p1 = 0.f, p2 = 0.f;
  fetch(0, false);
  for (int i0 = 0; i0 < k; i0 += PH_CS) {
    stage(false);
    fetch(i0 + PH_CS, false);
    if (on) {
      for (int j = 0; j < PH_CS && i0 + j < k; ++j) {
        const float4 v = sv[lane][j];
        st[lane][j] = tr;                     // t_before
        const float w = __fmul_rn(tr, v.w);   // weights = t_before * alpha
        p0 = __fadd_rn(p0, __fmul_rn(w, v.x));
        p1 = __fadd_rn(p1, __fmul_rn(w, v.y));
        p2 = __fadd_rn(p2, __fmul_rn(w, v.z));
        tr = __fmul_rn(tr, __fsub_rn(1.0f, v.w));  // cumprod(1 - alpha)
      }
    }
    __syncwarp();
#pragma unroll
    for (int u = 0; u < PH_CS; ++u) {
      const int e = lane + 32 * u, r = e / PH_CS, j = e % PH_CS;
      if (r < nr && i0 + j < k) tb[(size_t)(b0 + r) * k + i0 + j] = st[r][j];
    }
    __syncwarp();
  }
  float r0 = 0.f, r1 = 0.f, r2 = 0.f;
  if (on) {
    r0 = __fsub_rn(__fadd_rn(p0, __fmul_rn(tr, A.bg[0])), A.gt[3 * b + 0]);
    r1 = __fsub_rn(__fadd_rn(p1, __fmul_rn(tr, A.bg[1])), A.gt[3 * b + 1]);
    r2 = __fsub_rn(__fadd_rn(p2, __fmul_rn(tr, A.bg[2])), A.gt[3 * b + 2]);
    loss_parts[b] = __dadd_rn(__dadd_rn(__dmul_rn((double)r0, (double)r0), __dmul_rn((double)r1, (double)r1)),
                              __dmul_rn((double)r2, (double)r2));
  }
  if (!A.d_color_q) return;
  const float d0 = __fmul_rn(A.two_over_b, r0), d1 = __fmul_rn(A.two_over_b, r1), d2 = __fmul_rn(A.two_over_b, r2);
  const float delta = on ? A.deltas[b] : 0.f;
  float re0 = A.bg[0], re1 = A.bg[1], re2 = A.bg[2];  // rest[:, k-1] = bg
  const int last = ((k - 1) / PH_CS) * PH_CS;
  fetch(last, true);  // t_before of these slots was stored above (same lanes' earlier stores: program order)
  for (int i0 = last; i0 >= 0; i0 -= PH_CS) {
    stage(true);
    fetch(i0 - PH_CS, true);
    if (on) {
      for (int j = min(PH_CS, k - i0) - 1; j >= 0; --j) {
        const float4 v = sv[lane][j];
        const int32_t q = sq[lane][j];
        if (q >= 0) {
          const float t = st[lane][j];
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
    __syncwarp();
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
  if (A.n_rays > 0)
    k_photo_ray<<<(unsigned)gf_div_up<int64_t>(A.n_rays, 32 * PH_WARPS), 32 * PH_WARPS, 0, st>>>(A, dense, qidx, nmask,
                                                                                               tb, parts);
  k_sum_f64<<<1, 1024, 0, st>>>(parts, A.n_rays, loss_sum);
}

// ---------------------------------------------------------------------------
// optimizer (train.py:130-160): Adam in place over one flat parameter array,
// float32 with numpy's operation order (NEP 50: Python-float coefficients are
// rounded to float32 before use); L2 term sum(x^2) in float64.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void adam_one(float& p, float g, float& m, float& v, const AdamCoef& c) {
  float mj = __fmul_rn(m, c.b1);                             // m *= b1
  mj = __fadd_rn(mj, __fmul_rn(c.one_minus_b1, g));          // m += (1 - b1) * g
  float vj = __fmul_rn(v, c.b2);                             // v *= b2
  vj = __fadd_rn(vj, __fmul_rn(__fmul_rn(c.one_minus_b2, g), g));  // v += (1 - b2) * g * g
  // p -= lr * (m / bc1) / (sqrt(v / bc2) + eps)
  const float num = __fmul_rn(c.lr, __fdiv_rn(mj, c.bc1));
  const float den = __fadd_rn(__fsqrt_rn(__fdiv_rn(vj, c.bc2)), c.eps);
  p = __fsub_rn(p, __fdiv_rn(num, den));
  m = mj;
  v = vj;
}

__global__ void k_adam(float* p, const float* g, float* m, float* v, int64_t n, AdamCoef c) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    float pj = p[j], mj = m[j], vj = v[j];
    adam_one(pj, g[j], mj, vj, c);
    p[j] = pj;
    m[j] = mj;
    v[j] = vj;
  }
}

// 16-byte aligned arrays: four parameters per thread and 16-byte accesses
// (same per-element arithmetic)
__global__ void __launch_bounds__(256) k_adam4(float4* p, const float4* g, float4* m, float4* v, int64_t n4,
                                               AdamCoef c) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x) {
    float4 pj = p[j], mj = m[j], vj = v[j];
    const float4 gj = g[j];
    adam_one(pj.x, gj.x, mj.x, vj.x, c);
    adam_one(pj.y, gj.y, mj.y, vj.y, c);
    adam_one(pj.z, gj.z, mj.z, vj.z, c);
    adam_one(pj.w, gj.w, mj.w, vj.w, c);
    p[j] = pj;
    m[j] = mj;
    v[j] = vj;
  }
}

void launch_adam(float* p, const float* g, float* m, float* v, int64_t n, const AdamCoef& c, cudaStream_t st) {
  if (n <= 0) return;
  const bool al = (((uintptr_t)p | (uintptr_t)g | (uintptr_t)m | (uintptr_t)v) & 15) == 0;
  const int64_t n4 = al ? n / 4 : 0;
  if (n4 > 0) {
    const unsigned grid = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(n4, 256), (int64_t)num_sms() * 8);
    k_adam4<<<grid, 256, 0, st>>>((float4*)p, (const float4*)g, (float4*)m, (float4*)v, n4, c);
  }
  const int64_t rest = n - 4 * n4;
  if (rest > 0) {
    const unsigned grid = (unsigned)std::min<int64_t>(gf_div_up<int64_t>(rest, 256), (int64_t)num_sms() * 16);
    k_adam<<<grid, 256, 0, st>>>(p + 4 * n4, g + 4 * n4, m + 4 * n4, v + 4 * n4, rest, c);
  }
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
