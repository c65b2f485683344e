// Fused positional-encoding + tiny-MLP on the 5th-gen tensor cores (sm_100a).
//
// Reference math: core.py:132-152 (encoding), mlp.py:222-266 (forward),
// batched.py:120-151 (one network per segment).  Design:
//
//  * one CTA = 128 threads working on TWO 128-row tiles of the same cell at
//    once (ping-pong): thread t owns row t of both tiles, which is TMEM lane
//    t, so every epilogue is a private tcgen05.ld of the thread's own
//    accumulator row; while the tensor core runs one tile's layer, the warps
//    run the other tile's epilogue, hiding the MMA / commit / barrier latency
//    of the 5-layer dependency chain;
//  * the cell's weights are pre-packed on the device (gf_pack_weights) into
//    the exact shared-memory image the MMAs consume (fp16, K-major,
//    no-swizzle canonical layout, fp32 biases) and brought in with ONE 1-D
//    bulk TMA copy (cp.async.bulk + mbarrier complete_tx) only when the
//    cell changes;
//  * the 6 affine layers run as 5 chains of tcgen05.mma.kind::f16
//    (M=128, N=32/32/48/32/16, K=64/32/32/64/32; density and feature share
//    one N=48 MMA), fp32 accumulators in TMEM, activations round-trip only
//    through shared memory (never HBM);
//  * persistent CTAs walk contiguous tile ranges so consecutive tiles of the
//    same cell reuse the staged weights; the next pair's row inputs are
//    prefetched while the current pair's first MMAs run.
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>

#include "gf_mlp.cuh"

namespace gf {

// ---------------------------------------------------------------------------
// layout of one cell's packed parameters == its shared-memory image
// ---------------------------------------------------------------------------
template <int W>
struct TcShape {
  static constexpr int P = 63, D = 27;
  static constexpr int K0 = 64, N0 = W;                        // trunk0   63 -> W
  static constexpr int K1 = W, N1 = W;                         // trunk1   W  -> W
  static constexpr int K2 = W, N2 = ((W + 1 + 15) / 16) * 16;  // feature (rows 0..W-1) + density (row W)
  static constexpr int K3 = ((W + D + 15) / 16) * 16, N3 = W;  // direction [feat, gamma(d)] -> W
  static constexpr int K4 = W, N4 = 16;                        // color W -> 3 (rows 0..2)
  // operand byte offsets (fp16, canonical K-major no-swizzle)
  static constexpr int B0 = 0;
  static constexpr int B1 = B0 + N0 * K0 * 2;
  static constexpr int B2 = B1 + N1 * K1 * 2;
  static constexpr int B3 = B2 + N2 * K2 * 2;
  static constexpr int B4 = B3 + N3 * K3 * 2;
  static constexpr int BIAS = B4 + N4 * K4 * 2;  // fp32 biases
  static constexpr int BB0 = 0, BB1 = N0, BB2 = N0 + N1, BB3 = N0 + N1 + N2, BB4 = N0 + N1 + N2 + N3;
  static constexpr int N_BIAS = N0 + N1 + N2 + N3 + N4;
  static constexpr int CELL_BYTES = ((BIAS + N_BIAS * 4) + 127) / 128 * 128;
  // per tile slot: A0 holds gamma(x) (128 x K0), later [feat, gamma(d)]
  // (128 x K3) once the trunk0 MMA has consumed gamma(x); A1 holds h0/h1/g.
  static constexpr int KA0 = K0 > K3 ? K0 : K3;
  static constexpr int SLOT_BYTES = 128 * KA0 * 2 + 128 * W * 2;
  static constexpr int A0(int s) { return CELL_BYTES + s * SLOT_BYTES; }
  static constexpr int A1(int s) { return CELL_BYTES + s * SLOT_BYTES + 128 * KA0 * 2; }
  static constexpr int BAR = CELL_BYTES + 2 * SLOT_BYTES;  // mma[0], mma[1], weights, tmem base
  static constexpr int SMEM = BAR + 32;
  static constexpr int NC = N2 <= 32 ? 32 : (N2 <= 64 ? 64 : (N2 <= 128 ? 128 : 256));  // TMEM cols per slot
  static constexpr int TMEM_COLS = 2 * NC;
};

// byte offset of element (r, k) in a canonical K-major no-swizzle operand of
// K columns: 8x8 core matrices (128 B), K-chunks adjacent (LBO = 128 B),
// 8-row groups SBO = K/8 * 128 B apart.
__host__ __device__ __forceinline__ int canon_off(int r, int k, int K) {
  return (r >> 3) * (K * 16) + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, int K) {
  const uint64_t lbo = 128, sbo = (uint64_t)K * 16;
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) | (1ull << 46);
}

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4)                       // D format f32
         | (0u << 7) | (0u << 10)        // A, B: f16
         | ((uint32_t)(N >> 3) << 17)    // N
         | ((uint32_t)(M >> 4) << 24);   // M
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

#define GF_LD16(taddr, r)                                                                                      \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
               "[%16];"                                                                                        \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),           \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),       \
                 "=r"(r[14]), "=r"(r[15])                                                                      \
               : "r"(taddr))

// load N accumulator columns (multiple of 16) of this thread's row
template <int N>
__device__ __forceinline__ void tmem_load(uint32_t taddr, float* out) {
  uint32_t r[N];
#pragma unroll
  for (int c = 0; c < N; c += 16) GF_LD16(taddr + c, (r + c));
  tmem_wait_ld();
#pragma unroll
  for (int c = 0; c < N; ++c) out[c] = __uint_as_float(r[c]);
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  uint32_t r;  // one F2FP.F16.F32.PACK_AB; low half = a
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

// write 8 consecutive features [k0, k0+8) of row r into a canonical operand
__device__ __forceinline__ void st_chunk(uint8_t* A, int K, int r, int k0, const float* v) {
  uint4 q = make_uint4(pack_h2(v[0], v[1]), pack_h2(v[2], v[3]), pack_h2(v[4], v[5]), pack_h2(v[6], v[7]));
  *reinterpret_cast<uint4*>(A + canon_off(r, k0, K)) = q;
}

// bias add (+ReLU) with 16-byte broadcast loads of the biases
template <int N, bool RELU>
__device__ __forceinline__ void add_bias(float* h, const float* __restrict__ b) {
  const float4* b4 = reinterpret_cast<const float4*>(b);
#pragma unroll
  for (int c = 0; c < N / 4; ++c) {
    const float4 q = b4[c];
    h[4 * c + 0] += q.x; h[4 * c + 1] += q.y; h[4 * c + 2] += q.z; h[4 * c + 3] += q.w;
    if (RELU) {
      h[4 * c + 0] = fmaxf(h[4 * c + 0], 0.f); h[4 * c + 1] = fmaxf(h[4 * c + 1], 0.f);
      h[4 * c + 2] = fmaxf(h[4 * c + 2], 0.f); h[4 * c + 3] = fmaxf(h[4 * c + 3], 0.f);
    }
  }
}

// sin / cos of x * 2^k * pi: the angle is formed exactly as numpy forms it
// (fl32(x * fl32(2^k pi)) == 2^k fl32(x*pi)), reduced by 2pi with a two-term
// Cody-Waite split, then MUFU sin/cos (~5e-7 abs).
__device__ __forceinline__ void sincos_scaled(float x, int k, float* s, float* c) {
  const float a = __fmul_rn(x, __int_as_float(0x40490FDB + (k << 23)));
  const float n = rintf(a * 0.15915494309189535f);
  float r = fmaf(-n, 6.28125f, a);          // 2pi_hi (exact times n <= 2^9)
  r = fmaf(-n, 1.9353071795864769e-3f, r);  // 2pi_lo
  __sincosf(r, s, c);
}

// octaves k < L: MUFU anchors every third octave, double-angle steps in
// between (max abs error 2.6e-6 vs 4.9e-4 fp16 operand rounding)
template <int L>
__device__ __forceinline__ void encode_octaves(float x, float* s, float* c) {
#pragma unroll
  for (int k = 0; k < L; ++k) {
    if (k % 3 == 0) {
      sincos_scaled(x, k, &s[k], &c[k]);
    } else {
      const float sp = s[k - 1], cp = c[k - 1];
      s[k] = 2.0f * sp * cp;
      c[k] = (cp - sp) * (cp + sp);
    }
  }
}

// one row's inputs
struct RowIn {
  uint32_t idx;
  bool valid;
  float x[3], d[3];
};

template <class IO>
__device__ __forceinline__ void load_row(const TileSched& S, const IO& io, uint2 tl, int tid, RowIn& r) {
  const uint32_t seg0 = S.offsets[tl.x], seg_n = S.offsets[tl.x + 1] - seg0;
  r.valid = tl.y + (uint32_t)tid < seg_n;
  r.idx = 0;
  r.x[0] = r.x[1] = r.x[2] = 0.f;
  r.d[0] = r.d[1] = r.d[2] = 0.f;
  if (r.valid) {
    r.idx = S.sorted[seg0 + tl.y + tid];
    io.load(r.idx, r.x, r.d);
  }
}

// tiles [t, t+1) or [t, t+2): the second slot is used only for a tile of the
// same cell (both slots share the staged weights)
__device__ __forceinline__ bool pair_second(const TileSched& S, uint32_t t, uint32_t t_end, uint32_t cell) {
  return t + 1 < t_end && S.tiles[t + 1].x == cell;
}

template <int W>
__device__ __forceinline__ void encode_position(uint8_t* A0, int tid, const float* x) {
  using T = TcShape<W>;
  float e[64];
  e[0] = x[0]; e[1] = x[1]; e[2] = x[2];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float s[10], c[10];
    encode_octaves<10>(x[a], s, c);
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      e[3 + 6 * k + a] = s[k];
      e[6 + 6 * k + a] = c[k];
    }
  }
  e[63] = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) st_chunk(A0, T::K0, tid, 8 * c, e + 8 * c);
}

template <int W>
__device__ __forceinline__ void encode_direction(uint8_t* A3, int tid, const float* d) {
  using T = TcShape<W>;
  float e[T::K3 - W];
  e[0] = d[0]; e[1] = d[1]; e[2] = d[2];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    float s[4], c[4];
    encode_octaves<4>(d[a], s, c);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      e[3 + 6 * k + a] = s[k];
      e[6 + 6 * k + a] = c[k];
    }
  }
#pragma unroll
  for (int j = 27; j < T::K3 - W; ++j) e[j] = 0.f;
#pragma unroll
  for (int c = 0; c < (T::K3 - W) / 8; ++c) st_chunk(A3, T::K3, tid, W + 8 * c, e + 8 * c);
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int W, class IO>
__global__ void __launch_bounds__(128) k_mlp_tc(const uint8_t* __restrict__ packed, TileSched S, IO io) {
  using T = TcShape<W>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const float* sbias = reinterpret_cast<const float*>(smem + T::BIAS);
  const uint32_t bar0 = smem_u32(smem + T::BAR), bar_w = bar0 + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + T::BAR + 24);
  const int tid = threadIdx.x, warp = tid >> 5;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)T::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar0 + 8, 1);
    mbar_init(bar_w, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;  // this warp's TMEM lane quarter
  const uint32_t wb = smem_u32(smem);

  const uint32_t nt = *S.n_tiles;
  const uint32_t per = (nt + gridDim.x - 1) / gridDim.x;
  const uint32_t t_begin = blockIdx.x * per, t_end = min(nt, t_begin + per);
  int cur = -1;
  uint32_t ph[2] = {0, 0}, ph_w = 0;

  // MMA issue for layer L of slot s (one elected thread)
  auto issue = [&](int L, int s) {
    if (tid != 0) return;
    const uint32_t a0 = wb + T::A0(s), a1 = wb + T::A1(s), d = tmem + s * T::NC;
    uint32_t a = a1, b = wb + T::B1, idesc = idesc_f16(128, T::N1);
    int K = T::K1;
    if (L == 0) { a = a0; b = wb + T::B0; K = T::K0; idesc = idesc_f16(128, T::N0); }
    if (L == 2) { b = wb + T::B2; K = T::K2; idesc = idesc_f16(128, T::N2); }
    if (L == 3) { a = a0; b = wb + T::B3; K = T::K3; idesc = idesc_f16(128, T::N3); }
    if (L == 4) { b = wb + T::B4; K = T::K4; idesc = idesc_f16(128, T::N4); }
    for (int ks = 0; ks < K / 16; ++ks)
      mma_f16(d, umma_desc(a + ks * 256, K), umma_desc(b + ks * 256, K), idesc, ks > 0 ? 1u : 0u);
    mma_commit(bar0 + 8 * s);
  };
  auto wait_mma = [&](int s) {
    mbar_wait(bar0 + 8 * s, ph[s]);
    ph[s] ^= 1;
    fence_after();
  };
  auto publish = [&]() {  // smem operand writes -> visible to the tensor core, TMEM reads retired
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
  };

  RowIn nxt[2];
  if (t_begin < t_end) {
    const uint2 tl = S.tiles[t_begin];
    load_row(S, io, tl, tid, nxt[0]);
    if (pair_second(S, t_begin, t_end, tl.x)) load_row(S, io, S.tiles[t_begin + 1], tid, nxt[1]);
  }

  for (uint32_t t = t_begin; t < t_end;) {
    const uint2 tl = S.tiles[t];
    const bool two = pair_second(S, t, t_end, tl.x);
    const uint32_t t_next = t + (two ? 2 : 1);
    __syncthreads();  // previous pair fully retired (bias reads, output stores)
    const bool new_cell = (int)tl.x != cur;
    if (new_cell && tid == 0) bulk_load(wb, packed + (size_t)tl.x * T::CELL_BYTES, T::CELL_BYTES, bar_w);
    cur = (int)tl.x;
    RowIn row[2] = {nxt[0], nxt[1]};

    encode_position<W>(smem + T::A0(0), tid, row[0].x);
    if (two) encode_position<W>(smem + T::A0(1), tid, row[1].x);
    publish();
    if (new_cell) {
      mbar_wait(bar_w, ph_w);
      ph_w ^= 1;
    }
    issue(0, 0);
    if (two) issue(0, 1);
    // prefetch the next pair while trunk0 runs
    if (t_next < t_end) {
      const uint2 tn = S.tiles[t_next];
      load_row(S, io, tn, tid, nxt[0]);
      if (pair_second(S, t_next, t_end, tn.x)) load_row(S, io, S.tiles[t_next + 1], tid, nxt[1]);
    }

    float sigma[2] = {0.f, 0.f};
#pragma unroll
    for (int L = 0; L < 5; ++L) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (s == 1 && !two) continue;
        uint8_t* A0 = smem + T::A0(s);
        uint8_t* A1 = smem + T::A1(s);
        const uint32_t trow = tmem + s * T::NC + lane_base;
        wait_mma(s);
        if (L == 0) {  // trunk0 -> A1; gamma(x) is dead, gamma(d) -> A0 as [., gamma(d)]
          float h[W];
          tmem_load<W>(trow, h);
          add_bias<W, true>(h, sbias + T::BB0);
#pragma unroll
          for (int c = 0; c < W / 8; ++c) st_chunk(A1, W, tid, 8 * c, h + 8 * c);
          encode_direction<W>(A0, tid, row[s].d);
        } else if (L == 1) {  // trunk1 -> A1
          float h[W];
          tmem_load<W>(trow, h);
          add_bias<W, true>(h, sbias + T::BB1);
#pragma unroll
          for (int c = 0; c < W / 8; ++c) st_chunk(A1, W, tid, 8 * c, h + 8 * c);
        } else if (L == 2) {  // feature (cols 0..W-1, unactivated) + density (col W)
          float h[T::N2];
          tmem_load<T::N2>(trow, h);
          add_bias<T::N2, false>(h, sbias + T::BB2);
          sigma[s] = fmaxf(h[W], 0.f);
#pragma unroll
          for (int c = 0; c < W / 8; ++c) st_chunk(A0, T::K3, tid, 8 * c, h + 8 * c);
        } else if (L == 3) {  // direction -> A1
          float h[W];
          tmem_load<W>(trow, h);
          add_bias<W, true>(h, sbias + T::BB3);
#pragma unroll
          for (int c = 0; c < W / 8; ++c) st_chunk(A1, W, tid, 8 * c, h + 8 * c);
        } else {  // color: sigmoid
          float z[16];
          tmem_load<16>(trow, z);
          float rgb[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const float v = z[c] + sbias[T::BB4 + c];
            rgb[c] = v >= 0.f ? __fdividef(1.f, 1.f + __expf(-v)) : __fdividef(__expf(v), 1.f + __expf(v));
          }
          if (row[s].valid) io.store(row[s].idx, rgb[0], rgb[1], rgb[2], sigma[s]);
        }
        if (L < 4) {
          publish();
          issue(L + 1, s);
        }
      }
    }
    fence_before();
    t = t_next;
  }
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)T::TMEM_COLS));
}

// ---------------------------------------------------------------------------
// packing (layer-major fp32 -> per-cell fp16 smem image)
// ---------------------------------------------------------------------------
struct PackArgsTc {
  const float* w[GF_MAX_LAYERS];
  const float* b[GF_MAX_LAYERS];
};

template <int W>
__global__ void k_pack_tc(PackArgsTc A, int64_t n_cells, uint8_t* packed) {
  using T = TcShape<W>;
  const int64_t cell = blockIdx.x;
  if (cell >= n_cells) return;
  uint8_t* dst = packed + cell * T::CELL_BYTES;
  // layer l weights (n_cells, out, in)
  auto w = [&](int l, int o, int i, int out, int in) -> float {
    return A.w[l][(cell * out + o) * (int64_t)in + i];
  };
  auto put = [&](int base, int K, int n, int k, float v) {
    *reinterpret_cast<__half*>(dst + base + canon_off(n, k, K)) = __float2half_rn(v);
  };
  for (int j = threadIdx.x; j < T::N0 * T::K0; j += blockDim.x) {
    int n = j / T::K0, k = j % T::K0;
    put(T::B0, T::K0, n, k, k < T::P ? w(0, n, k, W, T::P) : 0.f);
  }
  for (int j = threadIdx.x; j < T::N1 * T::K1; j += blockDim.x) {
    int n = j / T::K1, k = j % T::K1;
    put(T::B1, T::K1, n, k, w(1, n, k, W, W));
  }
  for (int j = threadIdx.x; j < T::N2 * T::K2; j += blockDim.x) {
    int n = j / T::K2, k = j % T::K2;
    float v = n < W ? w(3, n, k, W, W) : (n == W ? w(2, 0, k, 1, W) : 0.f);  // feature rows, then density
    put(T::B2, T::K2, n, k, v);
  }
  for (int j = threadIdx.x; j < T::N3 * T::K3; j += blockDim.x) {
    int n = j / T::K3, k = j % T::K3;
    put(T::B3, T::K3, n, k, k < W + T::D ? w(4, n, k, W, W + T::D) : 0.f);
  }
  for (int j = threadIdx.x; j < T::N4 * T::K4; j += blockDim.x) {
    int n = j / T::K4, k = j % T::K4;
    put(T::B4, T::K4, n, k, n < 3 ? w(5, n, k, 3, W) : 0.f);
  }
  float* bias = reinterpret_cast<float*>(dst + T::BIAS);
  for (int j = threadIdx.x; j < T::N_BIAS; j += blockDim.x) {
    float v = 0.f;
    if (j < T::BB1) v = A.b[0][cell * W + j];
    else if (j < T::BB2) v = A.b[1][cell * W + (j - T::BB1)];
    else if (j < T::BB3) {
      int c = j - T::BB2;
      v = c < W ? A.b[3][cell * W + c] : (c == W ? A.b[2][cell] : 0.f);
    } else if (j < T::BB4) v = A.b[4][cell * W + (j - T::BB3)];
    else {
      int c = j - T::BB4;
      v = c < 3 ? A.b[5][cell * 3 + c] : 0.f;
    }
    bias[j] = v;
  }
  for (int j = T::BIAS + T::N_BIAS * 4 + threadIdx.x; j < T::CELL_BYTES; j += blockDim.x) dst[j] = 0;
}

static bool tc_supported(const LayerTable& t) {
  return t.pos_dim == 63 && t.dir_dim == 27 && t.view == t.width && t.trunk == 2 && (t.width == 32 || t.width == 64);
}

size_t fp16_cell_bytes(const LayerTable& t) {
  if (!tc_supported(t)) return 0;
  return t.width == 32 ? TcShape<32>::CELL_BYTES : TcShape<64>::CELL_BYTES;
}

bool launch_pack_fp16(const LayerTable& t, int64_t n_cells, const float* const* w, const float* const* b, void* packed,
                      cudaStream_t st) {
  if (!tc_supported(t)) return false;
  PackArgsTc A;
  for (int l = 0; l < t.n_layers; ++l) { A.w[l] = w[l]; A.b[l] = b[l]; }
  if (n_cells <= 0) return true;
  if (t.width == 32) k_pack_tc<32><<<(unsigned)n_cells, 256, 0, st>>>(A, n_cells, (uint8_t*)packed);
  else k_pack_tc<64><<<(unsigned)n_cells, 256, 0, st>>>(A, n_cells, (uint8_t*)packed);
  return true;
}

template <int W, class IO>
static int tc_resident() {
  using T = TcShape<W>;
  auto k = k_mlp_tc<W, IO>;
  static thread_local int per_sm = 0;  // resident CTAs per SM for this instantiation
  if (per_sm == 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, T::SMEM);
    // residency from first principles (the occupancy API proved unreliable
    // here): shared memory (+1 KiB reserved per CTA), registers, TMEM columns
    int dev = 0, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaFuncAttributes fa;
    int regs = 128;
    if (cudaFuncGetAttributes(&fa, k) == cudaSuccess && fa.numRegs > 0) regs = fa.numRegs;
    const int by_smem = smem_sm / (T::SMEM + 1024);
    const int by_regs = 65536 / (((regs + 7) / 8 * 8) * 128);
    const int by_tmem = 512 / T::TMEM_COLS;
    per_sm = by_smem < by_regs ? by_smem : by_regs;
    per_sm = per_sm < by_tmem ? per_sm : by_tmem;
    if (per_sm < 1) per_sm = 1;
    if (getenv("GF_DEBUG"))
      fprintf(stderr, "[gf] k_mlp_tc<%d>: smem %d B, regs %d -> %d CTAs/SM (smem %d, regs %d, tmem %d)\n", W,
              T::SMEM, regs, per_sm, by_smem, by_regs, by_tmem);
    cudaGetLastError();
  }
  return per_sm;
}

template <int W, class IO>
static void launch_tc_w(const void* packed, const TileSched& S, const IO& io, cudaStream_t st) {
  using T = TcShape<W>;
  k_mlp_tc<W, IO><<<num_sms() * tc_resident<W, IO>(), 128, T::SMEM, st>>>((const uint8_t*)packed, S, io);
}

bool prepare_mlp_tc(const LayerTable& t) {
  if (!tc_supported(t)) return false;
  num_sms();
  if (t.width == 32) tc_resident<32, RenderIO>();
  else tc_resident<64, RenderIO>();
  return true;
}

template <class IO>
static bool launch_tc(const LayerTable& t, const void* packed, const TileSched& S, const IO& io, cudaStream_t st) {
  if (!tc_supported(t)) return false;
  if (t.width == 32) launch_tc_w<32>(packed, S, io, st);
  else launch_tc_w<64>(packed, S, io, st);
  return true;
}

bool launch_mlp_tc_render(const LayerTable& t, const void* packed, const TileSched& S, const RenderIO& io,
                          cudaStream_t st) {
  return launch_tc(t, packed, S, io, st);
}

bool launch_mlp_tc_query(const LayerTable& t, const void* packed, const TileSched& S, const QueryIO& io,
                         cudaStream_t st) {
  return launch_tc(t, packed, S, io, st);
}

}  // namespace gf
