// Fused positional-encoding + tiny-MLP on the 5th-gen tensor cores (sm_100a).
//
// Reference math: core.py:132-152 (encoding), mlp.py:222-266 (forward),
// batched.py:120-151 (one network per segment).  Design:
//
//  * activations live in TENSOR MEMORY: every layer is a chain of
//    tcgen05.mma.kind::f16 with the A operand (128 rows x K, fp16) read from
//    TMEM and the B operand (the cell's weights) from shared memory.  With A
//    in shared memory an M=128 x K=16 MMA moves 4 KB through the 128 B/clk
//    shared-memory port (~51 cycles at N=32, measured: scripts/ubench_tmem.cu);
//    from TMEM it runs at ~18 cycles, close to the N=32 floor of 16;
//  * one CTA = NS warpgroups + 1 loader warp.  Warpgroup g owns TMEM slot g
//    (SLOT columns: the accumulator D_L at [0, N_L), the A operand of layer L
//    at ACOL_L) and runs its own stream of 128-row tiles; thread gt of a
//    group owns row gt == TMEM lane gt, so every epilogue is a private
//    tcgen05.ld of the thread's accumulator row, fp32 -> fp16 (+ReLU) packs
//    and one tcgen05.st of the next layer's A row.  Groups never wait for
//    each other: while one group's MMAs run the others run epilogues;
//  * the CTA's contiguous tile range is cut into runs of one cell; the
//    loader warp finds the runs and brings each run's packed weights (the
//    exact shared-memory image of the B operands + bias tiles, k_pack_tc) into
//    one of two buffers with one bulk TMA copy, so the next cell's weights
//    arrive while the current run is evaluated.  Within a run group g takes
//    tiles g, g+NS, ...; a per-buffer mbarrier (count NS) frees the buffer;
//  * biases enter the accumulator through one K=16 MMA against a constant
//    TMEM operand of ones (bias tile row n = [hi(b_n), lo(b_n), 0...], 22
//    significant bits); density and feature share one N=W+16 MMA;
//  * gamma(x) (core.py layout) is generated octave by octave (exactly
//    reduced MUFU anchors + f32x2 double-angle steps) and flushed to TMEM
//    4 columns (8 fp16) at a time; the render path's gamma(d) is encoded
//    once per ray by k_ray_init and fetched while the first layers run.
#include <cuda_fp16.h>

#include <cstdio>
#include <cstdlib>

#include "gf_encode.cuh"
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
  // weight operand byte offsets (fp16, canonical K-major no-swizzle)
  static constexpr int B0 = 0;
  static constexpr int B1 = B0 + N0 * K0 * 2;
  static constexpr int B2 = B1 + N1 * K1 * 2;
  static constexpr int B3 = B2 + N2 * K2 * 2;
  static constexpr int B4 = B3 + N3 * K3 * 2;
  // bias operands: one K=16 tile per layer, row n = [hi(b_n), lo(b_n), 0 ...]
  // (fp16 hi + fp16 remainder: 22 significant bits); multiplied by the
  // constant ONES operand (columns 0 and 1 = 1) they initialise the accumulator
  static constexpr int BB0 = B4 + N4 * K4 * 2;
  static constexpr int BB1 = BB0 + N0 * 32;
  static constexpr int BB2 = BB1 + N1 * 32;
  static constexpr int BB3 = BB2 + N2 * 32;
  static constexpr int BB4 = BB3 + N3 * 32;
  static constexpr int CELL_BYTES = ((BB4 + N4 * 32) + 1023) / 1024 * 1024;

  // ---- TMEM slot of one tile (32-bit columns; fp16 A operands pack two
  // K values per column, low half = even k).  Layer L reads A_L at ACOL_L
  // and writes D_L at [0, N_L); the epilogue of L reads D_L completely before
  // it writes A_{L+1}, so A_{L+1} may overlap D_L.
  static constexpr int A0C = W, A1C = W, A2C = N2, A3C = W, A4C = W;
  static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  static constexpr int SLOT =
      cmax(cmax(A0C + K0 / 2, A1C + K1 / 2), cmax(cmax(A2C + K2 / 2, A3C + K3 / 2), A4C + K4 / 2));
  static_assert(A0C >= N0 && A1C >= N1 && A2C >= N2 && A3C >= N3 && A4C >= N4, "A operand overlaps its layer's D");
  static_assert(SLOT % 16 == 0, "slot columns");
};

// launch shape per width: warpgroups per CTA, tiles per warpgroup (TMEM
// slots each), CTAs per SM.  Measured on the C2 frame (MLP ms/frame,
// 2026-10-17): 7 groups x 1 tile x 1 CTA 0.361 (4 weight buffers), 0.364
// (3); 6 x 1 x 1 0.376; 3 x 1 x 2 0.376-0.386; 2 x 1 x 2 0.457; 3 x 1 x 1
// 0.550; two tiles per warpgroup 0.414; a dedicated MMA-issuer warp 0.589;
// the colour layer on the CUDA cores instead of a 5th MMA 0.41 -- tiles in
// flight per SM, each with its own warps, is what counts (latency-bound),
// and TMEM (64 columns per W=32 tile) caps them at 7.
#ifndef GF_TC_NS32
#define GF_TC_NS32 7
#endif
#ifndef GF_TC_CTAS32
#define GF_TC_CTAS32 1
#endif
#ifndef GF_TC_R32
#define GF_TC_R32 1
#endif
#ifndef GF_TC_WREL
#define GF_TC_WREL 2  // run hand-over: 0 unsafe (reference point only), 1 per-warp release, 2 group-synchronous
#endif
#ifndef GF_TC_NBUF32
#define GF_TC_NBUF32 4
#endif
template <int W>
struct TcCfg {
  static constexpr int NS = W == 32 ? GF_TC_NS32 : 2;
  static constexpr int CTAS = W == 32 ? GF_TC_CTAS32 : 2;
  static constexpr int R = W == 32 ? GF_TC_R32 : 1;        // tiles in flight per warpgroup (TMEM slots each)
  static constexpr int THREADS = NS * 128 + 32;
  static constexpr int ONES = NS * R * TcShape<W>::SLOT;  // 8 columns: [1, 1, 0 ...] fp16 per row
  static constexpr int tmem_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }
  static constexpr int TMEM_COLS = tmem_cols(ONES + 8);
  static_assert(ONES + 8 <= 512 && TMEM_COLS * CTAS <= 512, "TMEM budget");
  // shared memory: NBUF weight buffers, then barriers and the run table
  static constexpr int NBUF = W == 32 ? GF_TC_NBUF32 : 2;
  static constexpr int BAR = NBUF * TcShape<W>::CELL_BYTES;      // full[NBUF], free[NBUF], mma[NS]
  static constexpr int TSLOT = BAR + 16 * NBUF + 8 * NS;         // TMEM base address
  static constexpr int RUNS = (TSLOT + 4 + 15) / 16 * 16;        // uint4 runs[NBUF]: (cell, first tile, end tile, 0)
  static constexpr int GINFO = RUNS + 16 * NBUF;                 // uint32 per group: end tile of its current run
  static constexpr int SMEM = GINFO + 4 * NS;
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

// D[tmem] (+)= A[tmem] . B[smem]
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n" : "+r"(pred));
  return pred;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// parity wait with a suspend-time hint: the warp sleeps in the barrier unit
// until the phase flips (or the hint expires) instead of spinning on issue slots
#ifndef GF_TC_WATCHDOG
#define GF_TC_WATCHDOG 0
#endif
__device__ __forceinline__ uint64_t gtimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase, int site = 0) {
  uint32_t done;
#if GF_TC_WATCHDOG  // diagnostic build: report the first waiter stuck for 2 s, then trap
  const uint64_t t0 = gtimer_ns();
#endif
  do {
#if GF_TC_WATCHDOG
    if (gtimer_ns() - t0 > 2000000000ull) {
      printf("[gf watchdog] k_mlp_tc stuck: block %d thread %d site %d bar 0x%x phase %u\n", blockIdx.x, threadIdx.x,
             site, bar, phase);
      __trap();
    }
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase), "r"(1000000u)
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
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

#define GF_LD16(taddr, r)                                                                                      \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
               "[%16];"                                                                                        \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),           \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),       \
                 "=r"(r[14]), "=r"(r[15])                                                                      \
               : "r"(taddr))
#define GF_LD4(taddr, r)                                                   \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])             \
               : "r"(taddr))
#define GF_LD1(taddr, r) asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr))
#define GF_ST4(taddr, a, b, c, d)                                                                       \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(a), "r"(b), \
               "r"(c), "r"(d)                                                                           \
               : "memory")
#define GF_ST8(taddr, r)                                                                                        \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]), \
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])                       \
               : "memory")

// accumulator columns [0, N) of this thread's TMEM row -> fp16 (+ReLU) ->
// the next layer's A row at column `acol` (two K values per column); 16
// accumulator columns per load so only 16 fp32 values are live
template <int N, bool RELU>
__device__ __forceinline__ void epilogue_to_a(uint32_t trow, uint32_t acol) {
#pragma unroll
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16], o[8];
    GF_LD16(trow + c, r);
    tmem_wait_ld();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float a = __uint_as_float(r[2 * q]), b = __uint_as_float(r[2 * q + 1]);
      o[q] = RELU ? pack_h2_relu(a, b) : pack_h2(a, b);
    }
    GF_ST8(trow + acol + c / 2, o);
  }
}

// one row's inputs (prefetched one tile ahead within a run)
struct RowIn {
  uint32_t idx, row;  // caller / staging index, sorted row
  bool valid;
  float x[3], d[3];
};

template <class IO>
__device__ __forceinline__ void load_row(const TileSched& S, const IO& io, uint2 tl, int tid, RowIn& r) {
  r.valid = (uint32_t)tid < gf_tile_rows(tl);
  r.idx = 0;
  r.row = tl.y + (uint32_t)tid;
  r.x[0] = r.x[1] = r.x[2] = 0.f;
  if (!IO::kDirEnc) r.d[0] = r.d[1] = r.d[2] = 0.f;
  if (r.valid) io.template fetch<!IO::kDirEnc>(S, tl.y + (uint32_t)tid, r.idx, r.x, r.d);
}

// gamma(x) (core.py:132-152 layout: raw xyz, then per octave k sin xyz, cos
// xyz; column 63 zero).  Anchors at octaves 0 and 5 (MUFU after an exact
// 2pi reduction, abs error <= 3.6e-7), four double-angle steps after each
// (error at most doubles per step: <= 6e-6, against the 2.4e-4 fp16 operand
// rounding), all as f32x2 pairs.  Octaves 0-4 are flushed to the A0 operand
// in TMEM first (4 columns = 8 fp16 per store), then octaves 5-9, so few
// values are live at once.
template <int W>
__device__ __forceinline__ void encode_position(uint32_t ta0, const float* x) {
  float e[64];
  e[0] = x[0]; e[1] = x[1]; e[2] = x[2];
  e[63] = 0.f;
  auto put = [&](int k, int a, float sv, float cv) {
    e[3 + 6 * k + a] = sv;
    e[6 + 6 * k + a] = cv;
  };
  auto flush = [&](int c) {
    const float* v = e + 8 * c;
    GF_ST4(ta0 + 4 * c, pack_h2(v[0], v[1]), pack_h2(v[2], v[3]), pack_h2(v[4], v[5]), pack_h2(v[6], v[7]));
  };
  // four double-angle steps of two chains from anchors (ka, aa), (kb, ab)
  auto chains = [&](int ka, int aa, float sa, float ca, int kb, int ab, float sb, float cb) {
    F2 sv = f2(sa, sb), cv = f2(ca, cb);
#pragma unroll
    for (int st = 1; st <= 4; ++st) {
      double_angle2_fma(sv, cv);
      float s0, s1, c0, c1;
      f2_split(sv, s0, s1);
      f2_split(cv, c0, c1);
      put(ka + st, aa, s0, c0);
      put(kb + st, ab, s1, c1);
    }
  };
  float s0, c0, s1, c1, s2, c2, s3, c3;
  // octaves 0-4 of x, y, z (and 5-9 of z)
  sincos_scaled2(x[0], 0, x[1], 0, &s0, &c0, &s1, &c1);
  sincos_scaled2(x[2], 0, x[2], 5, &s2, &c2, &s3, &c3);
  put(0, 0, s0, c0); put(0, 1, s1, c1); put(0, 2, s2, c2); put(5, 2, s3, c3);
  chains(0, 0, s0, c0, 0, 1, s1, c1);
  chains(0, 2, s2, c2, 5, 2, s3, c3);
  flush(0); flush(1); flush(2); flush(3);
  // octaves 5-9 of x, y
  sincos_scaled2(x[0], 5, x[1], 5, &s0, &c0, &s1, &c1);
  put(5, 0, s0, c0); put(5, 1, s1, c1);
  chains(5, 0, s0, c0, 5, 1, s1, c1);
  flush(4); flush(5); flush(6); flush(7);
}

template <int W, class IO>
__device__ __forceinline__ void fetch_direction(const IO& io, const RowIn& row, uint4* de) {
  if (IO::kDirEnc) {
    if (row.valid) io.load_denc(row.idx, row.row, de);
    else de[0] = de[1] = de[2] = de[3] = make_uint4(0u, 0u, 0u, 0u);
  } else {
    encode_direction_h(row.d, de);
  }
}

__device__ __forceinline__ void QueryIO::load_denc(uint32_t idx, uint32_t row, uint4* de) const {
  float d[3];
  if (sdir) {
    const float4 q = sdir[row];
    d[0] = q.x; d[1] = q.y; d[2] = q.z;
  } else {
    const float* q = dir + 3ull * idx;
    d[0] = q[0]; d[1] = q[1]; d[2] = q[2];
  }
  encode_direction_h(d, de);
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int W, class IO>
__global__ void __launch_bounds__(TcCfg<W>::THREADS, TcCfg<W>::CTAS) k_mlp_tc(const uint8_t* __restrict__ packed,
                                                                              TileSched S, IO io) {
  using T = TcShape<W>;
  using C = TcCfg<W>;
  constexpr int NS = C::NS;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sb = smem_u32(smem);
  constexpr int NB = C::NBUF;
  const uint32_t bar_full = sb + C::BAR, bar_free = bar_full + 8 * NB, bar_mma = bar_free + 8 * NB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::TSLOT);
  uint4* runs = reinterpret_cast<uint4*>(smem + C::RUNS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = warp >> 2;  // warpgroup (TMEM slot); g == NS: the loader warp

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < NB; ++i) {
      mbar_init(bar_full + 8 * i, 1);
      // every warp of every group releases a run itself: a warp must never
      // lag two phases behind on full[] (parity aliasing), so the loader may
      // refill a buffer only once all 4*NS warps have left its run
      mbar_init(bar_free + 8 * i, GF_TC_WREL == 1 ? 4 * NS : NS);
    }
    for (int i = 0; i < NS; ++i) mbar_init(bar_mma + 8 * i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp < 4) {  // constant bias multiplier, row r = [1, 1, 0 ... 0] (fp16), lane quarter of this warp
    const uint32_t ta = tmem + C::ONES + ((uint32_t)(warp * 32) << 16);
    uint32_t o[8] = {0x3C003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
    GF_ST8(ta, o);
    tmem_wait_st();
  }
  fence_before();
  __syncthreads();
  fence_after();
  // setup above is private to this CTA (TMEM, barriers, constant operand):
  // it overlaps the previous kernel's tail under PDL
  gf_pdl_wait();

  const uint32_t nt = *S.n_tiles;
  const uint32_t per = (nt + gridDim.x - 1) / gridDim.x;
  const uint32_t t_begin = min(nt, blockIdx.x * per), t_end = min(nt, t_begin + per);

  if (g == NS) {
    // ---- loader warp: cut [t_begin, t_end) into runs of one cell; run r's
    // weights go to buffer r % NB once every group has released run r - NB
    uint32_t s = t_begin;
    for (uint32_t r = 0, k = 0;; ++r, k = k + 1 == NB ? 0 : k + 1) {
      uint32_t cell = 0, e = s;
      if (s < t_end) {
        cell = gf_tile_cell(S.tiles[s]);
        e = s + 1;
        for (;;) {
          if (e >= t_end) { e = t_end; break; }
          const uint32_t t = e + (uint32_t)lane;
          const bool diff = t >= t_end || gf_tile_cell(S.tiles[t]) != cell;
          const uint32_t m = __ballot_sync(0xffffffffu, diff);
          if (m) { e += (uint32_t)(__ffs(m) - 1); break; }
          e += 32;
        }
      }
      if (r >= NB) mbar_wait(bar_free + 8 * k, ((r - NB) / NB) & 1, 1);
      if (lane == 0) {
        runs[k] = make_uint4(cell, s, e, 0u);
        if (s < t_end) bulk_load(sb + k * T::CELL_BYTES, packed + (size_t)cell * T::CELL_BYTES, T::CELL_BYTES,
                                 bar_full + 8 * k);
        else mbar_arrive(bar_full + 8 * k);  // end of the range
      }
      __syncwarp();
      if (s >= t_end) break;
      s = e;
    }
  } else {
    // ---- warpgroup g: tiles t_begin + g, t_begin + g + NS, ... of the CTA's
    // range, up to R consecutive ones of the same run per pass (TMEM slots
    // g*R .. g*R + R-1): each thread owns row gt of every tile in flight, so
    // one barrier, one MMA commit and one wait per layer serve R tiles and
    // the R epilogues interleave
    constexpr int R = C::R;
    const int gt = tid & 127;
    const uint32_t lq = (uint32_t)((warp & 3) * 32) << 16;  // this warp's lane quarter
    const uint32_t slot0 = tmem + (uint32_t)(g * R * T::SLOT);
    const uint32_t ones = tmem + C::ONES;
    const uint32_t mbar = bar_mma + 8 * g;
    uint32_t ph = 0;
    // layer L's MMA chains for n tiles, issued by warp L % 4 of the group (one
    // elected lane): bias tile against the ones operand first (accumulator :=
    // bias), then the K steps; one commit for all of them
    auto issue = [&](int L, uint32_t wb, int n) {
      if ((warp & 3) != (L & 3)) return;
      fence_after();
      uint32_t b = wb + T::B1, bb = wb + T::BB1, idesc = idesc_f16(128, T::N1), acol = T::A1C;
      int K = T::K1;
      if (L == 0) { b = wb + T::B0; bb = wb + T::BB0; K = T::K0; idesc = idesc_f16(128, T::N0); acol = T::A0C; }
      if (L == 2) { b = wb + T::B2; bb = wb + T::BB2; K = T::K2; idesc = idesc_f16(128, T::N2); acol = T::A2C; }
      if (L == 3) { b = wb + T::B3; bb = wb + T::BB3; K = T::K3; idesc = idesc_f16(128, T::N3); acol = T::A3C; }
      if (L == 4) { b = wb + T::B4; bb = wb + T::BB4; K = T::K4; idesc = idesc_f16(128, T::N4); acol = T::A4C; }
#if (GF_EXP & 2)  // diagnostic: no tensor-core work, the commit barrier is arrived directly
      if (elect_one()) mbar_arrive(mbar);
      __syncwarp();
      return;
#endif
      if (elect_one()) {
        const uint64_t dbb = umma_desc(bb, 16), db = umma_desc(b, K);
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (j < n) {
            const uint32_t sl = slot0 + (uint32_t)(j * T::SLOT);
            mma_ts(sl, ones, dbb, idesc, 0u);
            // a K step of 16 columns: +8 TMEM columns of A, +256 B of B (+16 in
            // the descriptor's start-address field, no carry out of 14 bits)
#pragma unroll
            for (int ks = 0; ks < K / 16; ++ks) mma_ts(sl, sl + acol + 8 * ks, db + (uint64_t)(ks * 16), idesc, 1u);
          }
        }
        mma_commit(mbar);
      }
      __syncwarp();
    };
    auto wait_mma = [&]() {
      mbar_wait(mbar, ph, 2);
      ph ^= 1;
      fence_after();
    };
    // this group's TMEM stores done and its TMEM loads retired -> the MMA
    // issuer (named barrier over the group's 128 threads)
    auto publish = [&]() {
      tmem_wait_st();
      fence_before();
      asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
    };
    auto trow = [&](int j) { return slot0 + (uint32_t)(j * T::SLOT) + lq; };

    // before tile t the group releases every run ending at or before t (a
    // short run may hold none of its tiles) and waits for the weights of the
    // run holding t; rows are prefetched R tiles ahead, across runs
    uint32_t r = 0, k = 0, wb = sb, run_end = 0;
    mbar_wait(bar_full, 0, 3);
    run_end = runs[0].z;
    volatile uint32_t* ginfo = reinterpret_cast<volatile uint32_t*>(smem + C::GINFO);
    // leave run r for run r + 1 (group-uniform).  A warp waiting on full[]
    // must never lag two phases behind (parity aliasing): in mode 2 only the
    // group's first warp waits and releases, behind a group barrier that
    // proves all 4 warps are done with run r, and hands the new run's end to
    // the others through shared memory
    auto next_run = [&](int site) {
      if (GF_TC_WREL == 2) {
        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
        ++r;
        const uint32_t kp = k;
        k = k + 1 == NB ? 0 : k + 1;
        if ((warp & 3) == 0) {
          if (lane == 0) mbar_arrive(bar_free + 8 * kp);  // the group is done with run r - 1
          mbar_wait(bar_full + 8 * k, (r / NB) & 1, site);
          if (lane == 0) ginfo[g] = runs[k].z;
        }
        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
        run_end = ginfo[g];
      } else {
        __syncwarp();
        if (GF_TC_WREL == 1 ? lane == 0 : gt == 0) mbar_arrive(bar_free + 8 * k);
        ++r;
        k = k + 1 == NB ? 0 : k + 1;
        mbar_wait(bar_full + 8 * k, (r / NB) & 1, site);
        run_end = runs[k].z;
      }
      wb = sb + k * T::CELL_BYTES;
    };
    RowIn q[R];  // rows of this group's next R tiles
    uint32_t t = t_begin + (uint32_t)g;
#pragma unroll
    for (int j = 0; j < R; ++j)
      if (t + (uint32_t)(j * NS) < t_end) load_row(S, io, S.tiles[t + (uint32_t)(j * NS)], gt, q[j]);
    while (t < t_end) {
      while (t >= run_end) next_run(4);
      // tiles of this pass: t, t + NS, ... while they stay in this run
      int n = 1;
#pragma unroll
      for (int j = 1; j < R; ++j)
        if (n == j && t + (uint32_t)(j * NS) < run_end && t + (uint32_t)(j * NS) < t_end) n = j + 1;
      RowIn row[R];
#pragma unroll
      for (int j = 0; j < R; ++j) row[j] = q[j];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (j < n) {
#if (GF_EXP & 1)  // diagnostic: no encoding arithmetic, the operand gets the raw position
          const uint32_t xv = __float_as_uint(row[j].x[0]);
          GF_ST4(trow(j) + T::A0C, xv, xv, xv, xv);
#else
          encode_position<W>(trow(j) + T::A0C, row[j].x);
#endif
        }
      }
      publish();
      issue(0, wb, n);
      // refill the prefetch queue: the rows not consumed move up, the rest
      // load while this pass runs
      const uint32_t tn = t + (uint32_t)(n * NS);
#pragma unroll
      for (int j = 0; j < R; ++j) {
        if (j + n < R) {
          q[j] = row[j + n];
        } else if (tn + (uint32_t)(j * NS) < t_end) {
          load_row(S, io, S.tiles[tn + (uint32_t)(j * NS)], gt, q[j]);
        }
      }
      uint4 de[R][4];  // direction operand chunks, fetched one layer ahead of their use
      float sigma[R];
      constexpr int NL = 5;  // MMA layers
#pragma unroll
      for (int L = 0; L < NL; ++L) {
        wait_mma();
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (j >= n) continue;
          const uint32_t tr = trow(j);
          if (L == 0) {  // trunk0 -> h0
            epilogue_to_a<W, true>(tr, T::A1C);
          } else if (L == 1) {  // trunk1 -> h1
            epilogue_to_a<W, true>(tr, T::A2C);
            fetch_direction<W>(io, row[j], de[j]);  // in flight while the L2 MMA runs
          } else if (L == 2) {  // feature (cols 0..W-1, unactivated) + density (col W) -> [feat, gamma(d)]
            uint32_t z;
            GF_LD1(tr + W, z);
            epilogue_to_a<W, false>(tr, T::A3C);  // its first wait covers the density load too
            sigma[j] = fmaxf(__uint_as_float(z), 0.f);
            uint32_t o[8] = {de[j][0].x, de[j][0].y, de[j][0].z, de[j][0].w,
                             de[j][1].x, de[j][1].y, de[j][1].z, de[j][1].w};
            GF_ST8(tr + T::A3C + W / 2, o);
            uint32_t o2[8] = {de[j][2].x, de[j][2].y, de[j][2].z, de[j][2].w,
                              de[j][3].x, de[j][3].y, de[j][3].z, de[j][3].w};
            GF_ST8(tr + T::A3C + W / 2 + 8, o2);
          } else if (L == 3) {  // direction -> g
            epilogue_to_a<W, true>(tr, T::A4C);
          } else {  // color: sigmoid
            uint32_t z[4];
            GF_LD4(tr, z);
            tmem_wait_ld();
            float rgb[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {  // sign-split sigmoid (mlp.py:228-235): e = exp(-|v|), 1/(1+e) or e/(1+e)
              const float v = __uint_as_float(z[c]);
              float e, qv;
              asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-1.4426950408889634f * fabsf(v)));
              asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(qv) : "f"(1.f + e));
              rgb[c] = v >= 0.f ? qv : e * qv;
            }
            if (row[j].valid) io.store(row[j].idx, row[j].row, rgb[0], rgb[1], rgb[2], sigma[j]);
          }
        }
        if (L < NL - 1) {
          publish();
          issue(L + 1, wb, n);
        }
      }
      t = tn;
    }
    // release the current and any later runs (the loader waits on them
    // before it reuses their buffers; the end sentinel needs no release)
    for (;;) {
      if (GF_TC_WREL == 2 && run_end >= t_end) {  // the last run: release it (after the group barrier)
        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
        if (gt == 0) mbar_arrive(bar_free + 8 * k);
        break;
      }
      if (GF_TC_WREL != 2 && run_end >= t_end) {
        __syncwarp();
        if (GF_TC_WREL == 1 ? lane == 0 : gt == 0) mbar_arrive(bar_free + 8 * k);
        break;
      }
      next_run(5);
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)C::TMEM_COLS));
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
  // bias tiles: row n of layer L = [hi, lo, 0 ...] with hi = fp16(b), lo = fp16(b - hi)
  auto bias_of = [&](int L, int n) -> float {
    if (L == 0) return n < W ? A.b[0][cell * W + n] : 0.f;
    if (L == 1) return n < W ? A.b[1][cell * W + n] : 0.f;
    if (L == 2) return n < W ? A.b[3][cell * W + n] : (n == W ? A.b[2][cell] : 0.f);  // feature, then density
    if (L == 3) return n < W ? A.b[4][cell * W + n] : 0.f;
    return n < 3 ? A.b[5][cell * 3 + n] : 0.f;
  };
  const int bb[5] = {T::BB0, T::BB1, T::BB2, T::BB3, T::BB4}, nn[5] = {T::N0, T::N1, T::N2, T::N3, T::N4};
  for (int L = 0; L < 5; ++L) {
    for (int j = threadIdx.x; j < nn[L] * 16; j += blockDim.x) {
      const int n = j / 16, k = j % 16;
      float v = 0.f;
      if (k < 2) {
        const float b = bias_of(L, n);
        const float hi = __half2float(__float2half_rn(b));
        v = k == 0 ? hi : b - hi;
      }
      put(bb[L], 16, n, k, v);
    }
  }
  for (int j = T::BB4 + T::N4 * 32 + threadIdx.x; j < T::CELL_BYTES; j += blockDim.x) dst[j] = 0;
}

static bool tc_supported(const LayerTable& t) {
  return t.pos_dim == 63 && t.dir_dim == 27 && t.view == t.width && t.trunk == 2 && t.skip < 0 &&
         (t.width == 32 || t.width == 64);
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
static int tc_grid() {
  using C = TcCfg<W>;
  auto k = k_mlp_tc<W, IO>;
  static thread_local int grid = 0;
  if (grid == 0) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    // residency from first principles (the occupancy API reports 1 CTA/SM
    // here, apparently counting all 16 named barriers per CTA): shared
    // memory (+1 KiB reserved per CTA), registers, TMEM columns
    int dev = 0, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaFuncAttributes fa;
    int regs = 128;
    if (cudaFuncGetAttributes(&fa, k) == cudaSuccess && fa.numRegs > 0) regs = fa.numRegs;
    const int warps = (C::THREADS + 31) / 32;
    const int by_smem = smem_sm / (C::SMEM + 1024);
    const int by_regs = 65536 / (((regs + 7) / 8 * 8) * 32 * warps);
    const int by_warps = 64 / warps;
    int per_sm = by_smem < by_regs ? by_smem : by_regs;
    per_sm = per_sm < by_warps ? per_sm : by_warps;
    per_sm = per_sm < C::CTAS ? per_sm : C::CTAS;  // TMEM: CTAS x TMEM_COLS <= 512
    if (per_sm < 1) per_sm = 1;
    grid = num_sms() * per_sm;
    if (getenv("GF_DEBUG")) {
      fprintf(stderr, "[gf] k_mlp_tc<%d>: %d warpgroups + loader, smem %d B, regs %d, TMEM %d cols -> %d CTAs/SM\n", W,
              C::NS, C::SMEM, fa.numRegs, C::TMEM_COLS, per_sm);
    }
    cudaGetLastError();
  }
  return grid;
}

template <int W, class IO>
static void launch_tc_w(const void* packed, const TileSched& S, const IO& io, cudaStream_t st) {
  using C = TcCfg<W>;
  gf_launch_pdl(k_mlp_tc<W, IO>, dim3(tc_grid<W, IO>()), dim3(C::THREADS), (size_t)C::SMEM, st,
                (const uint8_t*)packed, S, io);
}

bool prepare_mlp_tc(const LayerTable& t) {
  if (!tc_supported(t)) return false;
  num_sms();
  if (t.width == 32) { tc_grid<32, RenderIO>(); tc_grid<32, QueryIO>(); }
  else { tc_grid<64, RenderIO>(); tc_grid<64, QueryIO>(); }
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
