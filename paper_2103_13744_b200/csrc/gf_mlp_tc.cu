// Fused positional-encoding + tiny-MLP on the 5th-gen tensor cores (sm_100a).
//
// Reference math: core.py:132-152 (encoding), mlp.py:222-266 (forward),
// batched.py:120-151 (one network per segment).  Design:
//
//  * one CTA = 256 threads = two warpgroups working on TWO 128-row tiles of
//    the same cell at once: group g owns tile slot g (its A operands, its
//    TMEM columns, its MMA commit barrier and its own elected issuing
//    thread); thread gt of a group owns row gt, which is TMEM lane gt, so
//    every epilogue is a private tcgen05.ld of the thread's own accumulator
//    row.  While the tensor core runs one group's layer the other group runs
//    its epilogue, hiding the MMA / commit / barrier latency of the 5-layer
//    dependency chain; groups synchronise with named barriers, the CTA only
//    at tile-pair boundaries (weight reuse);
//  * epilogues: FADD2 bias adds, F2FP.RELU packs, 16-byte operand stores;
//    the render path's direction chunk gamma(d) is encoded once per ray by
//    k_ray_init and copied, not recomputed per sample;
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
  // constant ONES tile (columns 0 and 1 = 1) they initialise the accumulator
  static constexpr int BB0 = B4 + N4 * K4 * 2;
  static constexpr int BB1 = BB0 + N0 * 32;
  static constexpr int BB2 = BB1 + N1 * 32;
  static constexpr int BB3 = BB2 + N2 * 32;
  static constexpr int BB4 = BB3 + N3 * 32;
  static constexpr int CELL_BYTES = ((BB4 + N4 * 32) + 1023) / 1024 * 1024;
  static constexpr int ONES = CELL_BYTES;  // 128 x 16 fp16 constant A operand
  // one A operand slot per tile, re-laid out in place layer by layer:
  // gamma(x) (K0) -> h0 (K1) -> h1 (K2) -> [feat, gamma(d)] (K3) -> g (K4)
  static constexpr int KA = K0 > K3 ? K0 : K3;
  static constexpr int SLOT_BYTES = 128 * KA * 2;
  static constexpr int A(int s) { return ONES + 4096 + s * SLOT_BYTES; }
  static constexpr int BAR = A(2);  // mma[0], mma[1], weights, tmem base
  // window of the CTA's tile descriptors (refilled at pair boundaries): tile
  // reads at the top of each pair are shared-memory loads, not global ones
  static constexpr int TILEBUF = BAR + 32;
  static constexpr int TB = 64;
  static constexpr int SMEM = TILEBUF + TB * 8;
  static constexpr int NC = N2 <= 32 ? 32 : (N2 <= 64 ? 64 : (N2 <= 128 ? 128 : 256));  // TMEM cols per slot
  static constexpr int TMEM_COLS = 2 * NC;
#if GF_EXP == 10
  static constexpr int CTAS_PER_SM = W == 32 ? 3 : 2;
#else
  static constexpr int CTAS_PER_SM = W == 32 ? 4 : 2;
#endif
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

// parity wait with a suspend-time hint: the warp sleeps in the barrier unit
// until the phase flips (or the hint expires) instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done;
  do {
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

// accumulator columns [c0, c0 + N) of this thread's TMEM row -> fp16 (+ReLU)
// into a canonical operand of K columns, 16 columns per TMEM load so only 16
// accumulator registers are live
template <int N, bool RELU>
__device__ __forceinline__ void tmem_to_operand(uint32_t trow, uint8_t* A, int K, int r) {
#pragma unroll
  for (int c = 0; c < N; c += 16) {
    float h[16];
    tmem_load<16>(trow + c, h);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float* v = h + 8 * q;
      uint4 o;
      if (RELU) {
        o = make_uint4(pack_h2_relu(v[0], v[1]), pack_h2_relu(v[2], v[3]), pack_h2_relu(v[4], v[5]),
                       pack_h2_relu(v[6], v[7]));
      } else {
        o = make_uint4(pack_h2(v[0], v[1]), pack_h2(v[2], v[3]), pack_h2(v[4], v[5]), pack_h2(v[6], v[7]));
      }
      *reinterpret_cast<uint4*>(A + canon_off(r, c + 8 * q, K)) = o;
    }
  }
}

// fp16 store (+ReLU) of accumulator columns [0, N) of row r into a
// canonical operand of K columns: per 8 columns four F2FP(.RELU) packs and
// one 16-byte store (the bias is already in the accumulator)
template <int N, bool RELU>
__device__ __forceinline__ void pack_store(const float* h, uint8_t* A, int K, int r) {
#pragma unroll
  for (int c = 0; c < N / 8; ++c) {
    const float* v = h + 8 * c;
    uint4 o;
    if (RELU) {
      o = make_uint4(pack_h2_relu(v[0], v[1]), pack_h2_relu(v[2], v[3]), pack_h2_relu(v[4], v[5]),
                     pack_h2_relu(v[6], v[7]));
    } else {
      o = make_uint4(pack_h2(v[0], v[1]), pack_h2(v[2], v[3]), pack_h2(v[4], v[5]), pack_h2(v[6], v[7]));
    }
    *reinterpret_cast<uint4*>(A + canon_off(r, 8 * c, K)) = o;
  }
}

// one row's inputs (prefetched one pair ahead); the render path's direction
// operand chunk (the ray's pre-encoded gamma(d), gf_encode.cuh) is fetched
// separately while the trunk0 MMA runs
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
// xyz; column 63 zero) generated octave by octave and flushed to the K0
// operand one 8-column chunk at a time, so only ~14 values are live
// gamma(x) (core.py:132-152 layout: raw xyz, then per octave k sin xyz, cos
// xyz; column 63 zero).  Anchors k = 0, 3, 6, 9 (MUFU after exact
// reduction), two double-angle steps after each of the first three; anchors
// and chains run as f32x2 pairs, in octave order, and every completed
// 8-column chunk is flushed to the K0 operand at once (few live registers).
template <int W>
__device__ __forceinline__ void encode_position(uint8_t* A0, int tid, const float* x) {
  using T = TcShape<W>;
  float e[64];
  e[0] = x[0]; e[1] = x[1]; e[2] = x[2];
  e[63] = 0.f;
  auto put = [&](int k, int a, float sv, float cv) {
    e[3 + 6 * k + a] = sv;
    e[6 + 6 * k + a] = cv;
  };
  auto flush = [&](int c) {
    const float* v = e + 8 * c;
    *reinterpret_cast<uint4*>(A0 + canon_off(tid, 8 * c, T::K0)) =
        make_uint4(pack_h2(v[0], v[1]), pack_h2(v[2], v[3]), pack_h2(v[4], v[5]), pack_h2(v[6], v[7]));
  };
  // two chains of two double-angle steps from anchors (ka, aa), (kb, ab)
  auto chains = [&](int ka, int aa, float sa, float ca, int kb, int ab, float sb, float cb) {
    F2 sv = f2(sa, sb), cv = f2(ca, cb);
#pragma unroll
    for (int st = 1; st <= 2; ++st) {
      double_angle2(sv, cv);
      float s0, s1, c0, c1;
      f2_split(sv, s0, s1);
      f2_split(cv, c0, c1);
      put(ka + st, aa, s0, c0);
      put(kb + st, ab, s1, c1);
    }
  };
  float s0, c0, s1, c1, s2, c2, s3, c3;
  // octaves 0-2 (and z of 3-5)
  sincos_scaled2(x[0], 0, x[1], 0, &s0, &c0, &s1, &c1);
  sincos_scaled2(x[2], 0, x[2], 3, &s2, &c2, &s3, &c3);
  put(0, 0, s0, c0); put(0, 1, s1, c1); put(0, 2, s2, c2); put(3, 2, s3, c3);
  chains(0, 0, s0, c0, 0, 1, s1, c1);
  chains(0, 2, s2, c2, 3, 2, s3, c3);
  flush(0); flush(1);
  // octaves 3-5
  sincos_scaled2(x[0], 3, x[1], 3, &s0, &c0, &s1, &c1);
  put(3, 0, s0, c0); put(3, 1, s1, c1);
  chains(3, 0, s0, c0, 3, 1, s1, c1);
  flush(2); flush(3);
  // octaves 6-8 (and z of 9)
  sincos_scaled2(x[0], 6, x[1], 6, &s0, &c0, &s1, &c1);
  sincos_scaled2(x[2], 6, x[2], 9, &s2, &c2, &s3, &c3);
  put(6, 0, s0, c0); put(6, 1, s1, c1); put(6, 2, s2, c2); put(9, 2, s3, c3);
  chains(6, 0, s0, c0, 6, 1, s1, c1);
#pragma unroll
  for (int st = 1; st <= 2; ++st) {  // 6z alone (scalar, same roundings)
    const float sp = s2, cp = c2;
    s2 = 2.0f * sp * cp;
    c2 = (cp - sp) * (cp + sp);
    put(6 + st, 2, s2, c2);
  }
  flush(4); flush(5); flush(6);
  // octave 9
  sincos_scaled2(x[0], 9, x[1], 9, &s0, &c0, &s1, &c1);
  put(9, 0, s0, c0); put(9, 1, s1, c1);
  flush(7);
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

template <int W>
__device__ __forceinline__ void store_direction(uint8_t* A3, int tid, const uint4* de) {
  using T = TcShape<W>;
  static_assert(T::K3 - W == 32, "direction operand chunk is 32 fp16 wide");
#pragma unroll
  for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(A3 + canon_off(tid, W + 8 * q, T::K3)) = de[q];
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
__global__ void __launch_bounds__(256, TcShape<W>::CTAS_PER_SM) k_mlp_tc(const uint8_t* __restrict__ packed,
                                                                         TileSched S, IO io) {
  using T = TcShape<W>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t bar0 = smem_u32(smem + T::BAR), bar_w = bar0 + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + T::BAR + 24);
  const int tid = threadIdx.x, warp = tid >> 5;
  // two warpgroups: group g owns tile slot g (its A operand, its TMEM
  // columns, its commit barrier); row gt of the tile is TMEM lane gt
  const int g = tid >> 7, gt = tid & 127;

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
  {  // constant bias multiplier: row r = [1, 1, 0 ... 0]
    const int r = tid >> 1, c = tid & 1;
    *reinterpret_cast<uint4*>(smem + T::ONES + canon_off(r, 8 * c, 16)) =
        c ? make_uint4(0u, 0u, 0u, 0u) : make_uint4(0x3C003C00u, 0u, 0u, 0u);
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  // setup above is private to this CTA (TMEM, barriers, constant tile): it
  // overlaps the previous kernel's tail under PDL; its results are read below
  gf_pdl_wait();
  const uint32_t tmem = *tmem_slot;
  const uint32_t wb = smem_u32(smem);
  uint8_t* Ag = smem + T::A(g);
  const uint32_t trow = tmem + g * T::NC + ((uint32_t)((warp & 3) * 32) << 16);  // lane quarter of this warp

  const uint32_t nt = *S.n_tiles;
  const uint32_t per = (nt + gridDim.x - 1) / gridDim.x;
  const uint32_t t_begin = blockIdx.x * per, t_end = min(nt, t_begin + per);
  uint2* s_tiles = reinterpret_cast<uint2*>(smem + T::TILEBUF);
  uint32_t tbase = t_begin;
  auto fill_tiles = [&](uint32_t from) {  // all threads, then a CTA barrier
    tbase = from;
    for (uint32_t j = tid; j < (uint32_t)T::TB && from + j < t_end; j += blockDim.x) s_tiles[j] = S.tiles[from + j];
    __syncthreads();
  };
  fill_tiles(t_begin);
  auto tile_at = [&](uint32_t u) -> uint2 { return s_tiles[u - tbase]; };
  int cur = -1;
  uint32_t ph = 0, ph_w = 0;

  // MMA chain of layer L for this group's slot (thread gt == 0 of the group):
  // bias tile first (accumulator := bias), then the K steps
  auto issue = [&](int L) {
#if GF_EXP == 3
    if (gt == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar0 + 8 * g) : "memory");
    return;
#endif
    if (gt != 0) return;
    const uint32_t a = wb + T::A(g), d = tmem + g * T::NC;
    uint32_t b = wb + T::B1, bb = wb + T::BB1, idesc = idesc_f16(128, T::N1);
    int K = T::K1;
    if (L == 0) { b = wb + T::B0; bb = wb + T::BB0; K = T::K0; idesc = idesc_f16(128, T::N0); }
    if (L == 2) { b = wb + T::B2; bb = wb + T::BB2; K = T::K2; idesc = idesc_f16(128, T::N2); }
    if (L == 3) { b = wb + T::B3; bb = wb + T::BB3; K = T::K3; idesc = idesc_f16(128, T::N3); }
    if (L == 4) { b = wb + T::B4; bb = wb + T::BB4; K = T::K4; idesc = idesc_f16(128, T::N4); }
    mma_f16(d, umma_desc(wb + T::ONES, 16), umma_desc(bb, 16), idesc, 0u);
    // a K step of 16 columns is 256 B further in both operands: +16 in the
    // descriptors' start-address field (>> 4), no carry out of 14 bits
    const uint64_t da = umma_desc(a, K), db = umma_desc(b, K);
    for (int ks = 0; ks < K / 16; ++ks) mma_f16(d, da + (uint64_t)(ks * 16), db + (uint64_t)(ks * 16), idesc, 1u);
    mma_commit(bar0 + 8 * g);
  };
  auto wait_mma = [&]() {
    mbar_wait(bar0 + 8 * g, ph);
    ph ^= 1;
    fence_after();
  };
  // this group's smem operand writes -> visible to the tensor core; its TMEM
  // reads retired (named barrier over the group's 128 threads)
  auto publish = [&]() {
    fence_async_smem();
    fence_before();
    asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
    fence_after();
  };
  // tile of this group inside the pair starting at t (slot 1 only for a
  // second tile of the same cell: both slots share the staged weights)
  auto second = [&](uint32_t t, uint32_t cell) -> bool {
    return t + 1 < t_end && gf_tile_cell(tile_at(t + 1)) == cell;
  };
  auto my_tile = [&](uint32_t t, uint2& tl) -> bool {
    if (t >= t_end) return false;
    tl = tile_at(t);
    if (g == 0) return true;
    if (!second(t, gf_tile_cell(tl))) return false;
    tl = tile_at(t + 1);
    return true;
  };

  RowIn nxt;
  {
    uint2 tl;
    if (my_tile(t_begin, tl)) load_row(S, io, tl, gt, nxt);
  }

  for (uint32_t t = t_begin; t < t_end;) {
    __syncthreads();  // previous pair fully retired (weight operands and the tile window may be replaced)
    if (t + 4 > tbase + (uint32_t)T::TB && tbase + (uint32_t)T::TB < t_end) fill_tiles(t);  // CTA-uniform
    const uint32_t cell = gf_tile_cell(tile_at(t));
    const bool two = second(t, cell);
    const uint32_t t_next = t + (two ? 2 : 1);
    const bool active = g == 0 || two;
    const bool new_cell = (int)cell != cur;
    if (new_cell && tid == 0) bulk_load(wb, packed + (size_t)cell * T::CELL_BYTES, T::CELL_BYTES, bar_w);
    cur = (int)cell;
    const RowIn row = nxt;
    if (active) {
#if GF_EXP == 1
      for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(Ag + canon_off(gt, 8 * c, T::K0)) = make_uint4(__float_as_uint(row.x[0]), 0u, 0u, 0u);
#else
      encode_position<W>(Ag, gt, row.x);
#endif
      publish();
    }
    if (new_cell) {
      mbar_wait(bar_w, ph_w);
      ph_w ^= 1;
    }
    if (active) issue(0);
    {  // prefetch this group's row of the next pair while trunk0 runs
      uint2 tn;
      if (my_tile(t_next, tn)) load_row(S, io, tn, gt, nxt);
    }
    if (active) {
      float sigma = 0.f;
      uint4 de[4];  // direction operand chunk, fetched one layer ahead of its use
#pragma unroll
      for (int L = 0; L < 5; ++L) {
        wait_mma();
        if (L == 0) {  // trunk0 -> h0 (K1 layout, over the dead gamma(x))
          tmem_to_operand<W, true>(trow, Ag, T::K1, gt);
        } else if (L == 1) {  // trunk1 -> h1 (K2 layout)
          tmem_to_operand<W, true>(trow, Ag, T::K2, gt);
          fetch_direction<W>(io, row, de);  // in flight while the L2 MMA runs
        } else if (L == 2) {  // feature (cols 0..W-1, unactivated) + density (col W) -> [feat, gamma(d)] (K3)
          store_direction<W>(Ag, gt, de);
          tmem_to_operand<W, false>(trow, Ag, T::K3, gt);
          float z[16];
          tmem_load<16>(trow + W, z);
          sigma = fmaxf(z[0], 0.f);
        } else if (L == 3) {  // direction -> g (K4 layout)
          tmem_to_operand<W, true>(trow, Ag, T::K4, gt);
        } else {  // color: sigmoid
          float z[16];
          tmem_load<16>(trow, z);
          float rgb[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const float v = z[c];
            const float e = __expf(-fabsf(v)), r = __fdividef(1.f, 1.f + e);  // sign-split sigmoid (mlp.py:228-235)
            rgb[c] = v >= 0.f ? r : e * r;
          }
          if (row.valid) io.store(row.idx, row.row, rgb[0], rgb[1], rgb[2], sigma);
        }
        if (L < 4) {
          publish();
          issue(L + 1);
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
    const int by_regs = 65536 / (((regs + 7) / 8 * 8) * 256);
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
  gf_launch_pdl(k_mlp_tc<W, IO>, dim3(num_sms() * tc_resident<W, IO>()), dim3(256), (size_t)T::SMEM, st,
                (const uint8_t*)packed, S, io);
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
