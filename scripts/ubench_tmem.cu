// Microbenchmark: TMEM load/store throughput and small-N tcgen05.mma rates
// (A from shared memory vs A from TMEM) on one B200 SM -- the constants that
// decide the tiny-MLP kernel's structure (DESIGN.md §5 K3).
//
//   nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o ubench_tmem scripts/ubench_tmem.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define LD16(taddr, r)                                                                                         \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, " \
               "[%16];"                                                                                        \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),           \
                 "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),       \
                 "=r"(r[14]), "=r"(r[15])                                                                      \
               : "r"(taddr))
#define ST16(taddr, r)                                                                                          \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),      \
               "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),     \
               "r"(r[15]))

__device__ __forceinline__ void alloc512(uint32_t* slot, uint32_t ncols = 512) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
}
__device__ __forceinline__ void free512(uint32_t t, uint32_t ncols = 512) {
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(ncols));
}

// MODE 0: ld x16 + wait each; MODE 1: 4 x ld x16 then one wait; MODE 2: st x16 + wait::st; MODE 3: 4 x st then wait
template <int MODE>
__global__ void k_tmem_bw(int iters, unsigned long long* cyc, uint32_t* sink) {
  extern __shared__ uint32_t sm[];
  alloc512(sm);
  const uint32_t tmem = sm[0];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint32_t lane_q = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col = (uint32_t)((warp >> 2) * 64) & 511u;
  const uint32_t ta = tmem + lane_q + col;
  uint32_t acc = 0, r[16], q[16], s[16], u[16];
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * 7 + i;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
      LD16(ta, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= r[0] ^ r[15];
    } else if (MODE == 1) {
      LD16(ta, r);
      LD16(ta + 16, q);
      LD16(ta + 32, s);
      LD16(ta + 48, u);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc ^= r[0] ^ q[15] ^ s[3] ^ u[7];
    } else if (MODE == 2) {
      r[0] += it;
      ST16(ta, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else {
      r[0] += it;
      ST16(ta, r);
      ST16(ta + 16, r);
      ST16(ta + 32, r);
      ST16(ta + 48, r);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  (void)nw;
  free512(tmem);
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, int K) {
  const uint64_t lbo = 128, sbo = (uint64_t)K * 16;
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((lbo >> 4) << 16) | ((sbo >> 4) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// one thread issues `iters` M=128 x N x K=16 MMAs into one accumulator; A from
// smem (TS=0) or TMEM (TS=1); commit + wait every `batch`
template <int N, int TS>
__global__ void k_mma_rate(int iters, int batch, unsigned long long* cyc, int nd, int cols) {
  extern __shared__ __align__(1024) uint8_t smb[];
  uint32_t* slot = reinterpret_cast<uint32_t*>(smb + 65536);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smb + 65536 + 64);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  alloc512(slot, cols);
  const uint32_t tmem = *slot;
  unsigned long long t0 = 0, t1 = 0;
  const uint32_t dstride = (uint32_t)(cols / 2 / nd);
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smb), b = smem_u32(smb + 32768);
    const uint64_t da = umma_desc(a, 64), db = umma_desc(b, 64);
    const uint32_t id = idesc_f16(128, N);
    uint32_t ph = 0;
    t0 = clock64();
    for (int it = 0; it < iters; it += batch) {
      for (int j = 0; j < batch; ++j) {
        const uint64_t dbj = db + (uint64_t)((j & 3) * 16);
        if (TS) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem + (j % nd) * dstride),
              "r"(tmem + (uint32_t)cols / 2 + (uint32_t)((j & 3) * 8)), "l"(dbj), "r"(id), "r"(1u));
        } else {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + (j % nd) * dstride),
              "l"(da + (uint64_t)((j & 3) * 16)), "l"(dbj), "r"(id), "r"(1u));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                   : "memory");
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(ph)
            : "memory");
      }
      ph ^= 1;
    }
    t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  free512(tmem, cols);
}

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n"
      : "+r"(pred));
  return pred;
}

// unrolled issue: ND accumulators in rotation, 16 MMAs per commit; WARP=1:
// warp 0 runs the loop and elect.sync picks the issuing lane
template <int N, int TS, int ND, int WARP>
__global__ void k_mma_rate2(int iters, unsigned long long* cyc, int cols) {
  extern __shared__ __align__(1024) uint8_t smb[];
  uint32_t* slot = reinterpret_cast<uint32_t*>(smb + 65536);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smb + 65536 + 64);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  alloc512(slot, cols);
  const uint32_t tmem = *slot;
  const bool run = WARP ? (threadIdx.x >> 5) == 0 : threadIdx.x == 0;
  if (run) {
    const uint32_t a = smem_u32(smb), b = smem_u32(smb + 32768);
    const uint64_t da = umma_desc(a, 64), db = umma_desc(b, 64);
    const uint32_t id = idesc_f16(128, N);
    const uint32_t ta = tmem + (uint32_t)cols / 2;
    uint32_t ph = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it += 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t d = tmem + (uint32_t)((j % ND) * N);
        const uint64_t dbj = db + (uint64_t)((j & 3) * 16);
        if (!WARP || elect_one()) {
          if (TS) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
                "r"(ta + (uint32_t)((j & 3) * 8)), "l"(dbj), "r"(id), "r"(1u));
          } else {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
                "l"(da + (uint64_t)((j & 3) * 16)), "l"(dbj), "r"(id), "r"(1u));
          }
        }
        if (WARP) __syncwarp();
      }
      if (!WARP || elect_one())
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                     : "memory");
      if (WARP) __syncwarp();
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(ph)
            : "memory");
      }
      ph ^= 1;
    }
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  }
  free512(tmem, cols);
}

static double med(unsigned long long* h, int n) {
  double s = 0;
  for (int i = 0; i < n; ++i) s += (double)h[i];
  return s / n;
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int nsm = 148, iters = 4096;
  unsigned long long *d_cyc, h[148];
  uint32_t* sink;
  cudaMalloc(&d_cyc, sizeof(h));
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int smem = 150 * 1024;  // one CTA per SM
  cudaFuncSetAttribute(k_tmem_bw<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tmem_bw<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tmem_bw<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tmem_bw<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[4] = {"ld x16 +wait", "ld 4x16 +wait", "st x16 +wait", "st 4x16 +wait"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int warps = 4; warps <= 32; warps *= 2) {
      void (*k)(int, unsigned long long*, uint32_t*) =
          mode == 0 ? k_tmem_bw<0> : mode == 1 ? k_tmem_bw<1> : mode == 2 ? k_tmem_bw<2> : k_tmem_bw<3>;
      k<<<nsm, warps * 32, smem>>>(iters, d_cyc, sink);
      k<<<nsm, warps * 32, smem>>>(iters, d_cyc, sink);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d_cyc, sizeof(h), cudaMemcpyDeviceToHost);
      const double c = med(h, nsm);
      const double bytes = (double)warps * 32 * 16 * 4 * iters * (mode & 1 ? 4 : 1);
      printf("TMEM %-14s warps/SM %2d: %8.0f cyc, %7.1f B/cyc/SM, %6.1f cyc per warp-op (%s)\n", names[mode], warps, c,
             bytes / c, c / iters, cudaGetErrorString(e));
    }
  }
  // (N, TS, distinct accumulators nd, CTAs per SM): smem 65 KB per CTA
#define RUN_MMA(N, TS, ND, CPS)                                                                            \
  {                                                                                                        \
    const int cols = 512 / CPS;                                                                            \
    const int msmem = (CPS == 1 ? 150 * 1024 : (CPS == 2 ? 100 * 1024 : 66 * 1024));                       \
    cudaFuncSetAttribute(k_mma_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, msmem);           \
    const int batch = 64;                                                                                  \
    k_mma_rate<N, TS><<<nsm * CPS, 128, msmem>>>(iters, batch, d_cyc2, ND, cols);                          \
    k_mma_rate<N, TS><<<nsm * CPS, 128, msmem>>>(iters, batch, d_cyc2, ND, cols);                          \
    cudaError_t e = cudaDeviceSynchronize();                                                               \
    cudaMemcpy(h2, d_cyc2, sizeof(unsigned long long) * nsm * CPS, cudaMemcpyDeviceToHost);                \
    const double c = med(h2, nsm * CPS);                                                                   \
    printf("MMA M=128 N=%3d %s accs %d CTAs/SM %d: %6.2f cyc/MMA per CTA, SM rate %7.0f MAC/cyc (floor %d cyc) (%s)\n", \
           N, TS ? "A=TMEM" : "A=SMEM", ND, CPS, c / iters, CPS * 128.0 * N * 16 * iters / c, 128 * N / 256,        \
           cudaGetErrorString(e));                                                                         \
  }
  unsigned long long *d_cyc2, h2[148 * 8];
  cudaMalloc(&d_cyc2, sizeof(h2));
#define RUN2(N, TS, ND, W, CPS)                                                                               \
  {                                                                                                        \
    const int cols = 512 / CPS;                                                                            \
    const int msmem = (CPS == 1 ? 150 * 1024 : (CPS == 2 ? 100 * 1024 : (CPS == 4 ? 50 * 1024 : 26 * 1024))); \
    cudaFuncSetAttribute(k_mma_rate2<N, TS, ND, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, msmem);   \
    k_mma_rate2<N, TS, ND, W><<<nsm * CPS, 128, msmem>>>(iters, d_cyc2, cols);                              \
    k_mma_rate2<N, TS, ND, W><<<nsm * CPS, 128, msmem>>>(iters, d_cyc2, cols);                              \
    cudaError_t e = cudaDeviceSynchronize();                                                               \
    cudaMemcpy(h2, d_cyc2, sizeof(unsigned long long) * nsm * CPS, cudaMemcpyDeviceToHost);                \
    const double c = med(h2, nsm * CPS);                                                                   \
    printf("MMA2 N=%3d %s accs %d %s CTAs/SM %d: %6.2f cyc/MMA per CTA, SM %6.2f cyc/MMA, %5.0f MAC/cyc (floor %d) (%s)\n", N, \
           TS ? "A=TMEM" : "A=SMEM", ND, W ? "warp+elect" : "thread0   ", CPS, c / iters, c / iters / CPS,           \
           CPS * 128.0 * N * 16 * iters / c, 128 * N / 256, cudaGetErrorString(e));                         \
  }
  RUN2(32, 1, 1, 0, 1) RUN2(32, 1, 1, 1, 1) RUN2(32, 1, 4, 0, 1) RUN2(32, 1, 4, 1, 1)
  RUN2(32, 0, 1, 1, 1) RUN2(32, 0, 4, 1, 1)
  RUN2(32, 1, 1, 1, 2) RUN2(32, 1, 1, 1, 4) RUN2(32, 1, 1, 1, 8) RUN2(32, 1, 2, 1, 4)
  RUN2(32, 0, 1, 1, 4) RUN2(32, 0, 1, 1, 8)
  RUN2(16, 1, 1, 1, 1) RUN2(16, 1, 4, 1, 1) RUN2(16, 1, 1, 1, 8)
  RUN2(48, 1, 1, 1, 1) RUN2(48, 1, 2, 1, 1) RUN2(48, 1, 1, 1, 4)
  RUN2(64, 1, 1, 1, 1) RUN2(64, 1, 2, 1, 1) RUN2(64, 1, 1, 1, 4)
  RUN2(128, 1, 1, 1, 1) RUN2(128, 1, 1, 1, 2)
  return 0;
}
