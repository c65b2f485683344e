// Stable counting sort by key: batched.py:60-85 group_by_network
// (np.argsort(kind="stable"), inverse permutation, bincount + cumsum).
//
// Items are split into contiguous ranges, one warp per range.  Pass 1 counts
// keys per range into a key-major (key x range) table; pass 2 scans the
// table in memory order (multi-CTA: per-CTA sums, their scan, then each
// CTA's slice), which gives every (key, range) pair its first output slot
// and the segment offsets; pass 3 replays each range in input order, ranking
// equal keys inside 32-item chunks with __match_any_sync, so ties keep their
// arrival order exactly as the stable argsort does.
#include "gf_common.cuh"

namespace gf {

__global__ void __launch_bounds__(32) k_group_count(const int64_t* __restrict__ keys, int64_t n, int64_t n_keys,
                                                    int64_t per, uint32_t* table, int64_t* err) {
  const int64_t w = blockIdx.x;
  const int64_t lo = w * per, hi = min(n, lo + per), nw = gridDim.x;
  for (int64_t i = lo + threadIdx.x; i < hi; i += 32) {
    int64_t k = keys[i];
    if (k < 0 || k >= n_keys) {
      atomicMin((unsigned long long*)err, (unsigned long long)i);
      continue;
    }
    atomicAdd(&table[k * nw + w], 1u);
  }
}

// exclusive scan of the key-major table: slot(key, w) = sum over (key' < key)
// + sum over (key, w' < w).  GS_ITEMS consecutive entries per CTA, 4 per thread.
#define GS_ITEMS 4096

__device__ __forceinline__ uint32_t block_scan_excl(uint32_t v, uint32_t* wsum, uint32_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
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
  total = wsum[31];
  const uint32_t r = (wid ? wsum[wid - 1] : 0u) + x - v;
  __syncthreads();  // wsum reusable
  return r;
}

__global__ void __launch_bounds__(1024) k_group_scan_sums(const uint32_t* __restrict__ table, uint32_t total,
                                                          uint32_t* sums) {
  __shared__ uint32_t wsum[32];
  const uint32_t e0 = blockIdx.x * GS_ITEMS + threadIdx.x * 4;
  uint32_t v = 0;
  if (e0 + 3 < total) {
    const uint4 q = *reinterpret_cast<const uint4*>(table + e0);
    v = q.x + q.y + q.z + q.w;
  } else {
    for (uint32_t j = 0; j < 4; ++j) v += e0 + j < total ? table[e0 + j] : 0u;
  }
  uint32_t tot;
  block_scan_excl(v, wsum, tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_group_scan_top(uint32_t* sums, uint32_t nb, int64_t n_keys,
                                                         int64_t* offsets) {
  __shared__ uint32_t wsum[32];
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < nb; b0 += 1024) {
    const uint32_t b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? sums[b] : 0u;
    uint32_t tot;
    const uint32_t ex = block_scan_excl(v, wsum, tot);
    if (b < nb) sums[b] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) offsets[n_keys] = (int64_t)carry;
}

__global__ void __launch_bounds__(1024) k_group_scan_apply(uint32_t* table, uint32_t total, uint32_t nw,
                                                           const uint32_t* __restrict__ sums, int64_t* offsets) {
  __shared__ uint32_t wsum[32];
  const uint32_t e0 = blockIdx.x * GS_ITEMS + threadIdx.x * 4;
  uint32_t v[4];
  for (uint32_t j = 0; j < 4; ++j) v[j] = e0 + j < total ? table[e0 + j] : 0u;
  uint32_t tot;
  uint32_t ex = sums[blockIdx.x] + block_scan_excl(v[0] + v[1] + v[2] + v[3], wsum, tot);
  for (uint32_t j = 0; j < 4; ++j) {
    const uint32_t e = e0 + j;
    if (e < total) {
      table[e] = ex;
      if (e % nw == 0) offsets[e / nw] = (int64_t)ex;
    }
    ex += v[j];
  }
}

__global__ void __launch_bounds__(32) k_group_place(const int64_t* __restrict__ keys, int64_t n, int64_t n_keys,
                                                    int64_t per, uint32_t* table, int64_t* order, int64_t* inverse) {
  const int64_t w = blockIdx.x;
  const int64_t lo = w * per, hi = min(n, lo + per), nw = gridDim.x;
  const unsigned lane = threadIdx.x;
  for (int64_t c = lo; c < hi; c += 32) {
    int64_t i = c + lane;
    bool p = i < hi;
    int64_t k = p ? keys[i] : 0;
    p = p && k >= 0 && k < n_keys;
    unsigned act = __ballot_sync(0xffffffffu, p);
    if (p) {
      unsigned peers = __match_any_sync(act, (unsigned long long)k);
      int leader = __ffs(peers) - 1;
      uint32_t b = 0;
      if ((int)lane == leader) {
        b = table[k * nw + w];
        table[k * nw + w] = b + __popc(peers);
      }
      b = __shfl_sync(peers, b, leader);
      int64_t pos = (int64_t)b + __popc(peers & ((1u << lane) - 1u));
      order[pos] = i;
      inverse[i] = pos;
    }
    __syncwarp();
  }
}

static int64_t group_warps(int64_t n) {
  int64_t w = (n + 2047) / 2048;
  return w < 1 ? 1 : (w > 4096 ? 4096 : w);
}

static uint32_t group_scan_blocks(int64_t n, int64_t n_keys) {
  return (uint32_t)((group_warps(n) * n_keys + GS_ITEMS - 1) / GS_ITEMS);
}

size_t group_workspace(int64_t n, int64_t n_keys) {
  return gf_align((size_t)group_warps(n) * n_keys * 4) + gf_align((size_t)group_scan_blocks(n, n_keys) * 4 + 4);
}

void launch_group(const int64_t* keys, int64_t n, int64_t n_keys, int64_t* order, int64_t* inverse,
                  int64_t* offsets, int64_t* err, void* ws, cudaStream_t st) {
  const int64_t nw = group_warps(n);
  const int64_t per = (n + nw - 1) / nw;
  uint32_t* table = (uint32_t*)ws;
  uint32_t* sums = (uint32_t*)((char*)ws + gf_align((size_t)nw * n_keys * 4));
  const uint32_t total = (uint32_t)(nw * n_keys), nb = group_scan_blocks(n, n_keys);
  cudaMemsetAsync(table, 0, (size_t)total * 4, st);
  if (n > 0) k_group_count<<<(unsigned)nw, 32, 0, st>>>(keys, n, n_keys, per, table, err);
  if (nb > 0) k_group_scan_sums<<<nb, 1024, 0, st>>>(table, total, sums);
  k_group_scan_top<<<1, 1024, 0, st>>>(sums, nb, n_keys, offsets);
  if (nb > 0) k_group_scan_apply<<<nb, 1024, 0, st>>>(table, total, (uint32_t)nw, sums, offsets);
  if (n > 0) k_group_place<<<(unsigned)nw, 32, 0, st>>>(keys, n, n_keys, per, table, order, inverse);
}

}  // namespace gf
