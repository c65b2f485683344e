// Stable counting sort by key: batched.py:60-85 group_by_network
// (np.argsort(kind="stable"), inverse permutation, bincount + cumsum).
//
// Items are split into contiguous ranges, one warp per range.  Pass 1 counts
// keys per range into a (range x key) table; pass 2 scans the table in
// key-major order, which gives every (key, range) pair its first output slot
// and the segment offsets; pass 3 replays each range in input order, ranking
// equal keys inside 32-item chunks with __match_any_sync, so ties keep their
// arrival order exactly as the stable argsort does.
#include "gf_common.cuh"

namespace gf {

__global__ void __launch_bounds__(32) k_group_count(const int64_t* __restrict__ keys, int64_t n, int64_t n_keys,
                                                    int64_t per, uint32_t* table, int64_t* err) {
  const int64_t w = blockIdx.x;
  const int64_t lo = w * per, hi = min(n, lo + per);
  uint32_t* row = table + w * n_keys;
  for (int64_t i = lo + threadIdx.x; i < hi; i += 32) {
    int64_t k = keys[i];
    if (k < 0 || k >= n_keys) {
      atomicMin((unsigned long long*)err, (unsigned long long)i);
      continue;
    }
    atomicAdd(&row[k], 1u);
  }
}

// exclusive scan of table in key-major order: slot(key, w) = sum over
// (key' < key) + sum over (key, w' < w)
__global__ void __launch_bounds__(1024) k_group_scan(uint32_t* table, int64_t n_keys, int64_t n_warps,
                                                     int64_t* offsets) {
  __shared__ uint64_t wsum[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t carry = 0;
  const int64_t total = n_keys * n_warps;
  for (int64_t base = 0; base < total; base += 1024) {
    int64_t e = base + threadIdx.x;  // key-major flat index
    int64_t key = e / n_warps, w = e % n_warps;
    uint64_t v = e < total ? table[w * n_keys + key] : 0;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint64_t t = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      wsum[lane] = t;
    }
    __syncthreads();
    uint64_t ex = carry + (wid ? wsum[wid - 1] : 0) + x - v;
    if (e < total) {
      table[w * n_keys + key] = (uint32_t)ex;
      if (w == 0) offsets[key] = (int64_t)ex;
    }
    carry += wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) offsets[n_keys] = (int64_t)carry;
}

__global__ void __launch_bounds__(32) k_group_place(const int64_t* __restrict__ keys, int64_t n, int64_t n_keys,
                                                    int64_t per, uint32_t* table, int64_t* order, int64_t* inverse) {
  const int64_t w = blockIdx.x;
  const int64_t lo = w * per, hi = min(n, lo + per);
  uint32_t* row = table + w * n_keys;
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
        b = row[k];
        row[k] = b + __popc(peers);
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

size_t group_workspace(int64_t n, int64_t n_keys) { return gf_align((size_t)group_warps(n) * n_keys * 4); }

void launch_group(const int64_t* keys, int64_t n, int64_t n_keys, int64_t* order, int64_t* inverse,
                  int64_t* offsets, int64_t* err, void* ws, cudaStream_t st) {
  int64_t nw = group_warps(n);
  int64_t per = (n + nw - 1) / nw;
  uint32_t* table = (uint32_t*)ws;
  cudaMemsetAsync(table, 0, (size_t)nw * n_keys * 4, st);
  if (n > 0) k_group_count<<<(unsigned)nw, 32, 0, st>>>(keys, n, n_keys, per, table, err);
  k_group_scan<<<1, 1024, 0, st>>>(table, n_keys, nw, offsets);
  if (n > 0) k_group_place<<<(unsigned)nw, 32, 0, st>>>(keys, n, n_keys, per, table, order, inverse);
}

}  // namespace gf
