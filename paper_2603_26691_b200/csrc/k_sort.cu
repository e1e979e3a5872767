// KB3 (general form) — stable counting sort of the SoA store by chunk id
// (C-15: ties keep the prior store order).  LSD radix with 8-bit digits; each
// pass is  count (per block, per warp, per digit)  ->  exclusive scan over
// (digit, block)  ->  stable scatter of the full payload (x, u, d, w, id, key).
// Within a block of 4096 items each warp owns 512 consecutive items and ranks
// equal digits with __match_any_sync, so the order is deterministic and stable.
// Used at injection (arbitrary displacement) and as the fallback rebin.
#include <cuda_runtime.h>

#include "st_internal.h"

namespace st {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kPerWarp = 512;
constexpr int kItems = kWarps * kPerWarp;   // 4096 items per block
constexpr int kRadix = 256;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Per-warp digit counts of this block's items into cnt[warp][digit].
__device__ __forceinline__ void warp_counts(const int32_t* __restrict__ key, int64_t n, int shift, int64_t blk0,
                                            uint32_t (*cnt)[kRadix]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t w0 = blk0 + (int64_t)warp * kPerWarp;
  for (int b = 0; b < kPerWarp; b += 32) {
    const int64_t i = w0 + b + lane;
    const bool valid = i < n;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!act) break;
    if (valid) {
      const int dg = (key[i] >> shift) & (kRadix - 1);
      const unsigned peers = __match_any_sync(act, dg);
      if ((peers & lanemask_lt()) == 0) cnt[warp][dg] += __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads) k_sort_count(const int32_t* __restrict__ key, int64_t n, int shift,
                                                         int64_t nblocks, uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[kWarps][kRadix];
  const int64_t blk0 = (int64_t)blockIdx.x * kItems;
  warp_counts(key, n, shift, blk0, cnt);
  for (int dg = threadIdx.x; dg < kRadix; dg += kThreads) {
    uint32_t s = 0;
    for (int w = 0; w < kWarps; ++w) s += cnt[w][dg];
    hist[(int64_t)dg * nblocks + blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kThreads) k_sort_scatter(Store src, Store dst, int64_t cap,
                                                           const int32_t* __restrict__ key,
                                                           int32_t* __restrict__ key_dst, int64_t n, int shift,
                                                           int64_t nblocks, const int64_t* __restrict__ offs) {
  __shared__ uint32_t cnt[kWarps][kRadix];
  __shared__ int64_t base[kWarps][kRadix];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t blk0 = (int64_t)blockIdx.x * kItems;
  warp_counts(key, n, shift, blk0, cnt);
  for (int dg = threadIdx.x; dg < kRadix; dg += kThreads) {
    int64_t s = offs[(int64_t)dg * nblocks + blockIdx.x];
    for (int w = 0; w < kWarps; ++w) {
      base[w][dg] = s;
      s += cnt[w][dg];
    }
  }
  __syncthreads();
  const int64_t w0 = blk0 + (int64_t)warp * kPerWarp;
  for (int b = 0; b < kPerWarp; b += 32) {
    const int64_t i = w0 + b + lane;
    const bool valid = i < n;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    if (!act) break;
    if (valid) {
      const int32_t k = key[i];
      const int dg = (k >> shift) & (kRadix - 1);
      const unsigned peers = __match_any_sync(act, dg);
      const unsigned below = peers & lanemask_lt();
      const int64_t dest = base[warp][dg] + __popc(below);
      __syncwarp(act);
      if (below == 0) base[warp][dg] += __popc(peers);
      for (int a = 0; a < 3; ++a) {
        dst.x[a * cap + dest] = src.x[a * cap + i];
        dst.u[a * cap + dest] = src.u[a * cap + i];
      }
      dst.d[dest] = src.d[i];
      dst.w[dest] = src.w[i];
      dst.id[dest] = src.id[i];
      key_dst[dest] = k;
    }
    __syncwarp();
  }
}

// ---- exclusive scan of uint32 -> int64 (three phases) ----
constexpr int kScanItems = 4096;

__global__ void __launch_bounds__(256) k_scan_partial(const uint32_t* __restrict__ in, int64_t m,
                                                      int64_t* __restrict__ partial) {
  __shared__ int64_t red[256];
  const int64_t b0 = (int64_t)blockIdx.x * kScanItems;
  int64_t s = 0;
  for (int j = threadIdx.x; j < kScanItems; j += 256) {
    const int64_t i = b0 + j;
    if (i < m) s += in[i];
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// Single block: exclusive scan of the partials in place (sequential chunks of 1024).
__global__ void __launch_bounds__(1024) k_scan_partials(int64_t* __restrict__ partial, int64_t np,
                                                        int64_t* __restrict__ total_out) {
  __shared__ int64_t sh[1024];
  __shared__ int64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < np; c0 += 1024) {
    const int64_t i = c0 + threadIdx.x;
    const int64_t v = i < np ? partial[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int64_t t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < np) partial[i] = carry + sh[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

__global__ void __launch_bounds__(256) k_scan_final(const uint32_t* __restrict__ in, int64_t m,
                                                    const int64_t* __restrict__ partial, int64_t* __restrict__ out) {
  // each thread scans 16 consecutive items, then a block scan of thread sums
  __shared__ int64_t sh[256];
  const int64_t b0 = (int64_t)blockIdx.x * kScanItems + (int64_t)threadIdx.x * 16;
  uint32_t v[16];
  int64_t s = 0;
  for (int j = 0; j < 16; ++j) {
    const int64_t i = b0 + j;
    v[j] = i < m ? in[i] : 0u;
    s += v[j];
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 256; o <<= 1) {
    const int64_t t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
    __syncthreads();
    sh[threadIdx.x] += t;
    __syncthreads();
  }
  int64_t run = partial[blockIdx.x] + sh[threadIdx.x] - s;
  for (int j = 0; j < 16; ++j) {
    const int64_t i = b0 + j;
    if (i < m) out[i] = run;
    run += v[j];
  }
}

__global__ void k_chunk_offsets(const int32_t* __restrict__ key, int64_t n, int32_t key_lo, int32_t nkeys,
                                int64_t* __restrict__ off) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > nkeys) return;
  const int32_t target = key_lo + k;
  int64_t lo = 0, hi = n;   // first index with key >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (key[mid] < target) lo = mid + 1;
    else hi = mid;
  }
  off[k] = lo;
}

}  // namespace

int launch_exclusive_scan_u32(const uint32_t* in, int64_t m, int64_t* out, int64_t* partial, cudaStream_t s) {
  const int64_t nb = (m + kScanItems - 1) / kScanItems;
  k_scan_partial<<<(unsigned)nb, 256, 0, s>>>(in, m, partial);
  k_scan_partials<<<1, 1024, 0, s>>>(partial, nb, out + m);
  k_scan_final<<<(unsigned)nb, 256, 0, s>>>(in, m, partial, out);
  return 3;
}

int launch_stable_sort(Store a, Store b, int64_t cap, int64_t n, int32_t* key_a, int32_t* key_b, int key_bits,
                       SortScratch& sc, int* result_in_b, cudaStream_t s) {
  *result_in_b = 0;
  if (n <= 1) return 0;
  const int64_t nblocks = (n + kItems - 1) / kItems;
  if (nblocks > sc.max_blocks) return -1;
  int launches = 0;
  Store src = a, dst = b;
  int32_t* ksrc = key_a;
  int32_t* kdst = key_b;
  const int passes = key_bits <= 0 ? 1 : (key_bits + 7) / 8;
  for (int p = 0; p < passes; ++p) {
    const int shift = 8 * p;
    k_sort_count<<<(unsigned)nblocks, kThreads, 0, s>>>(ksrc, n, shift, nblocks, sc.hist);
    launches += 1 + launch_exclusive_scan_u32(sc.hist, (int64_t)kRadix * nblocks, sc.offs, sc.partial, s);
    k_sort_scatter<<<(unsigned)nblocks, kThreads, 0, s>>>(src, dst, cap, ksrc, kdst, n, shift, nblocks, sc.offs);
    ++launches;
    Store t = src; src = dst; dst = t;
    int32_t* kt = ksrc; ksrc = kdst; kdst = kt;
    *result_in_b ^= 1;
  }
  return launches;
}

int launch_chunk_offsets(const int32_t* key_sorted, int64_t n, int32_t key_lo, int32_t nkeys, int64_t* offsets,
                         cudaStream_t s) {
  const int total = nkeys + 1;
  k_chunk_offsets<<<(total + 255) / 256, 256, 0, s>>>(key_sorted, n, key_lo, nkeys, offsets);
  return 1;
}

}  // namespace st
