// stats.cuh -- per-iteration population statistics on the device
// (the reference computes them on the host,
// stats.py:21-100).
//
//   * frozen-range PMF histogram, binned exactly as numpy does
//     (stats.py:45-47): idx = clip(int64((f64(x) - lo) / width), 0, bins-1)
//     with IEEE double subtract / divide and truncation;
//   * the minimum;
//   * nearest-rank percentiles (stats.py:21-29): the k-th smallest cost for up
//     to four ranks at once, by an MSB radix select over the order-preserving
//     64-bit keys (8 passes of 8-bit digits; the last block of each pass turns
//     the digit histograms into the next prefix).
#pragma once
#include <type_traits>
#include "common.cuh"

namespace qsb {

constexpr int STATS_RANKS = 4;

struct StatsWork {
  // per pass, per rank: 256-bin digit histogram
  unsigned int hist[STATS_RANKS][256];
  unsigned long long prefix[STATS_RANKS];   // key bits fixed so far
  unsigned long long kth[STATS_RANKS];      // remaining rank (0-based) inside the prefix
  unsigned int done;
  unsigned int pad;
  unsigned long long min_key;
};

template <typename CT>
__device__ __forceinline__ unsigned long long cost_key(CT c) {
  if constexpr (std::is_floating_point<CT>::value) {
    // canonicalise -0.0 (costs are sums of non-negative products)
    return okey(c == 0.0 ? 0.0 : (double)c);
  } else {
    return (unsigned long long)c ^ 0x8000000000000000ULL;
  }
}

// PMF histogram + minimum key.
template <typename CT>
__global__ void stats_hist_kernel(const CT* cost, int64_t P, double lo, double width, int bins,
                                  unsigned int* hist, StatsWork* w) {
  extern __shared__ unsigned int sh[];
  for (int b = threadIdx.x; b < bins; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  unsigned long long mn = ~0ULL;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    const CT c = cost[i];
    const double a = (double)c;
    long long idx = (long long)__ddiv_rn(__dsub_rn(a, lo), width);   // astype(int64): truncation
    idx = idx < 0 ? 0 : (idx > bins - 1 ? bins - 1 : idx);
    atomicAdd(&sh[idx], 1u);
    const unsigned long long k = cost_key(c);
    mn = k < mn ? k : mn;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(FULL, mn, o);
    mn = t < mn ? t : mn;
  }
  if ((threadIdx.x & 31) == 0) atomicMin(&w->min_key, mn);
  __syncthreads();
  for (int b = threadIdx.x; b < bins; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

// One radix-select pass (digit = bits [shift, shift+8) of the key) for all
// ranks; the last block folds the histograms into prefix / kth.
template <typename CT>
__global__ void stats_select_kernel(const CT* cost, int64_t P, int shift, int nranks, StatsWork* w) {
  __shared__ unsigned int sh[STATS_RANKS][256];
  __shared__ bool last;
  for (int i = threadIdx.x; i < STATS_RANKS * 256; i += blockDim.x) sh[i / 256][i % 256] = 0;
  __syncthreads();
  const unsigned long long hmask = shift >= 56 ? 0ULL : (~0ULL << (shift + 8));
  unsigned long long pre[STATS_RANKS];
  for (int r = 0; r < nranks; ++r) pre[r] = w->prefix[r];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = cost_key(cost[i]);
    const unsigned d = (unsigned)((k >> shift) & 0xffULL);
    for (int r = 0; r < nranks; ++r)
      if ((k & hmask) == pre[r]) atomicAdd(&sh[r][d], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nranks * 256; i += blockDim.x)
    if (sh[i / 256][i % 256]) atomicAdd(&w->hist[i / 256][i % 256], sh[i / 256][i % 256]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&w->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < nranks) {
    const int r = threadIdx.x;
    unsigned long long kk = w->kth[r];
    volatile unsigned int* h = w->hist[r];
    int d = 0;
    for (; d < 256; ++d) {
      const unsigned long long c = h[d];
      if (kk < c) break;
      kk -= c;
    }
    w->prefix[r] |= (unsigned long long)d << shift;
    w->kth[r] = kk;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < STATS_RANKS * 256; i += blockDim.x) w->hist[i / 256][i % 256] = 0;
  if (threadIdx.x == 0) w->done = 0;
}

}  // namespace qsb

namespace qsb {

__global__ void stats_init_kernel(StatsWork* w, unsigned long long k0, unsigned long long k1,
                                  unsigned long long k2, unsigned long long k3) {
  w->prefix[0] = w->prefix[1] = w->prefix[2] = w->prefix[3] = 0;
  w->kth[0] = k0; w->kth[1] = k1; w->kth[2] = k2; w->kth[3] = k3;
  w->done = 0;
  w->min_key = ~0ULL;
}

// out[0] = minimum, out[1 + r] = k_r-th smallest, as the cost's raw bits.
template <typename CT>
__global__ void stats_finish_kernel(const StatsWork* w, int nranks, long long* out) {
  auto val = [](unsigned long long k) -> long long {
    if constexpr (std::is_floating_point<CT>::value) return __double_as_longlong(from_okey(k));
    else return (long long)(k ^ 0x8000000000000000ULL);
  };
  out[0] = val(w->min_key);
  for (int r = 0; r < nranks; ++r) out[1 + r] = val(w->prefix[r]);
}

}  // namespace qsb
