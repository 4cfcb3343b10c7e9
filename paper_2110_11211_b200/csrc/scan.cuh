// Deterministic device-wide exclusive scan (three phases: tile sums, scan of
// tile sums, tile scans).  Used by the SFC rank computation and the radix
// sort; hand-written, no CUB.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace sfcdd {

constexpr int SCAN_THREADS = 512;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// Functor-based input so callers can scan derived quantities (e.g. popcounts)
template <typename T, typename F>
__global__ void scan_tile_sums(F in, int64_t n, T* tile_sums) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  T s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + (int64_t)k * SCAN_THREADS + threadIdx.x;
    if (i < n) s += in(i);
  }
  __shared__ T red[SCAN_THREADS / 32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    T t = threadIdx.x < SCAN_THREADS / 32 ? red[threadIdx.x] : T(0);
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = t;
  }
}

// single block: exclusive scan of m tile sums in place; grand total to *total
template <typename T>
__global__ void scan_tile_offsets(T* sums, int64_t m, T* total) {
  __shared__ T carry;
  __shared__ T wsum[SCAN_THREADS / 32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t b = 0; b < m; b += SCAN_THREADS) {
    int64_t i = b + threadIdx.x;
    T v = i < m ? sums[i] : T(0);
    T inc = warp_inclusive_scan(v);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      T w = lane < SCAN_THREADS / 32 ? wsum[lane] : T(0);
      T wi = warp_inclusive_scan(w);
      if (lane < SCAN_THREADS / 32) wsum[lane] = wi - w;
    }
    __syncthreads();
    T ex = inc - v + wsum[warp] + carry;
    if (i < m) sums[i] = ex;
    __syncthreads();
    if (threadIdx.x == SCAN_THREADS - 1) carry = ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

// per tile: exclusive scan of in(i) plus the tile offset; out(i, value)
template <typename T, typename F, typename G>
__global__ void scan_tiles(F in, G out, int64_t n, const T* tile_offsets) {
  __shared__ T wsum[SCAN_THREADS / 32];
  __shared__ T carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  if (threadIdx.x == 0) carry = tile_offsets[blockIdx.x];
  __syncthreads();
  // thread-contiguous items for coalescing-friendly access per round
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + (int64_t)k * SCAN_THREADS + threadIdx.x;
    T v = i < n ? in(i) : T(0);
    T inc = warp_inclusive_scan(v);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      T w = lane < SCAN_THREADS / 32 ? wsum[lane] : T(0);
      T wi = warp_inclusive_scan(w);
      if (lane < SCAN_THREADS / 32) wsum[lane] = wi - w;
    }
    __syncthreads();
    T ex = inc - v + wsum[warp] + carry;
    if (i < n) out(i, ex);
    __syncthreads();
    if (threadIdx.x == SCAN_THREADS - 1) carry = ex + v;
    __syncthreads();
  }
}

}  // namespace sfcdd
