// device.cuh — warp/block primitives shared by the kernels.
#pragma once
#include "internal.h"

namespace remat {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ u64 shfl_xor_u64(u64 v, int m) {
  return __shfl_xor_sync(kFull, v, m);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(kFull, v, m);
  return v;
}

__device__ __forceinline__ u64 warp_or(u64 v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v |= __shfl_xor_sync(kFull, v, m);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

__device__ __forceinline__ u64 warp_inclusive_min(u64 v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    u64 o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v = o < v ? o : v;
  }
  return v;
}

// Block-wide exclusive sum over blockDim.x threads (a multiple of 32, <= 1024).
// `scratch` holds >= 33 elements.  Returns the exclusive prefix; *total gets the
// block total.  Ends with the scratch free for reuse after a __syncthreads.
template <typename T>
__device__ T block_exclusive_sum(T v, T* scratch, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  T inc = warp_inclusive_sum(v);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T s = lane < nw ? scratch[lane] : T(0);
    T si = warp_inclusive_sum(s);
    if (lane < nw) scratch[lane] = si - s;
    if (lane == nw - 1) scratch[32] = si;
  }
  __syncthreads();
  T out = scratch[warp] + inc - v;
  *total = scratch[32];
  __syncthreads();
  return out;
}

// Block-wide exclusive min (identity ~0ull).
__device__ __forceinline__ u64 block_exclusive_min(u64 v, u64* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  u64 inc = warp_inclusive_min(v);
  u64 exc = __shfl_up_sync(kFull, inc, 1);
  if (lane == 0) exc = ~0ull;
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    u64 s = lane < nw ? scratch[lane] : ~0ull;
    u64 si = warp_inclusive_min(s);
    u64 se = __shfl_up_sync(kFull, si, 1);
    if (lane == 0) se = ~0ull;
    if (lane < nw) scratch[lane] = se;
  }
  __syncthreads();
  u64 w = scratch[warp];
  __syncthreads();
  return w < exc ? w : exc;
}

// Weighted popcount Σ_{v ∈ x} cost[v] over one 64-bit word (word index q).
__device__ __forceinline__ long long word_weight(u64 x, int q, const long long* __restrict__ cost) {
  long long s = 0;
  while (x) {
    int b = __ffsll((long long)x) - 1;
    x &= x - 1;
    s += __ldg(cost + q * 64 + b);
  }
  return s;
}

}  // namespace remat
