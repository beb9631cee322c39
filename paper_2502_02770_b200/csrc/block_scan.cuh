// Small block-wide primitives (scan, reductions, radix select) shared by the
// selection and pruning kernels.
#pragma once
#include "common.cuh"

namespace tw {

// Inclusive block scan of one u32 per thread; returns the inclusive prefix and
// writes the block total.  `tmp` must hold blockDim/32 + 1 words.
__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, uint32_t* tmp, uint32_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < nw ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) tmp[lane] = s;
  }
  __syncthreads();
  if (wid > 0) x += tmp[wid - 1];
  total = tmp[nw - 1];
  __syncthreads();
  return x;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* tmp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) tmp[wid] = v;
  __syncthreads();
  T r = 0;
  for (int i = 0; i < nw; ++i) r += tmp[i];
  __syncthreads();
  return r;
}

__device__ __forceinline__ uint32_t block_max_u32(uint32_t v, uint32_t* tmp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max_u32(v);
  if (lane == 0) tmp[wid] = v;
  __syncthreads();
  uint32_t r = 0;
  for (int i = 0; i < nw; ++i) r = max(r, tmp[i]);
  __syncthreads();
  return r;
}

// Given per-bin counts hist[0..nbins) (nbins a multiple of blockDim.x),
// find the bin d* scanning from the TOP bin down such that
//   above = sum_{d > d*} hist[d] < need <= above + hist[d*].
// Returns d* and writes `above` (uniform across the block).
__device__ __forceinline__ int block_find_from_top(const uint32_t* hist, int nbins, uint32_t need, uint32_t* tmp,
                                                   uint32_t& above_out) {
  const int per = nbins / blockDim.x;
  // thread t owns bins in descending order: [nbins - (t+1)*per, nbins - t*per)
  const int hi_bin = nbins - threadIdx.x * per - 1;
  uint32_t local = 0;
  for (int i = 0; i < per; ++i) local += hist[hi_bin - i];
  uint32_t total;
  uint32_t incl = block_incl_scan(local, tmp, total);
  uint32_t excl = incl - local;
  __shared__ int s_bin;
  __shared__ uint32_t s_above;
  if (threadIdx.x == 0) { s_bin = -1; s_above = 0; }
  __syncthreads();
  if (excl < need && need <= incl) {
    uint32_t run = excl;
    for (int i = 0; i < per; ++i) {
      uint32_t c = hist[hi_bin - i];
      if (run + c >= need) { s_bin = hi_bin - i; s_above = run; break; }
      run += c;
    }
  }
  __syncthreads();
  int b = s_bin;
  above_out = s_above;
  __syncthreads();
  return b;
}

// K-th largest (1-based k) of n u32 keys held in shared memory.
// Three radix passes (11, 11, 10 bits); `hist` needs 2048 words.
__device__ __forceinline__ uint32_t block_kth_largest(const uint32_t* keys, int n, uint32_t k, uint32_t* hist,
                                                      uint32_t* tmp) {
  uint32_t prefix = 0, mask = 0, need = k;
  const int shifts[3] = {21, 10, 0};
  const int widths[3] = {11, 11, 10};
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    const int sh = shifts[pass], nb = 1 << widths[pass];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      uint32_t kk = keys[i];
      if ((kk & mask) == prefix) atomicAdd(&hist[(kk >> sh) & (nb - 1)], 1u);
    }
    __syncthreads();
    uint32_t above;
    int d = block_find_from_top(hist, 2048, need, tmp, above);  // bins >= nb are zero
    need -= above;
    prefix |= (uint32_t)d << sh;
    mask |= (uint32_t)(nb - 1) << sh;
  }
  return prefix;
}

}  // namespace tw
