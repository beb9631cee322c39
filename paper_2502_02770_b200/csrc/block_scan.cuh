// Block- and warp-group-wide primitives (scan, reductions, radix select)
// shared by the selection and pruning kernels.  A Group is a run of whole
// warps synchronised by a named barrier, so several independent selections
// can proceed inside one CTA (e.g. the G query heads of a KV head).
#pragma once
#include "common.cuh"

namespace tw {

struct Group {
  int bar;       // named barrier id; 0 = __syncthreads (whole block)
  int nthreads;  // threads in the group (multiple of 32)
  int tid;       // thread index inside the group
  __device__ __forceinline__ void sync() const {
    if (bar == 0) __syncthreads();
    else named_bar_sync(bar, nthreads);
  }
  __device__ __forceinline__ int warp() const { return tid >> 5; }
  __device__ __forceinline__ int nwarps() const { return nthreads >> 5; }
};

__device__ __forceinline__ Group whole_block() { return Group{0, (int)blockDim.x, (int)threadIdx.x}; }

// Inclusive scan of one u32 per thread; `tmp` needs nwarps words.
__device__ __forceinline__ uint32_t group_incl_scan(const Group& g, uint32_t v, uint32_t* tmp, uint32_t& total) {
  const int lane = g.tid & 31, wid = g.warp(), nw = g.nwarps();
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  g.sync();
  uint32_t pre = 0, tot = 0;
  for (int i = 0; i < nw; ++i) {
    const uint32_t s = tmp[i];
    pre += i < wid ? s : 0u;
    tot += s;
  }
  g.sync();
  total = tot;
  return x + pre;
}

__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, uint32_t* tmp, uint32_t& total) {
  return group_incl_scan(whole_block(), v, tmp, total);
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

__device__ __forceinline__ void group_minmax_u32(const Group& g, uint32_t& mn, uint32_t& mx, uint32_t* tmp) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((g.tid & 31) == 0) {
    tmp[2 * g.warp()] = mn;
    tmp[2 * g.warp() + 1] = mx;
  }
  g.sync();
  for (int i = 0; i < g.nwarps(); ++i) {
    mn = min(mn, tmp[2 * i]);
    mx = max(mx, tmp[2 * i + 1]);
  }
  g.sync();
}

// Given per-bin counts hist[0..nbins) (nbins a multiple of the group size),
// find bin d* scanning from the TOP bin down with
//   above = sum_{d > d*} hist[d] < need <= above + hist[d*].
// `res` (2 words of shared memory per group) receives {d*, above}.
__device__ __forceinline__ int group_find_from_top(const Group& g, const uint32_t* hist, int nbins, uint32_t need,
                                                   uint32_t* tmp, int* res, uint32_t& above_out) {
  const int per = nbins / g.nthreads;
  const int hi_bin = nbins - g.tid * per - 1;
  uint32_t local = 0;
  for (int i = 0; i < per; ++i) local += hist[hi_bin - i];
  uint32_t total;
  const uint32_t incl = group_incl_scan(g, local, tmp, total);
  const uint32_t excl = incl - local;
  if (g.tid == 0) { res[0] = -1; res[1] = 0; }
  g.sync();
  if (excl < need && need <= incl) {
    uint32_t run = excl;
    for (int i = 0; i < per; ++i) {
      const uint32_t c = hist[hi_bin - i];
      if (run + c >= need) { res[0] = hi_bin - i; res[1] = (int)run; break; }
      run += c;
    }
  }
  g.sync();
  const int b = res[0];
  above_out = (uint32_t)res[1];
  g.sync();
  return b;
}

// k-th largest (1-based) of n u32 keys in shared memory.  Only the bits below
// the highest bit where the keys differ are radix-scanned (11 bits a pass), so
// clustered keys (e.g. fp32 scores of similar magnitude) need two passes.
// `hist` needs 2048 words, `tmp` 2*nwarps words, `res` 2 words.
__device__ __forceinline__ uint32_t group_kth_largest(const Group& g, const uint32_t* keys, int n, uint32_t k,
                                                      uint32_t* hist, uint32_t* tmp, int* res) {
  uint32_t mn = 0xFFFFFFFFu, mx = 0;
  for (int i = g.tid; i < n; i += g.nthreads) {
    mn = min(mn, keys[i]);
    mx = max(mx, keys[i]);
  }
  group_minmax_u32(g, mn, mx, tmp);
  if (mn == mx) return mn;
  int hi = 31 - __clz(mn ^ mx);
  uint32_t mask = hi == 31 ? 0u : ~((2u << hi) - 1u);
  uint32_t prefix = mn & mask;
  uint32_t need = k;
  while (hi >= 0) {
    const int width = hi + 1 < 11 ? hi + 1 : 11;
    const int sh = hi + 1 - width;
    const uint32_t dm = (1u << width) - 1u;
    for (int i = g.tid; i < 2048; i += g.nthreads) hist[i] = 0;
    g.sync();
    for (int i = g.tid; i < n; i += g.nthreads) {
      const uint32_t kk = keys[i];
      if ((kk & mask) == prefix) atomicAdd(&hist[(kk >> sh) & dm], 1u);
    }
    g.sync();
    uint32_t above;
    const int d = group_find_from_top(g, hist, 2048, need, tmp, res, above);
    need -= above;
    prefix |= (uint32_t)d << sh;
    mask |= dm << sh;
    hi = sh - 1;
  }
  return prefix;
}

// Same result as group_kth_largest, by a bitwise search over the informative
// bits: for each bit, one counting pass over the keys (shared memory) and one
// group reduction.  Cheaper than histogram passes when keys cluster.
// `tmp` needs nwarps words.
__device__ __forceinline__ uint32_t group_kth_largest_bs(const Group& g, const uint32_t* keys, int n, uint32_t k,
                                                         uint32_t* tmp) {
  uint32_t mn = 0xFFFFFFFFu, mx = 0;
  for (int i = g.tid; i < n; i += g.nthreads) {
    mn = min(mn, keys[i]);
    mx = max(mx, keys[i]);
  }
  group_minmax_u32(g, mn, mx, tmp);
  if (mn == mx) return mn;
  const int hi = 31 - __clz(mn ^ mx);
  uint32_t res = hi == 31 ? 0u : (mn & ~((2u << hi) - 1u));
  for (int bit = hi; bit >= 0; --bit) {
    const uint32_t cand = res | (1u << bit);
    uint32_t c = 0;
#pragma unroll 8
    for (int i = g.tid; i < n; i += g.nthreads) c += keys[i] >= cand ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((g.tid & 31) == 0) tmp[g.warp()] = c;
    g.sync();
    uint32_t tot = 0;
    for (int w = 0; w < g.nwarps(); ++w) tot += tmp[w];
    g.sync();
    if (tot >= k) res = cand;
  }
  return res;
}

// k-th largest of n ordered float keys (f2key) in shared memory with ONE
// histogram pass: 1024 bins linearly spaced between the min and max value
// (monotone in the value), then the few members of the crossing bin are
// ranked directly.  Falls back to the bitwise search when that bin is crowded
// (ties / clustered values).  `hist` needs 1024 words, `mem` 64 words,
// `tmp` 2*nwarps words, `res` 4 words.
__device__ __forceinline__ uint32_t group_kth_largest_lin(const Group& g, const uint32_t* keys, int n, uint32_t k,
                                                          uint32_t* hist, uint32_t* mem, uint32_t* tmp, int* res) {
  constexpr int kNb = 1024, kMem = 64;
  uint32_t mn = 0xFFFFFFFFu, mx = 0;
  for (int i = g.tid; i < n; i += g.nthreads) {
    mn = min(mn, keys[i]);
    mx = max(mx, keys[i]);
  }
  for (int i = g.tid; i < kNb; i += g.nthreads) hist[i] = 0;
  group_minmax_u32(g, mn, mx, tmp);
  if (mn == mx) return mn;
  const float vmin = key2f(mn), vmax = key2f(mx);
  const float scale = (float)kNb / (vmax - vmin);
  if (!(scale > 0.f) || isinf(scale)) return group_kth_largest_bs(g, keys, n, k, tmp);
  auto bin = [&](uint32_t kk) {
    const float x = (key2f(kk) - vmin) * scale;
    return x >= (float)(kNb - 1) ? kNb - 1 : (int)x;
  };
  for (int i = g.tid; i < n; i += g.nthreads) atomicAdd(&hist[bin(keys[i])], 1u);
  g.sync();
  uint32_t above;
  const int b = group_find_from_top(g, hist, kNb, k, tmp, res, above);
  const int members = (int)hist[b];
  if (members > kMem) return group_kth_largest_bs(g, keys, n, k, tmp);
  if (g.tid == 0) res[2] = 0;
  g.sync();
  for (int i = g.tid; i < n; i += g.nthreads)
    if (bin(keys[i]) == b) mem[atomicAdd(&res[2], 1)] = keys[i];
  g.sync();
  const uint32_t need = k - above;  // 1-based rank inside the bin
  if (g.tid < members) {
    const uint32_t x = mem[g.tid];
    uint32_t gt = 0, ge = 0;
    for (int j = 0; j < members; ++j) {
      gt += mem[j] > x;
      ge += mem[j] >= x;
    }
    if (gt < need && need <= ge) res[3] = (int)x;  // all writers agree
  }
  g.sync();
  const uint32_t r = (uint32_t)res[3];
  g.sync();
  return r;
}

}  // namespace tw
