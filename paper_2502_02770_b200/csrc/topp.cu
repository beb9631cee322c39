// K3b/K3c: per-head softmax over the candidates, top-p threshold, group union.
//
// Reference: stable_softmax (attention.py:79-86) in fp64 over the candidate
// logits (pipeline.py:344), binary_search_top_p (pruner.py:57-114): the
// returned set is {w >= l}, and with the default epsilon/max_iters the search
// runs until that set is the MINIMAL TIE-CLOSED top set whose mass reaches
// p_eff = min(p, sum w) - 1e-9 (break rules :99-104).  We compute that set
// directly instead of bisecting (~50 passes): a mass-weighted radix select.
//
//   pass 1   e_i = exp(z_i - max) (SFU exp2, ~1e-6 relative), quantised to
//            u64 fixed point (exact, order-independent sums => deterministic);
//            histogram of (count, mass) over 4096 bins of (max - z) ; the
//            crossing bin is the first (highest-z) bin where the running mass
//            reaches p_eff * Z.
//   pass 2+  the crossing bin's members are compacted to shared memory and
//            ranked exactly by their fp32 logit key (ties = equal logits =
//            equal weights); bins too full to rank are split again by key.
// The selected set is {z >= z_thr}: the same tie-closed set the reference
// returns, up to weights within ~1e-7 relative of the threshold.
//
// K3c: the group's final set is the union over its G heads (pipeline.py:347);
// it is compacted in ascending token order and cut into attention work items.
#include "block_scan.cuh"
#ifdef TW_TOPP_TRACE
#include <cstdio>
#endif

namespace tw {

#ifdef TW_TOPP_TRACE
__device__ unsigned long long g_trace[512 * 8];
__device__ int g_trace_phase[512];
#define TRACE(tag)                                                                                  \
  do {                                                                                              \
    if (threadIdx.x == 0 && blockIdx.x < 512) {                                                     \
      unsigned long long now;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));                                      \
      int ph = g_trace_phase[blockIdx.x]++;                                                         \
      if (ph < 8) g_trace[blockIdx.x * 8 + ph] = now;                                               \
    }                                                                                               \
  } while (0)
#else
#define TRACE(tag) do {} while (0)
#endif

constexpr int kTopThreads = 512;
constexpr int kBins = 4096;
constexpr int kRankCap = 512;          // members ranked O(k^2) in shared memory
constexpr float kBinPerLogit = 120.0f; // bins cover (max - z) in [0, 34.1)

__device__ __forceinline__ void atomic_add_u64_split(uint32_t* lo, uint32_t* hi, uint64_t v) {
  const uint32_t vlo = (uint32_t)v, vhi = (uint32_t)(v >> 32);
  const uint32_t old = atomicAdd(lo, vlo);
  const uint32_t carry = (uint32_t)(old + vlo < old);
  if (vhi + carry) atomicAdd(hi, vhi + carry);
}

// Fixed-point softmax mass of logit z under max m: round(e * 2^sh) with
// e = 2^((z - m) log2 e) on the SFU (rel. error ~1e-6 for z - m >= -40; the
// scale is a power of two so the float->u64 conversion adds no error).
__device__ __forceinline__ uint64_t mass_fx(float z, float m, float fscale) {
  const float e = exp2f((z - m) * 1.4426950408889634f);
  return __float2ull_rn(e * fscale);
}

__device__ __forceinline__ int dbin(float z, float m) {
  const float d = (m - z) * kBinPerLogit;
  return d >= (float)(kBins - 1) ? kBins - 1 : (int)d;
}

// u64 inclusive block scan (one value per thread)
__device__ __forceinline__ uint64_t block_incl_scan_u64(uint64_t v, uint64_t* tmp, uint64_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t s = lane < nw ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
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

struct TopSmem {
  uint32_t cnt[kBins];
  uint32_t mlo[kBins];
  uint32_t mhi[kBins];
  uint32_t mkey[kRankCap];
  uint64_t mmass[kRankCap];
  uint64_t scan_tmp[32];
  uint32_t tmp32[40];
  int nmem;
  uint32_t kmin, kmax;
  int bin;
  uint64_t above_mass;
  uint32_t above_cnt;
  uint32_t thr;
  uint32_t sel_cnt;
  uint64_t sel_mass;
};

// Find the first bin in `order` (ascending index = descending logit when
// `descending_index` is false) whose running mass reaches target.
__device__ __forceinline__ void find_crossing(TopSmem& S, double target, uint64_t base_mass, bool top_is_high) {
  const int per = kBins / kTopThreads;
  // thread t owns `per` consecutive bins in priority order
  uint64_t local = 0;
  uint32_t lcnt = 0;
  for (int i = 0; i < per; ++i) {
    const int rank = threadIdx.x * per + i;
    const int bb = top_is_high ? (kBins - 1 - rank) : rank;
    local += ((uint64_t)S.mhi[bb] << 32) | S.mlo[bb];
    lcnt += S.cnt[bb];
  }
  uint64_t total;
  const uint64_t incl = block_incl_scan_u64(local, S.scan_tmp, total);
  uint32_t ctot;
  const uint32_t cincl = block_incl_scan(lcnt, S.tmp32, ctot);
  const uint64_t excl = incl - local;
  const uint32_t cexcl = cincl - lcnt;
  if (threadIdx.x == 0) S.bin = -1;
  __syncthreads();
  if ((double)(base_mass + excl) < target && target <= (double)(base_mass + incl)) {
    uint64_t run = excl;
    uint32_t crun = cexcl;
    for (int i = 0; i < per; ++i) {
      const int rank = threadIdx.x * per + i;
      const int bb = top_is_high ? (kBins - 1 - rank) : rank;
      const uint64_t m = ((uint64_t)S.mhi[bb] << 32) | S.mlo[bb];
      if ((double)(base_mass + run + m) >= target) {
        S.bin = bb;
        S.above_mass = base_mass + run;
        S.above_cnt = crun;
        break;
      }
      run += m;
      crun += S.cnt[bb];
    }
  }
  __syncthreads();
}

// Vectorised walk over a head's logits: 4 x float4 in flight per thread.
template <typename F>
__device__ __forceinline__ void for_each_logit(const float* __restrict__ z, int npos, F&& f) {
  const float4* z4 = reinterpret_cast<const float4*>(z);
  const int n4 = npos >> 2;
  for (int base = threadIdx.x; base < n4; base += blockDim.x * 4) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = base + u * blockDim.x;
      v[u] = i < n4 ? __ldcg(z4 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = base + u * blockDim.x;
      if (i < n4) {
        f(4 * i, v[u].x);
        f(4 * i + 1, v[u].y);
        f(4 * i + 2, v[u].z);
        f(4 * i + 3, v[u].w);
      }
    }
  }
}

// One CTA per query head; the last head of a unit to finish also forms the
// group's final set (K3c) and reserves its attention work items.
__global__ void __launch_bounds__(kTopThreads) topp_head_kernel(tw_paged_kv kv, tw_decode_params prm,
                                                                tw_decode_buffers buf) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TopSmem& S = *reinterpret_cast<TopSmem*>(smem_raw);
  __shared__ int s_last;
  __shared__ uint32_t s_selc;
  __shared__ unsigned long long s_selm;
  const int qh = blockIdx.x;
  const int G = kv.group_size;
  const int unit = qh / G;
  const int npos = buf.cand_count[unit] * kPage;
  const size_t T = (size_t)kv.max_pages * kPage;
  const float* z = buf.logits + (size_t)qh * T;
  const float M = key2f(buf.head_max[qh]);
  const double p_eff = fmin(prm.p, 1.0) - 1e-9;
  float* stats = buf.head_stats + (size_t)qh * 4;
  uint32_t thr = 0xFFFFFFFFu;  // selects nothing
  uint32_t b0 = 0;
  uint64_t Z = 0;
  float fscale = 1.f;
  uint32_t sel_cnt = 0;        // |{z >= thr}|   (counted from the histograms, no extra pass)
  uint64_t sel_mass = 0;       // its fixed-point mass
  const bool empty = p_eff <= 0.0 || npos == 0 || !(M > -INFINITY);
  TRACE("start");
  if (!empty) {
    // fixed-point scale: sums of up to npos terms stay below 2^63
    const int lg = 32 - __clz(npos);
    fscale = ldexpf(1.f, 62 - lg);
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) { S.cnt[i] = 0; S.mlo[i] = 0; S.mhi[i] = 0; }
    __syncthreads();
    uint64_t zt = 0;
    uint32_t nvalid = 0;
    for_each_logit(z, npos, [&](int, float zi) {
      if (zi == -INFINITY) return;
      ++nvalid;
      const uint64_t mf = mass_fx(zi, M, fscale);
      const int bb = dbin(zi, M);
      atomicAdd(&S.cnt[bb], 1u);
      if (mf) atomic_add_u64_split(&S.mlo[bb], &S.mhi[bb], mf);
      zt += mf;
    });
    TRACE("pass1");
    block_incl_scan_u64(zt, S.scan_tmp, Z);
    block_incl_scan(nvalid, S.tmp32, b0);
    const double target = p_eff * (double)Z;

    // level 0: bins of (max - z), highest logit first (= ascending bin index)
    find_crossing(S, target, 0, false);
    TRACE("crossing");
    int bin = S.bin;
    uint64_t above_mass = S.above_mass;
    uint32_t above_cnt = S.above_cnt;
    uint32_t klo = 0, khi = 0xFFFFFFFFu;
    bool resolved = false;
    if (bin < 0) {  // rounding: the whole set is needed
      thr = 0;
      sel_cnt = b0;
      sel_mass = Z;
      resolved = true;
    }
    int members = resolved ? 0 : (int)S.cnt[bin];
    uint64_t range_mass = resolved ? 0 : (((uint64_t)S.mhi[bin] << 32) | S.mlo[bin]);
    while (!resolved) {
      __syncthreads();
      if (members <= kRankCap) {
        // compact the members, then rank them exactly
        if (threadIdx.x == 0) { S.nmem = 0; s_selc = 0; s_selm = 0; }
        __syncthreads();
        for_each_logit(z, npos, [&](int, float zi) {
          if (zi == -INFINITY || dbin(zi, M) != bin) return;
          const uint32_t k = f2key(zi);
          if (k < klo || k > khi) return;
          const int slot = atomicAdd(&S.nmem, 1);
          if (slot < kRankCap) {
            S.mkey[slot] = k;
            S.mmass[slot] = mass_fx(zi, M, fscale);
          }
        });
        __syncthreads();
        TRACE("members");
        const int nm = min(S.nmem, kRankCap);
        if (threadIdx.x == 0) S.thr = klo;  // fallback (rounding): keep the whole range
        __syncthreads();
        for (int a = threadIdx.x; a < nm; a += blockDim.x) {
          const uint32_t ka = S.mkey[a];
          uint64_t above = 0, eq = 0;
          for (int j = 0; j < nm; ++j) {
            const uint32_t kj = S.mkey[j];
            const uint64_t mj = S.mmass[j];
            above += kj > ka ? mj : 0;
            eq += kj == ka ? mj : 0;
          }
          if ((double)(above_mass + above) < target && target <= (double)(above_mass + above + eq))
            S.thr = ka;  // every writer of this class writes the same key
        }
        __syncthreads();
        thr = S.thr;
        for (int a = threadIdx.x; a < nm; a += blockDim.x)
          if (S.mkey[a] >= thr) {
            atomicAdd(&s_selc, 1u);
            atomicAdd(&s_selm, (unsigned long long)S.mmass[a]);
          }
        __syncthreads();
        TRACE("ranked");
        sel_cnt = above_cnt + s_selc;
        sel_mass = above_mass + s_selm;
        resolved = true;
      } else {
        // split the range by key: min/max key of the members, 4096 key bins
        if (threadIdx.x == 0) { S.kmin = 0xFFFFFFFFu; S.kmax = 0; }
        for (int i = threadIdx.x; i < kBins; i += blockDim.x) { S.cnt[i] = 0; S.mlo[i] = 0; S.mhi[i] = 0; }
        __syncthreads();
        for_each_logit(z, npos, [&](int, float zi) {
          if (zi == -INFINITY || dbin(zi, M) != bin) return;
          const uint32_t k = f2key(zi);
          if (k < klo || k > khi) return;
          atomicMin(&S.kmin, k);
          atomicMax(&S.kmax, k);
        });
        __syncthreads();
        const uint32_t kmin = S.kmin, kmax = S.kmax;
        if (kmin == kmax) {  // one tie class fills the range: it is the threshold
          thr = kmin;
          sel_cnt = above_cnt + members;
          sel_mass = above_mass + range_mass;
          break;
        }
        const int sh = max(0, (32 - __clz(kmax - kmin)) - 12);
        for_each_logit(z, npos, [&](int, float zi) {
          if (zi == -INFINITY || dbin(zi, M) != bin) return;
          const uint32_t k = f2key(zi);
          if (k < klo || k > khi) return;
          const int sb = (int)((k - kmin) >> sh);
          atomicAdd(&S.cnt[sb], 1u);
          const uint64_t mf = mass_fx(zi, M, fscale);
          if (mf) atomic_add_u64_split(&S.mlo[sb], &S.mhi[sb], mf);
        });
        __syncthreads();
        find_crossing(S, target, above_mass, true);  // highest key first
        if (S.bin < 0) {
          thr = kmin;
          sel_cnt = above_cnt + members;
          sel_mass = above_mass + range_mass;
          break;
        }
        const int sb = S.bin;
        above_mass = S.above_mass;
        above_cnt += S.above_cnt;
        members = (int)S.cnt[sb];
        range_mass = ((uint64_t)S.mhi[sb] << 32) | S.mlo[sb];
        klo = kmin + ((uint32_t)sb << sh);
        khi = min(kmax, klo + ((1u << sh) - 1u));
      }
    }
    __syncthreads();
  }
  TRACE("resolved");
  // selection bitmap of the head's pruned set {z >= thr} (key compares only)
  uint32_t* bits = buf.sel_bits + (size_t)qh * (T / 32);
  {
    const float4* z4 = reinterpret_cast<const float4*>(z);
    const int n4 = npos >> 2;
    const int lane = threadIdx.x & 31;
    for (int i0 = 0; i0 < n4; i0 += blockDim.x) {
      const int i = i0 + threadIdx.x;
      uint32_t nib = 0;
      if (i < n4) {
        const float4 v = __ldcg(z4 + i);
        nib = (v.x != -INFINITY && f2key(v.x) >= thr ? 1u : 0u) | (v.y != -INFINITY && f2key(v.y) >= thr ? 2u : 0u) |
              (v.z != -INFINITY && f2key(v.z) >= thr ? 4u : 0u) | (v.w != -INFINITY && f2key(v.w) >= thr ? 8u : 0u);
      }
      uint32_t w = nib << (4 * (lane & 7));
      w |= __shfl_xor_sync(0xffffffffu, w, 1);
      w |= __shfl_xor_sync(0xffffffffu, w, 2);
      w |= __shfl_xor_sync(0xffffffffu, w, 4);
      if ((lane & 7) == 0 && i < n4) bits[i >> 3] = w;
    }
  }
  if (threadIdx.x == 0) {
    buf.head_thr[qh] = thr;
    stats[0] = (float)sel_cnt;
    stats[1] = empty ? 0.f : (float)((double)sel_mass / (double)Z);
    stats[2] = empty ? 0.f : (float)((double)mass_fx(key2f(thr), M, fscale) / (double)Z);
    stats[3] = (float)b0;
  }
  TRACE("bitmap");
  // ---- K3c: the last head of the unit forms the group set
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(buf.unit_done + unit, 1) == G - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int* cand = buf.cand_pages + (size_t)unit * kv.max_pages;
  int* out = buf.final_idx + (size_t)unit * T;
  const int words = (npos + 31) >> 5;
  const uint32_t* hb = buf.sel_bits + (size_t)unit * G * (T / 32);
  uint32_t base = 0;
  for (int w0 = 0; w0 < words; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    uint32_t x = 0;
    if (w < words)
      for (int g = 0; g < G; ++g) x |= __ldcg(hb + (size_t)g * (T / 32) + w);
    uint32_t total;
    const uint32_t incl = block_incl_scan(__popc(x), S.tmp32, total);
    uint32_t pos = base + incl - __popc(x);
    while (x) {
      const int bit = __ffs(x) - 1;
      x &= x - 1;
      const int pp = w * 32 + bit;
      out[pos++] = cand[pp >> 4] * kPage + (pp & 15);
    }
    base += total;
  }
  if (threadIdx.x == 0) {
    buf.final_count[unit] = (int)base;
    const int chunk = prm.chunk_tokens > 0 ? prm.chunk_tokens : TW_DEFAULT_CHUNK;
    const int nitems = ((int)base + chunk - 1) / chunk;
    const int first = nitems ? (int)atomicAdd(&buf.counters[0], (uint32_t)nitems) : 0;
    buf.unit_items[2 * unit] = first;
    buf.unit_items[2 * unit + 1] = nitems;
    for (int i = 0; i < nitems; ++i) {
      if (first + i < buf.max_items) {
        buf.work_items[2 * (first + i)] = unit;
        buf.work_items[2 * (first + i) + 1] = i * chunk;
      }
    }
  }
}

// ---------------------------------------------------------------- Algorithm 1, literally

__device__ __forceinline__ double block_sum_d(double v, double* tmp) { return block_sum<double>(v, tmp); }

__device__ __forceinline__ double block_min_d(double v, double* tmp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) tmp[wid] = v;
  __syncthreads();
  double r = INFINITY;
  for (int i = 0; i < nw; ++i) r = fmin(r, tmp[i]);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) topp_bisect_kernel(const double* __restrict__ weights, int n, double p,
                                                          double eps, int max_iters, uint8_t* mask,
                                                          double* thr_out, int32_t* it_out) {
  __shared__ double tmp[32];
  const double* w = weights + (size_t)blockIdx.x * n;
  double s = 0.0, mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) { s += w[i]; mx = fmax(mx, w[i]); }
  const double total = block_sum_d(s, tmp);
  const double wmax = -block_min_d(-mx, tmp);
  const double p_eff = fmin(p, total) - 1e-9;
  uint8_t* mk = mask + (size_t)blockIdx.x * n;
  if (p_eff <= 0.0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) mk[i] = 0;
    if (threadIdx.x == 0) { thr_out[blockIdx.x] = INFINITY; it_out[blockIdx.x] = 0; }
    return;
  }
  double l = 0.0, r = wmax;
  int it = 0;
  while (true) {
    // live = {w >= l}
    double lm = INFINITY;
    for (int i = threadIdx.x; i < n; i += blockDim.x) if (w[i] >= l) lm = fmin(lm, w[i]);
    const double smallest = block_min_d(lm, tmp);
    const double m = 0.5 * (l + r);
    double above = 0.0, kept = 0.0, inside = 0.0, nabove = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double x = w[i];
      if (x < l) continue;
      if (x > smallest) { above += x; nabove += 1.0; }
      if (x < r && x > l) inside += 1.0;
      if (x >= m) kept += x;
    }
    above = block_sum_d(above, tmp);
    nabove = block_sum_d(nabove, tmp);
    inside = block_sum_d(inside, tmp);
    kept = block_sum_d(kept, tmp);
    if (nabove == 0.0) break;
    if (above < p_eff) break;
    if (it >= max_iters) break;
    if (r - l < eps) break;
    if (inside == 0.0) break;
    if (!(l < m && m < r)) break;
    if (kept >= p_eff) l = m; else r = m;
    ++it;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) mk[i] = w[i] >= l ? 1 : 0;
  if (threadIdx.x == 0) { thr_out[blockIdx.x] = l; it_out[blockIdx.x] = it; }
}

}  // namespace tw

using namespace tw;

#ifdef TW_TOPP_TRACE
extern "C" int tw_debug_trace(unsigned long long* host_out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, g_trace, sizeof(g_trace));
  int zeros[512] = {0};
  cudaMemcpyToSymbol(g_trace_phase, zeros, sizeof(zeros));
  return 0;
}
#endif

extern "C" int tw_topp(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
                       cudaStream_t stream) {
  if (!kv || !prm || !buf || !buf->logits || !buf->head_thr || !buf->head_stats || !buf->final_idx ||
      !buf->final_count || !buf->unit_items || !buf->work_items || !buf->counters)
    return TW_ERR_INVALID;
  if (!(prm->p >= 0.0 && prm->p <= 1.0)) return TW_ERR_INVALID;
  const int units = kv->num_seqs * kv->num_kv_heads;
  if (!buf->sel_bits || !buf->unit_done) return TW_ERR_INVALID;
  const size_t smem = sizeof(TopSmem);
  cudaFuncSetAttribute(topp_head_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaMemsetAsync(buf->unit_done, 0, sizeof(int32_t) * units, stream);
  topp_head_kernel<<<units * kv->group_size, kTopThreads, smem, stream>>>(*kv, *prm, *buf);
  return launch_status();
}

extern "C" int tw_topp_bisect(const double* weights, int32_t rows, int32_t n, double p, double epsilon,
                              int32_t max_iters, uint8_t* mask_out, double* threshold_out, int32_t* iters_out,
                              cudaStream_t stream) {
  if (!weights || rows < 1 || n < 1 || !(p >= 0.0 && p <= 1.0) || !(epsilon > 0.0) || max_iters < 1 ||
      !mask_out || !threshold_out || !iters_out)
    return TW_ERR_INVALID;
  topp_bisect_kernel<<<rows, 256, 0, stream>>>(weights, n, p, epsilon, max_iters, mask_out, threshold_out,
                                                iters_out);
  return launch_status();
}
