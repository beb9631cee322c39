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
#include <cfloat>

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

#ifndef TW_TOPP_THREADS
#define TW_TOPP_THREADS 512
#endif
constexpr int kTopThreads = TW_TOPP_THREADS;
#ifndef TW_TOPP_MINB
#define TW_TOPP_MINB 2
#endif
constexpr int kBins = 4096;
constexpr int kRankCap = 512;           // members ranked O(k^2) in shared memory
constexpr float kBinPerLogit = 120.0f;  // bins cover (max - z) in [0, 34.1)
constexpr int kNW = kTopThreads / 32;
constexpr int kPer = kBins / kTopThreads;
static_assert(kPer <= 8, "find_crossing's step table covers 8 bins per thread");
// exp(-i/120), i = 0..7
__device__ constexpr double kStepExp[8] = {1.0, 0.991701292638876, 0.9834714538216175, 0.9753099120283326,
                                           0.9672161004820059, 0.9591894571091382, 0.951229424500714,
                                           0.9433354498734922};

// Masses.  Bin b of (max - z) has top t_b = M - b/120 (float) and weight
// w_b = exp(t_b - M) (fp64).  A member has e_i = exp(z_i - M) = w_b r_i with
// r_i = exp(z_i - t_b) in (0.9917, 1]; it is summed as the u32 fixed-point
// deficit u_i = rint((1 - r_i) 2^kq) (< 2^kq / 120), so
//     bin mass = w_b (count - sum u / 2^kq).
// Counts and deficits are plain u32 shared-memory adds (no 64-bit carries),
// exact and order-independent => deterministic.  r_i comes from the SFU over
// a 1/120-logit range (~2e-7 relative); w_b is fp64.  The deepest bin (34+
// logits below the max, weights < 2e-15) takes whatever lands there.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// bin of z: floor((M - z) * 120), clamped to the last bin
__device__ __forceinline__ int dbin(float z, float M120) {
  return min(__float2int_rz(fmaf(-z, kBinPerLogit, M120)), kBins - 1);
}

// Largest float z with dbin(z) >= b (dbin is non-increasing in z), so bin b is
// the float interval (bin_ceiling(b + 1), bin_ceiling(b)].
__device__ __forceinline__ float bin_ceiling(int b, float M, float M120) {
  if (b <= 0) return INFINITY;
  if (b >= kBins) return -INFINITY;
  float e = M - (float)b / kBinPerLogit;
  for (int i = 0; i < 64 && dbin(e, M120) < b; ++i) e = nextafterf(e, -INFINITY);
  for (int i = 0; i < 64; ++i) {
    const float up = nextafterf(e, INFINITY);
    if (dbin(up, M120) < b) break;
    e = up;
  }
  return e;
}

__device__ __forceinline__ float bin_top(float M, int b) { return fmaf(-(float)b, 1.0f / kBinPerLogit, M); }

__device__ __forceinline__ uint32_t deficit(float z, float M, int b, float uscale) {
  const float r = ex2_approx((z - bin_top(M, b)) * 1.4426950408889634f);
  return (uint32_t)__float2int_rn(fmaxf(fmaf(-r, uscale, uscale), 0.0f));
}

__device__ __forceinline__ double class_mass(double w, uint64_t cnt, uint64_t usum, double inv_uscale) {
  return w * ((double)cnt - (double)usum * inv_uscale);
}

// CTA-wide inclusive scan with a compile-time warp count.
template <typename T>
__device__ __forceinline__ T cta_incl_scan(T v, T* tmp, T& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T s = lane < kNW ? tmp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kNW) tmp[lane] = s;
  }
  __syncthreads();
  if (wid > 0) x += tmp[wid - 1];
  total = tmp[kNW - 1];
  __syncthreads();
  return x;
}

struct TopSmem {
  uint32_t cnt[kBins];
  uint32_t usum[kBins];
  uint32_t mkey[kRankCap];
  uint32_t mu[kRankCap];
  double dtmp[32];
  uint32_t utmp[32];
  int nmem;
  uint32_t kmin, kmax;
  int bin;
  double above_mass;
  uint32_t above_cnt;
  uint32_t thr;
  uint32_t selc;
  unsigned long long selu;
};

// First bin in priority order whose running mass (from base_mass) reaches
// the target.  Level 0 (wconst <= 0): bins of (max - z) weighted w_b,
// priority = ascending b, target = p_eff * (total mass), returned as Z.
// Deeper levels: key sub-bins of one parent bin, all weighted wconst,
// priority = descending index (highest key first).  Also returns the count
// of everything scanned in `count_total`.
__device__ __forceinline__ double find_crossing(TopSmem& S, double target, double base_mass, float M, double wconst,
                                                double inv_uscale, double p_eff, uint32_t& count_total) {
  const bool level0 = !(wconst > 0.0);
  double m[kPer];
  uint32_t c[kPer];
  double w0 = wconst;
  float t0 = 0.f;
  if (level0) {  // w_b for this thread's kPer consecutive bins: one exp, then exact small-step corrections
    t0 = bin_top(M, threadIdx.x * kPer);
    w0 = exp((double)t0 - (double)M);
  }
  double local = 0.0;
  uint32_t lcnt = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int rank = threadIdx.x * kPer + i;
    const int bb = level0 ? rank : (kBins - 1 - rank);
    c[i] = S.cnt[bb];
    double w = wconst;
    if (level0) {
      // exp(t_b - M) = w0 * exp(t_b - t0);  t_b - t0 = -i/120 + d (d ~ float rounding, tiny)
      const double d = ((double)bin_top(M, bb) - (double)t0) + (double)i / (double)kBinPerLogit;
      w = w0 * kStepExp[i] * (1.0 + d * (1.0 + 0.5 * d));
    }
    m[i] = c[i] ? class_mass(w, c[i], S.usum[bb], inv_uscale) : 0.0;
    local += m[i];
    lcnt += c[i];
  }
  double total;
  const double incl = cta_incl_scan<double>(local, S.dtmp, total);
  uint32_t ctot;
  const uint32_t cincl = cta_incl_scan<uint32_t>(lcnt, S.utmp, ctot);
  count_total = ctot;
  if (level0) target = p_eff * total;
  const double excl = incl - local;
  if (threadIdx.x == 0) S.bin = -1;
  __syncthreads();
  if (base_mass + excl < target && target <= base_mass + incl) {
    double run = base_mass + excl;
    uint32_t crun = cincl - lcnt;
    bool found = false;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      if (!found && c[i] && run + m[i] >= target) {
        found = true;
        S.bin = level0 ? threadIdx.x * kPer + i : kBins - 1 - (threadIdx.x * kPer + i);
        S.above_mass = run;
        S.above_cnt = crun;
      }
      run += m[i];
      crun += c[i];
    }
  }
  __syncthreads();
  return total;
}

// Vectorised walk over a head's logits: kUnroll float4 in flight per thread.
#ifndef TW_TOPP_UNROLL
#define TW_TOPP_UNROLL 4
#endif
constexpr int kUnroll = TW_TOPP_UNROLL;
template <typename F>
__device__ __forceinline__ void for_each_logit(const float* __restrict__ z, int npos, F&& f) {
  const float4* z4 = reinterpret_cast<const float4*>(z);
  const int n4 = npos >> 2;
  for (int base = threadIdx.x; base < n4; base += kTopThreads * kUnroll) {
    float4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int i = base + u * kTopThreads;
      v[u] = i < n4 ? __ldcg(z4 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      f(v[u].x);
      f(v[u].y);
      f(v[u].z);
      f(v[u].w);
    }
  }
}

// One CTA per query head; the last head of a unit to finish also forms the
// group's final set (K3c) and reserves its attention work items.
__global__ void __launch_bounds__(kTopThreads, TW_TOPP_MINB) topp_head_kernel(tw_paged_kv kv, tw_decode_params prm,
                                                                               tw_decode_buffers buf) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TopSmem& S = *reinterpret_cast<TopSmem*>(smem_raw);
  __shared__ int s_last;
  const int qh = blockIdx.x;
  const int G = kv.group_size;
  const int unit = qh / G;
  const int npos = buf.cand_count[unit] * kPage;
  const size_t T = (size_t)kv.max_pages * kPage;
  const float* z = buf.logits + (size_t)qh * T;
  const float M = key2f(buf.head_max[qh]);
  const float M120 = M * kBinPerLogit;
  const double p_eff = fmin(prm.p, 1.0) - 1e-9;
  float* stats = buf.head_stats + (size_t)qh * 4;
  uint32_t thr = 0xFFFFFFFFu;  // selects nothing
  uint32_t b0 = 0;
  double Z = 0.0;
  uint32_t sel_cnt = 0;        // |{z >= thr}|   (from the histograms, no extra pass)
  double sel_mass = 0.0;       // its mass
  // deficit scale: a bin's u32 sum holds up to 2^32 / (2^kq / 120) members
  const float uscale = npos > 120000 ? 1048576.0f : 4194304.0f;
  const double inv_uscale = 1.0 / (double)uscale;
  const bool empty = p_eff <= 0.0 || npos == 0 || !(M > -INFINITY);
  TRACE("start");
  if (!empty) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      S.cnt[threadIdx.x + i * kTopThreads] = 0;
      S.usum[threadIdx.x + i * kTopThreads] = 0;
    }
    __syncthreads();
    for_each_logit(z, npos, [&](float zi) {
      if (zi > -INFINITY) {
        const int bb = dbin(zi, M120);
        atomicAdd(&S.cnt[bb], 1u);
        atomicAdd(&S.usum[bb], deficit(zi, M, bb, uscale));
      }
    });
    __syncthreads();
    TRACE("pass1");
    Z = find_crossing(S, 0.0, 0.0, M, 0.0, inv_uscale, p_eff, b0);
    const double target = p_eff * Z;
    TRACE("crossing");
    int bin = S.bin;
    double above_mass = S.above_mass;
    uint32_t above_cnt = S.above_cnt;
    uint32_t klo = 0, khi = 0xFFFFFFFFu;
    bool resolved = false;
    if (bin < 0) {  // rounding: the whole set is needed
      thr = 0;
      sel_cnt = b0;
      sel_mass = Z;
      resolved = true;
    }
    const int pbin = bin;  // parent bin of every deeper level
    __shared__ float s_zr[2];
    if (!resolved && threadIdx.x == 0) {
      s_zr[0] = bin_ceiling(pbin + 1, M, M120);  // members: zlo < z <= zhi
      s_zr[1] = bin_ceiling(pbin, M, M120);
    }
    __syncthreads();
    const float zlo = s_zr[0], zhi = s_zr[1];
    const double wb = resolved ? 0.0 : exp((double)bin_top(M, pbin) - (double)M);
    int members = resolved ? 0 : (int)S.cnt[bin];
    double range_mass = resolved ? 0.0 : class_mass(wb, S.cnt[bin], S.usum[bin], inv_uscale);
    while (!resolved) {
      __syncthreads();
      if (members <= kRankCap) {
        // compact the members, then rank them exactly
        if (threadIdx.x == 0) { S.nmem = 0; S.selc = 0; S.selu = 0; }
        __syncthreads();
        for_each_logit(z, npos, [&](float zi) {
          if (zi > zlo && zi <= zhi) {
            const uint32_t k = f2key(zi);
            if (k >= klo && k <= khi) {
              const int slot = atomicAdd(&S.nmem, 1);
              if (slot < kRankCap) {
                S.mkey[slot] = k;
                S.mu[slot] = deficit(zi, M, pbin, uscale);
              }
            }
          }
        });
        __syncthreads();
        TRACE("members");
        const int nm = min(S.nmem, kRankCap);
        if (threadIdx.x == 0) S.thr = klo;  // fallback (rounding): keep the whole range
        __syncthreads();
        for (int a = threadIdx.x; a < nm; a += kTopThreads) {
          const uint32_t ka = S.mkey[a];
          uint32_t cgt = 0, ceq = 0;
          uint64_t ugt = 0, ueq = 0;
          for (int j = 0; j < nm; ++j) {
            const uint32_t kj = S.mkey[j];
            const uint32_t uj = S.mu[j];
            cgt += kj > ka;
            ugt += kj > ka ? uj : 0u;
            ceq += kj == ka;
            ueq += kj == ka ? uj : 0u;
          }
          const double lo = above_mass + class_mass(wb, cgt, ugt, inv_uscale);
          const double hi = lo + class_mass(wb, ceq, ueq, inv_uscale);
          if (lo < target && target <= hi) S.thr = ka;  // every writer of this class writes the same key
        }
        __syncthreads();
        thr = S.thr;
        for (int a = threadIdx.x; a < nm; a += kTopThreads)
          if (S.mkey[a] >= thr) {
            atomicAdd(&S.selc, 1u);
            atomicAdd(&S.selu, (unsigned long long)S.mu[a]);
          }
        __syncthreads();
        TRACE("ranked");
        sel_cnt = above_cnt + S.selc;
        sel_mass = above_mass + class_mass(wb, S.selc, S.selu, inv_uscale);
        resolved = true;
      } else {
        // split the range by key: min/max key of the members, 4096 key sub-bins
        if (threadIdx.x == 0) { S.kmin = 0xFFFFFFFFu; S.kmax = 0; }
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
          S.cnt[threadIdx.x + i * kTopThreads] = 0;
          S.usum[threadIdx.x + i * kTopThreads] = 0;
        }
        __syncthreads();
        for_each_logit(z, npos, [&](float zi) {
          if (zi > zlo && zi <= zhi) {
            const uint32_t k = f2key(zi);
            if (k >= klo && k <= khi) {
              atomicMin(&S.kmin, k);
              atomicMax(&S.kmax, k);
            }
          }
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
        for_each_logit(z, npos, [&](float zi) {
          if (zi > zlo && zi <= zhi) {
            const uint32_t k = f2key(zi);
            if (k >= klo && k <= khi) {
              const int sb = (int)((k - kmin) >> sh);
              atomicAdd(&S.cnt[sb], 1u);
              atomicAdd(&S.usum[sb], deficit(zi, M, pbin, uscale));
            }
          }
        });
        __syncthreads();
        uint32_t dummy;
        find_crossing(S, target, above_mass, M, wb, inv_uscale, p_eff, dummy);  // highest key first
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
        range_mass = class_mass(wb, S.cnt[sb], S.usum[sb], inv_uscale);
        klo = kmin + ((uint32_t)sb << sh);
        khi = min(kmax, klo + ((1u << sh) - 1u));
      }
    }
    __syncthreads();
  }
  TRACE("resolved");
  // selection bitmap of the head's pruned set {z >= z_thr} (float compares; -inf never selected)
  uint32_t* bits = buf.sel_bits + (size_t)qh * (T / 32);
  {
    const float zthr = thr == 0u ? -FLT_MAX : key2f(thr);  // thr = ~0 -> NaN: selects nothing
    const float4* z4 = reinterpret_cast<const float4*>(z);
    const int n4 = npos >> 2;
    const int lane = threadIdx.x & 31;
    for (int i0 = 0; i0 < n4; i0 += kTopThreads * kUnroll) {
      float4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int i = i0 + u * kTopThreads + threadIdx.x;
        v[u] = i < n4 ? __ldcg(z4 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int i = i0 + u * kTopThreads + threadIdx.x;
        const uint32_t nib = (v[u].x >= zthr ? 1u : 0u) | (v[u].y >= zthr ? 2u : 0u) | (v[u].z >= zthr ? 4u : 0u) |
                             (v[u].w >= zthr ? 8u : 0u);
        uint32_t w = nib << (4 * (lane & 7));
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        w |= __shfl_xor_sync(0xffffffffu, w, 4);
        if ((lane & 7) == 0 && i < n4) bits[i >> 3] = w;
      }
    }
  }
  if (threadIdx.x == 0) {
    buf.head_thr[qh] = thr;
    stats[0] = (float)sel_cnt;
    stats[1] = empty ? 0.f : (float)(sel_mass / Z);
    stats[2] = empty ? 0.f : (float)(exp((double)key2f(thr) - (double)M) / Z);
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
  for (int w0 = 0; w0 < words; w0 += kTopThreads) {
    const int w = w0 + threadIdx.x;
    uint32_t x = 0;
    if (w < words)
      for (int g = 0; g < G; ++g) x |= __ldcg(hb + (size_t)g * (T / 32) + w);
    // a word covers candidate pages 2w and 2w+1: fetch both page ids before the scan
    const int c0 = x & 0xFFFFu ? cand[2 * w] * kPage : 0;
    const int c1 = x >> 16 ? cand[2 * w + 1] * kPage - 16 : 0;
    uint32_t total;
    const uint32_t incl = cta_incl_scan<uint32_t>(__popc(x), S.utmp, total);
    uint32_t pos = base + incl - __popc(x);
    while (x) {
      const int bit = __ffs(x) - 1;
      x &= x - 1;
      out[pos++] = (bit < 16 ? c0 : c1) + bit;
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
