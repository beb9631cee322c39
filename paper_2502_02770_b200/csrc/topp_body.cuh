// Top-p body shared by the per-unit top-p kernel (topp.cu) and the fused
// per-unit select/estimate/top-p kernel (unit.cu).  See topp.cu for the method.
#pragma once
#include <cfloat>

#include "block_scan.cuh"

namespace tw {

#ifdef TW_TOPP_TRACE
static __device__ unsigned long long g_tt[1024][8];
#define TT(ph)                                                                                       \
  do {                                                                                               \
    if (threadIdx.x == 0 && blockIdx.x < 1024) {                                                     \
      unsigned long long now_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_));                                      \
      g_tt[blockIdx.x][ph] = now_;                                                                   \
    }                                                                                                \
  } while (0)
#else
#define TT(ph) do {} while (0)
#endif

constexpr int kBins = TW_TOPP_BINS;      // 4096
// per-head histograms are stored with one pad word per 16 bins, so the crossing
// scan's threads (16 consecutive bins each) read different banks
constexpr int kBinsP = kBins + kBins / 16;
__device__ __forceinline__ int hidx(int b) { return b + (b >> 4); }
constexpr float kBinPerLogit = 120.0f;   // bins cover (max - z) in [0, 34.1); the last bin takes the rest
constexpr int kHB = 4;                   // heads whose histograms are resident at once (4 x 32 KB)
constexpr int kMemberCap = TW_TOPP_MEMBER_CAP;
constexpr int kResBuckets = 1024;        // key buckets per refinement level
constexpr int kRankCap = 64;             // members ranked exactly (O(k^2))
constexpr float kUscale = 4194304.0f;    // deficits in units of 2^-22
constexpr double kInvUscale = 1.0 / 4194304.0;
// exp(-i/120), i = 0..15
static __constant__ float kStepExpF[16] = {
    1.0f, 0.991701292638876f, 0.9834714538216175f, 0.9753099120283326f, 0.9672161004820059f, 0.9591894571091382f,
    0.951229424500714f, 0.9433354498734922f, 0.9355069850316178f, 0.9277434863285529f, 0.9200444146293233f,
    0.9124092352730778f, 0.9048374180359595f, 0.8973284370942841f, 0.8898817709880238f, 0.8824969025845955f};
// Masses.  Bin b of (max - z) has top t_b = M - b/120 (float) and weight
// w_b = exp(t_b - M) (fp64).  A member has e_i = exp(z_i - M) = w_b r_i with
// r_i = exp(z_i - t_b) in (0.9917, 1]; it is summed as the fixed-point deficit
// u_i = rint((1 - r_i) 2^22), so bin mass = w_b (count - sum u / 2^22).  r_i
// comes from the SFU over a 1/120-logit range (~2e-7 relative); w_b is fp64.
// The deepest bin (34+ logits below the max, weights < 2e-15) takes whatever
// lands there.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ int dbin(float z, float M120) {
  return min(__float2int_rz(fmaf(-z, kBinPerLogit, M120)), kBins - 1);
}
__device__ __forceinline__ float bin_top(float M, int b) { return fmaf(-(float)b, 1.0f / kBinPerLogit, M); }
// Largest float z with dbin(z) >= b (dbin is non-increasing in z), so bin b
// is the float interval (bin_ceiling(b + 1), bin_ceiling(b)].  The guess
// M - b/120 is off by the rounding of M120 (~|M| 3e-8 absolute), which near
// z = 0 is hundreds of ulps, so the exact boundary is found by bisection over
// the ordered float keys of a bracket much wider than that error and much
// narrower than a bin.
static __device__ __noinline__ float bin_ceiling(int b, float M, float M120) {
  if (b <= 0) return INFINITY;
  if (b >= kBins) return -INFINITY;
  const float e = M - (float)b / kBinPerLogit;
#ifdef TW_OLD_BIN_CEILING  // the round-1 64-ulp walk, kept only to show the regression test catches it
  float x = e;
  for (int i = 0; i < 64 && dbin(x, M120) < b; ++i) x = nextafterf(x, -INFINITY);
  for (int i = 0; i < 64; ++i) {
    const float up = nextafterf(x, INFINITY);
    if (dbin(up, M120) < b) break;
    x = up;
  }
  return x;
#endif
  // fast path: the edge is usually within a few ulps of the guess
  {
    float x = e;
    int i = 0;
    for (; i < 8 && dbin(x, M120) < b; ++i) x = nextafterf(x, -INFINITY);
    if (i < 8) {
      for (i = 0; i < 8; ++i) {
        const float up = nextafterf(x, INFINITY);
        if (dbin(up, M120) < b) return x;
        x = up;
      }
    }
  }
  const float d = 2e-3f;  // a quarter bin
  uint32_t lo = f2key(e - d), hi = f2key(e + d);  // dbin(lo) >= b > dbin(hi)
  while (hi - lo > 1) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (dbin(key2f(mid), M120) >= b) lo = mid;
    else hi = mid;
  }
  return key2f(lo);
}
__device__ __forceinline__ uint32_t deficit(float z, float M, int b) {
  const float r = ex2_approx((z - bin_top(M, b)) * 1.4426950408889634f);
  return (uint32_t)__float2int_rn(fmaxf(fmaf(-r, kUscale, kUscale), 0.0f));
}
__device__ __forceinline__ double class_mass(double w, uint64_t cnt, uint64_t usum) {
  return w * ((double)cnt - (double)usum * kInvUscale);
}
__device__ __forceinline__ float4 ninf4() { return make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY); }
__device__ __forceinline__ float comp(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }

// Inclusive scans of a (double, u32) pair per thread in one pass (two group barriers).
__device__ __forceinline__ void grp_scan2(const Group& g, double v, uint32_t u, double* dtmp, uint32_t* utmp,
                                          double& incl, uint32_t& uincl, double& total, uint32_t& utotal) {
  const int lane = g.tid & 31, wid = g.warp(), nw = g.nwarps();
  double x = v;
  uint32_t y = u;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double xs = __shfl_up_sync(0xffffffffu, x, o);
    const uint32_t ys = __shfl_up_sync(0xffffffffu, y, o);
    if (lane >= o) { x += xs; y += ys; }
  }
  if (lane == 31) { dtmp[wid] = x; utmp[wid] = y; }
  g.sync();
  double pre = 0.0, tot = 0.0;
  uint32_t upre = 0, utot = 0;
  for (int i = 0; i < nw; ++i) {
    const double sd = dtmp[i];
    const uint32_t su = utmp[i];
    pre += i < wid ? sd : 0.0;
    tot += sd;
    upre += i < wid ? su : 0u;
    utot += su;
  }
  g.sync();
  incl = x + pre;
  uincl = y + upre;
  total = tot;
  utotal = utot;
}

template <typename T>
__device__ __forceinline__ T grp_scan(const Group& g, T v, T* tmp, T& total) {
  const int lane = g.tid & 31, wid = g.warp(), nw = g.nwarps();
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  g.sync();
  T pre = T(0), tot = T(0);
  for (int i = 0; i < nw; ++i) {
    const T s = tmp[i];
    pre += i < wid ? s : T(0);
    tot += s;
  }
  g.sync();
  total = tot;
  return x + pre;
}

struct ResGroupSmem {
  uint32_t bc[kResBuckets];
  unsigned long long bu[kResBuckets];
  uint32_t rk[kRankCap], ru[kRankCap];
  double dtmp[32];
  uint32_t utmp[32];
  unsigned long long ltmp[32];
  uint32_t kmin, kmax, live, thr;
  int nr, bin;
  double above;
};

// members of one head's crossing bin: a segment of the shared member list ...
struct SmemSrc {
  const uint32_t* keys;
  const uint32_t* pos;
  int m;
  float M;
  int cb;
  template <class F>
  __device__ __forceinline__ void each(const Group& g, F&& f) const {
    for (int i = g.tid; i < m; i += g.nthreads) {
      const uint32_t k = keys[i];
      f(k, deficit(key2f(k), M, cb), pos[i]);
    }
  }
};
// ... or, when the list overflowed, found again by re-reading the head's logits
struct LogitSrc {
  const float* z;
  int npos;
  float M;
  int cb;
  template <class F>
  __device__ __forceinline__ void each(const Group& g, F&& f) const {
    const float4* z4 = reinterpret_cast<const float4*>(z);
    const float M120 = M * kBinPerLogit;
    for (int i = g.tid; i < (npos >> 2); i += g.nthreads) {
      const float4 v = __ldcg(z4 + i);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float x = comp(v, e);
        if (x > -INFINITY && dbin(x, M120) == cb) f(f2key(x), deficit(x, M, cb), (uint32_t)(4 * i + e));
      }
    }
  }
};

// Threshold key inside the crossing bin: the key of the class at which the
// running mass (highest key first, from `base`) reaches `target`.  Members
// share the bin weight wb, so a class's mass is wb (count - sum u / 2^22).
template <class Src>
__device__ uint32_t resolve_threshold(const Group& g, const Src& src, double base, double target, double wb,
                                      ResGroupSmem& S) {
  const int lane = g.tid & 31;
  uint32_t klo = 0, khi = 0xFFFFFFFFu;
  for (int level = 0; level < 6; ++level) {
    if (g.tid == 0) { S.kmin = 0xFFFFFFFFu; S.kmax = 0; S.live = 0; S.nr = 0; S.bin = -1; }
    g.sync();
    uint32_t lmin = 0xFFFFFFFFu, lmax = 0, lc = 0;
    src.each(g, [&](uint32_t k, uint32_t, uint32_t) {
      if (k >= klo && k <= khi) { lmin = min(lmin, k); lmax = max(lmax, k); ++lc; }
    });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lmin = min(lmin, __shfl_xor_sync(0xffffffffu, lmin, o));
      lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
      lc += __shfl_xor_sync(0xffffffffu, lc, o);
    }
    if (lane == 0 && lc) { atomicMin(&S.kmin, lmin); atomicMax(&S.kmax, lmax); atomicAdd(&S.live, lc); }
    g.sync();
    const uint32_t kmin = S.kmin, kmax = S.kmax, live = S.live;
    if (live == 0) return klo;
    if (kmin == kmax) return kmin;  // one tie class fills the range: it is the threshold
    if (live <= kRankCap) {
      src.each(g, [&](uint32_t k, uint32_t u, uint32_t) {
        if (k >= klo && k <= khi) {
          const int s = atomicAdd(&S.nr, 1);
          S.rk[s] = k;
          S.ru[s] = u;
        }
      });
      if (g.tid == 0) S.thr = kmin;  // rounding fallback: keep the whole range
      g.sync();
      for (int a = g.tid; a < (int)live; a += g.nthreads) {
        const uint32_t ka = S.rk[a];
        uint32_t cgt = 0, ceq = 0;
        uint64_t ugt = 0, ueq = 0;
        for (int j = 0; j < (int)live; ++j) {
          const uint32_t kj = S.rk[j], uj = S.ru[j];
          cgt += kj > ka;
          ugt += kj > ka ? uj : 0u;
          ceq += kj == ka;
          ueq += kj == ka ? uj : 0u;
        }
        const double lo = base + class_mass(wb, cgt, ugt);
        const double hi = lo + class_mass(wb, ceq, ueq);
        if (lo < target && target <= hi) S.thr = ka;  // every writer of this class writes the same key
      }
      g.sync();
      return S.thr;
    }
    // split the live range into key buckets, highest key first
    const int sh = max(0, (32 - __clz(kmax - kmin)) - 10);
    for (int i = g.tid; i < kResBuckets; i += g.nthreads) { S.bc[i] = 0; S.bu[i] = 0; }
    g.sync();
    src.each(g, [&](uint32_t k, uint32_t u, uint32_t) {
      if (k >= klo && k <= khi) {
        const int bk = (int)((k - kmin) >> sh);
        atomicAdd(&S.bc[bk], 1u);
        atomicAdd(&S.bu[bk], (unsigned long long)u);
      }
    });
    g.sync();
    const int per = kResBuckets / g.nthreads;  // buckets per thread, highest key first
    double local = 0.0;
    for (int i = 0; i < per; ++i) {
      const int bk = kResBuckets - 1 - (g.tid * per + i);
      local += S.bc[bk] ? class_mass(wb, S.bc[bk], S.bu[bk]) : 0.0;
    }
    double total;
    const double incl = grp_scan<double>(g, local, S.dtmp, total);
    const double excl = incl - local;
    if (base + excl < target && target <= base + incl) {
      double run = base + excl;
      for (int i = 0; i < per; ++i) {
        const int bk = kResBuckets - 1 - (g.tid * per + i);
        const double mb = S.bc[bk] ? class_mass(wb, S.bc[bk], S.bu[bk]) : 0.0;
        if (S.bc[bk] && run + mb >= target) {
          S.bin = bk;
          S.above = run;
          break;
        }
        run += mb;
      }
    }
    g.sync();
    if (S.bin < 0) return kmin;  // rounding: keep the whole range
    base = S.above;
    klo = kmin + ((uint32_t)S.bin << sh);
    khi = kmax - klo > (1u << sh) - 1u ? klo + ((1u << sh) - 1u) : kmax;
    g.sync();
  }
  return klo;
}


// Per-head record (shared memory of the unit's CTA).
struct HeadRec {
  double above_mass;  // mass of the bins above the crossing bin
  double target;      // p_eff * Z
  double Z;           // total mass (in units of exp(z - max))
  double wb;          // weight of the crossing bin's top, exp(t_cb - max)
  int cb;             // crossing bin; -1: keep every candidate; -2: keep nothing
  uint32_t above_cnt, members, b0;
  float M;            // max logit
  float zhi, zlo;     // crossing bin = (zlo, zhi]: kept outright iff z > zhi
  int seg;            // member-list segment start (-1: resolved by re-reading the logits)
};

// HB = heads whose histograms are resident at once.  The wide variant (HB = 4)
// runs one 1024-thread CTA per SM; the narrow one (HB = 2 for G = 4, half the
// member list) fits two per SM, for batches with more units than SMs.
template <int G, int HB, int GTO = 0>
struct UnitCfg {
  static constexpr int GB = G < HB ? G : HB;    // heads per histogram batch
  static constexpr int GT = GTO ? GTO : G <= 2 ? 512 : 256;  // threads per head (warp group)
  static constexpr int NT = GT * GB;            // threads
  static constexpr int MC = HB >= kHB ? kMemberCap : kMemberCap / 2;  // member-list capacity
  static constexpr size_t kHistBytes = (size_t)GB * kBinsP * 8;
  static constexpr size_t kResBytes = (size_t)GB * sizeof(ResGroupSmem);
  static constexpr size_t kSmem = (kHistBytes > kResBytes ? kHistBytes : kResBytes) + (size_t)MC * 8;
  // the union bitmap lives in the histogram region (dead after the crossing
  // scan) behind the resolve scratch, when the context fits
  static constexpr size_t kBitsOff = (kResBytes + 15) & ~size_t(15);
  static constexpr size_t kBitsCap = kHistBytes > kBitsOff ? (kHistBytes - kBitsOff) / 4 : 0;  // words
};

// One unit's top-p (CTA of UnitCfg<G, HB>::NT threads; `sm` = UnitCfg::kSmem bytes of dynamic shared memory).
template <int G, int HB, bool SB, int GTO = 0>
__device__ __forceinline__ void topp_unit_body(const int unit, const tw_paged_kv& kv, const tw_decode_params& prm,
                                               const tw_decode_buffers& buf, unsigned char* sm) {
  using Cfg = UnitCfg<G, HB, GTO>;
  constexpr int GB = Cfg::GB, NT = Cfg::NT, kGT = Cfg::GT, MC = Cfg::MC;
  constexpr int kPerT = kBins / kGT;  // bins per thread in the crossing scan
  uint32_t* Hc = reinterpret_cast<uint32_t*>(sm);                           // [GB][kBinsP] counts
  uint32_t* Hu = Hc + GB * kBinsP;                                           // [GB][kBinsP] deficit sums
  ResGroupSmem* RS = reinterpret_cast<ResGroupSmem*>(sm);                    // [GB] (aliases the bins)
  uint32_t* mkey = reinterpret_cast<uint32_t*>(sm + Cfg::kSmem - (size_t)MC * 8);  // [MC]
  uint32_t* mpos = mkey + MC;                                                 // [MC]
  __shared__ HeadRec R[G];
  __shared__ unsigned long long s_deep[GB];
  __shared__ int s_fill[G];
  __shared__ int s_first;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gp = tid / kGT;
  const Group grp{1 + gp, kGT, tid % kGT};
  const size_t T = (size_t)kv.max_pages * kPage;
  const int npos = buf.cand_count[unit] * kPage;
  const int n4 = npos >> 2;
  const float* zu = buf.logits + (size_t)unit * G * T;
  // SB: the bitmap in shared memory (pass 2 writes every word it covers, so no zeroing)
  uint32_t* ubits = SB ? reinterpret_cast<uint32_t*>(sm + Cfg::kBitsOff)
                       : buf.sel_bits + (size_t)unit * ((T + 31) / 32);
  auto ld_bits = [&](int w) -> uint32_t {
    if constexpr (SB) return ubits[w];
    else return __ldcg(ubits + w);
  };
  const double p_eff = fmin(prm.p, 1.0) - 1e-9;
  if (tid < G) {
    const float M = key2f(buf.head_max[(size_t)unit * G + tid]);  // NaN when the head has no valid logit
    HeadRec r{};
    r.M = M;
    r.cb = (p_eff <= 0.0 || npos == 0 || !(M > -INFINITY)) ? -2 : 0;
    r.zhi = r.zlo = INFINITY;
    r.seg = -1;
    R[tid] = r;
    s_fill[tid] = 0;
  }
  __syncthreads();
  TT(0);

  // ---- pass 1 (per batch of GB heads): bins, then each head's crossing bin
#pragma unroll 1
  for (int g0 = 0; g0 < G; g0 += GB) {
    for (int i = tid; i < GB * kBinsP; i += NT) Hc[i] = Hu[i] = 0;
    if (tid < GB) s_deep[tid] = 0;
    __syncthreads();
    {
      float Mh[GB], m120[GB];
      bool act[GB];
      unsigned long long deep[GB];
#pragma unroll
      for (int h = 0; h < GB; ++h) {
        act[h] = g0 + h < G && R[g0 + h].cb != -2;
        Mh[h] = act[h] ? R[g0 + h].M : 0.f;
        m120[h] = Mh[h] * kBinPerLogit;
        deep[h] = 0;
      }
#pragma unroll (G >= 4 ? 4 : 2)  // logit-pass unrolling, measured per G (C2/C5 vs C3)
      for (int i = tid; i < n4; i += NT) {
        float4 v[GB];
#pragma unroll
        for (int h = 0; h < GB; ++h)
          v[h] = act[h] ? __ldcg(reinterpret_cast<const float4*>(zu + (size_t)(g0 + h) * T) + i) : ninf4();
#pragma unroll
        for (int h = 0; h < GB; ++h)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float z = comp(v[h], e);
            if (z > -INFINITY) {
              const int b = dbin(z, m120[h]);
              const uint32_t d = deficit(z, Mh[h], b);
              atomicAdd(&Hc[h * kBinsP + hidx(b)], 1u);
              if (b < kBins - 1) atomicAdd(&Hu[h * kBinsP + hidx(b)], d);
              else deep[h] += d;  // the deepest bin's deficits (up to 2^22 each) need 64 bits
            }
          }
      }
#pragma unroll
      for (int h = 0; h < GB; ++h) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) deep[h] += __shfl_xor_sync(0xffffffffu, deep[h], o);
        if (lane == 0 && deep[h]) atomicAdd(&s_deep[h], deep[h]);
      }
    }
    __syncthreads();
    TT(1);
    const int g = g0 + gp;
    if (g < G && R[g].cb != -2) {  // uniform per warp group
      const uint32_t* hc = Hc + gp * kBinsP;
      const uint32_t* hu = Hu + gp * kBinsP;
      const float M = R[g].M;
      const float M120 = M * kBinPerLogit;
      const int bfirst = grp.tid * kPerT;
      const float t0 = bin_top(M, bfirst);
      // Bin masses in fp32 (relative error ~2e-7 each, all terms positive, summed in
      // fp64): the crossing search tolerates that (the top-p contract allows 1e-6),
      // and fp64 per bin was the slowest part of this phase.
      const float w0 = (float)exp((double)t0 - (double)M);
#ifdef TW_TT_SPLIT
      if (gp == 0) TT(6);
#endif
      auto mass = [&](int i, uint32_t& c) -> double {
        const int bb = bfirst + i;
        c = hc[hidx(bb)];
        if (!c) return 0.0;
        const uint64_t us = bb == kBins - 1 ? (uint64_t)s_deep[gp] : (uint64_t)hu[hidx(bb)];
        // exp(t_b - M) = w0 * exp(t_b - t0);  t_b - t0 = -i/120 + d (d ~ float rounding, tiny)
        const float d = (bin_top(M, bb) - t0) + (float)i * (1.0f / 120.0f);
        const float w = w0 * kStepExpF[i] * (1.0f + d);
        return (double)(w * ((float)c - (float)us * (float)kInvUscale));
      };
      static_assert(kPerT <= 16, "kStepExp covers 16 bins per thread");
      double local = 0.0;
      uint32_t lc = 0;
#pragma unroll 4
      for (int i = 0; i < kPerT; ++i) {
        uint32_t c;
        local += mass(i, c);
        lc += c;
      }
      double Z;
      uint32_t b0;
      __shared__ double s_dtmp[GB][kGT / 32];
      __shared__ uint32_t s_utmp[GB][kGT / 32];
#ifndef TW_TT_SPLIT
      if (gp == 0) TT(6);
#endif
      double incl;
      uint32_t cincl;
      grp_scan2(grp, local, lc, s_dtmp[gp], s_utmp[gp], incl, cincl, Z, b0);
      const double target = p_eff * Z;
      HeadRec& r = R[g];
      if (grp.tid == 0) {  // defaults: -1 = rounding left the target above the total -> keep everything
        r.cb = -1;
        r.Z = Z;
        r.target = target;
        r.b0 = b0;
        r.zhi = r.zlo = -INFINITY;
      }
      grp.sync();
      const double excl = incl - local;
      if (excl < target && target <= incl) {  // the one thread holding the crossing bin records it
        double run = excl;
        uint32_t crun = cincl - lc;
#pragma unroll 1
        for (int i = 0; i < kPerT; ++i) {
          uint32_t c;
          const double m = mass(i, c);
          if (c && run + m >= target) {
            const int cb = bfirst + i;
            r.cb = cb;
            r.above_mass = run;
            r.above_cnt = crun;
            r.members = c;
            r.wb = exp((double)bin_top(M, cb) - (double)M);
            r.zhi = bin_ceiling(cb, M, M120);
            r.zlo = bin_ceiling(cb + 1, M, M120);
            break;
          }
          run += m;
          crun += c;
        }
      }
      if (gp == 0) TT(7);
    }
    __syncthreads();
  }
  TT(2);
  // member-list segments: heads in order while they fit; the rest re-read their logits
  if (tid == 0) {
    uint32_t acc = 0;
    for (int g = 0; g < G; ++g) {
      HeadRec& r = R[g];
      if (r.cb >= 0 && acc + r.members <= (uint32_t)MC) {
        r.seg = (int)acc;
        acc += r.members;
      } else if (r.cb >= 0) {
        r.zlo = r.zhi;  // empty member range in pass 2
      }
    }
  }
  __syncthreads();

  // ---- pass 2: union of the heads' outright-kept positions + crossing-bin members
  {
    float zhi[G], zlo[G];
    int sg[G];
#pragma unroll
    for (int g = 0; g < G; ++g) { zhi[g] = R[g].zhi; zlo[g] = R[g].zlo; sg[g] = R[g].seg; }
#pragma unroll (G >= 4 ? 1 : 2)
    for (int i0 = 0; i0 < n4; i0 += NT) {
      const int i = i0 + tid;
      const bool valid = i < n4;
      uint32_t nib = 0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float4 v = valid ? __ldcg(reinterpret_cast<const float4*>(zu + (size_t)g * T) + i) : ninf4();
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float z = comp(v, e);
          nib |= (z > zhi[g] ? 1u : 0u) << e;
          if (z > zlo[g] && z <= zhi[g]) {
            const int s = sg[g] + atomicAdd(&s_fill[g], 1);
            mkey[s] = f2key(z);
            mpos[s] = (uint32_t)(4 * i + e);
          }
        }
      }
      uint32_t w = nib << (4 * (lane & 7));
      w |= __shfl_xor_sync(0xffffffffu, w, 1);
      w |= __shfl_xor_sync(0xffffffffu, w, 2);
      w |= __shfl_xor_sync(0xffffffffu, w, 4);
      if ((lane & 7) == 0 && valid) ubits[i >> 3] = w;
    }
  }
  __syncthreads();
#ifdef TW_TOPP_CHECK
  if (tid < G && R[tid].seg >= 0 && s_fill[tid] != (int)R[tid].members)
    printf("topp member mismatch unit %d head %d counted %u listed %d cb %d M %a zhi %a zlo %a\n", unit, tid,
           R[tid].members, s_fill[tid], R[tid].cb, R[tid].M, R[tid].zhi, R[tid].zlo);
#endif

  TT(3);
  // ---- resolve: exact threshold class inside each head's crossing bin (warp group per head)
#pragma unroll 1
  for (int g = gp; g < G; g += GB) {
    const HeadRec& h = R[g];
    const size_t qh = (size_t)unit * G + g;
    uint32_t thr, sel_cnt = 0;
    double sel_mass = 0.0;
    ResGroupSmem& S = RS[gp];
    if (h.cb == -2) {
      thr = 0xFFFFFFFFu;
    } else if (h.cb == -1) {
      thr = 0u;
      sel_cnt = h.b0;
      sel_mass = h.Z;
    } else {
      uint32_t c = 0;
      unsigned long long us = 0;
      auto pick = [&](uint32_t k, uint32_t u, uint32_t pos) {
#ifdef TW_TOPP_CHECK
        if (pos >= (uint32_t)npos)
          printf("topp bad pos unit %d head %d pos %u npos %d seg %d members %u MC %d\n", unit, g, pos, npos, h.seg,
                 h.members, MC);
#endif
        if (k >= thr) {
          ++c;
          us += u;
          atomicOr(ubits + (pos >> 5), 1u << (pos & 31));
        }
      };
      if (h.seg >= 0) {
        const SmemSrc src{mkey + h.seg, mpos + h.seg, (int)h.members, h.M, h.cb};
        thr = resolve_threshold(grp, src, h.above_mass, h.target, h.wb, S);
        src.each(grp, pick);
      } else {
        const LogitSrc src{zu + (size_t)g * T, npos, h.M, h.cb};
        thr = resolve_threshold(grp, src, h.above_mass, h.target, h.wb, S);
        src.each(grp, pick);
      }
      uint32_t ct;
      grp_scan<uint32_t>(grp, c, S.utmp, ct);
      unsigned long long ut;
      grp_scan<unsigned long long>(grp, us, S.ltmp, ut);
      sel_cnt = h.above_cnt + ct;
      sel_mass = h.above_mass + class_mass(h.wb, ct, ut);
    }
    if (grp.tid == 0) {
      float* stats = buf.head_stats + qh * 4;
      const bool empty = h.cb == -2;
      buf.head_thr[qh] = thr;
      stats[0] = (float)sel_cnt;
      stats[1] = empty ? 0.f : (float)(sel_mass / h.Z);
      stats[2] = empty || thr == 0u ? 0.f : (float)(exp((double)key2f(thr) - (double)h.M) / h.Z);
      stats[3] = (float)h.b0;
    }
    grp.sync();
  }
  __syncthreads();  // member bits (atomics of this CTA) are visible to the loads below
  TT(4);

  // ---- K3c: compact the union bitmap -> ascending token ids + attention work items.
  // Each warp owns a contiguous run of words: one pass counts, one CTA scan of
  // the warp totals, then each warp emits its run (lane l writes bit l of a
  // word: consecutive lanes -> consecutive ids, coalesced) with no further barriers.
  const int* cand = buf.cand_pages + (size_t)unit * kv.max_pages;
  int* out = buf.final_idx + (size_t)unit * T;
  const int words = (npos + 31) >> 5;
  constexpr int NW = NT / 32;
  __shared__ uint32_t s_wtot[NW];
  const int per_w = (words + NW - 1) / NW;
  const int wlo = min(words, warp * per_w), whi = min(words, wlo + per_w);
  // the first emission group's candidate pages, loaded ahead of the count and the CTA scan
  const int pa0 = 2 * wlo + lane < kv.max_pages ? __ldcg(cand + 2 * wlo + lane) : 0;
  const int pb0 = 2 * wlo + 32 + lane < kv.max_pages ? __ldcg(cand + 2 * wlo + 32 + lane) : 0;
  uint32_t cnt = 0;
  for (int w = wlo + lane; w < whi; w += 32) cnt += __popc(ld_bits(w));
  cnt = warp_sum(cnt);
  if (lane == 0) s_wtot[warp] = cnt;
  __syncthreads();
  uint32_t run = 0, basei = 0;
#pragma unroll
  for (int i = 0; i < NW; ++i) {
    run += i < warp ? s_wtot[i] : 0u;
    basei += s_wtot[i];
  }
  // claim the unit's attention work items now: the atomic's latency overlaps the emission
  const int chunk = prm.chunk_tokens > 0 ? prm.chunk_tokens : TW_DEFAULT_CHUNK;
  const int nitems = ((int)basei + chunk - 1) / chunk;
  if (tid == 0) {
    buf.final_count[unit] = (int)basei;
    s_first = nitems ? (int)atomicAdd(&buf.counters[0], (uint32_t)nitems) : 0;
  }
  for (int w0 = wlo; w0 < whi; w0 += 32) {
    const int w = w0 + lane;
    const uint32_t x = w < whi ? ld_bits(w) : 0u;
    const int pa = w0 == wlo ? pa0 : 2 * w0 + lane < kv.max_pages ? cand[2 * w0 + lane] : 0;
    const int pb = w0 == wlo ? pb0 : 2 * w0 + 32 + lane < kv.max_pages ? cand[2 * w0 + 32 + lane] : 0;
    uint32_t incl = __popc(x);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t wbase = run + incl - __popc(x);
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const uint32_t xw = __shfl_sync(0xffffffffu, x, j);
      const uint32_t bw = __shfl_sync(0xffffffffu, wbase, j);
      const int src = (2 * j + (lane >> 4)) & 31;
      const int qa = __shfl_sync(0xffffffffu, pa, src), qb = __shfl_sync(0xffffffffu, pb, src);
      if ((xw >> lane) & 1u)
        out[bw + __popc(xw & ((1u << lane) - 1u))] = (j < 16 ? qa : qb) * kPage + (lane & 15);
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  TT(5);
  __syncthreads();
  if (tid == 0) {
    buf.unit_items[2 * unit] = s_first;
    buf.unit_items[2 * unit + 1] = nitems;
  }
  for (int i = tid; i < nitems; i += NT) {
    if (s_first + i < buf.max_items) {
      buf.work_items[2 * (s_first + i)] = unit;
      buf.work_items[2 * (s_first + i) + 1] = i * chunk;
    }
  }
}

}  // namespace tw
