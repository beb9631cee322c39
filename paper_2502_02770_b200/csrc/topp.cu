// K3b/K3c: per-head softmax over the candidates, top-p threshold, group union.
//
// Reference: stable_softmax (attention.py:79-86) in fp64 over the candidate
// logits (pipeline.py:344), binary_search_top_p (pruner.py:57-114): the
// returned set is {w >= l}, and with the default epsilon/max_iters the search
// runs until that set is the MINIMAL TIE-CLOSED top set whose mass reaches
// p_eff = min(p, sum w) - 1e-9 (break rules :99-104).  We compute that set
// directly instead of bisecting (~50 passes over the weights): a mass-weighted
// radix select, split into two grid-wide kernels so that every pass over the
// logits runs on the whole GPU (not one CTA per head):
//
//   topp_hist   grid (head, 8192-logit chunk).  e_i = exp(z_i - max) is binned
//               by (max - z) into 4096 bins of 1/120 logit; a bin holds
//               (count, sum of u32 fixed-point deficits) packed in one u64, so
//               bin masses are exact, order-independent integer sums (the
//               result is deterministic).  Chunks merge into a per-head global
//               histogram with u64 atomics; the head's last chunk CTA finds the
//               crossing bin (first bin, highest z first, where the running mass
//               reaches p_eff * Z) and writes the head record.
//   topp_union  grid (unit, slice of candidate positions).  One read of the G
//               heads' logits: a position is kept if, for some head, its bin
//               lies above that head's crossing bin; crossing-bin members go to
//               a per-unit list.  The unit's last slice CTA ranks each head's
//               members exactly by fp32 logit key (key buckets, then an exact
//               rank of <= 64 members; ties = equal logits = equal weights),
//               adds them to the union bitmap, and compacts the group's final
//               set (pipeline.py:347) into ascending token ids and attention
//               work items.
//
// The selected set is {z >= z_thr}: the reference's tie-closed set, up to
// weights within ~1e-7 relative of the threshold (SFU exp inside a bin).
#include <algorithm>
#include <cfloat>

#include <cooperative_groups.h>

#include "block_scan.cuh"

namespace cg = cooperative_groups;

namespace tw {

#ifdef TW_TOPP_TRACE
constexpr int kTrCta = 8192;
__device__ unsigned long long g_tt[3][kTrCta][8];
#define TT(k, ph)                                                                                    \
  do {                                                                                               \
    const int c_ = blockIdx.x + blockIdx.y * gridDim.x;                                              \
    if (threadIdx.x == 0 && c_ < kTrCta) {                                                           \
      unsigned long long now_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_));                                      \
      g_tt[k][c_][ph] = now_;                                                                        \
    }                                                                                                \
  } while (0)
#else
#define TT(k, ph) do {} while (0)
#endif

constexpr int kBins = TW_TOPP_BINS;      // 4096
constexpr float kBinPerLogit = 120.0f;   // bins cover (max - z) in [0, 34.1); the last bin takes the rest
constexpr int kTT = 256;                 // threads of both kernels
constexpr int kTW = kTT / 32;
constexpr int kPerT = kBins / kTT;       // 16 bins per thread in the scans
constexpr int kClusterLogits = 16384;    // candidate positions per histogram CTA (cluster size)
constexpr int kUnionLogits = 16384;      // logits (positions x G) per union CTA
constexpr int kMemberCap = TW_TOPP_MEMBER_CAP;
constexpr uint64_t kCntOne = 1ull << 43; // packed bin: count << 43 | deficit sum
constexpr uint64_t kUsMask = kCntOne - 1;
constexpr float kUscale = 4194304.0f;    // deficits in units of 2^-22
constexpr double kInvUscale = 1.0 / 4194304.0;
// exp(-i/120), i = 0..15
__constant__ double kStepExp[16] = {
    1.0, 0.991701292638876, 0.9834714538216175, 0.9753099120283326, 0.9672161004820059, 0.9591894571091382,
    0.951229424500714, 0.9433354498734922, 0.9355069850316178, 0.9277434863285529, 0.9200444146293233,
    0.9124092352730778, 0.9048374180359595, 0.8973284370942841, 0.8898817709880238, 0.8824969025845955};

// Per-head record written by topp_hist, read by topp_union.
struct TopHead {
  double above_mass;  // mass of the bins above the crossing bin
  double target;      // p_eff * Z
  double Z;           // total mass (in units of exp(z - max))
  double wb;          // weight of the crossing bin's top, exp(t_cb - max)
  int32_t cb;         // crossing bin; -1: keep every candidate; -2: keep nothing
  uint32_t above_cnt, members, b0;
  float M;            // max logit
  float zhi, zlo;     // crossing bin = (zlo, zhi] in logit space: kept outright iff z > zhi
  uint32_t pad;
};
static_assert(sizeof(TopHead) == TW_TOPP_HEAD_BYTES, "head record size");

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
// is the float interval (bin_ceiling(b + 1), bin_ceiling(b)].
__device__ float bin_ceiling(int b, float M, float M120) {
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
__device__ __forceinline__ uint32_t deficit(float z, float M, int b) {
  const float r = ex2_approx((z - bin_top(M, b)) * 1.4426950408889634f);
  return (uint32_t)__float2int_rn(fmaxf(fmaf(-r, kUscale, kUscale), 0.0f));
}
__device__ __forceinline__ double class_mass(double w, uint64_t cnt, uint64_t usum) {
  return w * ((double)cnt - (double)usum * kInvUscale);
}
__device__ __forceinline__ float4 ninf4() { return make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY); }
__device__ __forceinline__ float comp(const float4& v, int e) { return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w; }

// CTA-wide (kTT threads) inclusive scan.
template <typename T>
__device__ __forceinline__ T cta_scan(T v, T* tmp, T& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  T pre = T(0), tot = T(0);
#pragma unroll
  for (int i = 0; i < kTW; ++i) {
    const T s = tmp[i];
    pre += i < wid ? s : T(0);
    tot += s;
  }
  __syncthreads();
  total = tot;
  return x + pre;
}
template <typename T>
__device__ __forceinline__ T cta_sum(T v, T* tmp) {
  T total;
  cta_scan<T>(v, tmp, total);
  return total;
}

struct ScanSmem {
  double dtmp[kTW];
  uint32_t utmp[kTW];
  uint64_t ltmp[kTW];
  int bin;
  double above;
  uint32_t above_cnt;
};

// First entry, in priority order (thread-major, then i), whose running mass
// from `base` reaches `target`: -> S.bin (= rank, or -1), S.above, S.above_cnt.
// `entry(i, m, c)` gives the mass and count of the thread's i-th entry (it is
// evaluated twice instead of holding 16 doubles live).  Returns the total
// mass; `ctot` receives the total count.
template <class Entry>
__device__ __forceinline__ double scan_crossing(Entry&& entry, double base, double target, bool target_is_fraction,
                                                ScanSmem& S, uint32_t& ctot, double& target_out) {
  double local = 0.0;
  uint32_t lc = 0;
#pragma unroll 4
  for (int i = 0; i < kPerT; ++i) {
    double m;
    uint32_t c;
    entry(i, m, c);
    local += m;
    lc += c;
  }
  double total;
  const double incl = cta_scan<double>(local, S.dtmp, total);
  const uint32_t cincl = cta_scan<uint32_t>(lc, S.utmp, ctot);
  if (target_is_fraction) target *= total;
  target_out = target;
  if (threadIdx.x == 0) S.bin = -1;
  __syncthreads();
  const double excl = incl - local;
  if (base + excl < target && target <= base + incl) {
    double run = base + excl;
    uint32_t crun = cincl - lc;
#pragma unroll 1
    for (int i = 0; i < kPerT; ++i) {
      double m;
      uint32_t c;
      entry(i, m, c);
      if (c && run + m >= target) {
        S.bin = threadIdx.x * kPerT + i;
        S.above = run;
        S.above_cnt = crun;
        break;
      }
      run += m;
      crun += c;
    }
  }
  __syncthreads();
  return total;
}

// ---------------------------------------------------------------- K3b-1: histogram + crossing bin

// grid (cluster size cs, Hq), cluster (cs, 1, 1): CTA `rank` of a head's
// cluster bins positions [rank * chunk, (rank + 1) * chunk); the per-CTA bins
// are merged through distributed shared memory (each rank sums a 1/cs slice of
// the bins over the cluster into rank 0), and rank 0 finds the crossing bin.
__global__ void __launch_bounds__(kTT, 4) topp_hist_kernel(tw_paged_kv kv, tw_decode_params prm, tw_decode_buffers buf) {
  // per-CTA bins as two u32 arrays (native shared atomics; a u64 shared add
  // is a CAS loop on sm_100a).  A regular bin's deficits are < 2^22/120 each;
  // the deepest bin's (up to 2^22 each) go to a u64.
  __shared__ uint32_t Hc[kBins], Hu[kBins];
  __shared__ unsigned long long s_deep;
  __shared__ ScanSmem S;
  cg::cluster_group cluster = cg::this_cluster();
  const int cs = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int qh = blockIdx.y, tid = threadIdx.x;
  const int unit = qh / kv.group_size;
  const int npos = buf.cand_count[unit] * kPage;
  TopHead* rec = reinterpret_cast<TopHead*>(buf.topp_heads) + qh;
  const float M = key2f(buf.head_max[qh]);  // NaN when the head has no valid logit
  const double p_eff = fmin(prm.p, 1.0) - 1e-9;
  if (p_eff <= 0.0 || npos == 0 || !(M > -INFINITY)) {  // uniform over the cluster: nobody syncs
    if (rank == 0 && tid == 0) {
      TopHead r{};
      r.cb = -2;
      r.M = M;
      r.zhi = r.zlo = INFINITY;
      *rec = r;
    }
    return;
  }
  TT(0, 0);
  const float M120 = M * kBinPerLogit;
  for (int i = tid; i < kBins; i += kTT) Hc[i] = Hu[i] = 0;
  if (tid == 0) s_deep = 0;
  __syncthreads();
  TT(0, 1);
  {
    const size_t T = (size_t)kv.max_pages * kPage;
    const int chunk = ((npos + cs - 1) / cs + 1023) & ~1023;  // even split of the head's positions
    const int lo = rank * chunk, hi = min(npos, lo + chunk);
    const float4* z4 = reinterpret_cast<const float4*>(buf.logits + (size_t)qh * T);
    unsigned long long deep = 0;
    for (int p0 = lo; p0 < hi; p0 += 16 * kTT) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = p0 + 4 * (tid + u * kTT);
        v[u] = p < hi ? __ldcg(z4 + (p >> 2)) : ninf4();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float z = comp(v[u], e);
          if (z > -INFINITY) {
            const int b = dbin(z, M120);
            const uint32_t d = deficit(z, M, b);
            atomicAdd(&Hc[b], 1u);
            if (b < kBins - 1) atomicAdd(&Hu[b], d);
            else deep += d;
          }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) deep += __shfl_xor_sync(0xffffffffu, deep, o);
    if ((tid & 31) == 0 && deep) atomicAdd(&s_deep, deep);
  }
  TT(0, 2);
  if (cs > 1) {
    cluster.sync();
    TT(0, 3);
    // rank r sums bins [r * 4096 / cs, (r + 1) * 4096 / cs) over the cluster into rank 0
    const int per = kBins / cs;
    const uint32_t* rc[8];
    const uint32_t* ru[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      rc[r] = cluster.map_shared_rank(Hc, r < cs ? r : 0);
      ru[r] = cluster.map_shared_rank(Hu, r < cs ? r : 0);
    }
    uint32_t* c0 = cluster.map_shared_rank(Hc, 0);
    uint32_t* u0 = cluster.map_shared_rank(Hu, 0);
    for (int i = rank * per + tid; i < (rank + 1) * per; i += kTT) {
      uint32_t c[8], u[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        c[r] = r < cs ? rc[r][i] : 0u;
        u[r] = r < cs ? ru[r][i] : 0u;
      }
      uint32_t cc = 0, uu = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) { cc += c[r]; uu += u[r]; }
      c0[i] = cc;
      u0[i] = uu;
    }
    TT(0, 7);
    if (rank == cs - 1 && tid == 0) {
      unsigned long long d = 0;
      for (int r = 0; r < cs; ++r) d += *cluster.map_shared_rank(&s_deep, r);
      *cluster.map_shared_rank(&s_deep, 0) = d;
    }
    cluster.sync();
    TT(0, 4);
    if (rank != 0) return;
  }
  auto packed = [&](int i) -> uint64_t {
    return ((uint64_t)Hc[i] << 43) | (i == kBins - 1 ? (uint64_t)s_deep : (uint64_t)Hu[i]);
  };
  // masses of this thread's 16 consecutive bins: one exp, then exact small steps
  const int bfirst = tid * kPerT;
  const float t0 = bin_top(M, bfirst);
  const double w0 = exp((double)t0 - (double)M);
  auto entry = [&](int i, double& m, uint32_t& c) {
    const int bb = bfirst + i;
    c = Hc[bb];
    // exp(t_b - M) = w0 * exp(t_b - t0);  t_b - t0 = -i/120 + d (d ~ float rounding, tiny)
    const double d = ((double)bin_top(M, bb) - (double)t0) + (double)i * (1.0 / 120.0);
    const double w = w0 * kStepExp[i] * (1.0 + d * (1.0 + 0.5 * d));
    m = c ? class_mass(w, c, packed(bb) & kUsMask) : 0.0;
  };
  uint32_t b0;
  double target;
  const double Z = scan_crossing(entry, 0.0, p_eff, true, S, b0, target);
  TT(0, 6);
  if (tid == 0) {
    TopHead r{};
    r.cb = S.bin;  // -1: rounding left the target above the total -> keep everything
    r.above_mass = S.bin >= 0 ? S.above : 0.0;
    r.above_cnt = S.bin >= 0 ? S.above_cnt : 0u;
    r.members = S.bin >= 0 ? Hc[S.bin] : 0u;
    r.b0 = b0;
    r.Z = Z;
    r.target = target;
    r.wb = S.bin >= 0 ? exp((double)bin_top(M, S.bin) - (double)M) : 0.0;
    r.M = M;
    r.zhi = S.bin >= 0 ? bin_ceiling(S.bin, M, M120) : -INFINITY;
    r.zlo = S.bin >= 0 ? bin_ceiling(S.bin + 1, M, M120) : -INFINITY;
    *rec = r;
  }
  TT(0, 5);
}

// ---------------------------------------------------------------- K3b-2: union scan

// One read of the G heads' logits over a slice of candidate positions: a
// position is in the union bitmap if some head keeps it outright (bin above
// the head's crossing bin); crossing-bin members are appended to the unit's
// member list as (key << 32 | head << 24 | position).
template <int G>
__global__ void __launch_bounds__(kTT, 3) topp_union_kernel(tw_paged_kv kv, tw_decode_buffers buf) {
  constexpr int kSlice = kUnionLogits / G;  // candidate positions per CTA
  __shared__ float s_hi[G], s_lo[G];
  const int unit = blockIdx.y, slice = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const int npos = buf.cand_count[unit] * kPage;
  const int base = slice * kSlice;
  if (base >= npos) return;
  TT(1, 0);
  if (tid == 0) {
    // heads whose crossing-bin members fit the unit's list (greedy, in head order); the
    // others get an empty member range and are resolved by re-reading their logits
    const TopHead* R = reinterpret_cast<const TopHead*>(buf.topp_heads) + (size_t)unit * G;
    uint32_t acc = 0;
    for (int g = 0; g < G; ++g) {
      const bool in = R[g].cb >= 0 && acc + R[g].members <= (uint32_t)kMemberCap;
      if (in) acc += R[g].members;
      s_hi[g] = R[g].zhi;
      s_lo[g] = in ? R[g].zlo : R[g].zhi;
    }
  }
  __syncthreads();
  float zhi[G], zlo[G];
#pragma unroll
  for (int g = 0; g < G; ++g) { zhi[g] = s_hi[g]; zlo[g] = s_lo[g]; }
  const size_t T = (size_t)kv.max_pages * kPage;
  const float* zu = buf.logits + (size_t)unit * G * T;
  uint32_t* ubits = buf.sel_bits + (size_t)unit * (T / 32);
  uint64_t* mem = buf.topp_members + (size_t)unit * kMemberCap;
  uint32_t* mcount = reinterpret_cast<uint32_t*>(buf.topp_ctr) + unit;
  const int len = min(kSlice, npos - base);
  constexpr int kIters = kSlice / (4 * kTT);
  float4 v[kIters][G];
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    const int p0 = 4 * tid + it * 4 * kTT;
#pragma unroll
    for (int g = 0; g < G; ++g)
      v[it][g] = p0 < len ? __ldcg(reinterpret_cast<const float4*>(zu + g * T + base + p0)) : ninf4();
  }
  uint32_t nmem = 0;
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    const int p0 = 4 * tid + it * 4 * kTT;
    const int p = base + p0;
    uint32_t nib = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float z = comp(v[it][g], e);
        nib |= (z > zhi[g] ? 1u : 0u) << e;
        nmem += (z > zlo[g]) & (z <= zhi[g]);
      }
    }
    uint32_t w = nib << (4 * (lane & 7));
    w |= __shfl_xor_sync(0xffffffffu, w, 1);
    w |= __shfl_xor_sync(0xffffffffu, w, 2);
    w |= __shfl_xor_sync(0xffffffffu, w, 4);
    if ((lane & 7) == 0 && p0 < len) ubits[p >> 5] = w;
  }
  TT(1, 1);
  // crossing-bin members: one list reservation per CTA
  __shared__ uint32_t s_tmp[kTT / 32];
  __shared__ uint32_t s_base;
  uint32_t total;
  const uint32_t incl = cta_scan<uint32_t>(nmem, s_tmp, total);
  if (total) {
    if (tid == 0) s_base = atomicAdd(mcount, total);
    __syncthreads();
    TT(1, 2);
    uint32_t slot = s_base + incl - nmem;
    if (nmem) {
#pragma unroll
      for (int it = 0; it < kIters; ++it) {
        const int p = base + 4 * tid + it * 4 * kTT;
#pragma unroll
        for (int g = 0; g < G; ++g) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float z = comp(v[it][g], e);
            if (z > zlo[g] && z <= zhi[g]) {
              if (slot < (uint32_t)kMemberCap)
                mem[slot] = ((uint64_t)f2key(z) << 32) | ((uint64_t)g << 24) | (uint64_t)(p + e);
              ++slot;
            }
          }
        }
      }
    }
  }
  TT(1, 3);
}

// ---------------------------------------------------------------- K3b-3 / K3c: exact thresholds + group union

constexpr int kResThreads = 512;
constexpr int kResBuckets = 1024;  // key buckets per level
constexpr int kRankCap = 64;       // members ranked exactly (O(k^2))

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
  double dtmp[16];
  uint32_t utmp[16];
  unsigned long long ltmp[16];
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

// One CTA per unit; its G heads are resolved concurrently by G warp groups
// (named barriers), then the CTA compacts the group's final set.
template <int G>
__global__ void __launch_bounds__(kResThreads) topp_resolve_kernel(tw_paged_kv kv, tw_decode_params prm,
                                                                    tw_decode_buffers buf) {
  extern __shared__ __align__(16) unsigned char rsm[];
  ResGroupSmem* GS = reinterpret_cast<ResGroupSmem*>(rsm);                 // [G]
  uint32_t* keys = reinterpret_cast<uint32_t*>(rsm + G * sizeof(ResGroupSmem));  // [kMemberCap]
  uint32_t* posn = keys + kMemberCap;                                        // [kMemberCap]
  __shared__ TopHead R[G];
  __shared__ int seg[G + 1], fill[G];
  __shared__ uint32_t btmp[kResThreads / 32];
  __shared__ int s_first;
  const int unit = blockIdx.x, tid = threadIdx.x;
  const size_t T = (size_t)kv.max_pages * kPage;
  const int npos = buf.cand_count[unit] * kPage;
  uint32_t* ubits = buf.sel_bits + (size_t)unit * (T / 32);
  const uint64_t* mem = buf.topp_members + (size_t)unit * kMemberCap;
  uint32_t* mcount = reinterpret_cast<uint32_t*>(buf.topp_ctr) + unit;
  TT(2, 0);
  if (tid < G) R[tid] = reinterpret_cast<const TopHead*>(buf.topp_heads)[(size_t)unit * G + tid];
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 0;
    seg[0] = 0;
    for (int g = 0; g < G; ++g) {
      const bool in = R[g].cb >= 0 && acc + R[g].members <= (uint32_t)kMemberCap;
      if (in) acc += R[g].members;
      seg[g + 1] = acc;
      fill[g] = 0;
    }
  }
  __syncthreads();
  // distribute the member list into per-head segments
  const int m = (int)min(*mcount, (uint32_t)kMemberCap);
  for (int i = tid; i < m; i += kResThreads) {
    const uint64_t r = mem[i];
    const int g = (int)(((uint32_t)r >> 24) & 0xFFu);
    const int s = seg[g] + atomicAdd(&fill[g], 1);
    keys[s] = (uint32_t)(r >> 32);
    posn[s] = (uint32_t)r & 0xFFFFFFu;
  }
  __syncthreads();
  TT(2, 1);
  {
    constexpr int kGT = kResThreads / G;
    const int g = tid / kGT;
    const Group grp{1 + g, kGT, tid % kGT};
    ResGroupSmem& S = GS[g];
    const TopHead& h = R[g];
    const size_t qh = (size_t)unit * G + g;
    uint32_t thr, sel_cnt = 0;
    double sel_mass = 0.0;
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
        if (k >= thr) {
          ++c;
          us += u;
          atomicOr(ubits + (pos >> 5), 1u << (pos & 31));
        }
      };
      if (seg[g + 1] - seg[g] == (int)h.members && h.members > 0) {
        const SmemSrc src{keys + seg[g], posn + seg[g], (int)h.members, h.M, h.cb};
        thr = resolve_threshold(grp, src, h.above_mass, h.target, h.wb, S);
        src.each(grp, pick);
      } else {
        const LogitSrc src{buf.logits + qh * T, npos, h.M, h.cb};
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
  }
  __syncthreads();  // member bits (global atomics of this CTA) are visible to its ld.cg below
  TT(2, 2);
  // ---- K3c: compact the union bitmap -> ascending token ids + attention work items
  const int* cand = buf.cand_pages + (size_t)unit * kv.max_pages;
  int* out = buf.final_idx + (size_t)unit * T;
  const int words = (npos + 31) >> 5;
  uint32_t basei = 0;
  const int lane = tid & 31, warp = tid >> 5;
  // the warp owns words w0 + 32 warp + j (j = lane) and their 64 candidate pages;
  // the next block's words and pages are prefetched while this one is written
  auto fetch = [&](int w0, uint32_t& x, int& pa, int& pb) {
    const int w = w0 + tid;
    x = w < words ? __ldcg(ubits + w) : 0u;
    const int p0 = 2 * (w0 + 32 * warp);
    pa = p0 + lane < kv.max_pages ? cand[p0 + lane] : 0;
    pb = p0 + 32 + lane < kv.max_pages ? cand[p0 + 32 + lane] : 0;
  };
  uint32_t xn;
  int pan, pbn;
  fetch(0, xn, pan, pbn);
  for (int w0 = 0; w0 < words; w0 += kResThreads) {
    const uint32_t x = xn;
    const int pa = pan, pb = pbn;
    if (w0 + kResThreads < words) fetch(w0 + kResThreads, xn, pan, pbn);
    uint32_t total;
    const uint32_t incl = block_incl_scan(__popc(x), btmp, total);
    const uint32_t wbase = basei + incl - __popc(x);
    // lane l writes bit l of each word: consecutive lanes -> consecutive ids (coalesced)
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const uint32_t xw = __shfl_sync(0xffffffffu, x, j);
      const uint32_t bw = __shfl_sync(0xffffffffu, wbase, j);
      const int src = (2 * j + (lane >> 4)) & 31;
      const int qa = __shfl_sync(0xffffffffu, pa, src), qb = __shfl_sync(0xffffffffu, pb, src);
      if ((xw >> lane) & 1u)
        out[bw + __popc(xw & ((1u << lane) - 1u))] = (j < 16 ? qa : qb) * kPage + (lane & 15);
    }
    basei += total;
  }
  TT(2, 3);
  const int chunk = prm.chunk_tokens > 0 ? prm.chunk_tokens : TW_DEFAULT_CHUNK;
  const int nitems = ((int)basei + chunk - 1) / chunk;
  if (tid == 0) {
    buf.final_count[unit] = (int)basei;
    s_first = nitems ? (int)atomicAdd(&buf.counters[0], (uint32_t)nitems) : 0;
    buf.unit_items[2 * unit] = s_first;
    buf.unit_items[2 * unit + 1] = nitems;
    *mcount = 0;
  }
  __syncthreads();
  for (int i = tid; i < nitems; i += kResThreads) {
    if (s_first + i < buf.max_items) {
      buf.work_items[2 * (s_first + i)] = unit;
      buf.work_items[2 * (s_first + i) + 1] = i * chunk;
    }
  }
  TT(2, 4);
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
extern "C" int tw_debug_ttrace(unsigned long long* host_out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, g_tt, sizeof(g_tt));
  cudaMemset(host_out, 0, 0);
  static unsigned long long zeros[3 * kTrCta * 8];
  cudaMemcpyToSymbol(g_tt, zeros, sizeof(zeros));
  return 0;
}
#endif

template <int G>
static void launch_union(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
                         cudaStream_t stream) {
  constexpr int kSlice = kUnionLogits / G;
  const int T = kv->max_pages * kPage;
  const int units = kv->num_seqs * kv->num_kv_heads;
  topp_union_kernel<G><<<dim3((T + kSlice - 1) / kSlice, units), kTT, 0, stream>>>(*kv, *buf);
  const int smem = G * (int)sizeof(ResGroupSmem) + 2 * kMemberCap * 4;
  cudaFuncSetAttribute(topp_resolve_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  topp_resolve_kernel<G><<<units, kResThreads, smem, stream>>>(*kv, *prm, *buf);
}

extern "C" int tw_topp(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
                       cudaStream_t stream) {
  if (!kv || !prm || !buf || !buf->logits || !buf->head_max || !buf->head_thr || !buf->head_stats ||
      !buf->final_idx || !buf->final_count || !buf->unit_items || !buf->work_items || !buf->counters ||
      !buf->sel_bits || !buf->topp_heads || !buf->topp_members ||
      !buf->topp_ctr)
    return TW_ERR_INVALID;
  if (!(prm->p >= 0.0 && prm->p <= 1.0)) return TW_ERR_INVALID;
  const long long T = (long long)kv->max_pages * kPage;
  if (T > (1ll << 21)) return TW_ERR_INVALID;  // packed bin counts / member positions
  const int units = kv->num_seqs * kv->num_kv_heads;
  const int Hq = units * kv->group_size;
  // histogram cluster: <= 8 CTAs (portable) of >= 8192 positions each
  const int cs = (int)std::min<long long>(8, std::max<long long>(1, (T + kClusterLogits - 1) / kClusterLogits));
  {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, Hq);
    cfg.blockDim = dim3(kTT);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    tw_decode_params p = *prm;
    tw_decode_buffers b = *buf;
    tw_paged_kv k = *kv;
    if (cudaLaunchKernelEx(&cfg, topp_hist_kernel, k, p, b) != cudaSuccess) return TW_ERR_CUDA;
  }
  switch (kv->group_size) {
    case 1: launch_union<1>(kv, prm, buf, stream); break;
    case 2: launch_union<2>(kv, prm, buf, stream); break;
    case 4: launch_union<4>(kv, prm, buf, stream); break;
    case 8: launch_union<8>(kv, prm, buf, stream); break;
    default: return TW_ERR_INVALID;
  }
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
