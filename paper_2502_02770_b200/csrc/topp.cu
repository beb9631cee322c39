// K3b/K3c: per-head softmax over the candidates, top-p threshold, group union.
//
// Reference: stable_softmax (attention.py:79-86) in fp64 over the candidate
// logits (pipeline.py:344), binary_search_top_p (pruner.py:57-114): the
// returned set is {w >= l}, and with the default epsilon/max_iters the search
// runs until that set is the MINIMAL TIE-CLOSED top set whose mass reaches
// p_eff = min(p, sum w) - 1e-9 (break rules :99-104).  We compute that set
// directly instead of bisecting (~50 passes over the weights): a mass-weighted
// radix select.  One CTA per unit (sequence, KV head) handles its G query
// heads, with everything between the two reads of the logits on chip:
//
//   pass 1   e_i = exp(z_i - max) is binned by (max - z) into 4096 bins of
//            1/120 logit per head (shared memory); a bin holds (count, sum of
//            u32 fixed-point deficits), so bin masses are exact,
//            order-independent integer sums (deterministic results).  The
//            crossing bin of each head -- the first bin, highest z first,
//            where the running mass reaches p_eff * Z -- is found by a scan
//            (one warp group per head).
//   pass 2   one read of the G heads' logits: a candidate position is kept if
//            some head keeps it outright (bin above that head's crossing bin,
//            a float compare against the bin's boundary); crossing-bin members
//            are listed per head in shared memory.
//   resolve  each head's members are ranked exactly by fp32 logit key (key
//            buckets, then an exact rank of <= 64 members; ties = equal
//            logits = equal weights); the union bitmap gets the members above
//            the threshold, and the group's final set (pipeline.py:347) is
//            compacted into ascending token ids and attention work items.
//
// The histogram pass is bound by shared-memory atomic throughput (two per
// logit); the rest is a few microseconds per unit.  The selected set is
// {z >= z_thr}: the reference's tie-closed set, up to weights within ~1e-7
// relative of the threshold (SFU exp inside a bin).
#include <algorithm>
#include <cfloat>

#include "topp_body.cuh"

namespace tw {

template <int G, int HB, bool SB>
__global__ void __launch_bounds__(UnitCfg<G, HB>::NT) topp_unit_kernel(tw_paged_kv kv, tw_decode_params prm,
                                                                      tw_decode_buffers buf) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char sm[];
  topp_unit_body<G, HB, SB>(blockIdx.x, kv, prm, buf, sm);
}

// ---------------------------------------------------------------- small batches: one CTA per query head

// When the batch has fewer (unit x head) pairs than SMs, one CTA per unit
// leaves most SMs idle: here every query head gets its own CTA (pass 1, its
// crossing, its pass 2 and resolve), the heads' kept positions are ORed into
// the unit's bitmap in global memory, and the unit's last CTA compacts the
// group union and leaves the bitmap and its counter zeroed.
constexpr int kHeadThreads = 512;
constexpr int kHeadMC = kMemberCap / 2;

template <int G>
__global__ void __launch_bounds__(kHeadThreads) topp_head_kernel(tw_paged_kv kv, tw_decode_params prm,
                                                                 tw_decode_buffers buf) {
  pdl_wait();
  pdl_trigger();
  constexpr int NT = kHeadThreads, NW = NT / 32, kPerT = kBins / NT;
  extern __shared__ __align__(16) unsigned char sm[];
  uint32_t* Hc = reinterpret_cast<uint32_t*>(sm);
  uint32_t* Hu = Hc + kBins;
  ResGroupSmem& S = *reinterpret_cast<ResGroupSmem*>(sm);  // aliases the bins once the crossing is known
  uint32_t* mkey = reinterpret_cast<uint32_t*>(sm + (size_t)kBins * 8);
  uint32_t* mpos = mkey + kHeadMC;
  __shared__ HeadRec R;
  __shared__ unsigned long long s_deep;
  __shared__ int s_fill, s_last, s_first;
  __shared__ double s_dtmp[NW];
  __shared__ uint32_t s_utmp[NW], s_wtot[NW];
  const int unit = blockIdx.x / G, g = blockIdx.x % G, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Group grp = whole_block();
  const size_t T = (size_t)kv.max_pages * kPage;
  const size_t qh = (size_t)unit * G + g;
  const int npos = buf.cand_count[unit] * kPage;
  const int n4 = npos >> 2;
  const float* z = buf.logits + qh * T;
  uint32_t* ubits = buf.sel_bits + (size_t)unit * ((T + 31) / 32);
  const double p_eff = fmin(prm.p, 1.0) - 1e-9;
  const float M = key2f(buf.head_max[qh]);
  const bool empty = p_eff <= 0.0 || npos == 0 || !(M > -INFINITY);
  if (tid == 0) {
    HeadRec r{};
    r.M = M;
    r.cb = empty ? -2 : 0;
    r.zhi = r.zlo = INFINITY;
    r.seg = -1;
    R = r;
    s_fill = 0;
    s_deep = 0;
  }
  TT(0);
  if (!empty) {
    for (int i = tid; i < kBins; i += NT) Hc[i] = Hu[i] = 0;
    __syncthreads();
    const float M120 = M * kBinPerLogit;
    unsigned long long deep = 0;
    for (int i = tid; i < n4; i += NT) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(z) + i);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float x = comp(v, e);
        if (x > -INFINITY) {
          const int b = dbin(x, M120);
          const uint32_t d = deficit(x, M, b);
          atomicAdd(&Hc[b], 1u);
          if (b < kBins - 1) atomicAdd(&Hu[b], d);
          else deep += d;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) deep += __shfl_xor_sync(0xffffffffu, deep, o);
    if (lane == 0 && deep) atomicAdd(&s_deep, deep);
    __syncthreads();
    TT(1);
    const int bfirst = tid * kPerT;
    const float t0 = bin_top(M, bfirst);
    const float w0 = (float)exp((double)t0 - (double)M);
    auto mass = [&](int i, uint32_t& c) -> double {
      const int bb = bfirst + i;
      c = Hc[bb];
      if (!c) return 0.0;
      const uint64_t us = bb == kBins - 1 ? (uint64_t)s_deep : (uint64_t)Hu[bb];
      const float d = (bin_top(M, bb) - t0) + (float)i * (1.0f / 120.0f);
      const float w = w0 * kStepExpF[i] * (1.0f + d);
      return (double)(w * ((float)c - (float)us * (float)kInvUscale));
    };
    double local = 0.0;
    uint32_t lc = 0;
#pragma unroll
    for (int i = 0; i < kPerT; ++i) {
      uint32_t c;
      local += mass(i, c);
      lc += c;
    }
    double Z;
    uint32_t b0;
    double incl;
    uint32_t cincl;
    grp_scan2(grp, local, lc, s_dtmp, s_utmp, incl, cincl, Z, b0);
    const double target = p_eff * Z;
    if (tid == 0) {  // defaults: -1 = rounding left the target above the total -> keep everything
      R.cb = -1;
      R.Z = Z;
      R.target = target;
      R.b0 = b0;
      R.zhi = R.zlo = -INFINITY;
    }
    __syncthreads();
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
          R.cb = cb;
          R.above_mass = run;
          R.above_cnt = crun;
          R.members = c;
          R.wb = exp((double)bin_top(M, cb) - (double)M);
          R.zhi = bin_ceiling(cb, M, M120);
          R.zlo = bin_ceiling(cb + 1, M, M120);
          if (c <= (uint32_t)kHeadMC) R.seg = 0;
          else R.zlo = R.zhi;  // members re-read from the logits
          break;
        }
        run += m;
        crun += c;
      }
    }
  }
  __syncthreads();
  TT(2);
  // ---- pass 2 (this head): kept positions ORed into the unit bitmap, crossing-bin members listed
  {
    const float zhi = R.zhi, zlo = R.zlo;
    for (int i0 = 0; i0 < n4; i0 += NT) {
      const int i = i0 + tid;
      const bool valid = i < n4;
      const float4 v = valid ? __ldcg(reinterpret_cast<const float4*>(z) + i) : ninf4();
      uint32_t nib = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float x = comp(v, e);
        nib |= (x > zhi ? 1u : 0u) << e;
        if (x > zlo && x <= zhi) {
          const int sl = atomicAdd(&s_fill, 1);
          mkey[sl] = f2key(x);
          mpos[sl] = (uint32_t)(4 * i + e);
        }
      }
      uint32_t w = nib << (4 * (lane & 7));
      w |= __shfl_xor_sync(0xffffffffu, w, 1);
      w |= __shfl_xor_sync(0xffffffffu, w, 2);
      w |= __shfl_xor_sync(0xffffffffu, w, 4);
      if ((lane & 7) == 0 && valid && w) atomicOr(ubits + (i >> 3), w);
    }
  }
  __syncthreads();
  TT(3);
  // ---- resolve the threshold class of this head
  {
    const HeadRec& h = R;
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
      if (h.seg >= 0) {
        const SmemSrc src{mkey, mpos, (int)h.members, h.M, h.cb};
        thr = resolve_threshold(grp, src, h.above_mass, h.target, h.wb, S);
        src.each(grp, pick);
      } else {
        const LogitSrc src{z, npos, h.M, h.cb};
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
    if (tid == 0) {
      float* stats = buf.head_stats + qh * 4;
      const bool emp = h.cb == -2;
      buf.head_thr[qh] = thr;
      stats[0] = (float)sel_cnt;
      stats[1] = emp ? 0.f : (float)(sel_mass / h.Z);
      stats[2] = emp || thr == 0u ? 0.f : (float)(exp((double)key2f(thr) - (double)h.M) / h.Z);
      stats[3] = (float)h.b0;
    }
  }
  TT(4);
  // ---- the unit's last head CTA compacts the union
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(buf.topp_done + unit, 1) == G - 1;
  __syncthreads();
  if (!s_last) return;
  TT(5);
  __threadfence();
  const int* cand = buf.cand_pages + (size_t)unit * kv.max_pages;
  int* out = buf.final_idx + (size_t)unit * T;
  const int words = (npos + 31) >> 5;
  const int per_w = (words + NW - 1) / NW;
  const int wlo = min(words, warp * per_w), whi = min(words, wlo + per_w);
  uint32_t cnt = 0;
  for (int w = wlo + lane; w < whi; w += 32) cnt += __popc(__ldcg(ubits + w));
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
    const uint32_t x = w < whi ? __ldcg(ubits + w) : 0u;
    if (w < whi) ubits[w] = 0u;  // leave the bitmap zeroed for the next step
    const int pa = 2 * w0 + lane < kv.max_pages ? cand[2 * w0 + lane] : 0;
    const int pb = 2 * w0 + 32 + lane < kv.max_pages ? cand[2 * w0 + 32 + lane] : 0;
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
  __syncthreads();
  TT(6);
  if (tid == 0) {
    buf.unit_items[2 * unit] = s_first;
    buf.unit_items[2 * unit + 1] = nitems;
    buf.topp_done[unit] = 0;
  }
  for (int i = tid; i < nitems; i += NT) {
    if (s_first + i < buf.max_items) {
      buf.work_items[2 * (s_first + i)] = unit;
      buf.work_items[2 * (s_first + i) + 1] = i * chunk;
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
extern "C" int tw_debug_ttrace(unsigned long long* host_out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, g_tt, sizeof(g_tt));
  static unsigned long long zeros[1024 * 8];
  cudaMemcpyToSymbol(g_tt, zeros, sizeof(zeros));
  return 0;
}
#endif

template <int G, int HB, bool SB>
static int launch_unit_sb(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
                          cudaStream_t stream) {
  const size_t smem = UnitCfg<G, HB>::kSmem;
  if (cudaFuncSetAttribute(topp_unit_kernel<G, HB, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return TW_ERR_CUDA;
  launch_pdl(topp_unit_kernel<G, HB, SB>, dim3(kv->num_seqs * kv->num_kv_heads), dim3(UnitCfg<G, HB>::NT), smem,
             stream, *kv, *prm, *buf);
  return launch_status();
}

template <int G, int HB>
static int launch_unit_hb(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
                          cudaStream_t stream) {
  const size_t words = ((size_t)kv->max_pages * kPage + 31) / 32;
  if (words <= UnitCfg<G, HB>::kBitsCap) return launch_unit_sb<G, HB, true>(kv, prm, buf, stream);
  return launch_unit_sb<G, HB, false>(kv, prm, buf, stream);
}

template <int G>
static int launch_unit(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
                       cudaStream_t stream) {
  // more units than SMs: the narrow CTA (two per SM) avoids a second wave of wide CTAs
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = kv->num_seqs * kv->num_kv_heads;
  static const int force_head = getenv("TW_TOPP_HEAD") ? atoi(getenv("TW_TOPP_HEAD")) : -1;  // A/B knob
  if (G >= 2 && buf->topp_done && (force_head > 0 || (force_head < 0 && units * G <= sms))) {
    // few (unit, head) pairs: one CTA per query head
    const size_t smem = (size_t)kBins * 8 + (size_t)kHeadMC * 8;
    if (cudaFuncSetAttribute(topp_head_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return TW_ERR_CUDA;
    launch_pdl(topp_head_kernel<G>, dim3(units * G), dim3(kHeadThreads), smem, stream, *kv, *prm, *buf);
    return launch_status();
  }
  if (G >= 2 && units > sms) return launch_unit_hb<G, kHB / 2>(kv, prm, buf, stream);
  return launch_unit_hb<G, kHB>(kv, prm, buf, stream);
}

extern "C" int tw_topp(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
                       cudaStream_t stream) {
  if (!kv || !prm || !buf || !buf->logits || !buf->head_max || !buf->head_thr || !buf->head_stats ||
      !buf->final_idx || !buf->final_count || !buf->unit_items || !buf->work_items || !buf->counters ||
      !buf->sel_bits)
    return TW_ERR_INVALID;
  if (!(prm->p >= 0.0 && prm->p <= 1.0)) return TW_ERR_INVALID;
  const long long T = (long long)kv->max_pages * kPage;
  if (T > (1ll << 24)) return TW_ERR_INVALID;  // member positions are 24-bit
  switch (kv->group_size) {
    case 1: return launch_unit<1>(kv, prm, buf, stream);
    case 2: return launch_unit<2>(kv, prm, buf, stream);
    case 4: return launch_unit<4>(kv, prm, buf, stream);
    case 8: return launch_unit<8>(kv, prm, buf, stream);
    default: return TW_ERR_INVALID;
  }
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
