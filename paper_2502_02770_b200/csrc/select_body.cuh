// Quest page selection body (exact fp64 page score, per-unit top-k + GQA
// union) shared by quest_select_kernel (quest.cu) and the fused per-unit
// kernel (unit.cu).  See quest.cu for the method.
#pragma once
#include "block_scan.cuh"

#ifdef TW_TOPP_TRACE
static __device__ unsigned long long g_strace[512 * 16];
static __device__ int g_strace_phase[512];
#define STRACE()                                                                                    \
  do {                                                                                              \
    if (threadIdx.x == 0 && blockIdx.x < 512) {                                                     \
      unsigned long long now;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));                                      \
      int ph = g_strace_phase[blockIdx.x]++;                                                        \
      if (ph < 16) g_strace[blockIdx.x * 16 + ph] = now;                                            \
    }                                                                                               \
  } while (0)
#else
#define STRACE() do {} while (0)
#endif

namespace tw {

constexpr int kSelThreads = 512;

// ---------------------------------------------------------------- exact fp64 bound

// One warp computes the reference's fp64 score of one (query head, page):
// bit-identical to NumPy (products exact, NumPy's summation order, fp64 divide).
template <typename T>
__device__ __forceinline__ double exact_page_score(const T* q, const T* lo, const T* hi, double* terms) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int c = 4 * lane + i;
    const double qd = (double)Elem<T>::to_f(q[c]);
    const double a = qd * (double)Elem<T>::to_f(lo[c]);
    const double bb = qd * (double)Elem<T>::to_f(hi[c]);
    terms[c] = (a >= bb) ? a : bb;  // np.maximum: first operand on ties
  }
  __syncwarp();
  double r = 0.0;
  if (lane < 8) {
    r = terms[lane];
#pragma unroll
    for (int k = 1; k < 16; ++k) r += terms[lane + 8 * k];
  }
  double r0 = __shfl_sync(0xffffffffu, r, 0), r1 = __shfl_sync(0xffffffffu, r, 1);
  double r2 = __shfl_sync(0xffffffffu, r, 2), r3 = __shfl_sync(0xffffffffu, r, 3);
  double r4 = __shfl_sync(0xffffffffu, r, 4), r5 = __shfl_sync(0xffffffffu, r, 5);
  double r6 = __shfl_sync(0xffffffffu, r, 6), r7 = __shfl_sync(0xffffffffu, r, 7);
  __syncwarp();
  return (((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))) / sqrt((double)kHeadDim);
}

// ---------------------------------------------------------------- select + union

constexpr int kSelGroups = 4;  // default warp groups: query heads selected concurrently

struct SelGroupSmem {
  uint32_t tmp[64];  // 2 words per warp of a group (up to 32 warps)
  uint32_t mem[64];
  int res[4];
  int namb, cin;
  float margin;
};

// One CTA per unit (b, kv head); its G query heads are spread over NG warp
// groups (named barriers 1..NG), each running filter-threshold -> band
// rescoring -> rank on its own head; the CTA then compacts the union.
// One unit's selection (CTA of NT threads; `smem` = select_smem_bytes(max_pages, NT, NG)).
// n_tokens: the unit's context length (< 0: read seq_lens).
template <typename T, int NT = kSelThreads, int NG = kSelGroups>
__device__ __forceinline__ void select_unit_body(const int unit, const tw_paged_kv& kv, const T* __restrict__ q,
                                                 const tw_decode_params& prm, const tw_decode_buffers& buf,
                                                 unsigned char* smem, const int n_tokens = -1) {
  __shared__ SelGroupSmem GS[NG];
  constexpr int kGroupThreads = NT / NG;
  __shared__ uint32_t btmp[NT / 32];
  const int G = kv.group_size;
  const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
  const int n = n_tokens >= 0 ? n_tokens : kv.seq_lens[b];
  const int P = (n + kPage - 1) / kPage;
  const int Pmax = kv.max_pages;
  const int words = (Pmax + 31) / 32;
  const int gp = threadIdx.x / kGroupThreads;
  const Group grp{1 + gp, kGroupThreads, (int)threadIdx.x % kGroupThreads};
  uint32_t* ubits = reinterpret_cast<uint32_t*>(smem);                                  // [words]
  uint32_t* gbase = ubits + words + gp * (Pmax + 2048 + words);
  uint32_t* keys = gbase;                                                                // [Pmax]
  uint32_t* hist = keys + Pmax;                                                          // [2048]
  uint32_t* hbits = hist + 2048;                                                         // [words]
  size_t toff = ((size_t)words + NG * ((size_t)Pmax + 2048 + words)) * 4;
  toff = (toff + 7) & ~size_t(7);
  double* terms = reinterpret_cast<double*>(smem + toff) + (threadIdx.x >> 5) * kHeadDim;  // [NT / 32 warps][128]
  SelGroupSmem& gs = GS[gp];

  STRACE();
  if ((int)threadIdx.x < G) buf.head_max[(size_t)unit * G + threadIdx.x] = 0u;  // estimate's running max starts at 0
  for (int i = threadIdx.x; i < words; i += blockDim.x) ubits[i] = 0;
  const int k = min(P, prm.budget_pages);
  const int* pt = kv.page_table + (size_t)b * Pmax;
  const T* meta = reinterpret_cast<const T*>(kv.kmeta);
  __syncthreads();

  // sink-window (selectors.py:164-175): pages [0, sw_a) and [sw_b, P); every page when the two meet
  const bool sw = prm.selector == TW_SELECT_SINK_WINDOW;
  const int sw_a = sw ? (prm.sink + kPage - 1) / kPage : 0;
  const int sw_b = sw ? max(0, n - prm.window) / kPage : 0;
  const bool all = prm.selector == TW_SELECT_FULL || (!sw && k >= P) ||
                   (sw && (prm.sink + prm.window >= n || sw_b <= sw_a));
  if (sw && !all) {
    if (buf.head_page_bits)
      for (int g = 0; g < G; ++g)
        for (int i = threadIdx.x; i < words; i += blockDim.x) {
          uint32_t w = 0;
          for (int j = 0; j < 32; ++j) {
            const int pg = i * 32 + j;
            w |= (pg < P && (pg < sw_a || pg >= sw_b)) ? 1u << j : 0u;
          }
          buf.head_page_bits[((size_t)unit * G + g) * words + i] = w;
        }
  } else if (all) {
    if (buf.head_page_bits) {
      for (int g = 0; g < G; ++g)
        for (int i = threadIdx.x; i < words; i += blockDim.x) {
          const int lo = i * 32;
          const uint32_t w = lo + 32 <= P ? 0xffffffffu : (lo >= P ? 0u : ((1u << (P - lo)) - 1u));
          buf.head_page_bits[((size_t)unit * G + g) * words + i] = w;
        }
    }
  } else {
    const float amax = kv.kabsmax[unit];
    const int wig = grp.warp(), lane = threadIdx.x & 31;
    for (int g = gp; g < G; g += NG) {
      const size_t qhi = (size_t)unit * G + g;
      const T* qh = q + qhi * kHeadDim;
      const float* sc = buf.page_scores + qhi * Pmax;
      int* band_idx = buf.band_idx + qhi * Pmax;
      double* band_s = buf.band_scores + qhi * Pmax;
      // margin: ||q||_1 * max|k| * 300 u  (+ relative slack so fp64-divide ties are rescored);
      // its q loads are issued before, and summed after, the key loads
      float qv[kHeadDim / 32];
      if (wig == 0)
#pragma unroll
        for (int c = 0; c < kHeadDim / 32; ++c) qv[c] = fabsf(Elem<T>::to_f(qh[lane + 32 * c]));
      for (int i = grp.tid; i < words; i += grp.nthreads) hbits[i] = 0;
      if ((Pmax & 3) == 0) {  // rows 16-byte aligned: four scores per load, all in flight at once
        const int P4 = P >> 2;
#pragma unroll 4
        for (int i = grp.tid; i < P4; i += grp.nthreads) {
          const float4 v = __ldcg(reinterpret_cast<const float4*>(sc) + i);
          keys[4 * i] = f2key(v.x);
          keys[4 * i + 1] = f2key(v.y);
          keys[4 * i + 2] = f2key(v.z);
          keys[4 * i + 3] = f2key(v.w);
        }
        for (int i = 4 * P4 + grp.tid; i < P; i += grp.nthreads) keys[i] = f2key(__ldcg(sc + i));
      } else {
#pragma unroll 8
        for (int i = grp.tid; i < P; i += grp.nthreads) keys[i] = f2key(__ldcg(sc + i));
      }
      if (wig == 0) {
        float qa = 0.f;
#pragma unroll
        for (int c = 0; c < kHeadDim / 32; ++c) qa += qv[c];
        qa = warp_sum(qa);
        if (lane == 0) { gs.margin = qa * amax * (300.0f / 16777216.0f); gs.namb = 0; gs.cin = 0; }
      }
      grp.sync();
      STRACE();
      // the k-th largest fp32 bound, exactly (a bin-wide window instead made the band --
      // rescored in fp64 -- wider and the select slower: C2 K2 51 -> 55 us, C5 250 -> 282 us)
      const float tlo = key2f(group_kth_largest_lin(grp, keys, P, (uint32_t)k, hist, gs.mem, gs.tmp, gs.res));
      const float thi = tlo;
      STRACE();
      const float m2 = 2.f * gs.margin + 1e-6f * fmaxf(fabsf(tlo), fabsf(thi)) + 1e-30f;
      const float hi_cut = thi + m2, lo_cut = tlo - m2;
      // classify 32 consecutive pages per warp: in-set bits by ballot, band members appended
      // with one shared atomic per warp
      uint32_t cin = 0;
      for (int i0 = grp.tid - lane; i0 < P; i0 += grp.nthreads) {
        const int i = i0 + lane;
        const float sv = i < P ? key2f(keys[i]) : -INFINITY;
        const bool in = i < P && sv > hi_cut;
        const bool band = i < P && !in && sv >= lo_cut;
        const uint32_t bin_ = __ballot_sync(0xffffffffu, in), bband = __ballot_sync(0xffffffffu, band);
        if (lane == 0) hbits[i0 >> 5] = bin_;
        cin += __popc(bin_);
        if (bband) {
          int base = 0;
          if (lane == 0) base = atomicAdd(&gs.namb, __popc(bband));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (band) band_idx[base + __popc(bband & ((1u << lane) - 1u))] = i;
        }
      }
      if (lane == 0 && cin) atomicAdd(&gs.cin, (int)cin);
      grp.sync();
      STRACE();
      const int namb = gs.namb;
      const int need = k - gs.cin;
      if (grp.tid == 0) atomicAdd(&buf.counters[1], (uint32_t)namb);  // diagnostic: rescored pages
      // exact fp64 rescoring of the band, one warp per page
      for (int a = wig; a < namb; a += grp.nwarps()) {
        const int lp = band_idx[a];
        const T* lo = meta + ((size_t)pt[lp] * kv.num_kv_heads + h) * 2 * kHeadDim;
        const double s = exact_page_score<T>(qh, lo, lo + kHeadDim, terms);
        if (lane == 0) band_s[a] = s;
      }
      grp.sync();
      STRACE();
      // rank inside the band: (score desc, page asc); keep the best `need`
      for (int a = grp.tid; a < namb; a += grp.nthreads) {
        const double sa = band_s[a];
        const int ia = band_idx[a];
        int rank = 0;
        for (int j = 0; j < namb; ++j) {
          const double sj = band_s[j];
          rank += (sj > sa) || (sj == sa && band_idx[j] < ia);
        }
        if (rank < need) atomicOr(&hbits[ia >> 5], 1u << (ia & 31));
      }
      grp.sync();
      for (int i = grp.tid; i < words; i += grp.nthreads) {
        atomicOr(&ubits[i], hbits[i]);
        if (buf.head_page_bits) buf.head_page_bits[qhi * words + i] = hbits[i];
      }
      grp.sync();
    }
  }
  __syncthreads();
  STRACE();
  // compact the union bitmap -> ascending candidate page list
  int* out = buf.cand_pages + (size_t)unit * Pmax;
  if (all) {  // every page: no bitmap
    for (int i = threadIdx.x; i < P; i += blockDim.x) out[i] = i;
    if (threadIdx.x == 0) {
      buf.cand_count[unit] = P;
      atomicMax(buf.counters + 6, (uint32_t)P);  // the estimate's item range
    }
    return;
  }
  if (sw) {  // two page ranges
    const int nb = P - sw_b;
    for (int i = threadIdx.x; i < sw_a + nb; i += blockDim.x) out[i] = i < sw_a ? i : sw_b + (i - sw_a);
    if (threadIdx.x == 0) {
      buf.cand_count[unit] = sw_a + nb;
      atomicMax(buf.counters + 6, (uint32_t)(sw_a + nb));
    }
    return;
  }
  uint32_t base = 0;
  for (int w0 = 0; w0 < words; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    const uint32_t bits = w < words ? ubits[w] : 0u;
    uint32_t total;
    const uint32_t incl = block_incl_scan(__popc(bits), btmp, total);
    uint32_t pos = base + incl - __popc(bits);
    uint32_t x = bits;
    while (x) {
      const int bit = __ffs(x) - 1;
      x &= x - 1;
      out[pos++] = w * 32 + bit;
    }
    base += total;
  }
  if (threadIdx.x == 0) {
    buf.cand_count[unit] = (int)base;
    atomicMax(buf.counters + 6, base);
  }
  STRACE();
}

inline size_t select_smem_bytes(int Pmax, int nt = kSelThreads, int ng = kSelGroups) {
  const int words = (Pmax + 31) / 32;
  size_t bytes = ((size_t)words + ng * ((size_t)Pmax + 2048 + words)) * 4;
  bytes = (bytes + 7) & ~size_t(7);
  return bytes + (size_t)(nt / 32) * kHeadDim * 8;
}

}  // namespace tw
