// K2: Quest page bounds, exact page top-k per query head, GQA union.
//
// Reference (pkg/src/nucleuskv/selectors.py):
//   quest_page_scores :97-109   score_p = sum_c max(q_c lo_c, q_c hi_c) / sqrt(d)  (fp64)
//   select_quest      :112-132  k = min(ceil(n/16), ceil(B0/16)) pages, stable
//                               argsort(-score) -> ties go to the lower page
//   group_union       :178-186  sorted union over the G query heads (pipeline.py:338)
//
// Exactness without an fp64 scan of every page: the HBM-bound filter pass
// computes fp32 bounds with a rigorous error bound m (products of bf16 values
// are exact in fp32; the 128-term sum errs by at most ~128 u sum|t|, and
// sum|t| <= ||q||_1 * max|k| of the unit).  The select pass finds the k-th
// largest fp32 bound t; pages above t + 2m are certainly in, below t - 2m
// certainly out, and only the thin band between is rescored in fp64 with
// NumPy's exact summation order (8 strided partial sums, then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), see oracle.numpy_rowsum_order) and
// ranked by (score desc, page asc).  The result is the reference's page set.
#include "block_scan.cuh"

namespace tw {

constexpr int kSelThreads = 512;
constexpr int kAmbMax = 8192;   // ambiguous pages ranked in shared memory per head
__host__ __device__ inline int amb_cap(int Pmax) { return Pmax < kAmbMax ? Pmax : kAmbMax; }
constexpr int kFilterPagesPerCta = 64;

// ---------------------------------------------------------------- filter pass

// grid (ceil(max_pages/64), B*H_kv); 8 warps; 16 lanes per page, 8 channels per lane.
template <typename T, int G>
__global__ void __launch_bounds__(256) quest_filter_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                           float* __restrict__ scores) {
  const int unit = blockIdx.y;
  const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
  const int npages = (kv.seq_lens[b] + kPage - 1) / kPage;
  const int p0 = blockIdx.x * kFilterPagesPerCta;
  if (p0 >= npages) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane & 15, half = lane >> 4;
  float qr[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) load8(q + ((size_t)unit * G + g) * kHeadDim + 8 * sub, qr[g]);
  const int pend = min(p0 + kFilterPagesPerCta, npages);
  const int* pt = kv.page_table + (size_t)b * kv.max_pages;
  for (int lp = p0 + warp * 2 + half; lp < pend; lp += 16) {
    const int phys = pt[lp];
    const T* lo = reinterpret_cast<const T*>(kv.kmeta) + ((size_t)phys * kv.num_kv_heads + h) * 2 * kHeadDim + 8 * sub;
    float l8[8], h8[8];
    load8(lo, l8);
    load8(lo + kHeadDim, h8);
    float acc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) a = fmaf(qr[g][i], qr[g][i] >= 0.f ? h8[i] : l8[i], a);
      acc[g] = a;
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1)
#pragma unroll
      for (int g = 0; g < G; ++g) acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], o);
    if (sub < G) {
      float v = acc[0];
#pragma unroll
      for (int g = 1; g < G; ++g) if (sub == g) v = acc[g];
      scores[((size_t)unit * G + sub) * kv.max_pages + lp] = v;
    }
  }
}

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

// tw_quest_scores: grid (ceil(max_pages/8), B*H_kv*G), 8 warps, warp per page.
template <typename T>
__global__ void __launch_bounds__(256) quest_exact_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                          double* __restrict__ out) {
  __shared__ double terms[8][kHeadDim];
  const int qh = blockIdx.y;  // global query head = unit * G + g
  const int G = kv.group_size;
  const int unit = qh / G;
  const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
  const int npages = (kv.seq_lens[b] + kPage - 1) / kPage;
  const int warp = threadIdx.x >> 5;
  const int lp = blockIdx.x * 8 + warp;
  if (lp >= kv.max_pages) return;
  double s = -INFINITY;
  if (lp < npages) {
    const int phys = kv.page_table[(size_t)b * kv.max_pages + lp];
    const T* lo = reinterpret_cast<const T*>(kv.kmeta) + ((size_t)phys * kv.num_kv_heads + h) * 2 * kHeadDim;
    s = exact_page_score<T>(q + (size_t)qh * kHeadDim, lo, lo + kHeadDim, terms[warp]);
  }
  if ((threadIdx.x & 31) == 0) out[(size_t)qh * kv.max_pages + lp] = s;
}

// ---------------------------------------------------------------- select + union

// One CTA per unit (b, kv head); heads processed in turn.
template <typename T>
__global__ void __launch_bounds__(kSelThreads) quest_select_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                                   tw_decode_params prm, tw_decode_buffers buf) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int unit = blockIdx.x;
  const int G = kv.group_size;
  const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
  const int n = kv.seq_lens[b];
  const int P = (n + kPage - 1) / kPage;
  const int Pmax = kv.max_pages;
  const int words = (Pmax + 31) / 32;
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem);                 // [Pmax]
  uint32_t* hist = keys + Pmax;                                        // [2048]
  uint32_t* ubits = hist + 2048;                                       // [words] union bitmap
  uint32_t* hbits = ubits + words;                                     // [words] this head's bitmap
  const int cap = amb_cap(Pmax);
  int* amb_idx = reinterpret_cast<int*>(hbits + words);                // [cap]
  size_t off = ((size_t)Pmax + 2048 + 2 * words + cap) * 4;
  off = (off + 7) & ~size_t(7);
  double* amb_s = reinterpret_cast<double*>(smem + off);               // [cap]
  double* terms = amb_s + cap;                                         // [16 warps][128]
  __shared__ uint32_t tmp[40];
  __shared__ int s_namb, s_cin;
  __shared__ float s_m;

  for (int i = threadIdx.x; i < words; i += blockDim.x) ubits[i] = 0;
  const int k = min(P, prm.budget_pages);
  const int* pt = kv.page_table + (size_t)b * Pmax;
  const T* meta = reinterpret_cast<const T*>(kv.kmeta);
  __syncthreads();

  if (prm.selector == TW_SELECT_FULL || k >= P) {
    for (int i = threadIdx.x; i < P; i += blockDim.x) atomicOr(&ubits[i >> 5], 1u << (i & 31));
    if (buf.head_page_bits) {
      for (int g = 0; g < G; ++g)
        for (int i = threadIdx.x; i < words; i += blockDim.x) {
          int lo = i * 32;
          uint32_t w = lo + 32 <= P ? 0xffffffffu : (lo >= P ? 0u : ((1u << (P - lo)) - 1u));
          buf.head_page_bits[((size_t)unit * G + g) * words + i] = w;
        }
    }
  } else {
    const float amax = kv.kabsmax[unit];
    for (int g = 0; g < G; ++g) {
      const T* qh = q + ((size_t)unit * G + g) * kHeadDim;
      const float* sc = buf.page_scores + ((size_t)unit * G + g) * Pmax;
      // margin: ||q||_1 * max|k| * 300 u  (+ relative slack so fp64 divide ties are rescored)
      float qa = 0.f;
      if (threadIdx.x < 32)
        for (int c = threadIdx.x; c < kHeadDim; c += 32) qa += fabsf(Elem<T>::to_f(qh[c]));
      if (threadIdx.x < 32) {
        qa = warp_sum(qa);
        if (threadIdx.x == 0) { s_m = qa * amax * (300.0f / 16777216.0f); s_namb = 0; s_cin = 0; }
      }
      for (int i = threadIdx.x; i < words; i += blockDim.x) hbits[i] = 0;
      for (int i = threadIdx.x; i < P; i += blockDim.x) keys[i] = f2key(sc[i]);
      __syncthreads();
      const float t = key2f(block_kth_largest(keys, P, (uint32_t)k, hist, tmp));
      const float m2 = 2.f * s_m + 1e-6f * fabsf(t) + 1e-30f;
      const float hi_cut = t + m2, lo_cut = t - m2;
      // classify
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const float s = key2f(keys[i]);
        if (s > hi_cut) {
          atomicOr(&hbits[i >> 5], 1u << (i & 31));
          atomicAdd(&s_cin, 1);
        } else if (s >= lo_cut) {
          int slot = atomicAdd(&s_namb, 1);
          if (slot < cap) amb_idx[slot] = i;
          else buf.counters[7] = 1;  // band overflow: flagged, checked by the host in debug runs
        }
      }
      __syncthreads();
      const int namb = min(s_namb, cap);
      const int need = k - s_cin;
      // exact fp64 rescoring of the ambiguous band, one warp per page
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int a = warp; a < namb; a += blockDim.x / 32) {
        const int lp = amb_idx[a];
        const T* lo = meta + ((size_t)pt[lp] * kv.num_kv_heads + h) * 2 * kHeadDim;
        double s = exact_page_score<T>(qh, lo, lo + kHeadDim, terms + warp * kHeadDim);
        if (lane == 0) amb_s[a] = s;
      }
      __syncthreads();
      // rank inside the band: (score desc, page asc); keep the best `need`
      for (int a = threadIdx.x; a < namb; a += blockDim.x) {
        const double sa = amb_s[a];
        const int ia = amb_idx[a];
        int rank = 0;
        for (int j = 0; j < namb; ++j) {
          const double sj = amb_s[j];
          rank += (sj > sa) || (sj == sa && amb_idx[j] < ia);
        }
        if (rank < need) atomicOr(&hbits[ia >> 5], 1u << (ia & 31));
      }
      __syncthreads();
      for (int i = threadIdx.x; i < words; i += blockDim.x) {
        ubits[i] |= hbits[i];
        if (buf.head_page_bits) buf.head_page_bits[((size_t)unit * G + g) * words + i] = hbits[i];
      }
      __syncthreads();
    }
  }
  __syncthreads();
  // compact the union bitmap -> ascending candidate page list
  int* out = buf.cand_pages + (size_t)unit * Pmax;
  uint32_t base = 0;
  for (int w0 = 0; w0 < words; w0 += blockDim.x) {
    const int w = w0 + threadIdx.x;
    const uint32_t bits = w < words ? ubits[w] : 0u;
    uint32_t total;
    const uint32_t incl = block_incl_scan(__popc(bits), tmp, total);
    uint32_t pos = base + incl - __popc(bits);
    uint32_t x = bits;
    while (x) {
      const int bit = __ffs(x) - 1;
      x &= x - 1;
      out[pos++] = w * 32 + bit;
    }
    base += total;
  }
  if (threadIdx.x == 0) buf.cand_count[unit] = (int)base;
}

inline size_t select_smem_bytes(int Pmax) {
  const int words = (Pmax + 31) / 32;
  const int cap = amb_cap(Pmax);
  size_t bytes = ((size_t)Pmax + 2048 + 2 * words + cap) * 4;
  bytes = (bytes + 7) & ~size_t(7);
  return bytes + (size_t)cap * 8 + (kSelThreads / 32) * kHeadDim * 8;
}

}  // namespace tw

using namespace tw;

template <typename T>
static int launch_select(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                         const tw_decode_buffers* buf, cudaStream_t stream) {
  const int units = kv->num_seqs * kv->num_kv_heads;
  cudaMemsetAsync(buf->counters, 0, 8 * sizeof(uint32_t), stream);
  if (prm->selector == TW_SELECT_QUEST) {
    dim3 grid((kv->max_pages + kFilterPagesPerCta - 1) / kFilterPagesPerCta, units);
    const T* qq = (const T*)q;
    switch (kv->group_size) {
      case 1: quest_filter_kernel<T, 1><<<grid, 256, 0, stream>>>(*kv, qq, buf->page_scores); break;
      case 2: quest_filter_kernel<T, 2><<<grid, 256, 0, stream>>>(*kv, qq, buf->page_scores); break;
      case 4: quest_filter_kernel<T, 4><<<grid, 256, 0, stream>>>(*kv, qq, buf->page_scores); break;
      case 8: quest_filter_kernel<T, 8><<<grid, 256, 0, stream>>>(*kv, qq, buf->page_scores); break;
      default: return TW_ERR_INVALID;
    }
  }
  const size_t smem = select_smem_bytes(kv->max_pages);
  if (smem > 227 * 1024) return TW_ERR_INVALID;
  cudaFuncSetAttribute(quest_select_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  quest_select_kernel<T><<<units, kSelThreads, smem, stream>>>(*kv, (const T*)q, *prm, *buf);
  return launch_status();
}

extern "C" int tw_select(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                         const tw_decode_buffers* buf, cudaStream_t stream) {
  if (!kv || !prm || !buf || kv->head_dim != kHeadDim || !buf->cand_pages || !buf->cand_count || !buf->counters)
    return TW_ERR_INVALID;
  if (prm->selector != TW_SELECT_FULL && prm->selector != TW_SELECT_QUEST) return TW_ERR_INVALID;
  if (prm->selector == TW_SELECT_QUEST && (prm->budget_pages < 1 || !buf->page_scores || !q)) return TW_ERR_INVALID;
  return kv->dtype == TW_BF16 ? launch_select<__nv_bfloat16>(kv, q, prm, buf, stream)
                              : launch_select<float>(kv, q, prm, buf, stream);
}

extern "C" int tw_quest_scores(const tw_paged_kv* kv, const void* q, double* scores_out, cudaStream_t stream) {
  if (!kv || !q || !scores_out || kv->head_dim != kHeadDim) return TW_ERR_INVALID;
  dim3 grid((kv->max_pages + 7) / 8, kv->num_seqs * kv->num_kv_heads * kv->group_size);
  if (kv->dtype == TW_BF16)
    quest_exact_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(*kv, (const __nv_bfloat16*)q, scores_out);
  else
    quest_exact_kernel<float><<<grid, 256, 0, stream>>>(*kv, (const float*)q, scores_out);
  return launch_status();
}
