// Channel-pruned base selector (the paper's "DS" baseline): per unit, the
// `count` channels with the largest mean |K| over the context, then per query
// head the B0 tokens with the largest partial logit over those channels; the
// group's candidate set is the union of its heads' token sets.
//
// Reference (pkg/src/nucleuskv/selectors.py):
//   top_channels_by_magnitude :135-143  mean |K| per channel in fp64 (NumPy's
//       axis-0 mean adds the rows in token order -- reproduced exactly below),
//       stable argsort(-magnitude)[:count], returned ascending
//   select_channel_pruned :146-161      scores = (K[:, ids] @ q[ids]) / sqrt(d)
//       in fp64, stable argsort(-scores)[:B0] (ties -> lower token)
//   build_selector :203-209             count = top_channels or max(1, d // 8); the
//       slice is fixed once per context (prm.channels_fixed reuses buf.chan_ids)
//
// One CTA per unit.  Scores are computed once per token for all G heads (the
// products of fp32/bf16 inputs are exact in fp64; the 16-term sum runs in
// ascending channel order -- the reference's BLAS order is not observable, so
// tokens whose fp64 scores tie to the last bit may differ), kept as fp32 keys
// (rounding is monotone, so only the fp32 tie class of the k-th key is
// ambiguous) and that class is ranked exactly by (fp64 score desc, token asc).
// The union becomes the candidate pages plus a token mask the INT estimate
// applies (tw_decode_buffers.tok_mask).  The ordered keys of the head being
// selected live in the unit's logits rows (global memory, L2-resident: the
// estimate overwrites them afterwards), so any context length is covered;
// shared memory holds the histogram, the token bitmap and the tie band.
#include "block_scan.cuh"

namespace tw {

constexpr int kChanThreads = 512;
constexpr int kChanBand = 4096;

// byte offset of the fp64 band scores in dynamic shared memory (8-byte aligned)
__host__ __device__ inline size_t chan_band_s_offset(int T_max) {
  const size_t bytes = ((size_t)2048 + (T_max + 31) / 32 + kChanBand) * 4;
  return (bytes + 7) & ~size_t(7);
}

template <typename T>
__global__ void __launch_bounds__(kChanThreads) chan_select_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                                   tw_decode_params prm, tw_decode_buffers buf) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem[];
  const int T_max = kv.max_pages * kPage;
  const int words = (T_max + 31) / 32;
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem);          // [2048]
  uint32_t* ubits = hist + 2048;                                 // [words]
  int* band_idx = reinterpret_cast<int*>(ubits + words);         // [kChanBand]
  double* band_s = reinterpret_cast<double*>(smem + chan_band_s_offset(T_max));  // [kChanBand]
  __shared__ double mean[kHeadDim];
  __shared__ int ids[kHeadDim];
  __shared__ double qsel[8][kHeadDim];
  __shared__ uint32_t gtmp[2 * (kChanThreads / 32)];
  __shared__ uint32_t mem[64];
  __shared__ int res[4];
  __shared__ int sel_flag[kHeadDim];
  __shared__ int s_namb, s_cgt;
  const int G = kv.group_size;
  const int unit = blockIdx.x, tid = threadIdx.x;
  const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
  const int n = kv.seq_lens[b];
  const int P = (n + kPage - 1) / kPage;
  const int count = prm.top_channels > 0 ? min(prm.top_channels, kHeadDim) : kHeadDim / 8;
  const int b0 = min(n, prm.budget_tokens);
  const int* pt = kv.page_table + (size_t)b * kv.max_pages;
  const T* kc = reinterpret_cast<const T*>(kv.k_cache);
  auto key_at = [&](int t, int c) -> double {
    const size_t row = ((size_t)pt[t / kPage] * kv.num_kv_heads + h) * kPage + (t % kPage);
    return (double)Elem<T>::to_f(kc[row * kHeadDim + c]);
  };
  const Group grp = whole_block();
  if (tid < G) buf.head_max[(size_t)unit * G + tid] = 0u;  // estimate's running max starts at 0
  for (int i = tid; i < words; i += kChanThreads) ubits[i] = 0;
  int* ids_g = buf.chan_ids + (size_t)unit * kHeadDim;
  if (prm.channels_fixed) {  // the slice fixed once per context (selectors.py:203-208)
    if (tid < count) ids[tid] = ids_g[tid];
  } else {
    // ---- channel magnitudes: rows added in token order, as np.abs(K).mean(axis=0)
    if (tid < kHeadDim) {
      double acc = 0.0;
      for (int t = 0; t < n; ++t) acc += fabs(key_at(t, tid));
      mean[tid] = n > 0 ? acc / (double)n : 0.0;
    }
    __syncthreads();
    if (tid < kHeadDim) {  // stable argsort(-magnitude)[:count]: ties -> lower channel
      const double m = mean[tid];
      int rank = 0;
      for (int j = 0; j < kHeadDim; ++j) rank += (mean[j] > m) || (mean[j] == m && j < tid);
      sel_flag[tid] = rank < count;
    }
    __syncthreads();
    if (tid < kHeadDim && sel_flag[tid]) {  // the chosen channels, ascending
      int pos = 0;
      for (int j = 0; j < tid; ++j) pos += sel_flag[j];
      ids[pos] = tid;
      ids_g[pos] = tid;
    }
  }
  __syncthreads();
  for (int i = tid; i < G * count; i += kChanThreads) {
    const int g = i / count, j = i % count;
    qsel[g][j] = (double)Elem<T>::to_f(q[((size_t)unit * G + g) * kHeadDim + ids[j]]);
  }
  __syncthreads();
  // ---- fp32 keys of every head (fp64 scores rounded: monotone), staged in the logits buffer
  const size_t Ts = (size_t)T_max;
  float* zs = buf.logits + (size_t)unit * G * Ts;
  for (int t = tid; t < n; t += kChanThreads) {
    double kv16[kHeadDim / 8];  // count <= 16 on the fast path
    if (count <= kHeadDim / 8) {
      for (int j = 0; j < count; ++j) kv16[j] = key_at(t, ids[j]);
      for (int g = 0; g < G; ++g) {
        double s = 0.0;
        for (int j = 0; j < count; ++j) s += kv16[j] * qsel[g][j];
        zs[(size_t)g * Ts + t] = (float)(s / sqrt((double)kHeadDim));
      }
    } else {
      for (int g = 0; g < G; ++g) {
        double s = 0.0;
        for (int j = 0; j < count; ++j) s += key_at(t, ids[j]) * qsel[g][j];
        zs[(size_t)g * Ts + t] = (float)(s / sqrt((double)kHeadDim));
      }
    }
  }
  __syncthreads();
  // ---- per head: top-B0 tokens, ties in the fp32 class of the k-th key ranked exactly
  for (int g = 0; g < (b0 > 0 ? G : 0); ++g) {
    // the head's fp32 scores become ordered keys in place (its logits row, global memory)
    uint32_t* keys = reinterpret_cast<uint32_t*>(zs + (size_t)g * Ts);
    for (int t = tid; t < n; t += kChanThreads) keys[t] = f2key(__ldcg(zs + (size_t)g * Ts + t));
    if (tid == 0) { s_namb = 0; s_cgt = 0; }
    __syncthreads();
    const uint32_t kth = group_kth_largest_lin(grp, keys, n, (uint32_t)b0, hist, mem, gtmp, res);
    for (int t = tid; t < n; t += kChanThreads) {
      const uint32_t k = keys[t];
      if (k > kth) {
        atomicOr(&ubits[t >> 5], 1u << (t & 31));
        atomicAdd(&s_cgt, 1);
      } else if (k == kth) {
        const int s = atomicAdd(&s_namb, 1);
        if (s < kChanBand) band_idx[s] = t;
      }
    }
    __syncthreads();
    const int namb = min(s_namb, kChanBand);
    const int need = b0 - s_cgt;
    for (int a = tid; a < namb; a += kChanThreads) {
      const int t = band_idx[a];
      double s = 0.0;
      for (int j = 0; j < count; ++j) s += key_at(t, ids[j]) * qsel[g][j];
      band_s[a] = s / sqrt((double)kHeadDim);
    }
    __syncthreads();
    for (int a = tid; a < namb; a += kChanThreads) {
      const double sa = band_s[a];
      const int ia = band_idx[a];
      int rank = 0;
      for (int j = 0; j < namb; ++j) {
        const double sj = band_s[j];
        rank += (sj > sa) || (sj == sa && band_idx[j] < ia);
      }
      if (rank < need) atomicOr(&ubits[ia >> 5], 1u << (ia & 31));
    }
    __syncthreads();
  }
  // ---- token mask + candidate pages (pages holding a selected token), ascending
  uint32_t* mask = buf.tok_mask + (size_t)unit * words;
  for (int i = tid; i < words; i += kChanThreads) mask[i] = ubits[i];
  int* out = buf.cand_pages + (size_t)unit * kv.max_pages;
  uint32_t base = 0;
  for (int p0 = 0; p0 < P; p0 += kChanThreads) {
    const int p = p0 + tid;
    const uint32_t word = p < P ? ubits[p >> 1] : 0u;
    const int has = p < P && ((p & 1) ? (word >> 16) : (word & 0xFFFFu)) != 0u;
    uint32_t total;
    const uint32_t incl = block_incl_scan((uint32_t)has, gtmp, total);
    if (has) out[base + incl - 1] = p;
    base += total;
  }
  if (tid == 0) {
    buf.cand_count[unit] = (int)base;
    atomicMax(buf.counters + 6, base);  // the estimate's item range
  }
}

}  // namespace tw

using namespace tw;

inline size_t chan_smem_bytes(int max_pages) {
  return chan_band_s_offset(max_pages * kPage) + (size_t)kChanBand * 8;
}

int tw_select_channel_pruned(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                                        const tw_decode_buffers* buf, cudaStream_t stream) {
  if (!kv || !q || !prm || !buf || kv->head_dim != kHeadDim || !buf->cand_pages || !buf->cand_count ||
      !buf->logits || !buf->tok_mask || !buf->chan_ids || !buf->head_max || !buf->counters || prm->budget_tokens < 1)
    return TW_ERR_INVALID;
  if (kv->group_size > 8 || prm->top_channels < 0 || prm->top_channels > kHeadDim) return TW_ERR_INVALID;
  const size_t smem = chan_smem_bytes(kv->max_pages);
  if (smem > 200 * 1024) return TW_ERR_INVALID;  // token bitmap: contexts up to ~1.5 M tokens
  cudaMemsetAsync(buf->counters, 0, 8 * sizeof(uint32_t), stream);
  const int units = kv->num_seqs * kv->num_kv_heads;
  if (kv->dtype == TW_BF16) {
    cudaFuncSetAttribute(chan_select_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chan_select_kernel<__nv_bfloat16><<<units, kChanThreads, smem, stream>>>(*kv, (const __nv_bfloat16*)q, *prm,
                                                                             *buf);
  } else {
    cudaFuncSetAttribute(chan_select_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    chan_select_kernel<float><<<units, kChanThreads, smem, stream>>>(*kv, (const float*)q, *prm, *buf);
  }
  return launch_status();
}
