// K4 sparse / K5 dense paged decode attention.
//
// Reference: attention_weights (attention.py:89-103) + sparse_attention with
// renormalize=True (attention.py:106-136), as run per head over the group's
// shared final set at pipeline.py:366-375:  out = w[S] @ V[S] / sum(w[S]) with
// w = softmax(K q / sqrt d) -- i.e. the softmax restricted to S.  Dense decode
// (K5) is the same over every token (bypass_config, pipeline.py:129-136).
//
// Load balancing: the surviving sets of different units
// differ by orders of magnitude, so work is flattened into fixed-size
// (unit, token-chunk) items produced on device by K3c; a persistent grid walks
// the item list and a merge kernel combines split-KV partial (m, l, o) states.
// All G query heads of a KV head read each gathered K/V row once.
//
// Mapping: 4 warps per CTA, a half-warp per token row (16 lanes x 8 channels
// = one coalesced 256-B bf16 row), 8 rows per half-warp per 64-token
// sub-chunk, all K and V loads of a sub-chunk issued before any math.
#include "common.cuh"

namespace tw {

constexpr int kAttWarps = 4;
constexpr int kSub = 64;  // tokens per sub-chunk (8 half-warps x 8 rows)

template <typename T>
struct RowLoad;  // 8 channels of one row for one lane
template <>
struct RowLoad<__nv_bfloat16> {
  uint4 v;
  __device__ __forceinline__ void load(const __nv_bfloat16* p) { v = ld_stream(p); }
  __device__ __forceinline__ void get(float (&o)[8]) const { cvt8(v, (const __nv_bfloat16*)nullptr, o); }
  __device__ __forceinline__ void zero() { v = make_uint4(0, 0, 0, 0); }
};
template <>
struct RowLoad<float> {
  uint4 a, b;
  __device__ __forceinline__ void load(const float* p) { a = ld_stream(p); b = ld_stream(p + 4); }
  __device__ __forceinline__ void get(float (&o)[8]) const {
    o[0] = __uint_as_float(a.x); o[1] = __uint_as_float(a.y); o[2] = __uint_as_float(a.z); o[3] = __uint_as_float(a.w);
    o[4] = __uint_as_float(b.x); o[5] = __uint_as_float(b.y); o[6] = __uint_as_float(b.z); o[7] = __uint_as_float(b.w);
  }
  __device__ __forceinline__ void zero() { a = b = make_uint4(0, 0, 0, 0); }
};

template <int G>
struct AttnSmem {
  float s[kSub][G];             // scores of the sub-chunk
  float m_new[G], alpha[G];
  float m[G], l[G];
  float red[2 * kAttWarps][G][kHeadDim];  // cross-half-warp reduction of o
};

// Attend the query heads of `unit` over `count` tokens given by `ids`
// (or the contiguous range [t0, t0+count) when ids == nullptr).
// Leaves the un-normalised o in red[0], and m, l in smem.
template <typename T, int G>
__device__ __forceinline__ void attend(const tw_paged_kv& kv, const T* __restrict__ q, int unit,
                                       const int* __restrict__ ids, int t0, int count, AttnSmem<G>& S) {
  const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane & 15, hw = warp * 2 + (lane >> 4);  // half-warp 0..7
  const int* pt = kv.page_table + (size_t)b * kv.max_pages;
  const T* kc = reinterpret_cast<const T*>(kv.k_cache);
  const T* vc = reinterpret_cast<const T*>(kv.v_cache);
  const float inv_sqrt_d = 0.08838834764831845f;

  float qf[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    load8(q + ((size_t)unit * G + g) * kHeadDim + 8 * sub, qf[g]);
#pragma unroll
    for (int i = 0; i < 8; ++i) qf[g][i] *= inv_sqrt_d;
  }
  float o[G][8];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int i = 0; i < 8; ++i) o[g][i] = 0.f;
  if (threadIdx.x < G) { S.m[threadIdx.x] = -INFINITY; S.l[threadIdx.x] = 0.f; }

  for (int c0 = 0; c0 < count; c0 += kSub) {
    RowLoad<T> kr[8], vr[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = c0 + hw + 8 * i;
      if (j < count) {
        const int tok = ids ? ids[j] : t0 + j;
        const size_t row = (((size_t)pt[tok >> 4] * kv.num_kv_heads + h) * kPage + (tok & 15)) * kHeadDim + 8 * sub;
        kr[i].load(kc + row);
        vr[i].load(vc + row);
      } else {
        kr[i].zero();
        vr[i].zero();
      }
    }
    // scores
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float kf[8];
      kr[i].get(kf);
      float sc[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) a = fmaf(qf[g][e], kf[e], a);
        sc[g] = a;
      }
#pragma unroll
      for (int off = 8; off > 0; off >>= 1)
#pragma unroll
        for (int g = 0; g < G; ++g) sc[g] += __shfl_xor_sync(0xffffffffu, sc[g], off);
      const int j = hw + 8 * i;
      if (sub == 0) {
#pragma unroll
        for (int g = 0; g < G; ++g) S.s[j][g] = (c0 + j < count) ? sc[g] : -INFINITY;
      }
    }
    __syncthreads();
    // per-head max of the sub-chunk and rescale factor
    if (warp < G || (G > kAttWarps)) {
      for (int g = warp; g < G; g += kAttWarps) {
        float mx = fmaxf(S.s[lane][g], S.s[lane + 32][g]);
        mx = warp_max(mx);
        const float mo = S.m[g];
        const float mn = fmaxf(mo, mx);
        const float e0 = mn == -INFINITY ? 0.f : __expf(S.s[lane][g] - mn);
        const float e1 = mn == -INFINITY ? 0.f : __expf(S.s[lane + 32][g] - mn);
        const float ls = warp_sum(e0 + e1);
        __syncwarp();
        S.s[lane][g] = e0;
        S.s[lane + 32][g] = e1;
        if (lane == 0) {
          const float al = (mo == -INFINITY) ? 0.f : __expf(mo - mn);
          S.alpha[g] = al;
          S.m[g] = mn;
          S.l[g] = S.l[g] * al + ls;
        }
      }
    }
    __syncthreads();
    // o = o * alpha + sum p v
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float al = S.alpha[g];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[g][e] *= al;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float vf[8];
      vr[i].get(vf);
      const int j = hw + 8 * i;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float pj = S.s[j][g];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[g][e] = fmaf(pj, vf[e], o[g][e]);
      }
    }
    __syncthreads();
  }
  // reduce o over the 8 half-warps
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < 8; ++e) S.red[hw][g][8 * sub + e] = o[g][e];
  __syncthreads();
  for (int x = threadIdx.x; x < G * kHeadDim; x += blockDim.x) {
    const int g = x / kHeadDim, c = x % kHeadDim;
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 2 * kAttWarps; ++k) s += S.red[k][g][c];
    S.red[0][g][c] = s;
  }
  __syncthreads();
}

// write either the final normalised output or a split-KV partial
template <int G>
__device__ __forceinline__ void emit(AttnSmem<G>& S, int unit, bool single, float* out, float* partial) {
  for (int x = threadIdx.x; x < G * kHeadDim; x += blockDim.x) {
    const int g = x / kHeadDim, c = x % kHeadDim;
    const float o = S.red[0][g][c];
    if (single) {
      const float l = S.l[g];
      out[((size_t)unit * G + g) * kHeadDim + c] = l > 0.f ? o / l : 0.f;
    } else {
      partial[(size_t)g * (kHeadDim + 2) + c] = o;
      if (c == 0) {
        partial[(size_t)g * (kHeadDim + 2) + kHeadDim] = S.m[g];
        partial[(size_t)g * (kHeadDim + 2) + kHeadDim + 1] = S.l[g];
      }
    }
  }
}

// K4: persistent walk over the device-built work list
template <typename T, int G>
__global__ void __launch_bounds__(kAttWarps * 32) sparse_attn_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                                     tw_decode_params prm, tw_decode_buffers buf,
                                                                     float* __restrict__ out) {
  __shared__ AttnSmem<G> S;
  const int chunk = prm.chunk_tokens > 0 ? prm.chunk_tokens : 64;
  const int nitems = min((int)buf.counters[0], (int)buf.max_items);
  const size_t T_stride = (size_t)kv.max_pages * kPage;
  for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int unit = buf.work_items[2 * it];
    const int start = buf.work_items[2 * it + 1];
    const int cnt = min(chunk, buf.final_count[unit] - start);
    attend<T, G>(kv, q, unit, buf.final_idx + unit * T_stride + start, 0, cnt, S);
    const bool single = buf.unit_items[2 * unit + 1] == 1;
    emit<G>(S, unit, single, out, buf.partials + (size_t)it * G * (kHeadDim + 2));
    __syncthreads();
  }
  // units whose final set is empty: zeros (sparse_attention without renormalisation, attention.py:126-129)
  const int units = kv.num_seqs * kv.num_kv_heads;
  for (int u = blockIdx.x; u < units; u += gridDim.x)
    if (buf.final_count[u] == 0)
      for (int x = threadIdx.x; x < G * kHeadDim; x += blockDim.x) out[(size_t)u * G * kHeadDim + x] = 0.f;
}

// merge split-KV partials: one CTA per unit, thread per (head, channel)
template <int G>
__global__ void merge_kernel(const tw_paged_kv kv, const int32_t* __restrict__ unit_items,
                             const float* __restrict__ partials, float* __restrict__ out, int dense_chunks,
                             int dense_chunk) {
  const int unit = blockIdx.x;
  int first, n;
  if (dense_chunks > 0) {
    first = unit * dense_chunks;
    n = (kv.seq_lens[unit / kv.num_kv_heads] + dense_chunk - 1) / dense_chunk;
  } else {
    first = unit_items[2 * unit];
    n = unit_items[2 * unit + 1];
  }
  if (n <= 1 && dense_chunks == 0) return;
  for (int x = threadIdx.x; x < G * kHeadDim; x += blockDim.x) {
    const int g = x / kHeadDim, c = x % kHeadDim;
    float M = -INFINITY;
    for (int i = 0; i < n; ++i) M = fmaxf(M, partials[((size_t)(first + i) * G + g) * (kHeadDim + 2) + kHeadDim]);
    float L = 0.f, o = 0.f;
    for (int i = 0; i < n; ++i) {
      const float* pp = partials + ((size_t)(first + i) * G + g) * (kHeadDim + 2);
      const float mi = pp[kHeadDim];
      if (mi == -INFINITY) continue;
      const float sc = __expf(mi - M);
      L += pp[kHeadDim + 1] * sc;
      o += pp[c] * sc;
    }
    out[((size_t)unit * G + g) * kHeadDim + c] = L > 0.f ? o / L : 0.f;
  }
}

// K5: grid (chunks, units); every chunk writes a partial, merged afterwards
template <typename T, int G>
__global__ void __launch_bounds__(kAttWarps * 32) dense_attn_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                                    float* __restrict__ partials, int chunk) {
  __shared__ AttnSmem<G> S;
  const int unit = blockIdx.y;
  const int n = kv.seq_lens[unit / kv.num_kv_heads];
  const int t0 = blockIdx.x * chunk;
  if (t0 >= n) return;
  attend<T, G>(kv, q, unit, nullptr, t0, min(chunk, n - t0), S);
  emit<G>(S, unit, false, nullptr, partials + ((size_t)unit * gridDim.x + blockIdx.x) * G * (kHeadDim + 2));
}

}  // namespace tw

using namespace tw;

constexpr int kDenseChunk = 512;

template <typename T, int G>
static int launch_sparse(const tw_paged_kv* kv, const T* q, const tw_decode_params* prm,
                         const tw_decode_buffers* buf, float* out, cudaStream_t s) {
  const int units = kv->num_seqs * kv->num_kv_heads;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = sms * 8;
  sparse_attn_kernel<T, G><<<grid, kAttWarps * 32, 0, s>>>(*kv, q, *prm, *buf, out);
  merge_kernel<G><<<units, 256, 0, s>>>(*kv, buf->unit_items, buf->partials, out, 0, 0);
  return launch_status();
}

template <typename T, int G>
static int launch_dense(const tw_paged_kv* kv, const T* q, const tw_decode_buffers* buf, float* out,
                        cudaStream_t s) {
  const int units = kv->num_seqs * kv->num_kv_heads;
  const int chunks = (kv->max_pages * kPage + kDenseChunk - 1) / kDenseChunk;
  if ((int64_t)chunks * units > buf->max_items) return TW_ERR_INVALID;
  dense_attn_kernel<T, G><<<dim3(chunks, units), kAttWarps * 32, 0, s>>>(*kv, q, buf->partials, kDenseChunk);
  merge_kernel<G><<<units, 256, 0, s>>>(*kv, nullptr, buf->partials, out, chunks, kDenseChunk);
  return launch_status();
}

#define TW_DISPATCH_G(G_, CALL) \
  switch (G_) {                 \
    case 1: { constexpr int GG = 1; return CALL; } \
    case 2: { constexpr int GG = 2; return CALL; } \
    case 4: { constexpr int GG = 4; return CALL; } \
    case 8: { constexpr int GG = 8; return CALL; } \
    default: return TW_ERR_INVALID; \
  }

extern "C" int tw_sparse_attention(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                                   const tw_decode_buffers* buf, float* out, cudaStream_t stream) {
  if (!kv || !q || !prm || !buf || !out || kv->head_dim != kHeadDim || !buf->partials) return TW_ERR_INVALID;
  if (prm->renormalize != 1) return TW_ERR_INVALID;
  if (kv->dtype == TW_BF16) {
    TW_DISPATCH_G(kv->group_size, (launch_sparse<__nv_bfloat16, GG>(kv, (const __nv_bfloat16*)q, prm, buf, out, stream)))
  }
  TW_DISPATCH_G(kv->group_size, (launch_sparse<float, GG>(kv, (const float*)q, prm, buf, out, stream)))
}

extern "C" int tw_dense_attention(const tw_paged_kv* kv, const void* q, const tw_decode_buffers* buf, float* out,
                                  cudaStream_t stream) {
  if (!kv || !q || !buf || !out || kv->head_dim != kHeadDim || !buf->partials) return TW_ERR_INVALID;
  if (kv->dtype == TW_BF16) {
    TW_DISPATCH_G(kv->group_size, (launch_dense<__nv_bfloat16, GG>(kv, (const __nv_bfloat16*)q, buf, out, stream)))
  }
  TW_DISPATCH_G(kv->group_size, (launch_dense<float, GG>(kv, (const float*)q, buf, out, stream)))
}

extern "C" int64_t tw_max_work_items(const tw_paged_kv* kv, int32_t chunk_tokens) {
  if (!kv) return 0;
  const int64_t units = (int64_t)kv->num_seqs * kv->num_kv_heads;
  const int64_t T = (int64_t)kv->max_pages * kPage;
  const int64_t c = chunk_tokens > 0 ? chunk_tokens : 64;
  const int64_t sparse = units * ((T + c - 1) / c);
  const int64_t dense = units * ((T + kDenseChunk - 1) / kDenseChunk);
  return sparse > dense ? sparse : dense;
}
