// K1: INT4 key quantization on KV append, bulk cache build, row quantizer.
//
// Reference semantics (pkg/src/nucleuskv/quantcache.py):
//   quantize_row :95-114 / build_cache :199-207 -- lo = min, hi = max of the
//   row; hi == lo -> scale 0, codes 0, zero lo; else scale = (hi - lo) / 15 and
//   code = clip(rint((k - lo) / scale), 0, 15), all in IEEE fp64 with
//   half-even rounding.  We use the same fp64 ops (DADD, correctly rounded
//   DDIV, rint), so codes are bit-identical; a reciprocal multiply or fp32
//   would not be.
//   _pack_matrix :122-130 -- even channel in the low nibble.
//   build_page_metadata :163-175 -- per-channel min/max of the page's real rows.
//
// Mapping: one warp per (token row, kv head); lane l owns channels 4l..4l+3,
// so the 256-B bf16 row is read as one coalesced 8-B-per-lane access and the
// 64-B packed row is written as one 2-B-per-lane store.
#include "quant_row.cuh"

namespace tw {

template <typename T, int BITS>
__global__ void __launch_bounds__(1024) append_kernel(tw_paged_kv kv, const T* __restrict__ k_new,
                                                      const T* __restrict__ v_new,
                                                      const int32_t* positions) {
  const int b = blockIdx.x;
  const int h = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int pos = positions[b];
  append_row_warp<T, BITS>(kv, b, h, lane, k_new, v_new, pos);
  __syncthreads();
  if (threadIdx.x == 0 && pos >= 0 && pos < kv.max_pages * kPage) kv.seq_lens[b] = pos + 1;
}

// Bulk build: block (logical page, sequence), one warp per kv head walking the
// page's valid rows; also (re)computes the page metadata and the |k| bound.
template <typename T, int BITS>
__global__ void __launch_bounds__(1024) build_kernel(tw_paged_kv kv) {
  const int lp = blockIdx.x, b = blockIdx.y;
  const int len = kv.seq_lens[b];
  if (lp * kPage >= len) return;
  const int h = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int H = kv.num_kv_heads;
  const int phys = kv.page_table[(size_t)b * kv.max_pages + lp];
  const size_t ph = (size_t)phys * H + h;
  const int valid = min(kPage, len - lp * kPage);
  const T* kc = reinterpret_cast<const T*>(kv.k_cache) + ph * kPage * kHeadDim;
  uint8_t* qb = kv.kq + ph * qblock_bytes_for(BITS);
  float mn[4], mx[4], amax = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) { mn[i] = INFINITY; mx[i] = -INFINITY; }
  for (int s = 0; s < valid; ++s) {
    float k[4];
    load4<T>(kc + s * kHeadDim + 4 * lane, k);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mn[i] = fminf(mn[i], k[i]);
      mx[i] = fmaxf(mx[i], k[i]);
      amax = fmaxf(amax, fabsf(k[i]));
    }
    RowQuant r = quant_row_warp<BITS>(k);
    write_quant<BITS>(qb, s, lane, r);
  }
  T* lo = reinterpret_cast<T*>(kv.kmeta) + ph * 2 * kHeadDim + 4 * lane;
  store4<T>(lo, mn);
  store4<T>(lo + kHeadDim, mx);
  amax = warp_max(amax);
  if (lane == 0) atomicMax(reinterpret_cast<unsigned*>(kv.kabsmax) + (size_t)b * H + h, __float_as_uint(amax));
}

// Generic row quantizer for the per-row API (any d, bits in {2,4,8}).
template <typename T>
__global__ void quant_rows_kernel(const T* __restrict__ rows, int n, int d, int levels,
                                  uint8_t* __restrict__ codes, double* scale_out, double* zero_out) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const T* r = rows + (size_t)row * d;
  float mn = INFINITY, mx = -INFINITY;
  for (int c = lane; c < d; c += 32) {
    float x = Elem<T>::to_f(r[c]);
    mn = fminf(mn, x);
    mx = fmaxf(mx, x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const double lo = mn, hi = mx;
  const double scale = (hi == lo) ? 0.0 : (hi - lo) / (double)levels;
  for (int c = lane; c < d; c += 32) {
    uint8_t code = 0;
    if (scale > 0.0) {
      double q = rint(((double)Elem<T>::to_f(r[c]) - lo) / scale);
      code = (uint8_t)fmin(fmax(q, 0.0), (double)levels);
    }
    codes[(size_t)row * d + c] = code;
  }
  if (lane == 0) {
    scale_out[row] = scale;
    zero_out[row] = lo;
  }
}

}  // namespace tw

using namespace tw;

static int check_geometry(const tw_paged_kv* kv) {
  if (!kv || kv->head_dim != kHeadDim || kv->num_kv_heads < 1 || kv->num_kv_heads > 32 ||
      kv->num_seqs < 1 || kv->max_pages < 1 || kv->group_size < 1 || kv->group_size > 8 ||
      (kv->dtype != TW_F32 && kv->dtype != TW_BF16) || (kv->bits != 0 && kv->bits != 2 && kv->bits != 4 &&
                                                          kv->bits != 8))
    return TW_ERR_INVALID;
  return TW_OK;
}

#define TW_DISPATCH_BITS(bits_, CALL)                 \
  switch (bits_) {                                    \
    case 2: { constexpr int BB = 2; CALL; break; }    \
    case 8: { constexpr int BB = 8; CALL; break; }    \
    default: { constexpr int BB = 4; CALL; break; }   \
  }

extern "C" int tw_quant_append(const tw_paged_kv* kv, const void* k_new, const void* v_new,
                               const int32_t* positions, cudaStream_t stream) {
  if (int s = check_geometry(kv)) return s;
  if (!k_new || !v_new || !positions) return TW_ERR_INVALID;
  dim3 grid(kv->num_seqs), block(32 * kv->num_kv_heads);
  if (kv->dtype == TW_BF16) {
    TW_DISPATCH_BITS(cache_bits(*kv), (append_kernel<__nv_bfloat16, BB><<<grid, block, 0, stream>>>(
                                           *kv, (const __nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new, positions)))
  } else {
    TW_DISPATCH_BITS(cache_bits(*kv), (append_kernel<float, BB><<<grid, block, 0, stream>>>(
                                           *kv, (const float*)k_new, (const float*)v_new, positions)))
  }
  return launch_status();
}

extern "C" int tw_quant_build(const tw_paged_kv* kv, cudaStream_t stream) {
  if (int s = check_geometry(kv)) return s;
  dim3 grid(kv->max_pages, kv->num_seqs), block(32 * kv->num_kv_heads);
  if (kv->dtype == TW_BF16) {
    TW_DISPATCH_BITS(cache_bits(*kv), (build_kernel<__nv_bfloat16, BB><<<grid, block, 0, stream>>>(*kv)))
  } else {
    TW_DISPATCH_BITS(cache_bits(*kv), (build_kernel<float, BB><<<grid, block, 0, stream>>>(*kv)))
  }
  return launch_status();
}

extern "C" int tw_quant_rows(const void* rows, int32_t n, int32_t d, int32_t dtype, int32_t bits,
                             uint8_t* codes_out, double* scale_out, double* zero_out, cudaStream_t stream) {
  if (n < 1 || d < 1 || (bits != 2 && bits != 4 && bits != 8)) return TW_ERR_INVALID;
  const int warps = 8;
  dim3 grid((n + warps - 1) / warps), block(32 * warps);
  const int levels = (1 << bits) - 1;
  if (dtype == TW_BF16)
    quant_rows_kernel<__nv_bfloat16><<<grid, block, 0, stream>>>((const __nv_bfloat16*)rows, n, d, levels, codes_out,
                                                                 scale_out, zero_out);
  else if (dtype == TW_F32)
    quant_rows_kernel<float><<<grid, block, 0, stream>>>((const float*)rows, n, d, levels, codes_out, scale_out,
                                                         zero_out);
  else
    return TW_ERR_INVALID;
  return launch_status();
}
