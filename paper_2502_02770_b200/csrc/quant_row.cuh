// One KV row's K1 work, shared by the append kernel (quant.cu) and the Quest
// filter that fuses the append into the decode step (quest.cu).  Semantics in
// quant.cu's header comment (quantcache.py:95-130, :163-175).
#pragma once
#include "common.cuh"

namespace tw {

struct RowQuant {
  uint32_t packed;  // 2 bytes used: this lane's 4 codes
  double scale;
  double lo;
};

// Quantize the 128-channel row held 4-per-lane across the warp to BITS-bit
// codes (levels = 2^BITS - 1), packed lowest-order field first (_pack_matrix,
// quantcache.py:122-130): 2 bytes per lane for 4-bit, 4 for 8-bit, 1 for 2-bit.
template <int BITS>
__device__ __forceinline__ RowQuant quant_row_warp(const float (&k)[4]) {
  constexpr double kLevels = (double)((1 << BITS) - 1);
  float mn = fminf(fminf(k[0], k[1]), fminf(k[2], k[3]));
  float mx = fmaxf(fmaxf(k[0], k[1]), fmaxf(k[2], k[3]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  RowQuant r;
  r.lo = (double)mn;
  const double hi = (double)mx;
  r.packed = 0;
  if (hi == r.lo) {
    r.scale = 0.0;
    return r;
  }
  r.scale = (hi - r.lo) / kLevels;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double c = rint(((double)k[i] - r.lo) / r.scale);
    c = fmin(fmax(c, 0.0), kLevels);
    r.packed |= (uint32_t)c << (BITS * i);
  }
  // nibble order inside the 2 bytes: byte0 = c0 | c1 << 4, byte1 = c2 | c3 << 4
  return r;
}

template <typename T>
__device__ __forceinline__ void load4(const T* p, float (&o)[4]);
template <>
__device__ __forceinline__ void load4<__nv_bfloat16>(const __nv_bfloat16* p, float (&o)[4]) {
  uint2 v = *reinterpret_cast<const uint2*>(p);
  o[0] = __uint_as_float(v.x << 16);
  o[1] = __uint_as_float(v.x & 0xFFFF0000u);
  o[2] = __uint_as_float(v.y << 16);
  o[3] = __uint_as_float(v.y & 0xFFFF0000u);
}
template <>
__device__ __forceinline__ void load4<float>(const float* p, float (&o)[4]) {
  float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}
template <typename T>
__device__ __forceinline__ void store4(T* p, const float (&o)[4]);
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* p, const float (&o)[4]) {
  uint2 v;
  v.x = (__float_as_uint(o[0]) >> 16) | (__float_as_uint(o[1]) & 0xFFFF0000u);
  v.y = (__float_as_uint(o[2]) >> 16) | (__float_as_uint(o[3]) & 0xFFFF0000u);
  *reinterpret_cast<uint2*>(p) = v;
}
template <>
__device__ __forceinline__ void store4<float>(float* p, const float (&o)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
}

template <int BITS>
__device__ __forceinline__ void write_quant(uint8_t* qblock, int slot, int lane, const RowQuant& r) {
  uint8_t* row = qblock + slot * (kHeadDim * BITS / 8);
  if (BITS == 4) reinterpret_cast<uint16_t*>(row)[lane] = (uint16_t)r.packed;
  else if (BITS == 8) reinterpret_cast<uint32_t*>(row)[lane] = r.packed;
  else row[lane] = (uint8_t)r.packed;
  if (lane == 0) {
    float* prm = reinterpret_cast<float*>(qblock + code_bytes_for(BITS));
    prm[slot] = (float)r.scale;
    prm[kPage + slot] = (float)r.lo;
  }
}

// Append the row at `pos` of (sequence b, kv head h): bf16/fp32 K and V into
// the paged pool, b-bit codes + params, the open page's channel min/max, and
// the |k| bound.  One warp; lane l owns channels 4l..4l+3.  A position beyond
// the page table's capacity is dropped (no out-of-bounds write).
template <typename T, int BITS>
__device__ __forceinline__ void append_row_warp(const tw_paged_kv& kv, int b, int h, int lane, const T* k_new,
                                                const T* v_new, int pos) {
  const int H = kv.num_kv_heads;
  if (pos < 0 || pos >= kv.max_pages * kPage) return;  // outside the sequence's page table: dropped
  const int logical = pos / kPage, slot = pos % kPage;
  const int phys = kv.page_table[(size_t)b * kv.max_pages + logical];
  const size_t ph = (size_t)phys * H + h;
  float k[4], v[4];
  load4<T>(k_new + ((size_t)b * H + h) * kHeadDim + 4 * lane, k);
  load4<T>(v_new + ((size_t)b * H + h) * kHeadDim + 4 * lane, v);
  T* kc = reinterpret_cast<T*>(kv.k_cache) + (ph * kPage + slot) * kHeadDim;
  T* vc = reinterpret_cast<T*>(kv.v_cache) + (ph * kPage + slot) * kHeadDim;
  store4<T>(kc + 4 * lane, k);
  store4<T>(vc + 4 * lane, v);

  RowQuant r = quant_row_warp<BITS>(k);
  write_quant<BITS>(kv.kq + ph * qblock_bytes_for(BITS), slot, lane, r);

  // page channel min/max (read-modify-write of the open page)
  T* lo = reinterpret_cast<T*>(kv.kmeta) + ph * 2 * kHeadDim + 4 * lane;
  T* hi = lo + kHeadDim;
  float nlo[4], nhi[4];
  if (slot == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) nlo[i] = nhi[i] = k[i];
  } else {
    float olo[4], ohi[4];
    load4<T>(lo, olo);
    load4<T>(hi, ohi);
#pragma unroll
    for (int i = 0; i < 4; ++i) { nlo[i] = fminf(olo[i], k[i]); nhi[i] = fmaxf(ohi[i], k[i]); }
  }
  store4<T>(lo, nlo);
  store4<T>(hi, nhi);

  float amax = fmaxf(fmaxf(fabsf(k[0]), fabsf(k[1])), fmaxf(fabsf(k[2]), fabsf(k[3])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if (lane == 0) atomicMax(reinterpret_cast<unsigned*>(kv.kabsmax) + (size_t)b * H + h, __float_as_uint(amax));
}

}  // namespace tw
