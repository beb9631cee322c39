// INT estimate helpers (u8 x s8 integer MMA, q as 22-bit fixed point in three
// signed 8-bit digits) shared by estimate_kernel (estimate.cu) and the fused
// per-unit kernel (unit.cu).  See estimate.cu for the method.
#pragma once
#include "common.cuh"

namespace tw {

__device__ __forceinline__ void mma_u8s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

constexpr int kDigits = 3;         // q as 3 signed base-256 digits of a 22-bit fixed-point value

// vector loads of 4 / 32 consecutive q elements as float
__device__ __forceinline__ void load4(const __nv_bfloat16* p, float& a, float& b, float& c, float& d) {
  const uint2 w = __ldg(reinterpret_cast<const uint2*>(p));
  a = __uint_as_float(w.x << 16); b = __uint_as_float(w.x & 0xFFFF0000u);
  c = __uint_as_float(w.y << 16); d = __uint_as_float(w.y & 0xFFFF0000u);
}
__device__ __forceinline__ void load4(const float* p, float& a, float& b, float& c, float& d) {
  const float4 w = __ldg(reinterpret_cast<const float4*>(p));
  a = w.x; b = w.y; c = w.z; d = w.w;
}
__device__ __forceinline__ void load32(const __nv_bfloat16* p, float (&v)[32]) {
  uint4 w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = __ldg(reinterpret_cast<const uint4*>(p) + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t x[4] = {w[i].x, w[i].y, w[i].z, w[i].w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[8 * i + 2 * k] = __uint_as_float(x[k] << 16);
      v[8 * i + 2 * k + 1] = __uint_as_float(x[k] & 0xFFFF0000u);
    }
  }
}
__device__ __forceinline__ void load32(const float* p, float (&v)[32]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 w = __ldg(reinterpret_cast<const float4*>(p) + i);
    v[4 * i] = w.x; v[4 * i + 1] = w.y; v[4 * i + 2] = w.z; v[4 * i + 3] = w.w;
  }
}

// q fixed point + digit B fragments for the lane's B column (head r), and for
// the lane's two accumulator columns (heads 2t, 2t+1): sum(q) and 2^-S.
// K slot -> channel map of the lane's A/B fragments (k-slot 4t+i of chunk j,
// +16 for half 1), chosen per cache width so every A register is a few
// mask/shift ops on the lane's contiguous code bytes:
//   4-bit: channel 32t + 8j + 2i + half   (low / high nibbles of word j)
//   8-bit: channel 32t + 8j + 4 half + i  (words 2j, 2j+1 as they are)
//   2-bit: channel 32t + 16 half + 4i + j (field j of each byte of word half)
template <int BITS>
__device__ __forceinline__ int slot_channel(int t, int j, int half, int i) {
  if (BITS == 8) return 32 * t + 8 * j + 4 * half + i;
  if (BITS == 2) return 32 * t + 16 * half + 4 * i + j;
  return 32 * t + 8 * j + 2 * i + half;
}

template <typename T, int G, int BITS>
__device__ __forceinline__ void estimate_prologue(const T* __restrict__ q, int unit, uint32_t (&bd)[kDigits][4][2],
                                                  float (&sq)[2], float (&inv_scale)[2]) {
  const int lane = threadIdx.x & 31, t = lane & 3, r = lane >> 2;
  float my_maxabs = 0.f;
  sq[0] = sq[1] = 0.f;
  inv_scale[0] = inv_scale[1] = 1.f;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const T* qg = q + ((size_t)unit * G + g) * kHeadDim + 4 * lane;
    float v0, v1, v2, v3;
    load4(qg, v0, v1, v2, v3);
    float s = (v0 + v1) + (v2 + v3);
    float m = fmaxf(fmaxf(fabsf(v0), fabsf(v1)), fmaxf(fabsf(v2), fabsf(v3)));
    s = warp_sum(s);
    m = warp_max(m);
    const int S = m > 0.f ? min(21 - ilogbf(m), 126) : 0;
    if (g == r) my_maxabs = (float)S;
    if (g == 2 * t) { sq[0] = s; inv_scale[0] = ldexpf(1.f, -S); }
    if (g == 2 * t + 1) { sq[1] = s; inv_scale[1] = ldexpf(1.f, -S); }
  }
  const int S = (int)my_maxabs;
  // the lane's channels 32t .. 32t+31 of head r (one contiguous 64/128-B run)
  float qv[32];
  load32(q + ((size_t)unit * G + (r < G ? r : 0)) * kHeadDim + 32 * t, qv);
  const float qscale = ldexpf(1.f, S);  // exact power of two
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t dig[kDigits] = {0u, 0u, 0u};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int x = r < G ? __float2int_rn(qv[slot_channel<BITS>(t, j, half, i) - 32 * t] * qscale) : 0;
#pragma unroll
        for (int k = 0; k < kDigits; ++k) {
          const int d = k + 1 < kDigits ? ((x + 128) & 255) - 128 : x;  // balanced digit, last takes the rest
          x = (x - d) >> 8;
          dig[k] |= ((uint32_t)d & 255u) << (8 * i);
        }
      }
#pragma unroll
      for (int k = 0; k < kDigits; ++k) bd[k][j][half] = dig[k];
    }
  }
}

// G <= 4: the digit columns are packed -- MMA 1 holds digits 0 and 1 of every
// head (B column 2g + d), MMA 2 digit 2 (column 2g; 2g + 1 is zero) -- so a page
// takes 8 integer MMAs instead of 12 and lane (t, r) ends with head t's rows
// r and r + 8.  The digit sums are combined in the same order as the unpacked
// path, so the logits are bit-identical.
template <typename T, int G, int BITS>
__device__ __forceinline__ void estimate_prologue_packed(const T* __restrict__ q, int unit, uint32_t (&b1)[4][2],
                                                         uint32_t (&b2)[4][2], float& sq, float& inv_scale) {
  const int lane = threadIdx.x & 31, t = lane & 3, r = lane >> 2;
  const int hb = r >> 1, dsel = r & 1;  // this lane's B column r: head hb, digit dsel (MMA 1) / 2 (MMA 2, even r)
  int Sb = 0;
  sq = 0.f;
  inv_scale = 1.f;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const T* qg = q + ((size_t)unit * G + g) * kHeadDim + 4 * lane;
    float v0, v1, v2, v3;
    load4(qg, v0, v1, v2, v3);
    float s = (v0 + v1) + (v2 + v3);
    float m = fmaxf(fmaxf(fabsf(v0), fabsf(v1)), fmaxf(fabsf(v2), fabsf(v3)));
    s = warp_sum(s);
    m = warp_max(m);
    const int S = m > 0.f ? min(21 - ilogbf(m), 126) : 0;
    if (g == hb) Sb = S;
    if (g == t) { sq = s; inv_scale = ldexpf(1.f, -S); }
  }
  float qv[32];
  load32(q + ((size_t)unit * G + (hb < G ? hb : 0)) * kHeadDim + 32 * t, qv);
  const float qscale = ldexpf(1.f, Sb);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t d1 = 0u, d2 = 0u;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int x = hb < G ? __float2int_rn(qv[slot_channel<BITS>(t, j, half, i) - 32 * t] * qscale) : 0;
        int dig[kDigits];
#pragma unroll
        for (int k = 0; k < kDigits; ++k) {
          dig[k] = k + 1 < kDigits ? ((x + 128) & 255) - 128 : x;
          x = (x - dig[k]) >> 8;
        }
        d1 |= ((uint32_t)(dsel ? dig[1] : dig[0]) & 255u) << (8 * i);
        d2 |= ((uint32_t)(dsel ? 0 : dig[2]) & 255u) << (8 * i);
      }
      b1[j][half] = d1;
      b2[j][half] = d2;
    }
  }
}

}  // namespace tw
