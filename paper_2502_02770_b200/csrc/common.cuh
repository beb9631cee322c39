// Shared device helpers for the Twilight sm_100a kernels.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <utility>

#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/twilight.h"

namespace tw {

constexpr int kPage = 16;          // tokens per page (SelectorConfig.page_size, selectors.py:39)
constexpr int kHeadDim = 128;      // d: Llama-3.1-8B / LongChat-7B head dim
constexpr int kCodeBytes = kPage * kHeadDim / 2;      // 1024 B of packed nibbles per (page, kv head)
constexpr int kQBlockBytes = kCodeBytes + kPage * 8;  // + fp32 scale[16] + fp32 zero[16] = 1152 B
// b-bit caches (quantcache.py:38, SUPPORTED_BITS = 2, 4, 8): the page's codes in the
// reference's byte layout (lowest-order field first), then the 128 B of parameters
__host__ __device__ constexpr int code_bytes_for(int bits) { return kPage * kHeadDim * bits / 8; }
__host__ __device__ constexpr int qblock_bytes_for(int bits) { return code_bytes_for(bits) + kPage * 8; }
__host__ __device__ inline int cache_bits(const tw_paged_kv& kv) { return kv.bits ? kv.bits : 4; }
constexpr int kWarp = 32;

// ---------------------------------------------------------------- element types

template <typename T> struct Elem;
template <> struct Elem<float> {
  static constexpr int kId = TW_F32;
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <> struct Elem<__nv_bfloat16> {
  static constexpr int kId = TW_BF16;
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

// 8 consecutive elements (16 B for bf16, 32 B for fp32) -> 8 floats
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&o)[8]) {
  uint4 v = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[2 * i] = __uint_as_float(w[i] << 16);
    o[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}
__device__ __forceinline__ void load8(const float* p, float (&o)[8]) {
  float4 a = *reinterpret_cast<const float4*>(p);
  float4 b = *reinterpret_cast<const float4*>(p + 4);
  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; o[4] = b.x; o[5] = b.y; o[6] = b.z; o[7] = b.w;
}

// streaming (read-once) 16-byte load that does not allocate in L1
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ void cvt8(const uint4& v, const __nv_bfloat16*, float (&o)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    o[2 * i] = __uint_as_float(w[i] << 16);
    o[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

// ---------------------------------------------------------------- ordering keys

// Monotone map fp32 -> u32: a < b  <=>  key(a) < key(b) (for non-NaN).
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(b);
}

// ---------------------------------------------------------------- warp helpers

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// exp(z - m) for z <= m, accurate to a few fp32 ulp even when z - m is large:
// the difference is formed exactly (two-sum) and the reduction uses a
// Cody-Waite split of ln 2, so the only error is the degree-7 polynomial.
__device__ __forceinline__ float exp_diff(float z, float m) {
  float s = z - m;
  float bb = s - z;
  float err = (z - (s - bb)) + (-m - bb);
  if (s < -103.0f) return 0.0f;
  float k = rintf(s * 1.4426950408889634f);
  float r = fmaf(-k, 0.693145751953125f, s);
  r = fmaf(-k, 1.428606765330187e-06f, r);
  r += err;
  float p = 1.9841270e-4f;                 // 1/5040
  p = fmaf(p, r, 1.3888889e-3f);           // 1/720
  p = fmaf(p, r, 8.3333333e-3f);           // 1/120
  p = fmaf(p, r, 4.1666667e-2f);           // 1/24
  p = fmaf(p, r, 1.6666667e-1f);           // 1/6
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  int ki = (int)k;
  if (ki < -125) return ldexpf(p, ki);     // gradual underflow
  return p * __int_as_float((ki + 127) << 23);
}

// ---------------------------------------------------------------- launch check

// Internal (not a tw_status): the fused K1+K2 launch does not apply, nothing
// was enqueued, and the caller runs the separate append + select.
constexpr int TW_FUSE_UNAVAILABLE = -1;

inline int launch_status() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && getenv("TW_DEBUG")) fprintf(stderr, "twilight: CUDA error %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? TW_OK : TW_ERR_CUDA;
}

}  // namespace tw

// ---------------------------------------------------------------- TMA bulk copy + mbarrier (sm_90+/sm_100a)
namespace tw {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (TMA, non-tensor), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Ampere-style async 16-byte global -> shared copies (LDGSTS)
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Dynamic work distribution for persistent warp workers: lane 0 takes the
// next item index from a global counter and broadcasts it (items are then
// balanced even when CTAs start late, e.g. next to another stream's kernel).
__device__ __forceinline__ int warp_fetch(uint32_t* ctr) {
  int it = 0;
  if ((threadIdx.x & 31) == 0) it = (int)atomicAdd(ctr, 1u);
  return __shfl_sync(0xffffffffu, it, 0);
}


__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Programmatic dependent launch (PDL): kernels of the decode step are launched
// with programmatic stream serialization, so a kernel's CTAs can be scheduled
// while its predecessor drains; each waits (griddepcontrol.wait) before
// touching the predecessor's outputs.  TW_PDL=0 turns it off (A/B knob).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("TW_PDL");
    on = e ? atoi(e) != 0 : 1;  // r02: C1 61.4 -> 58.6 us, C2 e2e 319.6 -> 312.3 us, C2 step unchanged
  }
  return on != 0;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Experiment knob: cap the resident CTAs per SM of the persistent kernels
// (TW_PERSIST_CTAS=n; unset = as many as fit).
inline int persist_cap(int per_sm) {
  static int cap = -1;
  if (cap < 0) {
    const char* e = getenv("TW_PERSIST_CTAS");
    cap = e ? atoi(e) : 0;
  }
  if (per_sm < 1) per_sm = 1;
  return cap > 0 && cap < per_sm ? cap : per_sm;
}

}  // namespace tw
