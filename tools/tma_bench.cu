// How fast can one producer warp per CTA gather rows with cp.async.bulk (TMA)
// into a shared-memory ring?  Compared with plain LDG.128 row gathers.
// Rows are random 256-B rows (or `run` consecutive rows) of a 4 GB buffer.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)), "l"(src), "r"(n), "r"(su32(b)) : "memory");
}

constexpr int STAGE_BYTES = 16384;

// producer warp 0 issues copies of `copy` bytes (stage = STAGE_BYTES) from random offsets; warps 1.. consume
__global__ void tma_gather(const uint8_t* __restrict__ src, size_t nchunks, int copy, int nstages, int iters, int* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + nstages * STAGE_BYTES);
  uint64_t* empty = full + nstages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncons = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int per_stage = STAGE_BYTES / copy;
  if (warp == 0) {
    uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x + 1) + lane;
    for (int i = 0; i < iters; ++i) {
      const int slot = i % nstages;
      mbar_wait(&empty[slot], ((i / nstages) & 1) ^ 1);
      if (lane == 0) mbar_expect(&full[slot], STAGE_BYTES);
      __syncwarp();
      for (int c = lane; c < per_stage; c += 32) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        const size_t off = (x % nchunks) * (size_t)copy;
        bulk(sm + slot * STAGE_BYTES + c * copy, src + off, copy, &full[slot]);
      }
    }
  } else {
    int acc = 0;
    for (int i = warp - 1; i < iters; i += ncons) {
      const int slot = i % nstages;
      mbar_wait(&full[slot], (i / nstages) & 1);
      acc += sm[slot * STAGE_BYTES + lane * 4];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    if (acc == 0x7fffffff) sink[0] = acc;
  }
}

__device__ __forceinline__ int4 ldnc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
// LDG gathers: half-warp per 256-B row, `unroll` rows in flight per half-warp
template <int U>
__global__ void ldg_gather(const uint8_t* __restrict__ src, size_t nrows, int iters, int* sink) {
  const int lane = threadIdx.x & 31, sub = lane & 15;
  uint64_t x = 0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + (threadIdx.x >> 4) + 1);
  int acc = 0;
  for (int i = 0; i < iters; ++i) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      v[u] = ldnc(reinterpret_cast<const int4*>(src + (x % nrows) * 256) + sub);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x7fffffff) sink[0] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t bytes = (size_t)4 << 30;
  uint8_t* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  int* sink;
  CK(cudaMalloc(&sink, 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  printf("{\"sms\": %d", sms);
  for (int copy : {256, 1024, 4096, 16384}) {
    for (int nst : {4, 8}) {
      for (int cps : {1, 2, 4}) {
        int threads = 32 * 5;
        size_t smem = nst * STAGE_BYTES + 2 * nst * 8;
        if (smem * cps > 227 * 1024) continue;
        CK(cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int iters = 2000;
        tma_gather<<<sms * cps, threads, smem>>>(buf, bytes / copy, copy, nst, 10, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        tma_gather<<<sms * cps, threads, smem>>>(buf, bytes / copy, copy, nst, iters, sink);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf(", \"tma_copy%d_st%d_cps%d_gbs\": %.0f", copy, nst, cps, (double)sms * cps * iters * STAGE_BYTES / (ms * 1e-3) / 1e9);
      }
    }
  }
  for (int bpsm : {4, 8, 16}) {
    int iters = 200;
    ldg_gather<8><<<sms * bpsm, 128>>>(buf, bytes / 256, 2, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    ldg_gather<8><<<sms * bpsm, 128>>>(buf, bytes / 256, iters, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf(", \"ldg256_u8_b%d_gbs\": %.0f", bpsm, (double)sms * bpsm * 8 * iters * 8 * 256 / (ms * 1e-3) / 1e9);
  }
  printf("}\n");
  return 0;
}
