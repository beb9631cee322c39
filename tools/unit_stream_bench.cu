// Microbenchmark: one CTA (or W warps of it) streams one unit's scattered
// page blocks (BS bytes each, page-table order) -- the access pattern of a
// CTA-per-unit Quest filter (512-B metadata blocks) or INT4 estimate (1152-B
// blocks).  Measures aggregate GB/s for a grid of `units` CTAs, LDGSTS per-warp
// rings vs TMA bulk copies.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/unit_stream_bench tools/unit_stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// LDGSTS: warp w streams tiles w, w+W, ...; each tile = TP pages; STAGES-deep ring, continuous across tiles
template <int W, int STAGES, int TP, int BS>
__global__ void __launch_bounds__(W * 32) k_ldgsts(const uint8_t* __restrict__ pool, const int* __restrict__ pt, int np,
                                                   float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* R = sm + (size_t)warp * STAGES * TP * BS;
  const int* tab = pt + (size_t)blockIdx.x * np;
  const int ntiles = (np + TP - 1) / TP;
  const int my = ntiles > warp ? (ntiles - warp + W - 1) / W : 0;
  auto issue = [&](int j) {
    const int tile = warp + j * W;
    uint8_t* dst = R + (j % STAGES) * TP * BS;
    for (int i = 0; i < TP; ++i) {
      const int p = tile * TP + i;
      if (p < np) {
        const uint8_t* src = pool + (size_t)tab[p] * BS;
        for (int c = lane; c < BS / 16; c += 32) cp_async16(dst + i * BS + 16 * c, src + 16 * c);
      }
    }
  };
  for (int s = 0; s < STAGES - 1; ++s) { if (s < my) issue(s); cp_commit(); }
  float acc = 0.f;
  for (int j = 0; j < my; ++j) {
    if (j + STAGES - 1 < my) issue(j + STAGES - 1);
    cp_commit();
    cp_wait<STAGES - 1>();
    __syncwarp();
    const float* t = reinterpret_cast<const float*>(R + (j % STAGES) * TP * BS);
    for (int i = lane; i < TP * BS / 4; i += 32 * 8) acc += t[i];
    __syncwarp();
  }
  cp_wait<0>();
  if (acc == 12345.f) out[blockIdx.x] = acc;
}

// TMA bulk: warp w, lane 0 issues one bulk copy per page into stage slots; mbarrier per stage
template <int W, int STAGES, int TP, int BS>
__global__ void __launch_bounds__(W * 32) k_bulk(const uint8_t* __restrict__ pool, const int* __restrict__ pt, int np,
                                                 float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[W][STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* R = sm + (size_t)warp * STAGES * TP * BS;
  const int* tab = pt + (size_t)blockIdx.x * np;
  const int ntiles = (np + TP - 1) / TP;
  const int my = ntiles > warp ? (ntiles - warp + W - 1) / W : 0;
  if (lane < STAGES) mbar_init(&bars[warp][lane], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int j) {
    const int tile = warp + j * W;
    uint8_t* dst = R + (j % STAGES) * TP * BS;
    const int n = min(TP, np - tile * TP);
    if (lane == 0) mbar_arrive_expect_tx(&bars[warp][j % STAGES], n * BS);
    __syncwarp();
    if (lane < n) bulk_g2s(dst + lane * BS, pool + (size_t)tab[tile * TP + lane] * BS, BS, &bars[warp][j % STAGES]);
  };
  for (int s = 0; s < STAGES - 1; ++s) if (s < my) issue(s);
  float acc = 0.f;
  for (int j = 0; j < my; ++j) {
    if (j + STAGES - 1 < my) issue(j + STAGES - 1);
    mbar_wait(&bars[warp][j % STAGES], (j / STAGES) & 1);
    const float* t = reinterpret_cast<const float*>(R + (j % STAGES) * TP * BS);
    for (int i = lane; i < TP * BS / 4; i += 32 * 8) acc += t[i];
    __syncwarp();
  }
  if (acc == 12345.f) out[blockIdx.x] = acc;
}

template <class K>
float run(K kern, int grid, int threads, size_t smem, const uint8_t* pool, const int* pt, int np, float* out, int reps,
          int layers, size_t layer_pages) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) kern<<<grid, threads, smem>>>(pool, pt + (size_t)(i % layers) * grid * np, np, out);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) kern<<<grid, threads, smem>>>(pool, pt + (size_t)(i % layers) * grid * np, np, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return -1; }
  return ms * 1000.f / reps;
}

template <int W, int ST, int TP, int BS>
void both(int units, int np, int H = 0) {
  const int layers = 4;
  const size_t pages = (size_t)units * np * layers;
  uint8_t* pool; int* pt; float* out;
  cudaMalloc(&pool, pages * BS);
  cudaMemset(pool, 0, pages * BS);
  cudaMalloc(&out, 4096 * 4);
  std::vector<int> h(pages);
  for (size_t i = 0; i < pages; ++i) h[i] = (int)i;
  if (H) {  // paged layout: unit u = (seq b, head hh) owns blocks (b*np + p)*H + hh
    for (int l = 0; l < layers; ++l)
      for (int u = 0; u < units; ++u)
        for (int p = 0; p < np; ++p)
          h[((size_t)l * units + u) * np + p] = (int)((((size_t)l * (units / H) + u / H) * np + p) * H + u % H);
  } else {
    std::mt19937 rng(1);
    std::shuffle(h.begin(), h.end(), rng);
  }
  cudaMalloc(&pt, pages * 4);
  cudaMemcpy(pt, h.data(), pages * 4, cudaMemcpyHostToDevice);
  const size_t smem = (size_t)W * ST * TP * BS;
  const double bytes = (double)units * np * BS;
  float t1 = run(k_ldgsts<W, ST, TP, BS>, units, W * 32, smem, pool, pt, np, out, 20, layers, 0);
  float t2 = run(k_bulk<W, ST, TP, BS>, units, W * 32, smem, pool, pt, np, out, 20, layers, 0);
  printf("{\"H\":%d,\"units\":%d,\"np\":%d,\"BS\":%d,\"W\":%d,\"stages\":%d,\"tile_pages\":%d,\"smem_kb\":%.0f,"
         "\"ldgsts_us\":%.2f,\"ldgsts_gbs\":%.0f,\"bulk_us\":%.2f,\"bulk_gbs\":%.0f}\n",
         H, units, np, BS, W, ST, TP, smem / 1024.0, t1, bytes / t1 / 1e3, t2, bytes / t2 / 1e3);
  cudaFree(pool); cudaFree(pt); cudaFree(out);
}

int main() {
  both<12, 3, 8, 512>(128, 2049, 8);
  both<16, 3, 8, 512>(128, 2049, 8);
  both<24, 3, 4, 512>(128, 2049, 8);
  both<32, 3, 4, 512>(128, 2049, 8);
  both<8, 3, 16, 512>(128, 2049, 8);
  both<16, 3, 8, 512>(128, 2049, 0);
  both<32, 3, 4, 512>(128, 2049, 0);
  both<16, 3, 4, 1152>(128, 1195, 8);
  both<24, 3, 2, 1152>(128, 1195, 8);
  both<32, 3, 2, 1152>(128, 1195, 8);
  both<16, 3, 4, 1152>(128, 1195, 0);
  both<32, 3, 2, 1152>(128, 1195, 0);
  both<16, 3, 4, 1152>(256, 598, 8);
  both<32, 3, 4, 512>(256, 8193, 8);
  both<16, 3, 8, 512>(256, 8193, 8);
  both<32, 3, 4, 512>(16, 513, 8);
  both<32, 3, 4, 512>(64, 129, 8);
  return 0;
}
