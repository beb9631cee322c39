// Micro-benchmarks that size the Twilight kernels on B200 (sm_100a):
// FP32 FFMA vs packed FFMA2, FP64 DFMA, legacy HMMA (mma.sync bf16) issue
// rates, and HBM read bandwidth for streaming / per-SM / 256-B row gathers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void ffma_k(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  float bb = b + threadIdx.x * 1e-9f;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    x0 = fmaf(x0, a, bb); x1 = fmaf(x1, a, bb); x2 = fmaf(x2, a, bb); x3 = fmaf(x3, a, bb);
    x4 = fmaf(x4, a, bb); x5 = fmaf(x5, a, bb); x6 = fmaf(x6, a, bb); x7 = fmaf(x7, a, bb);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// register-register form: multiplier is a per-thread register, not an immediate/uniform
__global__ void ffma_rr_k(float* out, const float* in) {
  float a = in[threadIdx.x], b = in[threadIdx.x + 1];
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
    x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void ffma2(unsigned long long& x, unsigned long long a, unsigned long long b) {
  asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x) : "l"(a), "l"(b));
}

__global__ void ffma2_k(float* out, const float* in) {
  float2 af = make_float2(in[threadIdx.x], in[threadIdx.x + 1]);
  float2 bf = make_float2(in[threadIdx.x + 2], in[threadIdx.x + 3]);
  unsigned long long a = *reinterpret_cast<unsigned long long*>(&af);
  unsigned long long b = *reinterpret_cast<unsigned long long*>(&bf);
  unsigned long long x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { float2 t = make_float2(threadIdx.x + j, j); x[j] = *reinterpret_cast<unsigned long long*>(&t); }
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) ffma2(x[j], a, b);
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) { float2 t = *reinterpret_cast<float2*>(&x[j]); s += t.x + t.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_k(double* out, const double* in) {
  double a = in[threadIdx.x], b = in[threadIdx.x + 1];
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 16
  for (int i = 0; i < ITERS / 4; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void hmma_k(float* out, const uint32_t* in) {
  uint32_t a0 = in[threadIdx.x], a1 = in[threadIdx.x + 1], a2 = in[threadIdx.x + 2], a3 = in[threadIdx.x + 3];
  uint32_t b0 = in[threadIdx.x + 4], b1 = in[threadIdx.x + 5];
  float c[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) for (int t = 0; t < 4; ++t) c[j][t] = 0.f;
#pragma unroll 4
  for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void imma_k(int* out, const uint32_t* in) {
  uint32_t a0 = in[threadIdx.x], a1 = in[threadIdx.x + 1], a2 = in[threadIdx.x + 2], a3 = in[threadIdx.x + 3];
  uint32_t b0 = in[threadIdx.x + 4], b1 = in[threadIdx.x + 5];
  int c[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) for (int t = 0; t < 4; ++t) c[j][t] = 0;
#pragma unroll 4
  for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ int4 ld_nc(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// grid-stride streaming read, 4 x 16 B in flight per thread per iteration
__global__ void stream_k(const int4* __restrict__ in, size_t n16, int* out) {
  int acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x * 4;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; i < n16; i += stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { size_t j = i + u * blockDim.x; v[u] = j < n16 ? ld_nc(in + j) : make_int4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

// gather of 256-byte rows at random row indices (one row = 16 lanes x 16 B)
__global__ void gather_k(const int4* __restrict__ base, const int* __restrict__ rows, int nrows, int* out) {
  int acc = 0;
  int lane16 = threadIdx.x & 15;
  int grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  int ngrp = (gridDim.x * blockDim.x) >> 4;
  for (int r = grp; r < nrows; r += ngrp * 4) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { int rr = r + u * ngrp; v[u] = rr < nrows ? ld_nc(base + (size_t)rows[rr] * 16 + lane16) : make_int4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678) out[0] = acc;
}

__global__ void flush_k(int4* buf, size_t n16) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) buf[i] = make_int4(i, 0, 0, 0);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  float *fo, *fi; double *dout, *din; uint32_t* ui; int* io;
  CK(cudaMalloc(&fo, sizeof(float) * 148 * 8 * 1024));
  CK(cudaMalloc(&fi, 4096)); CK(cudaMemset(fi, 0, 4096));
  CK(cudaMalloc(&dout, sizeof(double) * 148 * 8 * 1024)); CK(cudaMalloc(&din, 8192)); CK(cudaMemset(din, 0, 8192));
  CK(cudaMalloc(&ui, 4096)); CK(cudaMemset(ui, 0, 4096)); CK(cudaMalloc(&io, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int blocks = sms * 4, threads = 256;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  auto timeit = [&](auto launch) { launch(); cudaDeviceSynchronize(); cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); return ms / 5; };
  double t;
  t = timeit([&] { ffma_k<<<blocks, threads>>>(fo, 1.0001f, 0.5f); });
  printf(", \"ffma_uniform_tflops\": %.1f", 2.0 * blocks * threads * ITERS * 8 / (t * 1e-3) / 1e12);
  t = timeit([&] { ffma_rr_k<<<blocks, threads>>>(fo, fi); });
  printf(", \"ffma_reg_tflops\": %.1f", 2.0 * blocks * threads * ITERS * 8 / (t * 1e-3) / 1e12);
  t = timeit([&] { ffma2_k<<<blocks, threads>>>(fo, fi); });
  printf(", \"ffma2_tflops\": %.1f", 2.0 * 2 * blocks * threads * ITERS * 8 / (t * 1e-3) / 1e12);
  t = timeit([&] { dfma_k<<<blocks, threads>>>(dout, din); });
  printf(", \"dfma_tflops\": %.2f", 2.0 * blocks * threads * (ITERS / 4) * 8 / (t * 1e-3) / 1e12);
  t = timeit([&] { hmma_k<<<blocks, threads>>>(fo, ui); });
  printf(", \"hmma_bf16_tflops\": %.1f", 2.0 * 16 * 8 * 16 * (blocks * threads / 32) * (ITERS / 8) * 8 / (t * 1e-3) / 1e12);
  t = timeit([&] { imma_k<<<blocks, threads>>>((int*)fo, ui); });
  printf(", \"imma_u8s8_tops\": %.1f", 2.0 * 16 * 8 * 32 * (blocks * threads / 32) * (ITERS / 8) * 8 / (t * 1e-3) / 1e12);
  CK(cudaGetLastError());
  fflush(stdout);

  size_t bytes = (size_t)4 << 30;
  int4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  size_t n16 = bytes / 16;
  for (int bpsm : {1, 2, 4, 8}) {
    for (int thr : {256, 512, 1024}) {
      if (bpsm * thr > 2048) continue;
      t = timeit([&] { stream_k<<<sms * bpsm, thr>>>(buf, n16, io); });
      printf(", \"stream_read_gbs_b%d_t%d\": %.0f", bpsm, thr, bytes / (t * 1e-3) / 1e9);
    }
  }
  // per-SM bandwidth: one CTA on a few SMs only, each streaming its own 64 MB slice
  for (int ncta : {1, 16, 32, 64}) {
    size_t sl = (size_t)ncta * (64 << 20) / 16;
    t = timeit([&] { stream_k<<<ncta, 1024>>>(buf, sl, io); });
    printf(", \"per_cta_gbs_n%d\": %.1f", ncta, sl * 16.0 / (t * 1e-3) / 1e9 / ncta);
  }
  // random 256-B row gather across the 4 GB buffer
  int nrows = 1 << 22;
  int* rows; CK(cudaMalloc(&rows, nrows * 4));
  {
    int* h = new int[nrows]; uint64_t s = 88172645463325252ull; size_t total_rows = bytes / 256;
    for (int i = 0; i < nrows; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % total_rows); }
    CK(cudaMemcpy(rows, h, nrows * 4, cudaMemcpyHostToDevice)); delete[] h;
  }
  int4* fl; size_t fbytes = (size_t)512 << 20; CK(cudaMalloc(&fl, fbytes));
  for (int bpsm : {4, 8}) {
    float tot = 0; int reps = 5;
    for (int r = 0; r < reps; ++r) {
      flush_k<<<sms * 4, 512>>>(fl, fbytes / 16);
      cudaEventRecord(e0); gather_k<<<sms * bpsm, 256>>>(buf, rows, nrows, io); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); tot += ms;
    }
    printf(", \"gather256_gbs_b%d\": %.0f", bpsm, (double)nrows * 256 / (tot / reps * 1e-3) / 1e9);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
