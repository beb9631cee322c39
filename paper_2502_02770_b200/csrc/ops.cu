// Per-vector operators of the reference API on CUDA tensors (off the decode
// hot path, which runs K1-K4; these serve callers of the reference's own
// operator signatures, attention.py:79-136):
//
//   tw_vec_logits   z = K q / float32(sqrt d)          attention_weights :89-103 (:102)
//   tw_vec_softmax  exp(z - max z) / sum               stable_softmax    :79-86
//   tw_vec_readout  w[S] @ V[S] (/ sum w[S])           sparse_attention  :106-136 (:130-135)
//
// Memory-bound GEMV / gather: warp-per-row dots for the logits, grid-stride
// block reductions (max by ordered key, sum in fp64) for the softmax, and a
// two-stage (per-block partials, then one finalising block) reduction for the
// readout, so results do not depend on atomic ordering.
#include <algorithm>

#include "common.cuh"

namespace tw {

template <typename T>
__global__ void __launch_bounds__(256) vec_logits_kernel(const T* __restrict__ q, const T* __restrict__ keys, int64_t n,
                                                         int d, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const float sd = (float)sqrt((double)d);  // the reference divides by float32(sqrt d) (attention.py:102)
  for (int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); row < n; row += (int64_t)gridDim.x * 8) {
    const T* k = keys + row * d;
    float acc = 0.f;
    for (int c = lane; c < d; c += 32) acc = fmaf(Elem<T>::to_f(k[c]), Elem<T>::to_f(q[c]), acc);
    acc = warp_sum(acc);
    if (lane == 0) out[row] = acc / sd;
  }
}

// scratch[0] = ordered key of the max, scratch[1..2] = fp64 sum (8-byte aligned at +8)
__global__ void __launch_bounds__(256) vec_max_kernel(const float* __restrict__ z, int64_t n, uint32_t* __restrict__ mx) {
  __shared__ uint32_t red[8];
  uint32_t m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, f2key(z[i]));
  m = warp_max_u32(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = max(m, red[w]);
    atomicMax(mx, max(m, red[0]));
  }
}

__global__ void __launch_bounds__(256) vec_expsum_kernel(const float* __restrict__ z, int64_t n,
                                                         const uint32_t* __restrict__ mx, double* __restrict__ sum) {
  __shared__ double red[8];
  const float M = key2f(*mx);
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += (double)expf(z[i] - M);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    atomicAdd(sum, s);
  }
}

__global__ void __launch_bounds__(256) vec_normalize_kernel(const float* __restrict__ z, int64_t n,
                                                            const uint32_t* __restrict__ mx,
                                                            const double* __restrict__ sum, float* __restrict__ out) {
  const float M = key2f(*mx);
  const float inv = (float)(1.0 / *sum);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = expf(z[i] - M) * inv;
}

// Stage 1: block b sums rows j = b, b + nblocks, ... of the selection into
// partial[b][0..d) (weighted values) and partial[b][d] (the weight mass).
template <typename WT, typename VT>
__global__ void __launch_bounds__(256) vec_readout_partial_kernel(const WT* __restrict__ w, const VT* __restrict__ v,
                                                                  int d, const int64_t* __restrict__ idx, int64_t m,
                                                                  double* __restrict__ partial) {
  double* part = partial + (size_t)blockIdx.x * (d + 1);
  for (int c = threadIdx.x; c <= d; c += blockDim.x) {
    double acc = 0.0;
    for (int64_t j = blockIdx.x; j < m; j += gridDim.x) {
      const int64_t t = idx[j];
      const double wt = (double)w[t];
      acc += c < d ? wt * (double)Elem<VT>::to_f(v[t * d + c]) : wt;
    }
    part[c] = acc;
  }
}
template <typename WT>
__global__ void __launch_bounds__(256) vec_readout_final_kernel(const double* __restrict__ partial, int parts, int d,
                                                                int renorm, WT* __restrict__ out,
                                                                double* __restrict__ mass_out) {
  __shared__ double mass;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int b = 0; b < parts; ++b) s += partial[(size_t)b * (d + 1) + d];
    mass = s;
    *mass_out = s;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < parts; ++b) s += partial[(size_t)b * (d + 1) + c];
    out[c] = (WT)(renorm ? (mass > 0.0 ? s / mass : 0.0) : s);
  }
}

}  // namespace tw

using namespace tw;

static int vec_grid(int64_t work, int per_block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (work + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * 8));
}

extern "C" int tw_vec_logits(const void* q, const void* keys, int64_t n, int32_t d, int32_t dtype, float* out,
                             cudaStream_t stream) {
  if (!q || !keys || !out || n < 1 || d < 1) return TW_ERR_INVALID;
  const int grid = vec_grid(n, 8);
  if (dtype == TW_BF16)
    vec_logits_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)keys,
                                                                n, d, out);
  else if (dtype == TW_F32)
    vec_logits_kernel<float><<<grid, 256, 0, stream>>>((const float*)q, (const float*)keys, n, d, out);
  else
    return TW_ERR_INVALID;
  return launch_status();
}

extern "C" int tw_vec_softmax(const float* z, int64_t n, float* out, void* scratch, cudaStream_t stream) {
  if (!z || !out || !scratch || n < 1) return TW_ERR_INVALID;
  uint32_t* mx = reinterpret_cast<uint32_t*>(scratch);
  double* sum = reinterpret_cast<double*>(reinterpret_cast<char*>(scratch) + 8);
  cudaMemsetAsync(scratch, 0, 16, stream);
  const int grid = vec_grid(n, 256);
  vec_max_kernel<<<grid, 256, 0, stream>>>(z, n, mx);
  vec_expsum_kernel<<<grid, 256, 0, stream>>>(z, n, mx, sum);
  vec_normalize_kernel<<<grid, 256, 0, stream>>>(z, n, mx, sum, out);
  return launch_status();
}

extern "C" int32_t tw_vec_readout_parts(void) { return 148; }

extern "C" int tw_vec_readout(const void* w, int32_t wdtype, const void* v, int32_t vdtype, int64_t n, int32_t d,
                              const int64_t* idx, int64_t m, int32_t renorm, void* out, double* partial,
                              double* mass_out, cudaStream_t stream) {
  if (!w || !v || !idx || !out || !partial || !mass_out || n < 1 || d < 1 || m < 1) return TW_ERR_INVALID;
  const int parts = (int)std::min<int64_t>(m, tw_vec_readout_parts());
  // wdtype: TW_F32 or 2 (= fp64); the output has the weights' type (the promotion of w and V)
  auto go = [&](auto wt, auto vt) {
    using WT = decltype(wt);
    using VT = decltype(vt);
    vec_readout_partial_kernel<WT, VT><<<parts, 256, 0, stream>>>((const WT*)w, (const VT*)v, d, idx, m, partial);
    vec_readout_final_kernel<WT><<<1, 256, 0, stream>>>(partial, parts, d, renorm, (WT*)out, mass_out);
  };
  if (wdtype == TW_F32 && vdtype == TW_F32) go(float(), float());
  else if (wdtype == TW_F32 && vdtype == TW_BF16) go(float(), __nv_bfloat16());
  else if (wdtype == 2 && vdtype == TW_F32) go(double(), float());
  else if (wdtype == 2 && vdtype == TW_BF16) go(double(), __nv_bfloat16());
  else return TW_ERR_INVALID;
  return launch_status();
}
