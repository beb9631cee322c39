// K3a: INT4 SpGEMV estimate q . k_hat / sqrt(d) over the candidate pages, all
// G query heads of a unit from ONE read of the packed codes.
//
// Reference: estimate_scores, quantcache.py:238-272 (k_hat = zero + scale*code,
// score = (k_hat . q) * (1/sqrt d)), called per head over the group union at
// pipeline.py:342.  Here score = (zero * sum(q) + scale * sum_c q_c code_c) / sqrt d.
//
// Why tensor cores here: per 72-byte token the estimate needs G*d = 512 MACs
// (G=4).  At B200's measured 35 T FFMA/s (tools/microbench.cu) CUDA cores
// would take longer than streaming the codes at HBM speed, so the
// code-times-query product runs on legacy mma.sync (bf16, m16n8k16): a page is
// exactly one 16-row A tile, the G heads (times 1 or 3 bf16 terms of q) are the
// N columns.  Codes 0..15 are exact in bf16, products are exact, accumulation
// is fp32 -- the arithmetic matches an fp32 FFMA dot product.
//
// Fragment trick (no shared memory, no ldmatrix): lane (t = lane%4, r = lane/4)
// loads the 16 contiguous bytes [16t, 16t+16) of rows r and r+8 of the page --
// one fully coalesced 512-B LDG.128 per 8 rows, straight from the reference
// byte layout.  The K dimension of the MMA is permuted so that each 32-bit
// word of nibbles expands to bf16x2 A registers with one LOP3 (+ shift) and a
// bf16 subtract of the 0x4300 magic; q's B fragments use the same permutation.
#include "common.cuh"

namespace tw {

constexpr int kEstPagesPerCta = 32;  // 4 warps x 8 pages
constexpr int kEstWarps = 4;

__device__ __forceinline__ uint32_t bf16x2_bits(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// (n_a, n_b) nibble pair of `w` at bit offsets (sh, sh+16) -> exact bf16x2
__device__ __forceinline__ uint32_t nib2bf16(uint32_t w, int sh) {
  uint32_t x = ((w >> sh) & 0x000F000Fu) | 0x43004300u;  // bf16(128 + n)
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&x);
  const __nv_bfloat162 off = __floats2bfloat162_rn(128.f, 128.f);
  v = __hsub2(v, off);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// channel that k-slot `slot` (0..15) of k-step s maps to for lane group t
__device__ __forceinline__ int kslot_channel(int t, int s, int slot) {
  const int m = s >> 1, hf = s & 1;
  const int j = slot & 7;            // 0,1 -> first pair; 8,9 handled by caller
  const int base = 32 * t + 8 * m + 2 * hf;
  return base + (slot >= 8 ? 1 : 0) + ((j & 1) ? 4 : 0);
}

template <typename T, int G, int TERMS>
__global__ void __launch_bounds__(kEstWarps * 32) estimate_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                                  tw_decode_buffers buf) {
  const int unit = blockIdx.y;
  const int ncand = buf.cand_count[unit];
  const int c0 = blockIdx.x * kEstPagesPerCta;
  if (c0 >= ncand) return;
  const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
  const int n = kv.seq_lens[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane & 3, r = lane >> 2;
  const int T_stride = kv.max_pages * kPage;

  // ---- B fragments: q of head n = r (lanes with r >= G carry zeros), split into TERMS bf16 parts
  uint32_t bf[TERMS][8][2];
  {
    const T* qh = q + ((size_t)unit * G + (r < G ? r : 0)) * kHeadDim;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      float v[4];
      const int slots[4] = {2 * t, 2 * t + 1, 2 * t + 8, 2 * t + 9};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int sl = slots[e] - 2 * t;  // 0,1,8,9
        v[e] = r < G ? Elem<T>::to_f(qh[kslot_channel(t, s, sl)]) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < TERMS; ++j) {
        float hi[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hi[e] = __bfloat162float(__float2bfloat16_rn(v[e]));
          if (j + 1 < TERMS) v[e] -= hi[e];  // exact residual
        }
        bf[j][s][0] = bf16x2_bits(hi[0], hi[1]);
        bf[j][s][1] = bf16x2_bits(hi[2], hi[3]);
      }
    }
  }
  // sum_c q_c of the two heads whose accumulator columns this lane holds
  float sq[2] = {0.f, 0.f};
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const T* qh = q + ((size_t)unit * G + g) * kHeadDim + 4 * lane;
    float s = (Elem<T>::to_f(qh[0]) + Elem<T>::to_f(qh[1])) + (Elem<T>::to_f(qh[2]) + Elem<T>::to_f(qh[3]));
    s = warp_sum(s);
    if (g == 2 * t) sq[0] = s;
    if (g == 2 * t + 1) sq[1] = s;
  }
  const float inv_sqrt_d = 0.08838834764831845f;  // float32(1/sqrt(128)), as quantcache.py:258
  float run_max[2] = {-INFINITY, -INFINITY};

  const int* cand = buf.cand_pages + (size_t)unit * kv.max_pages;
  const int* pt = kv.page_table + (size_t)b * kv.max_pages;
  const int cend = min(c0 + kEstPagesPerCta, ncand);
  // all pages of this warp (ci = c0 + warp + 4*i, i < 8) are loaded up front:
  // 16 x 16 B of codes + 8 params per lane in flight before the first MMA
  constexpr int kPPW = kEstPagesPerCta / kEstWarps;
  int lp_all = 0;
  {
    const int ci = c0 + warp + kEstWarps * lane;
    if (lane < kPPW && ci < cend) lp_all = cand[ci];
  }
  uint4 lo4[kPPW], hi4[kPPW];
  float prmv[kPPW];
#pragma unroll
  for (int i = 0; i < kPPW; ++i) {
    const int ci = c0 + warp + kEstWarps * i;
    const int lpi = __shfl_sync(0xffffffffu, lp_all, i);
    if (ci < cend) {
      const uint8_t* qb = kv.kq + ((size_t)pt[lpi] * kv.num_kv_heads + h) * kQBlockBytes;
      lo4[i] = ld_stream(qb + r * 64 + t * 16);
      hi4[i] = ld_stream(qb + (r + 8) * 64 + t * 16);
      prmv[i] = __ldg(reinterpret_cast<const float*>(qb + kCodeBytes) + lane);
    }
  }
#pragma unroll
  for (int i = 0; i < kPPW; ++i) {
    const int ci = c0 + warp + kEstWarps * i;
    if (ci >= cend) break;
    const int lp = __shfl_sync(0xffffffffu, lp_all, i);
    // ---- MMA over the 8 k-steps
    float acc[TERMS][4];
#pragma unroll
    for (int j = 0; j < TERMS; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    const uint32_t wl[4] = {lo4[i].x, lo4[i].y, lo4[i].z, lo4[i].w};
    const uint32_t wh[4] = {hi4[i].x, hi4[i].y, hi4[i].z, hi4[i].w};
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int m = s >> 1, sh = (s & 1) ? 8 : 0;
      uint32_t a[4];
      a[0] = nib2bf16(wl[m], sh);
      a[1] = nib2bf16(wh[m], sh);
      a[2] = nib2bf16(wl[m], sh + 4);
      a[3] = nib2bf16(wh[m], sh + 4);
#pragma unroll
      for (int j = 0; j < TERMS; ++j) mma_bf16(acc[j], a, bf[j][s][0], bf[j][s][1]);
    }
    // ---- epilogue: rows r and r+8, heads 2t and 2t+1
    const float pv = prmv[i];
    const float sc_r = __shfl_sync(0xffffffffu, pv, r), sc_r8 = __shfl_sync(0xffffffffu, pv, r + 8);
    const float z_r = __shfl_sync(0xffffffffu, pv, 16 + r), z_r8 = __shfl_sync(0xffffffffu, pv, 24 + r);
    float d[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float x = acc[0][e];
#pragma unroll
      for (int j = 1; j < TERMS; ++j) x += acc[j][e];
      d[e] = x;
    }
    const int tok_r = lp * kPage + r;
    const bool v_r = tok_r < n, v_r8 = tok_r + 8 < n;
    if (2 * t < G) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int g = 2 * t + e;
        if (g < G) {
          float l0 = v_r ? fmaf(sc_r, d[e], z_r * sq[e]) * inv_sqrt_d : -INFINITY;
          float l1 = v_r8 ? fmaf(sc_r8, d[2 + e], z_r8 * sq[e]) * inv_sqrt_d : -INFINITY;
          float* lg = buf.logits + ((size_t)unit * G + g) * T_stride + (size_t)ci * kPage;
          lg[r] = l0;
          lg[r + 8] = l1;
          run_max[e] = fmaxf(run_max[e], fmaxf(l0, l1));
        }
      }
    }
  }
  // per-head max over this warp -> global (ordered-key atomicMax)
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    float mx = run_max[e];
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    const int g = 2 * t + e;
    if (r == 0 && g < G && mx > -INFINITY) atomicMax(buf.head_max + (size_t)unit * G + g, f2key(mx));
  }
}

// ---------------------------------------------------------------- per-token API

// estimate_scores at arbitrary token ids (quantcache.py:238-272): warp per
// token, k_hat formed in fp64 and rounded to fp32 per element like :269.
template <typename T>
__global__ void estimate_tokens_kernel(tw_paged_kv kv, int seq, int kvh, const T* __restrict__ q,
                                       const int32_t* __restrict__ idx, int m, float* __restrict__ out,
                                       int32_t* status) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= m) return;
  const int tok = idx[w];
  const int n = kv.seq_lens[seq];
  if (tok < 0 || tok >= n) {
    if (lane == 0) *status = TW_ERR_INDEX;
    return;
  }
  const int phys = kv.page_table[(size_t)seq * kv.max_pages + tok / kPage];
  const uint8_t* qb = kv.kq + ((size_t)phys * kv.num_kv_heads + kvh) * kQBlockBytes;
  const int slot = tok % kPage;
  const uint16_t codes = reinterpret_cast<const uint16_t*>(qb + slot * (kHeadDim / 2))[lane];
  const float* prm = reinterpret_cast<const float*>(qb + kCodeBytes);
  const double scale = prm[slot], zero = prm[kPage + slot];
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float kh = (float)(zero + scale * (double)((codes >> (4 * i)) & 0xF));
    acc = fmaf(kh, Elem<T>::to_f(q[4 * lane + i]), acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) out[w] = acc * 0.08838834764831845f;
}

}  // namespace tw

using namespace tw;

template <typename T, int TERMS>
static int launch_estimate(const tw_paged_kv* kv, const T* q, const tw_decode_buffers* buf, cudaStream_t stream) {
  const int units = kv->num_seqs * kv->num_kv_heads;
  dim3 grid((kv->max_pages + kEstPagesPerCta - 1) / kEstPagesPerCta, units), block(kEstWarps * 32);
  switch (kv->group_size) {
    case 1: estimate_kernel<T, 1, TERMS><<<grid, block, 0, stream>>>(*kv, q, *buf); break;
    case 2: estimate_kernel<T, 2, TERMS><<<grid, block, 0, stream>>>(*kv, q, *buf); break;
    case 4: estimate_kernel<T, 4, TERMS><<<grid, block, 0, stream>>>(*kv, q, *buf); break;
    case 8: estimate_kernel<T, 8, TERMS><<<grid, block, 0, stream>>>(*kv, q, *buf); break;
    default: return TW_ERR_INVALID;
  }
  return launch_status();
}

extern "C" int tw_estimate(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                           const tw_decode_buffers* buf, cudaStream_t stream) {
  (void)prm;
  if (!kv || !q || !buf || kv->head_dim != kHeadDim || !buf->logits || !buf->head_max) return TW_ERR_INVALID;
  cudaMemsetAsync(buf->head_max, 0, sizeof(uint32_t) * kv->num_seqs * kv->num_kv_heads * kv->group_size, stream);
  if (kv->dtype == TW_BF16) return launch_estimate<__nv_bfloat16, 1>(kv, (const __nv_bfloat16*)q, buf, stream);
  return launch_estimate<float, 3>(kv, (const float*)q, buf, stream);
}

extern "C" int tw_estimate_tokens(const tw_paged_kv* kv, int32_t seq, int32_t kv_head, const void* q,
                                  const int32_t* token_idx, int32_t m, float* scores_out, int32_t* status_out,
                                  cudaStream_t stream) {
  if (!kv || !q || !token_idx || !scores_out || m < 1 || kv->head_dim != kHeadDim) return TW_ERR_INVALID;
  const int warps = 8;
  dim3 grid((m + warps - 1) / warps), block(32 * warps);
  if (kv->dtype == TW_BF16)
    estimate_tokens_kernel<__nv_bfloat16><<<grid, block, 0, stream>>>(*kv, seq, kv_head, (const __nv_bfloat16*)q,
                                                                      token_idx, m, scores_out, status_out);
  else
    estimate_tokens_kernel<float><<<grid, block, 0, stream>>>(*kv, seq, kv_head, (const float*)q, token_idx, m,
                                                              scores_out, status_out);
  return launch_status();
}
