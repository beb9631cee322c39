// K3a: INT4 SpGEMV estimate q . k_hat / sqrt(d) over the candidate pages, all
// G query heads of a unit from ONE read of the packed codes.
//
// Reference: estimate_scores, quantcache.py:238-272 (k_hat = zero + scale*code,
// score = (k_hat . q) * (1/sqrt d)), called per head over the group union at
// pipeline.py:342.  Here score = (zero * sum(q) + scale * sum_c q_c code_c) / sqrt d.
//
// Why tensor cores here: per 72-byte token the estimate needs G*d = 512 MACs
// (G=4).  At B200's measured 35 T FFMA/s (tools/microbench.cu) CUDA cores
// would take longer than streaming the codes at HBM speed.  The code-times-
// query product runs on legacy integer MMA (mma.sync m16n8k32 u8 x s8 -> s32,
// 1.1 POPS measured): a page is one 16-row A tile; q is a 22-bit fixed-point
// vector split into three signed 8-bit digits (one MMA column block per digit),
// so every product and sum is exact integer arithmetic and the only rounding
// is q -> fixed point (2^-22 of max|q|).  Nibbles become u8 A operands with
// one AND (+ one shift) per 8 codes, 4x fewer instructions than a bf16 expand.
//
// Fragment trick (no ldmatrix): lane (t = lane%4, r = lane/4) reads the 16
// contiguous bytes [16t, 16t+16) of rows r and r+8 of the page -- the
// reference's own byte layout, staged through a per-warp cp.async ring.  The
// MMA's K order is permuted so the low nibbles of a 32-bit word are one A
// register and the high nibbles another; q's B fragments use the same order.
#include <algorithm>
#include <type_traits>

#include "estimate_body.cuh"

namespace tw {

#ifdef TW_EST_TRACE
// per work item: start, end (globaltimer ns), global warp id (tools/att_trace.py --kernel estimate)
static __device__ unsigned long long g_et[65536][3];
extern "C" int tw_debug_etrace(unsigned long long* host_out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, g_et, sizeof(g_et));
  static unsigned long long zeros[65536 * 3];
  cudaMemcpyToSymbol(g_et, zeros, sizeof(zeros));
  return 0;
}
__device__ __forceinline__ unsigned long long etimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

#ifndef TW_EST_ITEM
#define TW_EST_ITEM 32
#endif
#ifndef TW_EST_STAGES
#define TW_EST_STAGES 6
#endif
constexpr int kEstPagesPerCta = TW_EST_ITEM;  // candidate pages per work item (<= 32: one per lane)
constexpr int kEstWarps = 4;

constexpr int kEstStages = TW_EST_STAGES;  // pages in flight per warp (ring stages)
#ifndef TW_EST_IPW
#define TW_EST_IPW 1
#endif
constexpr int kEstItemsPerWarp = TW_EST_IPW;
#ifndef TW_EST_BULK
#define TW_EST_BULK 0  // r02: bulk copies measured 1-2% slower (C2 47.5 vs 46.9 us, C3 401 vs 392 us)
#endif

// Persistent warp workers over (unit, 32-candidate-page) items, chunk-major;
// each warp streams its pages' 1152-B INT4 blocks through a 4-deep ring of
// 72 16-byte cp.async per page; built with -DTW_EST_BULK=1 every page is ONE
// TMA bulk copy (cp.async.bulk, issued by the lane that holds the page's
// address) completing on a per-stage mbarrier (measured 1-2% slower).
// MASKED: the sink-window or channel-pruned selectors' token masks are
// applied; the plain (Quest / full) variant drops those per-page tests.
template <typename T, int G, int BITS, bool MASKED>
__global__ void __launch_bounds__(kEstWarps * 32) estimate_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                                  tw_decode_buffers buf, int max_chunks,
                                                                  int sw_sink, int sw_window,
                                                                  const uint32_t* __restrict__ tok_mask,
                                                                  int item) {
  pdl_wait();
  pdl_trigger();
  constexpr int kSt = BITS == 8 && kEstStages > 4 ? 4 : kEstStages;  // 8-bit blocks: static smem cap
  constexpr int kBlock = qblock_bytes_for(BITS), kCodes = code_bytes_for(BITS), kRowBytes = kHeadDim * BITS / 8;
  __shared__ __align__(128) uint8_t ring[kEstWarps][kSt][kBlock];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#if TW_EST_BULK
  __shared__ __align__(8) uint64_t bars[kEstWarps][kSt];
  if (lane < kSt) mbar_init(&bars[warp][lane], 1);
  mbar_fence_init();
  __syncwarp();
  uint32_t issued = 0;  // pages this warp has issued: page j of all items uses slot j % kSt, parity (j / kSt) & 1
#endif
  const int t = lane & 3, r = lane >> 2;
  const int units = kv.num_seqs * kv.num_kv_heads;
  const int T_stride = kv.max_pages * kPage;
  const float inv_sqrt_d = 0.08838834764831845f;  // float32(1/sqrt(128)), as quantcache.py:258
  uint8_t (*R)[kBlock] = ring[warp];
  constexpr bool kPacked = G <= 4;
  uint32_t bd[kPacked ? 1 : kDigits][4][2];
  uint32_t pb1[4][2], pb2[4][2];
  float sq[2], isc[2];
  int cur_unit = -1;
  float run_max[2] = {-INFINITY, -INFINITY};
  auto flush_max = [&](int u) {
    if constexpr (kPacked) {
      float mx = run_max[0];
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      if (r == 0 && t < G && mx > -INFINITY) atomicMax(buf.head_max + (size_t)u * G + t, f2key(mx));
      run_max[0] = -INFINITY;
    } else {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      float mx = run_max[e];
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      const int g = 2 * t + e;
      if (r == 0 && g < G && mx > -INFINITY) atomicMax(buf.head_max + (size_t)u * G + g, f2key(mx));
      run_max[e] = -INFINITY;
    }
    }
  };
  // chunks past the longest candidate list are empty: the select left the
  // maximum candidate-page count in counters[6]
  // items per warp: `item` (host) shrinks on the device while the live items (the longest
  // candidate list in counters[6] sets the chunk count) leave fewer than
  // kEstItemsPerWarp per warp -- at C2 32-page items were ~1.2 per warp, so the warps
  // that drew a second one set the kernel's length
  const int maxc = (int)buf.counters[6];
  while (item > 4 && (long long)units * ((maxc + item - 1) / item) < (long long)kEstItemsPerWarp * gridDim.x * kEstWarps)
    item >>= 1;
  const int live_chunks = (min(maxc, kv.max_pages) + item - 1) / item;
  for (int it = warp_fetch(buf.counters + 3); it < units * live_chunks; it = warp_fetch(buf.counters + 3)) {
    const int unit = it % units;  // chunk-major: non-empty items come first, spread over all warps
    const int c0 = (it / units) * item;
    const int ncand = buf.cand_count[unit];
    if (c0 >= ncand) continue;
#ifdef TW_EST_TRACE
    if (lane == 0 && it < 65536) { g_et[it][0] = etimer(); g_et[it][2] = blockIdx.x * kEstWarps + warp; }
#endif
    const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
    const int n = kv.seq_lens[b];
    const int np = min(item, ncand - c0);
    // candidate page -> physical block, one page per lane
    int lp_l = 0;
    const uint8_t* src_l = kv.kq;
    if (lane < np) {
      lp_l = buf.cand_pages[(size_t)unit * kv.max_pages + c0 + lane];
      src_l = kv.kq + ((size_t)kv.page_table[(size_t)b * kv.max_pages + lp_l] * kv.num_kv_heads + h) * kBlock;
    }
#if TW_EST_BULK
    const uint32_t base = issued;
    auto issue = [&](int i) {
      const uint32_t slot = (base + i) % kSt;
      if (lane == 0) mbar_arrive_expect_tx(&bars[warp][slot], kBlock);
      __syncwarp();
      if (lane == i) bulk_g2s(R[slot], src_l, kBlock, &bars[warp][slot]);
    };
#pragma unroll
    for (int i = 0; i < kSt - 1; ++i)
      if (i < np) issue(i);
#else
    auto issue = [&](int i) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, (unsigned long long)src_l, i));
      uint8_t* dst = R[i % kSt];
#pragma unroll
      for (int c = lane; c < kBlock / 16; c += 32) cp_async16(dst + 16 * c, src + 16 * c);
    };
#pragma unroll
    for (int i = 0; i < kSt - 1; ++i) {
      if (i < np) issue(i);
      cp_commit();
    }
#endif
    if (unit != cur_unit) {
      if (cur_unit >= 0) flush_max(cur_unit);
      if constexpr (kPacked) estimate_prologue_packed<T, G, BITS>(q, unit, pb1, pb2, sq[0], isc[0]);
      else estimate_prologue<T, G, BITS>(q, unit, reinterpret_cast<uint32_t (&)[kDigits][4][2]>(bd), sq, isc);
      cur_unit = unit;
    }
    for (int i = 0; i < np; ++i) {
      if (i + kSt - 1 < np) issue(i + kSt - 1);
#if TW_EST_BULK
      const uint32_t slot = (base + i) % kSt;
      mbar_wait(&bars[warp][slot], ((base + i) / kSt) & 1);
      const uint8_t* pg = R[slot];
#else
      cp_commit();
      cp_wait<kSt - 1>();
      __syncwarp();
      const uint8_t* pg = R[i % kSt];
#endif
      // the lane's code bytes of rows r and r+8: channels 32t .. 32t+31
      uint32_t wl[BITS], wh[BITS];
      if (BITS == 8) {
        const uint4 a0 = *reinterpret_cast<const uint4*>(pg + r * kRowBytes + t * 32);
        const uint4 a1 = *reinterpret_cast<const uint4*>(pg + r * kRowBytes + t * 32 + 16);
        const uint4 b0 = *reinterpret_cast<const uint4*>(pg + (r + 8) * kRowBytes + t * 32);
        const uint4 b1 = *reinterpret_cast<const uint4*>(pg + (r + 8) * kRowBytes + t * 32 + 16);
        const uint32_t x[16] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w,
                                b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int k = 0; k < BITS; ++k) { wl[k] = x[k]; wh[k] = x[8 + k]; }
      } else if (BITS == 4) {
        const uint4 lo4 = *reinterpret_cast<const uint4*>(pg + r * kRowBytes + t * 16);
        const uint4 hi4 = *reinterpret_cast<const uint4*>(pg + (r + 8) * kRowBytes + t * 16);
        const uint32_t x[8] = {lo4.x, lo4.y, lo4.z, lo4.w, hi4.x, hi4.y, hi4.z, hi4.w};
#pragma unroll
        for (int k = 0; k < BITS; ++k) { wl[k] = x[k]; wh[k] = x[4 + k]; }
      } else {
        const uint2 lo2 = *reinterpret_cast<const uint2*>(pg + r * kRowBytes + t * 8);
        const uint2 hi2 = *reinterpret_cast<const uint2*>(pg + (r + 8) * kRowBytes + t * 8);
        wl[0] = lo2.x; wl[1] = lo2.y; wh[0] = hi2.x; wh[1] = hi2.y;
      }
      const float pv = reinterpret_cast<const float*>(pg + kCodes)[lane];
      __syncwarp();
      const int lp = __shfl_sync(0xffffffffu, lp_l, i);
      int acc[kPacked ? 2 : kDigits][4];
#pragma unroll
      for (int k = 0; k < (kPacked ? 2 : kDigits); ++k) acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t a[4];
        if (BITS == 4) {
          a[0] = wl[j] & 0x0F0F0F0Fu;         // row r,   channels 32t+8j + {0,2,4,6}
          a[1] = wh[j] & 0x0F0F0F0Fu;         // row r+8
          a[2] = (wl[j] >> 4) & 0x0F0F0F0Fu;  // row r,   channels 32t+8j + {1,3,5,7}
          a[3] = (wh[j] >> 4) & 0x0F0F0F0Fu;  // row r+8
        } else if (BITS == 8) {
          a[0] = wl[2 * j];                   // row r,   channels 32t+8j + {0..3}
          a[1] = wh[2 * j];
          a[2] = wl[2 * j + 1];               // row r,   channels 32t+8j + {4..7}
          a[3] = wh[2 * j + 1];
        } else {
          a[0] = (wl[0] >> (2 * j)) & 0x03030303u;  // row r, channels 32t + 4i + j
          a[1] = (wh[0] >> (2 * j)) & 0x03030303u;
          a[2] = (wl[1] >> (2 * j)) & 0x03030303u;  // row r, channels 32t + 16 + 4i + j
          a[3] = (wh[1] >> (2 * j)) & 0x03030303u;
        }
        if constexpr (kPacked) {
          mma_u8s8(acc[0], a, pb1[j][0], pb1[j][1]);
          mma_u8s8(acc[1], a, pb2[j][0], pb2[j][1]);
        } else {
#pragma unroll
          for (int k = 0; k < kDigits; ++k)
            mma_u8s8(acc[k], a, reinterpret_cast<uint32_t (&)[kDigits][4][2]>(bd)[k][j][0],
                     reinterpret_cast<uint32_t (&)[kDigits][4][2]>(bd)[k][j][1]);
        }
      }
      // ---- epilogue: rows r and r+8, heads 2t and 2t+1
      const float sc_r = __shfl_sync(0xffffffffu, pv, r), sc_r8 = __shfl_sync(0xffffffffu, pv, r + 8);
      const float z_r = __shfl_sync(0xffffffffu, pv, 16 + r), z_r8 = __shfl_sync(0xffffffffu, pv, 24 + r);
      float d[4];
      if constexpr (kPacked) {  // head t: digits 0, 1 in acc[0] columns (2t, 2t+1), digit 2 in acc[1] column 2t
        d[0] = fmaf((float)acc[1][0], 65536.f, fmaf((float)acc[0][1], 256.f, (float)acc[0][0])) * isc[0];
        d[2] = fmaf((float)acc[1][2], 65536.f, fmaf((float)acc[0][3], 256.f, (float)acc[0][2])) * isc[0];
        d[1] = d[3] = 0.f;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          d[e] = fmaf((float)acc[2][e], 65536.f, fmaf((float)acc[1][e], 256.f, (float)acc[0][e])) * isc[e & 1];
      }
      const int tok_r = lp * kPage + r;
      // sink-window selection (selectors.py:164-175): tokens between the sink and the window are not candidates
      bool v_r = tok_r < n, v_r8 = tok_r + 8 < n;
      if constexpr (MASKED) {
        const bool swm = sw_window >= 0 && sw_sink + sw_window < n;
        v_r = v_r && (!swm || tok_r < sw_sink || tok_r >= n - sw_window);
        v_r8 = v_r8 && (!swm || tok_r + 8 < sw_sink || tok_r + 8 >= n - sw_window);
      }
      if (MASKED && tok_mask) {  // channel-pruned selection: only the selected tokens of a candidate page
        const uint32_t mw = __ldg(tok_mask + (size_t)unit * ((T_stride + 31) / 32) + (tok_r >> 5));
        v_r = v_r && ((mw >> (tok_r & 31)) & 1u);
        v_r8 = v_r8 && ((mw >> ((tok_r + 8) & 31)) & 1u);
      }
      const int ci = c0 + i;
      if constexpr (kPacked) {
        if (t < G) {
          const float l0 = v_r ? fmaf(sc_r, d[0], z_r * sq[0]) * inv_sqrt_d : -INFINITY;
          const float l1 = v_r8 ? fmaf(sc_r8, d[2], z_r8 * sq[0]) * inv_sqrt_d : -INFINITY;
          float* lg = buf.logits + ((size_t)unit * G + t) * T_stride + (size_t)ci * kPage;
          lg[r] = l0;
          lg[r + 8] = l1;
          run_max[0] = fmaxf(run_max[0], fmaxf(l0, l1));
        }
      } else if (2 * t < G) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int g = 2 * t + e;
          if (g < G) {
            const float l0 = v_r ? fmaf(sc_r, d[e], z_r * sq[e]) * inv_sqrt_d : -INFINITY;
            const float l1 = v_r8 ? fmaf(sc_r8, d[2 + e], z_r8 * sq[e]) * inv_sqrt_d : -INFINITY;
            float* lg = buf.logits + ((size_t)unit * G + g) * T_stride + (size_t)ci * kPage;
            lg[r] = l0;
            lg[r + 8] = l1;
            run_max[e] = fmaxf(run_max[e], fmaxf(l0, l1));
          }
        }
      }
    }
#if TW_EST_BULK
    issued = base + np;  // every issued page was waited on above
#else
    cp_wait<0>();
#endif
#ifdef TW_EST_TRACE
    if (lane == 0 && it < 65536) g_et[it][1] = etimer();
#endif
  }
  if (cur_unit >= 0) flush_max(cur_unit);
}

// ---------------------------------------------------------------- exact estimator

// estimator_bits = "exact" (_candidate_logits, pipeline.py:212-214): the
// candidates' logits K[idx] @ q / float32(sqrt d) from the full-precision key
// cache, same candidate layout and -inf padding as the INT estimate.  Warp per
// (unit, candidate page); lane (row = lane / 2, half = lane % 2) dots 64
// channels of its row with the G queries staged in shared memory.  Off the
// decode hot path (the API's exact estimator and the bypass layers of
// bypass_config, pipeline.py:129-136), so CUDA cores suffice.
template <typename T, int G>
__global__ void __launch_bounds__(kEstWarps * 32) estimate_exact_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                                        tw_decode_buffers buf, int sw_sink,
                                                                        int sw_window,
                                                                        const uint32_t* __restrict__ tok_mask) {
  __shared__ float qs[kEstWarps][G][kHeadDim];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = lane >> 1, half = lane & 1;
  const int units = kv.num_seqs * kv.num_kv_heads;
  const int T_stride = kv.max_pages * kPage;
  const float sqrt_d = 11.313708498984761f;  // float32(sqrt(128)), divided as pipeline.py:213
  int cur_unit = -1;
  float run_max[G];
#pragma unroll
  for (int g = 0; g < G; ++g) run_max[g] = -INFINITY;
  auto flush = [&](int u) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float mx = warp_max(run_max[g]);
      if (lane == 0 && mx > -INFINITY) atomicMax(buf.head_max + (size_t)u * G + g, f2key(mx));
      run_max[g] = -INFINITY;
    }
  };
  const long long items = (long long)units * kv.max_pages;
  for (long long it = (long long)blockIdx.x * kEstWarps + warp; it < items; it += (long long)gridDim.x * kEstWarps) {
    const int unit = (int)(it % units), c = (int)(it / units);
    if (c >= buf.cand_count[unit]) continue;
    const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
    const int n = kv.seq_lens[b];
    if (unit != cur_unit) {
      if (cur_unit >= 0) flush(cur_unit);
      __syncwarp();
      for (int i = lane; i < G * kHeadDim; i += 32)
        qs[warp][i / kHeadDim][i % kHeadDim] = Elem<T>::to_f(q[(size_t)unit * G * kHeadDim + i]);
      __syncwarp();
      cur_unit = unit;
    }
    const int lp = buf.cand_pages[(size_t)unit * kv.max_pages + c];
    const int phys = kv.page_table[(size_t)b * kv.max_pages + lp];
    const T* krow = reinterpret_cast<const T*>(kv.k_cache) +
                    (((size_t)phys * kv.num_kv_heads + h) * kPage + row) * kHeadDim + 64 * half;
    float acc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) acc[g] = 0.f;
#pragma unroll
    for (int c8 = 0; c8 < 8; ++c8) {
      float k8[8];
      load8(krow + 8 * c8, k8);
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[g] = fmaf(k8[i], qs[warp][g][64 * half + 8 * c8 + i], acc[g]);
    }
    const int tok = lp * kPage + row;
    bool valid = tok < n && (sw_window < 0 || sw_sink + sw_window >= n || tok < sw_sink || tok >= n - sw_window);
    if (tok_mask) valid = valid && ((__ldg(tok_mask + (size_t)unit * ((T_stride + 31) / 32) + (tok >> 5)) >>
                                     (tok & 31)) & 1u);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float z = valid ? (acc[g] + __shfl_xor_sync(0xffffffffu, acc[g], 1)) / sqrt_d : -INFINITY;
      run_max[g] = fmaxf(run_max[g], z);
      if (half == 0) buf.logits[((size_t)unit * G + g) * T_stride + (size_t)c * kPage + row] = z;
    }
  }
  if (cur_unit >= 0) flush(cur_unit);
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
  const int bits = cache_bits(kv);
  const uint8_t* qb = kv.kq + ((size_t)phys * kv.num_kv_heads + kvh) * qblock_bytes_for(bits);
  const int slot = tok % kPage;
  const uint8_t* row = qb + slot * (kHeadDim * bits / 8);
  const uint32_t codes = bits == 8 ? reinterpret_cast<const uint32_t*>(row)[lane]
                         : bits == 4 ? (uint32_t)reinterpret_cast<const uint16_t*>(row)[lane] : (uint32_t)row[lane];
  const uint32_t cmask = (1u << bits) - 1u;
  const float* prm = reinterpret_cast<const float*>(qb + code_bytes_for(bits));
  const double scale = prm[slot], zero = prm[kPage + slot];
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float kh = (float)(zero + scale * (double)((codes >> (bits * i)) & cmask));
    acc = fmaf(kh, Elem<T>::to_f(q[4 * lane + i]), acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) out[w] = acc * 0.08838834764831845f;
}

}  // namespace tw

using namespace tw;

template <typename T, int G, int BITS>
static void launch_estimate_g(const tw_paged_kv* kv, const T* q, const tw_decode_buffers* buf, int sw_sink,
                              int sw_window, const uint32_t* tok_mask, cudaStream_t stream) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, estimate_kernel<T, G, BITS, false>, kEstWarps * 32, 0);
  int grid = sms * persist_cap(per_sm);
  // item size: 32 pages (amortises the per-item index lookups and ring fill) unless
  // that leaves warps idle -- small batches split into 16-, 8- or 4-page items
  const int units = kv->num_seqs * kv->num_kv_heads;
  int item = kEstPagesPerCta;
  while (item > 4 && (long long)units * ((kv->max_pages + item - 1) / item) < (long long)grid * kEstWarps) item /= 2;
  const int max_chunks = (kv->max_pages + item - 1) / item;
  const int items = units * max_chunks;
  if (grid * kEstWarps > items) grid = (items + kEstWarps - 1) / kEstWarps;
  if (sw_window >= 0 || tok_mask)
    launch_pdl(estimate_kernel<T, G, BITS, true>, dim3(grid), dim3(kEstWarps * 32), 0, stream, *kv, q, *buf,
               max_chunks, sw_sink, sw_window, tok_mask, item);
  else
    launch_pdl(estimate_kernel<T, G, BITS, false>, dim3(grid), dim3(kEstWarps * 32), 0, stream, *kv, q, *buf,
               max_chunks, sw_sink, sw_window, tok_mask, item);
}

template <typename T>
static int launch_estimate(const tw_paged_kv* kv, const T* q, const tw_decode_buffers* buf, int ss, int sw,
                           const uint32_t* tm, bool exact, cudaStream_t stream) {
  auto by_bits = [&](auto gtag) {
    constexpr int GG = decltype(gtag)::value;
    if (exact) {
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const long long items = (long long)kv->num_seqs * kv->num_kv_heads * kv->max_pages;
      const int grid = (int)std::min<long long>((items + kEstWarps - 1) / kEstWarps, (long long)sms * 16);
      estimate_exact_kernel<T, GG><<<grid, kEstWarps * 32, 0, stream>>>(*kv, q, *buf, ss, sw, tm);
      return;
    }
    switch (cache_bits(*kv)) {
      case 2: launch_estimate_g<T, GG, 2>(kv, q, buf, ss, sw, tm, stream); break;
      case 8: launch_estimate_g<T, GG, 8>(kv, q, buf, ss, sw, tm, stream); break;
      default: launch_estimate_g<T, GG, 4>(kv, q, buf, ss, sw, tm, stream); break;
    }
  };
  switch (kv->group_size) {
    case 1: by_bits(std::integral_constant<int, 1>{}); break;
    case 2: by_bits(std::integral_constant<int, 2>{}); break;
    case 4: by_bits(std::integral_constant<int, 4>{}); break;
    case 8: by_bits(std::integral_constant<int, 8>{}); break;
    default: return TW_ERR_INVALID;
  }
  return launch_status();
}

extern "C" int tw_estimate(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                           const tw_decode_buffers* buf, cudaStream_t stream) {
  if (!kv || !q || !buf || kv->head_dim != kHeadDim || !buf->logits || !buf->head_max) return TW_ERR_INVALID;
  const bool sw = prm && prm->selector == TW_SELECT_SINK_WINDOW;
  const int ss = sw ? prm->sink : 0, swin = sw ? prm->window : -1;
  const uint32_t* tm = prm && prm->selector == TW_SELECT_CHANNEL_PRUNED ? buf->tok_mask : nullptr;
  if (prm && prm->selector == TW_SELECT_CHANNEL_PRUNED && !tm) return TW_ERR_INVALID;
  // head_max is zeroed by tw_select (quest_select_kernel), which always precedes this call
  const bool exact = prm && prm->estimator == TW_ESTIMATE_EXACT;
  if (prm && prm->estimator != TW_ESTIMATE_INT && !exact) return TW_ERR_INVALID;
  if (kv->dtype == TW_BF16)
    return launch_estimate<__nv_bfloat16>(kv, (const __nv_bfloat16*)q, buf, ss, swin, tm, exact, stream);
  return launch_estimate<float>(kv, (const float*)q, buf, ss, swin, tm, exact, stream);
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
