// K2 + K3 fused per unit: one CTA per unit (sequence, KV head) runs, back to
// back and on its own unit only,
//
//   A  the K1 append of the unit's new row (fused decode step) and the Quest
//      filter: the unit's page metadata streamed through per-warp cp.async
//      rings, fp32 page bounds on tensor cores            (selectors.py:97-109)
//   B  the exact page top-k per query head + GQA union    (selectors.py:112-132,
//      :178-186; select_body.cuh), or every page for the full selector (:90-94)
//   C  the INT4 estimate over the union's pages, all G heads from one read of
//      the codes                                          (quantcache.py:238-272)
//   D  softmax + top-p per head + group union + work items (pruner.py:57-114,
//      pipeline.py:341-347; topp_body.cuh)
//
// Why one CTA per unit: the separate kernels of the same stages are each
// bound by a per-unit latency chain (select, top-p) or by work-item boundaries
// of persistent warps (filter, estimate), and each launch drains the GPU.  Here
// every phase streams one unit's blocks with no item boundaries (16 warps,
// 3-stage rings, ~128 KB in flight per SM: tools/unit_stream_bench.cu measures
// 5.4-5.8 TB/s for this pattern with 128 CTAs), units drift out of phase so one
// CTA's select / top-p chain overlaps other CTAs' streams, and the page scores
// and logits make a round trip through L2 only.  The per-unit results are
// bit-identical to the separate kernels': the same select and top-p bodies,
// the same integer-exact estimate.
#include "estimate_body.cuh"
#include "quant_row.cuh"
#include "select_body.cuh"
#include "topp_body.cuh"

#ifdef TW_UNIT_TRACE
static __device__ unsigned long long g_ut[4096][8];
#define UT(ph)                                                                                       \
  do {                                                                                               \
    if (threadIdx.x == 0 && blockIdx.x < 4096) {                                                     \
      unsigned long long now_;                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_));                                      \
      g_ut[blockIdx.x][ph] = now_;                                                                   \
    }                                                                                                \
  } while (0)
extern "C" int tw_debug_utrace(unsigned long long* host_out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, g_ut, sizeof(g_ut));
  static unsigned long long zeros[4096 * 8];
  cudaMemcpyToSymbol(g_ut, zeros, sizeof(zeros));
  return 0;
}
#else
#define UT(ph) do {} while (0)
#endif
#ifdef TW_TOPP_TRACE
extern "C" int tw_debug_unit_ttrace(unsigned long long* host_out) {  // the top-p body's phase stamps in this kernel
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, tw::g_tt, sizeof(tw::g_tt));
  static unsigned long long zeros[1024 * 8];
  cudaMemcpyToSymbol(tw::g_tt, zeros, sizeof(zeros));
  return 0;
}
extern "C" int tw_debug_unit_strace(unsigned long long* host_out) {  // the select body's phase stamps
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, g_strace, sizeof(g_strace));
  int zeros[512] = {0};
  cudaMemcpyToSymbol(g_strace_phase, zeros, sizeof(zeros));
  static unsigned long long z2[512 * 16];
  cudaMemcpyToSymbol(g_strace, z2, sizeof(z2));
  return 0;
}
#endif

namespace tw {

constexpr int kUnitThreads = 1024;  // one CTA per SM: 32 warps stream, 4 x 256-thread groups select
constexpr int kUnitWarps = kUnitThreads / 32;
// phase A: per-warp ring of 4-page tiles (512 B of bf16 lo|hi per page, rows padded to
// 528 B so the ldmatrix rows of a tile fall in different banks)
constexpr int kUfTile = 4, kUfStages = 3, kUfRow = 528;
constexpr size_t kUfRing = (size_t)kUfStages * kUfTile * kUfRow;  // per warp
// phase C: per-warp ring of 2-page tiles of 1152-B INT4 blocks
constexpr int kUeTile = 2, kUeStages = 3;
constexpr size_t kUeRing = (size_t)kUeStages * kUeTile * kQBlockBytes;  // per warp
constexpr int kRingStages = 3;  // mbarriers per warp (both phases)

// top-p histogram batch and warp-group size per group size: UnitCfg<G, HB, GT>::NT == 1024
template <int G> struct UnitHB { static constexpr int value = G == 1 ? 1 : G == 2 ? 2 : 4; };
template <int G> struct UnitGT { static constexpr int value = G == 1 ? 1024 : 0; };

__device__ __forceinline__ void ldsm_x4_u(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma_bf16_u(float (&c)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

// ---------------------------------------------------------------- per-warp page streams
// Each warp streams a contiguous run [lo, hi) of one unit's pages through a
// ring of mbarrier-tracked stages filled by TMA bulk copies (cp.async.bulk:
// one instruction per page, issued by the lane that holds the page's address,
// so the issue cost is a few instructions per tile instead of one LDGSTS per
// 16 bytes per lane).  Page addresses come in batches of 32 (one per lane),
// the next batch's loads in flight while the current one is used.
__device__ __forceinline__ void ring_init(uint64_t* bars) {
  const int lane = threadIdx.x & 31;
  if (lane < kRingStages) mbar_init(bars + lane, 1);
  mbar_fence_init();
  __syncwarp();
}

// ---------------------------------------------------------------- phase A: Quest filter
// The bound is linear in the metadata row (lo | hi): score = qneg . lo + qpos . hi.
// The G query rows are the MMA's A operand (rows >= G are zero; fragments in
// shared memory, the same for every warp) and a tile's pages its N columns
// (B = the metadata rows via ldmatrix; columns >= kUfTile repeat): 16 k-steps
// of m16n8k16 per tile.  bf16 products are exact in fp32; the select's margin
// covers the fp32 sum.
template <int G>
__device__ __forceinline__ void unit_filter(const int unit, const int b, const int h, const int P,
                                            const tw_paged_kv& kv, const __nv_bfloat16* __restrict__ q,
                                            float* __restrict__ scores, unsigned char* sm, uint2* s_qa,
                                            uint64_t* bars) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane & 3, r = lane >> 2;
  uint8_t* R = sm + (size_t)warp * kUfRing;
  // A fragments: s_qa[kk][lane] = row r (head), k = 16kk + {2t, 2t+1} | + 8
  if (warp < 16) {
    const int kk = warp;
    const uint32_t* qw = reinterpret_cast<const uint32_t*>(q + ((size_t)unit * G + (r < G ? r : 0)) * kHeadDim);
    const __nv_bfloat162 zero2 = __float2bfloat162_rn(0.f);
    uint32_t w2[2];
#pragma unroll
    for (int hb = 0; hb < 2; ++hb) {
      const uint32_t w = r < G ? __ldg(qw + 8 * (kk & 7) + 4 * hb + t) : 0u;
      const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&w);
      const __nv_bfloat162 x = kk < 8 ? __hmin2(v, zero2) : __hmax2(v, zero2);  // lo channels: qneg, hi: qpos
      w2[hb] = *reinterpret_cast<const uint32_t*>(&x);
    }
    s_qa[kk * 32 + lane] = make_uint2(w2[0], w2[1]);
  }
  ring_init(bars);
  __syncthreads();
  const int* pt = kv.page_table + (size_t)b * kv.max_pages;
  const uint8_t* meta = reinterpret_cast<const uint8_t*>(kv.kmeta);
  const int H = kv.num_kv_heads;
  const int per = (P + kUnitWarps - 1) / kUnitWarps;
  const int lo = min(P, warp * per), np = min(P, lo + per) - lo;
  const int my = (np + kUfTile - 1) / kUfTile;
  int ph_cur = lane < np ? __ldg(pt + lo + lane) : 0;
  int ph_nxt = 32 + lane < np ? __ldg(pt + lo + 32 + lane) : 0;
  int ib = 0;
  auto issue = [&](int j) {
    const int i0 = j * kUfTile, st = j % kUfStages;
    if ((i0 >> 5) != ib) {
      ib = i0 >> 5;
      ph_cur = ph_nxt;
      const int nx = 32 * (ib + 1) + lane;
      ph_nxt = nx < np ? __ldg(pt + lo + nx) : 0;
    }
    const int cnt = min(kUfTile, np - i0);
    if (lane == 0) mbar_arrive_expect_tx(bars + st, cnt * 512);
    __syncwarp();
    const int x = lane - (i0 & 31);
    if (x >= 0 && x < cnt)
      bulk_g2s(R + (st * kUfTile + x) * kUfRow, meta + ((size_t)ph_cur * H + h) * 512, 512, bars + st);
  };
#pragma unroll
  for (int s = 0; s < kUfStages - 1; ++s)
    if (s < my) issue(s);
  const size_t srow = (size_t)kv.max_pages;
  const int m = lane >> 3, row = lane & (kUfTile - 1);  // ldmatrix: matrix m = chunk 4kk2 + m; rows >= kUfTile repeat
  for (int j = 0; j < my; ++j) {
    if (j + kUfStages - 1 < my) issue(j + kUfStages - 1);
    mbar_wait(bars + j % kUfStages, (j / kUfStages) & 1);
    const uint8_t* tile = R + (j % kUfStages) * kUfTile * kUfRow;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk2 = 0; kk2 < 8; ++kk2) {
      uint32_t bf[4];
      ldsm_x4_u(bf, tile + row * kUfRow + (4 * kk2 + m) * 16);
      const uint2 a0 = s_qa[(2 * kk2) * 32 + lane], a1 = s_qa[(2 * kk2 + 1) * 32 + lane];
      mma_bf16_u(acc, a0.x, a0.y, bf[0], bf[1]);
      mma_bf16_u(acc, a1.x, a1.y, bf[2], bf[3]);
    }
    __syncwarp();  // the stage is read: it may be refilled
    const int p = lo + j * kUfTile + 2 * t;  // c0, c1: head r, pages 2t, 2t+1 (t < 2 real)
    if (r < G && 2 * t < kUfTile) {
      float* so = scores + ((size_t)unit * G + r) * srow;
      if (p < lo + np) so[p] = acc[0];
      if (p + 1 < lo + np) so[p + 1] = acc[1];
    }
  }
}

// ---------------------------------------------------------------- phase C: INT4 estimate
// Warp w streams a contiguous run of the unit's candidate pages (2-page tiles,
// 3-stage TMA ring); per page the packed-digit integer MMAs of estimate.cu
// (G <= 4), logits for rows r, r + 8 of head t.
template <int G>
__device__ __forceinline__ void unit_estimate(const int unit, const int b, const int h, const int n, const int ncand,
                                              const tw_paged_kv& kv, const __nv_bfloat16* __restrict__ q,
                                              const tw_decode_buffers& buf, unsigned char* sm, uint32_t* s_hmax,
                                              uint64_t* bars, int* s_lp) {
  static_assert(G <= 4, "packed digits");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane & 3, r = lane >> 2;
  uint8_t* R = sm + (size_t)warp * kUeRing;
  const int T_stride = kv.max_pages * kPage;
  const float inv_sqrt_d = 0.08838834764831845f;  // float32(1/sqrt(128)), as quantcache.py:258
  const int* cand = buf.cand_pages + (size_t)unit * kv.max_pages;
  const int* pt = kv.page_table + (size_t)b * kv.max_pages;
  const int H = kv.num_kv_heads;
  ring_init(bars);
  const int per = (ncand + kUnitWarps - 1) / kUnitWarps;
  const int lo = min(ncand, warp * per), np = min(ncand, lo + per) - lo;
  const int my = (np + kUeTile - 1) / kUeTile;
  int lp_cur = lane < np ? __ldcg(cand + lo + lane) : 0;
  int lp_nxt = 32 + lane < np ? __ldcg(cand + lo + 32 + lane) : 0;
  int ph_cur = lane < np ? __ldg(pt + lp_cur) : 0;
  int ib = 0;
  uint32_t pb1[4][2], pb2[4][2];
  float sq, isc;
  estimate_prologue_packed<__nv_bfloat16, G, 4>(q, unit, pb1, pb2, sq, isc);
  int* lps = s_lp + warp * kRingStages * kUeTile;
  auto issue = [&](int j) {
    const int i0 = j * kUeTile, st = j % kUeStages;
    if ((i0 >> 5) != ib) {
      ib = i0 >> 5;
      lp_cur = lp_nxt;
      ph_cur = 32 * ib + lane < np ? __ldg(pt + lp_cur) : 0;
      const int nx = 32 * (ib + 1) + lane;
      lp_nxt = nx < np ? __ldcg(cand + lo + nx) : 0;
    }
    const int cnt = min(kUeTile, np - i0);
    if (lane == 0) mbar_arrive_expect_tx(bars + st, cnt * kQBlockBytes);
    __syncwarp();
    const int x = lane - (i0 & 31);
    if (x >= 0 && x < cnt) {
      bulk_g2s(R + (st * kUeTile + x) * kQBlockBytes, kv.kq + ((size_t)ph_cur * H + h) * kQBlockBytes, kQBlockBytes,
               bars + st);
      lps[st * kUeTile + x] = lp_cur;
    }
  };
#pragma unroll
  for (int s = 0; s < kUeStages - 1; ++s)
    if (s < my) issue(s);
  float run_max = -INFINITY;
  float* lg_head = buf.logits + ((size_t)unit * G + (t < G ? t : 0)) * T_stride + r;
  for (int j = 0; j < my; ++j) {
    if (j + kUeStages - 1 < my) issue(j + kUeStages - 1);
    const int st = j % kUeStages;
    mbar_wait(bars + st, (j / kUeStages) & 1);
    __syncwarp();  // the issuing lanes' page ids
    const uint8_t* stage = R + st * kUeTile * kQBlockBytes;
    const int c0 = lo + j * kUeTile;
    const int cnt = min(kUeTile, np - j * kUeTile);
#pragma unroll
    for (int i = 0; i < kUeTile; ++i) {
      if (i < cnt) {
        const uint8_t* pg = stage + i * kQBlockBytes;
        const uint4 lo4 = *reinterpret_cast<const uint4*>(pg + r * 64 + t * 16);
        const uint4 hi4 = *reinterpret_cast<const uint4*>(pg + (r + 8) * 64 + t * 16);
        const uint32_t wl[4] = {lo4.x, lo4.y, lo4.z, lo4.w}, wh[4] = {hi4.x, hi4.y, hi4.z, hi4.w};
        const float* prm = reinterpret_cast<const float*>(pg + kCodeBytes);
        const float sc_r = prm[r], sc_r8 = prm[r + 8], z_r = prm[16 + r], z_r8 = prm[24 + r];
        const int lp = lps[st * kUeTile + i];
        int acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const uint32_t a[4] = {wl[jj] & 0x0F0F0F0Fu, wh[jj] & 0x0F0F0F0Fu, (wl[jj] >> 4) & 0x0F0F0F0Fu,
                                 (wh[jj] >> 4) & 0x0F0F0F0Fu};
          mma_u8s8(acc[0], a, pb1[jj][0], pb1[jj][1]);
          mma_u8s8(acc[1], a, pb2[jj][0], pb2[jj][1]);
        }
        const float d0 = fmaf((float)acc[1][0], 65536.f, fmaf((float)acc[0][1], 256.f, (float)acc[0][0])) * isc;
        const float d2 = fmaf((float)acc[1][2], 65536.f, fmaf((float)acc[0][3], 256.f, (float)acc[0][2])) * isc;
        const int tok_r = lp * kPage + r;
        const float l0 = tok_r < n ? fmaf(sc_r, d0, z_r * sq) * inv_sqrt_d : -INFINITY;
        const float l1 = tok_r + 8 < n ? fmaf(sc_r8, d2, z_r8 * sq) * inv_sqrt_d : -INFINITY;
        if (t < G) {
          float* lg = lg_head + (size_t)(c0 + i) * kPage;
          lg[0] = l0;
          lg[8] = l1;
          run_max = fmaxf(run_max, fmaxf(l0, l1));
        }
      }
    }
    __syncwarp();  // the stage is read: it may be refilled
  }
  run_max = fmaxf(run_max, __shfl_xor_sync(0xffffffffu, run_max, 4));
  run_max = fmaxf(run_max, __shfl_xor_sync(0xffffffffu, run_max, 8));
  run_max = fmaxf(run_max, __shfl_xor_sync(0xffffffffu, run_max, 16));
  if (r == 0 && t < G && run_max > -INFINITY) atomicMax(s_hmax + t, f2key(run_max));
}

// ---------------------------------------------------------------- the fused kernel
// SELECT_ONLY: phases A + B only (K1 + K2: the candidate pages), for the
// separate estimate / top-p kernels.
template <int G, bool SB, bool SELECT_ONLY = false>
__global__ void __launch_bounds__(kUnitThreads, 1) unit_step_kernel(tw_paged_kv kv, const __nv_bfloat16* __restrict__ q,
                                                                    tw_decode_params prm, tw_decode_buffers buf,
                                                                    const __nv_bfloat16* __restrict__ k_new,
                                                                    const __nv_bfloat16* __restrict__ v_new,
                                                                    const int32_t* positions) {
  extern __shared__ __align__(128) unsigned char usm[];
  __shared__ uint32_t s_hmax[G];
  __shared__ int s_ncand;
  __shared__ __align__(8) uint64_t s_bars[2][kUnitWarps][kRingStages];  // filter | estimate rings
  __shared__ int s_lp[kUnitWarps * kRingStages * kUeTile];
  const int unit = blockIdx.x;
  const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int n;
  if (positions) {
    const int pos = __ldg(positions + b);
    n = min(pos + 1, kv.max_pages * kPage);
  } else {
    n = kv.seq_lens[b];
  }
  const int P = (n + kPage - 1) / kPage;
  UT(0);
  if ((int)threadIdx.x < G) s_hmax[threadIdx.x] = 0u;
  if (prm.selector == TW_SELECT_QUEST) {
    // K1: the warp that streams the open page appends the new row to it first
    const int per = (P + kUnitWarps - 1) / kUnitWarps;
    if (positions && P > 0 && warp == (P - 1) / per) {
      append_row_warp<__nv_bfloat16, 4>(kv, b, h, lane, k_new, v_new, n - 1);
      if (h == 0 && lane == 0 && __ldg(positions + b) < kv.max_pages * kPage) kv.seq_lens[b] = n;
      __threadfence();  // the row's metadata precedes this warp's TMA reads of the page
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __syncwarp();
    }
    // the A fragments sit behind the filter's rings (both dead after phase A)
    unit_filter<G>(unit, b, h, P, kv, q, buf.page_scores, usm,
                   reinterpret_cast<uint2*>(usm + kUfRing * kUnitWarps), s_bars[0][warp]);
  } else if (positions && warp == 0) {
    append_row_warp<__nv_bfloat16, 4>(kv, b, h, lane, k_new, v_new, n - 1);
    if (h == 0 && lane == 0 && __ldg(positions + b) < kv.max_pages * kPage) kv.seq_lens[b] = n;
    __threadfence();
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  __syncthreads();
  UT(1);
  select_unit_body<__nv_bfloat16, kUnitThreads>(unit, kv, q, prm, buf, usm, n);
  if constexpr (SELECT_ONLY) return;
  __syncthreads();
  UT(2);
  if (threadIdx.x == 0) s_ncand = buf.cand_count[unit];
  __syncthreads();
  unit_estimate<G>(unit, b, h, n, s_ncand, kv, q, buf, usm, s_hmax, s_bars[1][warp], s_lp);
  __syncthreads();
  UT(3);
  if ((int)threadIdx.x < G) buf.head_max[(size_t)unit * G + threadIdx.x] = s_hmax[threadIdx.x];
  __syncthreads();
  topp_unit_body<G, UnitHB<G>::value, SB, UnitGT<G>::value>(unit, kv, prm, buf, usm);
  UT(4);
}

inline size_t unit_select_smem_bytes(int max_pages) {
  return std::max<size_t>(kUfRing * kUnitWarps + 16 * 32 * sizeof(uint2), select_smem_bytes(max_pages, kUnitThreads));
}

template <int G>
inline size_t unit_smem_bytes(int max_pages) {
  size_t s = std::max<size_t>(kUfRing * kUnitWarps + 16 * 32 * sizeof(uint2), kUeRing * kUnitWarps);
  s = std::max(s, select_smem_bytes(max_pages, kUnitThreads));
  s = std::max(s, UnitCfg<G, UnitHB<G>::value, UnitGT<G>::value>::kSmem);
  return s;
}

}  // namespace tw

using namespace tw;

static int unit_min_units() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("TW_UNIT_MIN");
    v = e ? atoi(e) : 64;
  }
  return v;
}

// 1 when the fused per-unit kernel covers this step's geometry and options.
int tw_unit_step_applies(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
                         const int32_t* positions) {
  const char* e = getenv("TW_UNIT");  // opt-in until it beats the separate kernels at every config
  if (!e || atoi(e) == 0) return 0;
  if (!kv || !prm || !buf || kv->dtype != TW_BF16 || kv->head_dim != kHeadDim || (kv->bits != 0 && kv->bits != 4))
    return 0;
  if (prm->estimator != TW_ESTIMATE_INT || prm->renormalize != 1) return 0;
  if (prm->selector != TW_SELECT_QUEST && prm->selector != TW_SELECT_FULL) return 0;
  if (prm->selector == TW_SELECT_QUEST && (prm->budget_pages < 1 || !buf->page_scores || !buf->band_idx ||
                                           !buf->band_scores))
    return 0;
  const int G = kv->group_size;
  if (G != 1 && G != 2 && G != 4) return 0;
  if (kv->num_seqs * kv->num_kv_heads < unit_min_units()) return 0;
  if (positions && positions == kv->seq_lens) return 0;  // every CTA of a sequence must see the same position
  if ((long long)kv->max_pages * kPage > (1ll << 24)) return 0;
  size_t smem = 0;
  switch (G) {
    case 1: smem = unit_smem_bytes<1>(kv->max_pages); break;
    case 2: smem = unit_smem_bytes<2>(kv->max_pages); break;
    default: smem = unit_smem_bytes<4>(kv->max_pages); break;
  }
  if (smem + 4096 > 227 * 1024) return 0;
  if (!buf->cand_pages || !buf->cand_count || !buf->logits || !buf->head_max || !buf->head_thr ||
      !buf->head_stats || !buf->final_idx || !buf->final_count || !buf->unit_items || !buf->work_items ||
      !buf->counters || !buf->sel_bits)
    return 0;
  return 1;
}

extern "C" int32_t tw_select_estimate_topp_applies(const tw_paged_kv* kv, const tw_decode_params* prm,
                                                   const tw_decode_buffers* buf) {
  return tw_unit_step_applies(kv, prm, buf, nullptr);
}

template <int G, bool SB>
static int launch_unit_step(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                            const int32_t* positions, const tw_decode_params* prm, const tw_decode_buffers* buf,
                            cudaStream_t stream) {
  const size_t smem = unit_smem_bytes<G>(kv->max_pages);
  auto kern = unit_step_kernel<G, SB>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return TW_ERR_CUDA;
  cudaMemsetAsync(buf->counters, 0, 8 * sizeof(uint32_t), stream);
  kern<<<kv->num_seqs * kv->num_kv_heads, kUnitThreads, smem, stream>>>(
      *kv, (const __nv_bfloat16*)q, *prm, *buf, (const __nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new, positions);
  return launch_status();
}

template <int G>
static int launch_unit_step_g(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                              const int32_t* positions, const tw_decode_params* prm, const tw_decode_buffers* buf,
                              cudaStream_t stream) {
  const size_t words = ((size_t)kv->max_pages * kPage + 31) / 32;
  if (words <= UnitCfg<G, UnitHB<G>::value, UnitGT<G>::value>::kBitsCap)
    return launch_unit_step<G, true>(kv, q, k_new, v_new, positions, prm, buf, stream);
  return launch_unit_step<G, false>(kv, q, k_new, v_new, positions, prm, buf, stream);
}

// K1 (when positions is given) + K2 in one per-unit launch: the Quest filter
// streamed by the unit's CTA and its page selection (phases A + B above), for
// the separate estimate and top-p kernels.  Returns TW_FUSE_UNAVAILABLE when
// the geometry is not covered (nothing launched).
int tw_unit_select(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                   const int32_t* positions, const tw_decode_params* prm, const tw_decode_buffers* buf,
                   cudaStream_t stream) {
  const char* e = getenv("TW_USELECT");  // opt-in: measured no faster than quest_filter + quest_select (r02)
  if (!e || atoi(e) == 0) return TW_FUSE_UNAVAILABLE;
  if (!kv || !prm || !buf || !q || kv->dtype != TW_BF16 || kv->head_dim != kHeadDim ||
      (kv->bits != 0 && kv->bits != 4) || prm->selector != TW_SELECT_QUEST || prm->budget_pages < 1 ||
      !buf->page_scores || !buf->band_idx || !buf->band_scores || !buf->cand_pages || !buf->cand_count ||
      !buf->counters || !buf->head_max || (positions && (!k_new || !v_new || positions == kv->seq_lens)))
    return TW_FUSE_UNAVAILABLE;
  const int G = kv->group_size;
  if (G != 1 && G != 2 && G != 4) return TW_FUSE_UNAVAILABLE;
  const size_t smem = unit_select_smem_bytes(kv->max_pages);
  if (smem + 4096 > 227 * 1024) return TW_FUSE_UNAVAILABLE;
  auto go = [&](auto kern) -> int {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return TW_ERR_CUDA;
    cudaMemsetAsync(buf->counters, 0, 8 * sizeof(uint32_t), stream);
    kern<<<kv->num_seqs * kv->num_kv_heads, kUnitThreads, smem, stream>>>(
        *kv, (const __nv_bfloat16*)q, *prm, *buf, (const __nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new,
        positions);
    return launch_status();
  };
  switch (G) {
    case 1: return go(unit_step_kernel<1, false, true>);
    case 2: return go(unit_step_kernel<2, false, true>);
    default: return go(unit_step_kernel<4, false, true>);
  }
}

// K1 (when positions is given) + K2 + K3 of one decode step in one launch.
extern "C" int tw_select_estimate_topp(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                                       const int32_t* positions, const tw_decode_params* prm,
                                       const tw_decode_buffers* buf, cudaStream_t stream) {
  if (!kv || !prm || !buf || !q || (positions && (!k_new || !v_new))) return TW_ERR_INVALID;
  if (!(prm->p >= 0.0 && prm->p <= 1.0)) return TW_ERR_INVALID;
  if (!tw_unit_step_applies(kv, prm, buf, positions)) return TW_ERR_INVALID;
  switch (kv->group_size) {
    case 1: return launch_unit_step_g<1>(kv, q, k_new, v_new, positions, prm, buf, stream);
    case 2: return launch_unit_step_g<2>(kv, q, k_new, v_new, positions, prm, buf, stream);
    default: return launch_unit_step_g<4>(kv, q, k_new, v_new, positions, prm, buf, stream);
  }
}
