// K2: Quest page bounds, exact page top-k per query head, GQA union.
//
// Reference (pkg/src/nucleuskv/selectors.py):
//   quest_page_scores :97-109   score_p = sum_c max(q_c lo_c, q_c hi_c) / sqrt(d)  (fp64)
//   select_quest      :112-132  k = min(ceil(n/16), ceil(B0/16)) pages, stable
//                               argsort(-score) -> ties go to the lower page
//   group_union       :178-186  sorted union over the G query heads (pipeline.py:338)
//
// Exactness without an fp64 scan of every page: the HBM-bound filter pass
// computes fp32 bounds with a rigorous error bound m (products of bf16 values
// are exact in fp32; the 128-term sum errs by at most ~128 u sum|t|, and
// sum|t| <= ||q||_1 * max|k| of the unit).  The select pass finds the k-th
// largest fp32 bound t; pages above t + 2m are certainly in, below t - 2m
// certainly out, and only the thin band between is rescored in fp64 with
// NumPy's exact summation order (8 strided partial sums, then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), see oracle.numpy_rowsum_order) and
// ranked by (score desc, page asc).  The result is the reference's page set.
#include "block_scan.cuh"
#include "quant_row.cuh"

#include "select_body.cuh"
#ifdef TW_TOPP_TRACE
extern "C" int tw_debug_strace(unsigned long long* host_out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, g_strace, sizeof(g_strace));
  int zeros[512] = {0};
  cudaMemcpyToSymbol(g_strace_phase, zeros, sizeof(zeros));
  return 0;
}
#endif

namespace tw {

#ifndef TW_QF_ITEM
#define TW_QF_ITEM 64
#endif
constexpr int kFilterPagesPerCta = TW_QF_ITEM;  // largest filter item (<= 64: two pages per lane)

// ---------------------------------------------------------------- filter pass

// Persistent warp workers over (unit, 16..64-page) items, chunk-major.  Each warp
// streams its pages' metadata (lo|hi, 512 B in bf16) through a 4-stage
// cp.async ring of 2-page stages; a half-warp scores one page (16 lanes x 8
// channels) for all G heads and reduces with shuffles.
constexpr int kQfWarps = 4;
constexpr int kQfStages = 4;

template <typename T, int G>
__global__ void __launch_bounds__(kQfWarps * 32) quest_filter_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                                     float* __restrict__ scores, int max_chunks,
                                                                     uint32_t* __restrict__ ctr, int item) {
  __shared__ __align__(128) T ring[kQfWarps][kQfStages][2][2 * kHeadDim];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sub = lane & 15, half = lane >> 4;
  const int units = kv.num_seqs * kv.num_kv_heads;
  constexpr int kPageBytes = 2 * kHeadDim * sizeof(T);
  constexpr int kChunks = kPageBytes / 16;  // 32 (bf16) or 64 (fp32) per page
  T (*R)[2][2 * kHeadDim] = ring[warp];
  float qr[G][8];
  int cur_unit = -1;
  for (int it = warp_fetch(ctr); it < units * max_chunks; it = warp_fetch(ctr)) {
    const int unit = it % units;
    const int p0 = (it / units) * item;
    const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
    const int npages = (kv.seq_lens[b] + kPage - 1) / kPage;
    if (p0 >= npages) continue;
    const int np = min(item, npages - p0);
    const int* pt = kv.page_table + (size_t)b * kv.max_pages;
    // physical metadata blocks of pages p0 + lane and p0 + 32 + lane
    const T* src0 = reinterpret_cast<const T*>(kv.kmeta);
    const T* src1 = src0;
    if (lane < np) src0 += ((size_t)pt[p0 + lane] * kv.num_kv_heads + h) * 2 * kHeadDim;
    if (lane + 32 < np) src1 += ((size_t)pt[p0 + 32 + lane] * kv.num_kv_heads + h) * 2 * kHeadDim;
    const int nst = (np + 1) / 2;
    auto issue = [&](int s) {
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int pg = 2 * s + j;
        if (pg < np) {
          const T* src = reinterpret_cast<const T*>(
              __shfl_sync(0xffffffffu, (unsigned long long)(pg < 32 ? src0 : src1), pg & 31));
          char* dst = reinterpret_cast<char*>(&R[s % kQfStages][j][0]);
#pragma unroll
          for (int c = lane; c < kChunks; c += 32)
            cp_async16(dst + 16 * c, reinterpret_cast<const char*>(src) + 16 * c);
        }
      }
    };
#pragma unroll
    for (int s = 0; s < kQfStages - 1; ++s) {
      if (s < nst) issue(s);
      cp_commit();
    }
    if (unit != cur_unit) {
#pragma unroll
      for (int g = 0; g < G; ++g) load8(q + ((size_t)unit * G + g) * kHeadDim + 8 * sub, qr[g]);
      cur_unit = unit;
    }
    for (int s = 0; s < nst; ++s) {
      if (s + kQfStages - 1 < nst) issue(s + kQfStages - 1);
      cp_commit();
      cp_wait<kQfStages - 1>();
      __syncwarp();
      const int pg = 2 * s + half;
      float l8[8], h8[8];
      load8(&R[s % kQfStages][half][8 * sub], l8);
      load8(&R[s % kQfStages][half][kHeadDim + 8 * sub], h8);
      __syncwarp();
      float acc[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float a = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) a = fmaf(qr[g][i], qr[g][i] >= 0.f ? h8[i] : l8[i], a);
        acc[g] = a;
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1)
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] += __shfl_xor_sync(0xffffffffu, acc[g], o);
      if (sub < G && pg < np) {
        float v = acc[0];
#pragma unroll
        for (int g = 1; g < G; ++g) if (sub == g) v = acc[g];
        scores[((size_t)unit * G + sub) * kv.max_pages + p0 + pg] = v;
      }
    }
    cp_wait<0>();
  }
}

// bf16 metadata: the bound is linear in the metadata row (lo | hi):
//   score = qneg . lo + qpos . hi,  qpos = max(q, 0), qneg = min(q, 0),
// i.e. a [pages x 256] x [256 x heads] product -> legacy mma.sync m16n8k16
// (bf16 products exact, fp32 accumulation, covered by the select margin).
// Per warp: 16-page tiles through a TW_QM_STAGES-deep (2) ring of TMA bulk
// copies (below); one ldmatrix.x4 + one MMA per page-tile k-step.
#ifndef TW_QM_STAGES
#define TW_QM_STAGES 2
#endif
constexpr int kQmStages = TW_QM_STAGES;
constexpr int kQmTile = 16;  // pages per stage (= the MMA's rows)
// Every page is ONE TMA bulk copy (cp.async.bulk, issued by the lane holding
// its address) into a row padded to 528 B (bulk copies cannot swizzle; the pad
// keeps ldmatrix's 8 rows in different banks), completing on a per-stage
// mbarrier (measured: C2 K2 49.4 -> 48.8 us, step 282.5 -> 280.5 us; C4 K2
// 246 -> 237 us).  TW_QF_BULK=0: 32 LDGSTS of 16 B per page into swizzled rows.
#ifndef TW_QF_BULK
#define TW_QF_BULK 1
#endif
constexpr int kQmRow = TW_QF_BULK ? 528 : 512;
constexpr int kQmStageBytes = kQmTile * kQmRow;

__device__ __forceinline__ void ldsm_x4_q(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma_bf16_q(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// With `positions` (the fused decode step) the warp whose item holds a unit's
// open page first appends that unit's new row (K1, append_row_warp) and then
// streams the page's updated metadata; page counts come from positions + 1.
template <int G>
__global__ void __launch_bounds__(kQfWarps * 32) quest_filter_mma_kernel(tw_paged_kv kv,
                                                                         const __nv_bfloat16* __restrict__ q,
                                                                         float* __restrict__ scores, int max_chunks,
                                                                         uint32_t* __restrict__ ctr, int item,
                                                                         const __nv_bfloat16* __restrict__ k_new,
                                                                         const __nv_bfloat16* __restrict__ v_new,
                                                                         const int32_t* positions) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) uint8_t qm_ring[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = lane & 3, r = lane >> 2, q8 = lane >> 3, rr = lane & 7;
  const int units = kv.num_seqs * kv.num_kv_heads;
  uint8_t (*R)[kQmStageBytes] =
      reinterpret_cast<uint8_t (*)[kQmStageBytes]>(qm_ring + (size_t)warp * kQmStages * kQmStageBytes);
#if TW_QF_BULK
  __shared__ __align__(8) uint64_t qbars[kQfWarps][kQmStages];
  if (lane < kQmStages) mbar_init(&qbars[warp][lane], 1);
  mbar_fence_init();
  __syncwarp();
  uint32_t issued = 0;  // tiles this warp has issued: tile j of all items uses slot j % stages, parity (j / stages) & 1
#endif
  uint32_t qb[16][2];  // B fragments of [qneg ; qpos] for head column r
  int cur_unit = -1;
  for (int it = warp_fetch(ctr); it < units * max_chunks; it = warp_fetch(ctr)) {
    const int unit = it % units;
    // chunks in reverse order: the item holding the open page (the append, a
    // latency chain) is taken first instead of last
    const int p0 = (max_chunks - 1 - it / units) * item;
    const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
    const int pos = positions ? __ldg(positions + b) : -1;
    const int n = positions ? min(pos + 1, kv.max_pages * kPage) : kv.seq_lens[b];
    const int npages = (n + kPage - 1) / kPage;
    if (p0 >= npages) continue;
    const int np = min(item, npages - p0);
    if (positions && npages - 1 < p0 + np) {  // this item holds the open page: append first
      switch (kv.bits) {
        case 2: append_row_warp<__nv_bfloat16, 2>(kv, b, h, lane, k_new, v_new, pos); break;
        case 8: append_row_warp<__nv_bfloat16, 8>(kv, b, h, lane, k_new, v_new, pos); break;
        default: append_row_warp<__nv_bfloat16, 4>(kv, b, h, lane, k_new, v_new, pos); break;
      }
      if (h == 0 && lane == 0 && pos < kv.max_pages * kPage)
        kv.seq_lens[b] = n;  // every reader in this kernel uses positions
      __threadfence();  // the metadata stores precede this warp's cp.async reads of the page
#if TW_QF_BULK
      asm volatile("fence.proxy.async.global;" ::: "memory");  // ... and its bulk (async-proxy) reads
#endif
      __syncwarp();
    }
    const int* pt = kv.page_table + (size_t)b * kv.max_pages;
    const uint8_t* base = reinterpret_cast<const uint8_t*>(kv.kmeta);
    const uint8_t* src0 = base;
    const uint8_t* src1 = base;
    if (lane < np) src0 += ((size_t)pt[p0 + lane] * kv.num_kv_heads + h) * 512;
    if (lane + 32 < np) src1 += ((size_t)pt[p0 + 32 + lane] * kv.num_kv_heads + h) * 512;
    const int ntile = (np + kQmTile - 1) / kQmTile;
#if TW_QF_BULK
    const uint32_t tbase = issued;
    auto issue = [&](int s) {  // tile s = pages 16s .. 16s+15, held by lanes 16(s&1) + x of src0 (s < 2) / src1
      const uint32_t slot = (tbase + s) % kQmStages;
      const int cnt = min(kQmTile, np - kQmTile * s);
      if (lane == 0) mbar_arrive_expect_tx(&qbars[warp][slot], cnt * 512);
      __syncwarp();
      const int x = lane - 16 * (s & 1);
      if (x >= 0 && x < cnt) bulk_g2s(R[slot] + x * kQmRow, s >= 2 ? src1 : src0, 512, &qbars[warp][slot]);
    };
#pragma unroll
    for (int s = 0; s < kQmStages - 1; ++s)
      if (s < ntile) issue(s);
#else
    auto issue = [&](int s) {
      uint8_t* dst = R[s % kQmStages];
#pragma unroll 4
      for (int i = 0; i < kQmTile; ++i) {
        const int pg = kQmTile * s + i;
        if (pg < np) {
          const uint8_t* src = reinterpret_cast<const uint8_t*>(
              __shfl_sync(0xffffffffu, (unsigned long long)(pg < 32 ? src0 : src1), pg & 31));
          // 32 chunks of 16 B per row; chunk c stored at c ^ (i & 7)
          cp_async16(dst + i * 512 + ((lane ^ (i & 7)) << 4), src + 16 * lane);
        }
      }
    };
#pragma unroll
    for (int s = 0; s < kQmStages - 1; ++s) {
      if (s < ntile) issue(s);
      cp_commit();
    }
#endif
    if (unit != cur_unit) {
      // k = 16kk + {2t, 2t+1 | 2t+8, 2t+9}; k < 128 -> qneg[k], else qpos[k - 128]:
      // the bf16 pair (c, c+1), c = k & 127, is 32-bit word 8(kk & 7) + t + 4hb of the head's row
      const uint32_t* qw = reinterpret_cast<const uint32_t*>(q + ((size_t)unit * G + (r < G ? r : 0)) * kHeadDim);
      uint32_t w[8][2];
#pragma unroll
      for (int k8 = 0; k8 < 8; ++k8) {
        w[k8][0] = r < G ? __ldg(qw + 8 * k8 + t) : 0u;
        w[k8][1] = r < G ? __ldg(qw + 8 * k8 + t + 4) : 0u;
      }
      const __nv_bfloat162 zero2 = __float2bfloat162_rn(0.f);
#pragma unroll
      for (int k8 = 0; k8 < 8; ++k8) {
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {
          const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&w[k8][hb]);
          const __nv_bfloat162 neg = __hmin2(v, zero2), pos = __hmax2(v, zero2);
          qb[k8][hb] = *reinterpret_cast<const uint32_t*>(&neg);
          qb[k8 + 8][hb] = *reinterpret_cast<const uint32_t*>(&pos);
        }
      }
      cur_unit = unit;
    }
    for (int s = 0; s < ntile; ++s) {
      if (s + kQmStages - 1 < ntile) issue(s + kQmStages - 1);
#if TW_QF_BULK
      const uint32_t slot = (tbase + s) % kQmStages;
      mbar_wait(&qbars[warp][slot], ((tbase + s) / kQmStages) & 1);
      const uint8_t* tile = R[slot];
#else
      cp_commit();
      cp_wait<kQmStages - 1>();
      __syncwarp();
      const uint8_t* tile = R[s % kQmStages];
#endif
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      {
        const int row = (q8 & 1) * 8 + rr;
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          uint32_t a[4];
          const int chunk = 2 * kk + (q8 >> 1);
#if TW_QF_BULK
          ldsm_x4_q(a, tile + row * kQmRow + (chunk << 4));
#else
          ldsm_x4_q(a, tile + row * 512 + ((chunk ^ (row & 7)) << 4));
#endif
          mma_bf16_q(acc, a, qb[kk][0], qb[kk][1]);
        }
        __syncwarp();
        // rows r, r+8 (pages), cols 2t, 2t+1 (heads)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int pg = 16 * s + r + (e >= 2 ? 8 : 0);
          const int g = 2 * t + (e & 1);
          if (g < G && pg < np) scores[((size_t)unit * G + g) * kv.max_pages + p0 + pg] = acc[e];
        }
      }
    }
#if TW_QF_BULK
    issued = tbase + ntile;  // every issued tile was waited on above
#else
    cp_wait<0>();
#endif
  }
}

// tw_quest_scores: grid (ceil(max_pages/8), B*H_kv*G), 8 warps, warp per page.
template <typename T>
__global__ void __launch_bounds__(256) quest_exact_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                          double* __restrict__ out) {
  __shared__ double terms[8][kHeadDim];
  const int qh = blockIdx.y;  // global query head = unit * G + g
  const int G = kv.group_size;
  const int unit = qh / G;
  const int b = unit / kv.num_kv_heads, h = unit % kv.num_kv_heads;
  const int npages = (kv.seq_lens[b] + kPage - 1) / kPage;
  const int warp = threadIdx.x >> 5;
  const int lp = blockIdx.x * 8 + warp;
  if (lp >= kv.max_pages) return;
  double s = -INFINITY;
  if (lp < npages) {
    const int phys = kv.page_table[(size_t)b * kv.max_pages + lp];
    const T* lo = reinterpret_cast<const T*>(kv.kmeta) + ((size_t)phys * kv.num_kv_heads + h) * 2 * kHeadDim;
    s = exact_page_score<T>(q + (size_t)qh * kHeadDim, lo, lo + kHeadDim, terms[warp]);
  }
  if ((threadIdx.x & 31) == 0) out[(size_t)qh * kv.max_pages + lp] = s;
}

// NG < 4 (the C4/C5 shapes): two CTAs per SM (64 registers), so more units start at once.
template <typename T, int NG, int NT>
__global__ void __launch_bounds__(NT, NT == 512 && NG < 4 ? 2 : 1)
    quest_select_kernel(tw_paged_kv kv, const T* __restrict__ q, tw_decode_params prm, tw_decode_buffers buf) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char smem[];
  select_unit_body<T, NT, NG>(blockIdx.x, kv, q, prm, buf, smem);
}

}  // namespace tw

using namespace tw;

#ifdef TW_TOPP_TRACE
extern "C" int tw_debug_select_strace(unsigned long long* host_out) {  // quest_select_kernel's phase stamps
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, g_strace, sizeof(g_strace));
  int zeros[512] = {0};
  cudaMemcpyToSymbol(g_strace_phase, zeros, sizeof(zeros));
  static unsigned long long z2[512 * 16];
  cudaMemcpyToSymbol(g_strace, z2, sizeof(z2));
  return 0;
}
#endif

// Warp groups of the select CTA (query heads selected concurrently, 512 / ng
// threads each): up to 4, fewer when the unit has fewer heads, when the
// per-group key arrays would not fit shared memory, or when the smaller CTA
// (two per SM) needs fewer waves for all units.  Measured: C5 (256 units of
// 8193 pages) select 246.7 -> 230.7 us with 2 groups, C4 (512 units of 4097)
// 259.7 -> 236.9; C2 (128 units) keeps 4 (2 groups: 53.9 -> 56.8).
// 0: no configuration fits.  TW_SEL_GROUPS=1|2|4 pins it (A/B).
static int select_threads() {
  static const int nt = [] {
    const char* e = getenv("TW_SEL_THREADS");
    return e && atoi(e) == 1024 ? 1024 : kSelThreads;
  }();
  return nt;
}
static int select_groups(int units, int G, int Pmax, int sms, int nt) {
  static const int pinned = [] {
    const char* e = getenv("TW_SEL_GROUPS");
    return e ? atoi(e) : 0;
  }();
  auto fits = [&](int ng) { return select_smem_bytes(Pmax, nt, ng) <= 227 * 1024; };
  if (pinned == 1 || pinned == 2 || pinned == 4) return fits(pinned) ? pinned : 0;
  const int gmax = G >= 4 ? 4 : (G >= 2 ? 2 : 1);
  int ng = gmax;
  while (ng > 1 && !fits(ng)) ng /= 2;
  if (!fits(ng)) return 0;
  auto waves = [&](int g) {  // 4 groups: 1 CTA per SM (registers); fewer: 2
    const int per_sm = (int)std::min<size_t>(g == 4 || nt > 512 ? 1 : 2, (228 * 1024) / (select_smem_bytes(Pmax, nt, g) + 1024));
    return (units + sms * per_sm - 1) / (sms * per_sm);
  };
  while (ng > 1 && waves(ng / 2) < waves(ng)) ng /= 2;
  return ng;
}

template <typename T>
static int launch_select(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                         const tw_decode_buffers* buf, cudaStream_t stream, const void* k_new = nullptr,
                         const void* v_new = nullptr, const int32_t* positions = nullptr) {
  const int units = kv->num_seqs * kv->num_kv_heads;
  int dev0 = 0, sms0 = 148;
  cudaGetDevice(&dev0);
  cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0);
  const int nt = select_threads();
  const int ng = select_groups(units, kv->group_size, kv->max_pages, sms0, nt);
  if (ng == 0) return TW_ERR_INVALID;  // checked before anything is enqueued
  const size_t smem = select_smem_bytes(kv->max_pages, nt, ng);
  cudaMemsetAsync(buf->counters, 0, 8 * sizeof(uint32_t), stream);
  if (prm->selector == TW_SELECT_QUEST) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // item size: 64 pages, halved (to 16 at least) while units x chunks would leave warps idle
    int item = kFilterPagesPerCta;
    while (item > 16 && (long long)units * ((kv->max_pages + item - 1) / item) < (long long)sms * 3 * kQfWarps)
      item /= 2;
    const int max_chunks = (kv->max_pages + item - 1) / item;
    const int items = units * max_chunks;
    const T* qq = (const T*)q;
    auto go = [&](auto kern) {
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQfWarps * 32, 0);
      int grid = sms * persist_cap(per_sm);
      if (grid * kQfWarps > items) grid = (items + kQfWarps - 1) / kQfWarps;
      kern<<<grid, kQfWarps * 32, 0, stream>>>(*kv, qq, buf->page_scores, max_chunks, buf->counters + 2, item);
    };
    if constexpr (sizeof(T) == 2) {
      auto gom = [&](auto kern) {
        const int smem = kQfWarps * kQmStages * kQmStageBytes;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int per_sm = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kQfWarps * 32, smem);
        int grid = sms * persist_cap(per_sm);
        if (grid * kQfWarps > items) grid = (items + kQfWarps - 1) / kQfWarps;
        launch_pdl(kern, dim3(grid), dim3(kQfWarps * 32), smem, stream, *kv, (const __nv_bfloat16*)q,
                   buf->page_scores, max_chunks, buf->counters + 2, item, (const __nv_bfloat16*)k_new,
                   (const __nv_bfloat16*)v_new, positions);
      };
      switch (kv->group_size) {
        case 1: gom(quest_filter_mma_kernel<1>); break;
        case 2: gom(quest_filter_mma_kernel<2>); break;
        case 4: gom(quest_filter_mma_kernel<4>); break;
        case 8: gom(quest_filter_mma_kernel<8>); break;
        default: return TW_ERR_INVALID;
      }
    } else {
      switch (kv->group_size) {
        case 1: go(quest_filter_kernel<T, 1>); break;
        case 2: go(quest_filter_kernel<T, 2>); break;
        case 4: go(quest_filter_kernel<T, 4>); break;
        case 8: go(quest_filter_kernel<T, 8>); break;
        default: return TW_ERR_INVALID;
      }
    }
  }
  auto sel = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(kern, dim3(units), dim3(nt), smem, stream, *kv, (const T*)q, *prm, *buf);
  };
  if (nt == 1024) {
    if (ng == 4) sel(quest_select_kernel<T, 4, 1024>);
    else if (ng == 2) sel(quest_select_kernel<T, 2, 1024>);
    else sel(quest_select_kernel<T, 1, 1024>);
  } else {
    if (ng == 4) sel(quest_select_kernel<T, 4, kSelThreads>);
    else if (ng == 2) sel(quest_select_kernel<T, 2, kSelThreads>);
    else sel(quest_select_kernel<T, 1, kSelThreads>);
  }
  return launch_status();
}

int tw_select_channel_pruned(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                             const tw_decode_buffers* buf, cudaStream_t stream);  // channel.cu

// The decode step's K1 + K2 in one pass when the Quest filter runs on the bf16
// tensor-core kernel.  Returns TW_FUSE_UNAVAILABLE (nothing launched) when the
// step must append separately: fp32 cache, other selectors, a select kernel
// that would not fit shared memory, or `positions` aliasing kv->seq_lens (the
// filter writes seq_lens while later items still read their positions).
int tw_unit_select(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                   const int32_t* positions, const tw_decode_params* prm, const tw_decode_buffers* buf,
                   cudaStream_t stream);  // unit.cu

int tw_select_append(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                     const int32_t* positions, const tw_decode_params* prm, const tw_decode_buffers* buf,
                     cudaStream_t stream) {
  // one CTA per unit streams its metadata and selects (unit.cu) when it covers the geometry
  if (int s = tw_unit_select(kv, q, k_new, v_new, positions, prm, buf, stream); s != TW_FUSE_UNAVAILABLE) return s;
  if (!kv || !prm || !buf || !k_new || !v_new || !positions || kv->dtype != TW_BF16 ||
      prm->selector != TW_SELECT_QUEST || kv->head_dim != kHeadDim || kv->num_kv_heads < 1 ||
      kv->num_kv_heads > 32 || kv->num_seqs < 1 || kv->max_pages < 1 ||
      (kv->group_size != 1 && kv->group_size != 2 && kv->group_size != 4 && kv->group_size != 8) ||
      (kv->bits != 0 && kv->bits != 2 && kv->bits != 4 && kv->bits != 8) || prm->budget_pages < 1 ||
      !buf->page_scores || !buf->band_idx || !buf->band_scores || !q || !buf->cand_pages || !buf->cand_count ||
      !buf->counters || !buf->head_max || positions == kv->seq_lens ||
      select_smem_bytes(kv->max_pages, kSelThreads, 1) > 227 * 1024)
    return TW_FUSE_UNAVAILABLE;
  return launch_select<__nv_bfloat16>(kv, q, prm, buf, stream, k_new, v_new, positions);
}

extern "C" int tw_select(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                         const tw_decode_buffers* buf, cudaStream_t stream) {
  if (prm && prm->selector == TW_SELECT_CHANNEL_PRUNED) return tw_select_channel_pruned(kv, q, prm, buf, stream);
  if (!kv || !prm || !buf || kv->head_dim != kHeadDim || !buf->cand_pages || !buf->cand_count || !buf->counters ||
      !buf->head_max)
    return TW_ERR_INVALID;
  if (prm->selector != TW_SELECT_FULL && prm->selector != TW_SELECT_QUEST && prm->selector != TW_SELECT_SINK_WINDOW)
    return TW_ERR_INVALID;
  if (prm->selector == TW_SELECT_SINK_WINDOW && (prm->sink < 0 || prm->window < 0 || prm->sink + prm->window < 1))
    return TW_ERR_INVALID;
  if (prm->selector == TW_SELECT_QUEST &&
      (prm->budget_pages < 1 || !buf->page_scores || !buf->band_idx || !buf->band_scores || !q))
    return TW_ERR_INVALID;
  if (prm->selector == TW_SELECT_QUEST)
    if (int s = tw_unit_select(kv, q, nullptr, nullptr, nullptr, prm, buf, stream); s != TW_FUSE_UNAVAILABLE) return s;
  return kv->dtype == TW_BF16 ? launch_select<__nv_bfloat16>(kv, q, prm, buf, stream)
                              : launch_select<float>(kv, q, prm, buf, stream);
}

extern "C" int tw_quest_scores(const tw_paged_kv* kv, const void* q, double* scores_out, cudaStream_t stream) {
  if (!kv || !q || !scores_out || kv->head_dim != kHeadDim) return TW_ERR_INVALID;
  dim3 grid((kv->max_pages + 7) / 8, kv->num_seqs * kv->num_kv_heads * kv->group_size);
  if (kv->dtype == TW_BF16)
    quest_exact_kernel<__nv_bfloat16><<<grid, 256, 0, stream>>>(*kv, (const __nv_bfloat16*)q, scores_out);
  else
    quest_exact_kernel<float><<<grid, 256, 0, stream>>>(*kv, (const float*)q, scores_out);
  return launch_status();
}
