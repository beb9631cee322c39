// K4 sparse / K5 dense paged decode attention.
//
// Reference: attention_weights (attention.py:89-103) + sparse_attention with
// renormalize=True (attention.py:106-136), run per head over the group's
// shared final set at pipeline.py:366-375: out = w[S] @ V[S] / sum(w[S]), w =
// softmax(K q / sqrt d) -- the softmax restricted to S.  Dense decode (K5) is
// the same over every token (bypass_config, pipeline.py:129-136).
//
// Load balancing: surviving sets differ by orders of
// magnitude between units, so the work is flattened into fixed-size
// (unit, token chunk) items built on device by K3c.  Every WARP is an
// independent worker walking that list; split units are merged afterwards
// (split-KV log-sum-exp) by a small parallel merge kernel.
//
// Per warp: a 2-stage cp.async (LDGSTS, 16 B per lane) ring of 16-row K/V
// tiles, XOR-swizzled so ldmatrix is bank-conflict free.  (Measured on B200,
// tools/tma_bench.cu: cp.async.bulk costs ~70 cycles per copy per issuing
// CTA, i.e. ~1 TB/s for 256-B row gathers at one CTA/SM, while LDGSTS moves
// 512 B per instruction.)  Both products run on tensor cores (mma.sync bf16):
//   S^T[rows x heads]  = K[rows x d] . Q^T[d x heads]      (rows in M, G<=8 heads in N)
//   O^T[d x heads]    += V^T[d x rows] . P^T[rows x heads] (P split into bf16 hi+lo)
// so every gathered row is read once and used by all G heads at a handful of
// issued instructions per row.  The fp32 (parity) variant uses CUDA cores.
#include "common.cuh"

namespace tw {

constexpr int kAttWarps = 4;            // warps (= independent workers) per CTA
constexpr int kAttThreads = kAttWarps * 32;
constexpr int kTile = 16;               // rows per stage
#ifndef TW_ATT_STAGES
#define TW_ATT_STAGES 2
#endif
constexpr int kNS = TW_ATT_STAGES;      // stages per warp
constexpr int kMaxChunk = 512;          // tokens per work item (upper bound)
constexpr int kDefaultChunk = TW_DEFAULT_CHUNK;
constexpr int kDenseChunk = 512;  // dense work-item tokens once the batch fills the GPU (see dense_chunk)

template <typename T>
struct WarpSmem {
  alignas(128) T k[kNS][kTile][kHeadDim];
  alignas(128) T v[kNS][kTile][kHeadDim];
  uint32_t rows[kMaxChunk];  // row index (element offset / 128) of every row of the current item
};

struct ItemDesc {
  int unit, start, count, nitems, slot;
};

template <bool DENSE>
__device__ __forceinline__ ItemDesc get_item(const tw_paged_kv& kv, const tw_decode_buffers& buf, int it,
                                             int chunk, int max_chunks) {
  ItemDesc d;
  if (DENSE) {
    d.unit = it / max_chunks;
    const int c = it % max_chunks;
    const int n = kv.seq_lens[d.unit / kv.num_kv_heads];
    d.start = c * chunk;
    d.count = min(chunk, n - d.start);
    d.nitems = (n + chunk - 1) / chunk;
  } else {
    d.unit = buf.work_items[2 * it];
    d.start = buf.work_items[2 * it + 1];
    d.count = min(chunk, buf.final_count[d.unit] - d.start);
    d.nitems = buf.unit_items[2 * d.unit + 1];
  }
  d.slot = it;
  return d;
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// swizzled byte offset of 16-B chunk c (0..15) of row i inside a bf16 tile
__device__ __forceinline__ int swz(int i, int c) { return i * 256 + ((c ^ (i & 7)) << 4); }

// Issue the cp.async copies of stage s (rows 16s .. 16s+15 of the item).
template <typename T>
__device__ __forceinline__ void issue_stage(WarpSmem<T>& W, const tw_paged_kv& kv, int s, int count, int slot) {
  const int lane = threadIdx.x & 31;
  constexpr int kChunks = kHeadDim * sizeof(T) / 16;  // 16 (bf16) or 32 (fp32) per row
  constexpr int kRowsPerInst = 32 / kChunks;          // 2 or 1
  const int c = lane % kChunks;
  char* kd = reinterpret_cast<char*>(&W.k[slot][0][0]);
  char* vd = reinterpret_cast<char*>(&W.v[slot][0][0]);
#pragma unroll
  for (int i0 = 0; i0 < kTile; i0 += kRowsPerInst) {
    const int i = i0 + lane / kChunks;
    const int j = s * kTile + i;
    if (j < count) {
      const size_t off = (size_t)W.rows[j] * kHeadDim;
      const char* ks = reinterpret_cast<const char*>(reinterpret_cast<const T*>(kv.k_cache) + off) + 16 * c;
      const char* vs = reinterpret_cast<const char*>(reinterpret_cast<const T*>(kv.v_cache) + off) + 16 * c;
      const int o = sizeof(T) == 2 ? swz(i, c) : i * kHeadDim * 4 + 16 * c;
      cp_async16(kd + o, ks);
      cp_async16(vd + o, vs);
    }
  }
}

#ifdef TW_ATT_TRACE
// per work item: start, end (globaltimer ns), global warp id (tools/att_trace.py)
static __device__ unsigned long long g_at[32768][3];
extern "C" int tw_debug_atrace(unsigned long long* host_out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, g_at, sizeof(g_at));
  static unsigned long long zeros[32768 * 3];
  cudaMemcpyToSymbol(g_at, zeros, sizeof(zeros));
  return 0;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

// ------------------------------------------------------------------ bf16 consumer (tensor cores)

struct StateMMA {
  float m[2], l[2];
  float o[8][4];  // O^T: m-tile i (channels 16i..16i+15) x heads (2t, 2t+1)
};

// PACKED (G <= 4): the P split's hi and lo halves share one PV MMA as
// columns (2g, 2g+1) of head g, so the PV product takes 8 MMAs per tile
// instead of 16 and lane (t, r) accumulates head t (o = hi column + lo column).
template <bool PACKED>
__device__ __forceinline__ void consume_mma(StateMMA& st, const uint32_t (&qb)[8][2], const char* K,
                                            const char* V, int rows) {
  const int lane = threadIdx.x & 31;
  const int r = lane >> 2, t = lane & 3, q8 = lane >> 3, rr = lane & 7;
  float s[4] = {0.f, 0.f, 0.f, 0.f};
  {
    const int row = (q8 & 1) * 8 + rr;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t a[4];
      ldsm_x4(a, K + swz(row, kk * 2 + (q8 >> 1)));
      mma16816(s, a, qb[kk][0], qb[kk][1]);
    }
  }
  const float sc = 0.08838834764831845f;  // 1/sqrt(128)
  s[0] = r < rows ? s[0] * sc : -INFINITY;
  s[1] = r < rows ? s[1] * sc : -INFINITY;
  s[2] = r + 8 < rows ? s[2] * sc : -INFINITY;
  s[3] = r + 8 < rows ? s[3] * sc : -INFINITY;
  float alpha[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float mx = fmaxf(s[c], s[c + 2]);
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    const float mn = fmaxf(st.m[c], mx);
    alpha[c] = (st.m[c] == -INFINITY) ? 0.f : __expf(st.m[c] - mn);
    s[c] = (s[c] == -INFINITY) ? 0.f : __expf(s[c] - mn);
    s[c + 2] = (s[c + 2] == -INFINITY) ? 0.f : __expf(s[c + 2] - mn);
    float ps = s[c] + s[c + 2];
    ps += __shfl_xor_sync(0xffffffffu, ps, 4);
    ps += __shfl_xor_sync(0xffffffffu, ps, 8);
    ps += __shfl_xor_sync(0xffffffffu, ps, 16);
    st.l[c] = st.l[c] * alpha[c] + ps;
    st.m[c] = mn;
  }
  const uint32_t h01 = pack_bf16(s[0], s[1]), h23 = pack_bf16(s[2], s[3]);
  const __nv_bfloat162 hb01 = *reinterpret_cast<const __nv_bfloat162*>(&h01);
  const __nv_bfloat162 hb23 = *reinterpret_cast<const __nv_bfloat162*>(&h23);
  const uint32_t l01 = pack_bf16(s[0] - __low2float(hb01), s[1] - __high2float(hb01));
  const uint32_t l23 = pack_bf16(s[2] - __low2float(hb23), s[3] - __high2float(hb23));
  const int vrow = (q8 >> 1) * 8 + rr;
  if constexpr (PACKED) {
    // this lane's PV column r = (head r >> 1, hi | lo); its accumulators hold head t
    const int hb = r >> 1;
    const int srcA = 8 * t + (hb >> 1), srcB = srcA + 4;
    const uint32_t selp = (hb & 1) ? 0x7632u : 0x5410u;
    const bool lo = r & 1;
    const uint32_t ha = __shfl_sync(0xffffffffu, h01, srcA), hbv = __shfl_sync(0xffffffffu, h01, srcB);
    const uint32_t la = __shfl_sync(0xffffffffu, l01, srcA), lb = __shfl_sync(0xffffffffu, l01, srcB);
    const uint32_t ha8 = __shfl_sync(0xffffffffu, h23, srcA), hb8 = __shfl_sync(0xffffffffu, h23, srcB);
    const uint32_t la8 = __shfl_sync(0xffffffffu, l23, srcA), lb8 = __shfl_sync(0xffffffffu, l23, srcB);
    const uint32_t b0 = __byte_perm(lo ? la : ha, lo ? lb : hbv, selp);
    const uint32_t b1 = __byte_perm(lo ? la8 : ha8, lo ? lb8 : hb8, selp);
    // rescale head t's accumulators by its alpha (held by lanes t' = t >> 1, component t & 1)
    const int src = 4 * r + (t >> 1);
    const float a0 = __shfl_sync(0xffffffffu, alpha[0], src), a1 = __shfl_sync(0xffffffffu, alpha[1], src);
    const float at = (t & 1) ? a1 : a0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      st.o[i][0] *= at;
      st.o[i][1] *= at;
      st.o[i][2] *= at;
      st.o[i][3] *= at;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t a[4];
      ldsm_x4_t(a, V + swz(vrow, 2 * i + (q8 & 1)));
      mma16816(st.o[i], a, b0, b1);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      st.o[i][0] *= alpha[0];
      st.o[i][1] *= alpha[1];
      st.o[i][2] *= alpha[0];
      st.o[i][3] *= alpha[1];
    }
    // P^T B fragments from the S^T accumulators (rows 2t,2t+1 | 2t+8,2t+9 of head g)
    const int g = lane >> 2;
    const int srcA = 8 * t + (g >> 1), srcB = srcA + 4;
    const uint32_t selp = (g & 1) ? 0x7632u : 0x5410u;
    const uint32_t bh0 = __byte_perm(__shfl_sync(0xffffffffu, h01, srcA), __shfl_sync(0xffffffffu, h01, srcB), selp);
    const uint32_t bh1 = __byte_perm(__shfl_sync(0xffffffffu, h23, srcA), __shfl_sync(0xffffffffu, h23, srcB), selp);
    const uint32_t bl0 = __byte_perm(__shfl_sync(0xffffffffu, l01, srcA), __shfl_sync(0xffffffffu, l01, srcB), selp);
    const uint32_t bl1 = __byte_perm(__shfl_sync(0xffffffffu, l23, srcA), __shfl_sync(0xffffffffu, l23, srcB), selp);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t a[4];
      ldsm_x4_t(a, V + swz(vrow, 2 * i + (q8 & 1)));
      mma16816(st.o[i], a, bh0, bh1);
      mma16816(st.o[i], a, bl0, bl1);
    }
  }
}

// ------------------------------------------------------------------ fp32 consumer (CUDA cores)

template <int G>
struct StateF32 {
  float m[G], l[G], o[G][4];  // lane owns channels 4*lane .. 4*lane+3
};

template <int G>
__device__ __forceinline__ void consume_f32(StateF32<G>& st, const float (&qf)[G][4], const float* K,
                                            const float* V, int rows) {
  const int lane = threadIdx.x & 31;
  const float sc = 0.08838834764831845f;
  for (int i = 0; i < rows; ++i) {
    const float4 k4 = *reinterpret_cast<const float4*>(K + i * kHeadDim + 4 * lane);
    const float4 v4 = *reinterpret_cast<const float4*>(V + i * kHeadDim + 4 * lane);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float a = qf[g][0] * k4.x + qf[g][1] * k4.y + qf[g][2] * k4.z + qf[g][3] * k4.w;
      a = warp_sum(a) * sc;
      const float mn = fmaxf(st.m[g], a);
      const float al = st.m[g] == -INFINITY ? 0.f : expf(st.m[g] - mn);
      const float p = expf(a - mn);
      st.l[g] = st.l[g] * al + p;
      st.m[g] = mn;
      st.o[g][0] = fmaf(p, v4.x, st.o[g][0] * al);
      st.o[g][1] = fmaf(p, v4.y, st.o[g][1] * al);
      st.o[g][2] = fmaf(p, v4.z, st.o[g][2] * al);
      st.o[g][3] = fmaf(p, v4.w, st.o[g][3] * al);
    }
  }
}

// ------------------------------------------------------------------ the kernel

template <typename T, int G, bool DENSE>
__global__ void __launch_bounds__(kAttThreads) attn_kernel(tw_paged_kv kv, const T* __restrict__ q,
                                                           tw_decode_buffers buf, float* __restrict__ out,
                                                           int chunk, int max_chunks, int total_items) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem<T>& W = reinterpret_cast<WarpSmem<T>*>(smem_raw)[warp];
  const int nitems_total = DENSE ? total_items : min((int)buf.counters[0], total_items);
  const size_t T_stride = (size_t)kv.max_pages * kPage;
  const int H = kv.num_kv_heads;
  const int gw = blockIdx.x * kAttWarps + warp, nw = gridDim.x * kAttWarps;
  const int r = lane >> 2, t = lane & 3;

  uint32_t* ctr = buf.counters + (DENSE ? 5 : 4);
  for (int it = warp_fetch(ctr); it < nitems_total; it = warp_fetch(ctr)) {
    const ItemDesc d = get_item<DENSE>(kv, buf, it, chunk, max_chunks);
    if (d.count <= 0) continue;
#ifdef TW_ATT_TRACE
    if (lane == 0 && it < 32768) { g_at[it][0] = gtimer(); g_at[it][2] = gw; }
#endif
    const int b = d.unit / H, h = d.unit % H;
    // Row indices (token id -> page table -> row): the first 32 rows (the
    // ring's first stages) are resolved first and their copies issued, then
    // the rest resolve while those copies are in flight, all loads of a batch
    // in flight together (two dependent L2 round trips per 8 rows otherwise
    // stalled every item's start).
    const int* pt = kv.page_table + (size_t)b * kv.max_pages;
    const int* ids = DENSE ? nullptr : buf.final_idx + d.unit * T_stride + d.start;
    auto row_of = [&](int j) -> uint32_t {
      const int tok = DENSE ? d.start + j : __ldg(ids + j);
      return ((uint32_t)__ldg(pt + (tok >> 4)) * H + h) * kPage + (tok & 15);
    };
    __syncwarp();
    if (lane < d.count) W.rows[lane] = row_of(lane);
    __syncwarp();
    const int nst = (d.count + kTile - 1) / kTile;
    static_assert((kNS - 1) * kTile <= 32, "the prologue stages use the first 32 rows");
#pragma unroll
    for (int s = 0; s < kNS - 1; ++s) {
      if (s < nst) issue_stage<T>(W, kv, s, d.count, s);
      cp_commit();
    }
    {
      constexpr int kB = 8;  // rows per lane resolved together
      for (int j0 = 32; j0 < d.count; j0 += 32 * kB) {
        int tok[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int j = j0 + 32 * u + lane;
          tok[u] = j < d.count ? (DENSE ? d.start + j : __ldg(ids + j)) : 0;
        }
        uint32_t ph[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) ph[u] = j0 + 32 * u + lane < d.count ? (uint32_t)__ldg(pt + (tok[u] >> 4)) : 0u;
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int j = j0 + 32 * u + lane;
          if (j < d.count) W.rows[j] = (ph[u] * H + h) * kPage + (tok[u] & 15);
        }
      }
      __syncwarp();
    }
    const T* qu = q + (size_t)d.unit * G * kHeadDim;
    float* part = buf.partials + (size_t)d.slot * G * (kHeadDim + 2);
    const bool single = d.nitems == 1;
    if constexpr (sizeof(T) == 2) {
      uint32_t qb[8][2];
      const int g = lane >> 2;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (g < G) {
          const uint32_t* qw = reinterpret_cast<const uint32_t*>(qu + g * kHeadDim + kk * 16);
          qb[kk][0] = __ldg(qw + t);
          qb[kk][1] = __ldg(qw + t + 4);
        } else {
          qb[kk][0] = qb[kk][1] = 0u;
        }
      }
      StateMMA st;
      st.m[0] = st.m[1] = -INFINITY;
      st.l[0] = st.l[1] = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) st.o[i][0] = st.o[i][1] = st.o[i][2] = st.o[i][3] = 0.f;
      for (int s = 0; s < nst; ++s) {
        if (s + kNS - 1 < nst) issue_stage<T>(W, kv, s + kNS - 1, d.count, (s + kNS - 1) % kNS);
        cp_commit();
        cp_wait<kNS - 1>();
        __syncwarp();
        const int slot = s % kNS;
        const int rows = min(kTile, d.count - s * kTile);
        if (rows < kTile) {  // 0 * stale smem would poison the PV product: clear unused V rows
          uint4* vz = reinterpret_cast<uint4*>(&W.v[slot][rows][0]);
          for (int z = lane; z < (kTile - rows) * 16; z += 32) vz[z] = make_uint4(0, 0, 0, 0);
          __syncwarp();
        }
        consume_mma<(G <= 4)>(st, qb, reinterpret_cast<const char*>(&W.k[slot][0][0]),
                              reinterpret_cast<const char*>(&W.v[slot][0][0]), rows);
        __syncwarp();
      }
      if constexpr (G <= 4) {
        // packed: lane (t, r) holds head t (hi + lo columns) for channels 16i + r (+8); its
        // softmax state sits in lanes t' = t >> 1, component t & 1
        const int src = 4 * r + (t >> 1);
        const float m0 = __shfl_sync(0xffffffffu, st.m[0], src), m1 = __shfl_sync(0xffffffffu, st.m[1], src);
        const float l0 = __shfl_sync(0xffffffffu, st.l[0], src), l1 = __shfl_sync(0xffffffffu, st.l[1], src);
        const float mt = (t & 1) ? m1 : m0, lt = (t & 1) ? l1 : l0;
        if (t < G) {
          const float inv = lt > 0.f ? 1.f / lt : 0.f;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int c0 = 16 * i + r;
            const float o0 = st.o[i][0] + st.o[i][1], o8 = st.o[i][2] + st.o[i][3];
            if (single) {
              out[((size_t)d.unit * G + t) * kHeadDim + c0] = o0 * inv;
              out[((size_t)d.unit * G + t) * kHeadDim + c0 + 8] = o8 * inv;
            } else {
              part[t * (kHeadDim + 2) + c0] = o0;
              part[t * (kHeadDim + 2) + c0 + 8] = o8;
            }
          }
          if (!single && r == 0) {
            part[t * (kHeadDim + 2) + kHeadDim] = mt;
            part[t * (kHeadDim + 2) + kHeadDim + 1] = lt;
          }
        }
      } else {
      // emit: lane holds heads 2t, 2t+1 for channels 16i + r (+8)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int g2 = 2 * t + c;
        if (g2 < G) {
          const float inv = st.l[c] > 0.f ? 1.f / st.l[c] : 0.f;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int c0 = 16 * i + r;
            if (single) {
              out[((size_t)d.unit * G + g2) * kHeadDim + c0] = st.o[i][c] * inv;
              out[((size_t)d.unit * G + g2) * kHeadDim + c0 + 8] = st.o[i][c + 2] * inv;
            } else {
              part[g2 * (kHeadDim + 2) + c0] = st.o[i][c];
              part[g2 * (kHeadDim + 2) + c0 + 8] = st.o[i][c + 2];
            }
          }
          if (!single && r == 0) {
            part[g2 * (kHeadDim + 2) + kHeadDim] = st.m[c];
            part[g2 * (kHeadDim + 2) + kHeadDim + 1] = st.l[c];
          }
        }
      }
      }
    } else {
      float qf[G][4];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float4 v = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(qu) + g * kHeadDim + 4 * lane);
        qf[g][0] = v.x; qf[g][1] = v.y; qf[g][2] = v.z; qf[g][3] = v.w;
      }
      StateF32<G> st;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        st.m[g] = -INFINITY;
        st.l[g] = 0.f;
        st.o[g][0] = st.o[g][1] = st.o[g][2] = st.o[g][3] = 0.f;
      }
      for (int s = 0; s < nst; ++s) {
        if (s + kNS - 1 < nst) issue_stage<T>(W, kv, s + kNS - 1, d.count, (s + kNS - 1) % kNS);
        cp_commit();
        cp_wait<kNS - 1>();
        __syncwarp();
        const int slot = s % kNS;
        consume_f32<G>(st, qf, reinterpret_cast<const float*>(&W.k[slot][0][0]),
                       reinterpret_cast<const float*>(&W.v[slot][0][0]), min(kTile, d.count - s * kTile));
        __syncwarp();
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float inv = st.l[g] > 0.f ? 1.f / st.l[g] : 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (single)
            out[((size_t)d.unit * G + g) * kHeadDim + 4 * lane + e] = st.o[g][e] * inv;
          else
            part[g * (kHeadDim + 2) + 4 * lane + e] = st.o[g][e];
        }
        if (!single && lane == 0) {
          part[g * (kHeadDim + 2) + kHeadDim] = st.m[g];
          part[g * (kHeadDim + 2) + kHeadDim + 1] = st.l[g];
        }
      }
    }
    cp_wait<0>();
#ifdef TW_ATT_TRACE
    if (lane == 0 && it < 32768) g_at[it][1] = gtimer();
#endif
  }
  // units whose final set is empty: zeros (sparse_attention, attention.py:126-129)
  if (!DENSE) {
    const int units = kv.num_seqs * H;
    for (int u = gw; u < units; u += nw)
      if (buf.final_count[u] == 0)
        for (int x = lane; x < G * kHeadDim; x += 32) out[(size_t)u * G * kHeadDim + x] = 0.f;
  }
}

// Merge the split-KV partials of every unit with more than one item
// (log-sum-exp over the union of the items, attention.py:130-135): one CTA of
// kMergeThreads per (unit, head).  Every thread loads item maxima / masses
// (one round of loads for up to kMergeThreads items), the CTA reduces the max
// and the weights, then kMergeGroups groups of 128 threads each sum a quarter
// of the items' outputs for channel (tid % 128) with their loads in flight,
// and the groups' sums are added in a fixed order.
constexpr int kMergeGroups = 4;
constexpr int kMergeThreads = kMergeGroups * kHeadDim;

template <int G, bool DENSE>
__global__ void __launch_bounds__(kMergeThreads) merge_kernel(tw_paged_kv kv, tw_decode_buffers buf,
                                                              float* __restrict__ out, int chunk, int max_chunks) {
  pdl_wait();
  pdl_trigger();
  constexpr int kMaxItems = 1024;
  constexpr int NW = kMergeThreads / 32;
  __shared__ float e_s[kMaxItems];
  __shared__ float red[NW], red2[NW];
  __shared__ float osum[kMergeGroups][kHeadDim];
  const int unit = blockIdx.x / G, g = blockIdx.x % G, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int first, n;
  if (DENSE) {
    const int len = kv.seq_lens[unit / kv.num_kv_heads];
    first = unit * max_chunks;
    n = (len + chunk - 1) / chunk;
  } else {
    first = buf.unit_items[2 * unit];
    n = buf.unit_items[2 * unit + 1];
  }
  if (n <= 1) return;
  constexpr int kStride = G * (kHeadDim + 2);
  const float* P = buf.partials + (size_t)first * kStride + g * (kHeadDim + 2);
  // item maxima (n <= kMaxItems: tw_max_work_items bounds the items of one unit)
  float mloc = -INFINITY;
  for (int i = tid; i < n; i += kMergeThreads) {
    const float mi = P[(size_t)i * kStride + kHeadDim];
    e_s[i] = mi;
    mloc = fmaxf(mloc, mi);
  }
  mloc = warp_max(mloc);
  if (lane == 0) red[warp] = mloc;
  __syncthreads();
  float M = red[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) M = fmaxf(M, red[w]);
  float lloc = 0.f;
  for (int i = tid; i < n; i += kMergeThreads) {
    const float mi = e_s[i];
    const float e = mi == -INFINITY ? 0.f : __expf(mi - M);
    e_s[i] = e;
    lloc = fmaf(e, P[(size_t)i * kStride + kHeadDim + 1], lloc);
  }
  lloc = warp_sum(lloc);
  if (lane == 0) red2[warp] = lloc;
  __syncthreads();
  float L = 0.f;
#pragma unroll
  for (int w = 0; w < NW; ++w) L += red2[w];
  const int grp = tid / kHeadDim, c = tid % kHeadDim;
  float O = 0.f;
  int i = grp;
  for (; i + 8 * kMergeGroups <= n; i += 8 * kMergeGroups) {
    float o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = P[(size_t)(i + k * kMergeGroups) * kStride + c];
#pragma unroll
    for (int k = 0; k < 8; ++k) O = fmaf(e_s[i + k * kMergeGroups], o[k], O);
  }
  for (; i < n; i += kMergeGroups) O = fmaf(e_s[i], P[(size_t)i * kStride + c], O);
  osum[grp][c] = O;
  __syncthreads();
  if (grp == 0) {
    float t = osum[0][c];
#pragma unroll
    for (int k = 1; k < kMergeGroups; ++k) t += osum[k][c];
    out[((size_t)unit * G + g) * kHeadDim + c] = L > 0.f ? t / L : 0.f;
  }
}

}  // namespace tw

using namespace tw;

// Work-item geometry the attention + merge kernels accept: chunks of whole
// 16-row tiles, at most kMaxChunk tokens, and at most 1024 items per unit (the
// merge kernel's per-(unit, head) weights).  Checked by tw_decode_step before
// K1 mutates the cache.
int tw_attn_geometry(const tw_paged_kv* kv, int chunk) {
  if (chunk < kTile || chunk > kMaxChunk || chunk % kTile != 0) return TW_ERR_INVALID;
  const int64_t T_tokens = (int64_t)kv->max_pages * kPage;
  if ((T_tokens + chunk - 1) / chunk > 1024) return TW_ERR_INVALID;
  return TW_OK;
}

// part: 0 both kernels, 1 the attention kernel only, 2 the merge only (per-kernel timing)
template <typename T, int G, bool DENSE>
static int launch_attn(const tw_paged_kv* kv, const T* q, const tw_decode_buffers* buf, float* out, int chunk,
                       cudaStream_t s, int part = 0) {
  const int units = kv->num_seqs * kv->num_kv_heads;
  const int T_tokens = kv->max_pages * kPage;
  const int max_chunks = (T_tokens + chunk - 1) / chunk;
  const int total = DENSE ? units * max_chunks : (int)buf->max_items;
  if (int st = tw_attn_geometry(kv, chunk)) return st;
  if (DENSE && (int64_t)units * max_chunks > buf->max_items) return TW_ERR_INVALID;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = sizeof(WarpSmem<T>) * kAttWarps;
  auto kern = attn_kernel<T, G, DENSE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kAttThreads, smem);
  int grid = sms * persist_cap(per_sm);
  if (DENSE && grid * kAttWarps > total) grid = (total + kAttWarps - 1) / kAttWarps;
  if (part != 2) {
    if (DENSE) cudaMemsetAsync(buf->counters + 5, 0, sizeof(uint32_t), s);  // dense runs without tw_select
    else if (part == 1) cudaMemsetAsync(buf->counters + 4, 0, sizeof(uint32_t), s);  // re-runnable alone
    launch_pdl(kern, dim3(grid), dim3(kAttThreads), smem, s, *kv, q, *buf, out, chunk, max_chunks, total);
  }
  if (part != 1)
    launch_pdl(merge_kernel<G, DENSE>, dim3(units * G), dim3(kMergeThreads), 0, s, *kv, *buf, out, chunk, max_chunks);
  return launch_status();
}

#define TW_DISPATCH_G(G_, CALL)                    \
  switch (G_) {                                    \
    case 1: { constexpr int GG = 1; return CALL; } \
    case 2: { constexpr int GG = 2; return CALL; } \
    case 4: { constexpr int GG = 4; return CALL; } \
    case 8: { constexpr int GG = 8; return CALL; } \
    default: return TW_ERR_INVALID;                \
  }

static inline int sparse_chunk(const tw_decode_params* prm) {
  return prm->chunk_tokens > 0 ? prm->chunk_tokens : kDefaultChunk;
}

extern "C" int tw_sparse_attention_part(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                                        const tw_decode_buffers* buf, float* out, int32_t part,
                                        cudaStream_t stream) {
  if (!kv || !q || !prm || !buf || !out || kv->head_dim != kHeadDim || !buf->partials) return TW_ERR_INVALID;
  if (prm->renormalize != 1 || part < 0 || part > 2) return TW_ERR_INVALID;
  const int chunk = sparse_chunk(prm);
  if (kv->dtype == TW_BF16) {
    TW_DISPATCH_G(kv->group_size, (launch_attn<__nv_bfloat16, GG, false>(kv, (const __nv_bfloat16*)q, buf, out,
                                                                        chunk, stream, part)))
  }
  TW_DISPATCH_G(kv->group_size,
                (launch_attn<float, GG, false>(kv, (const float*)q, buf, out, chunk, stream, part)))
}

extern "C" int tw_sparse_attention(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                                   const tw_decode_buffers* buf, float* out, cudaStream_t stream) {
  return tw_sparse_attention_part(kv, q, prm, buf, out, 0, stream);
}

// Dense work-item size: 512 tokens once units x chunks give every worker warp
// of a full GPU (148 SMs x 12 warps) two items; smaller (down to 64, multiples
// of 16) for small batches, which would otherwise leave most SMs idle (batch 1
// x 8 KV heads at 8k: 136 items of 512 for 1776 workers); never more than 1024
// items per unit (the merge kernel's bound).
static int dense_chunk(const tw_paged_kv* kv) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t units = (int64_t)kv->num_seqs * kv->num_kv_heads;
  const int64_t T = (int64_t)kv->max_pages * kPage;
  const int64_t target = (int64_t)sms * 3 * kAttWarps * 2;
  int64_t c = (T * units + target - 1) / target;
  c = (c + kTile - 1) / kTile * kTile;
  c = c < 64 ? 64 : c > kDenseChunk ? kDenseChunk : c;
  const int64_t floor1024 = ((T + 1023) / 1024 + kTile - 1) / kTile * kTile;
  return (int)(c < floor1024 ? floor1024 : c);
}

extern "C" int tw_dense_attention(const tw_paged_kv* kv, const void* q, const tw_decode_buffers* buf, float* out,
                                  cudaStream_t stream) {
  if (!kv || !q || !buf || !out || kv->head_dim != kHeadDim || !buf->partials) return TW_ERR_INVALID;
  const int chunk = dense_chunk(kv);
  if (kv->dtype == TW_BF16) {
    TW_DISPATCH_G(kv->group_size,
                  (launch_attn<__nv_bfloat16, GG, true>(kv, (const __nv_bfloat16*)q, buf, out, chunk, stream)))
  }
  TW_DISPATCH_G(kv->group_size, (launch_attn<float, GG, true>(kv, (const float*)q, buf, out, chunk, stream)))
}

extern "C" int64_t tw_max_work_items(const tw_paged_kv* kv, int32_t chunk_tokens) {
  if (!kv) return 0;
  const int64_t units = (int64_t)kv->num_seqs * kv->num_kv_heads;
  const int64_t T = (int64_t)kv->max_pages * kPage;
  const int64_t c = chunk_tokens > 0 ? chunk_tokens : kDefaultChunk;
  const int64_t sparse = units * ((T + c - 1) / c);
  const int64_t dc = dense_chunk(kv);
  const int64_t dense = units * ((T + dc - 1) / dc);
  return sparse > dense ? sparse : dense;
}
