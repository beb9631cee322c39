/*
 * twilight.h -- C ABI of the B200 (sm_100a) Twilight decode-attention path.
 *
 * Plain C: device pointers, sizes and a cudaStream_t.  No torch types.  The
 * caller allocates every buffer (the library never allocates or frees); all
 * work is enqueued on the given stream, so the calls are CUDA-graph safe and
 * never synchronise with the host.  Every entry point returns a tw_status.
 *
 * The reference (/root/reference/pkg, Python/NumPy package "nucleuskv") has
 * no FFI; its seam is the Python operator API.  Each entry point below names
 * the reference function(s) it replaces (file:line under pkg/src/nucleuskv/).
 * The Python shim paper_2502_02770_b200 binds these with ctypes and restores
 * the reference signatures.
 *
 * Layout of one paged KV pool (one attention layer), page size 16:
 *   k_cache, v_cache : [num_phys_pages][H_kv][16][d]       dtype (bf16 | f32)
 *   kq               : [num_phys_pages][H_kv][1152] bytes:  packed INT4 codes
 *                      [16][d/2] (even channel in the low nibble, exactly the
 *                      reference's byte layout, quantcache.py:122-151), then
 *                      f32 scale[16], f32 zero[16]
 *   kmeta            : [num_phys_pages][H_kv][2][d] dtype:  per-page channel
 *                      min (lo) and max (hi) of the real rows
 *   kabsmax          : [B][H_kv] f32: max |k| over the unit (Quest filter bound)
 *   page_table       : [B][max_pages] int32 logical page -> physical page
 *   seq_lens         : [B] int32 tokens in each sequence
 */
#ifndef TWILIGHT_H_
#define TWILIGHT_H_

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TW_PAGE_SIZE 16
#define TW_QBLOCK_BYTES 1152  /* 4-bit block; a b-bit block is TW_QBLOCK_BYTES_FOR(b) */
#define TW_QBLOCK_BYTES_FOR(bits) (256 * (bits) + 128)
#define TW_DEFAULT_CHUNK 512 /* tokens per sparse-attention work item */
#define TW_TOPP_BINS 4096        /* top-p histogram bins per query head */
#define TW_TOPP_MEMBER_CAP 8192  /* crossing-bin members held on chip per unit (more: re-read path) */

/* Status codes; the shim maps them to the reference's exceptions
 * (attention.py:30-36, pruner.py:67-76, quantcache.py:246-267). */
typedef enum {
  TW_OK = 0,
  TW_ERR_INVALID = 1,    /* ValueError */
  TW_ERR_INDEX = 2,      /* IndexError */
  TW_ERR_DEGENERATE = 3, /* DegenerateSelectionError */
  TW_ERR_CUDA = 4        /* RuntimeError */
} tw_status;

typedef enum { TW_F32 = 0, TW_BF16 = 1 } tw_dtype;
typedef enum {
  TW_SELECT_FULL = 0,
  TW_SELECT_QUEST = 1,
  TW_SELECT_SINK_WINDOW = 2,
  TW_SELECT_CHANNEL_PRUNED = 3
} tw_selector;

typedef enum {
  TW_ESTIMATE_INT = 0,   /* INT-b key cache, PagedKVCache.bits */
  TW_ESTIMATE_EXACT = 1  /* K[idx] @ q / sqrt(d) from k_cache */
} tw_estimator;

typedef struct tw_paged_kv {
  int32_t num_seqs;       /* B */
  int32_t num_kv_heads;   /* H_kv */
  int32_t group_size;     /* G query heads per KV head (GroupMap, selectors.py:53-69) */
  int32_t head_dim;       /* d; 128 on this path */
  int32_t max_pages;      /* page_table row length */
  int32_t num_phys_pages; /* pages in the pool */
  int32_t dtype;          /* tw_dtype of K, V, q and kmeta */
  int32_t bits;           /* INT key cache width: 2, 4 or 8 (SUPPORTED_BITS, quantcache.py:38); 0 = 4 */
  void* k_cache;
  void* v_cache;
  uint8_t* kq;
  void* kmeta;
  float* kabsmax;
  const int32_t* page_table;
  int32_t* seq_lens;
} tw_paged_kv;

typedef struct tw_decode_params {
  int32_t selector;     /* tw_selector: full (selectors.py:90-94), quest (:112-132), sink_window (:164-175) */
  int32_t budget_pages; /* ceil(B0 / 16), B0 = resolve_budget(...) (selectors.py:72-87, :127) */
  double p;             /* top-p mass target, BinarySearchConfig.p (pruner.py:35) */
  int32_t chunk_tokens; /* sparse-attention work-item size (0 = TW_DEFAULT_CHUNK) */
  int32_t renormalize;  /* must be 1 on this path (PipelineConfig.renormalize_output, pipeline.py:58) */
  int32_t sink;         /* sink-window selector (select_sink_window, selectors.py:164-175): first tokens kept */
  int32_t window;       /* ... and last tokens kept; every token when sink + window >= n */
  int32_t top_channels; /* channel-pruned selector (select_channel_pruned, selectors.py:146-161): channels kept
                           (0 = d / 8, build_selector :205-207) */
  int32_t budget_tokens;/* channel-pruned selector: B0 in tokens (resolve_budget) */
  int32_t channels_fixed;/* channel-pruned selector: 0 = rank the channels by mean |K| and write them to
                           chan_ids; 1 = use the top_channels ids already in chan_ids (the slice fixed
                           once per context, selectors.py:203) */
  int32_t estimator;    /* tw_estimator: the cache's INT codes (estimate_scores, quantcache.py:238-272) or
                           the full-precision keys (estimator_bits="exact", pipeline.py:212-214) */
} tw_decode_params;

/* Intermediate buffers of one decode step (all caller-allocated, sizes in
 * elements; U = B*H_kv units, Hq = B*H_kv*G query heads, T = max_pages*16). */
typedef struct tw_decode_buffers {
  float* page_scores;       /* [Hq][max_pages]   fp32 Quest bounds (filter pass) */
  int32_t* cand_pages;      /* [U][max_pages]    sorted candidate logical pages (group union) */
  int32_t* cand_count;      /* [U] */
  float* logits;            /* [U][G][T]         INT4-estimated logits, -inf past seq end */
  uint32_t* head_max;       /* [Hq]              max logit (ordered key); zeroed by tw_select */
  uint32_t* head_thr;       /* [Hq]              top-p threshold (ordered key of the logit) */
  float* head_stats;        /* [Hq][4]           B1, candidate mass, threshold weight, B0 */
  int32_t* final_idx;       /* [U][T]            group-shared surviving token ids, ascending */
  int32_t* final_count;     /* [U] */
  int32_t* unit_items;      /* [U][2]            first work item, number of work items */
  int32_t* work_items;      /* [max_items][2]    (unit, first token slot) */
  uint32_t* counters;       /* [8]               device-side counters (zeroed by tw_select; [6] = max candidate pages) */
  float* partials;          /* [max_items][G][d+2] split-KV partial (o[d], m, l) */
  uint32_t* head_page_bits; /* optional [Hq][ceil(max_pages/32)] per-head Quest page sets */
  uint32_t* sel_bits;       /* [U][ceil(T/32)]   group-union bitmap over candidate positions */
  uint32_t* tok_mask;       /* [U][ceil(T/32)]        channel-pruned selector: selected tokens (the estimate's mask) */
  int32_t* chan_ids;        /* [U][128]          channel-pruned selector: the channel slice (ascending) */
  int32_t* topp_done;       /* [U]               small-batch top-p: heads finished per unit (zero-initialised;
                                                   left zeroed; with it, sel_bits must start zeroed too) */
  int32_t* band_idx;        /* [Hq][max_pages]   Quest pages in the fp32 filter's ambiguous band */
  double* band_scores;      /* [Hq][max_pages]   their exact fp64 bounds */
  int64_t max_items;
} tw_decode_buffers;

/* Library version (major*10000 + minor*100 + patch). */
int32_t tw_version(void);

/* Worst-case number of sparse/dense attention work items for this geometry. */
int64_t tw_max_work_items(const tw_paged_kv* kv, int32_t chunk_tokens);

/* K1 -- quantize-on-append.  For every sequence b, writes the new K/V row of
 * every KV head at token position positions[b] (k_new/v_new: [B][H_kv][d]),
 * its INT4 codes + params, updates the page's channel min/max and the unit's
 * |k| bound, and sets seq_lens[b] = positions[b] + 1.  Bit-exact with
 * build_cache over the grown matrix (quantcache.py:95-114, 178-235) and
 * build_page_metadata (quantcache.py:163-175).  positions may alias seq_lens. */
int tw_quant_append(const tw_paged_kv* kv, const void* k_new, const void* v_new,
                    const int32_t* positions, cudaStream_t stream);

/* K1 (bulk) -- quantize every cached token < seq_lens[b] (prefill / cache
 * build): build_cache + build_page_metadata (quantcache.py:163-235). */
int tw_quant_build(const tw_paged_kv* kv, cudaStream_t stream);

/* Row quantizer for an (n, d) matrix: codes [n][d] u8 and fp64 params,
 * bits in {2, 4, 8}: quantize_row (quantcache.py:95-114). */
int tw_quant_rows(const void* rows, int32_t n, int32_t d, int32_t dtype, int32_t bits,
                  uint8_t* codes_out, double* scale_out, double* zero_out, cudaStream_t stream);

/* Exact fp64 Quest page bounds for every query head: quest_page_scores
 * (selectors.py:97-109), bit-identical to NumPy (same summation order).
 * q: [B][H_kv*G][d]; scores_out: [B*H_kv*G][max_pages], -inf past the last page. */
int tw_quest_scores(const tw_paged_kv* kv, const void* q, double* scores_out, cudaStream_t stream);

/* K2 -- page selection + GQA union: select_quest (selectors.py:112-132) per
 * query head (exact top-k with ties to the lower page: fp32 filter, fp64
 * refine of the ambiguous band), group_union (selectors.py:178-186) per KV
 * head; or select_full (selectors.py:90-94).  Also zeroes buf->counters. */
int tw_select(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
              const tw_decode_buffers* buf, cudaStream_t stream);

/* K3a -- INT4 estimate over the candidate pages for all G heads of a unit:
 * estimate_scores (quantcache.py:238-272) as called at pipeline.py:342; with
 * prm->estimator == TW_ESTIMATE_EXACT the logits come from the full-precision
 * keys instead (_candidate_logits exact path, pipeline.py:212-214). */
int tw_estimate(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                const tw_decode_buffers* buf, cudaStream_t stream);

/* K3b/K3c -- per-head softmax over the candidates + top-p threshold
 * (stable_softmax attention.py:79-86 at pipeline.py:344; the minimal
 * tie-closed set of binary_search_top_p, pruner.py:57-114), then the group
 * union of the pruned sets (pipeline.py:347) and the attention work list. */
int tw_topp(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
            cudaStream_t stream);

/* K4 -- sparse decode attention of every query head over its group's final
 * set, subset softmax (attention_weights + sparse_attention(renormalize=True),
 * attention.py:89-136 at pipeline.py:366-375), head-flattened split-KV work
 * items merged on device.  out: [B][H_kv*G][d] f32. */
int tw_sparse_attention(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                        const tw_decode_buffers* buf, float* out, cudaStream_t stream);

/* tw_sparse_attention in parts, for per-kernel timing: part 1 launches only
 * the gather / subset-softmax kernel (split units' partials are left in
 * buf->partials, their out rows unwritten), part 2 only the split-KV merge;
 * 0 = both (= tw_sparse_attention). */
int tw_sparse_attention_part(const tw_paged_kv* kv, const void* q, const tw_decode_params* prm,
                             const tw_decode_buffers* buf, float* out, int32_t part, cudaStream_t stream);

/* K5 -- dense paged decode attention over all seq_lens[b] tokens (the bypass
 * layers' path, bypass_config pipeline.py:129-136; the speedup baseline). */
int tw_dense_attention(const tw_paged_kv* kv, const void* q, const tw_decode_buffers* buf,
                       float* out, cudaStream_t stream);

/* K2 + K3 (tw_select, tw_estimate, tw_topp) for every unit in ONE launch, one
 * CTA per unit (sequence, KV head) running its filter, page selection, INT4
 * estimate and top-p back to back; with positions (and k_new, v_new) the K1
 * append of each unit's new row runs first inside the same CTA (positions must
 * not alias seq_lens).  Same outputs as the separate calls.  Covers bf16
 * caches with 4-bit codes, the quest and full selectors, the INT estimator,
 * G in {1, 2, 4} and batches of at least 64 units (TW_UNIT_MIN); anything else
 * returns TW_ERR_INVALID (use the separate calls).  tw_decode_step takes this
 * path whenever it applies. */
int tw_select_estimate_topp(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                            const int32_t* positions, const tw_decode_params* prm,
                            const tw_decode_buffers* buf, cudaStream_t stream);

/* 1 when tw_select_estimate_topp covers this geometry and these options, else 0. */
int32_t tw_select_estimate_topp_applies(const tw_paged_kv* kv, const tw_decode_params* prm,
                                        const tw_decode_buffers* buf);

/* One full decode step of one layer: K1 append, K2, K3a, K3b/c, K4. */
int tw_decode_step(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                   const int32_t* positions, const tw_decode_params* prm,
                   const tw_decode_buffers* buf, float* out, cudaStream_t stream);

/* INT4 estimate at arbitrary token ids of one unit (seq, kv_head) for one
 * query (d,): estimate_scores (quantcache.py:238-272).  Returns
 * TW_ERR_INDEX via *status_out (device-written int) for ids >= seq_len. */
int tw_estimate_tokens(const tw_paged_kv* kv, int32_t seq, int32_t kv_head, const void* q,
                       const int32_t* token_idx, int32_t m, float* scores_out,
                       int32_t* status_out, cudaStream_t stream);

/* Literal Algorithm 1 threshold bisection on rows of normalised fp64 weights
 * (binary_search_top_p, pruner.py:57-114), any epsilon / max_iters:
 * weights [rows][n]; mask_out [rows][n] u8; threshold_out / iters_out [rows]. */
int tw_topp_bisect(const double* weights, int32_t rows, int32_t n, double p, double epsilon,
                   int32_t max_iters, uint8_t* mask_out, double* threshold_out,
                   int32_t* iters_out, cudaStream_t stream);

/* Per-vector operators of the reference API (off the decode path):
 *   tw_vec_logits  out[n] f32 = K[n][d] q[d] / float32(sqrt d)      attention.py:102 (attention_weights)
 *   tw_vec_softmax out[n] f32 = exp(z - max z) / sum, scratch >= 16 B attention.py:79-86 (stable_softmax)
 *   tw_vec_readout out[d] = w[idx] @ V[idx] (/ sum w[idx] if renorm), weights f32 (TW_F32) or f64 (2),
 *                  values f32 / bf16; out in the weights' type; partial: tw_vec_readout_parts() * (d+1)
 *                  doubles of scratch; *mass_out = sum w[idx]       attention.py:106-136 (sparse_attention)
 * dtype / vdtype are tw_dtype codes. */
int tw_vec_logits(const void* q, const void* keys, int64_t n, int32_t d, int32_t dtype, float* out,
                  cudaStream_t stream);
int tw_vec_softmax(const float* z, int64_t n, float* out, void* scratch, cudaStream_t stream);
int32_t tw_vec_readout_parts(void);
int tw_vec_readout(const void* w, int32_t wdtype, const void* v, int32_t vdtype, int64_t n, int32_t d,
                   const int64_t* idx, int64_t m, int32_t renorm, void* out, double* partial, double* mass_out,
                   cudaStream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TWILIGHT_H_ */
