// C-ABI glue: version and the fused one-layer decode step.
#include "common.cuh"

extern "C" int32_t tw_version(void) { return 100; }  // 0.1.0

int tw_select_append(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                     const int32_t* positions, const tw_decode_params* prm, const tw_decode_buffers* buf,
                     cudaStream_t stream);  // quest.cu
int tw_attn_geometry(const tw_paged_kv* kv, int chunk);  // attention.cu
int tw_unit_step_applies(const tw_paged_kv* kv, const tw_decode_params* prm, const tw_decode_buffers* buf,
                         const int32_t* positions);  // unit.cu

extern "C" int tw_decode_step(const tw_paged_kv* kv, const void* q, const void* k_new, const void* v_new,
                              const int32_t* positions, const tw_decode_params* prm,
                              const tw_decode_buffers* buf, float* out, cudaStream_t stream) {
  if (!kv || !prm || !buf || !out) return TW_ERR_INVALID;
  // reject a bad attention geometry before K1 appends and advances seq_lens
  if (int s = tw_attn_geometry(kv, prm->chunk_tokens > 0 ? prm->chunk_tokens : TW_DEFAULT_CHUNK)) return s;
  if (prm->renormalize != 1) return TW_ERR_INVALID;
  if (tw_unit_step_applies(kv, prm, buf, nullptr)) {  // K1..K3 in one per-unit launch (unit.cu)
    int s;
    if (positions == kv->seq_lens) {  // aliased: every CTA of a sequence must see the same position
      if ((s = tw_quant_append(kv, k_new, v_new, positions, stream))) return s;
      s = tw_select_estimate_topp(kv, q, nullptr, nullptr, nullptr, prm, buf, stream);
    } else {
      s = tw_select_estimate_topp(kv, q, k_new, v_new, positions, prm, buf, stream);
    }
    if (s) return s;
    return tw_sparse_attention(kv, q, prm, buf, out, stream);
  }
  int s = tw_select_append(kv, q, k_new, v_new, positions, prm, buf, stream);  // K1 fused into the Quest filter
  if (s == tw::TW_FUSE_UNAVAILABLE) {
    if ((s = tw_quant_append(kv, k_new, v_new, positions, stream))) return s;
    s = tw_select(kv, q, prm, buf, stream);
  }
  if (s) return s;
  if ((s = tw_estimate(kv, q, prm, buf, stream))) return s;
  if ((s = tw_topp(kv, prm, buf, stream))) return s;
  return tw_sparse_attention(kv, q, prm, buf, out, stream);
}
