#pragma once
#include "qcache.cuh"

namespace tkv {
// records a launch on `layer` (its len pointer) in `st`; false when the
// stream's previous sparse-layer launch was on the same layer (no PDL then)
bool pdl_note(cudaStream_t st, const void *layer);
int sparse_prefill(const SL &s, const uint16_t *keys, const uint16_t *values, int64_t n, cudaStream_t st);
int sparse_append(const SL &s, const uint16_t *nk, const uint16_t *nv, cudaStream_t st);
int64_t stage1_workspace(int B, int hq, int H, int d);
int stage1(const uint16_t *hidden, const uint16_t *w_q, int B, int hq, int H, int d, int G, const float *chmax,
           int d_s, double *q_hat, int32_t *channels, void *ws, cudaStream_t st, const SL *prefetch = nullptr);
int64_t select_workspace(int units, int64_t cap);
int select_tokens(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s, int n_local,
                  int n_topk, int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count, double *scores_out,
                  void *ws, cudaStream_t st);
int topk_from_scores(const double *scores, int units, int64_t n, int n_local, int n_topk, int32_t *sel_idx,
                     int32_t *sel_count, void *ws, cudaStream_t st);
int64_t sparse_attn_workspace(int units, int G, int d, int max_rows);
int sparse_attention(const SL &s, const uint16_t *queries, int G, const int32_t *sel_idx, const int32_t *sel_count,
                     int n_local, int max_rows, int keys_from_device, float *out, void *ws, cudaStream_t st);
bool sparse_decode_supported(const SL &s, int G, int n_local);
int max_active_clusters(int d, int G);
int last_cluster_size();  // cluster size the last sparse_decode_fused dispatch chose (8, 4 or 2)
int choose_cluster(const SL &s, int G, int n_local);  // the cluster size sparse_decode_fused picks
#define TKV_FZ_VARIANT_DECLS                                                                                      \
  bool sparse_decode_supported(const SL &s, int G, int n_local);                                                 \
  int max_active_clusters(int d, int G);                                                                         \
  int sparse_decode_fused(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s,          \
                          int n_local, int n_topk, int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count,    \
                          int keys_from_device, float *out, const uint16_t *new_keys, const uint16_t *new_values, \
                          cudaStream_t st);
namespace fz4 {  // the same kernel with 4-CTA clusters (sparse_fused.cu built with TKV_FZ_CTAS=4)
TKV_FZ_VARIANT_DECLS
}  // namespace fz4
namespace fz2 {  // and with 2-CTA clusters (TKV_FZ_CTAS=2)
TKV_FZ_VARIANT_DECLS
}  // namespace fz2
namespace wide {  // the wide decode (sparse_wide.cu): P CTAs per unit, for few units per GPU
bool supported(const SL &s, int G, int n_local, int d_s, int keys_from_device, bool cluster_ok);
int64_t ctl_bytes(int units, int d);      // per-unit counters + histograms (zero between launches)
int64_t scratch_bytes(int units, int d);  // per-unit headers, lists, partials
int parts_for(int units);
int decode(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s, int n_local, int n_topk,
           int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count, int keys_from_device, float *out,
           const uint16_t *new_keys, const uint16_t *new_values, void *ctl, void *scratch, cudaStream_t st);
}  // namespace wide
int sparse_decode_fused(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s, int n_local,
                        int n_topk, int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count, int keys_from_device,
                        float *out, const uint16_t *new_keys, const uint16_t *new_values, cudaStream_t st);
int64_t fidelity_workspace(int units, int G, int64_t n, int k);
int sparse_fidelity(const SL &s, const uint16_t *queries, int G, int64_t n, const int32_t *sel_idx,
                    const int32_t *sel_count, int sel_stride, int k, float *exact_out, double *metrics, void *ws,
                    cudaStream_t st);
int uva_probe(const void *host, size_t bytes, int row_bytes, const int32_t *rows, int nrows, float *sink,
              cudaStream_t st);
int64_t calibrate_workspace(int hq, int n_q, int64_t n);
int dense_preference(const uint16_t *queries, const uint16_t *keys, int hq, int h, int n_q, int64_t n, int d,
                     int64_t k, double *head_scores, void *ws, cudaStream_t st);
}  // namespace tkv
