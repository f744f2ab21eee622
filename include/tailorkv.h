/*
 * tailorkv.h -- C ABI of the B200-native TailorKV decode engine.
 *
 * Every entry point takes plain device/host pointers, integer sizes and a
 * cudaStream_t (passed as void*).  No torch types cross this boundary.  The
 * caller owns every buffer; the library never allocates on the decode path
 * (the only allocator is tkv_host_store_create, which owns its pinned arena).
 *
 * The reference (hybridkv, /root/reference/pkg/src/hybridkv) has no FFI: its
 * boundary is a Python API.  Each function below names the reference
 * function(s) it replaces; paper_2505_19586_b200/_lib.py is the ctypes binding
 * (the "reference-side binding" described in INTEGRATION.md).
 *
 * Status codes map 1:1 onto hybridkv/errors.py:9-38 classes.
 *
 * Device-resident counters: every cache keeps its token count in device memory
 * (int32 *len) so a whole decode step can be captured once in a CUDA graph and
 * replayed; appends advance the counter on the device.
 */
#ifndef TAILORKV_H_
#define TAILORKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TKV_OK = 0,
  TKV_ERR_SHAPE = 1,       /* ShapeError       (errors.py:13) */
  TKV_ERR_PARAMETER = 2,   /* ParameterError   (errors.py:25) */
  TKV_ERR_EMPTY_CACHE = 3, /* EmptyCacheError  (errors.py:17) */
  TKV_ERR_NUMERIC = 4,     /* NumericError     (errors.py:21) */
  TKV_ERR_ENCODING = 5,    /* EncodingError    (errors.py:29) */
  TKV_ERR_SCHEDULING = 6,  /* SchedulingError  (errors.py:33) */
  TKV_ERR_CUDA = 7         /* CUDA runtime failure (no reference counterpart) */
};

/* Last error message of the calling thread ("" when none). */
const char *tkv_last_error(void);
int tkv_abi_version(void);
/* Record a CUDA event on a stream; external != 0 makes the record a node of a
 * graph being captured on that stream (cudaEventRecordExternal), so kernels
 * can be timed inside a replayed decode-step graph. */
int tkv_event_record(void *event, void *stream, int32_t external);
/* Instantiate a captured decode-step graph (cudaGraph_t) so that kernel
 * nodes run at their launch priorities (the attention chain above stage 1 of
 * the next layer); launch / destroy the executable graph. */
int tkv_graph_instantiate(void *graph, void **exec);
int tkv_graph_launch(void *exec, void *stream);
int tkv_graph_destroy(void *exec);

/* ------------------------------------------------------------------------
 * Quantized layer cache (quantizer.py:187-497)
 * ------------------------------------------------------------------------
 * One cache holds `units` KV heads (units = batch * kv_heads on this rank).
 * Keys are per-channel groups of g tokens with an fp16 residual of < g rows
 * (quantizer.py:277-293); values are per-token groups of g channels
 * (quantizer.py:252-275).  Codes live in the MMA-native bit-plane layout
 * described in DESIGN.md section 3; tkv_qcache_export produces the
 * reference's GQT1 stream byte-for-byte.
 */
typedef struct tkv_qcache {
  int32_t units, d, bits, g;
  int64_t capacity;      /* tokens; multiple of the key tile (see tkv_qcache_sizes) */
  uint32_t *key_codes;   /* [units][capacity/Tk][d/32][32][4] */
  uint32_t *key_lohi;    /* half2(lo,hi) [units][capacity/g][d] */
  uint16_t *key_resid;   /* fp16 [units][g][d] */
  uint32_t *val_codes;   /* [units][capacity/32][sets][32][4] */
  uint32_t *val_lohi;    /* half2(lo,hi) [units][capacity][ceil(d/g)] */
  float *val_smax;       /* [units][2] running max group scale: [0] values, [1] keys */
  int32_t *len;          /* device scalar: tokens held (all units) */
  uint32_t *ticket;      /* device scalar scratch for append */
} tkv_qcache;

/* Byte sizes of each buffer of a cache (same order as the struct pointers:
 * key_codes, key_lohi, key_resid, val_codes, val_lohi, val_smax).  Returns the
 * token tile the capacity must be a multiple of in *tile. */
int tkv_qcache_sizes(int32_t units, int32_t d, int32_t bits, int32_t g, int64_t capacity,
                     int64_t sizes[6], int32_t *tile);

/* Prefill/compress: quantize keys/values [units][n][d] fp16 into an empty
 * cache (replaces quantize_layer_kv, quantizer.py:479-497).  Sets *len = n.
 * `check_finite` != 0 scans the input and fails with TKV_ERR_NUMERIC. */
int tkv_qcache_pack(const tkv_qcache *c, const uint16_t *keys, const uint16_t *values, int64_t n,
                    int32_t check_finite, void *stream);

/* Decode-step append of one token per unit (replaces
 * QuantizedLayerKV.append_token, quantizer.py:445-451). */
int tkv_qcache_append(const tkv_qcache *c, const uint16_t *new_keys, const uint16_t *new_values,
                      void *stream);

/* Export unit u as a GQT1 blob (replaces GroupQuantizedTensor.to_bytes,
 * quantizer.py:358-380).  `which` 0 = keys, 1 = values.  `out` is a DEVICE
 * buffer of at least tkv_qcache_export_size bytes; n is the host's copy of *len. */
int64_t tkv_qcache_export_size(const tkv_qcache *c, int32_t which, int64_t n);
int tkv_qcache_export(const tkv_qcache *c, int32_t unit, int32_t which, int64_t n, uint8_t *out,
                      void *stream);

/* Dequantize unit u to fp32 [n][d] (replaces GroupQuantizedTensor.dequantize,
 * quantizer.py:335-352); test/inspection helper. */
int tkv_qcache_dequant(const tkv_qcache *c, int32_t unit, int32_t which, int64_t n, float *out,
                       void *stream);

/* Quantized decode attention of one layer (replaces pipeline.py:331-337:
 * qgemv_scores quantizer.py:505-533 -> softmax(/sqrt d) -> qgemv_output
 * quantizer.py:536-558).  queries fp16 [units*G][d]; out fp32 [units*G][d].
 * `workspace` >= tkv_quant_decode_workspace bytes.  impl: 0 = auto,
 * 1 = reference-shaped SIMT kernel, 2 = tensor-core (IMMA) kernel, persistent
 * and TMA-pipelined, 3 = the per-chunk IMMA kernel it replaced. */
int64_t tkv_quant_decode_workspace(const tkv_qcache *c, int32_t G);
int tkv_quant_decode(const tkv_qcache *c, const uint16_t *queries, int32_t G, float *out,
                     void *workspace, int32_t impl, void *stream);

/* Raw quantized GEMVs for one unit (replace qgemv_scores quantizer.py:505-533
 * and qgemv_output :536-558), float64 like the reference: logits [n] of a
 * query [d] over the unit's keys (complete groups + fp16 residual rows), and
 * weights [n] @ the unit's dequantized values -> out [d].  Deterministic
 * (fixed-order reductions); qgemv_output needs a workspace of
 * tkv_qgemv_output_workspace bytes. */
int tkv_qgemv_scores(const tkv_qcache *c, int32_t unit, int64_t n, const double *query, double *logits,
                     void *stream);
int64_t tkv_qgemv_output_workspace(const tkv_qcache *c, int64_t n);
int tkv_qgemv_output(const tkv_qcache *c, int32_t unit, int64_t n, const double *weights, double *out,
                     void *workspace, void *stream);

/* GQT1 import (replaces GroupQuantizedTensor.from_bytes quantizer.py:383-422):
 * the HOST blob's codes, zero points / scales and key residual go into one
 * unit of the cache (which 0 = keys, PER_CHANNEL blob; 1 = values, PER_TOKEN)
 * and *len becomes the blob's row count.  device_ws: >= blob_len bytes of
 * device memory (staging).  Header/section checks raise TKV_ERR_ENCODING
 * like the reference.  Synchronous.  A blob exported from fp16 inputs
 * re-exports byte-identically. */
int tkv_qcache_import(const tkv_qcache *c, int32_t unit, int32_t which, const uint8_t *blob, int64_t blob_len,
                      uint8_t *device_ws, void *stream);

/* float64 helpers over caller device arrays for the reference-signature
 * API (paper_2505_19586_b200/hybridkv.py):
 * - attention: softmax(q K^T / sqrt(d)) per query row (kv_model.py:169-194),
 *   optionally over the index list sel[m] (sparse_attention retriever.py:214-226),
 *   weights [rows][m] and/or out = weights @ V [rows][d]; workspace rows*m doubles;
 * - approx_scores (retriever.py:166-189): critical_keys [n][d_s] @ sum_g q[g];
 * - channel selection (retriever.py:111-163): scores[c] = sum_g |q_hat[g][c]| *
 *   chmax[c] (channel_abs_max NULL: scores = q_hat[0][c] as given), top d_s
 *   with ties to the lower index, ascending;
 * - host gather (memsim.py:118-127): K and V rows of one unit from the pinned
 *   host store by UVA loads into device buffers [m][d];
 * - sum_at: sum of w[idx[i]] for i < *count (sparse_error's kept mass). */
int tkv_attention_f64(const double *queries, int32_t rows, const double *keys, const double *values, int64_t n,
                      int32_t d, const int64_t *sel, int64_t m, double *workspace, double *weights, double *out,
                      void *stream);
int tkv_approx_scores_f64(const double *query_critical, int32_t G, const double *critical_keys, int64_t n,
                          int32_t d_s, double *out, void *stream);
int tkv_channel_select_f64(const double *q_hat, int32_t G, const double *channel_abs_max, int32_t d, int32_t d_s,
                           double *scores, int32_t *selected, void *stream);
struct tkv_sparse_layer;
int tkv_host_gather(const struct tkv_sparse_layer *s, int32_t unit, const int64_t *indices, int64_t m, uint16_t *out_keys,
                    uint16_t *out_values, void *stream);
int tkv_sum_at(const double *w, const int32_t *indices, const int32_t *count, double *out, void *stream);

/* ------------------------------------------------------------------------
 * Sparsity-friendly layer (retriever.py:84-226, memsim.py:76-252)
 * ------------------------------------------------------------------------ */
typedef struct tkv_sparse_layer {
  int32_t units, d;
  int64_t capacity;       /* tokens */
  int64_t local_offset;   /* first token index held by the local mirror */
  int64_t local_capacity; /* rows of the local mirror */
  uint16_t *kt;           /* channel-major keys fp16 [units][d][capacity] (scorer) */
  float *chmax;           /* running max|K| [units][d] (memsim.py:93,109-111) */
  uint16_t *loc_k;        /* local mirror fp16 [units][local_capacity][d] */
  uint16_t *loc_v;
  uint16_t *kdev;         /* optional token-major device keys [units][capacity][d] or NULL */
  uint16_t *host_kv;      /* pinned host store [units][capacity][2][d] (K row | V row) */
  int32_t *len;           /* device scalar */
  uint32_t *ticket;       /* device scalar scratch */
  /* Optional HBM value-row cache (cache_slots == 0 disables it): a value row
   * fetched over PCIe stays in a slot until it has not been selected for
   * cache_window steps; a row selected again is read from HBM.  Rows never
   * change once written, so a cached (token, row) pair stays exact.  Needs
   * cache_slots >= cache_window * (n_local + n_topk). */
  int32_t cache_slots;    /* slots per unit */
  int32_t cache_window;   /* steps a selected row stays resident */
  int32_t *slot_tok;      /* [units][cache_slots] token held by the slot, -1 when empty */
  int32_t *slot_stamp;    /* [units][cache_slots] *len at the row's last selection */
  uint16_t *slot_v;       /* [units][cache_slots][2][d] cached (key | value) rows */
  int32_t *tok_slot;      /* [units][capacity] token -> slot, verified against slot_tok */
  unsigned long long *cache_stats; /* [2]: rows served from HBM, rows fetched over PCIe */
  /* Optional [units][4] float (16-byte aligned): per head, the last step's
   * top-k score threshold as a z-score of that step's scores and a running
   * mean of its step-to-step change (two spare floats); a hint that aims the
   * next step's threshold search (results never depend on it; NaN or NULL =
   * no hint). */
  float *thresh;
  /* [units][TKV_MAX_PARTS] (with cache_slots): per slot partition, the slot
   * the next allocation scan starts from (the cache's clock hand),
   * zero-initialised */
  int32_t *slot_hand;
  /* Attention-sink tokens (an extension; the reference has none, 0 = the
   * reference's selection): tokens [0, n_sink) are always selected besides
   * the local window and the n_topk best of [n_sink, n - n_local), so
   * sel_idx needs n_local + n_topk + n_sink entries per unit.  Fused decode
   * and cluster select only (other paths fail with TKV_ERR_PARAMETER). */
  int32_t n_sink;
  /* Optional [units][TKV_MAX_PARTS][2] float (NaN-initialised): the wide
   * decode's per-partition threshold hint (z-score of the last top-k
   * threshold against that partition's own score moments, running mean of
   * its step-to-step change).  Like `thresh`, it only aims the search. */
  float *part_hint;
  /* Optional [units] int32, zero-initialised: a device-side handshake with stage 1 that replaces a
   * stream/graph dependency of the decode on stage 1.  tkv_stage1 (given this layer as prefetch_layer)
   * stores 1 for a unit once its critical channels are written; the fused cluster decode waits for 1
   * before it reads the channels and stores 0 when it is done.  Only for decodes that leave SMs free for
   * stage 1 (the caller's choice; the wait is bounded: an error flag, never a hang).  NULL = none. */
  int32_t *s1_ready;
  /* stage-1 options for this layer: bit 0 = no scorer-column L2 prefetch */
  int32_t s1_flags;
} tkv_sparse_layer;

/* Token partitions per unit of the wide sparse decode (and slot_hand stride). */
#define TKV_MAX_PARTS 256

/* Prefill/offload (replaces HostPool.offload_layer memsim.py:88-93 and the
 * local mirror of pipeline.py:183-193): keys/values fp16 [units][n][d] on the
 * device.  Sets *len = n. */
int tkv_sparse_prefill(const tkv_sparse_layer *s, const uint16_t *keys, const uint16_t *values,
                       int64_t n, void *stream);
/* Append one token per unit (replaces HostPool.append memsim.py:106-111 and
 * the mirror append pipeline.py:412-413). */
int tkv_sparse_append(const tkv_sparse_layer *s, const uint16_t *new_keys, const uint16_t *new_values,
                      void *stream);

/* Stage 1 (replaces estimate_query retriever.py:84-108 + group_channel_scores
 * :138-148 + select_critical_channels :151-163, caller pipeline.py:271-286).
 * hidden fp16 [B][hidden]; w_q fp16 [hq][hidden][d] (this rank's q heads);
 * units = B * hq / G.  Writes q_hat f64 [B][hq][d] (may be NULL) and
 * channels int32 [units][d_s] sorted ascending.  The workspace must be zero
 * before its first use and belong to one (B, hq, hidden, d) shape: its
 * arrival counters re-arm themselves, so it can be reused (and replayed
 * from a CUDA graph) without clearing.  B > 2 with d in {64, 128, 256}
 * runs the tensor-core kernel (mma.sync, W_q read once per 16 sequences,
 * cluster reduction); otherwise the SIMT kernel. */
int64_t tkv_stage1_workspace(int32_t B, int32_t hq, int32_t hidden, int32_t d);
/* Stage 1 that also starts moving the selected channel rows of `layer`'s
 * channel-major scorer keys into L2 (TMA prefetch), so the layer's decode
 * scores from L2.  `layer` NULL = tkv_stage1. */
int tkv_stage1_prefetch(const uint16_t *hidden, const uint16_t *w_q, int32_t B, int32_t hq, int32_t hidden_dim,
                        int32_t d, int32_t G, const float *chmax, int32_t d_s, double *q_hat, int32_t *channels,
                        void *workspace, const tkv_sparse_layer *layer, void *stream);
int tkv_stage1(const uint16_t *hidden, const uint16_t *w_q, int32_t B, int32_t hq, int32_t hidden_dim,
               int32_t d, int32_t G, const float *chmax, int32_t d_s, double *q_hat, int32_t *channels,
               void *workspace, void *stream);

/* Stage 2 (replaces approx_scores retriever.py:166-189 + select_topk_tokens
 * :192-211): scores over the channel-major keys with the group-summed true
 * query, then the exact (score desc, index desc) top-k plus the local window.
 * sel_idx int32 [units][n_local+n_topk] ascending; sel_count/fetch_count
 * int32 [units] (fetch_count = selected indices below the local window). */
int64_t tkv_select_workspace(int32_t units, int64_t capacity);
int tkv_select_tokens(const tkv_sparse_layer *s, const uint16_t *queries, int32_t G, const int32_t *channels,
                      int32_t d_s, int32_t n_local, int32_t n_topk, int32_t *sel_idx, int32_t *sel_count,
                      int32_t *fetch_count, double *scores_out, void *workspace, void *stream);

/* Top-k selection over caller-provided f64 scores [units][n] (unit tests of
 * select_topk_tokens, retriever.py:192-211). */
int tkv_topk_from_scores(const double *scores, int32_t units, int64_t n, int32_t n_local, int32_t n_topk,
                         int32_t *sel_idx, int32_t *sel_count, void *workspace, void *stream);

/* Gather + sparse attention (replaces fetch_topk memsim.py:228-252 +
 * pipeline.py:364-376): rows below the local window come from the pinned host
 * store over PCIe (with keys_from_device != 0 only the value rows cross PCIe;
 * key rows come from kdev, or from the channel-major scorer copy kt when kdev
 * is NULL), the rest from the local mirror.  out fp32 [units*G][d]. */
int64_t tkv_sparse_attn_workspace(int32_t units, int32_t G, int32_t d, int32_t max_rows);
int tkv_sparse_attention(const tkv_sparse_layer *s, const uint16_t *queries, int32_t G, const int32_t *sel_idx,
                         const int32_t *sel_count, int32_t n_local, int32_t max_rows, int32_t keys_from_device,
                         float *out, void *workspace, void *stream);

/* Which kernel tkv_sparse_decode would run for these arguments (nothing is launched): the cluster size
 * (8, 4 or 2) of the fused cluster kernel, 0 the wide decode, -1 the unfused three-launch path, -2 an
 * invalid layer.  (A caller enabling the stage-1 handshake, tkv_sparse_layer.s1_ready, uses it to check
 * that the decode leaves SMs free.) */
int tkv_sparse_decode_plan(const tkv_sparse_layer *s, int32_t G, int32_t d_s, int32_t n_local,
                           int32_t keys_from_device);


/* One decode step of a sparsity-friendly layer in ONE launch (replaces
 * pipeline.py:351-376: approx_scores retriever.py:166-189 + select_topk_tokens
 * :192-211 + fetch_topk memsim.py:228-252 + sparse attention): proxy scores,
 * exact top-k plus the local window, gather (value rows over PCIe or from the
 * HBM row cache, key rows from HBM when keys_from_device != 0) and exact
 * softmax attention.  Outputs are those of tkv_select_tokens followed by
 * tkv_sparse_attention; `workspace` >= tkv_sparse_decode_workspace bytes, zero
 * before its first use (its tail holds the wide decode's per-unit barrier and
 * merge counters, which every launch leaves at zero again; the rest is
 * scratch).  With few units per GPU (units x partitions <= SMs) the decode
 * spreads each unit over several CTAs (the wide decode: one grid barrier per
 * unit on the common path); otherwise one thread-block cluster per unit.  With new_keys/new_values fp16
 * [units][d] (else NULL) the step's append (tkv_sparse_append) is fused into
 * the same launch, after the attention (attend-before-append,
 * pipeline.py:315-413). */
int64_t tkv_sparse_decode_workspace(int32_t units, int64_t capacity, int32_t G, int32_t d, int32_t max_rows);
int tkv_sparse_decode(const tkv_sparse_layer *s, const uint16_t *queries, int32_t G, const int32_t *channels,
                      int32_t d_s, int32_t n_local, int32_t n_topk, int32_t *sel_idx, int32_t *sel_count,
                      int32_t *fetch_count, int32_t keys_from_device, const uint16_t *new_keys,
                      const uint16_t *new_values, float *out, void *workspace, void *stream);
/* Fidelity metrics of one decode step of a sparsity-friendly layer against
 * exact attention over its first n tokens (replaces the oracle comparison of
 * pipeline.py:316-325, 377-403; kv_model.py:169-213; retriever.py:229-252):
 * exact_out fp32 [units*G][128] (exact softmax(qK^T/sqrt d)V, keys from HBM,
 * values from the host store), metrics f64 [units][2] = (recall@k of the
 * selection against the exact top-k group-weight tokens, selected attention
 * mass / G).  sel_idx/sel_count as written by tkv_sparse_decode; k = n_topk. */
int64_t tkv_sparse_fidelity_workspace(int32_t units, int32_t G, int64_t n, int32_t k);
int tkv_sparse_fidelity(const tkv_sparse_layer *s, const uint16_t *queries, int32_t G, int64_t n,
                        const int32_t *sel_idx, const int32_t *sel_count, int32_t sel_stride, int32_t k,
                        float *exact_out, double *metrics, void *workspace, void *stream);
/* Pinned, NUMA-local host arena for the KV store (memsim.py:76-135).  numa_node
 * < 0 leaves placement to the OS.  Returns a host pointer usable by kernels
 * (UVA) or NULL. */
void *tkv_host_store_create(size_t bytes, int32_t numa_node);
int tkv_host_store_destroy(void *ptr, size_t bytes);

/* PCIe H2D probe for the roofline: UVA zero-copy read kernel over `bytes` of a
 * pinned host buffer, rows of `row_bytes` at random row indices. */
int tkv_uva_read_probe(const void *host, size_t bytes, int32_t row_bytes, const int32_t *rows, int32_t nrows,
                       float *sink, void *stream);

/* ------------------------------------------------------------------------
 * Layer classification (identifier.py:89-187)
 * ------------------------------------------------------------------------
 * Per q head: mean over the n_q probe queries of (1 - top-k attention mass)
 * against all n keys of its KV head.  queries fp16 [hq][n_q][d], keys fp16
 * [h][n][d]; head_scores f64 [hq]. */
int64_t tkv_calibrate_workspace(int32_t hq, int32_t n_q, int64_t n);
int tkv_dense_preference(const uint16_t *queries, const uint16_t *keys, int32_t hq, int32_t h, int32_t n_q,
                         int64_t n, int32_t d, int64_t k, double *head_scores, void *workspace, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TAILORKV_H_ */
