#include <algorithm>
// extern "C" boundary: argument validation, status codes (errors.py:9-38),
// dispatch to the kernels.  See include/tailorkv.h.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "common.cuh"
#include "qcache.cuh"
#include "sparse.cuh"

namespace tkv {

static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

int check_launch(const char *what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TKV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return TKV_OK;
}

// Programmatic dependent launch guard.  The fused sparse kernel reads its
// layer's token count and starts its scorer loads before griddepcontrol.wait,
// and triggers its dependents before its own append.  That is only safe when
// the kernel ahead of it in the stream is NOT a launch on the same layer: for
// any other predecessor P, P itself passed its wait only after everything
// before it completed, so the layer's last writer has finished.  Every launch
// that touches a sparse layer notes (stream, layer) here; a fused launch whose
// stream's previous note is the same layer goes without the PDL attribute.
static std::mutex g_pdl_mu;
static std::unordered_map<cudaStream_t, const void *> g_pdl_last;

bool pdl_note(cudaStream_t st, const void *layer) {
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  const void *&last = g_pdl_last[st];
  const bool ok = last != layer;
  last = layer;
  return ok;
}

static int validate_qcache(const tkv_qcache *c) {
  TKV_REQUIRE(c != nullptr, TKV_ERR_PARAMETER, "null cache");
  TKV_REQUIRE(c->bits == 1 || c->bits == 2, TKV_ERR_PARAMETER, "bits must be one of (1, 2)");
  TKV_REQUIRE(c->d >= 32 && c->d <= 256 && c->d % 32 == 0, TKV_ERR_SHAPE,
              "head_dim must be a multiple of 32 in [32, 256] on the CUDA path");
  TKV_REQUIRE(c->g == 16 || c->g == 32 || c->g == 64 || (c->g == 128 && c->bits == 1), TKV_ERR_PARAMETER,
              "group_size must be 16, 32 or 64 (128 at 1 bit) on the CUDA path");
  TKV_REQUIRE(c->units >= 1, TKV_ERR_SHAPE, "units must be >= 1");
  TKV_REQUIRE(c->capacity % key_tile_tokens(c->bits) == 0 && c->capacity % c->g == 0, TKV_ERR_PARAMETER,
              "capacity must be a multiple of the key tile");
  return TKV_OK;
}

}  // namespace tkv

using namespace tkv;

extern "C" {

const char *tkv_last_error(void) { return g_err.c_str(); }
int tkv_abi_version(void) { return 1; }

int tkv_graph_instantiate(void *graph, void **exec) {
  cudaGraphExec_t e = nullptr;
  const cudaError_t r = cudaGraphInstantiateWithFlags(&e, static_cast<cudaGraph_t>(graph),
                                                      cudaGraphInstantiateFlagUseNodePriority);
  if (r != cudaSuccess) return fail(TKV_ERR_CUDA, std::string("tkv_graph_instantiate: ") + cudaGetErrorString(r));
  *exec = e;
  return TKV_OK;
}

int tkv_graph_launch(void *exec, void *stream) {
  const cudaError_t r = cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), as_stream(stream));
  if (r != cudaSuccess) return fail(TKV_ERR_CUDA, std::string("tkv_graph_launch: ") + cudaGetErrorString(r));
  return TKV_OK;
}

int tkv_graph_destroy(void *exec) {
  cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec));
  return TKV_OK;
}

int tkv_event_record(void *event, void *stream, int32_t external) {
  const cudaError_t e = external ? cudaEventRecordWithFlags(static_cast<cudaEvent_t>(event), as_stream(stream),
                                                            cudaEventRecordExternal)
                                 : cudaEventRecord(static_cast<cudaEvent_t>(event), as_stream(stream));
  if (e != cudaSuccess) return fail(TKV_ERR_CUDA, std::string("tkv_event_record: ") + cudaGetErrorString(e));
  return TKV_OK;
}

int tkv_qcache_sizes(int32_t units, int32_t d, int32_t bits, int32_t g, int64_t capacity, int64_t sizes[6],
                     int32_t *tile) {
  tkv_qcache c{};
  c.units = units; c.d = d; c.bits = bits; c.g = g; c.capacity = capacity;
  const int Tk = (bits == 1 || bits == 2) ? key_tile_tokens(bits) : 1;
  if (tile) *tile = Tk > g ? Tk : g;
  if (int r = validate_qcache(&c)) return r;
  const int nb = (d + g - 1) / g;
  sizes[0] = (int64_t)units * (capacity / Tk) * (d / 32) * 128 * 4;
  sizes[1] = (int64_t)units * (capacity / g) * d * 4;
  sizes[2] = (int64_t)units * g * d * 2;
  sizes[3] = (int64_t)units * (capacity / 32) * val_sets(d, bits) * 128 * 4;
  sizes[4] = (int64_t)units * capacity * nb * 4;
  sizes[5] = (int64_t)units * 8;  // [units][2]: max value scale, max key scale
  return TKV_OK;
}

int tkv_qcache_pack(const tkv_qcache *c, const uint16_t *keys, const uint16_t *values, int64_t n,
                    int32_t check_finite, void *stream) {
  if (int r = validate_qcache(c)) return r;
  TKV_REQUIRE(n >= 1, TKV_ERR_EMPTY_CACHE, "cannot quantize an empty cache");
  TKV_REQUIRE(n <= c->capacity, TKV_ERR_SHAPE, "sequence longer than the cache capacity");
  return pack(*c, keys, values, n, check_finite, as_stream(stream));
}

int tkv_qcache_append(const tkv_qcache *c, const uint16_t *nk, const uint16_t *nv, void *stream) {
  if (int r = validate_qcache(c)) return r;
  return append(*c, nk, nv, as_stream(stream));
}

int64_t tkv_qcache_export_size(const tkv_qcache *c, int32_t which, int64_t n) { return export_size(*c, which, n); }

int tkv_qcache_export(const tkv_qcache *c, int32_t unit, int32_t which, int64_t n, uint8_t *out, void *stream) {
  if (int r = validate_qcache(c)) return r;
  TKV_REQUIRE(unit >= 0 && unit < c->units, TKV_ERR_PARAMETER, "unit out of range");
  TKV_REQUIRE(which == 0 || which == 1, TKV_ERR_PARAMETER, "which must be 0 (keys) or 1 (values)");
  return export_blob(*c, unit, which, n, out, as_stream(stream));
}

int tkv_qcache_dequant(const tkv_qcache *c, int32_t unit, int32_t which, int64_t n, float *out, void *stream) {
  if (int r = validate_qcache(c)) return r;
  TKV_REQUIRE(unit >= 0 && unit < c->units, TKV_ERR_PARAMETER, "unit out of range");
  return dequant(*c, unit, which, n, out, as_stream(stream));
}

int64_t tkv_quant_decode_workspace(const tkv_qcache *c, int32_t G) { return quant_decode_workspace(*c, G); }

int tkv_quant_decode(const tkv_qcache *c, const uint16_t *queries, int32_t G, float *out, void *workspace,
                     int32_t impl, void *stream) {
  if (int r = validate_qcache(c)) return r;
  TKV_REQUIRE(G >= 1 && G <= 16, TKV_ERR_SHAPE, "query heads per KV head must be in [1, 16]");
  return quant_decode(*c, queries, G, out, workspace, impl, as_stream(stream));
}

int tkv_qgemv_scores(const tkv_qcache *c, int32_t unit, int64_t n, const double *query, double *logits,
                     void *stream) {
  if (int r = validate_qcache(c)) return r;
  TKV_REQUIRE(unit >= 0 && unit < c->units, TKV_ERR_PARAMETER, "unit out of range");
  TKV_REQUIRE(n >= 1 && n <= c->capacity, TKV_ERR_EMPTY_CACHE, "token count out of range");
  return qgemv_scores(*c, unit, n, query, logits, as_stream(stream));
}

int64_t tkv_qgemv_output_workspace(const tkv_qcache *c, int64_t n) { return qgemv_output_workspace(*c, n); }

int tkv_qgemv_output(const tkv_qcache *c, int32_t unit, int64_t n, const double *weights, double *out,
                     void *workspace, void *stream) {
  if (int r = validate_qcache(c)) return r;
  TKV_REQUIRE(unit >= 0 && unit < c->units, TKV_ERR_PARAMETER, "unit out of range");
  TKV_REQUIRE(n >= 1 && n <= c->capacity, TKV_ERR_EMPTY_CACHE, "token count out of range");
  return qgemv_output(*c, unit, n, weights, out, workspace, as_stream(stream));
}

int tkv_qcache_import(const tkv_qcache *c, int32_t unit, int32_t which, const uint8_t *blob, int64_t blob_len,
                      uint8_t *device_ws, void *stream) {
  if (int r = validate_qcache(c)) return r;
  TKV_REQUIRE(unit >= 0 && unit < c->units, TKV_ERR_PARAMETER, "unit out of range");
  TKV_REQUIRE(which == 0 || which == 1, TKV_ERR_PARAMETER, "which must be 0 (keys) or 1 (values)");
  TKV_REQUIRE(blob != nullptr && blob_len >= 24, TKV_ERR_ENCODING, "quantized tensor blob truncated");
  TKV_REQUIRE(std::memcmp(blob, "GQT1", 4) == 0, TKV_ERR_ENCODING, "bad quantized tensor magic");
  auto u32 = [&](int o) {
    return (uint32_t)blob[o] | ((uint32_t)blob[o + 1] << 8) | ((uint32_t)blob[o + 2] << 16) |
           ((uint32_t)blob[o + 3] << 24);
  };
  const int bits = blob[4], axis = blob[5], g = blob[6] | (blob[7] << 8);
  const int64_t rows = u32(8), d = u32(12), res_rows = u32(16), packed_len = u32(20);
  TKV_REQUIRE(axis == (which == 0 ? 1 : 2), TKV_ERR_ENCODING, "blob axis does not match keys/values");
  TKV_REQUIRE(bits == c->bits && g == c->g && d == c->d, TKV_ERR_ENCODING,
              "blob bits / group size / head_dim differ from the cache");
  TKV_REQUIRE(packed_len == (rows * d * bits + 7) / 8, TKV_ERR_ENCODING, "packed code section has the wrong length");
  TKV_REQUIRE(which == 0 ? rows % g == 0 && res_rows < g : res_rows == 0, TKV_ERR_ENCODING,
              "row counts inconsistent with the group size");
  const int64_t grid = which == 0 ? (rows / g) * d : rows * ((d + g - 1) / g);
  const int64_t need = 24 + packed_len + 4 * grid + 2 * res_rows * d;
  TKV_REQUIRE(blob_len >= need, TKV_ERR_ENCODING, "parameter or residual section truncated");
  TKV_REQUIRE(rows + res_rows <= c->capacity, TKV_ERR_SHAPE, "blob longer than the cache capacity");
  TKV_REQUIRE(device_ws != nullptr, TKV_ERR_PARAMETER, "device workspace of blob_len bytes required");
  cudaStream_t st = as_stream(stream);
  if (cudaMemcpyAsync(device_ws, blob, need, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return check_launch("tkv_qcache_import (copy)");
  int r = import_blob(*c, unit, which, device_ws, rows, res_rows, packed_len, st);
  if (r == TKV_OK && cudaStreamSynchronize(st) != cudaSuccess) return check_launch("tkv_qcache_import");
  return r;
}

int tkv_attention_f64(const double *queries, int32_t rows, const double *keys, const double *values, int64_t n,
                      int32_t d, const int64_t *sel, int64_t m, double *workspace, double *weights, double *out,
                      void *stream) {
  TKV_REQUIRE(rows >= 1 && d >= 1, TKV_ERR_SHAPE, "attention needs at least one query row");
  TKV_REQUIRE(n >= 1 && m >= 1, TKV_ERR_EMPTY_CACHE, "attention over an empty cache");
  TKV_REQUIRE(workspace != nullptr, TKV_ERR_PARAMETER, "workspace of rows * m doubles required");
  return attention_f64(queries, rows, keys, values, n, d, sel, m, workspace, weights, out, as_stream(stream));
}

int tkv_approx_scores_f64(const double *query_critical, int32_t G, const double *critical_keys, int64_t n,
                          int32_t d_s, double *out, void *stream) {
  TKV_REQUIRE(G >= 1 && d_s >= 1 && d_s <= 4096 && n >= 0, TKV_ERR_SHAPE, "bad approx_scores shape");
  if (n == 0) return TKV_OK;
  return approx_scores_f64(query_critical, G, critical_keys, n, d_s, out, as_stream(stream));
}

int tkv_channel_select_f64(const double *q_hat, int32_t G, const double *channel_abs_max, int32_t d, int32_t d_s,
                           double *scores, int32_t *selected, void *stream) {
  TKV_REQUIRE(G >= 1 && d >= 1 && d <= 4096, TKV_ERR_SHAPE, "bad channel-score shape");
  TKV_REQUIRE(d_s >= 1 && d_s <= d, TKV_ERR_PARAMETER, "d_s must lie in [1, head_dim]");
  return channel_select_f64(q_hat, G, channel_abs_max, d, d_s, scores, selected, as_stream(stream));
}

int tkv_host_gather(const tkv_sparse_layer *s, int32_t unit, const int64_t *indices, int64_t m, uint16_t *out_keys,
                    uint16_t *out_values, void *stream) {
  TKV_REQUIRE(s != nullptr && s->host_kv != nullptr, TKV_ERR_PARAMETER, "layer has no host store");
  TKV_REQUIRE(unit >= 0 && unit < s->units, TKV_ERR_PARAMETER, "unit out of range");
  TKV_REQUIRE(s->d % 8 == 0, TKV_ERR_SHAPE, "head_dim must be a multiple of 8");
  return host_gather(*s, unit, indices, m, out_keys, out_values, as_stream(stream));
}

int tkv_sum_at(const double *w, const int32_t *indices, const int32_t *count, double *out, void *stream) {
  return sum_at(w, indices, count, out, as_stream(stream));
}

static int validate_sparse(const tkv_sparse_layer *s) {
  TKV_REQUIRE(s != nullptr, TKV_ERR_PARAMETER, "null layer");
  TKV_REQUIRE(s->d >= 32 && s->d <= 256 && s->d % 32 == 0, TKV_ERR_SHAPE,
              "head_dim must be a multiple of 32 in [32, 256] on the CUDA path");
  TKV_REQUIRE(s->units >= 1 && s->capacity >= 1, TKV_ERR_SHAPE, "empty layer");
  TKV_REQUIRE(s->host_kv != nullptr, TKV_ERR_PARAMETER, "layer has no host store");
  return TKV_OK;
}

int tkv_sparse_prefill(const tkv_sparse_layer *s, const uint16_t *keys, const uint16_t *values, int64_t n,
                       void *stream) {
  if (int r = validate_sparse(s)) return r;
  TKV_REQUIRE(n >= 1, TKV_ERR_EMPTY_CACHE, "cannot offload an empty cache");
  TKV_REQUIRE(n <= s->capacity, TKV_ERR_SHAPE, "sequence longer than the layer capacity");
  TKV_REQUIRE(s->local_offset >= 0 && s->local_offset <= n, TKV_ERR_PARAMETER, "bad local offset");
  pdl_note(as_stream(stream), s->len);
  return sparse_prefill(*s, keys, values, n, as_stream(stream));
}

int tkv_sparse_append(const tkv_sparse_layer *s, const uint16_t *nk, const uint16_t *nv, void *stream) {
  if (int r = validate_sparse(s)) return r;
  pdl_note(as_stream(stream), s->len);
  return sparse_append(*s, nk, nv, as_stream(stream));
}

int64_t tkv_stage1_workspace(int32_t B, int32_t hq, int32_t hidden, int32_t d) {
  return stage1_workspace(B, hq, hidden, d);
}

int tkv_stage1(const uint16_t *hidden, const uint16_t *w_q, int32_t B, int32_t hq, int32_t hidden_dim, int32_t d,
               int32_t G, const float *chmax, int32_t d_s, double *q_hat, int32_t *channels, void *workspace,
               void *stream) {
  TKV_REQUIRE(B >= 1 && B <= 1024, TKV_ERR_SHAPE, "batch must be in [1, 1024] for stage 1");
  TKV_REQUIRE(d >= 32 && d <= 256 && d % 32 == 0, TKV_ERR_SHAPE, "head_dim must be a multiple of 32 in [32,256]");
  TKV_REQUIRE(G >= 1 && hq % G == 0, TKV_ERR_SHAPE, "query heads not divisible by the group size");
  TKV_REQUIRE(d_s >= 1 && d_s <= d, TKV_ERR_PARAMETER, "d_s must lie in [1, head_dim]");
  return stage1(hidden, w_q, B, hq, hidden_dim, d, G, chmax, d_s, q_hat, channels, workspace, as_stream(stream));
}

int tkv_stage1_prefetch(const uint16_t *hidden, const uint16_t *w_q, int32_t B, int32_t hq, int32_t hidden_dim,
                        int32_t d, int32_t G, const float *chmax, int32_t d_s, double *q_hat, int32_t *channels,
                        void *workspace, const tkv_sparse_layer *layer, void *stream) {
  TKV_REQUIRE(B >= 1 && B <= 1024, TKV_ERR_SHAPE, "batch must be in [1, 1024] for stage 1");
  TKV_REQUIRE(d >= 32 && d <= 256 && d % 32 == 0, TKV_ERR_SHAPE, "head_dim must be a multiple of 32 in [32,256]");
  TKV_REQUIRE(G >= 1 && hq % G == 0, TKV_ERR_SHAPE, "query heads not divisible by the group size");
  TKV_REQUIRE(d_s >= 1 && d_s <= d, TKV_ERR_PARAMETER, "d_s must lie in [1, head_dim]");
  if (layer) {
    if (int r = validate_sparse(layer)) return r;
    TKV_REQUIRE(layer->d == d && layer->units == B * (hq / G), TKV_ERR_SHAPE, "prefetch layer does not match stage 1");
  }
  return stage1(hidden, w_q, B, hq, hidden_dim, d, G, chmax, d_s, q_hat, channels, workspace, as_stream(stream),
                layer);
}

int64_t tkv_select_workspace(int32_t units, int64_t capacity) { return select_workspace(units, capacity); }

int tkv_select_tokens(const tkv_sparse_layer *s, const uint16_t *queries, int32_t G, const int32_t *channels,
                      int32_t d_s, int32_t n_local, int32_t n_topk, int32_t *sel_idx, int32_t *sel_count,
                      int32_t *fetch_count, double *scores_out, void *workspace, void *stream) {
  if (int r = validate_sparse(s)) return r;
  TKV_REQUIRE(n_local >= 0, TKV_ERR_PARAMETER, "n_local must be >= 0");
  TKV_REQUIRE(n_topk >= 1, TKV_ERR_PARAMETER, "n_topk must be >= 1");
  TKV_REQUIRE(d_s >= 1 && d_s <= s->d && d_s <= 128, TKV_ERR_PARAMETER, "d_s must lie in [1, min(head_dim,128)]");
  return select_tokens(*s, queries, G, channels, d_s, n_local, n_topk, sel_idx, sel_count, fetch_count, scores_out,
                       workspace, as_stream(stream));
}

int tkv_topk_from_scores(const double *scores, int32_t units, int64_t n, int32_t n_local, int32_t n_topk,
                         int32_t *sel_idx, int32_t *sel_count, void *workspace, void *stream) {
  TKV_REQUIRE(n >= 1, TKV_ERR_EMPTY_CACHE, "token selection over an empty cache");
  TKV_REQUIRE(n_local >= 0 && n_topk >= 1, TKV_ERR_PARAMETER, "token budgets out of range");
  return topk_from_scores(scores, units, n, n_local, n_topk, sel_idx, sel_count, workspace, as_stream(stream));
}

// byte sizes of the wide decode's regions at the front of the decode workspace
static void decode_ws_parts(int units, int d, int64_t *ctl_b, int64_t *scr_b) {
  *ctl_b = (wide::ctl_bytes(units, d) + 255) / 256 * 256;
  *scr_b = (wide::scratch_bytes(units, d) + 255) / 256 * 256;
}

// which kernel tkv_sparse_decode would dispatch for these arguments (same encoding as below), no launch
int tkv_sparse_decode_plan(const tkv_sparse_layer *s, int32_t G, int32_t d_s, int32_t n_local,
                           int32_t keys_from_device) {
  if (validate_sparse(s)) return -2;
  const bool cl = sparse_decode_supported(*s, G, n_local);
  if (wide::supported(*s, G, n_local, d_s, keys_from_device, cl)) return 0;
  return cl ? choose_cluster(*s, G, n_local) : -1;
}

// which kernel the last tkv_sparse_decode dispatched: cluster size (8, 4, 2) of the fused cluster kernel,
// 0 the wide decode, -1 the unfused three-launch path (host-side dispatch; a captured graph keeps it)
static int g_sparse_path = -2;
int tkv_debug_sparse_path(void) { return g_sparse_path; }

int tkv_sparse_decode(const tkv_sparse_layer *s, const uint16_t *queries, int32_t G, const int32_t *channels,
                      int32_t d_s, int32_t n_local, int32_t n_topk, int32_t *sel_idx, int32_t *sel_count,
                      int32_t *fetch_count, int32_t keys_from_device, const uint16_t *new_keys,
                      const uint16_t *new_values, float *out, void *workspace, void *stream) {
  if (int r = validate_sparse(s)) return r;
  TKV_REQUIRE(n_local >= 0 && n_local <= 4096, TKV_ERR_PARAMETER, "n_local must lie in [0, 4096]");
  TKV_REQUIRE(n_topk >= 1, TKV_ERR_PARAMETER, "n_topk must be >= 1");
  TKV_REQUIRE(d_s >= 1 && d_s <= s->d && d_s <= 128, TKV_ERR_PARAMETER, "d_s must lie in [1, min(head_dim,128)]");
  TKV_REQUIRE(G >= 1 && G <= 8, TKV_ERR_SHAPE, "group size must lie in [1, 8]");
  TKV_REQUIRE((new_keys == nullptr) == (new_values == nullptr), TKV_ERR_PARAMETER,
              "new_keys and new_values must both be given or both be NULL");
  // workspace: [wide counters | wide scratch | the unfused path's region] (decode_ws_parts)
  int64_t ctl_b, scr_b;
  decode_ws_parts(s->units, s->d, &ctl_b, &scr_b);
  char *ws0 = static_cast<char *>(workspace);
  if (wide::supported(*s, G, n_local, d_s, keys_from_device, sparse_decode_supported(*s, G, n_local))) {
    TKV_REQUIRE(s->s1_ready == nullptr, TKV_ERR_PARAMETER,
                "the stage-1 handshake (s1_ready) needs the fused cluster decode, not the wide decode");
    g_sparse_path = 0;
    return wide::decode(*s, queries, G, channels, d_s, n_local, n_topk, sel_idx, sel_count, fetch_count,
                        keys_from_device, out, new_keys, new_values, ws0, ws0 + ctl_b, as_stream(stream));
  }
  if (sparse_decode_supported(*s, G, n_local)) {
    const int r = sparse_decode_fused(*s, queries, G, channels, d_s, n_local, n_topk, sel_idx, sel_count,
                                      fetch_count, keys_from_device, out, new_keys, new_values, as_stream(stream));
    g_sparse_path = last_cluster_size();
    return r;
  }
  g_sparse_path = -1;
  // shapes outside the fused kernels: select, then gather + attention, then the append (three launches)
  TKV_REQUIRE(s->s1_ready == nullptr, TKV_ERR_PARAMETER,
              "the stage-1 handshake (s1_ready) needs the fused cluster decode");
  TKV_REQUIRE(s->n_sink == 0, TKV_ERR_PARAMETER, "attention sinks need the fused sparse decode (shape unsupported)");
  pdl_note(as_stream(stream), s->len);
  char *ws = ws0 + ctl_b + scr_b;
  const int64_t sel_ws = (select_workspace(s->units, s->capacity) + 255) / 256 * 256;
  if (int r = select_tokens(*s, queries, G, channels, d_s, n_local, n_topk, sel_idx, sel_count, fetch_count, nullptr,
                            ws, as_stream(stream)))
    return r;
  if (int r = sparse_attention(*s, queries, G, sel_idx, sel_count, n_local, n_local + n_topk, keys_from_device, out,
                               ws + sel_ws, as_stream(stream)))
    return r;
  return new_keys ? sparse_append(*s, new_keys, new_values, as_stream(stream)) : TKV_OK;
}

int64_t tkv_sparse_fidelity_workspace(int32_t units, int32_t G, int64_t n, int32_t k) {
  return fidelity_workspace(units, G, n, k);
}

int tkv_sparse_fidelity(const tkv_sparse_layer *s, const uint16_t *queries, int32_t G, int64_t n,
                        const int32_t *sel_idx, const int32_t *sel_count, int32_t sel_stride, int32_t k,
                        float *exact_out, double *metrics, void *workspace, void *stream) {
  if (int r = validate_sparse(s)) return r;
  TKV_REQUIRE(n >= 1 && n <= s->capacity, TKV_ERR_EMPTY_CACHE, "fidelity over an empty or oversized prefix");
  TKV_REQUIRE(k >= 1, TKV_ERR_PARAMETER, "k must be >= 1");
  return sparse_fidelity(*s, queries, G, n, sel_idx, sel_count, sel_stride, (int)std::min<int64_t>(k, n), exact_out,
                         metrics, workspace, as_stream(stream));
}

int64_t tkv_sparse_decode_workspace(int32_t units, int64_t capacity, int32_t G, int32_t d, int32_t max_rows) {
  int64_t ctl_b, scr_b;
  decode_ws_parts(units, d, &ctl_b, &scr_b);
  return ctl_b + scr_b + (select_workspace(units, capacity) + 255) / 256 * 256 +
         sparse_attn_workspace(units, G, d, max_rows);
}

int64_t tkv_sparse_attn_workspace(int32_t units, int32_t G, int32_t d, int32_t max_rows) {
  return sparse_attn_workspace(units, G, d, max_rows);
}

int tkv_sparse_attention(const tkv_sparse_layer *s, const uint16_t *queries, int32_t G, const int32_t *sel_idx,
                         const int32_t *sel_count, int32_t n_local, int32_t max_rows, int32_t keys_from_device,
                         float *out, void *workspace, void *stream) {
  if (int r = validate_sparse(s)) return r;
  pdl_note(as_stream(stream), s->len);
  return sparse_attention(*s, queries, G, sel_idx, sel_count, n_local, max_rows, keys_from_device, out, workspace,
                          as_stream(stream));
}

void *tkv_host_store_create(size_t bytes, int32_t numa_node) {
  const size_t page = 2u << 20;
  const size_t len = (bytes + page - 1) / page * page;
  void *p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) {
    set_error("mmap failed for the host KV store");
    return nullptr;
  }
  madvise(p, len, MADV_HUGEPAGE);
  if (numa_node >= 0 && numa_node < 64) {
    unsigned long mask = 1ul << numa_node;
    // MPOL_BIND = 2; ignore failure (single-node hosts, no permission)
    syscall(SYS_mbind, p, len, 2, &mask, 64, 0);
  }
  memset(p, 0, len);  // first touch places pages on the bound node
  const cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(p, len);
    set_error(std::string("cudaHostRegister: ") + cudaGetErrorString(e));
    return nullptr;
  }
  return p;
}

int tkv_host_store_destroy(void *ptr, size_t bytes) {
  const size_t page = 2u << 20;
  const size_t len = (bytes + page - 1) / page * page;
  cudaHostUnregister(ptr);
  munmap(ptr, len);
  return TKV_OK;
}

int tkv_uva_read_probe(const void *host, size_t bytes, int32_t row_bytes, const int32_t *rows, int32_t nrows,
                       float *sink, void *stream) {
  TKV_REQUIRE(row_bytes % 16 == 0, TKV_ERR_PARAMETER, "row_bytes must be a multiple of 16");
  return uva_probe(host, bytes, row_bytes, rows, nrows, sink, as_stream(stream));
}

int64_t tkv_calibrate_workspace(int32_t hq, int32_t n_q, int64_t n) { return calibrate_workspace(hq, n_q, n); }

int tkv_dense_preference(const uint16_t *queries, const uint16_t *keys, int32_t hq, int32_t h, int32_t n_q,
                         int64_t n, int32_t d, int64_t k, double *head_scores, void *workspace, void *stream) {
  TKV_REQUIRE(h >= 1 && hq % h == 0, TKV_ERR_SHAPE, "query heads not divisible by kv heads");
  TKV_REQUIRE(n_q >= 1 && n_q <= n, TKV_ERR_PARAMETER, "probe n_q out of range");
  TKV_REQUIRE(k >= 1 && k <= n, TKV_ERR_PARAMETER, "k must lie in [1, n]");
  TKV_REQUIRE(d % 2 == 0 && d <= 256, TKV_ERR_SHAPE, "head_dim must be even and <= 256");
  return dense_preference(queries, keys, hq, h, n_q, n, d, k, head_scores, workspace, as_stream(stream));
}

}  // extern "C"
