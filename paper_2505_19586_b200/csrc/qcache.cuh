#pragma once
#include "common.cuh"

namespace tkv {

using QC = tkv_qcache;
using SL = tkv_sparse_layer;

int pack(const QC &c, const uint16_t *keys, const uint16_t *values, int64_t n, int check_finite, cudaStream_t st);
int append(const QC &c, const uint16_t *nk, const uint16_t *nv, cudaStream_t st);
int64_t export_size(const QC &c, int which, int64_t n);
int export_blob(const QC &c, int u, int which, int64_t n, uint8_t *out, cudaStream_t st);
int dequant(const QC &c, int u, int which, int64_t n, float *out, cudaStream_t st);
int qgemv_scores(const QC &c, int u, int64_t n, const double *q, double *logits, cudaStream_t st);
int64_t qgemv_output_workspace(const QC &c, int64_t n);
int qgemv_output(const QC &c, int u, int64_t n, const double *w, double *out, void *ws, cudaStream_t st);

// reference-signature surface (refops.cu)
int import_blob(const QC &c, int u, int which, const uint8_t *blob, int64_t rows, int64_t res_rows,
                int64_t packed_len, cudaStream_t st);
int attention_f64(const double *q, int rows, const double *keys, const double *values, int64_t n, int d,
                  const int64_t *sel, int64_t m, double *ws, double *weights, double *out, cudaStream_t st);
int approx_scores_f64(const double *qc, int G, const double *keys, int64_t n, int d_s, double *out, cudaStream_t st);
int channel_select_f64(const double *qhat, int G, const double *chmax, int d, int d_s, double *scores, int32_t *sel,
                       cudaStream_t st);
int host_gather(const SL &s, int u, const int64_t *idx, int64_t m, uint16_t *out_k, uint16_t *out_v, cudaStream_t st);
int sum_at(const double *w, const int32_t *idx, const int32_t *cnt, double *out, cudaStream_t st);

int64_t quant_decode_workspace(const QC &c, int G);
int64_t quant_decode_arrive_offset(const QC &c, int G);
int quant_decode(const QC &c, const uint16_t *q, int G, float *out, void *ws, int impl, cudaStream_t st);

// Split-K partial combine shared by the quantized and sparse attention paths:
// part_m/part_l [units][chunks][G], part_acc [units][chunks][G][d].
// chunk_count (device, per unit) may be NULL -> all `chunks` valid.
void launch_combine(const float *part_m, const float *part_l, const float *part_acc, int units, int chunks, int G,
                    int d, const int32_t *chunk_rows, int rows_per_chunk, float *out, cudaStream_t st);

void launch_combine_scalar(const float *pm, const float *pl, const float *pacc, int units, int chunks, int G, int d,
                           const int32_t *len, int rows_per_chunk, float *out, cudaStream_t st);

}  // namespace tkv
