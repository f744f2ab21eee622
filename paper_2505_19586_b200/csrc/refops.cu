// Kernels behind the reference-signature surface (paper_2505_19586_b200/hybridkv.py):
// GQT1 import into the HBM cache, float64 attention / proxy scores / channel
// selection over caller arrays, a UVA gather from the pinned host store, and
// the top-k mass of a weight vector.  Everything here is called per API
// call (numpy in, numpy out in the reference), not from the decode step.
#include <cmath>

#include "common.cuh"
#include "qcache.cuh"

namespace tkv {

// ---------------------------------------------------------------------------
// GQT1 import (GroupQuantizedTensor.from_bytes, quantizer.py:383-422) into a
// cache unit.  The cache keeps each group's fp16 (lo, hi); the blob carries
// fp16 (zero point, scale).  lo = zero point; hi is the fp16 value whose
// float64 scale (hi - lo) / (2^b - 1), rounded to fp16 like the exporter
// (scale_f16 in qcache.cu), gives back the blob's scale: the one the
// reference quantizer started from when its inputs were fp16.  Without such
// a value (a blob from wider inputs) the nearest fp16 to lo + s (2^b - 1) is
// kept and decoding differs by that rounding.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint16_t imp_scale_f16(uint16_t lo, uint16_t hi, int bits) {
  const double l = h2d(lo), h = h2d(hi);
  double s = __ddiv_rn(__dsub_rn(h, l), (double)((1 << bits) - 1));
  if (s == 0.0) s = 1.0;
  return f64_to_f16_bits(s);
}

__device__ __forceinline__ uint16_t imp_next_f16(uint16_t x, int dir) {
  // neighbour of a finite fp16 in the direction of increasing (dir > 0) or decreasing value
  if ((x & 0x7fffu) == 0) return dir > 0 ? 0x0001u : 0x8001u;
  const bool neg = x & 0x8000u;
  return (dir > 0) != neg ? (uint16_t)(x + 1) : (uint16_t)(x - 1);
}

__device__ uint32_t imp_lohi(uint16_t zp, uint16_t sc, int bits) {
  const double span = h2d(sc) * (double)((1 << bits) - 1);
  uint16_t hi = f64_to_f16_bits(h2d(zp) + span);
  if (imp_scale_f16(zp, hi, bits) != sc) {
    const uint16_t a = imp_next_f16(hi, -1), b = imp_next_f16(hi, 1);
    if (imp_scale_f16(zp, a, bits) == sc) hi = a;
    else if (imp_scale_f16(zp, b, bits) == sc) hi = b;
  }
  if (h2d(hi) < h2d(zp)) hi = zp;
  return pack_lohi(zp, hi);
}

__device__ __forceinline__ uint16_t rd16(const uint8_t *p) { return (uint16_t)(p[0] | (p[1] << 8)); }

// keys blob: codes in (block, channel, token) order, params [blocks][d], residual [res][d]
__global__ void import_keys_kernel(QC c, int u, const uint8_t *__restrict__ packed, int64_t blocks, int64_t res_rows,
                                   const uint8_t *__restrict__ zp, const uint8_t *__restrict__ sc,
                                   const uint8_t *__restrict__ res) {
  const int d = c.d, bits = c.bits, g = c.g;
  const int Tk = key_tile_tokens(bits);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t ncomp = blocks * g;
  // native code words of every tile touched: rebuild word by word (gather from the LSB-first stream)
  const int64_t nwords = ((ncomp + Tk - 1) / Tk) * (d / 32) * 128;
  uint32_t *dst = c.key_codes + (size_t)u * (c.capacity / Tk) * (d / 32) * 128;
  const int kslots = 8 / bits;
  for (int64_t wi = tid; wi < nwords; wi += stride) {
    const int role = (int)(wi & 3), lane = (int)((wi >> 2) & 31);
    const int64_t rest = wi >> 7;
    const int ks = (int)(rest % (d / 32));
    const int64_t tile = rest / (d / 32);
    const int g8 = lane >> 2, tq = lane & 3;
    uint32_t word = 0;
    for (int i = 0; i < 4; ++i) {
      const int ch = 32 * ks + 4 * tq + i + 16 * (role >> 1);
      for (int k = 0; k < kslots; ++k) {
        const int64_t t = tile * Tk + 16 * k + g8 + 8 * (role & 1);
        if (t >= ncomp) continue;
        const int64_t p = (t / g) * ((int64_t)d * g) + (int64_t)ch * g + t % g;  // stream position
        const uint32_t code = (packed[(p * bits) >> 3] >> ((p * bits) & 7)) & ((1u << bits) - 1u);
        word |= code << (8 * i + k * bits);
      }
    }
    dst[wi] = word;
  }
  for (int64_t i = tid; i < blocks * d; i += stride) {
    const uint32_t w = imp_lohi(rd16(zp + 2 * i), rd16(sc + 2 * i), bits);
    c.key_lohi[((size_t)u * (c.capacity / g)) * d + i] = w;
    const float lo = h2f((uint16_t)(w & 0xffff)), hi = h2f((uint16_t)(w >> 16));
    atomic_max_pos(&c.val_smax[2 * u + 1], hi > lo ? (hi - lo) / (float)((1 << bits) - 1) : 0.0f);
  }
  for (int64_t i = tid; i < res_rows * d; i += stride) c.key_resid[(size_t)u * g * d + i] = rd16(res + 2 * i);
}

// values blob: codes row-major [n][d], params [n][ceil(d/g)]
__global__ void import_values_kernel(QC c, int u, const uint8_t *__restrict__ packed, int64_t n,
                                     const uint8_t *__restrict__ zp, const uint8_t *__restrict__ sc) {
  const int d = c.d, bits = c.bits, g = c.g;
  const int nb = (d + g - 1) / g;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  const int per = 16 * (8 / bits), sets = val_sets(d, bits);
  const int64_t nwords = ((n + 31) / 32) * sets * 128;
  uint32_t *dst = c.val_codes + (size_t)u * (c.capacity / 32) * sets * 128;
  const int kslots = 8 / bits;
  for (int64_t wi = tid; wi < nwords; wi += stride) {
    const int role = (int)(wi & 3), lane = (int)((wi >> 2) & 31);
    const int64_t rest = wi >> 7;
    const int set = (int)(rest % sets);
    const int64_t vt = rest / sets;
    const int g8 = lane >> 2, tq = lane & 3;
    uint32_t word = 0;
    for (int i = 0; i < 4; ++i) {
      const int64_t t = vt * 32 + 4 * tq + i + 16 * (role >> 1);
      if (t >= n) continue;
      for (int k = 0; k < kslots; ++k) {
        const int ch = set * per + 16 * k + g8 + 8 * (role & 1);
        if (ch >= d) continue;
        const int64_t p = t * d + ch;
        const uint32_t code = (packed[(p * bits) >> 3] >> ((p * bits) & 7)) & ((1u << bits) - 1u);
        word |= code << (8 * i + k * bits);
      }
    }
    dst[wi] = word;
  }
  for (int64_t i = tid; i < n * nb; i += stride) {
    const uint32_t w = imp_lohi(rd16(zp + 2 * i), rd16(sc + 2 * i), bits);
    c.val_lohi[(size_t)u * c.capacity * nb + i] = w;
    atomic_max_pos(&c.val_smax[2 * u], group_scale_f(h2f((uint16_t)(w & 0xffff)), h2f((uint16_t)(w >> 16)), bits));
  }
}

__global__ void import_len_kernel(int32_t *len, int64_t n) { *len = (int32_t)n; }

int import_blob(const QC &c, int u, int which, const uint8_t *blob, int64_t rows, int64_t res_rows,
                int64_t packed_len, cudaStream_t st) {
  const uint8_t *packed = blob + 24;
  if (which == 0) {
    const int64_t blocks = rows / c.g, grid = blocks * c.d;
    const uint8_t *zp = packed + packed_len, *sc = zp + 2 * grid, *res = sc + 2 * grid;
    import_keys_kernel<<<296, 256, 0, st>>>(c, u, packed, blocks, res_rows, zp, sc, res);
    import_len_kernel<<<1, 1, 0, st>>>(c.len, rows + res_rows);
  } else {
    const int64_t grid = rows * ((c.d + c.g - 1) / c.g);
    const uint8_t *zp = packed + packed_len, *sc = zp + 2 * grid;
    import_values_kernel<<<296, 256, 0, st>>>(c, u, packed, rows, zp, sc);
    import_len_kernel<<<1, 1, 0, st>>>(c.len, rows);
  }
  return check_launch("tkv_qcache_import");
}

// ---------------------------------------------------------------------------
// float64 exact attention over caller arrays (attention_weights /
// exact_attention kv_model.py:169-213, sparse_attention retriever.py:214-226):
// softmax(q K^T / sqrt(d)) (max-subtracted), then weights @ V.  One CTA per
// query row; `sel` (optional) restricts the rows to an index list.
// ---------------------------------------------------------------------------
constexpr int RO_THREADS = 256;

__device__ __forceinline__ double ro_block_reduce(double v, double *sh, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmax(v, x) : v + x;
  }
  if (lane == 0) sh[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = sh[0];
    for (int i = 1; i < RO_THREADS / 32; ++i) a = is_max ? fmax(a, sh[i]) : a + sh[i];
    sh[32] = a;
  }
  __syncthreads();
  const double r = sh[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(RO_THREADS) attention_f64_kernel(const double *__restrict__ q,
                                                                   const double *__restrict__ keys,
                                                                   const double *__restrict__ values, int64_t n,
                                                                   int d, const int64_t *__restrict__ sel,
                                                                   int64_t m, double *__restrict__ logits,
                                                                   double *__restrict__ weights,
                                                                   double *__restrict__ out) {
  __shared__ double sh[33];
  const int row = blockIdx.x;
  const double *qr = q + (size_t)row * d;
  double *lg = logits + (size_t)row * m;
  const double inv = 1.0 / sqrt((double)d);
  double mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < m; j += RO_THREADS) {
    const int64_t t = sel ? sel[j] : j;
    const double *kr = keys + (size_t)t * d;
    double a = 0.0;
    for (int c = 0; c < d; ++c) a = fma(kr[c], qr[c], a);
    a *= inv;
    lg[j] = a;
    mx = fmax(mx, a);
  }
  mx = ro_block_reduce(mx, sh, true);
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < m; j += RO_THREADS) {
    const double e = exp(lg[j] - mx);
    lg[j] = e;
    s += e;
  }
  s = ro_block_reduce(s, sh, false);
  const double rs = 1.0 / s;
  if (weights)
    for (int64_t j = threadIdx.x; j < m; j += RO_THREADS) weights[(size_t)row * m + j] = lg[j] * rs;
  if (out) {
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += RO_THREADS) {
      double a = 0.0;
      for (int64_t j = 0; j < m; ++j) a = fma(lg[j] * rs, values[(size_t)(sel ? sel[j] : j) * d + c], a);
      out[(size_t)row * d + c] = a;
    }
  }
}

int attention_f64(const double *q, int rows, const double *keys, const double *values, int64_t n, int d,
                  const int64_t *sel, int64_t m, double *ws, double *weights, double *out, cudaStream_t st) {
  attention_f64_kernel<<<rows, RO_THREADS, 0, st>>>(q, keys, values, n, d, sel, m, ws, weights, out);
  return check_launch("tkv_attention_f64");
}

// ---------------------------------------------------------------------------
// approx_scores (retriever.py:166-189): critical_keys [n][d_s] @ (sum over the
// group of query_critical [G][d_s]), float64.
// ---------------------------------------------------------------------------
__global__ void approx_scores_f64_kernel(const double *__restrict__ qc, int G, const double *__restrict__ keys,
                                         int64_t n, int d_s, double *__restrict__ out) {
  extern __shared__ double qsum[];
  for (int i = threadIdx.x; i < d_s; i += blockDim.x) {
    double a = 0.0;
    for (int j = 0; j < G; ++j) a += qc[(size_t)j * d_s + i];
    qsum[i] = a;
  }
  __syncthreads();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double a = 0.0;
    for (int i = 0; i < d_s; ++i) a = fma(keys[(size_t)t * d_s + i], qsum[i], a);
    out[t] = a;
  }
}

int approx_scores_f64(const double *qc, int G, const double *keys, int64_t n, int d_s, double *out, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>(296, (n + 255) / 256);
  approx_scores_f64_kernel<<<std::max(blocks, 1), 256, d_s * sizeof(double), st>>>(qc, G, keys, n, d_s, out);
  return check_launch("tkv_approx_scores_f64");
}

// ---------------------------------------------------------------------------
// group_channel_scores + select_critical_channels (retriever.py:111-163):
// s_c = (sum_j |q_hat[j][c]|) * chmax_c; top d_s, ties to the lower index,
// ascending.  One CTA; rank by counting.
// ---------------------------------------------------------------------------
__global__ void channel_select_f64_kernel(const double *__restrict__ qhat, int G, const double *__restrict__ chmax,
                                          int d, int d_s, double *__restrict__ scores, int32_t *__restrict__ sel) {
  extern __shared__ double sc[];
  int *flag = reinterpret_cast<int *>(sc + d);
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    double s;
    if (chmax) {
      double a = 0.0;
      for (int j = 0; j < G; ++j) a += fabs(qhat[(size_t)j * d + c]);  // ascending j (numpy axis-0 sum)
      s = a * chmax[c];
    } else {
      s = qhat[c];  // caller scores as they are (select_critical_channels)
    }
    sc[c] = s;
    if (scores) scores[c] = s;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const double s = sc[c];
    int rank = 0;
    for (int j = 0; j < d; ++j) rank += (sc[j] > s) || (sc[j] == s && j < c);
    flag[c] = rank < d_s;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    if (!flag[c]) continue;
    int pos = 0;
    for (int j = 0; j < c; ++j) pos += flag[j];
    sel[pos] = c;
  }
}

int channel_select_f64(const double *qhat, int G, const double *chmax, int d, int d_s, double *scores, int32_t *sel,
                       cudaStream_t st) {
  channel_select_f64_kernel<<<1, 256, d * (sizeof(double) + sizeof(int)), st>>>(qhat, G, chmax, d, d_s, scores, sel);
  return check_launch("tkv_channel_select_f64");
}

// ---------------------------------------------------------------------------
// Rows of one head from the pinned host store (HostPool.gather, memsim.py:118-127):
// UVA loads, one warp per row, K and V rows to device buffers [m][d].
// ---------------------------------------------------------------------------
__global__ void host_gather_kernel(SL s, int u, const int64_t *__restrict__ idx, int64_t m, uint16_t *out_k,
                                   uint16_t *out_v) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int vec = s.d / 8;  // 16-byte vectors per row
  for (int64_t r = warp; r < m; r += nw) {
    const uint4 *src = reinterpret_cast<const uint4 *>(s.host_kv + ((size_t)u * s.capacity + idx[r]) * 2 * s.d);
    for (int v = lane; v < 2 * vec; v += 32) {
      const uint4 x = src[v];
      uint16_t *dst = v < vec ? out_k + (size_t)r * s.d : out_v + (size_t)r * s.d;
      reinterpret_cast<uint4 *>(dst)[v % vec] = x;
    }
  }
}

int host_gather(const SL &s, int u, const int64_t *idx, int64_t m, uint16_t *out_k, uint16_t *out_v, cudaStream_t st) {
  if (m == 0) return TKV_OK;
  const int blocks = (int)std::min<int64_t>(296, (m + 7) / 8);
  host_gather_kernel<<<blocks, 256, 0, st>>>(s, u, idx, m, out_k, out_v);
  return check_launch("tkv_host_gather");
}

// ---------------------------------------------------------------------------
// sum of w over an index list, float64, fixed order (sparse_error's kept
// mass, identifier.py:89-107, after the top-k index selection)
// ---------------------------------------------------------------------------
__global__ void sum_at_kernel(const double *__restrict__ w, const int32_t *__restrict__ idx, const int32_t *cnt,
                              double *out) {
  __shared__ double sh[33];
  double a = 0.0;
  for (int i = threadIdx.x; i < *cnt; i += RO_THREADS) a += w[idx[i]];
  a = ro_block_reduce(a, sh, false);
  if (threadIdx.x == 0) *out = a;
}

int sum_at(const double *w, const int32_t *idx, const int32_t *cnt, double *out, cudaStream_t st) {
  sum_at_kernel<<<1, RO_THREADS, 0, st>>>(w, idx, cnt, out);
  return check_launch("tkv_sum_at");
}

}  // namespace tkv
