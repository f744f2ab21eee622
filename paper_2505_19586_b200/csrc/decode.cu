// Quantized-layer decode attention (pipeline.py:331-337 over
// quantizer.py:505-558) as split-K flash-decoding, plus the shared combine.
#include <cmath>

#include "common.cuh"
#include "qcache.cuh"

namespace tkv {

constexpr int SIMT_CHUNK = 256;  // tokens per CTA in the SIMT kernel

// ---------------------------------------------------------------------------
// Combine split-K partials: out = sum_c e^{m_c-M} acc_c / sum_c e^{m_c-M} l_c.
// Fixed chunk order -> bit-identical repeated runs (pipeline determinism,
// test_pipeline.py:189-195).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) combine_kernel(const float *__restrict__ pm, const float *__restrict__ pl,
                                                       const float *__restrict__ pacc, int chunks, int G, int d,
                                                       const int32_t *__restrict__ rows, int rows_stride,
                                                       int rows_per_chunk, float *__restrict__ out) {
  // grid (units*G, ceil(d/32)); 8 warps split the chunks, lanes own channels
  __shared__ float red_m[8];
  __shared__ float part_acc[8][32];
  __shared__ float part_l[8];
  const int u = blockIdx.x / G, h = blockIdx.x % G;
  const int ch = blockIdx.y * 32 + (threadIdx.x & 31);
  const int warp = threadIdx.x >> 5;
  const int nrows = rows ? rows[(size_t)u * rows_stride] : chunks * rows_per_chunk;
  const int valid = min(chunks, (nrows + rows_per_chunk - 1) / rows_per_chunk);
  const size_t base0 = (size_t)u * chunks * G + h;
  float M = -INFINITY;
  for (int ci = threadIdx.x; ci < valid; ci += blockDim.x) M = fmaxf(M, pm[base0 + (size_t)ci * G]);
  M = warp_max(M);
  if ((threadIdx.x & 31) == 0) red_m[warp] = M;
  __syncthreads();
  M = -INFINITY;
  for (int i = 0; i < 8; ++i) M = fmaxf(M, red_m[i]);
  float L = 0.0f, acc = 0.0f;
#pragma unroll 4
  for (int ci = warp; ci < valid; ci += 8) {
    const size_t base = base0 + (size_t)ci * G;
    const float m = pm[base];
    const float sc = m == -INFINITY ? 0.0f : __expf(m - M);
    L += sc * pl[base];
    if (ch < d) acc += sc * pacc[base * d + ch];
  }
  part_acc[warp][threadIdx.x & 31] = acc;
  if ((threadIdx.x & 31) == 0) part_l[warp] = L;
  __syncthreads();
  if (warp == 0 && ch < d) {
    float a = 0.0f, l = 0.0f;
    for (int w = 0; w < 8; ++w) {  // fixed order: deterministic
      a += part_acc[w][threadIdx.x];
      l += part_l[w];
    }
    out[((size_t)u * G + h) * d + ch] = a / l;
  }
}

void launch_combine(const float *pm, const float *pl, const float *pacc, int units, int chunks, int G, int d,
                    const int32_t *rows, int rows_per_chunk, float *out, cudaStream_t st) {
  combine_kernel<<<dim3(units * G, (d + 31) / 32), 256, 0, st>>>(pm, pl, pacc, chunks, G, d, rows, rows ? 1 : 0,
                                                                 rows_per_chunk, out);
}

// variant where every unit shares one device row count (quantized layers)
void launch_combine_scalar(const float *pm, const float *pl, const float *pacc, int units, int chunks, int G,
                                  int d, const int32_t *len, int rows_per_chunk, float *out, cudaStream_t st) {
  combine_kernel<<<dim3(units * G, (d + 31) / 32), 256, 0, st>>>(pm, pl, pacc, chunks, G, d, len, 0, rows_per_chunk,
                                                                 out);
}

// ---------------------------------------------------------------------------
// SIMT decode: one CTA per (256-token chunk, unit).  Each thread owns a token
// for the logits and a channel for the value GEMV.  Keys: logit = sum_c
// (code*s+lo) q_c; values: centred v = (code - (2^b-1)/2) s + mid, so the
// float sums do not cancel ("Accumulation order").
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) quant_decode_simt(QC c, const uint16_t *__restrict__ queries, int G,
                                                          float *__restrict__ pm, float *__restrict__ pl,
                                                          float *__restrict__ pacc, int chunks) {
  extern __shared__ __align__(16) float sm[];
  const int d = c.d, bits = c.bits, g = c.g;
  const int nb = (d + g - 1) / g;
  const int u = blockIdx.y, chunk = blockIdx.x;
  const int64_t n = *c.len;
  const int64_t cs = (int64_t)chunk * SIMT_CHUNK;
  if (cs >= n) return;
  const int rows = (int)imin64(SIMT_CHUNK, n - cs);
  const int64_t ncomp = (n / g) * g;
  float *q = sm;                          // [G][d]
  float *lg = q + G * d;                  // [G][CHUNK]
  const float inv_sqrt_d = 1.0f / sqrtf((float)d);
  for (int i = threadIdx.x; i < G * d; i += blockDim.x)
    q[i] = h2f(queries[((size_t)u * G) * d + i]);
  __syncthreads();
  const int Tk = key_tile_tokens(bits);
  const uint32_t *kc = c.key_codes + (size_t)u * (c.capacity / Tk) * (d / 32) * 128;
  const uint32_t cmask = (1u << bits) - 1u;
  // ---- phase 1: logits, one token per thread ----
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    const int64_t T = cs + t;
    float acc[16];
#pragma unroll
    for (int h = 0; h < 16; ++h) acc[h] = 0.0f;
    if (T < ncomp) {
      const uint32_t *lohi = c.key_lohi + ((size_t)u * (c.capacity / g) + T / g) * d;
      for (int ch0 = 0; ch0 < d; ch0 += 4) {
        int64_t wi;
        int bit;
        key_code_pos(T, ch0, d, bits, &wi, &bit);  // channels ch0..ch0+3 share the word
        const uint32_t w = kc[wi];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int ch = ch0 + i;
          const uint32_t pr = lohi[ch];
          const float lo = h2f(pr & 0xffff), hi = h2f(pr >> 16);
          const float kv = (float)((w >> (bit + 8 * i)) & cmask) * group_scale_f(lo, hi, bits) + lo;
#pragma unroll
          for (int h = 0; h < 16; ++h)
            if (h < G) acc[h] = fmaf(kv, q[h * d + ch], acc[h]);
        }
      }
    } else {
      const uint16_t *kr = c.key_resid + ((size_t)u * g + (T - ncomp)) * d;
      for (int ch = 0; ch < d; ++ch) {
        const float kv = h2f(kr[ch]);
#pragma unroll
        for (int h = 0; h < 16; ++h)
          if (h < G) acc[h] = fmaf(kv, q[h * d + ch], acc[h]);
      }
    }
#pragma unroll
    for (int h = 0; h < 16; ++h)
      if (h < G) lg[h * SIMT_CHUNK + t] = acc[h] * inv_sqrt_d;
  }
  __syncthreads();
  // ---- softmax statistics, one warp per head ----
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int h = warp; h < G; h += blockDim.x >> 5) {
    float m = -INFINITY;
    for (int t = lane; t < rows; t += 32) m = fmaxf(m, lg[h * SIMT_CHUNK + t]);
    m = warp_max(m);
    float l = 0.0f;
    for (int t = lane; t < rows; t += 32) {
      const float p = __expf(lg[h * SIMT_CHUNK + t] - m);
      lg[h * SIMT_CHUNK + t] = p;
      l += p;
    }
    l = warp_sum(l);
    if (lane == 0) {
      pm[((size_t)u * chunks + chunk) * G + h] = m;
      pl[((size_t)u * chunks + chunk) * G + h] = l;
    }
  }
  __syncthreads();
  // ---- phase 2: value GEMV, one channel per thread, token slices ----
  const int slices = blockDim.x / d;  // d <= 256 and divides 256 for supported d
  float *red = lg + G * SIMT_CHUNK;   // [slices][G][d]
  const int ch = threadIdx.x % d, slice = threadIdx.x / d;
  const int sets = val_sets(d, bits);
  const uint32_t *vc = c.val_codes + (size_t)u * (c.capacity / 32) * sets * 128;
  const float c0 = 0.5f * (float)cmask;
  float acc[16];
#pragma unroll
  for (int h = 0; h < 16; ++h) acc[h] = 0.0f;
  if (slice < slices) {
    for (int t = slice; t < rows; t += slices) {
      const int64_t T = cs + t;
      int64_t wi;
      int bit;
      val_code_pos(T, ch, d, bits, &wi, &bit);
      const float code = (float)((vc[wi] >> bit) & cmask);
      const uint32_t pr = c.val_lohi[((size_t)u * c.capacity + T) * nb + ch / g];
      const float lo = h2f(pr & 0xffff), hi = h2f(pr >> 16);
      const float s = group_scale_f(lo, hi, bits);
      const float v = (code - c0) * s + (lo + c0 * s);
#pragma unroll
      for (int h = 0; h < 16; ++h)
        if (h < G) acc[h] = fmaf(lg[h * SIMT_CHUNK + t], v, acc[h]);
    }
#pragma unroll
    for (int h = 0; h < 16; ++h)
      if (h < G) red[(slice * G + h) * d + ch] = acc[h];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * d; i += blockDim.x) {
    float s = 0.0f;
    for (int sl = 0; sl < slices; ++sl) s += red[sl * G * d + i];
    pacc[((size_t)u * chunks + chunk) * G * d + i] = s;
  }
}

// [split partials (m, l, acc) of the SIMT layout, which bounds the tensor-core kernels' | unit arrival
// counters at quant_decode_arrive_offset | slack]
int64_t quant_decode_arrive_offset(const QC &c, int G) {
  const int64_t chunks = (c.capacity + SIMT_CHUNK - 1) / SIMT_CHUNK;
  return ((int64_t)c.units * chunks * G * (2 + c.d) * (int64_t)sizeof(float) + 255) / 256 * 256;
}

int64_t quant_decode_workspace(const QC &c, int G) {
  return quant_decode_arrive_offset(c, G) + ((int64_t)c.units * 4 + 255) / 256 * 256 + 256;
}

int quant_decode_imma(const QC &c, const uint16_t *q, int G, float *out, void *ws, cudaStream_t st);
int quant_decode_pipe(const QC &c, const uint16_t *q, int G, float *out, void *ws, cudaStream_t st);
bool imma_supported(const QC &c, int G);

int quant_decode(const QC &c, const uint16_t *q, int G, float *out, void *ws, int impl, cudaStream_t st) {
  if (impl == 2 || impl == 3 || (impl == 0 && imma_supported(c, G))) {
    if (!imma_supported(c, G) || (impl == 3 && G > 4))
      return fail(TKV_ERR_PARAMETER, "tensor-core decode needs d=128, g=64 and G<=16 (G<=4 for impl 3)");
    return impl == 3 ? quant_decode_imma(c, q, G, out, ws, st) : quant_decode_pipe(c, q, G, out, ws, st);
  }
  const int chunks = (int)((c.capacity + SIMT_CHUNK - 1) / SIMT_CHUNK);
  float *pm = reinterpret_cast<float *>(ws);
  float *pl = pm + (size_t)c.units * chunks * G;
  float *pacc = pl + (size_t)c.units * chunks * G;
  const int slices = 256 / c.d;
  const size_t sm = sizeof(float) * ((size_t)G * c.d + (size_t)G * SIMT_CHUNK + (size_t)slices * G * c.d);
  cudaFuncSetAttribute(quant_decode_simt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 grid(chunks, c.units);
  quant_decode_simt<<<grid, 256, sm, st>>>(c, q, G, pm, pl, pacc, chunks);
  launch_combine_scalar(pm, pl, pacc, c.units, chunks, G, c.d, c.len, SIMT_CHUNK, out, st);
  return check_launch("tkv_quant_decode");
}

}  // namespace tkv
