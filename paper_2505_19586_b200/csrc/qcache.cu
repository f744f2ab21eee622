#include <algorithm>
// Quantized layer cache: prefill pack, decode append, GQT1 export, dequant,
// raw GEMVs.  Reference: hybridkv/quantizer.py:187-558.
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "qcache.cuh"

namespace tkv {

// ---------------------------------------------------------------------------
// Pack keys: one CTA per (key tile, unit).  quantizer.py:277-293.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) pack_keys_kernel(QC c, const uint16_t *__restrict__ keys, int64_t n,
                                                         int64_t n_complete) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int d = c.d, bits = c.bits, g = c.g;
  const int Tk = key_tile_tokens(bits);
  const int u = blockIdx.y;
  const int64_t t0 = (int64_t)blockIdx.x * Tk;
  if (t0 >= n_complete) return;
  const int rows = (int)imin64(Tk, n_complete - t0);  // complete groups only
  uint16_t *tile = reinterpret_cast<uint16_t *>(smem);               // [Tk][d]
  uint8_t *codes = reinterpret_cast<uint8_t *>(smem + (size_t)Tk * d * 2);  // [Tk][d]
  uint32_t *lohi = reinterpret_cast<uint32_t *>(codes + (size_t)Tk * d);      // [Tk/g][d]
  const uint16_t *src = keys + ((size_t)u * n + t0) * d;
  // stage the tile (16-byte vectors; d % 32 == 0 keeps rows 16B aligned)
  const int vec_per_row = d / 8;
  for (int v = threadIdx.x; v < rows * vec_per_row; v += blockDim.x) {
    reinterpret_cast<uint4 *>(tile)[v] = __ldg(reinterpret_cast<const uint4 *>(src) + v);
  }
  __syncthreads();
  const int groups = rows / g;
  for (int p = threadIdx.x; p < groups * d; p += blockDim.x) {
    const int grp = p / d, ch = p % d;
    float lo = h2f(tile[(grp * g) * d + ch]), hi = lo;
    uint16_t lob = tile[(grp * g) * d + ch], hib = lob;
    for (int r = 1; r < g; ++r) {
      uint16_t xb = tile[(grp * g + r) * d + ch];
      float x = h2f(xb);
      if (x < lo) { lo = x; lob = xb; }
      if (x > hi) { hi = x; hib = xb; }
    }
    // canonicalise -0.0 so the fp16 bits reproduce float64 min/max values
    if (lo == 0.0f) lob = 0x0000u;
    if (hi == 0.0f) hib = 0x0000u;
    const uint32_t w = pack_lohi(lob, hib);
    lohi[p] = w;
    c.key_lohi[((size_t)u * (c.capacity / g) + (t0 / g) + grp) * d + ch] = w;
    atomic_max_pos(&c.val_smax[2 * u + 1], hi > lo ? (hi - lo) / (float)((1 << bits) - 1) : 0.0f);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < Tk * d; p += blockDim.x) {
    const int t = p / d, ch = p % d;
    uint8_t code = 0;
    if (t < rows) {
      const uint32_t w = lohi[(t / g) * d + ch];
      code = (uint8_t)encode_code(h2f(tile[p]), h2f((uint16_t)(w & 0xffff)), h2f((uint16_t)(w >> 16)), bits);
    }
    codes[p] = code;
  }
  __syncthreads();
  // assemble native words for this tile: (d/32) * 32 lanes * 4 roles
  const int nwords = (d / 32) * 128;
  uint32_t *dst = c.key_codes + ((size_t)u * (c.capacity / Tk) + blockIdx.x) * nwords;
  const int kslots = 8 / bits;
  for (int wi = threadIdx.x; wi < nwords; wi += blockDim.x) {
    const int role = wi & 3, lane = (wi >> 2) & 31, ks = wi >> 7;
    const int g8 = lane >> 2, tq = lane & 3;
    uint32_t word = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int ch = 32 * ks + 4 * tq + i + 16 * (role >> 1);
      for (int k = 0; k < kslots; ++k) {
        const int t = 16 * k + g8 + 8 * (role & 1);
        word |= (uint32_t)codes[t * d + ch] << (8 * i + k * bits);
      }
    }
    dst[wi] = word;
  }
}

// ---------------------------------------------------------------------------
// Pack values: one CTA per (32-token tile, unit).  quantizer.py:252-275.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) pack_values_kernel(QC c, const uint16_t *__restrict__ values, int64_t n,
                                                           int64_t row0, int64_t src_rows) {
  // row0: first token index of this call (prefill: 0).  src holds rows [row0, row0+src_rows).
  extern __shared__ __align__(16) unsigned char smem[];
  const int d = c.d, bits = c.bits, g = c.g;
  const int nb = (d + g - 1) / g;
  const int u = blockIdx.y;
  const int64_t t0 = (int64_t)blockIdx.x * 32;
  if (t0 >= n) return;
  const int rows = (int)imin64(32, n - t0);
  uint16_t *tile = reinterpret_cast<uint16_t *>(smem);                  // [32][d]
  uint8_t *codes = reinterpret_cast<uint8_t *>(smem + 32 * d * 2);       // [32][d]
  uint32_t *lohi = reinterpret_cast<uint32_t *>(codes + 32 * d);         // [32][nb]
  __shared__ float smax;
  if (threadIdx.x == 0) smax = 0.0f;
  const uint16_t *src = values + ((size_t)u * src_rows + (t0 - row0)) * d;
  const int vec_per_row = d / 8;
  for (int v = threadIdx.x; v < rows * vec_per_row; v += blockDim.x)
    reinterpret_cast<uint4 *>(tile)[v] = __ldg(reinterpret_cast<const uint4 *>(src) + v);
  __syncthreads();
  for (int p = threadIdx.x; p < rows * nb; p += blockDim.x) {
    const int t = p / nb, b = p % nb;
    const int c0 = b * g, c1 = min(d, c0 + g);
    uint16_t lob = tile[t * d + c0], hib = lob;
    float lo = h2f(lob), hi = lo;
    for (int ch = c0 + 1; ch < c1; ++ch) {
      const uint16_t xb = tile[t * d + ch];
      const float x = h2f(xb);
      if (x < lo) { lo = x; lob = xb; }
      if (x > hi) { hi = x; hib = xb; }
    }
    if (lo == 0.0f) lob = 0;
    if (hi == 0.0f) hib = 0;
    const uint32_t w = pack_lohi(lob, hib);
    lohi[p] = w;
    c.val_lohi[((size_t)u * c.capacity + t0 + t) * nb + b] = w;
    atomic_max_pos(&smax, group_scale_f(lo, hi, bits));
  }
  __syncthreads();
  for (int p = threadIdx.x; p < 32 * d; p += blockDim.x) {
    const int t = p / d, ch = p % d;
    uint8_t code = 0;
    if (t < rows) {
      const uint32_t w = lohi[t * nb + ch / g];
      code = (uint8_t)encode_code(h2f(tile[p]), h2f((uint16_t)(w & 0xffff)), h2f((uint16_t)(w >> 16)), bits);
    }
    codes[p] = code;
  }
  __syncthreads();
  const int sets = val_sets(d, bits);
  const int per = 16 * (8 / bits);
  const int kslots = 8 / bits;
  const int nwords = sets * 128;
  uint32_t *dst = c.val_codes + ((size_t)u * (c.capacity / 32) + blockIdx.x) * nwords;
  for (int wi = threadIdx.x; wi < nwords; wi += blockDim.x) {
    const int role = wi & 3, lane = (wi >> 2) & 31, set = wi >> 7;
    const int g8 = lane >> 2, tq = lane & 3;
    uint32_t word = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int t = 4 * tq + i + 16 * (role >> 1);
      for (int k = 0; k < kslots; ++k) {
        const int ch = set * per + 16 * k + g8 + 8 * (role & 1);
        if (ch < d) word |= (uint32_t)codes[t * d + ch] << (8 * i + k * bits);
      }
    }
    // a partial tile (append path) must keep bits of tokens already present
    if (row0 > t0) word |= dst[wi];
    dst[wi] = word;
  }
  if (threadIdx.x == 0) atomic_max_pos(&c.val_smax[2 * u], smax);
}

__global__ void copy_residual_kernel(QC c, const uint16_t *__restrict__ keys, int64_t n, int64_t n_complete) {
  const int u = blockIdx.y;
  const int r = blockIdx.x;
  const int64_t t = n_complete + r;
  if (t >= n) return;
  for (int ch = threadIdx.x; ch < c.d; ch += blockDim.x)
    c.key_resid[((size_t)u * c.g + r) * c.d + ch] = keys[((size_t)u * n + t) * c.d + ch];
}

__global__ void set_len_kernel(int32_t *len, int64_t n) { *len = (int32_t)n; }

__global__ void finite_check_kernel(const uint16_t *__restrict__ x, int64_t count, int *flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    if ((x[i] & 0x7c00u) == 0x7c00u) { *flag = 1; return; }
  }
}

int pack(const QC &c, const uint16_t *keys, const uint16_t *values, int64_t n, int check_finite,
         cudaStream_t st) {
  if (check_finite) {
    int *flag = nullptr;
    if (cudaMallocAsync(&flag, sizeof(int), st) != cudaSuccess) return fail(TKV_ERR_CUDA, "cudaMallocAsync failed");
    cudaMemsetAsync(flag, 0, sizeof(int), st);
    finite_check_kernel<<<592, 256, 0, st>>>(keys, (int64_t)c.units * n * c.d, flag);
    finite_check_kernel<<<592, 256, 0, st>>>(values, (int64_t)c.units * n * c.d, flag);
    int h = 0;
    cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(flag, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(TKV_ERR_CUDA, "finite check failed");
    if (h) return fail(TKV_ERR_NUMERIC, "matrix contains non-finite values");
  }
  const int Tk = key_tile_tokens(c.bits);
  const int64_t n_complete = (n / c.g) * c.g;
  cudaMemsetAsync(c.val_smax, 0, sizeof(float) * 2 * c.units, st);
  if (n_complete > 0) {
    const size_t sm = (size_t)Tk * c.d * 3 + (size_t)(Tk / c.g) * c.d * 4;
    cudaFuncSetAttribute(pack_keys_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid((unsigned)((n_complete + Tk - 1) / Tk), c.units);
    pack_keys_kernel<<<grid, 256, sm, st>>>(c, keys, n, n_complete);
  }
  if (n > n_complete) {
    dim3 grid((unsigned)(n - n_complete), c.units);
    copy_residual_kernel<<<grid, 128, 0, st>>>(c, keys, n, n_complete);
  }
  {
    const int nb = (c.d + c.g - 1) / c.g;
    const size_t sm = (size_t)32 * c.d * 3 + (size_t)32 * nb * 4;
    cudaFuncSetAttribute(pack_values_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    dim3 grid((unsigned)((n + 31) / 32), c.units);
    pack_values_kernel<<<grid, 256, sm, st>>>(c, values, n, 0, n);
  }
  set_len_kernel<<<1, 1, 0, st>>>(c.len, n);
  return check_launch("tkv_qcache_pack");
}

// ---------------------------------------------------------------------------
// Append one token per unit (quantizer.py:445-451).  One CTA per unit.
// Values are packed immediately; keys go to the residual and a group is
// finalised when g rows are pending (quantizer.py:277-293).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) append_kernel(QC c, const uint16_t *__restrict__ nk,
                                                      const uint16_t *__restrict__ nv) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int d = c.d, bits = c.bits, g = c.g;
  const int nb = (d + g - 1) / g;
  const int u = blockIdx.x;
  const int64_t n = *c.len;  // token index being appended
  uint8_t *vcodes = smem;                                    // [d]
  uint32_t *vlohi = reinterpret_cast<uint32_t *>(smem + ((d + 15) & ~15));  // [nb]
  uint8_t *kcodes = smem + ((d + 15) & ~15) + 64 * 4;       // [g][d] when finalising
  // ---- values ----
  const uint16_t *vrow = nv + (size_t)u * d;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const int c0 = b * g, c1 = min(d, c0 + g);
    uint16_t lob = vrow[c0], hib = lob;
    float lo = h2f(lob), hi = lo;
    for (int ch = c0 + 1; ch < c1; ++ch) {
      const uint16_t xb = vrow[ch];
      const float x = h2f(xb);
      if (x < lo) { lo = x; lob = xb; }
      if (x > hi) { hi = x; hib = xb; }
    }
    if (lo == 0.0f) lob = 0;
    if (hi == 0.0f) hib = 0;
    vlohi[b] = pack_lohi(lob, hib);
    c.val_lohi[((size_t)u * c.capacity + n) * nb + b] = vlohi[b];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.0f;
    for (int b = 0; b < nb; ++b)
      m = fmaxf(m, group_scale_f(h2f(vlohi[b] & 0xffff), h2f(vlohi[b] >> 16), bits));
    atomic_max_pos(&c.val_smax[2 * u], m);
  }
  for (int ch = threadIdx.x; ch < d; ch += blockDim.x) {
    const uint32_t w = vlohi[ch / g];
    vcodes[ch] = (uint8_t)encode_code(h2f(vrow[ch]), h2f(w & 0xffff), h2f(w >> 16), bits);
  }
  __syncthreads();
  for (int ch = threadIdx.x; ch < d; ch += blockDim.x) {
    int64_t wi;
    int bit;
    val_code_pos(n, ch, d, bits, &wi, &bit);
    atomicOr(&c.val_codes[(size_t)u * (c.capacity / 32) * val_sets(d, bits) * 128 + wi], (uint32_t)vcodes[ch] << bit);
  }
  // ---- keys ----
  const int64_t n_complete = (n / g) * g;
  const int r = (int)(n - n_complete);
  const uint16_t *krow = nk + (size_t)u * d;
  uint16_t *res = c.key_resid + (size_t)u * g * d;
  for (int ch = threadIdx.x; ch < d; ch += blockDim.x) res[r * d + ch] = krow[ch];
  __syncthreads();
  if (r == g - 1) {  // the group is complete: quantize g rows x d channels
    const int64_t grp = n_complete / g;
    for (int ch = threadIdx.x; ch < d; ch += blockDim.x) {
      uint16_t lob = res[ch], hib = lob;
      float lo = h2f(lob), hi = lo;
      for (int rr = 1; rr < g; ++rr) {
        const uint16_t xb = res[rr * d + ch];
        const float x = h2f(xb);
        if (x < lo) { lo = x; lob = xb; }
        if (x > hi) { hi = x; hib = xb; }
      }
      if (lo == 0.0f) lob = 0;
      if (hi == 0.0f) hib = 0;
      c.key_lohi[((size_t)u * (c.capacity / g) + grp) * d + ch] = pack_lohi(lob, hib);
      atomic_max_pos(&c.val_smax[2 * u + 1], hi > lo ? (hi - lo) / (float)((1 << bits) - 1) : 0.0f);
      for (int rr = 0; rr < g; ++rr)
        kcodes[rr * d + ch] = (uint8_t)encode_code(h2f(res[rr * d + ch]), lo, hi, bits);
    }
    __syncthreads();
    const int Tk = key_tile_tokens(bits);
    uint32_t *kc = c.key_codes + (size_t)u * (c.capacity / Tk) * (d / 32) * 128;
    for (int p = threadIdx.x; p < g * d; p += blockDim.x) {
      const int rr = p / d, ch = p % d;
      int64_t wi;
      int bit;
      key_code_pos(n_complete + rr, ch, d, bits, &wi, &bit);
      const uint32_t v = (uint32_t)kcodes[p] << bit;
      if (v) atomicOr(&kc[wi], v);
    }
  }
  // ---- advance the shared length once every unit is done ----
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(c.ticket, 1u);
    if (prev == (unsigned)gridDim.x - 1) {
      *c.ticket = 0;
      __threadfence();
      *c.len = (int32_t)(n + 1);
    }
  }
}

int append(const QC &c, const uint16_t *nk, const uint16_t *nv, cudaStream_t st) {
  const size_t sm = ((c.d + 15) & ~15) + 64 * 4 + (size_t)c.g * c.d;
  cudaFuncSetAttribute(append_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  launch_prio(append_kernel, dim3(c.units), dim3(256), sm, st, true, c, nk, nv);
  return check_launch("tkv_qcache_append");
}

// ---------------------------------------------------------------------------
// GQT1 export (quantizer.py:358-380), bit-exact.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t key_code_at(const QC &c, int u, int64_t t, int ch) {
  int64_t wi;
  int bit;
  key_code_pos(t, ch, c.d, c.bits, &wi, &bit);
  const int Tk = key_tile_tokens(c.bits);
  const uint32_t w = c.key_codes[(size_t)u * (c.capacity / Tk) * (c.d / 32) * 128 + wi];
  return (w >> bit) & ((1u << c.bits) - 1u);
}

__device__ __forceinline__ uint32_t val_code_at(const QC &c, int u, int64_t t, int ch) {
  int64_t wi;
  int bit;
  val_code_pos(t, ch, c.d, c.bits, &wi, &bit);
  const uint32_t w = c.val_codes[(size_t)u * (c.capacity / 32) * val_sets(c.d, c.bits) * 128 + wi];
  return (w >> bit) & ((1u << c.bits) - 1u);
}

__device__ __forceinline__ uint16_t scale_f16(uint32_t lohi, int bits) {
  const double lo = h2d(lohi & 0xffff), hi = h2d(lohi >> 16);
  double s = __ddiv_rn(__dsub_rn(hi, lo), (double)((1 << bits) - 1));
  if (s == 0.0) s = 1.0;
  return f64_to_f16_bits(s);
}

__global__ void export_kernel(QC c, int u, int which, int64_t n, uint8_t *out, int64_t packed_len,
                              int64_t grid_rows, int64_t grid_cols, int64_t res_rows) {
  const int d = c.d, bits = c.bits, g = c.g;
  const int64_t ncomp = which == 0 ? (n / g) * g : n;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0) {  // header <4sBBHIIII
    out[0] = 'G'; out[1] = 'Q'; out[2] = 'T'; out[3] = '1';
    out[4] = (uint8_t)bits;
    out[5] = (uint8_t)(which == 0 ? 1 : 2);
    out[6] = (uint8_t)(g & 0xff); out[7] = (uint8_t)(g >> 8);
    const uint32_t f[4] = {(uint32_t)ncomp, (uint32_t)d, (uint32_t)res_rows, (uint32_t)packed_len};
    for (int j = 0; j < 4; ++j)
      for (int bte = 0; bte < 4; ++bte) out[8 + 4 * j + bte] = (uint8_t)(f[j] >> (8 * bte));
  }
  uint8_t *packed = out + 24;
  const int per_byte = 8 / bits;
  const int64_t total = ncomp * d;
  for (int64_t B = tid; B < packed_len; B += stride) {
    uint32_t byte = 0;
    for (int q = 0; q < per_byte; ++q) {
      const int64_t p = B * per_byte + q;
      if (p >= total) break;
      uint32_t code;
      if (which == 0) {
        const int64_t blk = p / ((int64_t)d * g), rem = p % ((int64_t)d * g);
        const int ch = (int)(rem / g);
        const int64_t t = blk * g + rem % g;
        code = key_code_at(c, u, t, ch);
      } else {
        code = val_code_at(c, u, p / d, (int)(p % d));
      }
      byte |= code << (q * bits);
    }
    packed[B] = (uint8_t)byte;
  }
  uint16_t *zp = reinterpret_cast<uint16_t *>(packed + packed_len);  // may be unaligned? packed_len even
  const int64_t G = grid_rows * grid_cols;
  for (int64_t i = tid; i < G; i += stride) {
    const int64_t r = i / grid_cols, col = i % grid_cols;
    uint32_t w;
    if (which == 0) w = c.key_lohi[((size_t)u * (c.capacity / g) + r) * d + col];
    else w = c.val_lohi[((size_t)u * c.capacity + r) * grid_cols + col];
    uint8_t *zb = reinterpret_cast<uint8_t *>(zp) + 2 * i;
    const uint16_t lo = (uint16_t)(w & 0xffff);
    zb[0] = lo & 0xff; zb[1] = lo >> 8;
    const uint16_t s = scale_f16(w, bits);
    uint8_t *sb = reinterpret_cast<uint8_t *>(zp) + 2 * G + 2 * i;
    sb[0] = s & 0xff; sb[1] = s >> 8;
  }
  uint8_t *res = reinterpret_cast<uint8_t *>(zp) + 4 * G;
  for (int64_t i = tid; i < res_rows * d; i += stride) {
    const uint16_t v = c.key_resid[(size_t)u * g * d + i];
    res[2 * i] = v & 0xff; res[2 * i + 1] = v >> 8;
  }
}

int64_t export_size(const QC &c, int which, int64_t n) {
  const int64_t ncomp = which == 0 ? (n / c.g) * c.g : n;
  const int64_t packed = (ncomp * c.d * c.bits + 7) / 8;
  const int64_t gr = which == 0 ? ncomp / c.g : n;
  const int64_t gc = which == 0 ? c.d : (c.d + c.g - 1) / c.g;
  const int64_t res = which == 0 ? (n - ncomp) : 0;
  return 24 + packed + 4 * gr * gc + 2 * res * c.d;
}

int export_blob(const QC &c, int u, int which, int64_t n, uint8_t *out, cudaStream_t st) {
  const int64_t ncomp = which == 0 ? (n / c.g) * c.g : n;
  const int64_t packed = (ncomp * c.d * c.bits + 7) / 8;
  const int64_t gr = which == 0 ? ncomp / c.g : n;
  const int64_t gc = which == 0 ? c.d : (c.d + c.g - 1) / c.g;
  const int64_t res = which == 0 ? (n - ncomp) : 0;
  export_kernel<<<296, 256, 0, st>>>(c, u, which, n, out, packed, gr, gc, res);
  return check_launch("tkv_qcache_export");
}

// ---------------------------------------------------------------------------
// Dequantize (quantizer.py:335-352) and raw GEMVs (quantizer.py:505-558).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float key_hat(const QC &c, int u, int64_t t, int ch, int64_t ncomp) {
  if (t >= ncomp) return h2f(c.key_resid[((size_t)u * c.g + (t - ncomp)) * c.d + ch]);
  const uint32_t w = c.key_lohi[((size_t)u * (c.capacity / c.g) + t / c.g) * c.d + ch];
  const float lo = h2f(w & 0xffff), hi = h2f(w >> 16);
  return (float)key_code_at(c, u, t, ch) * group_scale_f(lo, hi, c.bits) + lo;
}

__device__ __forceinline__ float val_hat(const QC &c, int u, int64_t t, int ch) {
  const int nb = (c.d + c.g - 1) / c.g;
  const uint32_t w = c.val_lohi[((size_t)u * c.capacity + t) * nb + ch / c.g];
  const float lo = h2f(w & 0xffff), hi = h2f(w >> 16);
  return (float)val_code_at(c, u, t, ch) * group_scale_f(lo, hi, c.bits) + lo;
}

__global__ void dequant_kernel(QC c, int u, int which, int64_t n, float *out) {
  const int64_t ncomp = (n / c.g) * c.g;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * c.d; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / c.d;
    const int ch = (int)(i % c.d);
    out[i] = which == 0 ? key_hat(c, u, t, ch, ncomp) : val_hat(c, u, t, ch);
  }
}

int dequant(const QC &c, int u, int which, int64_t n, float *out, cudaStream_t st) {
  dequant_kernel<<<296, 256, 0, st>>>(c, u, which, n, out);
  return check_launch("tkv_qcache_dequant");
}

// qgemv_scores (quantizer.py:505-533), float64 like the reference:
// logit_t = sum_c code[t,c] (q_c s[g,c]) + sum_c q_c z[g,c] over complete
// groups, residual rows @ q.  One warp per token, lanes over channels.
__global__ void __launch_bounds__(256) qgemv_scores_kernel(QC c, int u, int64_t n, const double *__restrict__ q,
                                                           double *__restrict__ logits) {
  const int lane = threadIdx.x & 31, d = c.d, g = c.g;
  const int64_t ncomp = (n / g) * g;
  const double den = (double)((1 << c.bits) - 1);
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < n;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double acc = 0.0;
    for (int ch = lane; ch < d; ch += 32) {
      if (t >= ncomp) {
        acc = fma(h2d(c.key_resid[((size_t)u * g + (t - ncomp)) * d + ch]), q[ch], acc);
      } else {
        const uint32_t w = c.key_lohi[((size_t)u * (c.capacity / g) + t / g) * d + ch];
        const double lo = h2d(w & 0xffff), hi = h2d(w >> 16);
        double s = (hi - lo) / den;
        if (s == 0.0) s = 1.0;
        acc = fma((double)key_code_at(c, u, t, ch), q[ch] * s, acc);
        acc = fma(q[ch], lo, acc);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) logits[t] = acc;
  }
}

// qgemv_output (quantizer.py:536-558), float64: out_c = sum_t w_t (code[t,c]
// s[t,cb] + z[t,cb]).  Pass 1: CTA per 1024-token chunk, threads over
// (token lane, channel), fixed-order partials; pass 2 sums the chunks in order.
constexpr int QG_CHUNK = 1024;
__global__ void __launch_bounds__(256) qgemv_output_part_kernel(QC c, int u, int64_t n, const double *__restrict__ w,
                                                                double *__restrict__ part) {
  __shared__ double red[256];
  const int d = c.d, nb = (d + c.g - 1) / c.g;
  const int lanes = 256 / d;  // token lanes (d <= 256)
  const int ch = threadIdx.x % d, tl = threadIdx.x / d;
  const double den = (double)((1 << c.bits) - 1);
  const int64_t t0 = (int64_t)blockIdx.x * QG_CHUNK, t1 = imin64(n, t0 + QG_CHUNK);
  double acc = 0.0;
  if (tl < lanes) {
    for (int64_t t = t0 + tl; t < t1; t += lanes) {
      const uint32_t pr = c.val_lohi[((size_t)u * c.capacity + t) * nb + ch / c.g];
      const double lo = h2d(pr & 0xffff), hi = h2d(pr >> 16);
      double s = (hi - lo) / den;
      if (s == 0.0) s = 1.0;
      acc = fma(w[t], fma((double)val_code_at(c, u, t, ch), s, lo), acc);
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < d) {
    double a = 0.0;
    for (int l = 0; l < lanes; ++l) a += red[l * d + threadIdx.x];
    part[(size_t)blockIdx.x * d + threadIdx.x] = a;
  }
}

__global__ void qgemv_output_sum_kernel(const double *__restrict__ part, int chunks, int d, double *__restrict__ out) {
  for (int ch = threadIdx.x; ch < d; ch += blockDim.x) {
    double a = 0.0;
    for (int k = 0; k < chunks; ++k) a += part[(size_t)k * d + ch];
    out[ch] = a;
  }
}

int64_t qgemv_output_workspace(const QC &c, int64_t n) { return ((n + QG_CHUNK - 1) / QG_CHUNK) * c.d * 8 + 256; }

int qgemv_scores(const QC &c, int u, int64_t n, const double *q, double *logits, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>(1184, (n + 7) / 8);
  qgemv_scores_kernel<<<std::max(blocks, 1), 256, 0, st>>>(c, u, n, q, logits);
  return check_launch("tkv_qgemv_scores");
}
int qgemv_output(const QC &c, int u, int64_t n, const double *w, double *out, void *ws, cudaStream_t st) {
  const int chunks = (int)((n + QG_CHUNK - 1) / QG_CHUNK);
  double *part = static_cast<double *>(ws);
  qgemv_output_part_kernel<<<chunks, 256, 0, st>>>(c, u, n, w, part);
  qgemv_output_sum_kernel<<<1, 256, 0, st>>>(part, chunks, c.d, out);
  return check_launch("tkv_qgemv_output");
}

}  // namespace tkv
