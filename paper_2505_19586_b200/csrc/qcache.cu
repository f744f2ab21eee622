#include <algorithm>
// Quantized layer cache: prefill pack, decode append, GQT1 export, dequant,
// raw GEMVs.  Reference: hybridkv/quantizer.py:187-558.
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "qcache.cuh"

namespace tkv {

// ---------------------------------------------------------------------------
// Prefill pack (quantize_layer_kv, quantizer.py:252-293, 479-497): HBM-bound.
// The codec is a monotone step function of x inside a group, so each group's
// codes are fixed by 2^b - 1 fp16 thresholds: T_k = the smallest fp16 x in
// [lo, hi] whose float64 reference code is >= k, found by a short search next
// to the real-valued boundary.  Encoding is then fp16x2 compares, with no
// division and no float64 per element; code(x) = sum_k [x >= T_k] is exactly
// the reference's code for every fp16 x in the group.  A degenerate group
// (hi == lo, code 0) gets NaN thresholds, which no compare passes.
// Persistent CTAs stage tiles with 16-byte cp.async into padded rows
// (conflict-free SMEM), double-buffered so the next tile's copy overlaps this
// tile's work; group min/max uses fp16x2 min/max (exact), the MMA-native words
// are assembled straight from the tile and written 8 bytes per thread
// (consecutive threads, consecutive words), and the largest group scale is
// kept per thread and published with one atomic per warp per unit.
// ---------------------------------------------------------------------------
// Group min/max with fp16 min/max, which order -0 below +0: a zero minimum is
// stored as -0 when the group holds a -0 (the reference's float64 min keeps
// the sign of the zero it meets; with both signs present its pick follows
// numpy's reduction order and is not reproduced).  The sign of a zero maximum
// never reaches an output (only hi - lo is used).
__device__ __forceinline__ uint16_t hmin_bits(uint16_t a, uint16_t b) {
  return __half_as_ushort(__hmin(__ushort_as_half(a), __ushort_as_half(b)));
}
__device__ __forceinline__ uint16_t hmax_bits(uint16_t a, uint16_t b) {
  return __half_as_ushort(__hmax(__ushort_as_half(a), __ushort_as_half(b)));
}

// fp16 bits <-> a signed order index (-0 and +0 both map to 0).
__device__ __forceinline__ int h_ord(uint16_t h) { return (h & 0x8000u) ? -(int)(h & 0x7fffu) : (int)h; }
__device__ __forceinline__ uint16_t h_unord(int o) { return o < 0 ? (uint16_t)(0x8000u | (uint32_t)(-o)) : (uint16_t)o; }

// T_k for one group (lo <= hi as fp16 bits), k = 1 .. 2^b - 1.
//   b = 1: code(x) = [2x >= hi + lo] (float64, exact: fp16 sums are exact there), so T_1 is the
//          fp16 round-up of the exact midpoint (hi + lo) / 2.
//   b = 2: code(x) >= k  <=>  (x - lo) / sd >= k - 1/2 up to float64 rounding, sd = (hi - lo) / 3
//          rounded as the reference does.  With m = lo + (k - 1/2) sd, T_k is the fp16 round-up c of
//          m, unless c or its fp16 predecessor p lies within 1e-12 (relative) of m -- an exact or
//          near tie, common because group bounds share the fp16 grid -- where the reference's
//          float64 code of that one candidate decides between it and its neighbour.
__device__ __forceinline__ uint16_t ceil_f16(double m) {  // the smallest fp16 >= m
  // fp32 round-to-nearest keeps every fp16 >= m above it, except when it lands exactly on an fp16 below m
  const uint16_t c = __half_as_ushort(__float2half_ru(__double2float_rn(m)));
  return h2d(c) < m ? h_unord(h_ord(c) + 1) : c;
}

// sd = (hi - lo) / 3 as the reference rounds it (b = 2; unused at b = 1)
template <int BITS>
__device__ __forceinline__ double group_sd(double lo, double hi) {
  return BITS == 2 ? __ddiv_rn(__dsub_rn(hi, lo), 3.0) : 0.0;
}

template <int BITS>
__device__ __forceinline__ uint16_t code_threshold(uint16_t lob, uint16_t hib, double sd, int k) {
  const double lo = h2d(lob), hi = h2d(hib);
  if (!(hi > lo)) return 0x7fffu;  // degenerate: code 0 everywhere
  if (BITS == 1) return ceil_f16(__dmul_rn(__dadd_rn(hi, lo), 0.5));
  const double m = __fma_rn((double)k - 0.5, sd, lo);
  const uint16_t c = ceil_f16(m);
  const int oc = h_ord(c);
  const uint16_t p = h_unord(oc - 1);
  const double band = 1e-12 * (fabs(lo) + fabs(m) + sd);
  const bool p_near = m - h2d(p) <= band, c_near = h2d(c) - m <= band;
  if (!p_near && !c_near) return c;
  // quantizer.py:99-107 on one candidate: round_half_away((x - lo) / sd) >= k
  const uint16_t cand = p_near ? p : c, alt = p_near ? c : h_unord(oc + 1);
  const double vd = __ddiv_rn(__dsub_rn(h2d(cand), lo), sd);
  return floor(__dadd_rn(fabs(vd), 0.5)) >= (double)k ? cand : alt;
}

__device__ __forceinline__ uint32_t hge2_mask(uint32_t x, uint32_t t) {
  return __hge2_mask(*reinterpret_cast<__half2 *>(&x), *reinterpret_cast<__half2 *>(&t));
}

// Code bits of two fp16 (x) against per-element thresholds t[0..NT) (half2 each): the masks are nested
// (T_1 <= T_2 <= T_3), so bit 0 of the count is their XOR and bit 1 is the second mask.  The result
// holds element 0's code at bit `sh` and element 1's at bit 16 + sh.
template <int BITS>
__device__ __forceinline__ uint32_t code_bits2(uint32_t x, const uint32_t *t, int sh) {
  if constexpr (BITS == 1) {
    return hge2_mask(x, t[0]) & (0x00010001u << sh);
  } else {
    const uint32_t m1 = hge2_mask(x, t[0]), m2 = hge2_mask(x, t[1]), m3 = hge2_mask(x, t[2]);
    return ((m1 ^ m2 ^ m3) & (0x00010001u << sh)) | (m2 & (0x00020002u << sh));
  }
}

// Stage rows x (8*vpr) fp16 from global (dense) into SMEM rows of stride RS with 16-byte cp.async
// (no registers held: the copy of the next tile overlaps this tile's work), one commit group.
__device__ __forceinline__ void tile_load_async(uint16_t *tile, int RS, const uint16_t *src, int rows, int vpr) {
  const int step_r = blockDim.x / vpr, step_c = blockDim.x % vpr;
  int r = threadIdx.x / vpr, col = threadIdx.x % vpr;
  const uint4 *s4 = reinterpret_cast<const uint4 *>(src);
  for (int v = threadIdx.x; v < rows * vpr; v += blockDim.x) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(tile + (size_t)r * RS + col * 8);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(s4 + v) : "memory");
    r += step_r;
    col += step_c;
    if (col >= vpr) {
      col -= vpr;
      ++r;
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// (u, i) += step over items laid out unit-major with `per` items per unit
__device__ __forceinline__ void item_advance(int &u, int &i, int step, int per) {
  i += step;
  while (i >= per) {
    i -= per;
    ++u;
  }
}

// Publish a running per-unit scale maximum (v >= 0): warp max, one atomic per warp.
__device__ __forceinline__ void flush_max(float v, float *gaddr) {
  const int vi = __reduce_max_sync(0xffffffffu, __float_as_int(v));
  if ((threadIdx.x & 31) == 0 && vi > 0) atomicMax(reinterpret_cast<int *>(gaddr), vi);
}

constexpr int PK_PAD = 16;  // key tile row padding (fp16): rows 8 banks apart for 8-byte loads
constexpr int PK_SEG = 4;   // row segments per key group in the min/max

// Pack keys: persistent CTAs over (unit, key tile of Tk = 16*8/b tokens) items, double-buffered;
// groups are G tokens x 1 channel.  D = head_dim when specialised, 0 = runtime c.d.
template <int BITS, int G, int D>
__global__ void __launch_bounds__(256) pack_keys_kernel(QC c, const uint16_t *__restrict__ keys, int64_t n,
                                                         int64_t n_complete, int tiles) {
  constexpr int Tk = 16 * (8 / BITS), NT = (1 << BITS) - 1, KS = 8 / BITS, GR = Tk / G, SR = G / PK_SEG;
  extern __shared__ __align__(16) unsigned char smem[];
  const int d = D ? D : c.d;
  const int RS = d + PK_PAD, P2 = d / 2, vpr = d / 8;  // row stride (fp16), channel pairs, 16-byte vectors
  uint16_t *tiles2 = reinterpret_cast<uint16_t *>(smem);                                    // [2][Tk][RS]
  uint32_t *thr = reinterpret_cast<uint32_t *>(tiles2 + (size_t)2 * Tk * RS);              // [GR][NT][d/2] fp16x2
  uint2 *red = reinterpret_cast<uint2 *>(thr + (size_t)GR * NT * P2);                      // [GR][SEG][d/2]
  double *gsd = reinterpret_cast<double *>(red + (size_t)GR * PK_SEG * P2);                 // [GR][d]
  uint32_t *bounds = reinterpret_cast<uint32_t *>(gsd + (size_t)GR * d);                    // [GR][d]
  uint16_t *thr16 = reinterpret_cast<uint16_t *>(thr);
  const int items = tiles * c.units;
  if ((int)blockIdx.x >= items) return;
  auto issue = [&](int uu, int tt, int bb) {
    const int64_t s0 = (int64_t)tt * Tk;
    tile_load_async(tiles2 + (size_t)bb * Tk * RS, RS, keys + ((size_t)uu * n + s0) * d, (int)imin64(Tk, n_complete - s0),
                    vpr);
  };
  int u = 0, ti = 0;
  item_advance(u, ti, blockIdx.x, tiles);
  issue(u, ti, 0);
  int cur_u = u;
  float smax = 0.0f;
  for (int w = blockIdx.x, buf = 0; w < items; w += gridDim.x, buf ^= 1) {
    int un = u, tn = ti;
    item_advance(un, tn, gridDim.x, tiles);
    if (w + (int)gridDim.x < items) issue(un, tn, buf ^ 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    cp_async_wait_prev();
    __syncthreads();
    const int64_t t0 = (int64_t)ti * Tk;
    const int groups = (int)imin64(Tk, n_complete - t0) / G;  // complete groups only
    if (u != cur_u) {
      flush_max(smax, &c.val_smax[2 * cur_u + 1]);
      cur_u = u;
      smax = 0.0f;
    }
    const uint16_t *tile = tiles2 + (size_t)buf * Tk * RS;
    for (int it = threadIdx.x; it < groups * PK_SEG * P2; it += blockDim.x) {
      const int p = it % P2, r0 = (it / P2) * SR;  // (grp, seg) rows are contiguous
      const uint32_t *col = reinterpret_cast<const uint32_t *>(tile) + (size_t)r0 * (RS / 2) + p;
      uint32_t x = col[0];
      __half2 lo = *reinterpret_cast<__half2 *>(&x), hi = lo;
#pragma unroll
      for (int r = 1; r < SR; ++r) {
        x = col[r * (RS / 2)];
        lo = __hmin2(lo, *reinterpret_cast<__half2 *>(&x));
        hi = __hmax2(hi, *reinterpret_cast<__half2 *>(&x));
      }
      red[it] = make_uint2(*reinterpret_cast<uint32_t *>(&lo), *reinterpret_cast<uint32_t *>(&hi));
    }
    __syncthreads();
    // (group, channel): bounds, sd; then one thread per (threshold k, group, channel); groups past a partial
    // tile get NaN thresholds (code 0)
    for (int it = threadIdx.x; it < groups * d; it += blockDim.x) {
      const int ch = it % d, grp = it / d;
      const int e = ch & 1;
      uint16_t lb = 0, hb = 0;
#pragma unroll
      for (int sg = 0; sg < PK_SEG; ++sg) {
        const uint2 lh = red[((size_t)grp * PK_SEG + sg) * P2 + (ch >> 1)];
        const uint16_t l = (uint16_t)(e ? lh.x >> 16 : lh.x), h = (uint16_t)(e ? lh.y >> 16 : lh.y);
        lb = sg ? hmin_bits(lb, l) : l;
        hb = sg ? hmax_bits(hb, h) : h;
      }
      const uint32_t w2 = pack_lohi(lb, hb);  // zero signs: hmin_bits
      bounds[it] = w2;
      if (BITS == 2) gsd[it] = group_sd<BITS>(h2d(lb), h2d(hb));
      c.key_lohi[((size_t)u * (c.capacity / G) + (t0 / G) + grp) * d + ch] = w2;
      const float lf = h2f(lb), hf = h2f(hb);
      smax = fmaxf(smax, hf > lf ? (hf - lf) / (float)NT : 0.0f);
    }
    __syncthreads();
    for (int it = threadIdx.x; it < NT * GR * d; it += blockDim.x) {
      const int gc = it % (GR * d), k = it / (GR * d) + 1;
      uint16_t tk = 0x7fffu;
      if (gc < groups * d) {
        const uint32_t w2 = bounds[gc];
        tk = code_threshold<BITS>((uint16_t)(w2 & 0xffffu), (uint16_t)(w2 >> 16), BITS == 2 ? gsd[gc] : 0.0, k);
      }
      thr16[((size_t)(gc / d) * NT + k - 1) * d + gc % d] = tk;
    }
    __syncthreads();
    // native words: thread (ks, lane, role pair rp) writes roles 2rp, 2rp+1 (tokens +0 / +8)
    // of channels ch0 .. ch0+3; token 16k + g8 + 8r lies in group 16k / G
    uint2 *dst = reinterpret_cast<uint2 *>(c.key_codes + ((size_t)u * (c.capacity / Tk) + ti) * (d / 32) * 128);
    for (int q = threadIdx.x; q < d * 2; q += blockDim.x) {
      const int rp = q & 1, lane = (q >> 1) & 31, ks = q >> 6;
      const int g8 = lane >> 2, tq = lane & 3;
      const int ch0 = 32 * ks + 16 * rp + 4 * tq;
      uint32_t a0[2] = {0u, 0u}, a1[2] = {0u, 0u};  // channels (0,1) and (2,3): slot k's code at bit k*b (+16)
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        const uint2 *tk = reinterpret_cast<const uint2 *>(thr + (size_t)((16 * k) / G) * NT * P2 + ch0 / 2);
        uint32_t tx[NT], ty[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const uint2 tt = tk[j * (P2 / 2)];
          tx[j] = tt.x;
          ty[j] = tt.y;
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const uint2 x = *reinterpret_cast<const uint2 *>(tile + (size_t)(16 * k + g8 + 8 * r) * RS + ch0);
          a0[r] |= code_bits2<BITS>(x.x, tx, k * BITS);
          a1[r] |= code_bits2<BITS>(x.y, ty, k * BITS);
        }
      }
      dst[(ks * 32 + lane) * 2 + rp] = make_uint2(__byte_perm(a0[0], a1[0], 0x6420), __byte_perm(a0[1], a1[1], 0x6420));
    }
    __syncthreads();  // the tile, red and thr are reused
    u = un;
    ti = tn;
  }
  flush_max(smax, &c.val_smax[2 * cur_u + 1]);
}

constexpr int PV_TOK = 128;           // tokens per value item (4 value tiles)
constexpr int PV_PAD = 8;             // value tile row padding (fp16): conflict-free 16-byte row loads
constexpr int PV_CT = PV_TOK + 16;    // code-byte row stride: 4-byte loads of 4 g8 rows on distinct banks

// Pack values: persistent CTAs over (unit, 128-token) items, double-buffered; groups are 1 token x G
// channels (a ragged last block allowed).  Thread (token, block) keeps its group in registers: min/max,
// thresholds, then codes.  Channel 16k + j of a word set (j < 16) contributes bits k*b of byte j, so the
// thread writes 16 code bytes per block into codes[set][part][j][token] (part = the block's slice of the
// set); a word then ORs its parts with one 4-token load each.
template <int BITS, int G, int D>
__global__ void __launch_bounds__(256) pack_values_kernel(QC c, const uint16_t *__restrict__ values, int64_t n,
                                                           int chunks) {
  constexpr int NT = (1 << BITS) - 1, KS = 8 / BITS, PER = 16 * KS, PARTS = PER / G;
  extern __shared__ __align__(16) unsigned char smem[];
  const int d = D ? D : c.d;
  const int nb = (d + G - 1) / G;
  const int RS = d + PV_PAD, vpr = d / 8;
  const int sets = val_sets(d, BITS);
  uint16_t *tiles2 = reinterpret_cast<uint16_t *>(smem);                              // [2][PV_TOK][RS]
  uint8_t *codes = reinterpret_cast<uint8_t *>(tiles2 + (size_t)2 * PV_TOK * RS);    // [sets][PARTS][16][PV_CT]
  const int items = chunks * c.units;
  if ((int)blockIdx.x >= items) return;
  auto issue = [&](int uu, int cc, int bb) {
    const int64_t s0 = (int64_t)cc * PV_TOK;
    tile_load_async(tiles2 + (size_t)bb * PV_TOK * RS, RS, values + ((size_t)uu * n + s0) * d,
                    (int)imin64(PV_TOK, n - s0), vpr);
  };
  int u = 0, ci = 0;
  item_advance(u, ci, blockIdx.x, chunks);
  issue(u, ci, 0);
  int cur_u = u;
  float smax = 0.0f;
  for (int w = blockIdx.x, buf = 0; w < items; w += gridDim.x, buf ^= 1) {
    int un = u, cn = ci;
    item_advance(un, cn, gridDim.x, chunks);
    if (w + (int)gridDim.x < items) issue(un, cn, buf ^ 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    cp_async_wait_prev();
    __syncthreads();
    const int64_t t0 = (int64_t)ci * PV_TOK;
    const int rows = (int)imin64(PV_TOK, n - t0);
    if (u != cur_u) {
      flush_max(smax, &c.val_smax[2 * cur_u]);
      cur_u = u;
      smax = 0.0f;
    }
    const uint16_t *tile = tiles2 + (size_t)buf * PV_TOK * RS;
    for (int p = threadIdx.x; p < PV_TOK * nb; p += blockDim.x) {
      const int t = p % PV_TOK, b = p / PV_TOK;
      const int c0 = b * G, nv = (min(d, c0 + G) - c0) / 8;  // 16-byte vectors in the block (>= 2)
      uint32_t acc[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // acc[q]: bytes j = 2q (bits 0-7), 2q+1 (bits 16-23)
      if (t < rows) {
        const uint4 *row = reinterpret_cast<const uint4 *>(tile + (size_t)t * RS + c0);
        uint32_t xs[G / 2];
        __half2 lo, hi;
#pragma unroll
        for (int v = 0; v < G / 8; ++v) {
          if (v < nv) {
            const uint4 x = row[v];
            xs[4 * v] = x.x;
            xs[4 * v + 1] = x.y;
            xs[4 * v + 2] = x.z;
            xs[4 * v + 3] = x.w;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const __half2 h = *reinterpret_cast<const __half2 *>(&xs[4 * v + j]);
              lo = (v | j) ? __hmin2(lo, h) : h;
              hi = (v | j) ? __hmax2(hi, h) : h;
            }
          }
        }
        const __half l = __hmin(__low2half(lo), __high2half(lo)), h = __hmax(__low2half(hi), __high2half(hi));
        const uint16_t lb = __half_as_ushort(l), hb = __half_as_ushort(h);  // zero signs: see hmin_bits
        c.val_lohi[((size_t)u * c.capacity + t0 + t) * nb + b] = pack_lohi(lb, hb);
        smax = fmaxf(smax, group_scale_f(__half2float(l), __half2float(h), BITS));
        uint32_t th[NT];
        const double sd = group_sd<BITS>(h2d(lb), h2d(hb));
#pragma unroll
        for (int k = 1; k <= NT; ++k) {
          const uint32_t tk = code_threshold<BITS>(lb, hb, sd, k);
          th[k - 1] = tk | (tk << 16);
        }
        const int kb = (b % PARTS) * (G / 16);  // the block's first k within its set
#pragma unroll
        for (int m = 0; m < G / 2; ++m)  // channel pair (2m, 2m+1): j = 2m % 16, k = kb + m / 8
          if (m < 4 * nv) acc[m % 8] |= code_bits2<BITS>(xs[m], th, (kb + m / 8) * BITS);
      }
      uint8_t *cb = codes + ((size_t)(c0 / PER) * PARTS + (b % PARTS)) * 16 * PV_CT + t;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        cb[(2 * q) * PV_CT] = (uint8_t)acc[q];
        cb[(2 * q + 1) * PV_CT] = (uint8_t)(acc[q] >> 16);
      }
    }
    __syncthreads();
    const int ntiles = (rows + 31) / 32;
    uint2 *dst = reinterpret_cast<uint2 *>(c.val_codes + ((size_t)u * (c.capacity / 32) + t0 / 32) * sets * 128);
    // thread (tile vt, set, lane, role pair rp) writes roles 2rp, 2rp+1 (channels +0 / +8): byte i holds
    // token 4tq + i + 16rp, bits k*b channel set*PER + 16k + g8 (+8)
    for (int q = threadIdx.x; q < ntiles * sets * 64; q += blockDim.x) {
      const int rp = q & 1, lane = (q >> 1) & 31, set = (q >> 6) % sets, vt = q / (sets * 64);
      const int g8 = lane >> 2, tq = lane & 3;
      const int tb = vt * 32 + 4 * tq + 16 * rp;
      uint32_t wv[2] = {0u, 0u};
#pragma unroll
      for (int pt = 0; pt < PARTS; ++pt) {
        if (set * PER + pt * G < d) {
          const uint8_t *cb = codes + ((size_t)set * PARTS + pt) * 16 * PV_CT + tb;
          wv[0] |= *reinterpret_cast<const uint32_t *>(cb + g8 * PV_CT);
          wv[1] |= *reinterpret_cast<const uint32_t *>(cb + (g8 + 8) * PV_CT);
        }
      }
      dst[((vt * sets + set) * 32 + lane) * 2 + rp] = make_uint2(wv[0], wv[1]);
    }
    __syncthreads();  // the tile and codes are reused
    u = un;
    ci = cn;
  }
  flush_max(smax, &c.val_smax[2 * cur_u]);
}

static int pack_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

template <typename K>
static unsigned persistent_grid(K kernel, size_t sm, int64_t items) {
  int per_sm = 0;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, sm) != cudaSuccess || per_sm < 1) per_sm = 1;
  return (unsigned)std::min<int64_t>(items, (int64_t)per_sm * pack_sms());
}

template <int BITS, int G, int D>
static void launch_pack(const QC &c, const uint16_t *keys, const uint16_t *values, int64_t n, int64_t n_complete,
                        cudaStream_t st) {
  constexpr int Tk = 16 * (8 / BITS), NT = (1 << BITS) - 1, GR = Tk / G;
  if (n_complete > 0) {
    const int tiles = (int)((n_complete + Tk - 1) / Tk);
    const size_t sm = (size_t)2 * Tk * (c.d + PK_PAD) * 2 + (size_t)GR * NT * c.d * 2 + (size_t)GR * PK_SEG * (c.d / 2) * 8 +
                      (size_t)GR * c.d * 12;
    const unsigned grid = persistent_grid(pack_keys_kernel<BITS, G, D>, sm, (int64_t)tiles * c.units);
    pack_keys_kernel<BITS, G, D><<<grid, 256, sm, st>>>(c, keys, n, n_complete, tiles);
  }
  const int chunks = (int)((n + PV_TOK - 1) / PV_TOK);
  const size_t sm = (size_t)2 * PV_TOK * (c.d + PV_PAD) * 2 + (size_t)val_sets(c.d, BITS) * (16 * (8 / BITS) / G) * 16 * PV_CT;
  const unsigned grid = persistent_grid(pack_values_kernel<BITS, G, D>, sm, (int64_t)chunks * c.units);
  pack_values_kernel<BITS, G, D><<<grid, 256, sm, st>>>(c, values, n, chunks);
}

template <int BITS, int G>
static void launch_pack_d(const QC &c, const uint16_t *keys, const uint16_t *values, int64_t n, int64_t n_complete,
                          cudaStream_t st) {
  if (c.d == 128) launch_pack<BITS, G, 128>(c, keys, values, n, n_complete, st);
  else if (c.d == 64) launch_pack<BITS, G, 64>(c, keys, values, n, n_complete, st);
  else launch_pack<BITS, G, 0>(c, keys, values, n, n_complete, st);
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
  const int64_t n_complete = (n / c.g) * c.g;
  cudaMemsetAsync(c.val_smax, 0, sizeof(float) * 2 * c.units, st);
  switch (c.bits * 1000 + c.g) {
    case 1016: launch_pack_d<1, 16>(c, keys, values, n, n_complete, st); break;
    case 1032: launch_pack_d<1, 32>(c, keys, values, n, n_complete, st); break;
    case 1064: launch_pack_d<1, 64>(c, keys, values, n, n_complete, st); break;
    case 1128: launch_pack_d<1, 128>(c, keys, values, n, n_complete, st); break;
    case 2016: launch_pack_d<2, 16>(c, keys, values, n, n_complete, st); break;
    case 2032: launch_pack_d<2, 32>(c, keys, values, n, n_complete, st); break;
    case 2064: launch_pack_d<2, 64>(c, keys, values, n, n_complete, st); break;
    default: return fail(TKV_ERR_PARAMETER, "unsupported (bits, group_size) for the CUDA pack");
  }
  if (n > n_complete) {
    dim3 grid((unsigned)(n - n_complete), c.units);
    copy_residual_kernel<<<grid, 128, 0, st>>>(c, keys, n, n_complete);
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
    for (int ch = c0 + 1; ch < c1; ++ch) {
      const uint16_t xb = vrow[ch];
      lob = hmin_bits(lob, xb);
      hib = hmax_bits(hib, xb);
    }
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
        lob = hmin_bits(lob, xb);
        hib = hmax_bits(hib, xb);
      }
      lo = h2f(lob);
      hi = h2f(hib);
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
