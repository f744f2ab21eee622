// Tensor-core quantized decode attention for d = 128,
// g = 64, 1/2-bit codes, up to 4 query heads per KV head.
//
// Keys:   logits[t, h] = sum_c code[t,c] * (q[h,c] s[g,c]) + q[h] . lo[g]
//         (quantizer.py:505-533).  MMA m16n8k32 u8 x s8 -> s32 with
//         A = key codes (tokens x channels) taken straight from the packed
//         bit-planes with ONE LOP3 per 4 codes: byte lanes of a code word hold
//         the codes of 8/b different m-tiles at bit offset k*b, so
//         (word & mask_k) is the u8 operand scaled by 2^(k b), undone on the
//         int32 result.  B = q*s quantised to a 16-bit fixed point split into
//         two s8 digits (hi, lo) that occupy the 8 N columns (4 heads x 2).
// Values: out^T[c, h] = sum_t code[t,c] * (p[t,h] s[t,cb]) + sum_t p lo
//         (quantizer.py:536-558), same operand trick with A = value codes
//         (channels x tokens).  Integer accumulation is exact, so the split-K
//         partial only carries the fixed-point rounding of B.
// Softmax: online max/rescale per 64-token group (pipeline.py:153-156, 336).
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "qcache.cuh"

namespace tkv {

constexpr int IM_D = 128;
constexpr int IM_G = 64;
constexpr int IM_CHUNK = 512;                  // tokens per CTA at b=1 (8 KB of key codes)
constexpr int IM_GROUPS = IM_CHUNK / IM_G;     // 8
constexpr int IM_WARPS = 4;
constexpr float IM_QMAX = 32512.0f;            // |x| bound of the 2-digit fixed point
constexpr float IM_MAGIC = 12582912.0f + 128.0f;  // 1.5*2^23 + 128: RNE to int, +128 digit bias

// the pipelined kernel takes any G in blocks of 4 query heads; the per-chunk kernel G <= 4
bool imma_supported(const QC &c, int G) {
  return c.d == IM_D && c.g == IM_G && (c.bits == 1 || c.bits == 2) && G >= 1 && G <= 16;
}

__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// pack the digit byte (sel: 0x1 hi = byte 1, 0x0 lo = byte 0) of four
// fixed-point floats into one s8x4 register; lo digits are re-centred by ^0x80
__device__ __forceinline__ uint32_t pack_digits(float x0, float x1, float x2, float x3, uint32_t sel2,
                                                uint32_t sel4, uint32_t xr) {
  const uint32_t a = __byte_perm(__float_as_uint(x0), __float_as_uint(x1), sel2);
  const uint32_t b = __byte_perm(__float_as_uint(x2), __float_as_uint(x3), sel2);
  return __byte_perm(a, b, 0x5410) ^ xr;
  (void)sel4;
}

// (TMA 1-D bulk copy and mbarrier helpers: common.cuh)

// Staging area: the chunk's packed codes and group parameters, brought in by
// four bulk copies at CTA start (16 KB keys + 16 KB values + params).
struct ImStage {
  uint4 kc[IM_CHUNK];             // key code words of the chunk (16 B per token at b=1)
  uint4 vc[IM_CHUNK];             // value code words of the chunk
  uint32_t klohi[IM_GROUPS * 128];  // key (lo, hi) per group x channel
  uint32_t vlohi[IM_CHUNK * 2];     // value (lo, hi) per token x channel block
  uint64_t bar[2];
};

struct ImSmem {
  float q[4][IM_D];             // query (h < G, else 0)
  float kscale[IM_GROUPS][4];   // per (group, head): max_c |q_hc s_gc| / 32512
  float off[IM_GROUPS][4];      // q_h . lo_g
  uint32_t bfrag[IM_GROUPS][4][36][2];  // key B fragments per group, k-step, lane (padded rows)
  union {
    struct {
      float s[IM_GROUPS][IM_D];  // key scales of the chunk's groups
      float lo[IM_GROUPS][IM_D];
    } k;
    struct {
      float sv[2][IM_CHUNK];     // value scale * 32512/Smax_v per (cb, token)
      float lov[2][IM_CHUNK];    // value zero-point per (cb, token)
    } v;
  } u;
  float p[IM_WARPS][4][IM_G + 8];  // per-warp softmax numerators of the current group (padded rows)
  float wm[IM_WARPS][4], wl[IM_WARPS][4];
};

template <int BITS>
__global__ void __launch_bounds__(IM_WARPS * 32, 4) quant_decode_imma_kernel(QC c, const uint16_t *__restrict__ queries,
                                                                              int G, float *__restrict__ pm,
                                                                              float *__restrict__ pl,
                                                                              float *__restrict__ pacc, int chunks,
                                                                              unsigned *__restrict__ arrive,
                                                                              float *__restrict__ out) {
  constexpr int CH = IM_CHUNK / BITS;      // tokens per CTA (16 KB of key codes)
  constexpr int NG = CH / IM_G;            // groups per CTA
  constexpr int KT = 128 / BITS;           // key tile tokens
  constexpr int GPT = KT / IM_G;           // groups per key tile
  constexpr int VS = BITS;                 // value code sets (d = 128)
  constexpr int SLOTS = 8 / BITS;
  constexpr uint32_t CM = BITS == 1 ? 0x01010101u : 0x03030303u;
  extern __shared__ __align__(16) unsigned char smraw[];
  ImSmem &S = *reinterpret_cast<ImSmem *>(smraw);
  ImStage &T = *reinterpret_cast<ImStage *>(smraw + ((sizeof(ImSmem) + 127) & ~size_t(127)));
  const int u = blockIdx.y, chunk = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g8 = lane >> 2, tq = lane & 3;
  const int64_t n = *c.len;
  const int64_t t0 = (int64_t)chunk * CH;
  if (t0 >= n) return;
  // ---- issue the chunk's bulk copies first; params on bar[0], codes on bar[1] ----
  if (tid == 0) {
    mbar_init(&T.bar[0], 1);
    mbar_init(&T.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    const int64_t cap = c.capacity;
    const int64_t g0c = t0 / IM_G, kt0 = t0 / KT, vt0 = t0 / 32;
    const uint32_t kl_bytes = (uint32_t)(imin64(NG, cap / IM_G - g0c) * IM_D * 4);
    const uint32_t vl_bytes = (uint32_t)(imin64(CH, cap - t0) * 8);
    const uint32_t kc_bytes = (uint32_t)(imin64(CH / KT, cap / KT - kt0) * 2048);
    const uint32_t vc_bytes = (uint32_t)(imin64(CH / 32, cap / 32 - vt0) * VS * 512);
    mbar_expect_tx(&T.bar[0], kl_bytes + vl_bytes);
    bulk_g2s(T.klohi, c.key_lohi + ((size_t)u * (cap / IM_G) + g0c) * IM_D, kl_bytes, &T.bar[0]);
    bulk_g2s(T.vlohi, c.val_lohi + ((size_t)u * cap + t0) * 2, vl_bytes, &T.bar[0]);
    mbar_expect_tx(&T.bar[1], kc_bytes + vc_bytes);
    bulk_g2s(T.kc, c.key_codes + ((size_t)u * (cap / KT) + kt0) * 512, kc_bytes, &T.bar[1]);
    bulk_g2s(T.vc, c.val_codes + ((size_t)u * (cap / 32) + vt0) * VS * 128, vc_bytes, &T.bar[1]);
  }
  const int64_t ncomp = (n / IM_G) * IM_G;
  const float inv_sqrt_d = 0.08838834764831845f;  // 1/sqrt(128)
  const float kmax_s = c.val_smax[2 * u + 1];
  const float vmax_s = c.val_smax[2 * u];
  (void)vmax_s;

  // ---- prologue: query, fixed-point scales, per-group key params ----
  for (int i = tid; i < 4 * IM_D; i += blockDim.x) {
    const int h = i / IM_D;
    S.q[h][i % IM_D] = h < G ? h2f(queries[((size_t)u * G + h) * IM_D + i % IM_D]) : 0.0f;
  }
  __syncthreads();
  (void)kmax_s;
  const int ngroups = (int)imin64(NG, (n - t0 + IM_G - 1) / IM_G);
  const int64_t g0 = t0 / IM_G;
  constexpr float KINV = 1.0f / (float)((1 << BITS) - 1);
  mbar_wait(&T.bar[0], 0);
  // Key groups, one warp per group, lane = one channel quad of the B-fragment
  // layout (ks, j, tq): decode (lo, s) from the staged params, offsets
  // q_h . lo_g, the per-(group, head) bound max_c |q_hc s_gc| (halving
  // butterflies), then the two s8 digits of every W = q s.
  {
    const int tqq = lane & 3, j = (lane >> 2) & 1, ks = lane >> 3;
    const int ch = 32 * ks + 16 * j + 4 * tqq;
    float4 qv[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) qv[h] = *reinterpret_cast<const float4 *>(&S.q[h][ch]);
    const bool b4 = lane & 16, b3 = lane & 8;
    for (int gi = warp; gi < NG; gi += IM_WARPS) {
      float lo[4] = {0.f, 0.f, 0.f, 0.f}, sc[4] = {0.f, 0.f, 0.f, 0.f};
      if (gi < ngroups && (g0 + gi + 1) * IM_G <= ncomp) {
        const uint4 raw = *reinterpret_cast<const uint4 *>(&T.klohi[gi * IM_D + ch]);
        const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          lo[i] = h2f(w[i] & 0xffff);
          sc[i] = (h2f(w[i] >> 16) - lo[i]) * KINV;  // 0 for degenerate groups (all codes 0)
        }
      }
      float W[4][4], dt[4], mx[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float qa[4] = {qv[h].x, qv[h].y, qv[h].z, qv[h].w};
        dt[h] = 0.0f;
        mx[h] = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          W[h][i] = qa[i] * sc[i];
          dt[h] = fmaf(qa[i], lo[i], dt[h]);
          mx[h] = fmaxf(mx[h], fabsf(W[h][i]));
        }
      }
      float d2[2], m2[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float sd = b4 ? dt[k] : dt[k + 2], sm = b4 ? mx[k] : mx[k + 2];
        const float rd = __shfl_xor_sync(0xffffffffu, sd, 16), rm = __shfl_xor_sync(0xffffffffu, sm, 16);
        d2[k] = (b4 ? dt[k + 2] : dt[k]) + rd;
        m2[k] = fmaxf(b4 ? mx[k + 2] : mx[k], rm);
      }
      float d1, m1;
      {
        const float sd = b3 ? d2[0] : d2[1], sm = b3 ? m2[0] : m2[1];
        const float rd = __shfl_xor_sync(0xffffffffu, sd, 8), rm = __shfl_xor_sync(0xffffffffu, sm, 8);
        d1 = (b3 ? d2[1] : d2[0]) + rd;
        m1 = fmaxf(b3 ? m2[1] : m2[0], rm);
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        d1 += __shfl_xor_sync(0xffffffffu, d1, o);
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
      }
      if ((lane & 7) == 0) {
        const int h = (b4 ? 2 : 0) + (b3 ? 1 : 0);
        S.off[gi][h] = d1;
        S.kscale[gi][h] = m1 * (1.0f / IM_QMAX);
      }
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float mh = __shfl_sync(0xffffffffu, m1, 8 * h);
        const float inv = mh > 0.0f ? __fdividef(IM_QMAX, mh) : 0.0f;
        const float x0 = fmaf(W[h][0], inv, IM_MAGIC), x1 = fmaf(W[h][1], inv, IM_MAGIC);
        const float x2 = fmaf(W[h][2], inv, IM_MAGIC), x3 = fmaf(W[h][3], inv, IM_MAGIC);
        S.bfrag[gi][ks][(2 * h) * 4 + tqq][j] = pack_digits(x0, x1, x2, x3, 0x0051, 0, 0u);              // hi: bytes 1
        S.bfrag[gi][ks][(2 * h + 1) * 4 + tqq][j] = pack_digits(x0, x1, x2, x3, 0x0040, 0, 0x80808080u);  // lo: bytes 0
      }
    }
  }
  // value params of the chunk's tokens: both channel blocks of a token at once
  for (int t = tid; t < CH; t += blockDim.x) {
    float s0 = 0.f, s1 = 0.f, l0 = 0.f, l1 = 0.f;
    if (t0 + t < n) {
      const uint2 w = *reinterpret_cast<const uint2 *>(&T.vlohi[2 * t]);
      l0 = h2f(w.x & 0xffff);
      l1 = h2f(w.y & 0xffff);
      s0 = (h2f(w.x >> 16) - l0) * KINV;
      s1 = (h2f(w.y >> 16) - l1) * KINV;
    }
    S.u.v.sv[0][t] = s0;
    S.u.v.sv[1][t] = s1;
    S.u.v.lov[0][t] = l0;
    S.u.v.lov[1][t] = l1;
  }
  __syncthreads();

  // ---- main loop: each warp walks whole key tiles of its chunk ----
  mbar_wait(&T.bar[1], 0);
  const uint16_t *kres = c.key_resid + (size_t)u * IM_G * IM_D;
  const uint32_t dsel = (g8 & 1) ? 0x0040u : 0x0051u;  // this lane's B column digit
  const uint32_t dxor = (g8 & 1) ? 0x80808080u : 0u;
  const int hB = g8 >> 1;                              // head of this lane's B column
  float m_run = -INFINITY, l_run = 0.0f, zsum[2] = {0.0f, 0.0f};
  float acc[8][2];
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) { acc[mt][0] = 0.0f; acc[mt][1] = 0.0f; }

  for (int kt = warp; kt < CH / KT; kt += IM_WARPS) {
    const int64_t tile_t0 = t0 + (int64_t)kt * KT;
    if (tile_t0 >= n) break;
    uint4 X[4];
    const bool any_complete = tile_t0 + IM_G <= ncomp;
    if (any_complete) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) X[ks] = T.kc[(kt * 4 + ks) * 32 + lane];
    }
#pragma unroll
    for (int gl = 0; gl < GPT; ++gl) {
      const int64_t gt0 = tile_t0 + gl * IM_G;  // group's first token
      if (gt0 >= n) break;
      const int gi = kt * GPT + gl;            // group index within the chunk
      float z[4][2];
      if (gt0 + IM_G <= ncomp) {
        uint32_t b[4][2];
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint2 bb = *reinterpret_cast<const uint2 *>(&S.bfrag[gi][ks][lane][0]);
          b[ks][0] = bb.x;
          b[ks][1] = bb.y;
        }
        const float off = S.off[gi][tq];
        const float ks_h = S.kscale[gi][tq];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          const int k = gl * 4 + mt;
          const uint32_t msk = CM << (k * BITS);
          int C[4] = {0, 0, 0, 0};
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            imma(C, X[ks].x & msk, X[ks].y & msk, X[ks].z & msk, X[ks].w & msk, b[ks][0], b[ks][1]);
          const float sc = ks_h * __int_as_float((127 - k * BITS) << 23);  // * 2^-(k b)
          z[mt][0] = fmaf(fmaf((float)C[0], 256.0f, (float)C[1]), sc, off) * inv_sqrt_d;
          z[mt][1] = fmaf(fmaf((float)C[2], 256.0f, (float)C[3]), sc, off) * inv_sqrt_d;
        }
      } else {
        // the fp16 residual group (< g rows, quantizer.py:529-530): plain FMAs
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int tl = mt * 16 + g8 + 8 * r;
            const int64_t T = gt0 + tl;
            float a = -INFINITY;
            if (T < n) {
              const uint16_t *kr = kres + (size_t)(T - ncomp) * IM_D;
              a = 0.0f;
              for (int ch = 0; ch < IM_D; ch += 2) {
                const uint32_t pr = *reinterpret_cast<const uint32_t *>(kr + ch);
                a = fmaf(h2f(pr & 0xffff), S.q[tq][ch], a);
                a = fmaf(h2f(pr >> 16), S.q[tq][ch + 1], a);
              }
              a *= inv_sqrt_d;
            }
            z[mt][r] = a;
          }
      }
      // mask tokens beyond n (complete groups never straddle n)
      if (gt0 + IM_G > n) {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int r = 0; r < 2; ++r)
            if (gt0 + mt * 16 + g8 + 8 * r >= n) z[mt][r] = -INFINITY;
      }
      // ---- online softmax over this group (head tq) ----
      float gmax = -INFINITY;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) gmax = fmaxf(gmax, fmaxf(z[mt][0], z[mt][1]));
      gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, 4));
      gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, 8));
      gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, 16));
      const float m_new = fmaxf(m_run, gmax);
      const float alpha = __expf(m_run - m_new);
      m_run = m_new;
      float psum = 0.0f, zl0 = 0.0f, zl1 = 0.0f;
      const int tl0 = (int)(gt0 - t0);
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int tl = mt * 16 + g8 + 8 * r;
          const float p = __expf(z[mt][r] - m_new);
          S.p[warp][tq][tl] = p;
          psum += p;
          zl0 = fmaf(p, S.u.v.lov[0][tl0 + tl], zl0);
          zl1 = fmaf(p, S.u.v.lov[1][tl0 + tl], zl1);
        }
      l_run = fmaf(l_run, alpha, psum);
      zsum[0] = fmaf(zsum[0], alpha, zl0);
      zsum[1] = fmaf(zsum[1], alpha, zl1);
      __syncwarp();
      // ---- value MMA over the group's two 32-token k-steps ----
      // B[t, (h,digit)] = p[t,h] * s[t,cb] in a 16-bit fixed point scaled by
      // this group's max_t,cb p*s of head h (adaptive, exact integer MMA)
      float prod[2][2][8];  // [vtile][cb][token slot]
      float pmax = 0.0f;
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int tb = v * 32 + 4 * tq;
        const float4 p0 = *reinterpret_cast<const float4 *>(&S.p[warp][hB][tb]);
        const float4 p1 = *reinterpret_cast<const float4 *>(&S.p[warp][hB][tb + 16]);
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          const float4 s0 = *reinterpret_cast<const float4 *>(&S.u.v.sv[cb][tl0 + tb]);
          const float4 s1 = *reinterpret_cast<const float4 *>(&S.u.v.sv[cb][tl0 + tb + 16]);
          float *pr = prod[v][cb];
          pr[0] = p0.x * s0.x; pr[1] = p0.y * s0.y; pr[2] = p0.z * s0.z; pr[3] = p0.w * s0.w;
          pr[4] = p1.x * s1.x; pr[5] = p1.y * s1.y; pr[6] = p1.z * s1.z; pr[7] = p1.w * s1.w;
#pragma unroll
          for (int e = 0; e < 8; ++e) pmax = fmaxf(pmax, pr[e]);
        }
      }
      pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, 1));
      pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, 2));
      pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, 4));
      const float pinv = pmax > 0.0f ? __fdividef(IM_QMAX, pmax) : 0.0f;
      const float vsc_h = __shfl_sync(0xffffffffu, pmax, (2 * tq) * 4) * (1.0f / IM_QMAX);  // head tq's scale
      int V[8][4];
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) { V[mt][0] = 0; V[mt][1] = 0; V[mt][2] = 0; V[mt][3] = 0; }
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int vt = (int)((gt0 - t0) >> 5) + v;
        uint4 A[VS];
#pragma unroll
        for (int st = 0; st < VS; ++st) A[st] = T.vc[(vt * VS + st) * 32 + lane];
        uint32_t B[2][2];
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          const float *pr = prod[v][cb];
          B[cb][0] = pack_digits(fmaf(pr[0], pinv, IM_MAGIC), fmaf(pr[1], pinv, IM_MAGIC), fmaf(pr[2], pinv, IM_MAGIC),
                                 fmaf(pr[3], pinv, IM_MAGIC), dsel, 0, dxor);
          B[cb][1] = pack_digits(fmaf(pr[4], pinv, IM_MAGIC), fmaf(pr[5], pinv, IM_MAGIC), fmaf(pr[6], pinv, IM_MAGIC),
                                 fmaf(pr[7], pinv, IM_MAGIC), dsel, 0, dxor);
        }
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const int st = mt / SLOTS, slot = mt % SLOTS;
          const uint32_t msk = CM << (slot * BITS);
          const uint4 a = A[st];
          imma(V[mt], a.x & msk, a.y & msk, a.z & msk, a.w & msk, B[mt / 4][0], B[mt / 4][1]);
        }
      }
      // ---- flush the exact integer partials into the float accumulators ----
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        const int slot = mt % SLOTS;
        const float sc = vsc_h * __int_as_float((127 - slot * BITS) << 23);
        acc[mt][0] = fmaf(acc[mt][0], alpha, fmaf((float)V[mt][0], 256.0f, (float)V[mt][1]) * sc);
        acc[mt][1] = fmaf(acc[mt][1], alpha, fmaf((float)V[mt][2], 256.0f, (float)V[mt][3]) * sc);
      }
      __syncwarp();
    }
  }
  // ---- reduce the warp: l and z-sums over the 8 lanes sharing head tq ----
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    l_run += __shfl_xor_sync(0xffffffffu, l_run, o);
    zsum[0] += __shfl_xor_sync(0xffffffffu, zsum[0], o);
    zsum[1] += __shfl_xor_sync(0xffffffffu, zsum[1], o);
  }
  __syncthreads();  // the chunk's value params are no longer needed: reuse as warp partials
  float *wacc = &S.u.v.sv[0][0];  // [warps][4][128]
  if (g8 == 0) {
    S.wm[warp][tq] = m_run;
    S.wl[warp][tq] = l_run;
  }
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int r = 0; r < 2; ++r) wacc[(warp * 4 + tq) * IM_D + mt * 16 + g8 + 8 * r] = acc[mt][r] + zsum[mt >> 2];
  __syncthreads();
  for (int i = tid; i < G * IM_D; i += blockDim.x) {
    const int h = i / IM_D, ch = i % IM_D;
    float M = -INFINITY;
    for (int w = 0; w < IM_WARPS; ++w) M = fmaxf(M, S.wm[w][h]);
    float L = 0.0f, A = 0.0f;
    for (int w = 0; w < IM_WARPS; ++w) {
      if (S.wm[w][h] == -INFINITY) continue;
      const float sc = __expf(S.wm[w][h] - M);
      L = fmaf(sc, S.wl[w][h], L);
      A = fmaf(sc, wacc[(w * 4 + h) * IM_D + ch], A);
    }
    const size_t base = ((size_t)u * chunks + chunk) * G + h;
    pacc[base * IM_D + ch] = A;
    if (ch == 0) {
      pm[base] = M;
      pl[base] = L;
    }
  }
  if (!arrive) return;  // separate combine kernel
  // ---- the last CTA of this unit merges the chunk partials (fixed order) ----
  __shared__ bool last;
  __syncthreads();
  const int nvalid = (int)((n + CH - 1) / CH);
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&arrive[u], 1u);
    last = prev == (unsigned)nvalid - 1;
    if (last) arrive[u] = 0;  // re-armed for the next launch / graph replay
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const size_t b0 = (size_t)u * chunks * G;
  merge_partials(pm + b0, pl + b0, pacc + b0 * IM_D, G, IM_D, nvalid, out + (size_t)u * G * IM_D,
                 &S.u.v.sv[0][0]);
}

// ---------------------------------------------------------------------------
// Persistent, pipelined variant: one 512-thread CTA per SM and a contiguous
// token range (split) of one unit per CTA.  Chunks stream through a 6-stage
// TMA ring (24 KB each), so the HBM reads stay in flight while the warps
// compute; each warp owns one key tile of a chunk and does the whole group
// computation (key B fragments, softmax, value MMA) on its own, with no CTA
// prologue per chunk.  The last warp to finish a chunk refills its stage.
// The CTA's 16 warp partials are merged in shared memory; the splits are
// merged by the combine kernel.
// ---------------------------------------------------------------------------
constexpr int QP_WARPS = 16;  // (20 warps at 96 registers spill and run 5 % slower)
constexpr int QP_NS = 6;

struct QpStage {
  uint4 kc[IM_CHUNK];
  uint4 vc[IM_CHUNK];
  uint32_t klohi[IM_GROUPS * 128];
  uint32_t vlohi[IM_CHUNK * 2];
};

struct QpWarp {
  uint32_t bfrag[4][36][2];      // key B fragments of the current group (padded rows)
  float off[4], kscale[4];       // q_h . lo_g and the fixed-point scale per head
  float ps[2][4][IM_G + 8];      // p[t,h] * s[t,cb] of the current group
};

struct QpSmem {
  QpStage st[QP_NS];
  float q[4][IM_D];
  QpWarp w[QP_WARPS];
  unsigned long long full[QP_NS];
  int done[QP_NS];
  float wm[QP_WARPS][4], wl[QP_WARPS][4];
};

// logits of the fp16 residual group for this lane's 8 token slots (mt, r): z[mt * 2 + r]
__device__ __noinline__ void qp_residual_logits(const uint16_t *kres, const float *qh, int64_t gt0, int64_t ncomp,
                                                int64_t n, int g8, float *z) {
  const float inv_sqrt_d = 0.08838834764831845f;
  for (int mt = 0; mt < 4; ++mt)
    for (int r = 0; r < 2; ++r) {
      const int tl = mt * 16 + g8 + 8 * r;
      const int64_t Tt = gt0 + tl;
      float a = -INFINITY;
      if (Tt < n) {
        const uint16_t *kr = kres + (size_t)(Tt - ncomp) * IM_D;
        a = 0.0f;
#pragma unroll 4
        for (int ch = 0; ch < IM_D; ch += 2) {
          const uint32_t pr = *reinterpret_cast<const uint32_t *>(kr + ch);
          a = fmaf(h2f(pr & 0xffff), qh[ch], a);
          a = fmaf(h2f(pr >> 16), qh[ch + 1], a);
        }
        a *= inv_sqrt_d;
      }
      z[mt * 2 + r] = a;
    }
}

template <int BITS>
__global__ void __launch_bounds__(QP_WARPS * 32, 1)
    quant_decode_pipe_kernel(QC c, const uint16_t *__restrict__ queries, int G, float *__restrict__ pm,
                             float *__restrict__ pl, float *__restrict__ pacc, int splits,
                             unsigned *__restrict__ arrive, float *__restrict__ out) {
  constexpr int CH = IM_CHUNK / BITS;  // tokens per chunk (16 KB of codes)
  constexpr int KT = 128 / BITS;       // key tile tokens
  constexpr int GPT = KT / IM_G;       // groups per key tile
  constexpr int TPC = CH / KT;         // tiles per chunk (4)
  constexpr int NWG = QP_WARPS / TPC;  // warp groups, each consuming whole chunks
  constexpr int VS = BITS;
  constexpr int SLOTS = 8 / BITS;
  constexpr uint32_t CM = BITS == 1 ? 0x01010101u : 0x03030303u;
  constexpr float KINV = 1.0f / (float)((1 << BITS) - 1);
  extern __shared__ __align__(128) unsigned char smraw[];
  QpSmem &S = *reinterpret_cast<QpSmem *>(smraw);
  const int u = blockIdx.y, split = blockIdx.x;
  // query heads [h0, h0 + Gb) of the unit: blocks of 4 (the MMA's N = 4 heads x 2 digits);
  // G > 4 runs ceil(G/4) head blocks whose CTAs stream the same codes (L2 serves the repeats)
  const int h0 = 4 * blockIdx.z, Gb = min(4, G - h0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g8 = lane >> 2, tq = lane & 3;
  const int64_t n = *c.len;
  const int64_t cap = c.capacity;
  const int64_t nch = (n + CH - 1) / CH;
  const int64_t cps = (nch + splits - 1) / splits;
  const int64_t cb = (int64_t)split * cps;
  const int cnt = (int)(cb < nch ? imin64(cps, nch - cb) : 0);
  if (tid == 0) {
    for (int s = 0; s < QP_NS; ++s) {
      mbar_init(reinterpret_cast<uint64_t *>(&S.full[s]), 1);
      S.done[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // one thread: chunk j of this split into stage j % QP_NS
  auto load = [&](int j) {
    const int s = j % QP_NS;
    QpStage &T = S.st[s];
    uint64_t *bar = reinterpret_cast<uint64_t *>(&S.full[s]);
    const int64_t t0 = (cb + j) * CH;
    const int64_t g0c = t0 / IM_G, kt0 = t0 / KT, vt0 = t0 / 32;
    const uint32_t kl_bytes = (uint32_t)(imin64(CH / IM_G, cap / IM_G - g0c) * IM_D * 4);
    const uint32_t vl_bytes = (uint32_t)(imin64(CH, cap - t0) * 8);
    const uint32_t kc_bytes = (uint32_t)(imin64(CH / KT, cap / KT - kt0) * 2048);
    const uint32_t vc_bytes = (uint32_t)(imin64(CH / 32, cap / 32 - vt0) * VS * 512);
    mbar_expect_tx(bar, kl_bytes + vl_bytes + kc_bytes + vc_bytes);
    bulk_g2s(T.kc, c.key_codes + ((size_t)u * (cap / KT) + kt0) * 512, kc_bytes, bar);
    bulk_g2s(T.vc, c.val_codes + ((size_t)u * (cap / 32) + vt0) * VS * 128, vc_bytes, bar);
    bulk_g2s(T.klohi, c.key_lohi + ((size_t)u * (cap / IM_G) + g0c) * IM_D, kl_bytes, bar);
    bulk_g2s(T.vlohi, c.val_lohi + ((size_t)u * cap + t0) * 2, vl_bytes, bar);
  };
  if (tid == 0)
    for (int j = 0; j < cnt && j < QP_NS; ++j) load(j);
  for (int i = tid; i < 4 * IM_D; i += blockDim.x) {
    const int h = i / IM_D;
    S.q[h][i % IM_D] = h < Gb ? h2f(queries[((size_t)u * G + h0 + h) * IM_D + i % IM_D]) : 0.0f;
  }
  __syncthreads();

  const int64_t ncomp = (n / IM_G) * IM_G;
  const float inv_sqrt_d = 0.08838834764831845f;  // 1/sqrt(128)
  QpWarp &Wp = S.w[warp];
  const uint16_t *kres = c.key_resid + (size_t)u * IM_G * IM_D;
  const uint32_t dsel = (g8 & 1) ? 0x0040u : 0x0051u;  // this lane's B column digit
  const uint32_t dxor = (g8 & 1) ? 0x80808080u : 0u;
  const int hB = g8 >> 1;                              // head of this lane's B column
  // this lane's channel quad in the B-fragment layout (ks, j, tq)
  const int fq = lane & 3, fj = (lane >> 2) & 1, fks = lane >> 3;
  const int fch = 32 * fks + 16 * fj + 4 * fq;
  const bool b4 = lane & 16, b3 = lane & 8;
  float m_run = -INFINITY, l_run = 0.0f, zsum[2] = {0.0f, 0.0f};
  float acc[8][2];
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    acc[mt][0] = 0.0f;
    acc[mt][1] = 0.0f;
  }
  const int wg = warp / TPC, tw = warp % TPC;
  for (int j = wg; j < cnt; j += NWG) {
    const int s = j % QP_NS;
    QpStage &T = S.st[s];
    mbar_wait(reinterpret_cast<uint64_t *>(&S.full[s]), (uint32_t)((j / QP_NS) & 1));
    const int64_t t0 = (cb + j) * CH;
    const int64_t tile_t0 = t0 + (int64_t)tw * KT;
    if (tile_t0 < n) {
      uint4 X[4];
      if (tile_t0 + IM_G <= ncomp) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) X[ks] = T.kc[(tw * 4 + ks) * 32 + lane];
      }
#pragma unroll 1  // one group's code (~12 KB of SASS) per iteration: the loop body stays in the I-cache
      for (int gl = 0; gl < GPT; ++gl) {
        const int64_t gt0 = tile_t0 + gl * IM_G;  // group's first token
        if (gt0 >= n) break;
        const int gi = tw * GPT + gl;            // group index within the chunk
        const int tl0 = (int)(gt0 - t0);
        float z[4][2];
        if (gt0 + IM_G <= ncomp) {
          // ---- this group's key B fragments: W = q s as two s8 digits, offsets q . lo ----
          {
            float lo[4], sc[4];
            const uint4 raw = *reinterpret_cast<const uint4 *>(&T.klohi[gi * IM_D + fch]);
            const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __half22float2(*reinterpret_cast<const __half2 *>(&w[i]));  // (lo, hi)
              lo[i] = f.x;
              sc[i] = (f.y - lo[i]) * KINV;  // 0 for degenerate groups (all codes 0)
            }
            float W[4][4], dt[4], mx[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float4 qh = *reinterpret_cast<const float4 *>(&S.q[h][fch]);
              const float qa[4] = {qh.x, qh.y, qh.z, qh.w};
              dt[h] = 0.0f;
              mx[h] = 0.0f;
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                W[h][i] = qa[i] * sc[i];
                dt[h] = fmaf(qa[i], lo[i], dt[h]);
                mx[h] = fmaxf(mx[h], fabsf(W[h][i]));
              }
            }
            float d2[2], m2[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const float sd = b4 ? dt[k] : dt[k + 2], sm = b4 ? mx[k] : mx[k + 2];
              const float rd = __shfl_xor_sync(0xffffffffu, sd, 16), rm = __shfl_xor_sync(0xffffffffu, sm, 16);
              d2[k] = (b4 ? dt[k + 2] : dt[k]) + rd;
              m2[k] = fmaxf(b4 ? mx[k + 2] : mx[k], rm);
            }
            float d1, m1;
            {
              const float sd = b3 ? d2[0] : d2[1], sm = b3 ? m2[0] : m2[1];
              const float rd = __shfl_xor_sync(0xffffffffu, sd, 8), rm = __shfl_xor_sync(0xffffffffu, sm, 8);
              d1 = (b3 ? d2[1] : d2[0]) + rd;
              m1 = fmaxf(b3 ? m2[1] : m2[0], rm);
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
              d1 += __shfl_xor_sync(0xffffffffu, d1, o);
              m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
            }
            if ((lane & 7) == 0) {
              const int h = (b4 ? 2 : 0) + (b3 ? 1 : 0);
              Wp.off[h] = d1;
              Wp.kscale[h] = m1 * (1.0f / IM_QMAX);
            }
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const float mh = __shfl_sync(0xffffffffu, m1, 8 * h);
              const float inv = mh > 0.0f ? __fdividef(IM_QMAX, mh) : 0.0f;
              const float x0 = fmaf(W[h][0], inv, IM_MAGIC), x1 = fmaf(W[h][1], inv, IM_MAGIC);
              const float x2 = fmaf(W[h][2], inv, IM_MAGIC), x3 = fmaf(W[h][3], inv, IM_MAGIC);
              Wp.bfrag[fks][(2 * h) * 4 + fq][fj] = pack_digits(x0, x1, x2, x3, 0x0051, 0, 0u);
              Wp.bfrag[fks][(2 * h + 1) * 4 + fq][fj] = pack_digits(x0, x1, x2, x3, 0x0040, 0, 0x80808080u);
            }
          }
          __syncwarp();
          uint32_t b[4][2];
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint2 bb = *reinterpret_cast<const uint2 *>(&Wp.bfrag[ks][lane][0]);
            b[ks][0] = bb.x;
            b[ks][1] = bb.y;
          }
          const float off = Wp.off[tq];
          const float ks_h = Wp.kscale[tq];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            const int k = gl * 4 + mt;
            const uint32_t msk = CM << (k * BITS);
            int Cc[4] = {0, 0, 0, 0};
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              imma(Cc, X[ks].x & msk, X[ks].y & msk, X[ks].z & msk, X[ks].w & msk, b[ks][0], b[ks][1]);
            const float sc = ks_h * __int_as_float((127 - k * BITS) << 23);  // * 2^-(k b)
            z[mt][0] = fmaf(fmaf((float)Cc[0], 256.0f, (float)Cc[1]), sc, off) * inv_sqrt_d;
            z[mt][1] = fmaf(fmaf((float)Cc[2], 256.0f, (float)Cc[3]), sc, off) * inv_sqrt_d;
          }
        } else {
          // the fp16 residual group (< g rows, quantizer.py:529-530): plain FMAs, out of line
          // (at most one group per launch; its code must not sit in the hot loop)
          qp_residual_logits(kres, &S.q[tq][0], gt0, ncomp, n, g8, &z[0][0]);
        }
        if (gt0 + IM_G > n) {  // mask tokens beyond n (complete groups never straddle n)
#pragma unroll
          for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int r = 0; r < 2; ++r)
              if (gt0 + mt * 16 + g8 + 8 * r >= n) z[mt][r] = -INFINITY;
        }
        // ---- online softmax over this group (head tq); p * s per value channel block ----
        float gmax = -INFINITY;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) gmax = fmaxf(gmax, fmaxf(z[mt][0], z[mt][1]));
        gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, 4));
        gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, 8));
        gmax = fmaxf(gmax, __shfl_xor_sync(0xffffffffu, gmax, 16));
        const float m_new = fmaxf(m_run, gmax);
        const float alpha = __expf(m_run - m_new);
        m_run = m_new;
        float psum = 0.0f, zl0 = 0.0f, zl1 = 0.0f;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const int tl = mt * 16 + g8 + 8 * r;
            const float p = __expf(z[mt][r] - m_new);
            float l0 = 0.0f, l1 = 0.0f, s0 = 0.0f, s1 = 0.0f;
            if (gt0 + tl < n) {
              const uint2 w = *reinterpret_cast<const uint2 *>(&T.vlohi[2 * (tl0 + tl)]);
              const float2 f0 = __half22float2(*reinterpret_cast<const __half2 *>(&w.x));  // (lo, hi)
              const float2 f1 = __half22float2(*reinterpret_cast<const __half2 *>(&w.y));
              l0 = f0.x;
              l1 = f1.x;
              s0 = (f0.y - l0) * KINV;
              s1 = (f1.y - l1) * KINV;
            }
            Wp.ps[0][tq][tl] = p * s0;
            Wp.ps[1][tq][tl] = p * s1;
            psum += p;
            zl0 = fmaf(p, l0, zl0);
            zl1 = fmaf(p, l1, zl1);
          }
        l_run = fmaf(l_run, alpha, psum);
        zsum[0] = fmaf(zsum[0], alpha, zl0);
        zsum[1] = fmaf(zsum[1], alpha, zl1);
        __syncwarp();
        // ---- value MMA over the group's two 32-token k-steps (see the kernel above) ----
        float prod[2][2][8];  // [vtile][cb][token slot]
        float pmax = 0.0f;
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int tb = v * 32 + 4 * tq;
#pragma unroll
          for (int cbk = 0; cbk < 2; ++cbk) {
            const float4 a0 = *reinterpret_cast<const float4 *>(&Wp.ps[cbk][hB][tb]);
            const float4 a1 = *reinterpret_cast<const float4 *>(&Wp.ps[cbk][hB][tb + 16]);
            float *pr = prod[v][cbk];
            pr[0] = a0.x; pr[1] = a0.y; pr[2] = a0.z; pr[3] = a0.w;
            pr[4] = a1.x; pr[5] = a1.y; pr[6] = a1.z; pr[7] = a1.w;
#pragma unroll
            for (int e = 0; e < 8; ++e) pmax = fmaxf(pmax, pr[e]);
          }
        }
        pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, 1));
        pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, 2));
        pmax = fmaxf(pmax, __shfl_xor_sync(0xffffffffu, pmax, 4));
        const float pinv = pmax > 0.0f ? __fdividef(IM_QMAX, pmax) : 0.0f;
        const float vsc_h = __shfl_sync(0xffffffffu, pmax, (2 * tq) * 4) * (1.0f / IM_QMAX);  // head tq's scale
        int V[8][4];
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          V[mt][0] = 0; V[mt][1] = 0; V[mt][2] = 0; V[mt][3] = 0;
        }
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int vt = (tl0 >> 5) + v;
          uint4 A[VS];
#pragma unroll
          for (int st = 0; st < VS; ++st) A[st] = T.vc[(vt * VS + st) * 32 + lane];
          uint32_t B[2][2];
#pragma unroll
          for (int cbk = 0; cbk < 2; ++cbk) {
            const float *pr = prod[v][cbk];
            B[cbk][0] = pack_digits(fmaf(pr[0], pinv, IM_MAGIC), fmaf(pr[1], pinv, IM_MAGIC),
                                    fmaf(pr[2], pinv, IM_MAGIC), fmaf(pr[3], pinv, IM_MAGIC), dsel, 0, dxor);
            B[cbk][1] = pack_digits(fmaf(pr[4], pinv, IM_MAGIC), fmaf(pr[5], pinv, IM_MAGIC),
                                    fmaf(pr[6], pinv, IM_MAGIC), fmaf(pr[7], pinv, IM_MAGIC), dsel, 0, dxor);
          }
#pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            const int st = mt / SLOTS, slot = mt % SLOTS;
            const uint32_t msk = CM << (slot * BITS);
            const uint4 a = A[st];
            imma(V[mt], a.x & msk, a.y & msk, a.z & msk, a.w & msk, B[mt / 4][0], B[mt / 4][1]);
          }
        }
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const int slot = mt % SLOTS;
          const float sc = vsc_h * __int_as_float((127 - slot * BITS) << 23);
          acc[mt][0] = fmaf(acc[mt][0], alpha, fmaf((float)V[mt][0], 256.0f, (float)V[mt][1]) * sc);
          acc[mt][1] = fmaf(acc[mt][1], alpha, fmaf((float)V[mt][2], 256.0f, (float)V[mt][3]) * sc);
        }
        __syncwarp();
      }
    }
    // ---- release the stage; the last of its TPC warps refills it ----
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      const int d = atomicAdd(&S.done[s], 1);
      if (d == TPC - 1) {
        __threadfence_block();
        S.done[s] = 0;
        if (j + QP_NS < cnt) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // our reads before the TMA writes
          load(j + QP_NS);
        }
      }
    }
  }
  // ---- merge the 16 warp partials (fixed order) into this split's partial ----
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    l_run += __shfl_xor_sync(0xffffffffu, l_run, o);
    zsum[0] += __shfl_xor_sync(0xffffffffu, zsum[0], o);
    zsum[1] += __shfl_xor_sync(0xffffffffu, zsum[1], o);
  }
  __syncthreads();  // every stage is consumed: its memory holds the warp partials now
  float *wacc = reinterpret_cast<float *>(&S.st[0]);  // [warps][4][128]
  if (g8 == 0) {
    S.wm[warp][tq] = m_run;
    S.wl[warp][tq] = l_run;
  }
#pragma unroll
  for (int mt = 0; mt < 8; ++mt)
#pragma unroll
    for (int r = 0; r < 2; ++r) wacc[(warp * 4 + tq) * IM_D + mt * 16 + g8 + 8 * r] = acc[mt][r] + zsum[mt >> 2];
  __syncthreads();
  for (int i = tid; i < Gb * IM_D; i += blockDim.x) {
    const int h = i / IM_D, ch = i % IM_D;
    float M = -INFINITY;
    for (int w = 0; w < QP_WARPS; ++w) M = fmaxf(M, S.wm[w][h]);
    float L = 0.0f, A = 0.0f;
    for (int w = 0; w < QP_WARPS; ++w) {
      if (S.wm[w][h] == -INFINITY) continue;
      const float sc = __expf(S.wm[w][h] - M);
      L = fmaf(sc, S.wl[w][h], L);
      A = fmaf(sc, wacc[(w * 4 + h) * IM_D + ch], A);
    }
    const size_t base = ((size_t)u * splits + split) * G + h0 + h;
    pacc[base * IM_D + ch] = A;
    if (ch == 0) {
      pm[base] = M;
      pl[base] = L;
    }
  }
  // ---- the last CTA of the unit (over splits x head blocks) merges the split partials
  // in a fixed order (no separate combine launch) ----
  __shared__ bool last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&arrive[u], 1u);
    last = prev == gridDim.x * gridDim.z - 1;
    if (last) arrive[u] = 0;  // re-armed for the next launch / graph replay
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const size_t b0 = (size_t)u * splits * G;
  merge_partials(pm + b0, pl + b0, pacc + b0 * IM_D, G, IM_D, splits, out + (size_t)u * G * IM_D,
                 reinterpret_cast<float *>(&S.st[0]) + QP_WARPS * 4 * IM_D);
}

static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int quant_decode_pipe(const QC &c, const uint16_t *q, int G, float *out, void *ws, cudaStream_t st) {
  const int CH = IM_CHUNK / c.bits;
  const int max_chunks = (int)((c.capacity + CH - 1) / CH);
  const int hblocks = (G + 3) / 4;
  const int splits = std::max(1, std::min(max_chunks, sm_count() / std::max(1, c.units * hblocks)));
  float *pm = reinterpret_cast<float *>(ws);
  float *pl = pm + (size_t)c.units * splits * G;
  float *pacc = pl + (size_t)c.units * splits * G;
  const size_t sm = sizeof(QpSmem);
  // per-unit arrival counters after the partials (quant_decode_workspace)
  unsigned *arrive = reinterpret_cast<unsigned *>(reinterpret_cast<char *>(ws) + quant_decode_arrive_offset(c, G));
  dim3 grid(splits, c.units, hblocks);
  if (c.bits == 1) {
    cudaFuncSetAttribute(quant_decode_pipe_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_prio(quant_decode_pipe_kernel<1>, grid, dim3(QP_WARPS * 32), sm, st, true, c, q, G, pm, pl, pacc, splits,
                arrive, out);
  } else {
    cudaFuncSetAttribute(quant_decode_pipe_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_prio(quant_decode_pipe_kernel<2>, grid, dim3(QP_WARPS * 32), sm, st, true, c, q, G, pm, pl, pacc, splits,
                arrive, out);
  }
  return check_launch("tkv_quant_decode(imma pipe)");
}

int quant_decode_imma(const QC &c, const uint16_t *q, int G, float *out, void *ws, cudaStream_t st) {
  const int CH = IM_CHUNK / c.bits;
  const int chunks = (int)((c.capacity + CH - 1) / CH);
  float *pm = reinterpret_cast<float *>(ws);
  float *pl = pm + (size_t)c.units * chunks * G;
  float *pacc = pl + (size_t)c.units * chunks * G;
  const size_t sm = ((sizeof(ImSmem) + 127) & ~size_t(127)) + sizeof(ImStage);
  dim3 grid(chunks, c.units);
  // fused last-CTA merge when the partials fit the merge buffer, else a combine kernel
  // measured: one CTA merging 128 chunk partials is slower than the parallel
  // combine kernel, so the fused merge stays off for the quantized decode
  const bool fused = false;
  // arrival counters live at the fixed tail of the workspace (the SIMT kernel
  // uses more partial space, so both implementations can share one workspace)
  unsigned *arrive =
      fused ? reinterpret_cast<unsigned *>(reinterpret_cast<char *>(ws) + quant_decode_arrive_offset(c, G)) : nullptr;
  if (c.bits == 1) {
    cudaFuncSetAttribute(quant_decode_imma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_prio(quant_decode_imma_kernel<1>, grid, dim3(IM_WARPS * 32), sm, st, true, c, q, G, pm, pl, pacc, chunks, arrive, out);
  } else {
    cudaFuncSetAttribute(quant_decode_imma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_prio(quant_decode_imma_kernel<2>, grid, dim3(IM_WARPS * 32), sm, st, true, c, q, G, pm, pl, pacc, chunks, arrive, out);
  }
  if (!fused) launch_combine_scalar(pm, pl, pacc, c.units, chunks, G, c.d, c.len, CH, out, st);
  return check_launch("tkv_quant_decode(imma)");
}

}  // namespace tkv
