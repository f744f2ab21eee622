// Shared helpers for the TailorKV sm_100a kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "tailorkv.h"

namespace tkv {

// ---- error plumbing (thread-local message, status codes from tailorkv.h) ----
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int check_launch(const char *what);

#define TKV_REQUIRE(cond, code, msg)            \
  do {                                          \
    if (!(cond)) return ::tkv::fail((code), (msg)); \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// ---- launch priorities ----
// The decode chain (attention kernels, appends) launches at the device's
// greatest priority and stage 1 of the next layer (side stream) at the least,
// so when both become ready together the CTA scheduler places the chain's
// kernels first and stage 1 fills the remaining SMs.  Captured graphs keep
// these as node priorities (instantiated with UseNodePriority, abi.cu).
inline int launch_priority(bool high) {
  static int lo = 1, hi = 1;
  if (lo == 1) {
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) lo = hi = 0;
  }
  return high ? hi : lo;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_prio(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                               bool high, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributePriority;
  at[0].val.priority = launch_priority(high);
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- numeric helpers ----
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ float h2f(uint16_t h) { return __half2float(__ushort_as_half(h)); }
__device__ __forceinline__ double h2d(uint16_t h) { return (double)__half2float(__ushort_as_half(h)); }
// Exact fp16 -> float64 by bit manipulation (integer pipe, no F2F.F64):
// normal numbers rebias the exponent (15 -> 1023); zero/subnormals are
// man * 2^-24 (finite inputs only).
__device__ __forceinline__ double h2d_fast(uint32_t h) {
  const uint32_t e = (h >> 10) & 0x1fu, man = h & 0x3ffu;
  const uint32_t sign = (h & 0x8000u) << 16;
  const double nrm = __hiloint2double((int)(sign | ((e + 1008u) << 20) | (man << 10)), 0);
  const double sub = __hiloint2double((int)(sign | 0x3e700000u), 0) * (double)man;  // +-2^-24 * man
  return e ? nrm : sub;
}

// float64 -> fp16 bits, round to nearest even (numpy's astype(float16) of a
// float64); written out because __double2half is not a direct conversion.
__device__ __forceinline__ uint16_t f64_to_f16_bits(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  const uint16_t sign = (uint16_t)((b >> 48) & 0x8000u);
  const int ex = (int)((b >> 52) & 0x7ff);
  if (ex == 0x7ff) return sign | ((b & 0xfffffffffffffull) ? 0x7e00u : 0x7c00u);
  const double a = fabs(x);
  if (a < 6.103515625e-05) {  // below 2^-14: subnormal grid of 2^-24
    const double q = rint(a * 16777216.0);
    return sign | (uint16_t)q;  // q == 1024 is the smallest normal
  }
  int e = ex - 1023;
  double q = rint(ldexp(a, 10 - e));  // in [1024, 2048]
  if (q >= 2048.0) { q = 1024.0; ++e; }
  if (e > 15) return sign | 0x7c00u;
  return sign | (uint16_t)(((e + 15) << 10) | ((int)q - 1024));
}

__device__ __forceinline__ uint32_t pack_lohi(uint16_t lo, uint16_t hi) {
  return (uint32_t)lo | ((uint32_t)hi << 16);
}

// Order-preserving map of an IEEE double onto uint64 (larger double -> larger key).
// -0.0 and +0.0 compare equal in the reference (numpy lexsort); map both to +0.
__device__ __forceinline__ uint64_t orderable(double x) {
  if (x == 0.0) x = 0.0;
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---- TMA 1-D bulk copies into shared memory, completion on an mbarrier ----
__device__ __forceinline__ uint32_t sm_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sm_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sm_addr(dst)),
      "l"(src), "r"(bytes), "r"(sm_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @p bra.uni DONE_%=;\n"
      " bra.uni WAIT_%=;\n DONE_%=:\n}\n" ::"r"(sm_addr(bar)),
      "r"(phase)
      : "memory");
}

// ---- quantization codec, bit-exact with quantizer.py:66-117 ----
// Codes are computed in float64 exactly as the reference (inputs are fp16,
// so x-lo, hi-lo, hi+lo are exact in float64).
//   b=1: code = [hi != lo] && 2x >= hi + lo           (DESIGN.md 3.2 proof)
//   b=2: fp32 fast path, float64 replay of the reference when the fp32
//        value lies within 1e-5 of a rounding boundary.
__device__ __forceinline__ uint32_t encode_code(float xf, float lof, float hif, int bits) {
  if (hif == lof) return 0u;  // degenerate group: scale 1, code 0 (quantizer.py:94-95)
  if (bits == 1) {
    double x2 = 2.0 * (double)xf;
    double s = __dadd_rn((double)hif, (double)lof);
    return x2 >= s ? 1u : 0u;
  }
  // bits == 2
  float a = xf - lof;          // relative error <= 2^-24
  float s = (hif - lof) / 3.0f;
  float v = a / s + 0.5f;
  float fl = floorf(v);
  float fr = v - fl;
  if (fr > 1e-5f && fr < 1.0f - 1e-5f) {
    int r = (int)fl;
    return (uint32_t)min(max(r, 0), 3);
  }
  double sd = __ddiv_rn(__dsub_rn((double)hif, (double)lof), 3.0);
  double vd = __ddiv_rn(__dsub_rn((double)xf, (double)lof), sd);
  double r = floor(__dadd_rn(fabs(vd), 0.5));
  if (vd < 0) r = -r;
  int ri = (int)r;
  return (uint32_t)min(max(ri, 0), 3);
}

__device__ __forceinline__ void atomic_max_pos(float *addr, float v) {
  atomicMax(reinterpret_cast<int *>(addr), __float_as_int(v));  // v >= 0
}

// Group scale as used by decode: (hi-lo)/(2^b-1), 1 when degenerate.
__device__ __forceinline__ float group_scale_f(float lo, float hi, int bits) {
  float s = (hi - lo) / (float)((1 << bits) - 1);
  return s == 0.0f ? 1.0f : s;
}

// ---- native (MMA fragment) layouts; DESIGN.md section 3 ----
// Key tile = 16 * (8/bits) tokens.  Word (tile, ks, lane, role) holds, in byte
// i at bits [k*b, k*b+b), the code of token 16k + (lane>>2) + 8(role&1) and
// channel 32ks + 4(lane&3) + i + 16(role>>1).
__host__ __device__ __forceinline__ int key_tile_tokens(int bits) { return 16 * (8 / bits); }

__device__ __forceinline__ void key_code_pos(int64_t t, int c, int d, int bits, int64_t *word, int *bit) {
  const int Tk = key_tile_tokens(bits);
  const int64_t tile = t / Tk;
  const int tt = (int)(t % Tk);
  const int k = tt >> 4, row = tt & 15;
  const int g8 = row & 7, rlo = row >> 3;
  const int ks = c >> 5, cc = c & 31;
  const int rhi = cc >> 4, c16 = cc & 15;
  const int tq = c16 >> 2, i = c16 & 3;
  const int lane = g8 * 4 + tq, role = rhi * 2 + rlo;
  *word = ((tile * (d >> 5) + ks) * 32 + lane) * 4 + role;
  *bit = 8 * i + k * bits;
}

// Value tile = 32 tokens.  sets = ceil(d / (16*8/bits)).  Word (vtile, set,
// lane, role) holds in byte i at bits [k*b, k*b+b) the code of token
// 32*vtile + 4(lane&3) + i + 16(role>>1) and channel
// set*16*(8/b) + 16k + (lane>>2) + 8(role&1).
__host__ __device__ __forceinline__ int val_sets(int d, int bits) {
  const int per = 16 * (8 / bits);
  return (d + per - 1) / per;
}

__device__ __forceinline__ void val_code_pos(int64_t t, int c, int d, int bits, int64_t *word, int *bit) {
  const int per = 16 * (8 / bits);
  const int64_t vt = t >> 5;
  const int tt = (int)(t & 31);
  const int rhi = tt >> 4, t16 = tt & 15;
  const int tq = t16 >> 2, i = t16 & 3;
  const int set = c / per, cs = c % per;
  const int k = cs >> 4, row = cs & 15;
  const int g8 = row & 7, rlo = row >> 3;
  const int lane = g8 * 4 + tq, role = rhi * 2 + rlo;
  *word = ((vt * val_sets(d, bits) + set) * 32 + lane) * 4 + role;
  *bit = 8 * i + k * bits;
}

// Merge split-K softmax partials of one unit, executed by one whole CTA
// (the last to finish): m/l [chunk][G], acc [chunk][G][d].  sm must hold
// 2*G*nvalid floats (G*nvalid <= 1024).  Fixed summation order.
__device__ __forceinline__ void merge_partials(const float *pm, const float *pl, const float *pacc, int G, int d,
                                               int nvalid, float *out, float *sm) {
  float *sc = sm, *ll = sm + G * nvalid;
  for (int i = threadIdx.x; i < G * nvalid; i += blockDim.x) {
    sc[i] = __ldcg(&pm[i]);  // i = ci*G + h
    ll[i] = __ldcg(&pl[i]);
  }
  __syncthreads();
  // one warp per head: the maximum, the rescale factors and the sum over the partials (lane-strided,
  // then a fixed butterfly: the summation order is deterministic)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int h = warp; h < G; h += nw) {
    float M = -INFINITY;
    for (int ci = lane; ci < nvalid; ci += 32) M = fmaxf(M, sc[ci * G + h]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = 0.0f;
    for (int ci = lane; ci < nvalid; ci += 32) {
      const float m = sc[ci * G + h];
      const float e = m == -INFINITY ? 0.0f : __expf(m - M);
      L = fmaf(e, ll[ci * G + h], L);
      sc[ci * G + h] = e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    __syncwarp();
    if (lane == 0) ll[h] = L;  // (slot h of chunk 0: its lane has consumed it above)
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * d; i += blockDim.x) {
    const int h = i / d, c = i % d;
    float A = 0.0f;
    for (int c0 = 0; c0 < nvalid; c0 += 16) {  // 16 partials in flight per thread
      float v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = c0 + j < nvalid ? __ldcg(&pacc[((size_t)(c0 + j) * G + h) * d + c]) : 0.0f;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j < nvalid) A = fmaf(sc[(c0 + j) * G + h], v[j], A);
    }
    out[(size_t)h * d + c] = A / ll[h];
  }
}

}  // namespace tkv
