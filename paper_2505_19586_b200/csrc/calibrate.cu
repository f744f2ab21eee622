// Offline layer classification on the GPU (identifier.py:89-187):
// dense preference score = mean over probe queries of
//   1 - (sum of the k largest softmax(K q / sqrt d) weights).
#include <cmath>

#include "common.cuh"
#include "sparse.cuh"

namespace tkv {

constexpr int CAL_NQ_MAX = 64;

// z[qh][p][j] = K[kvh(qh)][j] . q[qh][p] / sqrt(d); one thread per key row.
__global__ void __launch_bounds__(256) cal_logits_kernel(const uint16_t *__restrict__ queries,
                                                          const uint16_t *__restrict__ keys, int hq, int h, int n_q,
                                                          int64_t n, int d, float *__restrict__ z) {
  extern __shared__ float qs[];  // [n_q][d]
  const int qh = blockIdx.y;
  const int kvh = qh / (hq / h);  // kv_model.py:71-73
  for (int i = threadIdx.x; i < n_q * d; i += blockDim.x) qs[i] = h2f(queries[(size_t)qh * n_q * d + i]);
  __syncthreads();
  const float inv = 1.0f / sqrtf((float)d);
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const uint16_t *kr = keys + ((size_t)kvh * n + j) * d;
  float acc[CAL_NQ_MAX];
#pragma unroll
  for (int p = 0; p < CAL_NQ_MAX; ++p) acc[p] = 0.0f;
  for (int c = 0; c < d; c += 2) {
    const uint32_t pr = *reinterpret_cast<const uint32_t *>(kr + c);
    const float k0 = h2f(pr & 0xffff), k1 = h2f(pr >> 16);
#pragma unroll
    for (int p = 0; p < CAL_NQ_MAX; ++p) {
      if (p < n_q) acc[p] = fmaf(k1, qs[p * d + c + 1], fmaf(k0, qs[p * d + c], acc[p]));
    }
  }
#pragma unroll
  for (int p = 0; p < CAL_NQ_MAX; ++p)
    if (p < n_q) z[((size_t)qh * n_q + p) * n + j] = acc[p] * inv;
}

__device__ __forceinline__ uint32_t ford(float x) {
  if (x == 0.0f) x = 0.0f;
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

template <typename T>
__device__ T block_reduce_sum(T v, T *sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) sh[w] = v;
  __syncthreads();
  T r = 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += sh[i];
    sh[32] = r;
  }
  __syncthreads();
  r = sh[32];
  __syncthreads();
  return r;
}

// One CTA per (qh, probe) row: max, sum of exp, k-th largest by radix select,
// then the top-k mass (ties at the threshold counted exactly k times).
__global__ void __launch_bounds__(1024) cal_row_kernel(const float *__restrict__ z, int64_t n, int64_t k,
                                                        double *__restrict__ err) {
  __shared__ double dsh[33];
  __shared__ float fsh[33];
  __shared__ uint32_t hist[256];
  __shared__ uint32_t prefix, pmask;
  __shared__ int64_t need;
  const float *row = z + (size_t)blockIdx.x * n;
  float m = -INFINITY;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) m = fmaxf(m, row[j]);
  // block max
  {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    m = warp_max(m);
    if (lane == 0) fsh[w] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      float r = -INFINITY;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmaxf(r, fsh[i]);
      fsh[32] = r;
    }
    __syncthreads();
    m = fsh[32];
    __syncthreads();
  }
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) s += exp((double)row[j] - (double)m);
  s = block_reduce_sum<double>(s, dsh);
  if (threadIdx.x == 0) { prefix = 0; pmask = 0; need = k; }
  __syncthreads();
  for (int lvl = 0; lvl < 4; ++lvl) {
    const int shift = 24 - 8 * lvl;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const uint32_t pf = prefix, pmk = pmask;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const uint32_t key = ford(row[j]);
      if ((key & pmk) == pf) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t cum = 0;
      int D = 0;
      for (int dg = 255; dg >= 0; --dg) {
        if (cum + (int64_t)hist[dg] >= need) { D = dg; break; }
        cum += hist[dg];
      }
      need -= cum;
      prefix = pf | ((uint32_t)D << shift);
      pmask = pmk | (255u << shift);
    }
    __syncthreads();
  }
  const uint32_t T = prefix;
  double kept = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const float x = row[j];
    if (ford(x) > T) kept += exp((double)x - (double)m);
  }
  kept = block_reduce_sum<double>(kept, dsh);
  if (threadIdx.x == 0) {
    // the threshold value itself: decode T back to a float
    const uint32_t b = (T & 0x80000000u) ? (T & 0x7fffffffu) : ~T;
    const float tv = __uint_as_float(b);
    kept += (double)need * exp((double)tv - (double)m);
    err[blockIdx.x] = 1.0 - kept / s;
  }
}

__global__ void cal_mean_kernel(const double *__restrict__ err, int n_q, double *__restrict__ out) {
  const int qh = blockIdx.x;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int p = 0; p < n_q; ++p) t += err[qh * n_q + p];
    out[qh] = t / n_q;
  }
}

int64_t calibrate_workspace(int hq, int n_q, int64_t n) {
  return (int64_t)hq * n_q * n * 4 + (int64_t)hq * n_q * 8 + 512;
}

int dense_preference(const uint16_t *queries, const uint16_t *keys, int hq, int h, int n_q, int64_t n, int d,
                     int64_t k, double *head_scores, void *ws, cudaStream_t st) {
  if (n_q > CAL_NQ_MAX) return fail(TKV_ERR_PARAMETER, "n_q above 64 is not supported on the GPU path");
  float *z = reinterpret_cast<float *>(ws);
  double *err = reinterpret_cast<double *>(reinterpret_cast<char *>(ws) + (((size_t)hq * n_q * n * 4 + 255) & ~size_t(255)));
  const size_t sm = (size_t)n_q * d * 4;
  cudaFuncSetAttribute(cal_logits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cal_logits_kernel<<<dim3((unsigned)((n + 255) / 256), hq), 256, sm, st>>>(queries, keys, hq, h, n_q, n, d, z);
  cal_row_kernel<<<hq * n_q, 1024, 0, st>>>(z, n, k, err);
  cal_mean_kernel<<<hq, 32, 0, st>>>(err, n_q, head_scores);
  return check_launch("tkv_dense_preference");
}

}  // namespace tkv
