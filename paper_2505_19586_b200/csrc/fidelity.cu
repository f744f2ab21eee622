// Fidelity metrics of a sparsity-friendly layer, on the GPU:
// the reference's per-step oracle comparison (pipeline.py:316-325, 377-403)
// without the float64 CPU oracle.
//
// * exact attention of every query head over all n tokens of its KV head
//   (kv_model.py:169-213): keys from HBM, values from the pinned host store
//   (or the local mirror), fp32 split-K with a fixed-order combine;
// * group weights gw[j] = sum over the group's heads of the exact softmax
//   weight of token j (pipeline.py:380-383), as float64 for the top-k;
// * the exact top-k of gw by (weight desc, index desc) (retriever.py:229-243,
//   reusing the top-k kernels), recall@k of the engine's selection
//   (retriever.py:246-252) and its attention mass (pipeline.py:385).
// Cosine and max-abs against the engine's output are formed by the caller
// from the returned exact outputs (pipeline.py:143-150, 400-401).
#include <string>

#include "common.cuh"
#include "sparse.cuh"

namespace tkv {

constexpr int FD_CHUNK = 256;  // tokens per CTA
constexpr int FD_WARPS = 8;

template <int D>
__device__ __forceinline__ void fd_key_row(const SL &s, int u, int64_t j, int lane, float (&k)[D / 32]) {
  constexpr int CPL = D / 32;
  if (s.kdev) {
    const uint16_t *kp = s.kdev + ((size_t)u * s.capacity + j) * D + lane * CPL;
#pragma unroll
    for (int e = 0; e < CPL; ++e) k[e] = h2f(kp[e]);
  } else {
    const uint16_t *kt = s.kt + (size_t)u * s.d * s.capacity;
#pragma unroll
    for (int e = 0; e < CPL; ++e) k[e] = h2f(kt[((size_t)lane * CPL + e) * s.capacity + j]);
  }
}

template <int D>
__device__ __forceinline__ void fd_value_row(const SL &s, int u, int64_t j, int lane, float (&v)[D / 32]) {
  constexpr int CPL = D / 32;
  const uint16_t *vp = j >= s.local_offset ? s.loc_v + ((size_t)u * s.local_capacity + (j - s.local_offset)) * D
                                           : s.host_kv + ((size_t)u * s.capacity + j) * 2 * D + D;
#pragma unroll
  for (int e = 0; e < CPL; ++e) v[e] = h2f(vp[lane * CPL + e]);
}

// pass 1: per (chunk, unit) softmax partials of the G heads: m, l, acc[G][D]
template <int D>
__global__ void __launch_bounds__(FD_WARPS * 32) fidelity_partial_kernel(SL s, const uint16_t *__restrict__ queries,
                                                                         int G, int64_t n, int chunks,
                                                                         float *__restrict__ pm, float *__restrict__ pl,
                                                                         float *__restrict__ pacc) {
  constexpr int CPL = D / 32;
  __shared__ float wm[FD_WARPS][8], wl[FD_WARPS][8], wacc[FD_WARPS][8][D];
  const int u = blockIdx.y, chunk = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float zs = 1.4426950408889634f / sqrtf((float)D);
  float q[8][CPL], m[8], l[8], acc[8][CPL];
  for (int h = 0; h < 8; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.0f;
    for (int e = 0; e < CPL; ++e) {
      acc[h][e] = 0.0f;
      q[h][e] = h < G ? h2f(queries[((size_t)u * G + h) * D + lane * CPL + e]) * zs : 0.0f;
    }
  }
  const int64_t j0 = (int64_t)chunk * FD_CHUNK;
  for (int64_t j = j0 + warp; j < min(n, j0 + FD_CHUNK); j += FD_WARPS) {
    float k[CPL], v[CPL];
    fd_key_row<D>(s, u, j, lane, k);
    fd_value_row<D>(s, u, j, lane, v);
    for (int h = 0; h < G; ++h) {
      float dp = 0.0f;
#pragma unroll
      for (int e = 0; e < CPL; ++e) dp = fmaf(q[h][e], k[e], dp);
      const float z = warp_sum(dp);
      const float mn = fmaxf(m[h], z), sc = exp2f(m[h] - mn), p = exp2f(z - mn);
      l[h] = l[h] * sc + p;
      for (int e = 0; e < CPL; ++e) acc[h][e] = acc[h][e] * sc + p * v[e];
      m[h] = mn;
    }
  }
  for (int h = 0; h < G; ++h) {
    if (lane == 0) {
      wm[warp][h] = m[h];
      wl[warp][h] = l[h];
    }
    for (int e = 0; e < CPL; ++e) wacc[warp][h][lane * CPL + e] = acc[h][e];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < G * D; i += blockDim.x) {
    const int h = i / D, c = i % D;
    float M = -INFINITY;
    for (int w = 0; w < FD_WARPS; ++w) M = fmaxf(M, wm[w][h]);
    float L = 0.0f, A = 0.0f;
    for (int w = 0; w < FD_WARPS; ++w) {
      if (wm[w][h] == -INFINITY) continue;
      const float sc = exp2f(wm[w][h] - M);
      L += sc * wl[w][h];
      A += sc * wacc[w][h][c];
    }
    const size_t b = ((size_t)u * chunks + chunk) * G + h;
    pacc[b * D + c] = A;
    if (c == 0) {
      pm[b] = M;
      pl[b] = L;
    }
  }
}

// pass 2: fixed-order combine -> exact outputs and per-head (M, L)
__global__ void fidelity_combine_kernel(const float *__restrict__ pm, const float *__restrict__ pl,
                                        const float *__restrict__ pacc, int chunks, int G, int D,
                                        float *__restrict__ out, float *__restrict__ hm, float *__restrict__ hl) {
  const int uh = blockIdx.x, u = uh / G, h = uh % G, c = threadIdx.x;  // D threads = channels
  float M = -INFINITY;
  for (int ci = 0; ci < chunks; ++ci) M = fmaxf(M, pm[((size_t)u * chunks + ci) * G + h]);
  float L = 0.0f, A = 0.0f;
  for (int ci = 0; ci < chunks; ++ci) {
    const size_t b = ((size_t)u * chunks + ci) * G + h;
    if (pm[b] == -INFINITY) continue;
    const float sc = exp2f(pm[b] - M);
    L += sc * pl[b];
    A += sc * pacc[b * D + c];
  }
  out[(size_t)uh * D + c] = A / L;
  if (c == 0) {
    hm[uh] = M;
    hl[uh] = L;
  }
}

// pass 3: group weights gw[u][j] = sum_h exp2(z_hj - M_h) / L_h (float64 for the top-k)
template <int D>
__global__ void __launch_bounds__(FD_WARPS * 32) fidelity_group_weights_kernel(SL s, const uint16_t *__restrict__ queries,
                                                                               int G, int64_t n,
                                                                               const float *__restrict__ hm,
                                                                               const float *__restrict__ hl,
                                                                               double *__restrict__ gw) {
  constexpr int CPL = D / 32;
  const int u = blockIdx.y, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float zs = 1.4426950408889634f / sqrtf((float)D);
  float q[8][CPL];
  for (int h = 0; h < 8; ++h)
    for (int e = 0; e < CPL; ++e) q[h][e] = h < G ? h2f(queries[((size_t)u * G + h) * D + lane * CPL + e]) * zs : 0.0f;
  const int64_t j0 = (int64_t)blockIdx.x * FD_CHUNK;
  for (int64_t j = j0 + warp; j < min(n, j0 + FD_CHUNK); j += FD_WARPS) {
    float k[CPL];
    fd_key_row<D>(s, u, j, lane, k);
    double w = 0.0;
    for (int h = 0; h < G; ++h) {
      float dp = 0.0f;
#pragma unroll
      for (int e = 0; e < CPL; ++e) dp = fmaf(q[h][e], k[e], dp);
      const float z = warp_sum(dp);
      w += (double)exp2f(z - hm[u * G + h]) / (double)hl[u * G + h];
    }
    if (lane == 0) gw[(size_t)u * n + j] = w;
  }
}

// pass 4: per unit, recall@k of the selection against the exact top-k and its mass
__global__ void fidelity_recall_kernel(const int32_t *__restrict__ sel_idx, const int32_t *__restrict__ sel_count,
                                       int sel_stride, const int32_t *__restrict__ top_idx,
                                       const int32_t *__restrict__ top_count, int top_stride,
                                       const double *__restrict__ gw, int64_t n, int G, double *__restrict__ metrics) {
  __shared__ int hits;
  __shared__ double mass;
  const int u = blockIdx.x;
  if (threadIdx.x == 0) {
    hits = 0;
    mass = 0.0;
  }
  __syncthreads();
  const int ns = sel_count[u], nt = top_count[u];
  const int32_t *tp = top_idx + (size_t)u * top_stride;
  for (int i = threadIdx.x; i < ns; i += blockDim.x) {
    const int j = sel_idx[(size_t)u * sel_stride + i];
    int lo = 0, hi = nt;  // the exact top-k is sorted ascending
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (tp[mid] < j) lo = mid + 1;
      else hi = mid;
    }
    if (lo < nt && tp[lo] == j) atomicAdd(&hits, 1);
    atomicAdd(&mass, gw[(size_t)u * n + j]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    metrics[u * 2 + 0] = nt ? (double)hits / (double)nt : 0.0;  // retriever.py:246-252
    metrics[u * 2 + 1] = mass / (double)G;                       // pipeline.py:385
  }
}

int64_t fidelity_workspace(int units, int G, int64_t n, int k) {
  const int64_t chunks = (n + FD_CHUNK - 1) / FD_CHUNK;
  int64_t b = (int64_t)units * chunks * G * (2 + 256) * 4;  // partials (d <= 256)
  b += (int64_t)units * G * 2 * 4;                           // head M, L
  b = (b + 255) / 256 * 256;
  b += (int64_t)units * n * 8;                                // group weights
  b += (int64_t)units * k * 4 + (int64_t)units * 4;           // exact top-k
  b = (b + 255) / 256 * 256;
  return b + select_workspace(units, n) + 256;
}

int sparse_fidelity(const SL &s, const uint16_t *queries, int G, int64_t n, const int32_t *sel_idx,
                    const int32_t *sel_count, int sel_stride, int k, float *exact_out, double *metrics, void *ws,
                    cudaStream_t st) {
  if ((s.d != 128 && s.d != 64) || G > 8) return fail(TKV_ERR_SHAPE, "fidelity metrics support head_dim 64/128, G <= 8");
  const int chunks = (int)((n + FD_CHUNK - 1) / FD_CHUNK);
  char *w = static_cast<char *>(ws);
  float *pm = reinterpret_cast<float *>(w);
  float *pl = pm + (size_t)s.units * chunks * G;
  float *pacc = pl + (size_t)s.units * chunks * G;
  float *hm = pacc + (size_t)s.units * chunks * G * s.d;
  float *hl = hm + (size_t)s.units * G;
  int64_t off = ((int64_t)s.units * chunks * G * (2 + 256) * 4 + (int64_t)s.units * G * 2 * 4 + 255) / 256 * 256;
  double *gw = reinterpret_cast<double *>(w + off);
  off += (int64_t)s.units * n * 8;
  int32_t *top_idx = reinterpret_cast<int32_t *>(w + off);
  int32_t *top_cnt = top_idx + (size_t)s.units * k;
  off = ((off + (int64_t)s.units * k * 4 + (int64_t)s.units * 4) + 255) / 256 * 256;
  const dim3 grid(chunks, s.units);
  if (s.d == 128) fidelity_partial_kernel<128><<<grid, FD_WARPS * 32, 0, st>>>(s, queries, G, n, chunks, pm, pl, pacc);
  else fidelity_partial_kernel<64><<<grid, FD_WARPS * 32, 0, st>>>(s, queries, G, n, chunks, pm, pl, pacc);
  fidelity_combine_kernel<<<s.units * G, s.d, 0, st>>>(pm, pl, pacc, chunks, G, s.d, exact_out, hm, hl);
  if (s.d == 128) fidelity_group_weights_kernel<128><<<grid, FD_WARPS * 32, 0, st>>>(s, queries, G, n, hm, hl, gw);
  else fidelity_group_weights_kernel<64><<<grid, FD_WARPS * 32, 0, st>>>(s, queries, G, n, hm, hl, gw);
  // the multi-kernel top-k starts from a zeroed workspace (histograms, counters)
  cudaMemsetAsync(w + off, 0, (size_t)select_workspace(s.units, n), st);
  if (int r = topk_from_scores(gw, s.units, n, 0, k, top_idx, top_cnt, w + off, st)) return r;
  fidelity_recall_kernel<<<s.units, 256, 0, st>>>(sel_idx, sel_count, sel_stride, top_idx, top_cnt, k, gw, n, G,
                                                   metrics);
  return check_launch("tkv_sparse_fidelity");
}

}  // namespace tkv
