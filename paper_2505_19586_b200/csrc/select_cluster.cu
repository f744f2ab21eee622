// Fused stage 2 for one sparsity-friendly layer: proxy scores
// (retriever.py:166-189) + exact top-k by (score desc, index desc) plus the
// local window, sorted ascending (retriever.py:192-211) -- one launch.
//
// One 8-CTA thread-block cluster per unit (KV head).  Each CTA scores a
// contiguous slice of the candidate tokens into shared memory (8-byte
// order-preserving keys of the float64 scores), then the cluster runs an
// 8-bit-digit radix select over the 64-bit keys with the per-CTA histograms
// exchanged through distributed shared memory (DSMEM), so the 1 MB of keys of
// a 128k-token head never round-trips through HBM.  Exact score ties at the
// threshold are resolved toward the larger index, as the reference's
// lexsort does.  Output order is ascending because every CTA owns a
// contiguous index range and writes at its cluster-prefix offset.
#include <cooperative_groups.h>

#include "common.cuh"
#include "sparse.cuh"

namespace cg = cooperative_groups;

namespace tkv {

constexpr int SC_CTAS = 8;
constexpr int SC_THREADS = 1024;
constexpr int SC_CHUNK_CAP = 24576;  // keys per CTA (8 B each) -> 196608 candidates per unit

__device__ __forceinline__ int block_excl_scan(int v, int *sh, int *total) {
  // sh: >= 33 ints
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int s = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    sh[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  const int before = (w ? sh[w - 1] : 0) + x - v;
  if (total) *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

__global__ void __cluster_dims__(SC_CTAS, 1, 1) __launch_bounds__(SC_THREADS, 1)
    select_cluster_kernel(SL s, const uint16_t *__restrict__ queries, int G, const int32_t *__restrict__ channels,
                          int d_s, int n_local, int n_topk, int32_t *__restrict__ sel_idx, int sel_stride,
                          int32_t *__restrict__ sel_count, int32_t *__restrict__ fetch_count,
                          double *__restrict__ scores_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint32_t hist[2][256];
  __shared__ uint32_t tot[256];
  __shared__ double qsum[128];
  __shared__ int chs[128];
  __shared__ int scan_sh[40];
  __shared__ int cta_count;
  __shared__ unsigned long long sh_prefix, sh_mask;
  __shared__ int sh_need, sh_done;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int u = blockIdx.y;
  const int tid = threadIdx.x;
  const int64_t n = *s.len;
  int32_t *out_idx = sel_idx + (size_t)u * sel_stride;
  if (n <= (int64_t)n_local + n_topk) {  // select everything (retriever.py:204-205)
    if (rank == 0) {
      for (int64_t j = tid; j < n; j += blockDim.x) out_idx[j] = (int32_t)j;
      if (tid == 0) {
        sel_count[u] = (int32_t)n;
        if (fetch_count) fetch_count[u] = (int32_t)(n > n_local ? n - n_local : 0);
      }
    }
    return;  // uniform across the cluster
  }
  const int64_t ncand = n - n_local;
  const int64_t chunk = ((ncand + SC_CTAS - 1) / SC_CTAS + 7) & ~int64_t(7);
  const int64_t j0 = rank * chunk;
  const int m = (int)(j0 < ncand ? imin64(chunk, ncand - j0) : 0);
  uint64_t *keys = reinterpret_cast<uint64_t *>(smem);
  uint8_t *flags = smem + (size_t)SC_CHUNK_CAP * 8;

  for (int i = tid; i < d_s; i += blockDim.x) {
    const int ch = channels[(size_t)u * d_s + i];
    double q = 0.0;
    for (int j = 0; j < G; ++j) q += h2d(queries[((size_t)u * G + j) * s.d + ch]);  // group sum
    qsum[i] = q;
    chs[i] = ch;
  }
  __syncthreads();
  // ---- scores: 8 consecutive tokens per thread, 16-byte loads per channel row ----
  const uint16_t *kt = s.kt + (size_t)u * s.d * s.capacity;
  for (int e0 = tid * 8; e0 < m; e0 += SC_THREADS * 8) {
    const int64_t j = j0 + e0;
    double acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
    const bool full = e0 + 8 <= m;
    for (int i = 0; i < d_s; ++i) {
      const uint16_t *row = kt + (size_t)chs[i] * s.capacity + j;
      const double qv = qsum[i];
      if (full) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(row));
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = fma(h2d((uint16_t)(w[e >> 1] >> (16 * (e & 1)))), qv, acc[e]);
      } else {
        for (int e = 0; e < 8 && e0 + e < m; ++e) acc[e] = fma(h2d(row[e]), qv, acc[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (e0 + e < m) {
        keys[e0 + e] = orderable(acc[e]);
        if (scores_out) scores_out[(size_t)u * s.capacity + j + e] = acc[e];
      }
    }
  }
  if (tid == 0) { sh_prefix = 0; sh_mask = 0; sh_need = n_topk; sh_done = 0; }
  __syncthreads();
  // ---- cluster radix select over the 64-bit keys ----
  uint64_t prefix = 0, mask = 0;
  int need = n_topk;
  bool done = false;
  for (int pass = 0; pass < 8 && !done; ++pass) {
    const int shift = 56 - 8 * pass;
    uint32_t *H = hist[pass & 1];
    if (tid < 256) H[tid] = 0;
    __syncthreads();
    for (int e = tid; e < m; e += blockDim.x) {
      const uint64_t k = keys[e];
      if ((k & mask) == prefix) atomicAdd(&H[(uint32_t)(k >> shift) & 255u], 1u);
    }
    cluster.sync();
    if (tid < 256) {
      uint32_t t = 0;
      for (int r = 0; r < SC_CTAS; ++r) t += cluster.map_shared_rank(H, r)[tid];
      tot[tid] = t;
    }
    __syncthreads();
    if (tid < 32) {
      // warp-parallel descending scan: lane l owns bins 255-8l-7 .. 255-8l
      uint32_t v[8];
      int sum = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i] = tot[255 - 8 * tid - i];
        sum += (int)v[i];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += y;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, incl >= need);
      const int L = __ffs(hit) - 1;
      if (tid == L) {
        int cum = incl - sum, D = 255 - 8 * L;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (cum + (int)v[i] >= need) { D = 255 - 8 * L - i; break; }
          cum += (int)v[i];
        }
        sh_need = need - cum;
        sh_prefix = prefix | ((uint64_t)D << shift);
        sh_mask = mask | (255ull << shift);
        sh_done = (int)tot[D] == need - cum;
      }
    }
    __syncthreads();
    prefix = sh_prefix;
    mask = sh_mask;
    need = sh_need;
    done = sh_done;
  }
  // ---- selection flags ----
  int ties = 0;
  for (int e = tid; e < m; e += blockDim.x) {
    const uint64_t k = keys[e] & mask;
    uint8_t f = k > prefix ? 1 : 0;
    if (k == prefix) {
      if (done) f = 1;
      else { f = 2; ++ties; }
    }
    flags[e] = f;
  }
  if (!done) {
    // exact ties at the threshold: keep the `need` largest indices
    int tot_ties;
    block_excl_scan(ties, scan_sh, &tot_ties);
    if (tid == 0) cta_count = tot_ties;
    cluster.sync();
    int above = 0;
    for (int r = rank + 1; r < SC_CTAS; ++r) above += *cluster.map_shared_rank(&cta_count, r);
    const int allowed = max(0, min(tot_ties, need - above));
    // rank of a tie inside this CTA counted from the highest index
    const int per = (m + SC_THREADS - 1) / SC_THREADS;
    const int b0 = tid * per, b1 = min(m, b0 + per);
    int mine = 0;
    for (int e = b0; e < b1; ++e) mine += flags[e] == 2;
    int dummy;
    const int before = block_excl_scan(mine, scan_sh, &dummy);
    int higher = tot_ties - before - mine;  // ties at indices above this thread's range
    for (int e = b1 - 1; e >= b0; --e) {
      if (flags[e] == 2) {
        flags[e] = higher < allowed ? 1 : 0;
        ++higher;
      }
    }
    cluster.sync();  // cta_count reads complete before reuse
  }
  __syncthreads();
  // ---- ascending output: contiguous ownership + cluster prefix offsets ----
  const int per = (m + SC_THREADS - 1) / SC_THREADS;
  const int b0 = tid * per, b1 = min(m, b0 + per);
  int mine = 0;
  for (int e = b0; e < b1; ++e) mine += flags[e];
  int cta_total;
  int pos = block_excl_scan(mine, scan_sh, &cta_total);
  if (tid == 0) cta_count = cta_total;
  cluster.sync();
  int offset = 0;
  for (int r = 0; r < rank; ++r) offset += *cluster.map_shared_rank(&cta_count, r);
  for (int e = b0; e < b1; ++e)
    if (flags[e]) out_idx[offset + pos++] = (int32_t)(j0 + e);
  if (rank == SC_CTAS - 1) {
    for (int i = tid; i < n_local; i += blockDim.x) out_idx[n_topk + i] = (int32_t)(ncand + i);
    if (tid == 0) {
      sel_count[u] = n_topk + n_local;
      if (fetch_count) fetch_count[u] = n_topk;
    }
  }
  cluster.sync();  // no CTA leaves while its shared memory may still be read
}

bool select_cluster_ok(const SL &s, int n_local) {
  const int64_t ncand = s.capacity - n_local;
  const int64_t chunk = ((ncand + SC_CTAS - 1) / SC_CTAS + 7) & ~int64_t(7);
  return chunk <= SC_CHUNK_CAP && s.capacity % 8 == 0;
}

int select_cluster(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s, int n_local,
                   int n_topk, int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count, double *scores_out,
                   cudaStream_t st) {
  const size_t sm = (size_t)SC_CHUNK_CAP * 9;
  cudaFuncSetAttribute(select_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 grid(SC_CTAS, s.units);
  select_cluster_kernel<<<grid, SC_THREADS, sm, st>>>(s, queries, G, channels, d_s, n_local, n_topk, sel_idx,
                                                       n_local + n_topk, sel_count, fetch_count, scores_out);
  return check_launch("tkv_select_tokens(cluster)");
}

}  // namespace tkv
