// Fused stage 2 for one sparsity-friendly layer: proxy scores
// (retriever.py:166-189) + exact top-k by (score desc, index desc) plus the
// local window, sorted ascending (retriever.py:192-211) -- one launch.
//
// One thread-block cluster per unit (KV head): 16 CTAs when the GPU can
// co-schedule them (non-portable size), else 8.  Each CTA scores a contiguous
// slice of the candidate tokens into shared memory as 8-byte
// order-preserving keys of the float64 scores; the cluster then runs a radix
// select with 11-bit digits over the bits below the keys' common prefix,
// exchanging the per-CTA histograms through distributed shared memory (DSMEM),
// so the 1 MB of keys of a 128k-token head never round-trips through HBM.
// Exact score ties at the threshold go to the larger index, as the
// reference's lexsort does.  Output order is ascending because every CTA owns
// a contiguous index range and writes at its cluster-prefix offset.
#include <cooperative_groups.h>

#include <string>

#include "common.cuh"
#include "sparse.cuh"

namespace cg = cooperative_groups;

namespace tkv {

constexpr int SC_THREADS = 1024;
constexpr int SC_CHUNK_CAP = 18432;  // keys per CTA (8 B each): 8 CTAs cover 147,456 candidates
constexpr int SC_BITS = 11;
constexpr int SC_BINS = 1 << SC_BITS;

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

// phase timestamps of CTA 0 / unit 0 (debug: tkv_debug_select_phases)
__device__ unsigned long long g_sel_phase[8];
#define SC_MARK(i)                                                         \
  do {                                                                     \
    if (blockIdx.y == 0 && rank == 0 && tid == 0) {                        \
      unsigned long long t_;                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                \
      g_sel_phase[i] = t_;                                                 \
    }                                                                      \
  } while (0)

constexpr int SC_BAND = 256;  // per-CTA cap of fp32-ambiguous candidates

struct SelShared {
  union {
    uint64_t keys64[SC_CHUNK_CAP];  // exact path: order-preserving float64 score keys
    struct {
      uint32_t keys32[SC_CHUNK_CAP];  // fast path: order-preserving fp32 score keys
      unsigned long long band_key[SC_BAND];
      uint32_t band_idx[SC_BAND];
      unsigned long long all_key[SC_BAND * 8];
      uint32_t all_idx[SC_BAND * 8];
    } f;
  } k;
  uint8_t flags[SC_CHUNK_CAP];
  uint32_t hist[2][SC_BINS];
  uint32_t tot[SC_BINS];
};

struct SelCtl {
  unsigned long long prefix;
  int need, done;
  int cta_count, band_count, overflow;
  unsigned long long kmin[32], kmax[32], ck[2];
  int scan[40];
};

__device__ __forceinline__ uint32_t orderable32(float x) {
  if (x == 0.0f) x = 0.0f;
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float from_orderable32(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// Cluster-wide min/max of the keys -> number of undecided low bits (`top`)
// and the common prefix above them.
template <int CTAS, typename KT>
__device__ void cluster_common_prefix(cg::cluster_group &cluster, const KT *keys, int m, SelCtl &C, int &top,
                                      unsigned long long &prefix) {
  constexpr int NB = 8 * sizeof(KT);
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned long long lo = ~0ull, hi = 0ull;
  for (int e = tid; e < m; e += blockDim.x) {
    const unsigned long long k = keys[e];
    lo = k < lo ? k : lo;
    hi = k > hi ? k : hi;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o), b = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if (lane == 0) {
    C.kmin[tid >> 5] = lo;
    C.kmax[tid >> 5] = hi;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = C.kmin[w] < lo ? C.kmin[w] : lo;
      hi = C.kmax[w] > hi ? C.kmax[w] : hi;
    }
    C.ck[0] = lo;
    C.ck[1] = hi;
  }
  cluster.sync();
  lo = ~0ull;
  hi = 0ull;
  for (int r = 0; r < CTAS; ++r) {
    const unsigned long long *rk = cluster.map_shared_rank(C.ck, r);
    lo = rk[0] < lo ? rk[0] : lo;
    hi = rk[1] > hi ? rk[1] : hi;
  }
  const int diff = lo == hi ? 0 : 64 - __clzll((long long)(lo ^ hi));  // highest differing bit + 1
  top = diff;                                                           // bits [0, top) undecided
  prefix = top >= 64 ? 0ull : (lo >> top) << top;
  (void)NB;
}

// Radix select (11-bit digits) of the `need`-th largest key over the
// cluster's keys.  Returns with prefix/top describing the threshold bin;
// done == true when exactly `need` keys remain in it (all selected).
template <int CTAS, typename KT>
__device__ void cluster_radix(cg::cluster_group &cluster, const KT *keys, int m, SelShared &S, SelCtl &C, int &top,
                             unsigned long long &prefix, int &need, bool &done, bool early_exit) {
  const int tid = threadIdx.x;
  done = false;
  for (int pass = 0; top > 0 && !done; ++pass) {
    const int w = top < SC_BITS ? top : SC_BITS;
    const int shift = top - w;
    const unsigned long long mask = top >= 64 ? 0ull : ~0ull << top;
    const int nb = 1 << w;
    uint32_t *H = S.hist[pass & 1];
    for (int i = tid; i < nb; i += blockDim.x) H[i] = 0;
    __syncthreads();
    const uint32_t dmask = (uint32_t)nb - 1u;
    for (int e = tid; e < m; e += blockDim.x) {
      const unsigned long long k = keys[e];
      if ((k & mask) == prefix) atomicAdd(&H[(uint32_t)(k >> shift) & dmask], 1u);
    }
    cluster.sync();
    for (int b = tid; b < nb; b += blockDim.x) {
      uint32_t t = 0;
#pragma unroll
      for (int r = 0; r < CTAS; ++r) t += cluster.map_shared_rank(H, r)[b];
      S.tot[nb - 1 - b] = t;  // descending-bin order
    }
    __syncthreads();
    int v = 0;
    for (int p2 = tid * 2; p2 < tid * 2 + 2 && p2 < nb; ++p2) v += (int)S.tot[p2];
    int total;
    const int before = block_excl_scan(v, C.scan, &total);
    if (before < need && before + v >= need) {
      int cum = before;
      for (int p2 = tid * 2; p2 < tid * 2 + 2 && p2 < nb; ++p2) {
        const int c = (int)S.tot[p2];
        if (cum + c >= need) {
          const int bin = nb - 1 - p2;
          C.need = need - cum;
          C.prefix = prefix | ((unsigned long long)bin << shift);
          C.done = early_exit && c == need - cum;
          break;
        }
        cum += c;
      }
    }
    __syncthreads();
    prefix = C.prefix;
    need = C.need;
    done = C.done;
    top = shift;
  }
}

// Flags for the keys relative to the threshold bin (1 selected, 0 not);
// ties at the threshold keep the `need` largest indices.
template <int CTAS, typename KT>
__device__ void cluster_flags(cg::cluster_group &cluster, const KT *keys, int m, uint8_t *flags, SelCtl &C, int top,
                              unsigned long long prefix, int need, bool done) {
  const int tid = threadIdx.x;
  const int rank = (int)cluster.block_rank();
  const unsigned long long fmask = top >= 64 ? 0ull : ~0ull << top;
  int ties = 0;
  for (int e = tid; e < m; e += blockDim.x) {
    const unsigned long long k = (unsigned long long)keys[e] & fmask;
    uint8_t f = k > prefix ? 1 : 0;
    if (k == prefix) {
      if (done) f = 1;
      else { f = 2; ++ties; }
    }
    flags[e] = f;
  }
  if (done) return;
  int tot_ties;
  block_excl_scan(ties, C.scan, &tot_ties);
  if (tid == 0) C.cta_count = tot_ties;
  cluster.sync();
  int above = 0;
  for (int r = rank + 1; r < CTAS; ++r) above += cluster.map_shared_rank(&C, r)->cta_count;
  const int allowed = max(0, min(tot_ties, need - above));
  const int per = (m + SC_THREADS - 1) / SC_THREADS;
  const int b0 = tid * per, b1 = min(m, b0 + per);
  int mine = 0;
  for (int e = b0; e < b1; ++e) mine += flags[e] == 2;
  int dummy;
  const int before = block_excl_scan(mine, C.scan, &dummy);
  int higher = tot_ties - before - mine;  // ties at indices above this thread's range
  for (int e = b1 - 1; e >= b0; --e) {
    if (flags[e] == 2) {
      flags[e] = higher < allowed ? 1 : 0;
      ++higher;
    }
  }
  cluster.sync();  // cta_count reads complete before reuse
}

template <int CTAS>
__global__ void __launch_bounds__(SC_THREADS, 1)
    select_cluster_kernel(SL s, const uint16_t *__restrict__ queries, int G, const int32_t *__restrict__ channels,
                          int d_s, int n_local, int n_topk, int32_t *__restrict__ sel_idx, int sel_stride,
                          int32_t *__restrict__ sel_count, int32_t *__restrict__ fetch_count,
                          double *__restrict__ scores_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  SelShared &S = *reinterpret_cast<SelShared *>(smem);
  __shared__ SelCtl C;
  __shared__ double qsum[128];
  __shared__ float qsum32[128];
  __shared__ int chs[128];
  __shared__ double band_eps;
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
  const int64_t chunk = ((ncand + CTAS - 1) / CTAS + 7) & ~int64_t(7);
  const int64_t j0 = rank * chunk;
  const int m = (int)(j0 < ncand ? imin64(chunk, ncand - j0) : 0);
  uint8_t *flags = S.flags;
  SC_MARK(0);
  for (int i = tid; i < d_s; i += blockDim.x) {
    const int ch = channels[(size_t)u * d_s + i];
    double q = 0.0;
    for (int j = 0; j < G; ++j) q += h2d(queries[((size_t)u * G + j) * s.d + ch]);  // group sum (retriever.py:189)
    qsum[i] = q;
    qsum32[i] = (float)q;
    chs[i] = ch;
  }
  if (tid == 0) {
    C.band_count = 0;
    C.overflow = 0;
  }
  __syncthreads();
  if (tid == 0) {
    // |fp32 score - float64 score| <= 2^-20 * sum_i max|K_i| |q_i| (9 roundings of 2^-24)
    double e = 0.0;
    for (int i = 0; i < d_s; ++i) e += (double)s.chmax[(size_t)u * s.d + chs[i]] * fabs(qsum[i]);
    band_eps = e * 9.5367431640625e-07;  // 2^-20
  }
  const uint16_t *kt = s.kt + (size_t)u * s.d * s.capacity;
  // ---- fast path: fp32 proxy scores (retriever.py:189) into order-preserving keys ----
  uint32_t *keys32 = S.k.f.keys32;
  for (int e0 = tid * 8; e0 < m; e0 += SC_THREADS * 8) {
    const int64_t j = j0 + e0;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
    const bool full = e0 + 8 <= m;
    int i = 0;
    if (full) {
      for (; i + 8 <= d_s; i += 8) {
        uint4 v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = __ldg(reinterpret_cast<const uint4 *>(kt + (size_t)chs[i + r] * s.capacity + j));
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const float qv = qsum32[i + r];
          const uint32_t w[4] = {v[r].x, v[r].y, v[r].z, v[r].w};
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = fmaf(h2f((uint16_t)(w[e >> 1] >> (16 * (e & 1)))), qv, acc[e]);
        }
      }
    }
    for (; i < d_s; ++i) {
      const uint16_t *row = kt + (size_t)chs[i] * s.capacity + j;
      const float qv = qsum32[i];
      for (int e = 0; e < 8 && e0 + e < m; ++e) acc[e] = fmaf(h2f(row[e]), qv, acc[e]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e0 + e < m) keys32[e0 + e] = orderable32(acc[e]);
  }
  SC_MARK(1);
  int top, need = n_topk;
  unsigned long long prefix;
  bool done;
  cluster_common_prefix<CTAS>(cluster, keys32, m, C, top, prefix);
  SC_MARK(2);
  cluster_radix<CTAS>(cluster, keys32, m, S, C, top, prefix, need, done, false);
  SC_MARK(3);
  // threshold value T32 = the n_topk-th largest fp32 score; the float64 order
  // can differ only within +-2 eps of it (|T64 - T32| <= eps)
  const double T32 = (double)from_orderable32((uint32_t)prefix);
  const double eps2 = 2.0 * band_eps;
  int definite = 0;
  for (int e = tid; e < m; e += blockDim.x) {
    const double dv = (double)from_orderable32(keys32[e]) - T32;
    uint8_t f = 0;
    if (dv > eps2) {
      f = 1;
      ++definite;
    } else if (dv >= -eps2) {
      const int slot = atomicAdd(&C.band_count, 1);
      if (slot < SC_BAND) {
        // exact float64 score for the ambiguous candidate (reference arithmetic)
        const int64_t j = j0 + e;
        double sc = 0.0;
        for (int i = 0; i < d_s; ++i) sc = fma(h2d(kt[(size_t)chs[i] * s.capacity + j]), qsum[i], sc);
        S.k.f.band_key[slot] = orderable(sc);
        S.k.f.band_idx[slot] = (uint32_t)j;
      } else {
        C.overflow = 1;
      }
      f = 3;
    }
    flags[e] = f;
  }
  int tot_def;
  block_excl_scan(definite, C.scan, &tot_def);
  if (tid == 0) C.cta_count = tot_def;
  cluster.sync();
  int all_def = 0, all_band = 0, overflow = 0;
  for (int r = 0; r < CTAS; ++r) {
    const SelCtl *R = cluster.map_shared_rank(&C, r);
    all_def += R->cta_count;
    all_band += min(R->band_count, SC_BAND);
    overflow |= R->overflow;
  }
  if (!overflow) {
    // gather every CTA's band (<= 8 x 256), rank the local band members among them
    int off = 0;
    for (int r = 0; r < CTAS; ++r) {
      const SelShared *RS = cluster.map_shared_rank(&S, r);
      const int c = min(cluster.map_shared_rank(&C, r)->band_count, SC_BAND);
      for (int i = tid; i < c; i += blockDim.x) {
        S.k.f.all_key[off + i] = RS->k.f.band_key[i];
        S.k.f.all_idx[off + i] = RS->k.f.band_idx[i];
      }
      off += c;
    }
    __syncthreads();
    const int need_b = n_topk - all_def;
    const int mine = min(C.band_count, SC_BAND);
    for (int b = tid; b < mine; b += blockDim.x) {
      const unsigned long long kb = S.k.f.band_key[b];
      const uint32_t ib = S.k.f.band_idx[b];
      int beaten = 0;
      for (int o = 0; o < all_band; ++o) {
        const unsigned long long ko = S.k.f.all_key[o];
        const uint32_t io = S.k.f.all_idx[o];
        beaten += (ko > kb) || (ko == kb && io > ib);  // (score desc, index desc)
      }
      flags[ib - j0] = beaten < need_b ? 1 : 0;
    }
    cluster.sync();  // band arrays read by other CTAs before the output phase reuses nothing
    __syncthreads();
    for (int e = tid; e < m; e += blockDim.x)
      if (flags[e] == 3) flags[e] = 0;  // (never happens: every band member was ranked)
  } else {
    // ---- exact path (degenerate inputs, e.g. huge exact-tie sets): float64 keys ----
    uint64_t *keys64 = S.k.keys64;
    __syncthreads();
    for (int e = tid; e < m; e += blockDim.x) {
      const int64_t j = j0 + e;
      double sc = 0.0;
      for (int i = 0; i < d_s; ++i) sc = fma(h2d(kt[(size_t)chs[i] * s.capacity + j]), qsum[i], sc);
      keys64[e] = orderable(sc);
    }
    __syncthreads();
    need = n_topk;
    cluster_common_prefix<CTAS>(cluster, keys64, m, C, top, prefix);
    cluster_radix<CTAS>(cluster, keys64, m, S, C, top, prefix, need, done, true);
    cluster_flags<CTAS>(cluster, keys64, m, flags, C, top, prefix, need, done);
  }
  if (scores_out) {
    for (int e = tid; e < m; e += blockDim.x) {
      const int64_t j = j0 + e;
      double sc = 0.0;
      for (int i = 0; i < d_s; ++i) sc = fma(h2d(kt[(size_t)chs[i] * s.capacity + j]), qsum[i], sc);
      scores_out[(size_t)u * s.capacity + j] = sc;
    }
  }
  __syncthreads();
  SC_MARK(4);
  // ---- ascending output: contiguous ownership + cluster prefix offsets ----
  const int per = (m + SC_THREADS - 1) / SC_THREADS;
  const int b0 = tid * per, b1 = min(m, b0 + per);
  int mine = 0;
  for (int e = b0; e < b1; ++e) mine += flags[e];
  int cta_total;
  int pos = block_excl_scan(mine, C.scan, &cta_total);
  if (tid == 0) C.cta_count = cta_total;
  cluster.sync();
  int offset = 0;
  for (int r = 0; r < rank; ++r) offset += cluster.map_shared_rank(&C, r)->cta_count;
  for (int e = b0; e < b1; ++e)
    if (flags[e]) out_idx[offset + pos++] = (int32_t)(j0 + e);
  if (rank == CTAS - 1) {
    for (int i = tid; i < n_local; i += blockDim.x) out_idx[n_topk + i] = (int32_t)(ncand + i);
    if (tid == 0) {
      sel_count[u] = n_topk + n_local;
      if (fetch_count) fetch_count[u] = n_topk;
    }
  }
  cluster.sync();  // no CTA leaves while its shared memory may still be read
  SC_MARK(5);
}

static int cluster_ctas() {
  // 16-CTA clusters when the hardware co-schedules them, else 8 (portable)
  static int cached = 0;
  if (cached) return cached;
  const size_t sm = sizeof(SelShared);
  cudaFuncSetAttribute(select_cluster_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(select_cluster_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaFuncSetAttribute(select_cluster_kernel<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(16, 1);
  cfg.blockDim = dim3(SC_THREADS);
  cfg.dynamicSmemBytes = sm;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 16;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int nclusters = 0;
  const char *env = getenv("TKV_SELECT_CLUSTER");
  if (!env || atoi(env) != 16)
    cached = 8;  // measured: 16-CTA clusters are slower on B200 (fewer co-resident clusters)
  else if (cudaOccupancyMaxActiveClusters(&nclusters, select_cluster_kernel<16>, &cfg) == cudaSuccess && nclusters > 0)
    cached = 16;
  else
    cached = 8;
  cudaGetLastError();
  return cached;
}

bool select_cluster_ok(const SL &s, int n_local) {
  const int64_t ncand = s.capacity - n_local;
  const int ctas = cluster_ctas();
  const int64_t chunk = ((ncand + ctas - 1) / ctas + 7) & ~int64_t(7);
  return chunk <= SC_CHUNK_CAP && s.capacity % 8 == 0;
}

int select_cluster(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s, int n_local,
                   int n_topk, int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count, double *scores_out,
                   cudaStream_t st) {
  const int ctas = cluster_ctas();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas, s.units);
  cfg.blockDim = dim3(SC_THREADS);
  cfg.dynamicSmemBytes = sizeof(SelShared);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = ctas;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int stride = n_local + n_topk;
  cudaError_t e;
  if (ctas == 16)
    e = cudaLaunchKernelEx(&cfg, select_cluster_kernel<16>, s, queries, G, channels, d_s, n_local, n_topk, sel_idx,
                           stride, sel_count, fetch_count, scores_out);
  else
    e = cudaLaunchKernelEx(&cfg, select_cluster_kernel<8>, s, queries, G, channels, d_s, n_local, n_topk, sel_idx,
                           stride, sel_count, fetch_count, scores_out);
  if (e != cudaSuccess) return fail(TKV_ERR_CUDA, std::string("tkv_select_tokens(cluster): ") + cudaGetErrorString(e));
  return check_launch("tkv_select_tokens(cluster)");
}

}  // namespace tkv

extern "C" int tkv_debug_select_phases(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, tkv::g_sel_phase, sizeof(unsigned long long) * 8) == cudaSuccess ? 0 : 7;
}
