// One launch per sparsity-friendly layer: proxy scores (retriever.py:166-189)
// -> exact top-k by (score desc, index desc) plus the local window, sorted
// ascending (retriever.py:192-211) -> gather of the selected rows (value rows
// over PCIe from the pinned host store, memsim.py:228-252) -> exact softmax
// attention over them (pipeline.py:364-376).
//
// One 8-CTA thread-block cluster per unit (batch x KV head), 1024 threads per
// CTA.  Each CTA owns a contiguous slice of the candidate tokens:
//
// 1. score: fp32 proxy scores of the slice into shared memory as
//    order-preserving 32-bit keys; min/max in registers;
// 2. threshold: a 4096-bin linear histogram over [min, max] (no contention,
//    one pass), per-bin totals reduced across the cluster through distributed
//    shared memory, then the bin holding the n_topk-th largest score; crowded
//    bins are refined with a second histogram over the bin's own range;
// 3. exact band: fp32 scores differ from the reference's float64 scores by at
//    most eps (a rigorous bound), so every key more than 2 eps
//    above the threshold bin is selected, every key more than 2 eps below is
//    not, and the few keys in between are rescored in float64 and ranked
//    exactly with the reference's tie rule (larger index wins);
//    degenerate inputs (huge exact-tie sets) take a float64 radix select;
// 4. output: ascending indices via cluster prefix offsets (sel_idx, counts);
// 5. (ATTEND) each CTA gathers its own selected rows -- keys from HBM, values
//    from the step-to-step HBM row cache or over PCIe by zero-copy loads, all
//    issued before any use -- runs an online softmax per warp, and the
//    partials are merged in a fixed order: warps in shared memory, CTAs over
//    DSMEM into rank 0, which writes the head outputs.
//
// No intermediate touches global memory except the selection outputs the API
// returns; the 1 MB of keys of a 128k-token head stays on chip.
#include <cooperative_groups.h>

#include <climits>
#include <string>

#include "common.cuh"
#include "sparse.cuh"

namespace cg = cooperative_groups;

#ifndef TKV_FZ_CTAS
#define TKV_FZ_CTAS 8
#endif

namespace tkv {
// This file is compiled three times (build.py): 8-CTA clusters in namespace tkv, and 4- and
// 2-CTA clusters in tkv::fz4 / tkv::fz2 for many units at shorter contexts (batch decode:
// more co-resident units per wave).
#if TKV_FZ_CTAS != 8
#define TKV_FZ_NS_(n) fz##n
#define TKV_FZ_NS(n) TKV_FZ_NS_(n)
namespace TKV_FZ_NS(TKV_FZ_CTAS) {
#endif
constexpr int FZ_CTAS = TKV_FZ_CTAS;
constexpr int FZ_THREADS = 512;
constexpr int FZ_WARPS = FZ_THREADS / 32;
constexpr int FZ_CAP = 18432;        // candidate keys per CTA: 8 CTAs cover 147,456 tokens
constexpr int FZ_NB = 512;           // linear histogram bins per pass
constexpr int FZ_REFINE = 96;        // refine the threshold bin while it holds more keys (cluster-wide)
constexpr int FZ_BAND = 256;         // per-CTA cap of float64-rescored band members
constexpr int FZ_LIST = 1536;        // per-CTA cap of the aimed candidate list
constexpr int FZ_CAND = 6144;        // cluster-wide cap of the aimed candidate list
constexpr int FZ_XBITS = 11;         // exact fallback: radix digit
constexpr int FZ_XBINS = 1 << FZ_XBITS;

__device__ __forceinline__ int fz_block_excl_scan(int v, int *sh, int *total) {
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

// exclusive block scan of a 64-bit value (packed 16-bit fields; no field overflows)
__device__ __forceinline__ unsigned long long fz_block_excl_scan64(unsigned long long v, unsigned long long *sh,
                                                                   unsigned long long *total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned long long t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    sh[lane] = t;
  }
  __syncthreads();
  const unsigned long long before = (w ? sh[w - 1] : 0ull) + x - v;
  *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before;
}

__device__ __forceinline__ uint32_t fz_orderable32(float x) {
  if (x == 0.0f) x = 0.0f;
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fz_from_orderable32(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

struct FzCtl {
  uint32_t kmin, kmax;          // this CTA's min/max orderable key
  double ksum, ksq;             // this CTA's sum and sum of squares of the fp32 scores
  int cta_count, band_count, overflow;
  int bin, inbin, status;       // threshold bin and its keys (cluster-wide); status 0 ok, -1 below, 1 above
  unsigned long long xprefix;   // exact path
  int xneed, xdone;
  unsigned long long xk[2];
  unsigned long long wk[2][32];
  double wsum[2][32];
  int scan[40];
  unsigned long long scan64[33];
  int hits, misses;  // row-cache counters of the gather (use_cache)
  int definite;      // select: candidate-list keys above the exact band
  int list_count;
  unsigned long long bar;       // mbarrier of the row staging (HBM copies on the key|value slot-cache path)
  unsigned long long bar2;      // key|value slot-cache path: the value rows fetched over PCIe
};

// dynamic shared memory
constexpr int FZ_UNION = FZ_CAP * 8;  // bytes of the phase-overlaid region (float64 keys of the exact path)
constexpr int FZ_XSTAGE = 26624;      // extra staging bytes: ~360 (K|V) rows per CTA fit one round
constexpr int FZ_STAGE = FZ_UNION + FZ_CAP + FZ_XSTAGE;  // k.raw + flags (dead after the output) + xstage
struct FzShared {
  union {
    uint64_t keys64[FZ_CAP];  // exact fallback: order-preserving float64 score keys
    struct {
      uint32_t keys32[FZ_CAP];   // fp32 order-preserving keys
      uint32_t hist[FZ_NB + 4];  // linear bins + [NB] keys above the range
      uint32_t tot[FZ_NB + 4];   // cluster totals
      unsigned long long band_key[FZ_BAND];
      uint32_t band_idx[FZ_BAND];
      union {
        struct {  // full-range path: every CTA's band members
          unsigned long long all_key[FZ_BAND * FZ_CTAS];
          uint32_t all_idx[FZ_BAND * FZ_CTAS];
        };
        unsigned long long cand[FZ_CAND];  // candidate-list path, rank 0: the cluster's candidates
      };
      unsigned long long list64[FZ_LIST];  // aimed candidates (orderable key << 32 | token index)
      uint8_t band_sel[FZ_BAND];           // rank 0: band member selected
      uint32_t bitmap[FZ_CAP / 32];        // selected band members of this CTA
    } f;
    unsigned char raw[FZ_UNION];  // attention phase: staged rows, logits, row list, partials
  } k;
  uint8_t flags[FZ_CAP];
  uint8_t xstage[FZ_XSTAGE];  // with k and flags: the gather's staging region (contiguous)
  uint32_t xhist[2][FZ_XBINS];
  uint32_t xtot[FZ_XBINS];
  float cta_m[8], cta_l[8];
  float red_m[FZ_WARPS][8], m_new[8];  // softmax: per-warp round maxima, the CTA's new max
  float cta_acc[1024];  // this CTA's merged partial, read by rank 0 over DSMEM
  float qs[1024];       // queries [G][D] * log2(e)/sqrt(d)
};

// ---------------------------------------------------------------------------
// exact fallback (float64 keys): common prefix + 11-bit radix + tie flags
// ---------------------------------------------------------------------------
__device__ void fz_common_prefix(cg::cluster_group &cluster, const uint64_t *keys, int m, FzCtl &C, int &top,
                                 unsigned long long &prefix) {
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
    C.wk[0][tid >> 5] = lo;
    C.wk[1][tid >> 5] = hi;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      lo = C.wk[0][w] < lo ? C.wk[0][w] : lo;
      hi = C.wk[1][w] > hi ? C.wk[1][w] : hi;
    }
    C.xk[0] = lo;
    C.xk[1] = hi;
  }
  cluster.sync();
  lo = ~0ull;
  hi = 0ull;
  for (int r = 0; r < FZ_CTAS; ++r) {
    const FzCtl *R = cluster.map_shared_rank(&C, r);
    lo = R->xk[0] < lo ? R->xk[0] : lo;
    hi = R->xk[1] > hi ? R->xk[1] : hi;
  }
  const int diff = lo == hi ? 0 : 64 - __clzll((long long)(lo ^ hi));
  top = diff;
  prefix = top >= 64 ? 0ull : (lo >> top) << top;
}

__device__ void fz_radix(cg::cluster_group &cluster, const uint64_t *keys, int m, FzShared &S, FzCtl &C, int &top,
                         unsigned long long &prefix, int &need, bool &done) {
  const int tid = threadIdx.x;
  done = false;
  for (int pass = 0; top > 0 && !done; ++pass) {
    const int w = top < FZ_XBITS ? top : FZ_XBITS;
    const int shift = top - w;
    const unsigned long long mask = top >= 64 ? 0ull : ~0ull << top;
    const int nb = 1 << w;
    uint32_t *H = S.xhist[pass & 1];
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
      for (int r = 0; r < FZ_CTAS; ++r) t += cluster.map_shared_rank(H, r)[b];
      S.xtot[nb - 1 - b] = t;  // descending-bin order
    }
    __syncthreads();
    const int bpt = (nb + (int)blockDim.x - 1) / (int)blockDim.x;  // bins per thread
    int v = 0;
    for (int p2 = tid * bpt; p2 < tid * bpt + bpt && p2 < nb; ++p2) v += (int)S.xtot[p2];
    int total;
    const int before = fz_block_excl_scan(v, C.scan, &total);
    if (before < need && before + v >= need) {
      int cum = before;
      for (int p2 = tid * bpt; p2 < tid * bpt + bpt && p2 < nb; ++p2) {
        const int c = (int)S.xtot[p2];
        if (cum + c >= need) {
          C.xneed = need - cum;
          C.xprefix = prefix | ((unsigned long long)(nb - 1 - p2) << shift);
          C.xdone = c == need - cum;
          break;
        }
        cum += c;
      }
    }
    __syncthreads();
    prefix = C.xprefix;
    need = C.xneed;
    done = C.xdone;
    top = shift;
  }
}

__device__ void fz_exact_flags(cg::cluster_group &cluster, const uint64_t *keys, int m, uint8_t *flags, FzCtl &C,
                               int top, unsigned long long prefix, int need, bool done) {
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
  fz_block_excl_scan(ties, C.scan, &tot_ties);
  if (tid == 0) C.cta_count = tot_ties;
  cluster.sync();
  int above = 0;
  for (int r = rank + 1; r < FZ_CTAS; ++r) above += cluster.map_shared_rank(&C, r)->cta_count;
  const int allowed = max(0, min(tot_ties, need - above));
  const int per = (m + FZ_THREADS - 1) / FZ_THREADS;
  const int b0 = tid * per, b1 = min(m, b0 + per);
  int mine = 0;
  for (int e = b0; e < b1; ++e) mine += flags[e] == 2;
  int dummy;
  const int before = fz_block_excl_scan(mine, C.scan, &dummy);
  int higher = tot_ties - before - mine;  // ties at indices above this thread's range
  for (int e = b1 - 1; e >= b0; --e) {
    if (flags[e] == 2) {
      flags[e] = higher < allowed ? 1 : 0;
      ++higher;
    }
  }
  cluster.sync();  // cta_count reads complete before reuse
}

__device__ __forceinline__ double fz_exact_score(const uint16_t *kt, int64_t cap, const int *chs, const double *qsum,
                                                 int d_s, int64_t j) {
  double sc = 0.0;
  for (int i = 0; i < d_s; ++i) sc = fma(h2d(kt[(size_t)chs[i] * cap + j]), qsum[i], sc);
  return sc;
}

// cluster-wide min/max (orderable keys) and sum / sum of squares of the scores
// this CTA's min/max key and score moments into C (for the cluster or for rank 0)
__device__ __forceinline__ void fz_block_stats(FzCtl &C, uint32_t lo, uint32_t hi, double sum, double sq) {
  const int tid = threadIdx.x, lane = tid & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    sq += __shfl_xor_sync(0xffffffffu, sq, o);
  }
  if (lane == 0) {
    C.wk[0][tid >> 5] = lo;
    C.wk[1][tid >> 5] = hi;
    C.wsum[0][tid >> 5] = sum;
    C.wsum[1][tid >> 5] = sq;
  }
  __syncthreads();
  if (tid < 32) {
    const bool ok = tid < (int)(blockDim.x >> 5);
    uint32_t a = ok ? (uint32_t)C.wk[0][tid] : 0xffffffffu, b = ok ? (uint32_t)C.wk[1][tid] : 0u;
    double x = ok ? C.wsum[0][tid] : 0.0, y = ok ? C.wsum[1][tid] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
      x += __shfl_xor_sync(0xffffffffu, x, o);
      y += __shfl_xor_sync(0xffffffffu, y, o);
    }
    if (tid == 0) {
      C.kmin = a;
      C.kmax = b;
      C.ksum = x;
      C.ksq = y;
    }
  }
}

__device__ __forceinline__ void fz_cluster_stats(cg::cluster_group &cluster, FzCtl &C, uint32_t lo, uint32_t hi,
                                                 double sum, double sq, uint32_t &glo, uint32_t &ghi, double &gsum,
                                                 double &gsq) {
  fz_block_stats(C, lo, hi, sum, sq);
  cluster.sync();
  glo = 0xffffffffu;
  ghi = 0u;
  gsum = 0.0;
  gsq = 0.0;
#pragma unroll
  for (int r = 0; r < FZ_CTAS; ++r) {
    const FzCtl *R = cluster.map_shared_rank(&C, r);
    glo = min(glo, R->kmin);
    ghi = max(ghi, R->kmax);
    gsum += R->ksum;
    gsq += R->ksq;
  }
}

// upper-tail standard normal quantile: z with P(Z > z) = p (Acklam's rational
// approximation, |rel err| < 1.2e-9 -- only used to aim the first histogram)
__device__ double fz_normal_upper_quantile(double p) {
  const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                       1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                       6.680131188771972e+01, -1.328068155288572e+01};
  const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                       -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00, 3.754408661907416e+00};
  const double q0 = fmin(fmax(1.0 - p, 1e-12), 1.0 - 1e-12);  // lower-tail probability
  double x;
  if (q0 < 0.02425) {
    const double q = sqrt(-2.0 * log(q0));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  } else if (q0 <= 1.0 - 0.02425) {
    const double q = q0 - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  } else {
    const double q = sqrt(-2.0 * log(1.0 - q0));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  return x;
}

// 16-byte read-only load that stays where it is written (issued before the
// barrier that follows it, so its latency overlaps the next global round trip)
__device__ __forceinline__ uint4 fz_ld_nc_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Keys live in the scorer's layout: thread t owns the 8-key groups starting
// at g*STEP + 8t (g < FZ_KG).  Passes over them read 8 keys with two 16-byte
// shared loads (a per-key loop at 16 warps/SM is shared-memory-latency bound).
constexpr int FZ_STEP = FZ_THREADS * 8;
constexpr int FZ_KG = (FZ_CAP + FZ_STEP - 1) / FZ_STEP;
__device__ __forceinline__ void fz_load8(const uint32_t *keys, int e, int m, uint32_t kk[8]) {
  if (e + 8 <= m) {
    const uint4 a = *reinterpret_cast<const uint4 *>(keys + e), b = *reinterpret_cast<const uint4 *>(keys + e + 4);
    kk[0] = a.x; kk[1] = a.y; kk[2] = a.z; kk[3] = a.w;
    kk[4] = b.x; kk[5] = b.y; kk[6] = b.z; kk[7] = b.w;
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) kk[q] = e + q < m ? keys[e + q] : 0u;
  }
}

// mbarrier + TMA bulk copy helpers (value-row staging)
__device__ __forceinline__ uint32_t fz_smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void fz_mbar_init(unsigned long long *bar) {
  asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(fz_smem_addr(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fz_mbar_expect(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(fz_smem_addr(bar)), "r"(bytes) : "memory");
}
// add bytes to the current phase's transaction count (no arrival; one thread arrives once all are queued)
__device__ __forceinline__ void fz_mbar_expect_only(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(fz_smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fz_mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(fz_smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void fz_mbar_wait(unsigned long long *bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n FZW_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra FZW_%=;\n}\n" ::"r"(
          fz_smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fz_bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   fz_smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(fz_smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void fz_bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(fz_smem_addr(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fz_bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
}

// phase timestamps of unit 0, every CTA (debug: tkv_debug_sparse_phases)
constexpr int FZ_NMARK = 40;
// stage-1 handshake wait, bounded (~2 s): a missing signal becomes an error flag, never a hang
__device__ unsigned g_fz_s1_timeout = 0;
__device__ __forceinline__ void fz_wait_ready(const int32_t *flag) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
  if (v) return;
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(100);
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (!v && t - t0 > 2000000000ull) {
      atomicExch(&g_fz_s1_timeout, 1u);
      return;
    }
  } while (!v);
}

__device__ unsigned long long g_fz_phase[FZ_CTAS][FZ_NMARK];
__device__ int g_fz_trace;  // set by tkv_debug_sparse_trace
__device__ double g_fz_dbg[2][8];  // list-path attempts of unit 0 (debug)
__device__ unsigned long long g_fz_clk[FZ_CTAS][2];  // clock64 at the first and last mark (debug)
__device__ unsigned long long g_fz_unit[64][FZ_CTAS][2];  // per unit and rank: globaltimer at start / end (debug)
__device__ unsigned long long g_fz_launch[128][3];  // unit 0, rank 0, per launch: start, after the PDL wait, end (debug)
__device__ unsigned int g_fz_nlaunch;
__device__ int g_fz_upath[64][4];  // per unit: select path (0 list attempt 0, 1 list attempt 1, 2 full range), list size, rows, misses
__device__ unsigned int g_fz_pathcnt[4];  // launches x units per select path (trace mode)
__device__ float g_fz_aim = 0.0f;         // tuning: fixed half-width of the first aimed range (sd); 0 = adaptive

// The threshold hint of a (layer, head), float4: x the last top-k threshold
// as a z-score of that step's scores, y a running mean of its step-to-step
// change (the z-score is what stays stable: the scores' mean and spread move
// with the query; an absolute hint drifts several times faster).
__device__ __forceinline__ void fz_store_hint(float *th, float4 old, double z) {
  const float dz = isfinite(old.x) ? (float)fabs(z - (double)old.x) : __int_as_float(0x7fc00000);
  th[1] = isfinite(old.y) ? (isfinite(dz) ? 0.75f * old.y + 0.25f * dz : old.y) : dz;
  th[0] = (float)z;
}
#define FZ_MARK(i)                                                          \
  do {                                                                      \
    if (trace && blockIdx.y == 0 && tid == 0) {                             \
      unsigned long long t_;                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
      g_fz_phase[rank][i] = t_;                                             \
    }                                                                       \
  } while (0)

template <bool ATTEND, int D, int GMAX>
__global__ void __launch_bounds__(FZ_THREADS, 1)
    sparse_fused_kernel(SL s, const uint16_t *__restrict__ queries, int G, const int32_t *__restrict__ channels,
                        int d_s, int n_local, int n_topk, int32_t *__restrict__ sel_idx, int sel_stride,
                        int32_t *__restrict__ sel_count, int32_t *__restrict__ fetch_count,
                        double *__restrict__ scores_out, int keys_from_device, float *__restrict__ out,
                        const uint16_t *__restrict__ new_keys, const uint16_t *__restrict__ new_values) {
  extern __shared__ __align__(16) unsigned char smem[];
  FzShared &S = *reinterpret_cast<FzShared *>(smem);
  __shared__ FzCtl C;
  // attention sinks (extension, s.n_sink = 0 for the reference): their keys are forced above every
  // score, so the n_topk + n_sink best candidates are the sinks plus the n_topk best of the rest
  const int n_sink = s.n_sink;
  n_topk += n_sink;
  __shared__ double qsum[128];
  __shared__ float qsum32[128];
  __shared__ int chs[128];
  __shared__ double band_eps;
  __shared__ double eps_term[128];
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int u = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = *s.len;
  const int trace = g_fz_trace;
  const float qnan = __int_as_float(0x7fc00000);
  const float aim_fixed = g_fz_aim;
  const float4 hint = s.thresh ? *reinterpret_cast<const float4 *>(s.thresh + 4 * (size_t)u) : make_float4(qnan, qnan, qnan, qnan);
  int32_t *out_idx = sel_idx + (size_t)u * sel_stride;
  const bool select_all = n <= (int64_t)n_local + n_topk;  // retriever.py:204-205
  const int64_t ncand = n > n_local ? n - n_local : 0;     // local window starts here
  const int64_t chunk = ((ncand + FZ_CTAS - 1) / FZ_CTAS + 15) & ~int64_t(15);
  const int64_t j0 = rank * chunk;
  const int m = (int)(j0 < ncand ? imin64(chunk, ncand - j0) : 0);
  uint8_t *flags = S.flags;
  const uint16_t *kt = s.kt + (size_t)u * s.d * s.capacity;
  FZ_MARK(0);
  if (trace && blockIdx.y == 0 && tid == 0) g_fz_clk[rank][0] = clock64();
  __shared__ unsigned int lslot;
  if (trace && blockIdx.y < 64 && tid == 0) {
    unsigned long long t_;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
    g_fz_unit[blockIdx.y][rank][0] = t_;
    if (blockIdx.y == 0 && rank == 0) {
      lslot = atomicAdd(&g_fz_nlaunch, 1u) & 127u;
      g_fz_launch[lslot][0] = t_;
    }
  }
  if (tid == 0) {
    C.band_count = 0;
    C.overflow = 0;
    C.hits = 0;
    C.misses = 0;
    if (ATTEND) {
      fz_mbar_init(&C.bar);
      fz_mbar_init(&C.bar2);
    }
  }
  // The step's new row goes to the pinned host store now, not in the final append: nothing reads row
  // n during this step (attend before append), and a posted PCIe store still in flight when the grid
  // ends delays its completion -- and the next layer's PDL wait -- by ~3.5 us (tools/pdl_probe.cu).
  if (ATTEND && new_keys && rank == FZ_CTAS - 1 && tid < 2 * D / 8) {
    const int half = tid / (D / 8), c8 = (tid % (D / 8)) * 8;  // 16-byte pieces of K then V
    const uint16_t *src = (half ? new_values : new_keys) + (size_t)u * D + c8;
    *reinterpret_cast<uint4 *>(s.host_kv + (((size_t)u * s.capacity + n) * 2 + half) * D + c8) =
        *reinterpret_cast<const uint4 *>(src);
  }
  // stage-1 handshake (tkv_sparse_layer.s1_ready): wait until this unit's channels are written
  if (ATTEND && s.s1_ready) {
    if (tid == 0) fz_wait_ready(&s.s1_ready[u]);
    __syncthreads();
  }
  bool listed = false;                 // candidate-list path: flags come from keys32 + bitmap
  uint32_t ord_def = 0xffffffffu;      // (list path) keys above this orderable value are selected
  if (select_all) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int e = tid; e < m; e += blockDim.x) flags[e] = 1;
    __syncthreads();
  } else {
    for (int i = tid; i < d_s; i += blockDim.x) chs[i] = channels[(size_t)u * d_s + i];
    __syncthreads();
    FZ_MARK(1);
    // ---- 1. fp32 proxy scores (retriever.py:189) -> order-preserving keys ----
    // Every thread issues its first two 8-token groups of scorer loads before
    // the group-summed query is formed: the two round trips overlap.
    uint32_t *keys32 = S.k.f.keys32;
    uint32_t klo = 0xffffffffu, khi = 0u;
    float fsum = 0.0f, fsq = 0.0f;
    const bool fast8 = (d_s & 7) == 0;
    constexpr int STEP = FZ_THREADS * 8;
    uint4 v[2][8];
    int e0 = tid * 8;
    if (fast8) {
#pragma unroll
      for (int g2 = 0; g2 < 2; ++g2)
        if (e0 + g2 * STEP + 8 <= m) {
#pragma unroll
          for (int r = 0; r < 8; ++r) v[g2][r] = fz_ld_nc_v4(kt + (size_t)chs[r] * s.capacity + j0 + e0 + g2 * STEP);
        }
    }
    // Programmatic dependent launch: everything above (length, channels, the
    // first scorer loads) only touches this layer's own state, so it overlaps
    // the previous kernel's tail; the query is consumed after the wait.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (trace && blockIdx.y == 0 && rank == 0 && tid == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      g_fz_launch[lslot][1] = t_;
    }
    for (int i = tid; i < d_s; i += blockDim.x) {
      const int ch = chs[i];
      double q = 0.0;
      for (int j = 0; j < G; ++j) q += h2d(queries[((size_t)u * G + j) * s.d + ch]);  // group sum (retriever.py:189)
      qsum[i] = q;
      qsum32[i] = (float)q;
      // |fp32 score - float64 score| <= (d_s + 2) 2^-24 sum_i max|K_i| |q_i| (see band_eps)
      eps_term[i] = (double)s.chmax[(size_t)u * s.d + ch] * fabs(q);
    }
    __syncthreads();
    FZ_MARK(2);
    for (; e0 < m; e0 += 2 * STEP) {
#pragma unroll
      for (int g2 = 0; g2 < 2; ++g2) {
        const int eg = e0 + g2 * STEP;
        if (eg >= m) break;
        const int64_t j = j0 + eg;
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
        int i = 0;
        if (fast8 && eg + 8 <= m) {
          for (; i < d_s; i += 8) {
            if (i > 0) {  // channel group 0 of every round was prefetched
#pragma unroll
              for (int r = 0; r < 8; ++r) v[g2][r] = fz_ld_nc_v4(kt + (size_t)chs[i + r] * s.capacity + j);
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const float qv = qsum32[i + r];
              const uint32_t w[4] = {v[g2][r].x, v[g2][r].y, v[g2][r].z, v[g2][r].w};
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[e] = fmaf(h2f((uint16_t)(w[e >> 1] >> (16 * (e & 1)))), qv, acc[e]);
            }
          }
        }
        for (; i < d_s; ++i) {
          const uint16_t *row = kt + (size_t)chs[i] * s.capacity + j;
          const float qv = qsum32[i];
          for (int e = 0; e < 8 && eg + e < m; ++e) acc[e] = fmaf(h2f(row[e]), qv, acc[e]);
        }
        uint32_t kk[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const bool sink = j + e < n_sink;
          kk[e] = sink ? 0xffffffffu : fz_orderable32(acc[e]);
          if (eg + e < m && !sink) {
            klo = min(klo, kk[e]);
            khi = max(khi, kk[e]);
            fsum += acc[e];
            fsq = fmaf(acc[e], acc[e], fsq);
          }
        }
        if (eg + 8 <= m) {  // two 16-byte stores (no 8-way bank conflicts)
          uint4 *dst = reinterpret_cast<uint4 *>(keys32 + eg);
          dst[0] = make_uint4(kk[0], kk[1], kk[2], kk[3]);
          dst[1] = make_uint4(kk[4], kk[5], kk[6], kk[7]);
        } else {
          for (int e = 0; e < 8 && eg + e < m; ++e) keys32[eg + e] = kk[e];
        }
      }
      if (fast8 && e0 + 2 * STEP < m) {  // next round's first channel group
#pragma unroll
        for (int g2 = 0; g2 < 2; ++g2)
          if (e0 + 2 * STEP + g2 * STEP + 8 <= m) {
#pragma unroll
            for (int r = 0; r < 8; ++r)
              v[g2][r] = fz_ld_nc_v4(kt + (size_t)chs[r] * s.capacity + j0 + e0 + 2 * STEP + g2 * STEP);
          }
      }
    }
    if (tid == 0) {
      double e = 0.0;
      for (int i = 0; i < d_s; ++i) e += eps_term[i];
      // a d_s-term fmaf chain plus the fp32 rounding of the query: <= (d_s + 1) roundings of
      // 2^-24 relative to sum_i max|K_i| |q_i|; (d_s + 2) leaves margin, 16 keeps the tuned band
      band_eps = e * fmax(16.0, (double)d_s + 2.0) * 5.9604644775390625e-08;  // x 2^-24
    }
    FZ_MARK(3);
    uint32_t glo, ghi;
    double gsum, gsq;
    fz_cluster_stats(cluster, C, klo, khi, (double)fsum, (double)fsq, glo, ghi, gsum, gsq);
    FZ_MARK(4);
    // ---- 2a. aimed candidate list, resolved by one CTA ----
    // Aim at the previous step's threshold of this (layer, head), +-3x its
    // usual step-to-step move, else at the Gaussian estimate mean + z sd (+-0.2 sd).  One pass with no
    // per-key atomics: keys above the aimed range are counted, keys inside it
    // (widened by 2 eps) are appended as (key, index) pairs through
    // warp-aggregated positions.  Rank 0 gathers the cluster's short list
    // over DSMEM and finds the exact selection alone (fp32 radix select of the
    // threshold, float64 rescoring of the +-2 eps band, reference tie rule),
    // so the whole search costs two cluster barriers.  Each CTA then derives
    // its flags from one integer compare plus the selected band members.  If
    // the aim misses or a list overflows, the full-range path below runs.
    const double flo = (double)fz_from_orderable32(glo), fhi = (double)fz_from_orderable32(ghi);
    const double eps2 = 2.0 * band_eps;
    uint32_t *H = S.k.f.hist;  // [NB] bins + [NB] keys above the range
    uint32_t *T = S.k.f.tot;   // cluster totals
    unsigned long long *list = S.k.f.list64;
    {
      const double N = (double)(ncand - imin64(ncand, n_sink)), mu = gsum / N, var = fmax(gsq / N - mu * mu, 0.0), sd = sqrt(var);
      const bool hinted = isfinite(hint.x);
      // the Gaussian estimate of the threshold (only without a hint or after an overflow)
      auto gauss = [&]() { return mu + fz_normal_upper_quantile((double)(n_topk - n_sink) / N) * sd; };
      const double tprev = mu + (double)hint.x * sd;
      double last_lo = 0.0, last_hi = 0.0;
      int dir = 0;
      for (int attempt = 0; attempt < 2 && !listed; ++attempt) {
        // attempt 0 spans the previous threshold (or the Gaussian estimate); after a
        // miss, attempt 1 extends 0.6 sd beyond the side of the missed range that holds the threshold
        double a_lo, a_hi;
        if (attempt == 0) {
          // +-(3 x the usual step-to-step move of the threshold), within [0.03, 0.25] sd
          const double w = !hinted ? 0.2
                           : aim_fixed > 0.0f ? (double)aim_fixed
                           : isfinite(hint.y) ? fmin(0.25, fmax(0.03, 3.0 * (double)hint.y)) : 0.1;
          const double c = hinted ? tprev : gauss();
          a_lo = c - w * sd;
          a_hi = c + w * sd;
        } else if (dir > 0) {
          a_lo = last_hi;
          a_hi = last_hi + 0.6 * sd;
        } else if (dir < 0) {
          a_lo = last_lo - 0.6 * sd;
          a_hi = last_lo;
        } else {  // a list overflowed
          const double gs = gauss();
          a_lo = gs - 0.4 * sd;
          a_hi = gs + 0.4 * sd;
        }
        if (!(sd > 0.0) || !isfinite(a_lo) || !isfinite(a_hi)) break;
        const double center = 0.5 * (a_lo + a_hi), width = 0.5 * (a_hi - a_lo);
        a_lo = fmax(flo, a_lo);
        a_hi = fmin(fhi, a_hi);
        last_lo = a_lo;
        last_hi = a_hi;
        if (!(a_hi > a_lo)) continue;
        // the list spans the aimed range plus two band widths, so the final band always lies inside it
        const uint32_t ord_llo = fz_orderable32(__double2float_rd(a_lo - 2.0 * eps2));
        const uint32_t ord_lhi = fz_orderable32(__double2float_ru(a_hi + 2.0 * eps2));
        if (tid == 0) C.list_count = 0;
        __syncthreads();
        FZ_MARK(9);
        int above = 0, c = 0;
        uint32_t cm[FZ_KG];
#pragma unroll
        for (int g = 0; g < FZ_KG; ++g) {
          const int e = g * FZ_STEP + tid * 8;
          uint32_t kk[8];
          if (e < m) fz_load8(keys32, e, m, kk);
          uint32_t cmask = 0u;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const bool valid = e + q < m;
            above += valid && kk[q] > ord_lhi;
            cmask |= (uint32_t)(valid && kk[q] >= ord_llo && kk[q] <= ord_lhi) << q;
          }
          cm[g] = cmask;
          c += __popc(cmask);
        }
        // one warp-aggregated slot reservation for all of this thread's candidates
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int wtot = __shfl_sync(0xffffffffu, incl, 31);
        int base = 0;
        if (lane == 31 && wtot) base = atomicAdd(&C.list_count, wtot);
        int pos = __shfl_sync(0xffffffffu, base, 31) + incl - c;
#pragma unroll
        for (int g = 0; g < FZ_KG; ++g) {
          const int e = g * FZ_STEP + tid * 8;
          uint32_t cmask = cm[g];
          while (cmask) {
            const int q = __ffs(cmask) - 1;
            cmask &= cmask - 1u;
            if (pos < FZ_LIST) list[pos] = ((unsigned long long)keys32[e + q] << 32) | (uint32_t)(j0 + e + q);
            ++pos;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) above += __shfl_xor_sync(0xffffffffu, above, o);
        if (lane == 0) C.wk[0][warp] = (unsigned long long)above;
        __syncthreads();
        if (tid == 0) {
          int t = 0;
          for (int w = 0; w < FZ_WARPS; ++w) t += (int)C.wk[0][w];
          C.cta_count = t;
        }
        FZ_MARK(5);
        cluster.sync();  // #1: every CTA's list and counts are complete
        FZ_MARK(6);
        if (rank == 0) {
          // ---- rank 0: gather, fp32 radix select, float64 band, exact ranking ----
          int A = 0, L = 0, ovf = 0, Lr[FZ_CTAS];
#pragma unroll
          for (int r = 0; r < FZ_CTAS; ++r) {
            const FzCtl *R = cluster.map_shared_rank(&C, r);
            A += R->cta_count;
            Lr[r] = R->list_count;
            ovf |= Lr[r] > FZ_LIST;
            L += Lr[r];
          }
          const int need = n_topk - A;
          int verdict = (ovf || L > FZ_CAND || need <= 0 || need > L) ? 0 : 1;
          int dir = need <= 0 ? 1 : (!ovf && need > L ? -1 : 0);  // where the threshold lies if the aim missed
          if (trace && blockIdx.y == 0 && tid == 0) {
            g_fz_dbg[attempt][0] = attempt; g_fz_dbg[attempt][1] = A; g_fz_dbg[attempt][2] = L;
            g_fz_dbg[attempt][3] = need; g_fz_dbg[attempt][4] = verdict; g_fz_dbg[attempt][5] = center;
            g_fz_dbg[attempt][6] = width; g_fz_dbg[attempt][7] = sd;
          }
          unsigned long long *cand = S.k.f.cand;
          if (verdict) {
            for (int t = tid; t < L; t += blockDim.x) {
              int r = 0, base = 0, run = 0;
#pragma unroll
              for (int k = 0; k < FZ_CTAS - 1; ++k) {  // (static indices keep Lr in registers)
                run += Lr[k];
                if (t >= run) {
                  r = k + 1;
                  base = run;
                }
              }
              cand[t] = cluster.map_shared_rank(list, r)[t - base];
            }
            __syncthreads();
            FZ_MARK(7);
            // one 512-bin linear histogram over the list's range: the bin holding
            // the need-th largest key bounds the threshold to [e_lo, e_hi]
            const float r_lo = __double2float_rd(a_lo), r_hi = __double2float_ru(a_hi);
            const float scale = (float)FZ_NB / (r_hi - r_lo);
            const uint32_t o_lo = fz_orderable32(r_lo), o_hi = fz_orderable32(r_hi);
            for (int i = tid; i <= FZ_NB; i += blockDim.x) H[i] = 0;
            __syncthreads();
            int ab = 0;
            for (int t = tid; t < L; t += blockDim.x) {
              const uint32_t k = (uint32_t)(cand[t] >> 32);
              if (k > o_hi) {
                ++ab;
              } else if (k >= o_lo) {
                const float x = fz_from_orderable32(k);
                atomicAdd(&H[min(FZ_NB - 1, max(0, (int)((x - r_lo) * scale)))], 1u);
              }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ab += __shfl_xor_sync(0xffffffffu, ab, o);
            if (lane == 0 && ab) atomicAdd(&H[FZ_NB], (unsigned)ab);
            if (tid == 0) C.bin = -1;
            __syncthreads();
            const int need2 = need - (int)H[FZ_NB];  // list members above the aimed range are selected
            if (warp == 0 && need2 > 0) {
              constexpr int BPL = FZ_NB / 32;
              int cl = 0;
#pragma unroll
              for (int q = 0; q < BPL; ++q) cl += (int)H[FZ_NB - 1 - BPL * lane - q];
              int incl = cl;
#pragma unroll
              for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
              }
              int before = incl - cl;
              const unsigned hit = __ballot_sync(0xffffffffu, before < need2 && incl >= need2);
              if (hit && lane == __ffs(hit) - 1) {
                for (int q = 0; q < BPL; ++q) {
                  const int b = FZ_NB - 1 - BPL * lane - q;
                  if (before + (int)H[b] >= need2) {
                    C.bin = b;
                    break;
                  }
                  before += (int)H[b];
                }
              }
            }
            __syncthreads();
            FZ_MARK(8);
            const int B = max(0, C.bin);
            if (C.bin < 0) {  // the aim missed: the threshold lies outside [a_lo, a_hi]
              verdict = 0;
              dir = need2 <= 0 ? 1 : -1;
            }
            const double delta = 9.5367431640625e-07 * (fabs((double)r_lo) + fabs((double)r_hi) + ((double)r_hi - r_lo));
            const double e_lo = B == 0 ? (double)r_lo : (double)r_lo + (double)B / (double)scale - delta;
            const double e_hi = B == FZ_NB - 1 ? (double)r_hi : (double)r_lo + (double)(B + 1) / (double)scale + delta;
            const double T32 = 0.5 * (e_lo + e_hi);
            const uint32_t ord_hi = fz_orderable32(__double2float_ru(e_hi + eps2));
            const uint32_t ord_lo = fz_orderable32(__double2float_rd(e_lo - eps2));
            if (tid == 0) {
              C.band_count = 0;
              C.overflow = 0;
              C.definite = 0;  // keys of the list above the band
            }
            __syncthreads();
            int def = 0;
            for (int t = tid; t < L; t += blockDim.x) {
              const uint32_t k = (uint32_t)(cand[t] >> 32);
              if (k > ord_hi) {
                ++def;
              } else if (k >= ord_lo) {
                const int slot = atomicAdd(&C.band_count, 1);
                if (slot < FZ_BAND) S.k.f.band_idx[slot] = (uint32_t)cand[t];
                else C.overflow = 1;
              }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) def += __shfl_xor_sync(0xffffffffu, def, o);
            if (lane == 0 && def) atomicAdd(&C.definite, def);
            __syncthreads();
            const int nb = min(C.band_count, FZ_BAND);
            const int need_b = n_topk - A - C.definite;
            if (!verdict || C.overflow || need_b < 0 || need_b > nb) {
              verdict = 0;  // the aim missed (or a band overflow): take the next attempt / full-range path
            } else {
              for (int b = tid; b < nb; b += blockDim.x)
                S.k.f.band_key[b] = orderable(fz_exact_score(kt, s.capacity, chs, qsum, d_s, S.k.f.band_idx[b]));
              __syncthreads();
              for (int b = tid; b < nb; b += blockDim.x) {
                const unsigned long long kb = S.k.f.band_key[b];
                const uint32_t ib = S.k.f.band_idx[b];
                int beaten = 0;
                for (int o = 0; o < nb; ++o) {
                  const unsigned long long ko = S.k.f.band_key[o];
                  const uint32_t io = S.k.f.band_idx[o];
                  beaten += (ko > kb) || (ko == kb && io > ib);  // (score desc, index desc)
                }
                S.k.f.band_sel[b] = beaten < need_b ? 1 : 0;
              }
              if (tid == 0) {
                C.xprefix = ord_hi;  // keys above this orderable value are selected
                if (s.thresh && sd > 0.0) fz_store_hint(s.thresh + 4 * u, hint, (T32 - mu) / sd);
              }
            }
          }
          if (tid == 0) {
            C.status = verdict;
            C.inbin = dir;  // (reused) miss direction for the next attempt
          }
          FZ_MARK(21);
        }
        cluster.sync();  // #2: rank 0's verdict, threshold and band are ready
        FZ_MARK(22);
        const FzCtl *R0 = cluster.map_shared_rank(&C, 0);
        dir = R0->status ? 0 : R0->inbin;
        if (trace && blockIdx.y < 64 && rank == 0 && tid == 0 && R0->status) {
          g_fz_upath[blockIdx.y][0] = attempt;
          g_fz_upath[blockIdx.y][1] = R0->list_count;
          atomicAdd(&g_fz_pathcnt[attempt], 1u);
        }
        if (R0->status) {
          ord_def = (uint32_t)R0->xprefix;
          for (int i = tid; i < FZ_CAP / 32; i += blockDim.x) S.k.f.bitmap[i] = 0u;
          __syncthreads();
          const FzShared *S0 = cluster.map_shared_rank(&S, 0);
          const int nb = min(R0->band_count, FZ_BAND);
          for (int b = tid; b < nb; b += blockDim.x) {
            const int64_t ib = S0->k.f.band_idx[b];
            if (S0->k.f.band_sel[b] && ib >= j0 && ib < j0 + m)
              atomicOr(&S.k.f.bitmap[(ib - j0) >> 5], 1u << ((ib - j0) & 31));
          }
          listed = true;
        }
        __syncthreads();
        FZ_MARK(23);
        if (!listed) cluster.sync();  // rank 0's reads of the lists are over before they are rebuilt
      }
    }
    if (!listed) {
    if (trace && blockIdx.y < 64 && rank == 0 && tid == 0) {
      g_fz_upath[blockIdx.y][0] = 2;
      atomicAdd(&g_fz_pathcnt[2], 1u);
    }
    // ---- 2b. threshold range by linear histograms (full range) ----
    if (tid == 0) {
      C.band_count = 0;
      C.overflow = 0;
    }
    __syncthreads();
    // Invariant kept by every accepted pass: #{score > R_hi} < n_topk <= #{score >= R_lo}.
    // Pass 0 aims at the Gaussian estimate of the n_topk-th score (mean + z sd,
    // +-0.6 sd); only keys inside the aimed range touch the histogram.  A
    // pass whose range misses the threshold falls back to the full range.
    double R_lo = flo, R_hi = fhi;
    {
      const double N = (double)(ncand - imin64(ncand, n_sink)), mu = gsum / N, var = fmax(gsq / N - mu * mu, 0.0), sd = sqrt(var);
      const double z = fz_normal_upper_quantile((double)(n_topk - n_sink) / N);
      const double t = mu + z * sd;
      if (sd > 0.0 && isfinite(t)) {
        R_lo = fmax(flo, t - 0.6 * sd);
        R_hi = fmin(fhi, t + 0.6 * sd);
        if (!(R_hi > R_lo)) {
          R_lo = flo;
          R_hi = fhi;
        }
      }
    }
    bool aimed = R_lo > flo || R_hi < fhi;
    for (int pass = 0; pass < 5; ++pass) {
      const float r_lo = __double2float_rd(R_lo), r_hi = __double2float_ru(R_hi);
      const float scale = (float)FZ_NB / (r_hi - r_lo);
      if (!(r_hi > r_lo) || !(scale < 3.0e38f)) break;  // degenerate range: everything in it is band
      for (int i = tid; i < FZ_NB + 4; i += blockDim.x) H[i] = 0;
      __syncthreads();
      int above = 0;
      const uint32_t ord_lo = fz_orderable32(r_lo), ord_hi = fz_orderable32(r_hi), ord_w = ord_hi - ord_lo;
#pragma unroll 1
      for (int g = 0; g < FZ_KG; ++g) {
        const int e = g * FZ_STEP + tid * 8;
        if (e >= m) break;
        uint32_t kk[8];
        fz_load8(keys32, e, m, kk);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const bool valid = e + q < m;
          above += valid && kk[q] > ord_hi;                         // integer compares on the orderable keys
          if (valid && kk[q] - ord_lo <= ord_w) {                   // inside [r_lo, r_hi] (rare when aimed)
            const float x = fz_from_orderable32(kk[q]);
            const int b = min(FZ_NB - 1, max(0, (int)((x - r_lo) * scale)));
            atomicAdd(&H[b], 1u);
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) above += __shfl_xor_sync(0xffffffffu, above, o);
      if (lane == 0 && above) atomicAdd(&H[FZ_NB], (unsigned)above);
      if (pass == 0) FZ_MARK(5);
      cluster.sync();
      if (pass == 0) FZ_MARK(6);
      // cluster totals: 16-byte DSMEM reads (DSMEM moves ~20 B/clk per SM)
      if (tid < (FZ_NB + 4) / 4) {
        uint4 t = make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int r = 0; r < FZ_CTAS; ++r) {
          const uint4 x = reinterpret_cast<const uint4 *>(cluster.map_shared_rank(H, r))[tid];
          t.x += x.x; t.y += x.y; t.z += x.z; t.w += x.w;
        }
        reinterpret_cast<uint4 *>(T)[tid] = t;
      }
      __syncthreads();
      if (pass == 0) FZ_MARK(7);
      if (warp == 0) {
        // descending scan by one warp: lane l owns bins NB-1-BPL*l .. NB-BPL-BPL*l
        const int need = n_topk - (int)T[FZ_NB];
        constexpr int BPL = FZ_NB / 32;
        int cl = 0;
#pragma unroll
        for (int q = 0; q < BPL; ++q) cl += (int)T[FZ_NB - 1 - BPL * lane - q];
        int incl = cl;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int in_range = __shfl_sync(0xffffffffu, incl, 31);
        int before = incl - cl;
        if (need <= 0) {
          if (lane == 0) C.status = 1;  // threshold above the range
        } else if (in_range < need) {
          if (lane == 0) C.status = -1;  // threshold below the range
        } else {
          const unsigned hit = __ballot_sync(0xffffffffu, before < need && incl >= need);
          if (lane == __ffs(hit) - 1) {
            for (int q = 0; q < BPL; ++q) {
              const int b = FZ_NB - 1 - BPL * lane - q;
              const int c = (int)T[b];
              if (before + c >= need) {
                C.bin = b;
                C.inbin = c;
                break;
              }
              before += c;
            }
            C.status = 0;
          }
        }
      }
      __syncthreads();
      if (pass == 0) FZ_MARK(8);
      const int status = C.status, B = C.bin, inbin = C.inbin;
      if (status != 0) {
        // the aimed range missed the threshold: widen it to the side that holds it
        if (status > 0) R_lo = R_hi; else R_hi = R_lo;
        R_lo = status > 0 ? R_lo : flo;
        R_hi = status > 0 ? fhi : R_hi;
        aimed = false;
        cluster.sync();  // every CTA has read this CTA's histogram before it is cleared
        continue;
      }
      // bin B's value range, widened by a rounding margin, clamped to the current range
      const double delta = 9.5367431640625e-07 * (fabs((double)r_lo) + fabs((double)r_hi) + ((double)r_hi - r_lo));
      const double e_lo = B == 0 ? (double)r_lo : (double)r_lo + (double)B / (double)scale - delta;
      const double e_hi = B == FZ_NB - 1 ? (double)r_hi : (double)r_lo + (double)(B + 1) / (double)scale + delta;
      R_lo = fmax(R_lo, e_lo);
      R_hi = fmin(R_hi, e_hi);
      if (inbin <= FZ_REFINE || pass == 4) break;
      cluster.sync();  // every CTA has read this CTA's histogram before it is cleared
    }
    (void)aimed;
    FZ_MARK(9);
    // ---- 3. exact band: [R_lo - 2eps, R_hi + 2eps] rescored in float64 ----
    const float band_hi = __double2float_ru(R_hi + 2.0 * band_eps);
    const float band_lo = __double2float_rd(R_lo - 2.0 * band_eps);
    int definite = 0;
    const uint32_t ord_bhi = fz_orderable32(band_hi), ord_blo = fz_orderable32(band_lo);
#pragma unroll 1
    for (int g = 0; g < FZ_KG; ++g) {
      const int e = g * FZ_STEP + tid * 8;
      if (e >= m) break;
      uint32_t kk[8];
      fz_load8(keys32, e, m, kk);
      uint32_t fl[2] = {0u, 0u};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const bool valid = e + q < m;
        const bool def = valid && kk[q] > ord_bhi;
        const bool band = valid && !def && kk[q] >= ord_blo;
        definite += def;
        fl[q >> 2] |= (def ? 1u : band ? 3u : 0u) << (8 * (q & 3));
        if (band) {  // rescored in float64 below, all band members at once
          const int slot = atomicAdd(&C.band_count, 1);
          if (slot < FZ_BAND) S.k.f.band_idx[slot] = (uint32_t)(j0 + e + q);
          else C.overflow = 1;
        }
      }
      if (e + 8 <= m) {
        *reinterpret_cast<uint2 *>(flags + e) = make_uint2(fl[0], fl[1]);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)  // (static indices keep fl in registers)
          if (e + q < m) flags[e + q] = (uint8_t)(fl[q >> 2] >> (8 * (q & 3)));
      }
    }
    __syncthreads();
    for (int b = tid; b < min(C.band_count, FZ_BAND); b += blockDim.x)
      S.k.f.band_key[b] = orderable(fz_exact_score(kt, s.capacity, chs, qsum, d_s, S.k.f.band_idx[b]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) definite += __shfl_xor_sync(0xffffffffu, definite, o);
    if (lane == 0) C.wk[0][warp] = (unsigned long long)definite;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < FZ_WARPS; ++w) t += (int)C.wk[0][w];
      C.cta_count = t;
    }
    FZ_MARK(10);
    cluster.sync();
    FZ_MARK(11);
    int cnt_r[FZ_CTAS], all_def = 0, all_band = 0, overflow = 0;
#pragma unroll
    for (int r = 0; r < FZ_CTAS; ++r) {
      const FzCtl *R = cluster.map_shared_rank(&C, r);
      cnt_r[r] = min(R->band_count, FZ_BAND);
      all_def += R->cta_count;
      all_band += cnt_r[r];
      overflow |= R->overflow;
    }
    if (!overflow) {
      // every CTA's band members, concatenated in rank order
      for (int t = tid; t < all_band; t += blockDim.x) {
        int r = 0, base = 0, run = 0;
#pragma unroll
        for (int k = 0; k < FZ_CTAS - 1; ++k) {
          run += cnt_r[k];
          if (t >= run) {
            r = k + 1;
            base = run;
          }
        }
        const FzShared *RS = cluster.map_shared_rank(&S, r);
        S.k.f.all_key[t] = RS->k.f.band_key[t - base];
        S.k.f.all_idx[t] = RS->k.f.band_idx[t - base];
      }
      __syncthreads();
      const int need_b = n_topk - all_def;
      const int mine = min(C.band_count, FZ_BAND);
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
      cluster.sync();  // band arrays read by the other CTAs
    } else {
      // ---- float64 radix select (degenerate inputs, e.g. huge exact-tie sets) ----
      uint64_t *keys64 = S.k.keys64;
      cluster.sync();  // no CTA still reads this CTA's band arrays (aliased by keys64)
      for (int e = tid; e < m; e += blockDim.x)
        keys64[e] = j0 + e < n_sink ? ~0ull : orderable(fz_exact_score(kt, s.capacity, chs, qsum, d_s, j0 + e));
      __syncthreads();
      int top, need64 = n_topk;
      unsigned long long prefix;
      bool done;
      fz_common_prefix(cluster, keys64, m, C, top, prefix);
      fz_radix(cluster, keys64, m, S, C, top, prefix, need64, done);
      fz_exact_flags(cluster, keys64, m, flags, C, top, prefix, need64, done);
    }
    if (rank == 0 && tid == 0 && s.thresh) {
      const double N = (double)(ncand - imin64(ncand, n_sink)), mu = gsum / N, sd = sqrt(fmax(gsq / N - mu * mu, 0.0));
      if (sd > 0.0) fz_store_hint(s.thresh + 4 * u, hint, (0.5 * (R_lo + R_hi) - mu) / sd);
    }
    }  // full-range path
    if (scores_out) {
      for (int e = tid; e < m; e += blockDim.x)
        scores_out[(size_t)u * s.capacity + j0 + e] = fz_exact_score(kt, s.capacity, chs, qsum, d_s, j0 + e);
    }
    __syncthreads();
  }
  FZ_MARK(12);
  // ---- 4. ascending output: the key groups in index order (g, thread, q) + cluster prefix offsets ----
  // per-(group, thread) counts, packed 16 bits per group, prefix-summed in one 64-bit block scan
  uint32_t fw[FZ_KG][2];
  unsigned long long packed = 0ull, packed2 = 0ull;  // groups 0-3 / 4-7
  static_assert(FZ_KG <= 8, "two packed scans cover at most 8 key groups");
#pragma unroll
  for (int g = 0; g < FZ_KG; ++g) {
    const int e = g * FZ_STEP + tid * 8;
    fw[g][0] = fw[g][1] = 0u;
    if (e < m) {
      if (listed) {
        uint32_t kk[8];
        fz_load8(S.k.f.keys32, e, m, kk);
        const uint32_t bits = (S.k.f.bitmap[e >> 5] >> (e & 31)) & 0xffu;  // e is a multiple of 8
#pragma unroll
        for (int q = 0; q < 8; ++q)
          fw[g][q >> 2] |= (uint32_t)(e + q < m && (kk[q] > ord_def || ((bits >> q) & 1u))) << (8 * (q & 3));
      } else if (e + 8 <= m) {
        const uint2 x = *reinterpret_cast<const uint2 *>(flags + e);
        fw[g][0] = x.x;
        fw[g][1] = x.y;
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q)  // (static indices keep fw in registers)
          if (e + q < m) fw[g][q >> 2] |= (uint32_t)flags[e + q] << (8 * (q & 3));
      }
    }
    const unsigned long long c = (unsigned long long)(__popc(fw[g][0]) + __popc(fw[g][1]));  // flags are 0/1 bytes
    if (g < 4) packed |= c << (16 * g);
    else packed2 |= c << (16 * (g - 4));
  }
  unsigned long long tot1, tot2 = 0ull;
  const unsigned long long pre1 = fz_block_excl_scan64(packed, C.scan64, &tot1);
  unsigned long long pre2 = 0ull;
  if (FZ_KG > 4 && m > 4 * FZ_STEP) pre2 = fz_block_excl_scan64(packed2, C.scan64, &tot2);
  int gbase[FZ_KG], gpos[FZ_KG];
  {
    int run = 0;
#pragma unroll
    for (int g = 0; g < FZ_KG; ++g) {
      const unsigned long long T = g < 4 ? tot1 : tot2, P = g < 4 ? pre1 : pre2;
      const int sh = 16 * (g & 3);
      gbase[g] = run;
      gpos[g] = run + (int)((P >> sh) & 0xffffull);
      run += (int)((T >> sh) & 0xffffull);
    }
  }
  const int cta_total = (int)((tot1 & 0xffffull) + ((tot1 >> 16) & 0xffffull) + ((tot1 >> 32) & 0xffffull) +
                              ((tot1 >> 48) & 0xffffull) + (tot2 & 0xffffull) + ((tot2 >> 16) & 0xffffull) +
                              ((tot2 >> 32) & 0xffffull) + ((tot2 >> 48) & 0xffffull));
  (void)gbase;
  if (tid == 0) C.cta_count = cta_total;
  FZ_MARK(13);
  cluster.sync();
  FZ_MARK(14);
  int offset = 0, far_total = 0;
#pragma unroll
  for (int r = 0; r < FZ_CTAS; ++r) {
    const int c = cluster.map_shared_rank(&C, r)->cta_count;
    if (r < rank) offset += c;
    far_total += c;
  }
  const int n_loc = (int)(n - ncand);
  // the local-window rows are dealt round-robin over the cluster's CTAs (local row l -> rank l % FZ_CTAS)
  const int n_loc_mine = n_loc > rank ? (n_loc - rank + FZ_CTAS - 1) / FZ_CTAS : 0;
  const int nrows = cta_total + (ATTEND ? n_loc_mine : 0);
  // row list (32-bit token offsets from rbase, local rows after the far ones) at the top of the staging region
  const int64_t rbase = imin64(j0, ncand);
  // [32-bit row offsets | 32-bit cache slot codes] per row
  const int rows_bytes = ((nrows * 4 + 127) / 128) * 128 + (ATTEND ? ((nrows * 4 + 127) / 128) * 128 : 0);
  static_assert(offsetof(FzShared, flags) == FZ_UNION && offsetof(FzShared, xstage) == FZ_UNION + FZ_CAP &&
                    offsetof(FzShared, xhist) == FZ_STAGE && offsetof(FzShared, xtot) == FZ_STAGE + sizeof(S.xhist),
                "the staging region k.raw + flags + xstage (+ xhist + xtot) is contiguous");
  // ranks other than 0 also stage over the exact path's histograms (dead after the select); in
  // rank 0 they are the inbox the other CTAs push their partials into
  const int stage_bytes = ATTEND ? FZ_STAGE + (rank != 0 ? (int)(sizeof(S.xhist) + sizeof(S.xtot)) : 0) : FZ_UNION;
  int32_t *rows = reinterpret_cast<int32_t *>(S.k.raw + stage_bytes - rows_bytes);
#pragma unroll
  for (int g = 0; g < FZ_KG; ++g) {
    int p = gpos[g];
#pragma unroll
    for (int w = 0; w < 2; ++w) {
      uint32_t x = fw[g][w];
      while (x) {
        const int bit = __ffs(x) - 1;
        x &= x - 1u;
        const int e = g * FZ_STEP + tid * 8 + 4 * w + (bit >> 3);
        out_idx[offset + p] = (int32_t)(j0 + e);
        if (ATTEND) rows[p] = (int32_t)(j0 + e - rbase);
        ++p;
      }
    }
  }
  if (ATTEND)
    for (int i = tid; i < n_loc_mine; i += blockDim.x) rows[cta_total + i] = (int32_t)(ncand + rank + FZ_CTAS * i - rbase);
  if (rank == FZ_CTAS - 1) {
    for (int i = tid; i < n_loc; i += blockDim.x) out_idx[far_total + i] = (int32_t)(ncand + i);
    if (tid == 0) {
      sel_count[u] = far_total + n_loc;
      if (fetch_count) fetch_count[u] = far_total;
    }
  }
  if constexpr (!ATTEND) {
    cluster.sync();  // no CTA leaves while its shared memory may still be read
    return;
  } else {
    for (int i = tid; i < G * D; i += blockDim.x)
      S.qs[i] = h2f(queries[(size_t)u * G * D + i]) * (1.4426950408889634f / sqrtf((float)D));  // log2(e)/sqrt(d)
    __syncthreads();
    FZ_MARK(15);
    // ---- 5. gather + attention over this CTA's rows ----
    // Value rows (PCIe host store, HBM row cache or local mirror) are staged
    // in shared memory by TMA bulk copies, every row of a round at once
    // (one PCIe round trip); key rows come from HBM into registers while the
    // value copies are in flight; logits go to shared memory; then each warp
    // runs an online softmax over its rows.  Rows fetched over PCIe are
    // inserted into the HBM row cache (slots whose row was not selected in
    // the last cache_window steps are reused).
    constexpr int CPL = D / 32;  // channels per lane
    const bool keys_host = !keys_from_device;
    const bool use_cache = s.cache_slots > 0 && keys_from_device;
    // key|value slot-cache path: a cached row is one 512-byte (K|V) copy from its
    // HBM slot into a (K|V) staging row; logits are computed from the staged keys
    const bool kvc = use_cache && s.kdev != nullptr;
    const int row_bytes = D * 2 * (keys_host || kvc ? 2 : 1) + GMAX * 4;  // staged V (+K) + logits
    const int NR = min(1024, ((stage_bytes - rows_bytes) / row_bytes) & ~15);
    uint16_t *stage = reinterpret_cast<uint16_t *>(S.k.raw);
    // staged rows: keys over PCIe: V [NR][D] then K [NR][D]; slot-cache path: [NR][K|V]; else V [NR][D]
    auto vrow = [&](int i) -> uint16_t * { return kvc ? stage + (size_t)i * 2 * D + D : stage + (size_t)i * D; };
    auto krow = [&](int i) -> uint16_t * { return kvc ? stage + (size_t)i * 2 * D : stage + ((size_t)NR + i) * D; };
    float *zs = reinterpret_cast<float *>(S.k.raw + (size_t)NR * D * 2 * (keys_host || kvc ? 2 : 1));
    int32_t *rslot = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned char *>(rows) + ((nrows * 4 + 127) / 128) * 128);
    const int64_t local_start = ncand;
    const int CS = s.cache_slots;
    int32_t *stok = use_cache ? s.slot_tok + (size_t)u * CS : nullptr;
    int32_t *sstamp = use_cache ? s.slot_stamp + (size_t)u * CS : nullptr;
    uint16_t *sv = use_cache ? s.slot_v + (size_t)u * CS * 2 * D : nullptr;  // slots hold (K|V) rows
    int32_t *tslot = use_cache ? s.tok_slot + (size_t)u * s.capacity : nullptr;
    // Each CTA owns the slots [p0, p1) of its unit's cache: it serves hits and
    // allocates misses only there, so no cross-CTA coordination is needed.
    const int spc = (CS + FZ_CTAS - 1) / FZ_CTAS;
    const int p0 = min(CS, rank * spc), p1 = min(CS, p0 + spc);
    // (0) row codes: >= 0 cached slot (hit, stamped with this step), -1 fetch over PCIe, -2 local mirror
    int hits = 0, misses = 0;
    for (int i = tid; i < nrows; i += blockDim.x) {
      const int64_t idx = rbase + rows[i];
      int code = -2;
      if (idx < local_start) {
        code = -1;
        if (use_cache) {
          // tok_slot entries are cleared when their slot is recycled (below), so an entry
          // inside this CTA's partition is valid without reading the slot's token back
          const int p = tslot[idx];
          if (p >= p0 && p < p1) {
            code = p;
            sstamp[p] = (int)n;
          }
        }
        hits += code >= 0;
        misses += code < 0;
      }
      rslot[i] = code;
    }
    __syncthreads();
    FZ_MARK(24);
    float mrun[GMAX], lrun[GMAX], acc[GMAX][CPL];
#pragma unroll
    for (int h = 0; h < GMAX; ++h) {
      mrun[h] = -INFINITY;
      lrun[h] = 0.0f;
#pragma unroll
      for (int e = 0; e < CPL; ++e) acc[h][e] = 0.0f;
    }
    // (a) one thread per row issues the bulk copy of its value row (and key row over PCIe)
    // PCIe copies stall their issuing thread on host-page translations (one
    // translation per random row; the GPU resolves ~75M/s), and the TMA unit
    // serves its queue in order.  With the row cache on, the last warp issues
    // them after every HBM copy is queued, while the other warps compute the
    // key logits; otherwise every thread issues its rows.
    const bool pcie_warp = use_cache;
    const int NLW = pcie_warp ? FZ_WARPS - 1 : FZ_WARPS;  // warps computing key logits
    auto over_pcie = [](int code) { return code == -1 || code <= -3; };
    auto issue_round = [&](int base, int cnt) {
      if (kvc) {
        // every copy adds its own bytes to C.bar (HBM) or, from the PCIe warp, C.bar2;
        // one arrival each once every copy of the round is queued
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (base == 0) FZ_MARK(34);
        for (int i = tid; i < cnt; i += blockDim.x) {
          const int64_t idx = rbase + rows[base + i];
          const int code = rslot[base + i];
          if (code >= 0) {  // hit: the slot's (K|V) row
            fz_mbar_expect_only(&C.bar, D * 4);
            fz_bulk_g2s(krow(i), sv + (size_t)code * 2 * D, D * 4, &C.bar);
          } else if (code == -2) {  // local window mirror
            const size_t lr = (size_t)u * s.local_capacity + (size_t)(idx - s.local_offset);
            fz_mbar_expect_only(&C.bar, D * 4);
            fz_bulk_g2s(krow(i), s.loc_k + lr * D, D * 2, &C.bar);
            fz_bulk_g2s(vrow(i), s.loc_v + lr * D, D * 2, &C.bar);
          } else {  // miss: key row from HBM here, value row over PCIe by the PCIe warp
            fz_mbar_expect_only(&C.bar, D * 2);
            fz_bulk_g2s(krow(i), s.kdev + ((size_t)u * s.capacity + idx) * D, D * 2, &C.bar);
          }
        }
        __syncthreads();
        if (tid == 0) fz_mbar_arrive(&C.bar);
        return;
      }
      if (tid == 0) fz_mbar_expect(&C.bar, (uint32_t)(cnt * D * 2 * (keys_host ? 2 : 1)));
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic accesses before the TMA writes
      __syncthreads();
      if (base == 0) FZ_MARK(34);
      for (int i = tid; i < cnt; i += blockDim.x) {
        const int64_t idx = rbase + rows[base + i];
        const int code = rslot[base + i];
        const uint16_t *vp;
        if (code == -2) {
          const int64_t lr = idx - s.local_offset;
          vp = s.loc_v + ((size_t)u * s.local_capacity + lr) * D;
          if (keys_host) fz_bulk_g2s(krow(i), s.loc_k + ((size_t)u * s.local_capacity + lr) * D, D * 2, &C.bar);
        } else {
          const uint16_t *hrow = s.host_kv + ((size_t)u * s.capacity + idx) * 2 * D;
          if (pcie_warp && over_pcie(code)) continue;
          vp = code >= 0 ? sv + (size_t)code * 2 * D + D : hrow + D;
          if (keys_host) fz_bulk_g2s(krow(i), hrow, D * 2, &C.bar);
        }
        fz_bulk_g2s(vrow(i), vp, D * 2, &C.bar);
      }
    };
    if (nrows > 0) issue_round(0, min(NR, nrows));
    FZ_MARK(25);
    uint32_t parity = 0;
    for (int base = 0; base < nrows; base += NR) {
      const int cnt = min(NR, nrows - base);
      if (base > 0) issue_round(base, cnt);
      // (b) logits of this warp's rows: key rows from HBM while the value copies fly;
      // a batch's 16 row loads are issued before any use
      if (pcie_warp && warp == FZ_WARPS - 1) {
        // (b') the PCIe warp: value rows over PCIe, queued behind the HBM copies
        // (queued behind the HBM copies: in front, their host-page translations held up the
        // TMA queue by ~1 us, more than the earlier start gained)
        unsigned long long *pbar = kvc ? &C.bar2 : &C.bar;
        for (int i = lane; i < cnt; i += 32) {
          if (!over_pcie(rslot[base + i])) continue;
          if (kvc) fz_mbar_expect_only(pbar, D * 2);
          fz_bulk_g2s(vrow(i), s.host_kv + ((size_t)u * s.capacity + rbase + rows[base + i]) * 2 * D + D, D * 2, pbar);
        }
        if (kvc) {
          __syncwarp();
          if (lane == 0) fz_mbar_arrive(pbar);
        }
        if (trace && blockIdx.y == 0 && lane == 0 && base == 0) {
          unsigned long long t_;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
          g_fz_phase[rank][35] = t_;
        }
        // cache slots for this step's misses (every round's), chosen by this warp
        // while the others compute the key logits: free slots of this CTA's
        // partition (empty, or not selected in the last cache_window steps),
        // scanned from the partition's clock hand 32 at a time
        if (base == 0) {
          const int W = max(1, s.cache_window);
          int32_t *F = reinterpret_cast<int32_t *>(S.cta_acc);  // free-slot list (cta_acc is written at the merge)
          constexpr int FCAP = sizeof(S.cta_acc) / 4;
          const unsigned lt = (1u << lane) - 1u;
          int need = 0;
          for (int i0 = 0; i0 < nrows; i0 += 32) {
            const int i = i0 + lane;
            need += __popc(__ballot_sync(0xffffffffu, i < nrows && rslot[i] == -1));
          }
          need = min(need, FCAP);
          const int np = p1 - p0;
          int32_t *hand = s.slot_hand ? s.slot_hand + (size_t)u * TKV_MAX_PARTS + rank : nullptr;
          const int h0 = hand && np > 0 ? ((*hand % np) + np) % np : 0;
          int found = 0;
          for (int k0 = 0; found < need && k0 < np; k0 += 32) {  // warp-uniform: found, need, np
            const int k = k0 + lane;
            int p = 0;
            bool fr = false;
            if (k < np) {
              p = p0 + (h0 + k) % np;
              fr = stok[p] < 0 || sstamp[p] <= (int)n - W;
            }
            const unsigned b = __ballot_sync(0xffffffffu, fr);
            const int pos = found + __popc(b & lt);
            if (fr && pos < need) {
              F[pos] = p;
              const int old = stok[p];  // the recycled slot's token loses its entry (unless it moved on)
              if (old >= 0) atomicCAS(&tslot[old], p, -1);
              if (pos == need - 1 && hand) *hand = (h0 + k + 1) % np;  // the hand moves past the last slot taken
            }
            found += __popc(b);
          }
          __syncwarp();
          const int used = min(found, need);
          int ord = 0;
          for (int i0 = 0; i0 < nrows; i0 += 32) {
            const int i = i0 + lane;
            const bool m = i < nrows && rslot[i] == -1;
            const unsigned b = __ballot_sync(0xffffffffu, m);
            const int k = ord + __popc(b & lt);
            if (m && k < used) rslot[i] = -3 - F[k];  // misses beyond the free slots are simply not cached
            ord += __popc(b);
          }
        }
      } else if (kvc) {
        // (b'') slot-cache path: the round's key rows (cached K|V rows, local
        // mirror, misses' key rows from HBM) land in shared memory; this warp's
        // rows are row = warp mod NLW, as for the register path below
        fz_mbar_wait(&C.bar, parity);
        if (base == 0 && warp == 0) FZ_MARK(32);
        if constexpr (CPL == 4 && (GMAX == 4 || GMAX == 8)) {
          // batches of KR rows: all shared-memory loads first, then independent
          // FMA + butterfly chains the scheduler can interleave
          constexpr int KR = GMAX == 4 ? 8 : 4;
          float4 qv[GMAX];
#pragma unroll
          for (int h = 0; h < GMAX; ++h) qv[h] = *reinterpret_cast<const float4 *>(S.qs + h * D + lane * 4);
          for (int i0 = warp; i0 < cnt; i0 += NLW * KR) {
            uint2 kbs[KR];
#pragma unroll
            for (int j = 0; j < KR; ++j) {
              const int i = i0 + NLW * j;
              kbs[j] = i < cnt ? *reinterpret_cast<const uint2 *>(krow(i) + lane * 4) : make_uint2(0u, 0u);
            }
#pragma unroll
            for (int j = 0; j < KR; ++j) {
            const int i = i0 + NLW * j;
            if (i >= cnt) break;
            const uint2 kb = kbs[j];
            const float k0 = h2f((uint16_t)kb.x), k1 = h2f((uint16_t)(kb.x >> 16));
            const float k2 = h2f((uint16_t)kb.y), k3 = h2f((uint16_t)(kb.y >> 16));
            float dd[GMAX];
#pragma unroll
            for (int h = 0; h < GMAX; ++h) dd[h] = fmaf(qv[h].x, k0, fmaf(qv[h].y, k1, fmaf(qv[h].z, k2, qv[h].w * k3)));
            // transposed butterfly: log2(GMAX) halving steps, then plain steps
            float c;
            int hl;
            if constexpr (GMAX == 8) {
              const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
              float a[4], b2[2];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                a[j] = (b16 ? dd[j + 4] : dd[j]) + __shfl_xor_sync(0xffffffffu, b16 ? dd[j] : dd[j + 4], 16);
#pragma unroll
              for (int j = 0; j < 2; ++j)
                b2[j] = (b8 ? a[j + 2] : a[j]) + __shfl_xor_sync(0xffffffffu, b8 ? a[j] : a[j + 2], 8);
              c = (b4 ? b2[1] : b2[0]) + __shfl_xor_sync(0xffffffffu, b4 ? b2[0] : b2[1], 4);
              c += __shfl_xor_sync(0xffffffffu, c, 2);
              c += __shfl_xor_sync(0xffffffffu, c, 1);
              hl = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
              if ((lane & 3) == 0 && hl < G) zs[(size_t)i * GMAX + hl] = c;
            } else {
              const bool hi16 = lane & 16, hi8 = lane & 8;
              float a0 = hi16 ? dd[2] : dd[0], a1 = hi16 ? dd[3] : dd[1];
              a0 += __shfl_xor_sync(0xffffffffu, hi16 ? dd[0] : dd[2], 16);
              a1 += __shfl_xor_sync(0xffffffffu, hi16 ? dd[1] : dd[3], 16);
              c = hi8 ? a1 : a0;
              c += __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
              c += __shfl_xor_sync(0xffffffffu, c, 4);
              c += __shfl_xor_sync(0xffffffffu, c, 2);
              c += __shfl_xor_sync(0xffffffffu, c, 1);
              hl = (hi16 ? 2 : 0) + (hi8 ? 1 : 0);
              if ((lane & 7) == 0 && hl < G) zs[(size_t)i * GMAX + hl] = c;
            }
            }
          }
        } else {
          for (int i = warp; i < cnt; i += NLW) {
            const uint16_t *kp = krow(i) + lane * CPL;
            float kf[CPL];
#pragma unroll
            for (int e = 0; e < CPL; ++e) kf[e] = h2f(kp[e]);
            for (int h = 0; h < G; ++h) {
              const float *qh = S.qs + h * D + lane * CPL;
              float dp = 0.0f;
#pragma unroll
              for (int e = 0; e < CPL; ++e) dp = fmaf(qh[e], kf[e], dp);
              dp = warp_sum(dp);
              if (lane == 0) zs[(size_t)i * GMAX + h] = dp;
            }
          }
        }
        if (base == 0 && warp == 0) FZ_MARK(33);
      } else if (!keys_host) {
        constexpr int RB = (CPL == 4 && GMAX == 8) ? 8 : 16;  // rows per warp and batch
        for (int i0 = warp; i0 < cnt; i0 += NLW * RB) {
          if constexpr (CPL == 4 && GMAX == 4) {
            uint2 kr[16];
#pragma unroll
            for (int jr = 0; jr < 16; ++jr) {
              const int i = i0 + NLW * jr;
              kr[jr] = make_uint2(0u, 0u);
              if (i < cnt) {
                const int64_t idx = rbase + rows[base + i];
                const uint16_t *kp = idx >= local_start
                                         ? s.loc_k + ((size_t)u * s.local_capacity + (idx - s.local_offset)) * D
                                         : (s.kdev ? s.kdev + ((size_t)u * s.capacity + idx) * D : nullptr);
                if (kp) {
                  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(kr[jr].x), "=r"(kr[jr].y) : "l"(kp + lane * 4));
                } else {  // key row from the channel-major scorer copy (scattered 2-byte reads)
                  uint32_t w[4];
#pragma unroll
                  for (int e = 0; e < 4; ++e) w[e] = kt[((size_t)lane * 4 + e) * s.capacity + idx];
                  kr[jr] = make_uint2(w[0] | (w[1] << 16), w[2] | (w[3] << 16));
                }
              }
            }
            if (base == 0 && i0 == warp) FZ_MARK(32);
            const float4 q0 = *reinterpret_cast<const float4 *>(S.qs + 0 * D + lane * 4);
            const float4 q1 = *reinterpret_cast<const float4 *>(S.qs + 1 * D + lane * 4);
            const float4 q2 = *reinterpret_cast<const float4 *>(S.qs + 2 * D + lane * 4);
            const float4 q3 = *reinterpret_cast<const float4 *>(S.qs + 3 * D + lane * 4);
#pragma unroll
            for (int jr = 0; jr < 16; ++jr) {
              const int i = i0 + NLW * jr;
              if (i >= cnt) break;
              const float k0 = h2f((uint16_t)kr[jr].x), k1 = h2f((uint16_t)(kr[jr].x >> 16));
              const float k2 = h2f((uint16_t)kr[jr].y), k3 = h2f((uint16_t)(kr[jr].y >> 16));
              const float d0 = fmaf(q0.x, k0, fmaf(q0.y, k1, fmaf(q0.z, k2, q0.w * k3)));
              const float d1 = fmaf(q1.x, k0, fmaf(q1.y, k1, fmaf(q1.z, k2, q1.w * k3)));
              const float d2 = fmaf(q2.x, k0, fmaf(q2.y, k1, fmaf(q2.z, k2, q2.w * k3)));
              const float d3 = fmaf(q3.x, k0, fmaf(q3.y, k1, fmaf(q3.z, k2, q3.w * k3)));
              // transposed butterfly: 6 shuffles reduce the four head sums
              const bool hi16 = lane & 16, hi8 = lane & 8;
              float a0 = hi16 ? d2 : d0, a1 = hi16 ? d3 : d1;
              a0 += __shfl_xor_sync(0xffffffffu, hi16 ? d0 : d2, 16);
              a1 += __shfl_xor_sync(0xffffffffu, hi16 ? d1 : d3, 16);
              float c = hi8 ? a1 : a0;
              c += __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
              c += __shfl_xor_sync(0xffffffffu, c, 4);
              c += __shfl_xor_sync(0xffffffffu, c, 2);
              c += __shfl_xor_sync(0xffffffffu, c, 1);
              const int h = (hi16 ? 2 : 0) + (hi8 ? 1 : 0);
              if ((lane & 7) == 0 && h < G) zs[(size_t)i * GMAX + h] = c;
            }
            if (base == 0 && i0 == warp) FZ_MARK(33);
          } else if constexpr (CPL == 4 && GMAX == 8) {
            // up to 8 query heads (Qwen2.5-7B G=7, Llama-3.1-70B G=8): 8 head sums
            // reduced by a 3-level transposed butterfly + 2 plain steps (9 shuffles
            // per row instead of 8 warp sums)
            uint2 kr[RB];
#pragma unroll
            for (int jr = 0; jr < RB; ++jr) {
              const int i = i0 + NLW * jr;
              kr[jr] = make_uint2(0u, 0u);
              if (i < cnt) {
                const int64_t idx = rbase + rows[base + i];
                const uint16_t *kp = idx >= local_start
                                         ? s.loc_k + ((size_t)u * s.local_capacity + (idx - s.local_offset)) * D
                                         : (s.kdev ? s.kdev + ((size_t)u * s.capacity + idx) * D : nullptr);
                if (kp) {
                  asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(kr[jr].x), "=r"(kr[jr].y) : "l"(kp + lane * 4));
                } else {
                  uint32_t w[4];
#pragma unroll
                  for (int e = 0; e < 4; ++e) w[e] = kt[((size_t)lane * 4 + e) * s.capacity + idx];
                  kr[jr] = make_uint2(w[0] | (w[1] << 16), w[2] | (w[3] << 16));
                }
              }
            }
            const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
            const int hl = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
#pragma unroll
            for (int jr = 0; jr < RB; ++jr) {
              const int i = i0 + NLW * jr;
              if (i >= cnt) break;
              const float k0 = h2f((uint16_t)kr[jr].x), k1 = h2f((uint16_t)(kr[jr].x >> 16));
              const float k2 = h2f((uint16_t)kr[jr].y), k3 = h2f((uint16_t)(kr[jr].y >> 16));
              float dd[8];
#pragma unroll
              for (int h = 0; h < 8; ++h) {
                const float4 qh = *reinterpret_cast<const float4 *>(S.qs + h * D + lane * 4);
                dd[h] = fmaf(qh.x, k0, fmaf(qh.y, k1, fmaf(qh.z, k2, qh.w * k3)));
              }
              float a[4];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                a[j] = (b16 ? dd[j + 4] : dd[j]) + __shfl_xor_sync(0xffffffffu, b16 ? dd[j] : dd[j + 4], 16);
              float b2[2];
#pragma unroll
              for (int j = 0; j < 2; ++j)
                b2[j] = (b8 ? a[j + 2] : a[j]) + __shfl_xor_sync(0xffffffffu, b8 ? a[j] : a[j + 2], 8);
              float c = (b4 ? b2[1] : b2[0]) + __shfl_xor_sync(0xffffffffu, b4 ? b2[0] : b2[1], 4);
              c += __shfl_xor_sync(0xffffffffu, c, 2);
              c += __shfl_xor_sync(0xffffffffu, c, 1);
              if ((lane & 3) == 0 && hl < G) zs[(size_t)i * GMAX + hl] = c;
            }
          } else {
            float kf[8][CPL];
#pragma unroll
            for (int jr = 0; jr < 8; ++jr) {
              const int i = i0 + NLW * jr;
#pragma unroll
              for (int e = 0; e < CPL; ++e) kf[jr][e] = 0.0f;
              if (i >= cnt) continue;
              const int64_t idx = rbase + rows[base + i];
              if (idx >= local_start || s.kdev) {
                const uint16_t *kp = idx >= local_start
                                         ? s.loc_k + ((size_t)u * s.local_capacity + (idx - s.local_offset)) * D
                                         : s.kdev + ((size_t)u * s.capacity + idx) * D;
#pragma unroll
                for (int e = 0; e < CPL; ++e) kf[jr][e] = h2f(kp[lane * CPL + e]);
              } else {
#pragma unroll
                for (int e = 0; e < CPL; ++e) kf[jr][e] = h2f(kt[((size_t)lane * CPL + e) * s.capacity + idx]);
              }
            }
#pragma unroll
            for (int jr = 0; jr < 8; ++jr) {
              const int i = i0 + NLW * jr;
              if (i >= cnt) break;
#pragma unroll
              for (int h = 0; h < GMAX; ++h) {
                if (h >= G) break;
                const float *qh = S.qs + h * D + lane * CPL;
                float dp = 0.0f;
#pragma unroll
                for (int e = 0; e < CPL; ++e) dp = fmaf(qh[e], kf[jr][e], dp);
                dp = warp_sum(dp);
                if (lane == 0) zs[(size_t)i * GMAX + h] = dp;
              }
            }
            // rows 8..15 of this batch
            for (int jr = 8; jr < 16; ++jr) {
              const int i = i0 + NLW * jr;
              if (i >= cnt) break;
              const int64_t idx = rbase + rows[base + i];
              float kk2[CPL];
              if (idx >= local_start || s.kdev) {
                const uint16_t *kp = idx >= local_start
                                         ? s.loc_k + ((size_t)u * s.local_capacity + (idx - s.local_offset)) * D
                                         : s.kdev + ((size_t)u * s.capacity + idx) * D;
#pragma unroll
                for (int e = 0; e < CPL; ++e) kk2[e] = h2f(kp[lane * CPL + e]);
              } else {
#pragma unroll
                for (int e = 0; e < CPL; ++e) kk2[e] = h2f(kt[((size_t)lane * CPL + e) * s.capacity + idx]);
              }
              for (int h = 0; h < G; ++h) {
                const float *qh = S.qs + h * D + lane * CPL;
                float dp = 0.0f;
#pragma unroll
                for (int e = 0; e < CPL; ++e) dp = fmaf(qh[e], kk2[e], dp);
                dp = warp_sum(dp);
                if (lane == 0) zs[(size_t)i * GMAX + h] = dp;
              }
            }
          }
        }
      }
      if (base == 0) FZ_MARK(27);
      // (c) value rows (and key rows over PCIe) have landed
      fz_mbar_wait(kvc ? &C.bar2 : &C.bar, parity);
      parity ^= 1u;
      if (base == 0) FZ_MARK(28);
      if (keys_host) {
        for (int i = warp; i < cnt; i += FZ_WARPS) {
          const uint16_t *kp = krow(i);
          for (int h = 0; h < G; ++h) {
            const float *qh = S.qs + h * D + lane * CPL;
            float dp = 0.0f;
#pragma unroll
            for (int e = 0; e < CPL; ++e) dp = fmaf(qh[e], h2f(kp[lane * CPL + e]), dp);
            dp = warp_sum(dp);
            if (lane == 0) zs[(size_t)i * GMAX + h] = dp;
          }
        }
      }
      __syncwarp();
      if (!keys_host) {
        // (d) softmax, warp-local: a warp's rows are the rows whose logits it
        // computed (row = warp mod NLW), so each warp runs an online softmax over
        // them with no CTA barrier -- the round max per head (entries spread over
        // the lanes, lane % GMAX = head), one exp2 per (row, head) written back in
        // place, then p.v over its rows; the warp partials merge below as before
        if (warp < NLW) {
          const int nr = cnt > warp ? (cnt - warp + NLW - 1) / NLW : 0;
          const int hl = lane % GMAX;
          const int ne = nr * GMAX;
          float wm = -INFINITY;
          for (int e = lane; e < ne; e += 32)
            if (hl < G) wm = fmaxf(wm, zs[(size_t)(warp + NLW * (e / GMAX)) * GMAX + hl]);
#pragma unroll
          for (int o = GMAX; o < 32; o <<= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
          float mh = -INFINITY;  // this lane's head's new max
#pragma unroll
          for (int h = 0; h < GMAX; ++h) {
            const float mr = fmaxf(mrun[h], __shfl_sync(0xffffffffu, wm, h));
            if (h < G && mr != -INFINITY) {
              const float sc = exp2f(mrun[h] - mr);  // 0 on the warp's first rows (mrun = -inf)
              lrun[h] *= sc;
#pragma unroll
              for (int e = 0; e < CPL; ++e) acc[h][e] *= sc;
              mrun[h] = mr;
            }
            if (h == hl) mh = mrun[h];
          }
          float ps = 0.0f;
          for (int e = lane; e < ne; e += 32) {
            if (hl >= G) continue;
            float *zp = &zs[(size_t)(warp + NLW * (e / GMAX)) * GMAX + hl];
            const float pv = exp2f(*zp - mh);
            *zp = pv;
            ps += pv;
          }
#pragma unroll
          for (int o = GMAX; o < 32; o <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
#pragma unroll
          for (int h = 0; h < GMAX; ++h) {
            const float t = __shfl_sync(0xffffffffu, ps, h);
            if (h < G) lrun[h] += t;
          }
          __syncwarp();
          if constexpr (CPL == 4 && GMAX == 4) {
            // batches of 4 rows: value and p loads first, then the FMAs
            for (int i0 = warp; i0 < cnt; i0 += NLW * 4) {
              uint2 bv[4];
              float4 pv[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int i = i0 + NLW * j;
                bv[j] = i < cnt ? *reinterpret_cast<const uint2 *>(vrow(i) + lane * 4) : make_uint2(0u, 0u);
                pv[j] = i < cnt ? *reinterpret_cast<const float4 *>(&zs[(size_t)i * 4]) : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float vf[4] = {h2f((uint16_t)bv[j].x), h2f((uint16_t)(bv[j].x >> 16)), h2f((uint16_t)bv[j].y),
                                     h2f((uint16_t)(bv[j].y >> 16))};
                const float pp[4] = {pv[j].x, pv[j].y, pv[j].z, pv[j].w};  // heads >= G hold 0 (never written: masked below)
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                  if (h >= G) break;
#pragma unroll
                  for (int e = 0; e < 4; ++e) acc[h][e] = fmaf(pp[h], vf[e], acc[h][e]);
                }
              }
            }
          } else
          for (int i = warp; i < cnt; i += NLW) {
            const uint16_t *vr = vrow(i) + lane * CPL;
            float vf[CPL];
            if constexpr (CPL == 4) {
              const uint2 bv = *reinterpret_cast<const uint2 *>(vr);
              vf[0] = h2f((uint16_t)bv.x); vf[1] = h2f((uint16_t)(bv.x >> 16));
              vf[2] = h2f((uint16_t)bv.y); vf[3] = h2f((uint16_t)(bv.y >> 16));
            } else {
#pragma unroll
              for (int e = 0; e < CPL; ++e) vf[e] = h2f(vr[e]);
            }
#pragma unroll
            for (int h = 0; h < GMAX; ++h) {
              if (h >= G) break;
              const float p = zs[(size_t)i * GMAX + h];
#pragma unroll
              for (int e = 0; e < CPL; ++e) acc[h][e] = fmaf(p, vf[e], acc[h][e]);
            }
          }
        }
        __syncthreads();  // the PCIe warp's cache-slot codes (rslot) before the inserts below
      } else {
      // (d) softmax: the round's max per head over the whole CTA, p = exp2(z - m)
      // once per (row, head) in shared memory, then each warp accumulates its rows
      __syncthreads();  // every logit of the round is in zs
      {
        float ml[GMAX];
#pragma unroll
        for (int h = 0; h < GMAX; ++h) ml[h] = -INFINITY;
        for (int i = tid; i < cnt; i += blockDim.x)
#pragma unroll
          for (int h = 0; h < GMAX; ++h)
            if (h < G) ml[h] = fmaxf(ml[h], zs[(size_t)i * GMAX + h]);
#pragma unroll
        for (int h = 0; h < GMAX; ++h) {
          if (h >= G) break;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) ml[h] = fmaxf(ml[h], __shfl_xor_sync(0xffffffffu, ml[h], o));
          if (lane == 0) S.red_m[warp][h] = ml[h];
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < GMAX; ++h) {
          if (h >= G) break;
          float mr = mrun[h];
          for (int w = 0; w < FZ_WARPS; ++w) mr = fmaxf(mr, S.red_m[w][h]);
          if (mr != -INFINITY) {
            const float sc = exp2f(mrun[h] - mr);  // 0 on the first round (mrun = -inf)
            lrun[h] *= sc;
#pragma unroll
            for (int e = 0; e < CPL; ++e) acc[h][e] *= sc;
            mrun[h] = mr;
          }
          if (tid == 0) S.m_new[h] = mr;
        }
        __syncthreads();
        for (int t = tid; t < cnt * G; t += blockDim.x) {
          const int i = t / G, h = t - i * G;
          zs[(size_t)i * GMAX + h] = exp2f(zs[(size_t)i * GMAX + h] - S.m_new[h]);
        }
        __syncthreads();
        for (int i = warp; i < cnt; i += FZ_WARPS) {
          const uint16_t *vr = vrow(i) + lane * CPL;
          float vf[CPL];
          if constexpr (CPL == 4) {
            const uint2 bv = *reinterpret_cast<const uint2 *>(vr);
            vf[0] = h2f((uint16_t)bv.x); vf[1] = h2f((uint16_t)(bv.x >> 16));
            vf[2] = h2f((uint16_t)bv.y); vf[3] = h2f((uint16_t)(bv.y >> 16));
          } else {
#pragma unroll
            for (int e = 0; e < CPL; ++e) vf[e] = h2f(vr[e]);
          }
#pragma unroll
          for (int h = 0; h < GMAX; ++h) {
            if (h >= G) break;
            const float p = zs[(size_t)i * GMAX + h];
            lrun[h] += p;
#pragma unroll
            for (int e = 0; e < CPL; ++e) acc[h][e] = fmaf(p, vf[e], acc[h][e]);
          }
        }
      }
      }
      if (base == 0) FZ_MARK(29);
      if (base == 0) FZ_MARK(36);
      // (e) rows fetched over PCIe enter the HBM row cache in their assigned slots
      if (use_cache) {
        for (int i = tid; i < cnt; i += blockDim.x) {
          const int code = rslot[base + i];
          if (code > -3) continue;
          const int dst = -3 - code;
          const int32_t idx = (int32_t)(rbase + rows[base + i]);
          stok[dst] = idx;
          sstamp[dst] = (int)n;
          tslot[idx] = dst;
          if (kvc)
            fz_bulk_s2g(sv + (size_t)dst * 2 * D, krow(i), D * 4);  // the staged (K|V) row
          else
            fz_bulk_s2g(sv + (size_t)dst * 2 * D + D, vrow(i), D * 2);
        }
        fz_bulk_commit_wait_read();  // the staged rows are read before the next round overwrites them
      }
      if (base == 0) FZ_MARK(30);
      __syncthreads();
    }
    if (trace && blockIdx.y < 64 && tid == 0) {
      atomicAdd(&g_fz_upath[blockIdx.y][2], nrows);
    }
    if (use_cache) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        hits += __shfl_xor_sync(0xffffffffu, hits, o);
        misses += __shfl_xor_sync(0xffffffffu, misses, o);
      }
      if (trace && blockIdx.y < 64 && lane == 0) atomicAdd(&g_fz_upath[blockIdx.y][3], misses);
      if (lane == 0 && (hits | misses)) {
        atomicAdd(&C.hits, hits);
        atomicAdd(&C.misses, misses);
      }
    }
    FZ_MARK(16);
    asm volatile("griddepcontrol.launch_dependents;");  // the next layer's kernel may start its prologue
    // every CTA of the cluster read its channels before the selection's cluster barriers: re-arm the handshake
    if (s.s1_ready && rank == 0 && tid == 0) s.s1_ready[u] = 0;
    __syncthreads();  // the staging area (aliased by the partials) is no longer read
    FZ_MARK(17);
    float *pm = reinterpret_cast<float *>(S.k.raw), *pl = pm + FZ_WARPS * GMAX, *pa = pl + FZ_WARPS * GMAX;
#pragma unroll
    for (int h = 0; h < GMAX; ++h) {
      if (h >= G) break;
      if (lane == 0) {
        pm[warp * GMAX + h] = mrun[h];
        pl[warp * GMAX + h] = lrun[h];
      }
#pragma unroll
      for (int e = 0; e < CPL; ++e) pa[((size_t)warp * GMAX + h) * D + lane * CPL + e] = acc[h][e];
    }
    __syncthreads();
    // With G*D <= 512 every CTA pushes its partial into rank 0's inbox (the
    // exact path's histograms, dead by now) with DSMEM stores before the
    // barrier, so rank 0 merges from its own shared memory and the other CTAs
    // leave right after the barrier; otherwise rank 0 pulls them afterwards.
    static_assert(sizeof(S.xhist) + sizeof(S.xtot) >= (FZ_CTAS * 512 + 2 * FZ_CTAS * 8) * sizeof(float),
                  "rank 0's partial inbox overlays the exact path's histograms");
    const bool push = G * D <= 512;
    float *inbox = cluster.map_shared_rank(reinterpret_cast<float *>(&S.xhist[0][0]), 0);  // [CTAS][512] + m, l
    for (int i = tid; i < G * D; i += blockDim.x) {
      const int h = i / D, c = i % D;
      float M = -INFINITY;
      for (int w = 0; w < FZ_WARPS; ++w) M = fmaxf(M, pm[w * GMAX + h]);
      float L = 0.0f, A = 0.0f;
      if (M != -INFINITY) {
        for (int w = 0; w < FZ_WARPS; ++w) {
          const float mw = pm[w * GMAX + h];
          if (mw == -INFINITY) continue;
          const float sc = exp2f(mw - M);
          L = fmaf(sc, pl[w * GMAX + h], L);
          A = fmaf(sc, pa[((size_t)w * GMAX + h) * D + c], A);
        }
      }
      if (push) {
        inbox[rank * 512 + i] = A;
        if (c == 0) {
          inbox[FZ_CTAS * 512 + rank * 8 + h] = M;
          inbox[FZ_CTAS * 512 + FZ_CTAS * 8 + rank * 8 + h] = L;
        }
      } else {
        S.cta_acc[i] = A;
        if (c == 0) {
          S.cta_m[h] = M;
          S.cta_l[h] = L;
        }
      }
    }
    if (use_cache && tid == 0 && (C.hits | C.misses)) {
      atomicAdd(&s.cache_stats[0], (unsigned long long)C.hits);
      atomicAdd(&s.cache_stats[1], (unsigned long long)C.misses);
    }
    FZ_MARK(18);
    cluster.sync();
    FZ_MARK(19);
    // ---- 6. the step's append (HostPool.append + mirror append, memsim.py:106-111,
    // pipeline.py:405-413) after this step's attention (every CTA has passed the
    // merge barrier): the new token of unit u goes to position n of every store;
    // the last cluster to finish advances *len ----
    if (new_keys && rank == FZ_CTAS - 1) {  // (rank 0 is merging the partials meanwhile)
      for (int c = tid; c < D; c += blockDim.x) {
        const uint16_t k = new_keys[(size_t)u * D + c], v = new_values[(size_t)u * D + c];
        s.kt[((size_t)u * D + c) * s.capacity + n] = k;  // (the host store row went out at kernel start)
        float *cm = &s.chmax[(size_t)u * D + c];
        *cm = fmaxf(*cm, fabsf(h2f(k)));
        const int64_t lr = n - s.local_offset;
        s.loc_k[((size_t)u * s.local_capacity + lr) * D + c] = k;
        s.loc_v[((size_t)u * s.local_capacity + lr) * D + c] = v;
        if (s.kdev) s.kdev[((size_t)u * s.capacity + n) * D + c] = k;
      }
      __syncthreads();
      if (tid == 0) {
        const unsigned prev = atomicAdd(s.ticket, 1u);
        if (prev == (unsigned)s.units - 1) {
          *s.ticket = 0;
          __threadfence();
          *s.len = (int32_t)(n + 1);
        }
      }
    }
    if (rank == 0 && push) {
      const float *ib = reinterpret_cast<const float *>(&S.xhist[0][0]);
      for (int i = tid; i < G * D; i += blockDim.x) {
        const int h = i / D;
        float Mr[FZ_CTAS], M = -INFINITY;
#pragma unroll
        for (int r = 0; r < FZ_CTAS; ++r) {
          Mr[r] = ib[FZ_CTAS * 512 + r * 8 + h];
          M = fmaxf(M, Mr[r]);
        }
        float L = 0.0f, A = 0.0f;
#pragma unroll
        for (int r = 0; r < FZ_CTAS; ++r) {
          if (Mr[r] == -INFINITY) continue;
          const float sc = exp2f(Mr[r] - M);
          L = fmaf(sc, ib[FZ_CTAS * 512 + FZ_CTAS * 8 + r * 8 + h], L);
          A = fmaf(sc, ib[r * 512 + i], A);
        }
        out[(size_t)u * G * D + i] = A / L;
      }
    } else if (rank == 0) {
      for (int i = tid; i < G * D; i += blockDim.x) {
        const int h = i / D;
        float Mr[FZ_CTAS], M = -INFINITY;
#pragma unroll
        for (int r = 0; r < FZ_CTAS; ++r) {
          Mr[r] = cluster.map_shared_rank(&S, r)->cta_m[h];
          M = fmaxf(M, Mr[r]);
        }
        float L = 0.0f, A = 0.0f;
#pragma unroll
        for (int r = 0; r < FZ_CTAS; ++r) {
          if (Mr[r] == -INFINITY) continue;
          const FzShared *R = cluster.map_shared_rank(&S, r);
          const float sc = exp2f(Mr[r] - M);
          L = fmaf(sc, R->cta_l[h], L);
          A = fmaf(sc, R->cta_acc[i], A);
        }
        out[(size_t)u * G * D + i] = A / L;
      }
    }
    if (!push) cluster.sync();  // rank 0 has read every CTA's partial
    FZ_MARK(20);
    if (trace && blockIdx.y == 0 && tid == 0) g_fz_clk[rank][1] = clock64();
    if (trace && blockIdx.y < 64 && tid == 0) {
      unsigned long long t_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
      g_fz_unit[blockIdx.y][rank][1] = t_;
      if (blockIdx.y == 0 && rank == 0) g_fz_launch[lslot][2] = t_;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
bool fused_ok(const SL &s, int n_local) {
  const int64_t ncand = s.capacity > n_local ? s.capacity - n_local : 0;
  const int64_t chunk = ((ncand + FZ_CTAS - 1) / FZ_CTAS + 15) & ~int64_t(15);
  // per-thread flag granules (<= 64 flags) and 16-bit row offsets
  return chunk <= FZ_CAP && chunk <= (int64_t)FZ_THREADS * 64 && chunk + 4096 < 65536 && s.capacity % 8 == 0;
}

template <bool ATTEND, int D, int GMAX>
static cudaError_t launch_fused(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s,
                                int n_local, int n_topk, int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count,
                                double *scores_out, int keys_from_device, float *out, cudaStream_t st,
                                const uint16_t *new_keys = nullptr, const uint16_t *new_values = nullptr) {
  auto kern = sparse_fused_kernel<ATTEND, D, GMAX>;
  const size_t sm = sizeof(FzShared);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (FZ_CTAS > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(FZ_CTAS, s.units);
  cfg.blockDim = dim3(FZ_THREADS);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute at[3];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = FZ_CTAS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributePriority;
  at[1].val.priority = launch_priority(true);
  at[2].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (griddepcontrol in the kernel)
  static const bool no_pdl = getenv("TKV_NO_PDL") != nullptr;
  // the pre-wait prologue reads this layer's length: never overlap a launch on the same layer
  at[2].val.programmaticStreamSerializationAllowed = (pdl_note(st, s.len) && !no_pdl) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 3;
  return cudaLaunchKernelEx(&cfg, kern, s, queries, G, channels, d_s, n_local, n_topk, sel_idx,
                            n_local + n_topk + s.n_sink,
                            sel_count, fetch_count, scores_out, keys_from_device, out, new_keys, new_values);
}

// select only (tkv_select_tokens)
int select_cluster(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s, int n_local,
                   int n_topk, int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count, double *scores_out,
                   cudaStream_t st) {
  const cudaError_t e = launch_fused<false, 128, 1>(s, queries, G, channels, d_s, n_local, n_topk, sel_idx,
                                                    sel_count, fetch_count, scores_out, 1, nullptr, st);
  if (e != cudaSuccess) return fail(TKV_ERR_CUDA, std::string("tkv_select_tokens(cluster): ") + cudaGetErrorString(e));
  return check_launch("tkv_select_tokens(cluster)");
}

bool select_cluster_ok(const SL &s, int n_local) { return fused_ok(s, n_local); }

bool sparse_decode_supported(const SL &s, int G, int n_local) {
  if (!fused_ok(s, n_local)) return false;
  return (s.d == 128 && G <= 8) || (s.d == 64 && G <= 8) || (s.d == 256 && G <= 4) || (s.d == 32 && G <= 8);
}

// clusters of this size that can be resident at once (cudaOccupancyMaxActiveClusters), per kernel instance
template <int D, int GMAX>
static int active_clusters() {
  static int n = -1;
  if (n < 0) {
    auto kern = sparse_fused_kernel<true, D, GMAX>;
    const size_t sm = sizeof(FzShared);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(FZ_CTAS, 1024);
    cfg.blockDim = dim3(FZ_THREADS);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = FZ_CTAS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    n = c;
  }
  return n;
}

int max_active_clusters(int d, int G) {
  if (d == 128 && G <= 4) return active_clusters<128, 4>();
  if (d == 128 && G <= 8) return active_clusters<128, 8>();
  if (d == 64 && G <= 8) return active_clusters<64, 8>();
  if (d == 32 && G <= 8) return active_clusters<32, 8>();
  if (d == 256 && G <= 4) return active_clusters<256, 4>();
  return 0;
}

#if TKV_FZ_CTAS == 8
static int g_last_cluster = 0;
int last_cluster_size() { return g_last_cluster; }

// Cluster size: the fewest waves of co-resident clusters over the units (a launch takes about the same
// time per wave whatever the cluster size: DESIGN.md 4.7), larger clusters on ties; a size is eligible when
// its CTAs can hold a unit's candidate slice.  B200, d 128: 8-CTA clusters 15 at once, 4-CTA 33, 2-CTA 74.
// TKV_FZ_CLUSTER=8|4|2 forces a size (when eligible).
static int g_cluster_force = -1;  // tkv_debug_sparse_cluster: runtime override of TKV_FZ_CLUSTER (tests)
int choose_cluster(const SL &s, int G, int n_local) {
  static const int env_force = getenv("TKV_FZ_CLUSTER") ? atoi(getenv("TKV_FZ_CLUSTER")) : 0;
  const int force = g_cluster_force >= 0 ? g_cluster_force : env_force;
  const int m8 = max_active_clusters(s.d, G);
  const bool ok4 = fz4::sparse_decode_supported(s, G, n_local), ok2 = fz2::sparse_decode_supported(s, G, n_local);
  const int m4 = ok4 ? fz4::max_active_clusters(s.d, G) : 0, m2 = ok2 ? fz2::max_active_clusters(s.d, G) : 0;
  auto waves = [&](int m) { return m > 0 ? (s.units + m - 1) / m : INT_MAX; };
  int c = 8, w = waves(m8);
  if (waves(m4) < w) c = 4, w = waves(m4);
  if (waves(m2) < w) c = 2, w = waves(m2);
  if (force == 8 || (force == 4 && ok4) || (force == 2 && ok2)) c = force;
  return c;
}
#endif

// fused select + gather + attention (tkv_sparse_decode)
int sparse_decode_fused(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s, int n_local,
                        int n_topk, int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count, int keys_from_device,
                        float *out, const uint16_t *new_keys, const uint16_t *new_values, cudaStream_t st) {
#if TKV_FZ_CTAS == 8
  {  // cluster size (choose_cluster)
    const int c = choose_cluster(s, G, n_local);
    g_last_cluster = c;
    if (c == 4)
      return fz4::sparse_decode_fused(s, queries, G, channels, d_s, n_local, n_topk, sel_idx, sel_count, fetch_count,
                                      keys_from_device, out, new_keys, new_values, st);
    if (c == 2)
      return fz2::sparse_decode_fused(s, queries, G, channels, d_s, n_local, n_topk, sel_idx, sel_count, fetch_count,
                                      keys_from_device, out, new_keys, new_values, st);
  }
#endif
  cudaError_t e;
#define TKV_FZ(D, GM)                                                                                          \
  e = launch_fused<true, D, GM>(s, queries, G, channels, d_s, n_local, n_topk, sel_idx, sel_count, fetch_count, \
                                nullptr, keys_from_device, out, st, new_keys, new_values)
  if (s.d == 128 && G <= 4) TKV_FZ(128, 4);
  else if (s.d == 128 && G <= 8) TKV_FZ(128, 8);
  else if (s.d == 64 && G <= 8) TKV_FZ(64, 8);
  else if (s.d == 32 && G <= 8) TKV_FZ(32, 8);
  else if (s.d == 256 && G <= 4) TKV_FZ(256, 4);
  else return fail(TKV_ERR_PARAMETER, "fused sparse decode supports d in {32,64,128,256} with G<=8 (G<=4 at d=256)");
#undef TKV_FZ
  if (e != cudaSuccess) return fail(TKV_ERR_CUDA, std::string("tkv_sparse_decode: ") + cudaGetErrorString(e));
  return check_launch("tkv_sparse_decode");
}

#if TKV_FZ_CTAS != 8
}  // namespace fz4 / fz2
}  // namespace tkv
#else
}  // namespace tkv

// force the fused decode's cluster size (8, 4 or 2 when eligible; 0 = auto; -1 = TKV_FZ_CLUSTER)
extern "C" int tkv_debug_sparse_cluster(int c) {
  tkv::g_cluster_force = c;
  return 0;
}

// 1 when a fused decode (8-CTA build) gave up waiting for the stage-1 handshake (then reset to 0)
extern "C" int tkv_debug_sparse_s1_timeout(void) {
  unsigned v = 0, z = 0;
  if (cudaMemcpyFromSymbol(&v, tkv::g_fz_s1_timeout, sizeof(v)) != cudaSuccess) return -1;
  cudaMemcpyToSymbol(tkv::g_fz_s1_timeout, &z, sizeof(z));
  return (int)v;
}

extern "C" int tkv_debug_sparse_trace(int on) {
  return cudaMemcpyToSymbol(tkv::g_fz_trace, &on, sizeof(int)) == cudaSuccess ? 0 : 7;
}

extern "C" int tkv_debug_sparse_upath(int *out, int reset) {
  if (reset) {
    static const int zero[64 * 4] = {};
    return cudaMemcpyToSymbol(tkv::g_fz_upath, zero, sizeof(zero)) == cudaSuccess ? 0 : 7;
  }
  return cudaMemcpyFromSymbol(out, tkv::g_fz_upath, sizeof(tkv::g_fz_upath)) == cudaSuccess ? 0 : 7;
}

extern "C" int tkv_debug_sparse_units(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, tkv::g_fz_unit, sizeof(tkv::g_fz_unit)) == cudaSuccess ? 0 : 7;
}

// launch timeline of unit 0 (start, after the PDL wait, end) for the last
// up-to-128 launches in trace mode, in launch order; returns the count
extern "C" int tkv_debug_sparse_launches(unsigned long long *out, int reset) {
  if (reset) {
    const unsigned int z = 0;
    return cudaMemcpyToSymbol(tkv::g_fz_nlaunch, &z, sizeof(z)) == cudaSuccess ? 0 : -1;
  }
  unsigned int cnt = 0;
  if (cudaMemcpyFromSymbol(&cnt, tkv::g_fz_nlaunch, sizeof(cnt)) != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(out, tkv::g_fz_launch, sizeof(tkv::g_fz_launch)) != cudaSuccess) return -1;
  return (int)cnt;
}

// select-path counts since the last reset (trace mode): [list attempt 0, attempt 1, full range]
extern "C" int tkv_debug_sparse_pathcount(unsigned int *out, int reset) {
  if (reset) {
    const unsigned int z[4] = {0, 0, 0, 0};
    return cudaMemcpyToSymbol(tkv::g_fz_pathcnt, z, sizeof(z)) == cudaSuccess ? 0 : 7;
  }
  return cudaMemcpyFromSymbol(out, tkv::g_fz_pathcnt, sizeof(tkv::g_fz_pathcnt)) == cudaSuccess ? 0 : 7;
}

// tuning: half-width (in score standard deviations) of the first aimed range
extern "C" int tkv_debug_sparse_aim(float w) {
  return cudaMemcpyToSymbol(tkv::g_fz_aim, &w, sizeof(w)) == cudaSuccess ? 0 : 7;
}

extern "C" int tkv_debug_sparse_clocks(unsigned long long *out) {
  return cudaMemcpyFromSymbol(out, tkv::g_fz_clk, sizeof(tkv::g_fz_clk)) == cudaSuccess ? 0 : 7;
}

extern "C" int tkv_debug_sparse_attempts(double *out) {
  return cudaMemcpyFromSymbol(out, tkv::g_fz_dbg, sizeof(tkv::g_fz_dbg)) == cudaSuccess ? 0 : 7;
}

extern "C" int tkv_debug_sparse_phases(unsigned long long *out) {  // [8][32]
  return cudaMemcpyFromSymbol(out, tkv::g_fz_phase, sizeof(tkv::g_fz_phase)) == cudaSuccess ? 0 : 7;  // [8][40]
}
#endif  // TKV_FZ_CTAS == 8 (debug exports)
