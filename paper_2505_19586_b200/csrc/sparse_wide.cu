// The wide sparse-layer decode: one launch per sparsity-friendly layer when a
// GPU holds few units (batch x KV heads), e.g. config 2's 8 heads on one B200
// or one head per GPU at N = 8.  Same results as the cluster kernel
// (sparse_fused.cu): proxy scores (retriever.py:166-189) -> exact top-k by
// (score desc, index desc) plus the local window, ascending
// (retriever.py:192-211) -> gather of the selected rows (memsim.py:228-252)
// -> exact softmax attention (pipeline.py:364-376) -> the step's append
// (memsim.py:106-111, pipeline.py:405-413).
//
// Why a second kernel: the cluster kernel runs one 8-CTA cluster per unit, so
// 8 units use 64 of the 148 SMs, and its data phases (2 MB of scorer columns
// and ~1.4 MB of gathered rows per unit) are bound by per-SM bandwidth
// (~45-55 GB/s per SM, profiles/r1_kernels.md 4).  Here a unit is split into
// P token partitions, one CTA each (P = SMs / units: 18 for 8 units), and the
// CTAs of a unit cooperate through global memory:
//
// 0. prologue (before the PDL wait, overlapping the previous layer): one
//    thread issues TMA bulk copies of the partition's d_s critical scorer
//    columns (<= 8 x 16 KB, L2-resident after stage 1's prefetch) into SMEM;
// 1. fp32 proxy scores -> order-preserving u32 keys in SMEM, and the
//    partition's own score moments;
// 2. aimed candidate list: each partition aims at the last step's threshold
//    through its OWN moments (a per-partition z-score hint, so aiming needs no
//    exchange), counts its keys above the window and publishes the keys inside
//    it (+-2 eps) with a header -> ONE unit barrier -> every CTA merges the
//    unit's lists and resolves the threshold redundantly and identically: the
//    bin of the k-th largest key, float64 rescoring of the +-2 eps band (eps is
//    a rigorous fp32 error bound), exact ranking with the
//    reference's tie rule, and every partition's selected count (so the output
//    offsets need no second barrier).
//    Fallbacks (aim missed, list overflow, huge exact-tie bands): a second
//    aimed attempt with the unit's global moments, then an exact radix select
//    of the k-th fp32 key through global histograms, then -- for bands larger
//    than the rescoring buffer -- an exact radix select over (float64 score,
//    index).  Every decision is taken identically by every CTA of the unit.
// 3. ascending output (sel_idx, counts);
// 4. gather of the partition's own rows into SMEM by TMA bulk copies (HBM row
//    cache, local mirror, token-major keys; value rows of misses over PCIe from
//    one warp, queued behind the HBM copies), logits, warp-local online
//    softmax, p.v;
// 5. partials merged in a fixed order by last-arriver merges (groups of 16,
//    then the groups), so no CTA waits for another; the final merger runs the
//    step's append.
//
// Deadlock freedom: a unit barrier waits only on CTAs of the same grid; the
// grid (units x P <= SMs, one CTA per SM) lets its dependents launch only
// after every one of its CTAs has started (griddepcontrol semantics), and the
// other kernels that can hold SMs meanwhile (stage 1 on the side stream, the
// previous layer's decode) finish without waiting on this grid.  Spins are
// bounded: a timeout sets an error word instead of hanging the GPU.

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "sparse.cuh"

namespace tkv {
namespace wide {

constexpr int WK_THREADS = 512;
constexpr int WK_WARPS = WK_THREADS / 32;
constexpr int WK_D = 128;                       // head_dim of this kernel
constexpr int WK_MAXM = 8192;                   // candidate tokens per partition
constexpr int WK_MAXDS = 8;                     // critical channels staged by TMA
constexpr int WK_RAW = WK_MAXDS * WK_MAXM * 2;  // 128 KB: scorer columns -> merged lists -> staged rows
constexpr int WK_MAXLOC = 512;                  // local-window rows per partition
constexpr int WK_KEYS = (WK_MAXM + WK_MAXLOC) * 4;  // keys32, then the partition's row list
constexpr int WK_LCAP = 1024;                   // list entries per partition and attempt
constexpr int WK_GCAP = 4096;                   // merged list entries per unit (64 KB of SMEM)
constexpr int WK_BAND = 512;                    // band members rescored in float64
constexpr int WK_NB = 1024;                     // resolve histogram bins (two per thread)
constexpr int WK_HB = 2048;                     // radix bins (fallback)
constexpr int WK_NHIST = 12;                    // 3 fp32 passes + 9 (float64 score, index) passes
constexpr int WK_GS = 16;                       // merge group size when P > 32
constexpr int WK_FCAP = 512;                    // cache slots allocated per partition and round
constexpr int WK_NMARK = 32;
constexpr unsigned WK_SPIN_LIMIT = 1u << 26;    // ~seconds: a stuck barrier becomes an error, not a hang
// a list entry: (order-preserving fp32 key << 32 | token index) and the token's float64 score
// (exact: computed from the partition's fp16 scorer columns in SMEM, in the reference's channel order)
struct LEnt {
  unsigned long long kidx;
  double s;
};
static_assert(WK_GCAP * 16 + TKV_MAX_PARTS * 64 <= WK_RAW, "merged list + header table fit the scorer region");
static_assert(WK_NB == 2 * WK_THREADS && WK_MAXM / 32 <= WK_THREADS, "one thread per bin pair / mask word");

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ord32(float x) {
  if (x == 0.0f) x = 0.0f;
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float from_ord32(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar) {
  asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(saddr(bar)));
}
__device__ __forceinline__ void mbar_arrive_expect(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ unsigned g_wk_err;  // a bounded wait timed out (results of that launch are void)
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
  // bounded: a byte-count mismatch must surface as an error, never as a hung GPU
  for (unsigned it = 0;; ++it) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(saddr(bar)), "r"(parity)
        : "memory");
    if (ok) return;
    if (it > (1u << 22)) {
      atomicExch(&g_wk_err, 2u);
      return;
    }
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(saddr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait_read() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ double normal_upper_quantile(double p) {
  // Acklam's rational approximation (|rel err| < 1.2e-9); only aims the first list
  const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                       1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00};
  const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                       6.680131188771972e+01, -1.328068155288572e+01};
  const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                       -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00};
  const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00, 3.754408661907416e+00};
  const double q0 = fmin(fmax(1.0 - p, 1e-12), 1.0 - 1e-12);
  if (q0 < 0.02425) {
    const double q = sqrt(-2.0 * log(q0));
    return (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
           ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
  }
  if (q0 <= 1.0 - 0.02425) {
    const double q = q0 - 0.5, r = q * q;
    return (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
           (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0);
  }
  const double q = sqrt(-2.0 * log(1.0 - q0));
  return -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
         ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0);
}

// ---------------------------------------------------------------------------
// workspace: [ctl + histograms per unit (zero between launches)] [the
// unfused path's region] [scratch per unit: headers, lists, counts, partials]
// ---------------------------------------------------------------------------
struct Hdr {  // one partition's published state for one attempt (64 B)
  uint32_t above, count, llo, lhi;  // keys above lhi; list entries; list key range [llo, lhi]
  uint32_t klo, khi, nval, pad0;    // min/max key and count of the scored keys (no sinks)
  double sum, sq;                   // score moments
  float wlo, whi;                   // the aimed window (values)
  uint32_t pad1[2];
};
static_assert(sizeof(Hdr) == 64, "header layout");
constexpr int CTL_WORDS = 64;  // bar_count, bar_gen, merge_final, fallback, err, merge_group[16] ...
enum { C_BAR = 0, C_GEN = 1, C_FINAL = 2, C_FALLBACK = 3, C_ERR = 4, C_GROUP = 8 };  // [C_BAR, C_GEN]: one u64
__host__ __device__ constexpr int64_t ctl_unit_bytes() { return CTL_WORDS * 4 + (int64_t)WK_NHIST * WK_HB * 4; }
__host__ __device__ constexpr int part_floats(int gmax) { return gmax * WK_D + 2 * gmax; }
__host__ __device__ inline int64_t scratch_unit_bytes(int P) {
  const int64_t hdr = 2LL * P * 64, lists = 2LL * P * WK_LCAP * 16, counts = ((int64_t)P * 4 + 255) / 256 * 256;
  const int NG = (P + WK_GS - 1) / WK_GS + 1;
  const int64_t parts = (int64_t)(P + NG) * part_floats(8) * 4;
  return (hdr + lists + counts + parts + 255) / 256 * 256;
}

struct WArgs {
  const uint16_t *queries;  // [units][G][D]
  const int32_t *channels;  // [units][d_s]
  int G, d_s, n_local, n_topk;
  int32_t *sel_idx;
  int sel_stride;
  int32_t *sel_count, *fetch_count;
  int keys_from_device;
  float *out;
  const uint16_t *new_keys, *new_values;
  unsigned char *ctl;      // per unit ctl_unit_bytes()
  unsigned char *scratch;  // per unit scratch_unit_bytes(P)
  int64_t scratch_unit;
};

// static shared state
struct WSh {
  unsigned long long bar_tma, bar_hbm, bar_pcie;
  int chs[WK_MAXDS];
  double qsum[WK_MAXDS];
  float qsum32[WK_MAXDS];
  double eps_term[WK_MAXDS];
  double band_eps;
  uint32_t r_lo[WK_WARPS], r_hi[WK_WARPS];
  double r_sum[WK_WARPS], r_sq[WK_WARPS];
  int r_i[WK_WARPS], r_j[WK_WARPS];
  int list_count, above;
  // local moments
  uint32_t klo, khi;
  int nval;
  double mu, sd;
  // resolve (identical in every CTA of the unit)
  int status, dir;
  uint32_t ord_def;
  int A, Ltot, ovf;
  uint32_t LL, LH, XL, XH, gklo, gkhi;
  double gmu, gsd;
  float XLf, XHf;
  int lstart[TKV_MAX_PARTS + 1];
  int pcount[TKV_MAX_PARTS];
  uint32_t hist[WK_HB];
  int bin, band_n, band_ovf, definite;
  double e_lo, e_hi;
  unsigned long long band_key[WK_BAND];
  uint32_t band_idx[WK_BAND];
  uint8_t band_sel[WK_BAND];
  uint32_t bitmap[WK_MAXM / 32];
  // radix fallback
  int rneed, rabove, rdigit;
  uint32_t rprefix;
  unsigned long long xprefix;
  uint32_t xjprefix;
  int nm;
  // output + gather
  int scan[WK_WARPS + 1];
  int offset, far_total, cta_total;
  int hits, misses, last, free_slots[WK_FCAP];
  int nrest;
  float m_new[8];
  // compact-path state
  float fsum, fsq;
  uint32_t llo, lhi;
  float wlo_f, whi_f;
  int cnt_a, cnt_b, cnt_c;
  uint32_t amask[WK_MAXM / 32];  // selected keys of this partition, 32 per word (index order)

  int wtot[WK_WARPS], wbase[WK_WARPS];
};

struct UnitWs {
  unsigned *ctl;
  unsigned *hist;
  Hdr *hdr;                    // [2][P]
  LEnt *lists;                 // [2][P][LCAP]
  int *counts;                 // [P]
  float *part;                 // [P + NG][part_floats(8)]
};

__device__ __forceinline__ UnitWs unit_ws(const WArgs &a, int u, int P) {
  UnitWs w;
  unsigned char *c = a.ctl + (size_t)u * ctl_unit_bytes();
  w.ctl = reinterpret_cast<unsigned *>(c);
  w.hist = reinterpret_cast<unsigned *>(c + CTL_WORDS * 4);
  unsigned char *s = a.scratch + (size_t)u * a.scratch_unit;
  w.hdr = reinterpret_cast<Hdr *>(s);
  s += 2LL * P * 64;
  w.lists = reinterpret_cast<LEnt *>(s);
  s += 2LL * P * WK_LCAP * 16;
  w.counts = reinterpret_cast<int *>(s);
  s += ((int64_t)P * 4 + 255) / 256 * 256;
  w.part = reinterpret_cast<float *>(s);
  return w;
}

// one unit's grid barrier: a 64-bit word (arrivals | generation << 32).  The
// last of P arrivals adds 2^32 - (P - 1), which resets the arrivals and bumps
// the generation in one atomic; the others poll the generation.  Thread 0
// spins, bounded (a stuck barrier becomes an error flag, never a hang).
__device__ __forceinline__ unsigned long long ld_acquire64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// split form: arrive (thread 0; returns the generation to wait past), then wait
__device__ __forceinline__ unsigned unit_arrive(unsigned *ctl, int P) {
  __syncthreads();
  unsigned g = 0;
  if (threadIdx.x == 0) {
    unsigned long long *word = reinterpret_cast<unsigned long long *>(&ctl[C_BAR]);
    __threadfence();  // this CTA's lists and header before the arrival
    const unsigned long long old = atomicAdd(word, 1ull);
    g = (unsigned)(old >> 32);
    if ((unsigned)old == (unsigned)P - 1) atomicAdd(word, (1ull << 32) - (unsigned long long)P);
  }
  return g;
}
__device__ __forceinline__ void unit_wait(unsigned *ctl, unsigned g) {
  if (threadIdx.x == 0) {
    const unsigned long long *word = reinterpret_cast<const unsigned long long *>(&ctl[C_BAR]);
    unsigned it = 0;
    while ((unsigned)(ld_acquire64(word) >> 32) == g) {
      if (++it > WK_SPIN_LIMIT) {
        atomicExch(&ctl[C_ERR], 1u);
        atomicExch(&g_wk_err, 1u);
        break;
      }
    }
    __threadfence();
  }
  __syncthreads();
}
__device__ __forceinline__ void unit_barrier(unsigned *ctl, int P) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long *word = reinterpret_cast<unsigned long long *>(&ctl[C_BAR]);
    __threadfence();  // this CTA's lists and header before the arrival
    const unsigned long long old = atomicAdd(word, 1ull);
    const unsigned g = (unsigned)(old >> 32);
    if ((unsigned)old == (unsigned)P - 1) {
      atomicAdd(word, (1ull << 32) - (unsigned long long)P);
    } else {
      unsigned it = 0;
      while ((unsigned)(ld_acquire64(word) >> 32) == g) {
        if (++it > WK_SPIN_LIMIT) {
          atomicExch(&ctl[C_ERR], 1u);
          atomicExch(&g_wk_err, 1u);
          break;
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// block-wide exclusive scan of one int per thread
__device__ __forceinline__ int block_excl_scan(int v, int *sh, int *total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sh[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < WK_WARPS ? sh[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < WK_WARPS) sh[lane] = wi - w;
    if (lane == WK_WARPS - 1) sh[WK_WARPS] = wi;
  }
  __syncthreads();
  const int r = sh[warp] + incl - v;
  if (total) *total = sh[WK_WARPS];
  __syncthreads();
  return r;
}

// block-wide sum of one int per thread (result in every thread)
__device__ __forceinline__ int block_sum(int v, int *sh) {
  int t;
  block_excl_scan(v, sh, &t);
  return t;
}

// Warp 0 scans a histogram (in shared memory, nbins <= 2048, a multiple of 32)
// from the top: the bin holding the need-th largest element and the count above it.
__device__ __forceinline__ void top_bin(const uint32_t *H, int nbins, int need, int *bin_out, int *above_out) {
  const int lane = threadIdx.x & 31;
  const int bpl = nbins / 32;
  int cl = 0;
#pragma unroll 1
  for (int q = 0; q < bpl; ++q) cl += (int)H[nbins - 1 - bpl * lane - q];
  int incl = cl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  const int before0 = incl - cl;
  const unsigned hit = __ballot_sync(0xffffffffu, before0 < need && incl >= need);
  if (!hit) {  // need <= 0 or beyond the total
    if (lane == 0) {
      *bin_out = -1;
      *above_out = total;
    }
    return;
  }
  if (lane == __ffs(hit) - 1) {
    int before = before0;
#pragma unroll 1
    for (int q = 0; q < bpl; ++q) {
      const int b = nbins - 1 - bpl * lane - q;
      if (before + (int)H[b] >= need) {
        *bin_out = b;
        *above_out = before;
        break;
      }
      before += (int)H[b];
    }
  }
}

// float64 proxy score of token j (retriever.py:189), the reference's value: fp16 keys times the fp16 group
// sum are exact in float64; every load is issued before the first FMA (d_s <= 8)
__device__ __forceinline__ double exact_score(const uint16_t *kt, int64_t cap, const int *chs, const double *qsum,
                                              int d_s, int64_t j) {
  uint16_t v[WK_MAXDS];
#pragma unroll
  for (int i = 0; i < WK_MAXDS; ++i) v[i] = i < d_s ? __ldg(kt + (size_t)chs[i] * cap + j) : (uint16_t)0;
  double sc = 0.0;
#pragma unroll
  for (int i = 0; i < WK_MAXDS; ++i)
    if (i < d_s) sc = fma(h2d(v[i]), qsum[i], sc);
  return sc;
}

// trace marks of unit 0 (partitions < 32)
constexpr int WK_TRACE_P = 32;
__device__ int g_wk_trace;
__device__ unsigned long long g_wk_mark[WK_TRACE_P][WK_NMARK];
__device__ unsigned int g_wk_path[4];  // select paths taken (units x launches): list 0, list 1, radix, exact radix
__device__ int g_wk_dbg[8];  // unit 0, partition 0, last launch: merged list, band, need_b, keys above all lists
__device__ unsigned long long g_wk_launch[128][3];  // unit 0 per launch: start (partition 0), after the PDL wait, end
__device__ unsigned int g_wk_nlaunch;
__device__ unsigned long long g_wk_uend[64];  // last launch: each unit's final-merge end (trace mode)
__device__ unsigned long long g_wk_lastexit;  // latest CTA exit (trace mode)
#define WK_MARK(i)                                                      \
  do {                                                                  \
    if (trace && blockIdx.y == 0 && blockIdx.x < WK_TRACE_P && tid == 0) \
      g_wk_mark[blockIdx.x][i] = gtime();                               \
  } while (0)

// ---------------------------------------------------------------------------
// gather helpers (out of line: one copy of the code, however many rounds)
// ---------------------------------------------------------------------------
struct GCtx {
  const uint16_t *loc_k, *loc_v, *kdev, *host_kv;
  uint16_t *sv;
  int32_t *stok, *sstamp, *tslot, *hand;
  int64_t capacity, local_capacity, local_offset, ncand;
  int u, n, p0, p1, window;
  bool use_cache, kfd;
};

// row codes: >= 0 cached slot (a hit, stamped with this step), -1 over PCIe, -2 local mirror
__device__ __noinline__ void lookup_rows(const GCtx &c, const int32_t *rows, int32_t *codes, int cnt, int *hits,
                                         int *misses) {
  int h = 0, mm = 0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int64_t idx = rows[i];
    int code = -2;
    if (idx < c.ncand) {
      code = -1;
      if (c.use_cache) {
        const int p = c.tslot[idx];
        if (p >= c.p0 && p < c.p1) {
          code = p;
          c.sstamp[p] = c.n;
        }
      }
      h += code >= 0;
      mm += code < 0;
    }
    codes[i] = code;
  }
  h = __reduce_add_sync(0xffffffffu, h);
  mm = __reduce_add_sync(0xffffffffu, mm);
  if ((threadIdx.x & 31) == 0 && (h | mm)) {
    atomicAdd(hits, h);
    atomicAdd(misses, mm);
  }
}

// a round's HBM copies (every thread): cached (K|V) slot rows, local rows, the keys of misses from
// the token-major copy; one expect-tx per warp, one arrival
__device__ __noinline__ void issue_hbm(const GCtx &c, const int32_t *rows, const int32_t *codes, int cnt,
                                       uint16_t *stage, unsigned long long *bar) {
  const int tid = threadIdx.x, lane = tid & 31;
  uint32_t bytes = 0;
  for (int i = tid; i < cnt; i += blockDim.x) {
    const int code = codes[i];
    bytes += code >= 0 || code == -2 ? WK_D * 4 : (c.kfd ? WK_D * 2 : 0);
  }
  bytes = __reduce_add_sync(0xffffffffu, bytes);
  if (lane == 0 && bytes) mbar_expect(bar, bytes);
  __syncwarp();
  for (int i = tid; i < cnt; i += blockDim.x) {
    const int64_t idx = rows[i];
    const int code = codes[i];
    uint16_t *dst = stage + (size_t)i * 2 * WK_D;
    if (code >= 0) {
      bulk_g2s(dst, c.sv + (size_t)code * 2 * WK_D, WK_D * 4, bar);
    } else if (code == -2) {
      const size_t lr = (size_t)c.u * c.local_capacity + (size_t)(idx - c.local_offset);
      bulk_g2s(dst, c.loc_k + lr * WK_D, WK_D * 2, bar);
      bulk_g2s(dst + WK_D, c.loc_v + lr * WK_D, WK_D * 2, bar);
    } else if (c.kfd) {
      bulk_g2s(dst, c.kdev + ((size_t)c.u * c.capacity + idx) * WK_D, WK_D * 2, bar);
    }
  }
  __syncthreads();
  if (tid == 0) mbar_arrive(bar);
}

// a round's PCIe copies, queued behind the HBM ones: value rows of misses (keys from HBM) or whole
// (K|V) host rows (keys over PCIe); by one warp (with the row cache) or by every thread
__device__ __noinline__ void issue_pcie(const GCtx &c, const int32_t *rows, const int32_t *codes, int cnt,
                                        uint16_t *stage, unsigned long long *bar, bool one_warp) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int t0 = one_warp ? lane : tid, ts = one_warp ? 32 : (int)blockDim.x;
  uint32_t pbytes = 0;
  for (int i = t0; i < cnt; i += ts) {
    const int code = codes[i];
    if (code == -1 || code <= -3) pbytes += c.kfd ? WK_D * 2 : WK_D * 4;
  }
  pbytes = __reduce_add_sync(0xffffffffu, pbytes);
  if (lane == 0 && pbytes) mbar_expect(bar, pbytes);
  __syncwarp();
  for (int i = t0; i < cnt; i += ts) {
    const int code = codes[i];
    if (code != -1 && code > -3) continue;
    const uint16_t *hrow = c.host_kv + ((size_t)c.u * c.capacity + rows[i]) * 2 * WK_D;
    uint16_t *dst = stage + (size_t)i * 2 * WK_D;
    if (c.kfd) bulk_g2s(dst + WK_D, hrow + WK_D, WK_D * 2, bar);
    else bulk_g2s(dst, hrow, WK_D * 4, bar);
  }
  if (one_warp) {
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
  } else {
    __syncthreads();
    if (tid == 0) mbar_arrive(bar);
  }
}

// cache slots for the misses (code -1) among codes[0, cnt), picked by one warp: free slots (empty,
// or not selected in the last `window` steps) of this partition, scanned from its clock hand 32 at
// a time, so the slots recycled are the ones filled longest ago; a miss becomes -3 - slot
// (misses beyond the free slots stay uncached)
__device__ __noinline__ void alloc_slots(const GCtx &c, int32_t *codes, int cnt, int *free_slots) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int Wn = max(1, c.window);
  int need = 0;
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    need += __popc(__ballot_sync(0xffffffffu, i < cnt && codes[i] == -1));
  }
  need = min(need, WK_FCAP);
  const int np = c.p1 - c.p0;
  const int h0 = c.hand && np > 0 ? ((*c.hand % np) + np) % np : 0;
  int found = 0;
  for (int k0 = 0; found < need && k0 < np; k0 += 32) {
    const int kk = k0 + lane;
    int p = 0;
    bool fr = false;
    if (kk < np) {
      p = c.p0 + (h0 + kk) % np;
      fr = c.stok[p] < 0 || c.sstamp[p] <= c.n - Wn;
    }
    const unsigned b = __ballot_sync(0xffffffffu, fr);
    const int pos = found + __popc(b & lt);
    if (fr && pos < need) {
      free_slots[pos] = p;
      const int old = c.stok[p];  // the recycled slot's token loses its entry (unless it moved on)
      if (old >= 0) atomicCAS(&c.tslot[old], p, -1);
      if (pos == need - 1 && c.hand) *c.hand = (h0 + kk + 1) % np;
    }
    found += __popc(b);
  }
  __syncwarp();
  const int used = min(found, need);
  int ord = 0;
  for (int i0 = 0; i0 < cnt; i0 += 32) {
    const int i = i0 + lane;
    const bool mm = i < cnt && codes[i] == -1;
    const unsigned b = __ballot_sync(0xffffffffu, mm);
    const int kk = ord + __popc(b & lt);
    if (mm && kk < used) codes[i] = -3 - free_slots[kk];
    ord += __popc(b);
  }
  __syncwarp();
}

// The rare select paths (the aimed lists missed or overflowed): an exact radix
// select of the k-th fp32 key through global histograms, then the band around
// it -- ranked in SMEM when small, else by an exact radix select over (float64
// score, index).  Out of line, so the common path's code stays compact (its
// instruction fetch is on the critical path).  Returns the key above which
// every key is selected; S.bitmap and S.pcount hold the rest.
struct FbArgs {
  const uint16_t *kt;
  int64_t cap;
  uint32_t *keys32;
  unsigned char *smem;
  Hdr *htab;
  UnitWs W;
  int64_t j0, chunk;
  int m, P, r, k, d_s, buf;
  double eps2;
};
__device__ __noinline__ uint32_t select_fallback(WSh &S, const FbArgs &f, int &path) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  (void)lane;
  const uint16_t *kt = f.kt;
  const int64_t cap = f.cap;
  const uint32_t *keys32 = f.keys32;
  unsigned char *smem = f.smem;
  Hdr *htab = f.htab;
  const UnitWs W = f.W;
  const int64_t j0 = f.j0, chunk = f.chunk;
  const int m = f.m, P = f.P, r = f.r, k = f.k, d_s = f.d_s, buf = f.buf;
  const double eps2 = f.eps2;
      // ---- fallback A: exact k-th largest fp32 key by radix passes over global histograms ----
      if (tid == 0 && r == 0) atomicExch(&W.ctl[C_FALLBACK], 1u);
      uint32_t prefix = 0u;
      int need = k, bits = 0;
      for (int pass = 0; pass < 3; ++pass) {
        const int nbits = pass < 2 ? 11 : 10, shift = 32 - bits - nbits;
        for (int i = tid; i < WK_HB; i += blockDim.x) S.hist[i] = 0u;
        __syncthreads();
        for (int e = tid; e < m; e += blockDim.x) {
          const uint32_t key = keys32[e];
          if (bits > 0 && (key >> (32 - bits)) != prefix) continue;
          atomicAdd(&S.hist[(key >> shift) & ((1u << nbits) - 1u)], 1u);
        }
        __syncthreads();
        unsigned *gh = W.hist + (size_t)pass * WK_HB;
        for (int i = tid; i < (1 << nbits); i += blockDim.x)
          if (S.hist[i]) atomicAdd(&gh[i], S.hist[i]);
        unit_barrier(W.ctl, P);
        for (int i = tid; i < (1 << nbits); i += blockDim.x) S.hist[i] = __ldcg(gh + i);
        __syncthreads();
        if (warp == 0) top_bin(S.hist, 1 << nbits, need, &S.rdigit, &S.rabove);
        __syncthreads();
        prefix = (prefix << nbits) | (uint32_t)max(0, S.rdigit);
        need -= S.rabove;
        bits += nbits;
        __syncthreads();
      }
      // the band around the exact k-th fp32 value, resolved with lists (keys in the band only)
      const float vk = from_ord32(prefix);
      if (tid == 0) S.e_lo = S.e_hi = (double)vk;  // (the next step's aim)
      const uint32_t ord_lo = ord32(__double2float_rd((double)vk - eps2));
      const uint32_t ord_hi = ord32(__double2float_ru((double)vk + eps2));
      LEnt *mylist = W.lists + ((size_t)buf * P + r) * WK_LCAP;
      if (tid == 0) {
        S.list_count = 0;
        S.above = 0;
      }
      __syncthreads();
      int above = 0;
      for (int e = tid; e < m; e += blockDim.x) {
        const uint32_t key = keys32[e];
        above += key > ord_hi;
        if (key >= ord_lo && key <= ord_hi) {
          const int pos = atomicAdd(&S.list_count, 1);
          if (pos < WK_LCAP) mylist[pos].kidx = ((unsigned long long)key << 32) | (uint32_t)(j0 + e);
        }
      }
      above = block_sum(above, S.scan);
      if (tid == 0) {
        Hdr h = {};
        h.above = (uint32_t)above;
        h.count = (uint32_t)S.list_count;
        h.llo = ord_lo;
        h.lhi = ord_hi;
        W.hdr[(size_t)buf * P + r] = h;
      }
      unit_barrier(W.ctl, P);
      for (int i = tid; i < P; i += blockDim.x) {
        const uint4 *src = reinterpret_cast<const uint4 *>(W.hdr + (size_t)buf * P + i);
        uint4 *dst = reinterpret_cast<uint4 *>(htab + i);
#pragma unroll
        for (int q = 0; q < 4; ++q) dst[q] = __ldcg(src + q);
      }
      __syncthreads();
      if (tid == 0) {
        int A = 0, L = 0, ovf = 0;
        for (int i = 0; i < P; ++i) {
          S.lstart[i] = L;
          A += (int)htab[i].above;
          L += (int)min(htab[i].count, (uint32_t)WK_LCAP);
          ovf |= htab[i].count > (uint32_t)WK_LCAP;
        }
        S.lstart[P] = L;
        S.A = A;
        S.Ltot = L;
        S.ovf = ovf || L > WK_BAND;
      }
      __syncthreads();
      const int need_b = k - S.A;  // every key above the band is selected
      if (!S.ovf) {
        path = 2;
        const int nb = S.Ltot;
        for (int t = tid; t < nb; t += blockDim.x) {
          int lo = 0, hi = P;
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (S.lstart[mid] <= t) lo = mid;
            else hi = mid;
          }
          const unsigned long long c = __ldcg(&W.lists[((size_t)buf * P + lo) * WK_LCAP + (t - S.lstart[lo])].kidx);
          S.band_idx[t] = (uint32_t)c;
          S.band_key[t] = orderable(exact_score(kt, cap, S.chs, S.qsum, d_s, (uint32_t)c));
        }
        for (int i = tid; i < P; i += blockDim.x) S.pcount[i] = (int)htab[i].above;
        for (int i = tid; i < WK_MAXM / 32; i += blockDim.x) S.bitmap[i] = 0u;
        __syncthreads();
        for (int b = tid; b < nb; b += blockDim.x) {
          const unsigned long long kb = S.band_key[b];
          const uint32_t ib = S.band_idx[b];
          int beaten = 0;
          for (int o = 0; o < nb; ++o) {
            const unsigned long long ko = S.band_key[o];
            beaten += (ko > kb) || (ko == kb && S.band_idx[o] > ib);
          }
          if (beaten < need_b) {
            atomicAdd(&S.pcount[(int)((int64_t)ib / chunk)], 1);
            if ((int64_t)ib >= j0 && (int64_t)ib < j0 + m)
              atomicOr(&S.bitmap[((int64_t)ib - j0) >> 5], 1u << (((int64_t)ib - j0) & 31));
          }
        }
        __syncthreads();
      } else {
        // ---- fallback B: the band is too large to rank in SMEM (e.g. massive exact ties): exact
        // radix select over the composite (float64 score, index) of the band members ----
        path = 3;
        unsigned long long *mkey = reinterpret_cast<unsigned long long *>(smem);        // [<= m]
        uint16_t *midx = reinterpret_cast<uint16_t *>(smem + WK_MAXM * 8);              // [<= m]
        if (tid == 0) S.nm = 0;
        __syncthreads();
        for (int e = tid; e < m; e += blockDim.x) {
          const uint32_t key = keys32[e];
          if (key < ord_lo || key > ord_hi) continue;
          const int pos = atomicAdd(&S.nm, 1);
          mkey[pos] = orderable(exact_score(kt, cap, S.chs, S.qsum, d_s, j0 + e));
          midx[pos] = (uint16_t)e;
        }
        __syncthreads();
        const int nm = S.nm;
        unsigned long long kp = 0ull;  // prefix of the float64 key
        uint32_t jp = 0u;              // prefix of the token index
        int rneed = need_b, kbits = 0, jbits = 0;
        for (int pass = 0; pass < 9; ++pass) {
          const bool onk = pass < 6;
          const int nbits = onk ? (pass < 5 ? 11 : 9) : (pass < 8 ? 11 : 10);
          for (int i = tid; i < WK_HB; i += blockDim.x) S.hist[i] = 0u;
          __syncthreads();
          for (int i = tid; i < nm; i += blockDim.x) {
            const unsigned long long key = mkey[i];
            const uint32_t j = (uint32_t)(j0 + midx[i]);
            if (onk) {
              if (kbits > 0 && (key >> (64 - kbits)) != kp) continue;
              atomicAdd(&S.hist[(uint32_t)(key >> (64 - kbits - nbits)) & ((1u << nbits) - 1u)], 1u);
            } else {
              if (key != kp) continue;
              if (jbits > 0 && (j >> (32 - jbits)) != jp) continue;
              atomicAdd(&S.hist[(j >> (32 - jbits - nbits)) & ((1u << nbits) - 1u)], 1u);
            }
          }
          __syncthreads();
          unsigned *gh = W.hist + (size_t)(3 + pass) * WK_HB;
          for (int i = tid; i < (1 << nbits); i += blockDim.x)
            if (S.hist[i]) atomicAdd(&gh[i], S.hist[i]);
          unit_barrier(W.ctl, P);
          for (int i = tid; i < (1 << nbits); i += blockDim.x) S.hist[i] = __ldcg(gh + i);
          __syncthreads();
          if (warp == 0) top_bin(S.hist, 1 << nbits, rneed, &S.rdigit, &S.rabove);
          __syncthreads();
          const uint32_t dg = (uint32_t)max(0, S.rdigit);
          if (onk) {
            kp = (kp << nbits) | dg;
            kbits += nbits;
          } else {
            jp = (jp << nbits) | dg;
            jbits += nbits;
          }
          rneed -= S.rabove;
          __syncthreads();
        }
        // selected band members: composite >= (kp, jp); exactly need_b of them over the unit
        for (int i = tid; i < WK_MAXM / 32; i += blockDim.x) S.bitmap[i] = 0u;
        __syncthreads();
        for (int i = tid; i < nm; i += blockDim.x) {
          const unsigned long long key = mkey[i];
          const uint32_t j = (uint32_t)(j0 + midx[i]);
          if (key > kp || (key == kp && j >= jp)) atomicOr(&S.bitmap[midx[i] >> 5], 1u << (midx[i] & 31));
        }
        __syncthreads();
        // per-partition counts are not derivable here: exchange them
        int c = 0;
        for (int e = tid; e < m; e += blockDim.x)
          c += keys32[e] > ord_hi || ((S.bitmap[e >> 5] >> (e & 31)) & 1u);
        c = block_sum(c, S.scan);
        if (tid == 0) W.counts[r] = c;
        unit_barrier(W.ctl, P);
        for (int i = tid; i < P; i += blockDim.x) S.pcount[i] = __ldcg(W.counts + i);
        __syncthreads();
      }
  return ord_hi;
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
// Code-size discipline: one launch executes this kernel's common path once per
// SM, and SASS beyond the ~16-32 KB instruction cache streams in from L2 at
// ~5-10 KB/us per SM (tools/icache_probe.cu).  So loops stay rolled unless the
// unrolled body is the point, reductions use the single-instruction REDUX, and
// the rare select paths live out of line (select_fallback).
__device__ __forceinline__ float warp_sum_rolled(float v) {
#pragma unroll 1
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll 1
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// merge cnt partials (fixed order) into dst (a partial) or into the unit's
// head outputs; the partials' maxima and sums are staged in SMEM first
__device__ __noinline__ void merge_partials_w(const float *src, int cnt, int PF, int gmax, int G, float *mls,
                                              float *dst, float *out) {
  const int tid = threadIdx.x;
  // the first element's partials are requested before the maxima/sums are staged: one round trip
  float v[32];  // every partial of this element in flight at once (cnt <= 32)
#pragma unroll
  for (int q = 0; q < 32; ++q) v[q] = q < cnt && tid < G * WK_D ? __ldcg(src + (size_t)q * PF + tid) : 0.0f;
  for (int t = tid; t < cnt * 2 * gmax; t += blockDim.x) {
    const int q = t / (2 * gmax), j = t % (2 * gmax);
    mls[t] = __ldcg(src + (size_t)q * PF + gmax * WK_D + j);
  }
  __syncthreads();
  for (int i = tid; i < G * WK_D; i += blockDim.x) {
    const int h = i / WK_D;
    if (i != tid) {
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = q < cnt ? __ldcg(src + (size_t)q * PF + i) : 0.0f;
    }
    float M = -INFINITY;
#pragma unroll 1
    for (int q = 0; q < cnt; ++q) M = fmaxf(M, mls[q * 2 * gmax + h]);
    float L = 0.0f, Ac = 0.0f;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const float mq = q < cnt ? mls[q * 2 * gmax + h] : -INFINITY;
      if (mq == -INFINITY) continue;
      const float sc = exp2f(mq - M);
      L = fmaf(sc, mls[q * 2 * gmax + gmax + h], L);
      Ac = fmaf(sc, v[q], Ac);
    }
    if (out) {
      out[i] = Ac / L;
    } else {
      dst[i] = Ac;
      if ((i % WK_D) == 0) {
        dst[gmax * WK_D + h] = M;
        dst[gmax * WK_D + gmax + h] = L;
      }
    }
  }
  __syncthreads();
}

template <int GMAX>
__global__ void __maxnreg__(96) sparse_wide_kernel(SL s, WArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ WSh S;
  uint16_t *raw = reinterpret_cast<uint16_t *>(smem);
  uint32_t *keys32 = reinterpret_cast<uint32_t *>(smem + WK_RAW);
  float *qs = reinterpret_cast<float *>(smem + WK_RAW + WK_KEYS);  // [G][D] * log2(e)/sqrt(d)
  const int u = blockIdx.y, r = blockIdx.x, P = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int trace = g_wk_trace;
  const int G = a.G, d_s = a.d_s;
  const int64_t n = *s.len;  // same-layer launches never overlap under PDL (pdl_note)
  const int n_sink = s.n_sink;
  const int k = a.n_topk + n_sink;
  const int64_t ncand = n > a.n_local ? n - a.n_local : 0;
  const int64_t chunk = ((ncand + P - 1) / P + 15) & ~int64_t(15);
  const int64_t j0 = (int64_t)r * chunk;
  const int m = (int)(j0 < ncand ? imin64(chunk, ncand - j0) : 0);
  const bool select_all = n <= (int64_t)a.n_local + k;
  const uint16_t *kt = s.kt + (size_t)u * WK_D * s.capacity;
  const unsigned long long t_start = trace ? gtime() : 0ull;
  WK_MARK(0);
  if (tid == 0) {
    mbar_init(&S.bar_tma);
    mbar_init(&S.bar_hbm);
    mbar_init(&S.bar_pcie);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    S.klo = 0xffffffffu;
    S.khi = 0u;
    S.nval = 0;
    S.fsum = S.fsq = 0.0f;
  }
  if (!select_all && tid < d_s) S.chs[tid] = a.channels[(size_t)u * d_s + tid];
  __syncthreads();
  // ---- 0. prologue: the partition's scorer columns into SMEM (TMA), before the PDL wait ----
  if (!select_all && m > 0 && tid == 0) {
    const int64_t m8 = imin64(((int64_t)m + 7) & ~int64_t(7), s.capacity - j0);
    mbar_arrive_expect(&S.bar_tma, (uint32_t)(d_s * m8 * 2));
#pragma unroll 1
    for (int i = 0; i < d_s; ++i)
      bulk_g2s(raw + (size_t)i * WK_MAXM, kt + (size_t)S.chs[i] * s.capacity + j0, (uint32_t)(m8 * 2), &S.bar_tma);
  }
  // The step's new row goes to the pinned host store now, not in the final append: nothing reads row
  // n during this step (attend before append), and a posted PCIe store still in flight when the grid
  // ends delays its completion -- and the next layer's PDL wait -- by ~3.5 us (tools/pdl_probe.cu).
  if (a.new_keys && r == P - 1 && tid < 2 * WK_D / 8) {
    const int half = tid / (WK_D / 8), c8 = (tid % (WK_D / 8)) * 8;  // 16-byte pieces of K then V
    const uint16_t *src = (half ? a.new_values : a.new_keys) + (size_t)u * WK_D + c8;
    *reinterpret_cast<uint4 *>(s.host_kv + (((size_t)u * s.capacity + n) * 2 + half) * WK_D + c8) =
        *reinterpret_cast<const uint4 *>(src);
  }
  // every CTA of this grid is resident once all have passed this point, so the next layer's kernel
  // (which only reads its own layer before its own wait) may start placing CTAs
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ unsigned lslot;
  if (trace && u == 0 && r == 0 && tid == 0) {  // (after the wait: the previous launch has ended)
    lslot = atomicAdd(&g_wk_nlaunch, 1u) & 127u;
    g_wk_launch[lslot][0] = t_start;
    g_wk_launch[lslot][1] = gtime();
  }
  WK_MARK(1);
  const UnitWs W = unit_ws(a, u, P);
#pragma unroll 1
  for (int i = tid; i < G * WK_D; i += blockDim.x)
    qs[i] = h2f(a.queries[(size_t)u * G * WK_D + i]) * (1.4426950408889634f / sqrtf((float)WK_D));
  if (!select_all && tid < d_s) {  // every load of a channel's group sum and channel max in flight at once
    const int ch = S.chs[tid];
    uint16_t qv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) qv[j] = j < G ? a.queries[((size_t)u * G + j) * WK_D + ch] : (uint16_t)0;
    const float cm = s.chmax[(size_t)u * WK_D + ch];
    double q = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < G) q += h2d(qv[j]);  // retriever.py:189 (group sum, in head order)
    S.qsum[tid] = q;
    S.qsum32[tid] = (float)q;
    S.eps_term[tid] = (double)cm * fabs(q);
  }
  __syncthreads();
  if (tid == 0 && !select_all) {
    double e = 0.0;
#pragma unroll 1
    for (int i = 0; i < d_s; ++i) e += S.eps_term[i];
    // |fp32 score - float64 score| <= (d_s + 1) 2^-24 sum_i max|K_i| |q_i| (a d_s-term fmaf chain plus
    // the query's fp32 rounding); (d_s + 2), at least 16, as in the cluster kernel
    S.band_eps = e * fmax(16.0, (double)d_s + 2.0) * 5.9604644775390625e-08;
  }
  uint32_t ord_def = 0xffffffffu;  // keys above are selected (plus S.bitmap members)
  int path = -1;
  // gather context
  const int n_loc = (int)(n - ncand);
  const int n_loc_mine = n_loc > r ? (n_loc - r + P - 1) / P : 0;
  const int CS = s.cache_slots;
  const bool kfd = a.keys_from_device != 0;
  const bool use_cache = CS > 0 && kfd;  // (K|V) slot cache (needs the token-major keys: dispatch checks s.kdev)
  uint16_t *stage = reinterpret_cast<uint16_t *>(smem);
  GCtx gc;
  {
    const int spc = (CS + P - 1) / P;  // this partition owns the slots [p0, p1)
    gc.loc_k = s.loc_k;
    gc.loc_v = s.loc_v;
    gc.kdev = s.kdev;
    gc.host_kv = s.host_kv;
    gc.sv = use_cache ? s.slot_v + (size_t)u * CS * 2 * WK_D : nullptr;
    gc.stok = use_cache ? s.slot_tok + (size_t)u * CS : nullptr;
    gc.sstamp = use_cache ? s.slot_stamp + (size_t)u * CS : nullptr;
    gc.tslot = use_cache ? s.tok_slot + (size_t)u * s.capacity : nullptr;
    gc.hand = use_cache && s.slot_hand ? s.slot_hand + (size_t)u * TKV_MAX_PARTS + r : nullptr;
    gc.capacity = s.capacity;
    gc.local_capacity = s.local_capacity;
    gc.local_offset = s.local_offset;
    gc.ncand = ncand;
    gc.u = u;
    gc.n = (int)n;
    gc.p0 = min(CS, r * spc);
    gc.p1 = min(CS, gc.p0 + spc);
    gc.window = s.cache_window;
    gc.use_cache = use_cache;
    gc.kfd = kfd;
  }
  if (tid == 0) S.hits = S.misses = 0;
  if (!select_all) {
    // ---- 1. fp32 proxy scores -> order-preserving keys; the partition's moments ----
    if (m > 0) mbar_wait(&S.bar_tma, 0);
    WK_MARK(2);
    {
      uint32_t klo = 0xffffffffu, khi = 0u;
      float fsum = 0.0f, fsq = 0.0f;
      int nval = 0;
#pragma unroll 1
      for (int e = tid * 8; e < m; e += WK_THREADS * 8) {
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
#pragma unroll 1
        for (int i = 0; i < d_s; ++i) {  // same fmaf order as the cluster kernel (the eps bound)
          const uint4 v = *reinterpret_cast<const uint4 *>(raw + (size_t)i * WK_MAXM + e);
          const float qv = S.qsum32[i];
          const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = fmaf(h2f((uint16_t)(w4[q >> 1] >> (16 * (q & 1)))), qv, acc[q]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const bool valid = e + q < m, sink = j0 + e + q < n_sink;
          const uint32_t key = sink ? 0xffffffffu : ord32(acc[q]);
          if (valid) keys32[e + q] = key;
          if (valid && !sink) {
            klo = min(klo, key);
            khi = max(khi, key);
            fsum += acc[q];
            fsq = fmaf(acc[q], acc[q], fsq);
            ++nval;
          }
        }
      }
      klo = __reduce_min_sync(0xffffffffu, klo);
      khi = __reduce_max_sync(0xffffffffu, khi);
      nval = __reduce_add_sync(0xffffffffu, nval);
      fsum = warp_sum_rolled(fsum);
      fsq = warp_sum_rolled(fsq);
      if (lane == 0) {
        atomicMin(&S.klo, klo);
        atomicMax(&S.khi, khi);
        atomicAdd(&S.nval, nval);
        S.r_sum[warp] = (double)fsum;  // summed in warp order below: the moments (and so the aim, the
        S.r_sq[warp] = (double)fsq;    // partitions' aims and hints) are deterministic
      }
      __syncthreads();
      if (tid == 0) {
        double su = 0.0, sq = 0.0;
#pragma unroll 1
        for (int w = 0; w < WK_WARPS; ++w) {
          su += S.r_sum[w];
          sq += S.r_sq[w];
        }
        S.fsum = (float)su;
        S.fsq = (float)sq;
        const int nv = S.nval;
        S.mu = nv ? su / nv : 0.0;
        S.sd = nv ? sqrt(fmax(sq / nv - S.mu * S.mu, 0.0)) : 0.0;
      }
    }
    WK_MARK(3);
    const double eps2 = 2.0 * S.band_eps;
    const double N = (double)(ncand - imin64(ncand, n_sink));
    float2 *hint = s.part_hint ? reinterpret_cast<float2 *>(s.part_hint) + (size_t)u * TKV_MAX_PARTS + r : nullptr;
    const float2 hv = hint ? *hint : make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    // after the first list pass: [merged lists | the unit's headers]
    LEnt *cand = reinterpret_cast<LEnt *>(smem);
    Hdr *htab = reinterpret_cast<Hdr *>(smem + WK_GCAP * 16);
    int buf = 0, dir = 0;
    bool done = false;
    // ---- 2. aimed list attempts ----
#pragma unroll 1
    for (int attempt = 0; attempt < 2 && !done; ++attempt) {
      if (tid == 0) {  // this partition's window (values) and list range (keys)
        double wlo, whi;
        const double mu = S.mu, sd = S.sd;
        if (attempt == 0) {
          double c, w;
          if (isfinite(hv.x) && sd > 0.0) {
            c = mu + (double)hv.x * sd;
            w = isfinite(hv.y) ? fmin(0.3, fmax(0.06, 3.0 * (double)hv.y)) : 0.15;
          } else {
            c = mu + normal_upper_quantile((double)(k - n_sink) / fmax(N, 1.0)) * sd;
            w = 0.12;
          }
          wlo = c - w * sd;
          whi = c + w * sd;
        } else {  // the unit's moments: extend beyond the side of the missed window that holds the threshold
          wlo = dir > 0 ? (double)S.XHf : (double)S.XLf - 0.6 * S.gsd;
          whi = dir > 0 ? (double)S.XHf + 0.6 * S.gsd : (double)S.XLf;
          wlo = fmax(wlo, (double)from_ord32(S.gklo));
          whi = fmin(whi, (double)from_ord32(S.gkhi));
        }
        if (m == 0 || S.nval == 0) {  // nothing to aim with: this partition must not narrow the intersection
          S.llo = 0u;
          S.lhi = 0xffffffffu;
          S.wlo_f = -INFINITY;
          S.whi_f = INFINITY;
        } else {
          if (!(whi >= wlo) || !isfinite(wlo) || !isfinite(whi)) wlo = whi = mu;
          S.wlo_f = __double2float_rd(wlo);
          S.whi_f = __double2float_ru(whi);
          S.llo = ord32(__double2float_rd(wlo - 2.0 * eps2));
          S.lhi = ord32(__double2float_ru(whi + 2.0 * eps2));
        }
        S.list_count = 0;
        S.above = 0;
      }
      __syncthreads();
      // list keys in [llo, lhi] (global), count keys above lhi
      {
        const uint32_t llo = S.llo, lhi = S.lhi;
        LEnt *mylist = W.lists + ((size_t)buf * P + r) * WK_LCAP;
        int above = 0;
#pragma unroll 1
        for (int g = 0; g < 2; ++g) {  // uniform trip count: the warp votes below need every lane
          const int e = g * WK_THREADS * 8 + tid * 8;
          uint32_t mask = 0u;
          if (e < m) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint32_t key = keys32[e + q];
              const bool valid = e + q < m;
              above += valid && key > lhi;
              mask |= (uint32_t)(valid && key >= llo && key <= lhi) << q;
            }
          }
          {  // keys above the list are selected whenever this attempt succeeds: their mask words
            uint32_t amsk = 0u;
            if (e < m) {
#pragma unroll
              for (int q = 0; q < 8; ++q) amsk |= (uint32_t)(e + q < m && keys32[e + q] > lhi) << q;
            }
            amsk <<= 8 * (lane & 3);
            amsk |= __shfl_xor_sync(0xffffffffu, amsk, 1);
            amsk |= __shfl_xor_sync(0xffffffffu, amsk, 2);
            if ((lane & 3) == 0 && g * WK_THREADS * 8 + tid * 8 < WK_MAXM) S.amask[(g * WK_THREADS * 8 + tid * 8) >> 5] = amsk;
          }
          const int c = __popc(mask);
          const int incl = warp_incl_scan(c, lane);
          const int wtot = __shfl_sync(0xffffffffu, incl, 31);
          int base = 0;
          if (lane == 31 && wtot) base = atomicAdd(&S.list_count, wtot);
          int pos = __shfl_sync(0xffffffffu, base, 31) + incl - c;
#pragma unroll 1
          while (mask) {
            const int q = __ffs(mask) - 1;
            mask &= mask - 1u;
            if (pos < WK_LCAP) {
              // exact_score: from the SMEM columns on the first attempt (same channel order); later
              // attempts run after the merged lists overwrote them, and read the scorer copy in HBM
              double sc = 0.0;
              if (attempt == 0) {
#pragma unroll 1
                for (int i = 0; i < d_s; ++i) sc = fma(h2d(raw[(size_t)i * WK_MAXM + e + q]), S.qsum[i], sc);
              } else {
                sc = exact_score(kt, s.capacity, S.chs, S.qsum, d_s, j0 + e + q);
              }
              LEnt le;
              le.kidx = ((unsigned long long)keys32[e + q] << 32) | (uint32_t)(j0 + e + q);
              le.s = sc;
              mylist[pos] = le;
            }
            ++pos;
          }
        }
        above = __reduce_add_sync(0xffffffffu, above);
        if (lane == 0 && above) atomicAdd(&S.above, above);
      }
      __syncthreads();
      if (tid == 0) {
        Hdr h;
        h.above = (uint32_t)S.above;
        h.count = (uint32_t)S.list_count;
        h.llo = S.llo;
        h.lhi = S.lhi;
        h.klo = S.klo;
        h.khi = S.khi;
        h.nval = (uint32_t)S.nval;
        h.pad0 = 0;
        h.sum = (double)S.fsum;
        h.sq = (double)S.fsq;
        h.wlo = S.wlo_f;
        h.whi = S.whi_f;
        h.pad1[0] = h.pad1[1] = 0;
        W.hdr[(size_t)buf * P + r] = h;
      }
      WK_MARK(4 + attempt);
      unit_barrier(W.ctl, P);
      WK_MARK(6 + attempt);
      // ---- resolve (every CTA of the unit computes the same) ----
#pragma unroll 1
      for (int i = tid; i < P; i += blockDim.x) {
        const uint4 *src = reinterpret_cast<const uint4 *>(W.hdr + (size_t)buf * P + i);
        uint4 *dst = reinterpret_cast<uint4 *>(htab + i);
        const uint4 x0 = __ldcg(src), x1 = __ldcg(src + 1), x2 = __ldcg(src + 2), x3 = __ldcg(src + 3);
        dst[0] = x0;
        dst[1] = x1;
        dst[2] = x2;
        dst[3] = x3;
      }
      if (tid == 0) {
        S.cnt_a = S.cnt_b = S.cnt_c = 0;
        S.band_n = 0;
        S.band_ovf = 0;
      }
      __syncthreads();
      if (attempt == 0) WK_MARK(14);
      if (warp == 0) {
        int A = 0, ovf = 0, nv = 0, run = 0;
        uint32_t LL = 0u, LH = 0xffffffffu, glo = 0xffffffffu, ghi = 0u, xl = 0u, xh = 0xffffffffu;
        float su = 0.0f, sq = 0.0f;
        const int per = (P + 31) / 32;
#pragma unroll 1
        for (int q = 0; q < per; ++q) {
          const int i = lane * per + q;
          if (i >= P) break;
          const Hdr &h = htab[i];
          A += (int)h.above;
          run += (int)min(h.count, (uint32_t)WK_LCAP);
          ovf |= h.count > (uint32_t)WK_LCAP;
          LL = max(LL, h.llo);
          LH = min(LH, h.lhi);
          xl = max(xl, ord32(h.wlo));
          xh = min(xh, ord32(h.whi));
          if (h.nval) {
            glo = min(glo, h.klo);
            ghi = max(ghi, h.khi);
          }
          su += (float)h.sum;
          sq += (float)h.sq;
          nv += (int)h.nval;
        }
        const int incl = warp_incl_scan(run, lane);
        int p0 = incl - run;
#pragma unroll 1
        for (int q = 0; q < per; ++q) {
          const int i = lane * per + q;
          if (i >= P) break;
          S.lstart[i] = p0;
          p0 += (int)min(htab[i].count, (uint32_t)WK_LCAP);
        }
        A = __reduce_add_sync(0xffffffffu, A);
        ovf = __reduce_or_sync(0xffffffffu, ovf);
        nv = __reduce_add_sync(0xffffffffu, nv);
        LL = __reduce_max_sync(0xffffffffu, LL);
        LH = __reduce_min_sync(0xffffffffu, LH);
        xl = __reduce_max_sync(0xffffffffu, xl);
        xh = __reduce_min_sync(0xffffffffu, xh);
        glo = __reduce_min_sync(0xffffffffu, glo);
        ghi = __reduce_max_sync(0xffffffffu, ghi);
        su = warp_sum_rolled(su);
        sq = warp_sum_rolled(sq);
        if (lane == 31) {
          S.lstart[P] = incl;
          S.Ltot = incl;
          S.A = A;
          S.ovf = ovf || incl > WK_GCAP;
          S.LL = LL;
          S.LH = LH;
          S.XL = xl;
          S.XH = xh;
          S.XLf = from_ord32(xl);
          S.XHf = from_ord32(xh);
          S.gklo = glo;
          S.gkhi = ghi;
          const double gm = nv ? (double)su / nv : 0.0;
          S.gmu = gm;
          S.gsd = nv ? sqrt(fmax((double)sq / nv - gm * gm, 0.0)) : 0.0;
          S.status = 0;
          S.dir = 0;
        }
      }
      __syncthreads();
      if (attempt == 0) WK_MARK(15);
      if (trace && u == 0 && r == 0 && tid == 0 && attempt == 0) {
        g_wk_dbg[5] = S.ovf;
        g_wk_dbg[6] = S.Ltot;
        g_wk_dbg[7] = (int)S.XL - (int)S.XH;
      }
      if (!S.ovf && S.XL <= S.XH) {
        const int Ltot = S.Ltot;
        const uint32_t XL = S.XL, XH = S.XH;
        int ab = 0, in = 0;
#pragma unroll 1
        for (int t = tid; t < Ltot; t += blockDim.x) {
          int lo = 0, hi = P;  // last partition with lstart <= t
#pragma unroll 1
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (S.lstart[mid] <= t) lo = mid;
            else hi = mid;
          }
          const LEnt *src = W.lists + ((size_t)buf * P + lo) * WK_LCAP + (t - S.lstart[lo]);
          LEnt le;
          le.kidx = __ldcg(&src->kidx);
          le.s = __ldcg(&src->s);
          cand[t] = le;
          const uint32_t key = (uint32_t)(le.kidx >> 32);
          ab += key > XH;
          in += key >= XL && key <= XH;
        }
#pragma unroll 1
        for (int i = tid; i < WK_NB; i += blockDim.x) S.hist[i] = 0u;
        ab = __reduce_add_sync(0xffffffffu, ab);
        in = __reduce_add_sync(0xffffffffu, in);
        if (lane == 0) {
          atomicAdd(&S.cnt_a, ab);
          atomicAdd(&S.cnt_b, in);
        }
        __syncthreads();
        if (attempt == 0) WK_MARK(16);
        const int need = k - (S.A + S.cnt_a);
        int st = 0, dr = 0;
        if (need <= 0) dr = 1;
        else if (need > S.cnt_b) dr = -1;
        else st = 1;
        if (st) {
          // histogram of the in-window entries over [XL, XH] (values): the bin of the need-th largest
          const float r_lo = S.XLf, r_hi = S.XHf;
          const bool flat = !(r_hi > r_lo);
          const float scale = flat ? 0.0f : (float)WK_NB / (r_hi - r_lo);
#pragma unroll 1
          for (int t = tid; t < Ltot; t += blockDim.x) {
            const uint32_t key = (uint32_t)(cand[t].kidx >> 32);
            if (key < XL || key > XH) continue;
            const int b = flat ? 0 : min(WK_NB - 1, max(0, (int)((from_ord32(key) - r_lo) * scale)));
            atomicAdd(&S.hist[b], 1u);
          }
          __syncthreads();
          {
            // the bin holding the need-th largest entry: thread t owns bins NB-1-2t, NB-2-2t (descending)
            const int b0 = WK_NB - 1 - 2 * tid, b1 = b0 - 1;
            const int h0 = (int)S.hist[b0], c2 = h0 + (int)S.hist[b1];
            const int incl = warp_incl_scan(c2, lane);
            if (lane == 31) S.wtot[warp] = incl;
            if (tid == 0) S.bin = -1;
            __syncthreads();
            int pre = incl - c2;
#pragma unroll 1
            for (int w = 0; w < warp; ++w) pre += S.wtot[w];
            if (pre < need && pre + c2 >= need) S.bin = pre + h0 >= need ? b0 : b1;
          }
          __syncthreads();
          if (attempt == 0) WK_MARK(17);
          const int B = S.bin;
          const double delta =
              9.5367431640625e-07 * (fabs((double)r_lo) + fabs((double)r_hi) + ((double)r_hi - (double)r_lo));
          const double e_lo = (flat || B <= 0) ? (double)r_lo : (double)r_lo + (double)B / (double)scale - delta;
          const double e_hi = (flat || B == WK_NB - 1 || B < 0) ? (double)r_hi
                                                               : (double)r_lo + (double)(B + 1) / (double)scale + delta;
          const uint32_t ord_lo = ord32(__double2float_rd(e_lo - eps2));
          const uint32_t ord_hi = ord32(__double2float_ru(e_hi + eps2));
          // the band must lie where every list is complete
          st = B >= 0 && ord_lo >= S.LL && ord_hi <= S.LH;
          if (st) {
#pragma unroll 1
            for (int t = tid; t < Ltot; t += blockDim.x) {
              const uint32_t key = (uint32_t)(cand[t].kidx >> 32);
              if (key > ord_hi) {
                atomicAdd(&S.cnt_c, 1);
              } else if (key >= ord_lo) {
                const int slot = atomicAdd(&S.band_n, 1);
                if (slot < WK_BAND) {
                  S.band_idx[slot] = (uint32_t)cand[t].kidx;
                  S.band_key[slot] = orderable(cand[t].s);  // the exact score came with the list
                } else {
                  S.band_ovf = 1;
                }
              }
            }
            __syncthreads();
            if (attempt == 0) WK_MARK(18);
            const int nb = min(S.band_n, WK_BAND);
            const int need_b = k - S.A - S.cnt_c;
            if (trace && u == 0 && r == 0 && tid == 0) {
              g_wk_dbg[0] = Ltot;
              g_wk_dbg[1] = S.band_n;
              g_wk_dbg[2] = need_b;
              g_wk_dbg[3] = S.A;
              g_wk_dbg[4] = S.cnt_b;
            }
            st = !S.band_ovf && need_b >= 0 && need_b <= nb;
            if (st) {
#pragma unroll 1
              for (int i = tid; i < P; i += blockDim.x) S.pcount[i] = (int)htab[i].above;
              __syncthreads();
              if (attempt == 0) WK_MARK(19);
#pragma unroll 1
              for (int b = tid; b < nb; b += blockDim.x) {
                const unsigned long long kb = S.band_key[b];
                const uint32_t ib = S.band_idx[b];
                int beaten = 0;
#pragma unroll 1
                for (int o = 0; o < nb; ++o) {
                  const unsigned long long ko = S.band_key[o];
                  beaten += (ko > kb) || (ko == kb && S.band_idx[o] > ib);  // (score desc, index desc)
                }
                if (beaten < need_b) {
                  atomicAdd(&S.pcount[(int)((int64_t)ib / chunk)], 1);
                  if ((int64_t)ib >= j0 && (int64_t)ib < j0 + m)
                    atomicOr(&S.amask[((int64_t)ib - j0) >> 5], 1u << (((int64_t)ib - j0) & 31));
                }
              }
              if (attempt == 0) WK_MARK(20);
              // every partition's count: keys above its list + list keys above the band + band members
#pragma unroll 1
              for (int t = tid; t < Ltot; t += blockDim.x) {
                const uint32_t key = (uint32_t)(cand[t].kidx >> 32), ib = (uint32_t)cand[t].kidx;
                if (key <= ord_hi) continue;
                atomicAdd(&S.pcount[(int)(ib / (uint32_t)chunk)], 1);
                if ((int64_t)ib >= j0 && (int64_t)ib < j0 + m)  // this partition's list keys above the band
                  atomicOr(&S.amask[((int64_t)ib - j0) >> 5], 1u << (((int64_t)ib - j0) & 31));
              }
              if (tid == 0) {
                S.ord_def = ord_hi;
                S.e_lo = e_lo;
                S.e_hi = e_hi;
              }
              __syncthreads();
              if (attempt == 0) WK_MARK(21);
            }
          }
          dr = 0;
        }
        if (tid == 0) {
          S.status = st;
          S.dir = dr;
        }
        __syncthreads();
      }
      dir = S.dir;
      if (S.status) {
        done = true;
        path = attempt;
        ord_def = S.ord_def;
      }
      buf ^= 1;
      if (!done && dir == 0) break;  // overflow or an uncovered band: the radix path decides
      __syncthreads();
    }
    if (!done) {
      if (tid == 0) S.e_lo = S.e_hi = __longlong_as_double(0x7ff8000000000000ll);
      FbArgs fa;
      fa.kt = kt;
      fa.cap = s.capacity;
      fa.keys32 = keys32;
      fa.smem = smem;
      fa.htab = htab;
      fa.W = W;
      fa.j0 = j0;
      fa.chunk = chunk;
      fa.m = m;
      fa.P = P;
      fa.r = r;
      fa.k = k;
      fa.d_s = d_s;
      fa.buf = buf;
      fa.eps2 = eps2;
      ord_def = select_fallback(S, fa, path);
      __syncthreads();
#pragma unroll 1
      for (int w = warp; w < WK_MAXM / 32; w += WK_WARPS) {  // the fallback's selection as mask words
        const int e = w * 32 + lane;
        const bool sel = e < m && (keys32[e] > ord_def || ((S.bitmap[w] >> lane) & 1u));
        const unsigned b = __ballot_sync(0xffffffffu, sel);
        if (lane == 0) S.amask[w] = b;
      }
    }
  }
  if (!select_all && tid == 0) {  // this partition's hint for the next step (from whichever path decided)
    float2 *hint = s.part_hint ? reinterpret_cast<float2 *>(s.part_hint) + (size_t)u * TKV_MAX_PARTS + r : nullptr;
    const double T = 0.5 * (S.e_lo + S.e_hi);
    if (hint && S.sd > 0.0 && isfinite(T)) {
      const float2 hv = *hint;
      const double z = (T - S.mu) / S.sd;
      const float dz = isfinite(hv.x) ? (float)fabs(z - (double)hv.x) : __int_as_float(0x7fc00000);
      const float y = isfinite(hv.y) ? (isfinite(dz) ? 0.75f * hv.y + 0.25f * dz : hv.y) : dz;
      *hint = make_float2((float)z, y);
    }
  }
  WK_MARK(8);
  if (trace && tid == 0 && r == 0 && path >= 0) atomicAdd(&g_wk_path[path], 1u);
  // ---- 3. ascending output from the mask words: one word (32 keys) per thread ----
  if (select_all) {
#pragma unroll 1
    for (int w = tid; w < WK_MAXM / 32; w += blockDim.x) {
      const int e = w * 32;
      S.amask[w] = e >= m ? 0u : (m - e >= 32 ? 0xffffffffu : ((1u << (m - e)) - 1u));
    }
  }
  __syncthreads();
  const uint32_t myw = tid < WK_MAXM / 32 ? S.amask[tid] : 0u;
  int cta_total;
  const int wpos = block_excl_scan(__popc(myw), S.scan, &cta_total);
  if (tid == 0) {
    if (select_all) {
      S.offset = (int)j0;
      S.far_total = (int)ncand;
    } else {
      int off = 0, tot = 0;
#pragma unroll 1
      for (int i = 0; i < P; ++i) {
        if (i == r) off = tot;
        tot += S.pcount[i];
      }
      S.offset = off;
      S.far_total = tot;
    }
  }
  __syncthreads();
  const int offset = S.offset, far_total = S.far_total;
  int32_t *rows = reinterpret_cast<int32_t *>(keys32);  // rows still to gather (global token indices)
  int32_t *out_idx = a.sel_idx + (size_t)u * a.sel_stride;
  {
    uint32_t x = myw;
    int p = wpos;
#pragma unroll 1
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1u;
      const int32_t idx = (int32_t)(j0 + tid * 32 + b);
      out_idx[offset + p] = idx;
      rows[p++] = idx;
    }
  }
  const int nrest = cta_total + n_loc_mine;
#pragma unroll 1
  for (int i = tid; i < n_loc_mine; i += blockDim.x) rows[cta_total + i] = (int32_t)(ncand + r + (int64_t)P * i);
  if (r == P - 1) {
#pragma unroll 1
    for (int i = tid; i < n_loc; i += blockDim.x) out_idx[far_total + i] = (int32_t)(ncand + i);
    if (tid == 0) {
      a.sel_count[u] = far_total + n_loc;
      if (a.fetch_count) a.fetch_count[u] = far_total;
    }
  }
  __syncthreads();
  WK_MARK(9);
  // ---- 4. gather + attention over this partition's rows, in rounds of NR staged rows ----
  constexpr int CPL = WK_D / 32;  // channels per lane
  const int NW = use_cache ? WK_WARPS - 1 : WK_WARPS;  // warps computing logits (the last one issues PCIe copies)
  const int rs_bytes = ((nrest * 4 + 127) / 128) * 128;
  int32_t *rslot = reinterpret_cast<int32_t *>(smem + WK_RAW - rs_bytes);
  const int row_bytes = 2 * WK_D * 2 + GMAX * 4;  // staged (K|V) row + its logits
  const int NR = min(512, ((WK_RAW - rs_bytes) / row_bytes) & ~15);
  float *zs = reinterpret_cast<float *>(smem + (size_t)NR * 2 * WK_D * 2);
  lookup_rows(gc, rows, rslot, nrest, &S.hits, &S.misses);
  __syncthreads();
  WK_MARK(22);
  float mrun[GMAX], lrun[GMAX], acc[GMAX][CPL];
#pragma unroll
  for (int h = 0; h < GMAX; ++h) {
    mrun[h] = -INFINITY;
    lrun[h] = 0.0f;
#pragma unroll
    for (int e = 0; e < CPL; ++e) acc[h][e] = 0.0f;
  }
  uint32_t parity = 0;
#pragma unroll 1
  for (int base = 0; base < nrest; base += NR) {
    const int32_t *rr = rows + base;
    int32_t *cc = rslot + base;
    const int cnt = min(NR, nrest - base);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic SMEM accesses before the TMA writes
    __syncthreads();
    issue_hbm(gc, rr, cc, cnt, stage, &S.bar_hbm);
    if (base == 0) WK_MARK(23);
    // with the row cache the last warp issues the PCIe copies and then picks the misses' cache
    // slots (all rounds) while the others compute the logits
    if (!use_cache || warp == WK_WARPS - 1) issue_pcie(gc, rr, cc, cnt, stage, &S.bar_pcie, use_cache);
    if (use_cache && warp == WK_WARPS - 1 && base == 0) alloc_slots(gc, rslot, nrest, S.free_slots);
    // (c) logits of this warp's rows (row = warp mod NW); keys over PCIe wait for those rows first
    if (warp < NW) {
      mbar_wait(&S.bar_hbm, parity);
      if (!kfd) mbar_wait(&S.bar_pcie, parity);
      float4 qv[GMAX];
#pragma unroll
      for (int h = 0; h < GMAX; ++h)
        qv[h] = h < G ? *reinterpret_cast<const float4 *>(qs + h * WK_D + lane * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
      for (int i = warp; i < cnt; i += NW) {
        const uint2 kb = *reinterpret_cast<const uint2 *>(stage + (size_t)i * 2 * WK_D + lane * 4);
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
          float t4[4], t2[2];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            t4[q] = (b16 ? dd[q + 4] : dd[q]) + __shfl_xor_sync(0xffffffffu, b16 ? dd[q] : dd[q + 4], 16);
#pragma unroll
          for (int q = 0; q < 2; ++q)
            t2[q] = (b8 ? t4[q + 2] : t4[q]) + __shfl_xor_sync(0xffffffffu, b8 ? t4[q] : t4[q + 2], 8);
          c = (b4 ? t2[1] : t2[0]) + __shfl_xor_sync(0xffffffffu, b4 ? t2[0] : t2[1], 4);
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
      __syncwarp();
      if (base == 0) WK_MARK(24);
      // (d) value rows landed; warp-local online softmax over this warp's rows, then p.v
      if (kfd) mbar_wait(&S.bar_pcie, parity);
      const int nr = cnt > warp ? (cnt - warp + NW - 1) / NW : 0;
      const int hl = lane % GMAX;
      const int ne = nr * GMAX;
      float wm = -INFINITY;
#pragma unroll 1
      for (int e = lane; e < ne; e += 32)
        if (hl < G) wm = fmaxf(wm, zs[(size_t)(warp + NW * (e / GMAX)) * GMAX + hl]);
#pragma unroll
      for (int o = GMAX; o < 32; o <<= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
      float mh = -INFINITY;
#pragma unroll
      for (int h = 0; h < GMAX; ++h) {
        const float mr = fmaxf(mrun[h], __shfl_sync(0xffffffffu, wm, h));
        if (h < G && mr != -INFINITY) {
          const float sc = exp2f(mrun[h] - mr);
          lrun[h] *= sc;
#pragma unroll
          for (int e = 0; e < CPL; ++e) acc[h][e] *= sc;
          mrun[h] = mr;
        }
        if (h == hl) mh = mrun[h];
      }
      float ps = 0.0f;
#pragma unroll 1
      for (int e = lane; e < ne; e += 32) {
        if (hl >= G) continue;
        float *zp = &zs[(size_t)(warp + NW * (e / GMAX)) * GMAX + hl];
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
#pragma unroll 1
      for (int i = warp; i < cnt; i += NW) {
        const uint2 bv = *reinterpret_cast<const uint2 *>(stage + (size_t)i * 2 * WK_D + WK_D + lane * 4);
        const float vf[4] = {h2f((uint16_t)bv.x), h2f((uint16_t)(bv.x >> 16)), h2f((uint16_t)bv.y),
                             h2f((uint16_t)(bv.y >> 16))};
        const float *pz = zs + (size_t)i * GMAX;
#pragma unroll
        for (int h = 0; h < GMAX; ++h) {
          const float pp = h < G ? pz[h] : 0.0f;
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[h][e] = fmaf(pp, vf[e], acc[h][e]);
        }
      }
    }
    if (base == 0) WK_MARK(25);
    __syncthreads();  // the PCIe warp's slot codes before the inserts
    // (e) rows fetched over PCIe enter the HBM row cache in their assigned slots
    if (use_cache) {
#pragma unroll 1
      for (int i = tid; i < cnt; i += blockDim.x) {
        const int code = cc[i];
        if (code > -3) continue;
        const int dst = -3 - code;
        const int32_t idx = rr[i];
        gc.stok[dst] = idx;
        gc.sstamp[dst] = (int)n;
        gc.tslot[idx] = dst;
        bulk_s2g(gc.sv + (size_t)dst * 2 * WK_D, stage + (size_t)i * 2 * WK_D, WK_D * 4);
      }
      bulk_commit_wait_read();
    }
    if (base == 0) WK_MARK(26);
    parity ^= 1u;
    __syncthreads();
  }
  WK_MARK(10);
  // ---- 5. this partition's partial: warps merged in SMEM, then published ----
  float *pm = reinterpret_cast<float *>(smem), *pl = pm + WK_WARPS * GMAX, *pa = pl + WK_WARPS * GMAX;
#pragma unroll
  for (int h = 0; h < GMAX; ++h) {
    if (lane == 0) {
      pm[warp * GMAX + h] = mrun[h];
      pl[warp * GMAX + h] = lrun[h];
    }
    *reinterpret_cast<float4 *>(pa + ((size_t)warp * GMAX + h) * WK_D + lane * CPL) =
        make_float4(acc[h][0], acc[h][1], acc[h][2], acc[h][3]);
  }
  __syncthreads();
  const int PF = part_floats(GMAX);
  float *mypart = W.part + (size_t)r * PF;
#pragma unroll 1
  for (int i = tid; i < G * WK_D; i += blockDim.x) {
    const int h = i / WK_D, c = i % WK_D;
    float M = -INFINITY;
#pragma unroll 1
    for (int w = 0; w < WK_WARPS; ++w) M = fmaxf(M, pm[w * GMAX + h]);
    float L = 0.0f, Ac = 0.0f;
    if (M != -INFINITY) {
#pragma unroll 1
      for (int w = 0; w < WK_WARPS; ++w) {
        const float mw = pm[w * GMAX + h];
        if (mw == -INFINITY) continue;
        const float sc = exp2f(mw - M);
        L = fmaf(sc, pl[w * GMAX + h], L);
        Ac = fmaf(sc, pa[((size_t)w * GMAX + h) * WK_D + c], Ac);
      }
    }
    mypart[h * WK_D + c] = Ac;
    if (c == 0) {
      mypart[GMAX * WK_D + h] = M;
      mypart[GMAX * WK_D + GMAX + h] = L;
    }
  }
  WK_MARK(27);
  if (use_cache && tid == 0 && (S.hits | S.misses)) {
    atomicAdd(&s.cache_stats[0], (unsigned long long)S.hits);
    atomicAdd(&s.cache_stats[1], (unsigned long long)S.misses);
  }
  // ---- merge: last arriver of each group of GS partitions, then the last group ----
  const int GSZ = P > 32 ? WK_GS : P;
  const int NG = (P + GSZ - 1) / GSZ;
  const int g = r / GSZ, gcount = min(GSZ, P - g * GSZ);
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned old = atomicAdd(&W.ctl[C_GROUP + g], 1u);
    S.last = old == (unsigned)gcount - 1;
    if (S.last) {
      atomicExch(&W.ctl[C_GROUP + g], 0u);
      __threadfence();
    }
  }
  __syncthreads();
  WK_MARK(11);
  if (trace && tid == 0) atomicMax(&g_wk_lastexit, gtime());
  if (!S.last) return;
  float *mls = reinterpret_cast<float *>(smem + 96 * 1024);  // [<= 32][2 GMAX]
  float *gpart = W.part + (size_t)P * PF;
  float *uout = a.out + (size_t)u * G * WK_D;
  if (NG == 1) {
    merge_partials_w(W.part, P, PF, GMAX, G, mls, nullptr, uout);
  } else {
    merge_partials_w(W.part + (size_t)g * GSZ * PF, gcount, PF, GMAX, G, mls, gpart + (size_t)g * PF, nullptr);
    if (tid == 0) {
      __threadfence();
      const unsigned old = atomicAdd(&W.ctl[C_FINAL], 1u);
      S.last = old == (unsigned)NG - 1;
      if (S.last) {
        atomicExch(&W.ctl[C_FINAL], 0u);
        __threadfence();
      }
    }
    __syncthreads();
    if (!S.last) return;
    merge_partials_w(gpart, NG, PF, GMAX, G, mls, nullptr, uout);
  }
  WK_MARK(12);
  if (trace && tid == 0) {
    const unsigned long long t_ = gtime();
    if (u == 0) g_wk_launch[(__ldcg(&g_wk_nlaunch) - 1u) & 127u][2] = t_;
    if (u < 64) g_wk_uend[u] = t_;
  }
  // ---- the final merger: the step's append (HostPool.append + mirror append, memsim.py:106-111,
  // pipeline.py:405-413), after every partition of the unit finished reading this step's state ----
  if (a.new_keys) {
#pragma unroll 1
    for (int c = tid; c < WK_D; c += blockDim.x) {
      const uint16_t kx = a.new_keys[(size_t)u * WK_D + c], vx = a.new_values[(size_t)u * WK_D + c];
      s.kt[((size_t)u * WK_D + c) * s.capacity + n] = kx;  // (the host store row went out at kernel start)
      float *cm = &s.chmax[(size_t)u * WK_D + c];
      *cm = fmaxf(*cm, fabsf(h2f(kx)));
      const int64_t lr = n - s.local_offset;
      s.loc_k[((size_t)u * s.local_capacity + lr) * WK_D + c] = kx;
      s.loc_v[((size_t)u * s.local_capacity + lr) * WK_D + c] = vx;
      if (s.kdev) s.kdev[((size_t)u * s.capacity + n) * WK_D + c] = kx;
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
  // histograms used by a fallback return to zero (every CTA of the unit is past them)
  if (__ldcg(&W.ctl[C_FALLBACK])) {
    uint4 *h4 = reinterpret_cast<uint4 *>(W.hist);
#pragma unroll 1
    for (int i = tid; i < WK_NHIST * WK_HB / 4; i += blockDim.x) h4[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    if (tid == 0) atomicExch(&W.ctl[C_FALLBACK], 0u);
  }
  WK_MARK(13);
  if (trace && tid == 0) atomicMax(&g_wk_lastexit, gtime());
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  return sms;
}

// partitions per unit: one CTA per SM over the whole GPU
int parts_for(int units) {
  int P = sm_count() / std::max(1, units);
  if (const char *e = getenv("TKV_WIDE_PARTS")) P = std::min(P, std::max(1, atoi(e)));
  return std::max(1, std::min(P, TKV_MAX_PARTS));
}

static int mode() {  // TKV_WIDE: 0 never, 1 whenever the shape allows, unset = auto
  static const int m = getenv("TKV_WIDE") ? atoi(getenv("TKV_WIDE")) : -1;
  return m;
}
static int g_force = -1;  // tkv_debug_sparse_wide: runtime override of TKV_WIDE

bool reserve(int units, int d) { return d == WK_D && sm_count() / std::max(1, units) >= 4; }

// Auto (mode -1) prefers the cluster kernel: measured equal at 8 units per GPU and faster at 1-4 units
// (both are bound by the serial latency of their phases, and the wide decode's unit
// barrier, list exchange and two-level merge grow with its partitions); the wide decode runs when
// forced, or when the cluster kernel cannot take the shape.
bool supported(const SL &s, int G, int n_local, int d_s, int keys_from_device, bool cluster_ok) {
  const int md = g_force >= 0 ? g_force : mode();
  if (md == 0 || (md < 0 && cluster_ok)) return false;
  if (!(s.d == WK_D && G >= 1 && G <= 8 && d_s >= 1 && d_s <= WK_MAXDS && s.capacity % 8 == 0)) return false;
  if (keys_from_device && s.kdev == nullptr) return false;  // key rows from the scorer copy: cluster kernel
  if (!reserve(s.units, s.d)) return false;
  const int P = parts_for(s.units);
  if (P < 2) return false;
  const int64_t ncand = s.capacity > n_local ? s.capacity - n_local : 0;
  const int64_t chunk = ((ncand + P - 1) / P + 15) & ~int64_t(15);
  if (chunk > WK_MAXM) return false;
  if ((n_local + P - 1) / P > WK_MAXLOC) return false;
  return true;
}

int64_t ctl_bytes(int units, int d) { return reserve(units, d) ? (int64_t)units * ctl_unit_bytes() : 0; }
int64_t scratch_bytes(int units, int d) {
  return reserve(units, d) ? (int64_t)units * scratch_unit_bytes(parts_for(units)) : 0;
}

template <int GMAX>
static cudaError_t launch(const SL &s, const WArgs &a, int P, cudaStream_t st) {
  auto kern = sparse_wide_kernel<GMAX>;
  const size_t sm = WK_RAW + WK_KEYS + (size_t)GMAX * WK_D * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P, s.units);
  cfg.blockDim = dim3(WK_THREADS);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributePriority;
  at[0].val.priority = launch_priority(true);
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  static const bool no_pdl = getenv("TKV_NO_PDL") != nullptr;
  at[1].val.programmaticStreamSerializationAllowed = (pdl_note(st, s.len) && !no_pdl) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, s, a);
}

int decode(const SL &s, const uint16_t *queries, int G, const int32_t *channels, int d_s, int n_local, int n_topk,
           int32_t *sel_idx, int32_t *sel_count, int32_t *fetch_count, int keys_from_device, float *out,
           const uint16_t *new_keys, const uint16_t *new_values, void *ctl, void *scratch, cudaStream_t st) {
  const int P = parts_for(s.units);
  WArgs a;
  a.queries = queries;
  a.channels = channels;
  a.G = G;
  a.d_s = d_s;
  a.n_local = n_local;
  a.n_topk = n_topk;
  a.sel_idx = sel_idx;
  a.sel_stride = n_local + n_topk + s.n_sink;
  a.sel_count = sel_count;
  a.fetch_count = fetch_count;
  a.keys_from_device = keys_from_device;
  a.out = out;
  a.new_keys = new_keys;
  a.new_values = new_values;
  a.ctl = static_cast<unsigned char *>(ctl);
  a.scratch = static_cast<unsigned char *>(scratch);
  a.scratch_unit = scratch_unit_bytes(P);
  const cudaError_t e = G <= 4 ? launch<4>(s, a, P, st) : launch<8>(s, a, P, st);
  if (e != cudaSuccess) return fail(TKV_ERR_CUDA, std::string("tkv_sparse_decode(wide): ") + cudaGetErrorString(e));
  return check_launch("tkv_sparse_decode(wide)");
}

}  // namespace wide
}  // namespace tkv

// debug / experiments: 0 cluster kernel always, 1 wide whenever the shape allows, -1 auto
extern "C" int tkv_debug_sparse_wide(int mode) {
  tkv::wide::g_force = mode;
  return 0;
}
extern "C" int tkv_debug_wide_trace(int on) {
  if (on) {
    static const unsigned z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(tkv::wide::g_wk_path, z, sizeof(z));
  }
  return cudaMemcpyToSymbol(tkv::wide::g_wk_trace, &on, sizeof(int)) == cudaSuccess ? 0 : 7;
}
extern "C" int tkv_debug_wide_marks(unsigned long long *out) {  // [32][24]
  return cudaMemcpyFromSymbol(out, tkv::wide::g_wk_mark, sizeof(tkv::wide::g_wk_mark)) == cudaSuccess ? 0 : 7;
}
extern "C" int tkv_debug_wide_paths(unsigned *out) {  // [4]
  return cudaMemcpyFromSymbol(out, tkv::wide::g_wk_path, sizeof(tkv::wide::g_wk_path)) == cudaSuccess ? 0 : 7;
}
// launch timeline of unit 0 (start, after the PDL wait, end of the final merge), last <= 128 launches
extern "C" int tkv_debug_wide_launches(unsigned long long *out, int reset) {
  if (reset) {
    const unsigned z = 0;
    return cudaMemcpyToSymbol(tkv::wide::g_wk_nlaunch, &z, sizeof(z)) == cudaSuccess ? 0 : -1;
  }
  unsigned cnt = 0;
  if (cudaMemcpyFromSymbol(&cnt, tkv::wide::g_wk_nlaunch, sizeof(cnt)) != cudaSuccess) return -1;
  if (cudaMemcpyFromSymbol(out, tkv::wide::g_wk_launch, sizeof(tkv::wide::g_wk_launch)) != cudaSuccess) return -1;
  return (int)cnt;
}
extern "C" int tkv_debug_wide_dbg(int *out) {  // [8]
  return cudaMemcpyFromSymbol(out, tkv::wide::g_wk_dbg, sizeof(tkv::wide::g_wk_dbg)) == cudaSuccess ? 0 : 7;
}
extern "C" int tkv_debug_wide_unit_ends(unsigned long long *out) {  // [64] + latest CTA exit
  cudaMemcpyFromSymbol(out + 64, tkv::wide::g_wk_lastexit, sizeof(unsigned long long));
  return cudaMemcpyFromSymbol(out, tkv::wide::g_wk_uend, sizeof(tkv::wide::g_wk_uend)) == cudaSuccess ? 0 : 7;
}
extern "C" int tkv_wide_parts(int32_t units) { return tkv::wide::parts_for(units); }
// bounded-wait timeouts of the wide decode since the last reset (0 = none; 1 unit barrier, 2 mbarrier)
extern "C" int tkv_debug_wide_error(int reset) {
  unsigned v = 0;
  cudaMemcpyFromSymbol(&v, tkv::wide::g_wk_err, sizeof(v));
  if (reset) {
    const unsigned z = 0;
    cudaMemcpyToSymbol(tkv::wide::g_wk_err, &z, sizeof(z));
  }
  return (int)v;
}
