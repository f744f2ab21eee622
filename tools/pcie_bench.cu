// PCIe H2D gather microbenchmark (B200): random fixed-size rows read from a
// pinned host arena by GPU kernels, in several issue styles and host
// allocation modes.  Used to pick the design of the Top-K value-row gather
// (DESIGN.md 4.4).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/pcie_bench.cu -lcuda -o tools/pcie_bench
// Run:  tools/pcie_bench [arena_GiB=8]
#include <cuda.h>
#include <cuda_runtime.h>

#include <sys/mman.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <random>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));   \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

// ---- style A: each warp owns RPW rows, all loads issued before use ----
template <int VEC, int RPW, int LD>
__global__ void k_warp_rows(const char *__restrict__ base, int row_bytes, const int *__restrict__ rows, int nrows,
                            unsigned *sink) {
  if (row_bytes / VEC > 32) return;
  const int lanes_per_row = row_bytes / VEC;
  const int rows_per_inst = 32 / lanes_per_row;
  const int lane = threadIdx.x & 31;
  const int sub = lane / lanes_per_row, l = lane % lanes_per_row;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  unsigned x = 0;
  for (int r0 = gw * RPW * rows_per_inst; r0 < nrows; r0 += nw * RPW * rows_per_inst) {
    uint4 v[RPW];
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int r = r0 + j * rows_per_inst + sub;
      v[j] = make_uint4(0, 0, 0, 0);
      if (r < nrows) {
        const char *p = base + (size_t)rows[r] * row_bytes + (size_t)l * VEC;
        if (VEC == 16) {
          if (LD == 0) v[j] = *reinterpret_cast<const uint4 *>(p);
          else if (LD == 1) v[j] = __ldcv(reinterpret_cast<const uint4 *>(p));
          else v[j] = __ldg(reinterpret_cast<const uint4 *>(p));
        } else {
          uint2 a;
          if (LD == 0) a = *reinterpret_cast<const uint2 *>(p);
          else if (LD == 1) a = __ldcv(reinterpret_cast<const uint2 *>(p));
          else a = __ldg(reinterpret_cast<const uint2 *>(p));
          v[j].x = a.x;
          v[j].y = a.y;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < RPW; ++j) x ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
  }
  if (x == 0x9e3779b9u) sink[0] = x;
}

// ---- style B: TMA bulk copies (cp.async.bulk global->shared, mbarrier) ----
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes));
}
__device__ unsigned g_timeout;
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  // bounded wait: gives up after ~50 ms and flags g_timeout (no GPU hang if
  // the bulk engine cannot complete a copy)
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    unsigned ok;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(a), "r"(phase) : "memory");
    if (ok) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 50000000ull) { g_timeout = 1; return; }
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

// each CTA loops over batches of `batch` rows; rows of a batch are issued by
// `batch` threads (one bulk copy each) into a double-buffered smem ring
__global__ void k_bulk(const char *__restrict__ base, int row_bytes, const int *__restrict__ rows, int nrows,
                       int batch, unsigned *sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  unsigned x = 0;
  const int stride = gridDim.x * batch;
  int it = 0;
  // prologue: issue batch 0
  auto issue = [&](int r0, int slot) {
    const int cnt = min(batch, nrows - r0);
    if (cnt <= 0) return;
    if (tid == 0) mbar_expect_tx(&bar[slot], (unsigned)(cnt * row_bytes));
    __syncthreads();
    if (tid < cnt)
      bulk_g2s(sm + ((size_t)slot * batch + tid) * row_bytes, base + (size_t)rows[r0 + tid] * row_bytes,
               (unsigned)row_bytes, &bar[slot]);
  };
  int r0 = blockIdx.x * batch;
  issue(r0, 0);
  unsigned ph[2] = {0, 0};
  for (; r0 < nrows; r0 += stride, ++it) {
    const int slot = it & 1;
    issue(r0 + stride, slot ^ 1);
    mbar_wait(&bar[slot], ph[slot]);
    ph[slot] ^= 1;
    const int cnt = min(batch, nrows - r0);
    const uint4 *s4 = reinterpret_cast<const uint4 *>(sm + (size_t)slot * batch * row_bytes);
    for (int i = tid; i < cnt * row_bytes / 16; i += blockDim.x) {
      const uint4 v = s4[i];
      x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncthreads();
  }
  if (x == 0x9e3779b9u) sink[0] = x;
}

// ---- style C: cp.async (LDGSTS) 16 B per lane into smem ----
__global__ void k_ldgsts(const char *__restrict__ base, int row_bytes, const int *__restrict__ rows, int nrows,
                         int batch, unsigned *sink) {
  extern __shared__ __align__(128) char sm[];
  const int tid = threadIdx.x;
  const int vec_per_row = row_bytes / 16;
  unsigned x = 0;
  for (int r0 = blockIdx.x * batch; r0 < nrows; r0 += gridDim.x * batch) {
    const int cnt = min(batch, nrows - r0);
    for (int i = tid; i < cnt * vec_per_row; i += blockDim.x) {
      const int r = i / vec_per_row, v = i % vec_per_row;
      const char *src = base + (size_t)rows[r0 + r] * row_bytes + v * 16;
      const unsigned dst = (unsigned)__cvta_generic_to_shared(sm + (size_t)i * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const uint4 *s4 = reinterpret_cast<const uint4 *>(sm);
    for (int i = tid; i < cnt * vec_per_row; i += blockDim.x) {
      const uint4 v = s4[i];
      x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncthreads();
  }
  if (x == 0x9e3779b9u) sink[0] = x;
}

// touches one 16-byte vector every `step` bytes of [base, base+len)
__global__ void k_touch(const char *__restrict__ base, size_t len, size_t step, unsigned *sink) {
  unsigned x = 0;
  for (size_t o = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * step; o < len;
       o += (size_t)gridDim.x * blockDim.x * step) {
    const uint4 v = __ldcv(reinterpret_cast<const uint4 *>(base + o));
    x ^= v.x;
  }
  if (x == 0x9e3779b9u) sink[0] = x;
}

static void *alloc_host(int mode, size_t bytes, int dev, int numa) {
  if (mode == 0) {  // mmap + THP + mbind + cudaHostRegister (the library's current store)
    void *p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(p, bytes, MADV_HUGEPAGE);
    memset(p, 1, bytes);
    CK(cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    return p;
  }
  if (mode == 1) {  // driver-allocated pinned memory
    void *p;
    CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(p, 1, bytes);
    return p;
  }
  if (mode == 3) {  // mmap without THP (4 KB pages) + register
    void *p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(p, bytes, MADV_NOHUGEPAGE);
    memset(p, 1, bytes);
    CK(cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    return p;
  }
  // mode 2: VMM host-NUMA allocation mapped into the GPU's VA
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  prop.location.id = numa < 0 ? 0 : numa;
  size_t gran = 0;
  if (cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) return nullptr;
  const size_t len = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  if (cuMemCreate(&h, len, &prop, 0) != CUDA_SUCCESS) return nullptr;
  CUdeviceptr va;
  if (cuMemAddressReserve(&va, len, gran, 0, 0) != CUDA_SUCCESS) return nullptr;
  if (cuMemMap(va, len, 0, h, 0) != CUDA_SUCCESS) return nullptr;
  CUmemAccessDesc acc[2] = {};
  acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc[0].location.id = dev;
  acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  acc[1].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  acc[1].location.id = prop.location.id;
  acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (cuMemSetAccess(va, len, acc, 2) != CUDA_SUCCESS) {
    if (cuMemSetAccess(va, len, acc, 1) != CUDA_SUCCESS) return nullptr;
    CK(cudaMemset((void *)va, 1, len));
  } else {
    memset((void *)va, 1, len);
  }
  printf("  [vmm host-numa granularity %zu]\n", gran);
  return (void *)va;
}

int main(int argc, char **argv) {
  setvbuf(stdout, nullptr, _IOLBF, 0);
  const double arena_gib = argc > 1 ? atof(argv[1]) : 8.0;
  const int only_mode = argc > 2 ? atoi(argv[2]) : -1;
  CK(cudaSetDevice(0));
  cuInit(0);
  int numa = -1;
  cudaDeviceGetAttribute(&numa, cudaDevAttrHostNumaId, 0);
  printf("host numa of gpu0: %d, numa_available=%d\n", numa, 0);
  const size_t bytes = (size_t)(arena_gib * (1ull << 30));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  unsigned *sink;
  CK(cudaMalloc(&sink, 4));
  // memcpy peak
  {
    const size_t nb = 256u << 20;
    void *h, *d;
    CK(cudaHostAlloc(&h, nb, 0));
    CK(cudaMalloc(&d, nb));
    for (int i = 0; i < 2; ++i) CK(cudaMemcpyAsync(d, h, nb, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(a, st));
    for (int i = 0; i < 5; ++i) CK(cudaMemcpyAsync(d, h, nb, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("memcpy H2D 256MiB pinned: %.1f GB/s\n", 5.0 * nb / (ms * 1e-3) / 1e9);
    CK(cudaFreeHost(h));
    CK(cudaFree(d));
  }
  const int big = 262144, small = 11000;
  if (only_mode == 9 || only_mode == 10) {
    // per-layer windows: 30 windows of `win` bytes, 11000 random rows of 256 B
    // in each (row pitch 256 or 512), windows visited in turn (cold translations);
    // mode 9: mmap+THP+cudaHostRegister, mode 10: cuMemCreate HOST_NUMA (2 MiB granularity)
    void *host = alloc_host(only_mode == 9 ? 0 : 2, bytes, 0, numa);
    const int W = 30;
    int *d_rows;
    CK(cudaMalloc(&d_rows, sizeof(int) * small * W));
    for (int nsmall : {11000, 1500}) for (int pitch : {512, 256}) {
      const int small = nsmall;
      const size_t win = (size_t)8 * 131072 * pitch;  // 8 units x 131072 tokens
      if (win * W > bytes) { printf("arena too small\n"); return 1; }
      std::mt19937_64 g(7);
      std::vector<int> hr((size_t)small * W);
      for (int w = 0; w < W; ++w)
        for (int i = 0; i < small; ++i) hr[(size_t)w * small + i] = (int)((win * w + (g() % (win / pitch)) * pitch) / 256);
      CK(cudaMemcpy(d_rows, hr.data(), sizeof(int) * hr.size(), cudaMemcpyHostToDevice));
      for (size_t touch : {(size_t)0, (size_t)65536}) {
        for (int rep = 0; rep < 2; ++rep) {
          double tg = 0, tt = 0;
          for (int w = 0; w < W; ++w) {
            float ms;
            if (touch) {
              CK(cudaEventRecord(a, st));
              k_touch<<<592, 256, 0, st>>>((const char *)host + win * w, win, touch, sink);
              CK(cudaEventRecord(b, st));
              CK(cudaEventSynchronize(b));
              CK(cudaEventElapsedTime(&ms, a, b));
              tt += ms;
            }
            CK(cudaEventRecord(a, st));
            k_warp_rows<16, 4, 1><<<1184, 256, 0, st>>>((const char *)host, 256,
                                                       d_rows + (size_t)w * small, small, sink);
            CK(cudaEventRecord(b, st));
            CK(cudaEventSynchronize(b));
            CK(cudaEventElapsedTime(&ms, a, b));
            tg += ms;
          }
          printf("rows %5d pitch %d touch-step %8zu rep %d: gather %.1f us/window (%.1f GB/s), touch %.1f us/window\n",
                 small, pitch, touch, rep, tg * 1e3 / W, (double)small * 256 / (tg * 1e-3 / W) / 1e9, tt * 1e3 / W);
        }
      }
    }
    return 0;
  }
  int *d_rows;
  CK(cudaMalloc(&d_rows, sizeof(int) * big));
  for (int mode = 0; mode < 4; ++mode) {
    if (only_mode >= 0 && mode != only_mode) continue;
    printf("== host alloc mode %d (%s), arena %.1f GiB\n", mode,
           mode == 0 ? "mmap+THP+register" : mode == 1 ? "cudaHostAlloc" : mode == 2 ? "cuMemCreate HOST_NUMA" : "mmap 4K+register",
           arena_gib);
    auto t0 = std::chrono::steady_clock::now();
    void *host = alloc_host(mode, bytes, 0, numa);
    printf("  alloc+touch+register %.1f s\n", std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    if (!host) {
      printf("  alloc failed\n");
      continue;
    }
    const char *base = (const char *)host;
    for (int row_bytes : {256, 512}) {
      std::mt19937_64 g(1);
      std::vector<int> hr(big);
      const size_t nrow_total = bytes / row_bytes;
      for (auto &x : hr) x = (int)(g() % nrow_total);
      CK(cudaMemcpy(d_rows, hr.data(), sizeof(int) * big, cudaMemcpyHostToDevice));
      auto timeit = [&](const char *name, int nrows, auto launch) {
        for (int i = 0; i < 2; ++i) launch(nrows);
        CK(cudaStreamSynchronize(st));
        const int reps = nrows == big ? 5 : 30;
        CK(cudaEventRecord(a, st));
        for (int i = 0; i < reps; ++i) launch(nrows);
        CK(cudaEventRecord(b, st));
        CK(cudaEventSynchronize(b));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double us = ms * 1e3 / reps;
        printf("  row %4d B %-34s rows %6d: %7.1f us  %6.1f GB/s\n", row_bytes, name, nrows, us,
               (double)nrows * row_bytes / (us * 1e-6) / 1e9);
      };
      char name[128];
#define WARPV(VEC, RPW, LD, BLOCKS, THREADS)                                                                  \
  do {                                                                                                         \
    snprintf(name, sizeof name, "warp v%d rpw%d ld%d %dx%d", VEC, RPW, LD, BLOCKS, THREADS);                   \
    for (int nr : {big, small})                                                                                \
      timeit(name, nr, [&](int n) {                                                                            \
        k_warp_rows<VEC, RPW, LD><<<BLOCKS, THREADS, 0, st>>>(base, row_bytes, d_rows, n, sink);               \
      });                                                                                                      \
  } while (0)
      WARPV(8, 8, 0, 672, 128);
      WARPV(8, 8, 1, 672, 128);
      WARPV(16, 8, 0, 672, 128);
      WARPV(16, 8, 1, 672, 128);
      WARPV(16, 8, 2, 672, 128);
      WARPV(16, 4, 1, 1184, 256);
      WARPV(16, 16, 1, 296, 256);
      WARPV(16, 8, 1, 148 * 4, 512);
      WARPV(8, 16, 1, 148 * 2, 512);
      for (int batch : {32, 64, 128}) {
        for (int ctas : {148, 296, 592}) {
          const size_t smem = 2ull * batch * row_bytes;
          if (smem > 200 * 1024) continue;
          CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          snprintf(name, sizeof name, "bulk batch%d %dx128", batch, ctas);
          for (int nr : {big, small})
            timeit(name, nr, [&](int n) { k_bulk<<<ctas, 128, smem, st>>>(base, row_bytes, d_rows, n, batch, sink); });
          unsigned to = 0;
          CK(cudaMemcpyFromSymbol(&to, g_timeout, 4));
          if (to) { printf("  bulk copy from host memory TIMED OUT (not supported?)\n"); goto after_bulk; }
        }
      }
    after_bulk:
      for (int batch : {32, 64}) {
        const size_t smem = (size_t)batch * row_bytes;
        CK(cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        snprintf(name, sizeof name, "ldgsts batch%d 592x256", batch);
        for (int nr : {big, small})
          timeit(name, nr, [&](int n) { k_ldgsts<<<592, 256, smem, st>>>(base, row_bytes, d_rows, n, batch, sink); });
      }
    }
    if (mode == 0 || mode == 3) {
      cudaHostUnregister(host);
      munmap(host, bytes);
    } else if (mode == 1) {
      cudaFreeHost(host);
    }
  }
  return 0;
}
