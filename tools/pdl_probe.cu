// PDL chain probe: how long after the primary grid's last CTA exits does the
// dependent grid's griddepcontrol.wait return?  Primary: 144 CTAs x 512
// threads that spin ~20 us, optionally ending with a host (PCIe) store or a
// TMA shared->global bulk store; dependent: same shape, PDL attribute.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_probe tools/pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ unsigned long long g_exit, g_wait;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(512) primary(int mode, unsigned *host, float *gbuf) {
  extern __shared__ float sm[];
  asm volatile("griddepcontrol.launch_dependents;");
  const unsigned long long t0 = gt();
  while (gt() - t0 < 20000) {
  }
  if (threadIdx.x == 0) {
    if (mode == 1) host[blockIdx.x] = 1u;  // a posted PCIe write
    if (mode == 2) {
      sm[0] = 1.0f;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16;" ::"l"(gbuf + 4 * blockIdx.x),
                   "r"((unsigned)__cvta_generic_to_shared(sm))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    atomicMax(&g_exit, gt());
  }
}

__global__ void __launch_bounds__(512) dependent() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicMax(&g_wait, gt());
}

int main() {
  unsigned *host;
  cudaHostAlloc(&host, 4096, cudaHostAllocMapped);
  float *gbuf;
  cudaMalloc(&gbuf, 1 << 20);
  cudaFuncSetAttribute(primary, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
  cudaFuncSetAttribute(dependent, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
  cudaStream_t st;
  cudaStreamCreate(&st);
  for (int mode = 0; mode < 3; ++mode) {
    double tot = 0;
    const int R = 20;
    for (int rep = 0; rep < R; ++rep) {
      unsigned long long z = 0;
      cudaMemcpyToSymbol(g_exit, &z, 8);
      cudaMemcpyToSymbol(g_wait, &z, 8);
      primary<<<144, 512, 180 * 1024, st>>>(mode, host, gbuf);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(144);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = 180 * 1024;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, dependent);
      cudaStreamSynchronize(st);
      unsigned long long e = 0, w = 0;
      cudaMemcpyFromSymbol(&e, g_exit, 8);
      cudaMemcpyFromSymbol(&w, g_wait, 8);
      if (rep >= 2) tot += (double)(w - e) / 1e3;
    }
    printf("mode %d (%s): last primary exit -> last dependent wait-done %.2f us\n", mode,
           mode == 0 ? "plain" : mode == 1 ? "host store" : "bulk s2g", tot / (R - 2));
  }
  return 0;
}
