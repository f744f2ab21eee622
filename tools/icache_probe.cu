// Instruction-fetch probe: how long does one warp per SM take to run N
// straight-line, independent FFMAs (16 B of SASS each) when the code is cold
// vs. warm?  Each launch runs the code `reps` times in a loop: rep 0 pays the
// fetch, later reps run from the instruction cache.  Prints us per launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/icache_probe tools/icache_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int N>
__global__ void probe(float *out, int reps, float a) {
  if (threadIdx.x >= 32) return;
  float x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < N / 8; ++i) {
      const float c = 1.0f + 1e-7f * (float)i;  // distinct immediates: no folding
      x0 = fmaf(x0, c, 0.5f); x1 = fmaf(x1, c, 0.25f); x2 = fmaf(x2, c, 0.125f); x3 = fmaf(x3, c, 1.5f);
      x4 = fmaf(x4, c, 2.5f); x5 = fmaf(x5, c, 3.5f); x6 = fmaf(x6, c, 4.5f); x7 = fmaf(x7, c, 5.5f);
    }
  }
  out[blockIdx.x * 32 + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <int N>
static void run(float *out) {
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  for (int reps : {1, 2, 4}) {
    probe<N><<<148, 512>>>(out, reps, 1.0f);
    cudaDeviceSynchronize();
    cudaEventRecord(s);
    for (int i = 0; i < 20; ++i) probe<N><<<148, 512>>>(out, reps, 1.0f);
    cudaEventRecord(e);
    cudaEventSynchronize(e);
    float ms = 0;
    cudaEventElapsedTime(&ms, s, e);
    printf("N=%6d (%6.1f KB of FFMA)  reps=%d: %8.2f us per launch\n", N, N * 16 / 1024.0, reps, ms * 1e3 / 20);
  }
}

int main() {
  float *out;
  cudaMalloc(&out, 148 * 32 * 4);
  run<512>(out);
  run<2048>(out);
  run<4096>(out);
  run<8192>(out);
  run<16384>(out);
  return 0;
}
