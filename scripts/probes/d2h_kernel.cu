// D2H of a 1 MiB frame: copy engine (cudaMemcpyAsync) vs SM stores into
// mapped page-locked memory (16 B per thread, G blocks).  Event-timed.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void st_copy(const uint4* __restrict__ s, uint4* d, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}
int main() {
  const size_t n = 1 << 20;
  uint8_t *src, *host;
  cudaMalloc(&src, n);
  cudaMemset(src, 7, n);
  cudaHostAlloc(&host, n, cudaHostAllocMapped);
  uint8_t* hd;
  cudaHostGetDevicePointer((void**)&hd, host, 0);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    float best = 1e9, sum = 0;
    for (int i = 0; i < 50; ++i) {
      cudaEventRecord(a, st);
      cudaMemcpyAsync(host, src, n, cudaMemcpyDeviceToHost, st);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
      sum += ms;
    }
    printf("copy engine: best %.1f us mean %.1f us\n", best * 1e3, sum / 50 * 1e3);
    for (int g : {8, 32, 148, 296, 592}) {
      best = 1e9; sum = 0;
      for (int i = 0; i < 50; ++i) {
        cudaEventRecord(a, st);
        st_copy<<<g, 256, 0, st>>>((const uint4*)src, (uint4*)hd, n / 16);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
        sum += ms;
      }
      printf("SM stores, %d blocks: best %.1f us mean %.1f us (ok=%d)\n", g, best * 1e3, sum / 50 * 1e3, host[n - 1] == 7);
    }
  }
  return 0;
}
