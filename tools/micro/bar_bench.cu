// Microbenchmark: cycles per iteration of a CTA-barrier loop (256 threads, 1 CTA/SM),
// with 0..3 dependent shared-memory loads per iteration.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int iters, int mode, long long *out, int *sink) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7) & 1023;
  __syncthreads();
  int x = threadIdx.x & 1023, acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    if (mode >= 1) x = s[x];
    if (mode >= 2) x = s[(x + 1) & 1023];
    if (mode >= 3) x = s[(x + 3) & 1023];
    acc += x;
    if (mode != 4) __syncthreads();
    else __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345) sink[0] = acc;
}
int main() {
  long long *d, h[148];
  int *sink;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaMalloc(&sink, 4);
  for (int threads : {256, 512}) {
    for (int mode = 0; mode <= 4; mode++) {
      k<<<148, threads>>>(10000, mode, d, sink);
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("threads %d mode %d: %.1f cycles/iter\n", threads, mode, h[0] / 10000.0);
    }
  }
  return 0;
}
