// Microbenchmark: per-iteration cost of a CTA-barrier loop (256 threads, 1 CTA/SM) that
// prefetches data D iterations ahead with (0) plain LDG into registers, (1) __ldg, (2)
// cp.async into shared memory, (3) a TMA bulk copy + mbarrier (one thread issues).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int D>
__global__ void k(const double *__restrict__ g, const int *__restrict__ rowstart, int iters, int mode,
                  long long *out, double *sink) {
  __shared__ __align__(128) double ring[D][256];
  __shared__ __align__(8) uint64_t bar[D];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int d = 0; d < D; d++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[d])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  double reg[D];
  double acc = 0.0;
  unsigned phase = 0;
  auto issue = [&](int it, int d) {
    const double *src = g + rowstart[(it + blockIdx.x * 977) & 65535];
    if (mode == 0) reg[d] = src[tid];
    else if (mode == 1) reg[d] = __ldg(src + tid);
    else if (mode == 2) {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(su(&ring[d][tid])), "l"(src + tid));
      asm volatile("cp.async.commit_group;");
    } else if (mode == 3 && tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[d])), "r"(2048));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 2048, [%2];" ::"r"(
                       su(&ring[d][0])), "l"(src), "r"(su(&bar[d])) : "memory");
    }
  };
#pragma unroll
  for (int d = 0; d < D; d++) issue(d, d);
  long long t0 = clock64();
  for (int it = 0; it < iters; it += D) {
#pragma unroll
    for (int d = 0; d < D; d++) {
      double v;
      if (mode <= 1) v = reg[d];
      else if (mode == 2) {
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1));
        v = ring[d][tid];
      } else {
        asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(
                         su(&bar[d])), "r"((phase >> d) & 1u) : "memory");
        phase ^= 1u << d;
        v = ring[d][tid];
      }
      acc += v;
      __syncthreads();
      issue(it + d + D, d);
    }
  }
  long long t1 = clock64();
  if (mode == 2) asm volatile("cp.async.wait_group 0;");
  if (mode == 3) {
    for (int d = 0; d < D; d++)
      asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }" ::"r"(
                       su(&bar[d])), "r"((phase >> d) & 1u) : "memory");
  }
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 1.2345) sink[0] = acc;
}
int main() {
  const size_t N = (size_t)1 << 27;  // 1 GiB of doubles: beyond L2
  double *g, *sink;
  int *rs, h_rs[65536];
  long long *d_out, h_out[148];
  cudaMalloc(&g, N * sizeof(double));
  cudaMemset(g, 0, N * sizeof(double));
  cudaMalloc(&rs, sizeof(h_rs));
  cudaMalloc(&sink, 8);
  cudaMalloc(&d_out, sizeof(h_out));
  for (int l2 = 0; l2 < 2; l2++) for (int Dv : {2, 4, 8, 16}) {
    const size_t span = l2 ? ((size_t)1 << 20) : N - 1024;  // 8 MB (L2-resident) or 1 GiB
    unsigned x = 12345;
    for (int i = 0; i < 65536; i++) {
      x = x * 1664525u + 1013904223u;
      h_rs[i] = (int)((x % (span / 512)) * 512);
    }
    cudaMemcpy(rs, h_rs, sizeof(h_rs), cudaMemcpyHostToDevice);
    for (int mode = 0; mode < 4; mode++) {
      auto kf = Dv == 2 ? k<2> : Dv == 4 ? k<4> : Dv == 8 ? k<8> : k<16>;
      kf<<<148, 256>>>(g, rs, 4096, mode, d_out, sink);
      kf<<<148, 256>>>(g, rs, 4096, mode, d_out, sink);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h_out, d_out, sizeof(h_out), cudaMemcpyDeviceToHost);
      printf("%s D=%2d mode %d (%s): %.1f cycles/iter %s\n", l2 ? "L2-resident" : "HBM", Dv, mode,
             mode == 0 ? "LDG regs" : mode == 1 ? "__ldg regs" : mode == 2 ? "cp.async" : "TMA bulk+mbar",
             h_out[0] / 4096.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
