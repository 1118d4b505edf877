// fp64 throughput on the box (roofline denominators for the squaring kernels, VERDICT r1
// item 4): DFMA, DMUL+DADD pairs, the fp64 tensor instruction mma.sync.m8n8k4.f64 (DMMA),
// and the L2 -> SM gather rate of 512-byte blocks (the B-block stream of the block
// kernels).  Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/micro/fp64_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 8192;
constexpr int CH = 8;  // independent chains per thread

__global__ void k_dfma(double *out, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmuladd(double *out, double a, double b) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = __dadd_rn(__dmul_rn(x[c], a), b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void k_dmma(double *out, double a, double b) {
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; c++) d[c][0] = d[c][1] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int c = 0; c < CH; c++) dmma(d[c][0], d[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += d[c][0] + d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// warp-per-block gathers of 512-byte blocks at pseudo-random block indices within a
// working set of nblk blocks (each lane loads 16 bytes)
__global__ void k_gather(const double2 *blocks, int64_t nblk, int rounds, double *out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint64_t h = 0x9E3779B97F4A7C15ull * (w + 1);
  double s = 0.0;
  for (int r = 0; r < rounds; r++) {
    double2 v[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      h ^= h >> 33;
      h *= 0xff51afd7ed558ccdull;
      h ^= h >> 29;
      v[q] = blocks[(int64_t)(h % (uint64_t)nblk) * 32 + lane];
    }
#pragma unroll
    for (int q = 0; q < 4; q++) s += v[q].x + v[q].y;
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  const int grid = sms * 8, thr = 256;
  double *out;
  cudaMalloc(&out, (size_t)grid * thr * 8 * 4);
  const double fl_thread = 2.0 * ITERS * CH;  // flops per thread per kernel (FMA = 2)
  const double nthr = (double)grid * thr;
  float t_fma = time_ms([&] { k_dfma<<<grid, thr>>>(out, 0.999, 1e-3); });
  float t_ma = time_ms([&] { k_dmuladd<<<grid, thr>>>(out, 0.999, 1e-3); });
  float t_mma = time_ms([&] { k_dmma<<<grid, thr>>>(out, 0.999, 1e-3); });
  const double tf_fma = fl_thread * nthr / (t_fma * 1e-3) / 1e12;
  const double tf_ma = fl_thread * nthr / (t_ma * 1e-3) / 1e12;  // 1 mul + 1 add = 2 flops
  // DMMA: per warp per instruction 8x8x4 = 256 FMAs = 512 flops
  const double tf_mma = 512.0 * ITERS * CH * (nthr / 32) / (t_mma * 1e-3) / 1e12;
  // L2 gathers: working sets of 32 MB (L2 resident) and 2 GB (HBM)
  double gb[2];
  const int64_t sets[2] = {(32ll << 20) / 512, (2048ll << 20) / 512};
  double2 *blk;
  cudaMalloc(&blk, (size_t)sets[1] * 512);
  cudaMemset(blk, 0, (size_t)sets[1] * 512);
  const int rounds = 64;
  for (int s = 0; s < 2; s++) {
    float t = time_ms([&] { k_gather<<<sms * 16, 256>>>(blk, sets[s], rounds, out); });
    const double bytes = (double)sms * 16 * 8 * rounds * 4 * 512;
    gb[s] = bytes / (t * 1e-3) / 1e9;
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f, \"dfma_tflops\": %.2f, "
         "\"dmul_dadd_tflops\": %.2f, \"dmma_m8n8k4_tflops\": %.2f, \"gather512_l2_gbs\": %.0f, "
         "\"gather512_hbm_gbs\": %.0f, \"ms\": [%.3f, %.3f, %.3f]}\n",
         p.name, sms, clk / 1e3, tf_fma, tf_ma, tf_mma, gb[0], gb[1], t_fma, t_ma, t_mma);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
