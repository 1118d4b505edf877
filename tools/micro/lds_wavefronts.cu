// Shared-memory wavefronts per warp load for the K3b operand patterns (run under ncu:
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum per kernel; also timed alone).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
template <int MODE>
__global__ void k(double *out) {
  __shared__ __align__(16) double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = i * 0.5;
  __syncthreads();
  const int lane = threadIdx.x & 31, li = lane >> 3, lj = lane & 7;
  double acc = 0.0;
  int off = 0;
  for (int it = 0; it < ITERS; it++) {
    if (MODE == 0) {  // LDS.64, 8 distinct contiguous (b[k][lj]), broadcast over li
      acc += s[off + lj];
    } else if (MODE == 1) {  // LDS.64, 4 distinct, 64 B apart (a[li][k])
      acc += s[off + li * 8];
    } else if (MODE == 2) {  // LDS.128, 8 distinct contiguous 128 B (pair layout b)
      const double2 v = reinterpret_cast<const double2 *>(s + off)[lj];
      acc += v.x + v.y;
    } else if (MODE == 3) {  // LDS.128, 4 distinct 64 B apart (a[li][k..k+1])
      const double2 v = reinterpret_cast<const double2 *>(s + off + li * 8)[0];
      acc += v.x + v.y;
    } else if (MODE == 4) {  // LDS.64 all lanes distinct contiguous (256 B)
      acc += s[off + lane];
    } else if (MODE == 5) {  // LDS.128 all distinct (512 B)
      const double2 v = reinterpret_cast<const double2 *>(s + off)[lane];
      acc += v.x + v.y;
    } else if (MODE == 6) {  // LDS.64 broadcast (1 address)
      acc += s[off];
    } else if (MODE == 7) {  // LDS.128, 8 distinct, 2 per quarter-warp (column = lane >> 2)
      const double2 v = reinterpret_cast<const double2 *>(s + off)[lane >> 2];
      acc += v.x + v.y;
    } else if (MODE == 8) {  // LDS.128, 4 distinct 64 B apart, all 4 in every quarter (row = lane & 3)
      const double2 v = reinterpret_cast<const double2 *>(s + off + (lane & 3) * 8)[0];
      acc += v.x + v.y;
    } else if (MODE == 9) {  // LDS.64, 4 distinct 64 B apart, all 4 in every quarter
      acc += s[off + (lane & 3) * 8];
    } else if (MODE == 10) {  // LDS.64, 8 distinct contiguous, same 8 in each quarter (lane & 7)
      acc += s[off + (lane & 7)];
    } else if (MODE == 12) {  // LDS.128 A rows 0..3 (lane & 3), pairs of rows 2, 3 swapped by 4 columns
      const int r = lane & 3, kk = (it & 3) ^ (((r >> 1) & 1) << 1);
      const double2 v = reinterpret_cast<const double2 *>(s + off + r * 8)[kk];
      acc += v.x + v.y;
    } else if (MODE == 11) {  // LDS.128, 2 distinct adjacent (32 B), row = lane >> 4
      const double2 v = reinterpret_cast<const double2 *>(s + off)[lane >> 4];
      acc += v.x + v.y;
    }
    off = (off + 64) & 1023;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
template <int MODE>
void run(double *d) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<MODE><<<148 * 8, 256>>>(d);
  cudaEventRecord(a);
  k<MODE><<<148 * 8, 256>>>(d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double warp_loads = 148.0 * 8 * 8 * ITERS;
  printf("mode %d: %.3f ms, %.2f SM-cycles per warp load (1.965 GHz)\n", MODE, ms,
         ms * 1e-3 * 1.965e9 * 148 / warp_loads);
}
int main() {
  double *d;
  cudaMalloc(&d, 148 * 8 * 256 * 8);
  run<0>(d); run<1>(d); run<2>(d); run<3>(d); run<4>(d); run<5>(d); run<6>(d); run<7>(d); run<8>(d); run<9>(d); run<10>(d); run<11>(d); run<12>(d);
  return 0;
}
