// Microbenchmark: DFMA latency / throughput per SMSP vs warps and independent chains; SHFL latency.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k_dfma(double* out, int iters, double w) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < CH; ++c) a[c] = fma(a[c], w, 1.0);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0);
}
__global__ void k_shfl(double* out, int iters) {
  double a = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) a = __shfl_down_sync(0xffffffffu, a, 1) + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x + 1] = a;
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0);
}
template <int CH>
void run(int warps_per_sm, double* d) {
  int iters = 2000;
  k_dfma<CH><<<148, warps_per_sm * 32>>>(d, iters, 0.999);
  cudaDeviceSynchronize();
  double cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  double per_round = cyc / (iters * 8.0);          // cycles per round of CH dfma per warp
  double wps = warps_per_sm / 4.0;                 // warps per SMSP
  printf("chains %2d warps/SM %2d: %.2f cycles per round; per-SMSP DFMA issue interval %.2f cycles\n", CH, warps_per_sm,
         per_round, per_round / (CH * wps));
}
int main() {
  double* d;
  cudaMalloc(&d, 148 * 1024 * 8);
  for (int w : {4, 8, 16, 32}) { run<1>(w, d); run<2>(w, d); run<4>(w, d); run<8>(w, d); run<12>(w, d); }
  k_shfl<<<1, 32>>>(d, 2000);
  cudaDeviceSynchronize();
  double cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  printf("shfl64 + dadd dependent: %.2f cycles\n", cyc / 16000.0);
  return 0;
}
