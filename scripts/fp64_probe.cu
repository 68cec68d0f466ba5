// FP64 pipe probe: dependent-chain latency and throughput vs (warps/SM, chains/warp).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chains(int iters, double* out, double m, double c) {
  double a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int i = 0; i < CH; ++i) a[i] = fma(a[i], m, c);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += a[i];
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (double)(t1 - t0) / (iters * 8.0);
  if (s == 1.2345) out[0] = s;
}
template <int CH>
void run(int warps_per_sm) {
  double* d; cudaMalloc(&d, 16);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int threads = 32 * warps_per_sm; int iters = 4000;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  chains<CH><<<sms, threads>>>(100, d, 0.999999, 1e-7);
  cudaEventRecord(a);
  chains<CH><<<sms, threads>>>(iters, d, 0.999999, 1e-7);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  double flops = 2.0 * sms * threads * iters * 8.0 * CH;
  printf("warps/SM %2d chains %d: %.2f TFLOP/s, cycles per chain-step %.1f\n", warps_per_sm, CH,
         flops / ms / 1e9, h[1]);
  cudaFree(d);
}
int main() {
  for (int w : {1, 4, 8, 16, 32}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
  return 0;
}
