// Same-address ticket atomics: 296 CTAs x 8 warps, every warp claims tickets from ONE global
// counter (two outstanding, as the transport kernel does) until `cnt` are taken -- time per
// "sweep" of cnt tickets, against S counters 128 B apart (warps spread over them).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) k(int* ctr, int cnt, int S, int sweeps, int* sink) {
  const int lane = threadIdx.x & 31, w = blockIdx.x * 8 + (threadIdx.x >> 5);
  int acc = 0;
  for (int sw = 0; sw < sweeps; ++sw) {
    int* c = ctr + (size_t)sw * S * 32;
    const int seg = (cnt + S - 1) / S;
    int s = w % S, tried = 0;
    int t1 = 0, t2 = 0;
    if (lane == 0) { t1 = atomicAdd(c + s * 32, 1); t2 = atomicAdd(c + s * 32, 1); }
    for (;;) {
      int t = __shfl_sync(0xffffffffu, t1, 0);
      if (t < seg && s * seg + t < cnt) {
        acc += t;
        if (lane == 0) { t1 = t2; t2 = atomicAdd(c + s * 32, 1); }
      } else {
        if (++tried == S) break;
        s = (s + 1) % S;
        if (lane == 0) { t1 = atomicAdd(c + s * 32, 1); t2 = atomicAdd(c + s * 32, 1); }
      }
    }
    // a grid barrier would sit here; the probe only measures the claims
  }
  if (acc == 123456789) *sink = acc;
}
int main() {
  int *ctr, *sink;
  const int sweeps = 200, cnt = 54000;
  cudaMalloc(&ctr, (size_t)sweeps * 64 * 32 * 4);
  cudaMalloc(&sink, 4);
  for (int S : {1, 2, 4, 8, 16, 32}) {
    cudaMemset(ctr, 0, (size_t)sweeps * 64 * 32 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<296, 256>>>(ctr, cnt, S, sweeps, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("{\"counters\": %d, \"tickets_per_sweep\": %d, \"us_per_sweep\": %.2f}\n", S, cnt, 1000.0f * ms / sweeps);
  }
  return 0;
}
