// grid.sync cost probe: N grid barriers with various CTA counts / block sizes
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, int* ctr) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(ctr, 1);
    g.sync();
  }
}
__global__ void k2(int iters, int* ctr, int* take) {
  // barrier + one global atomic per warp (work fetch) per iteration
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) {
    if ((threadIdx.x & 31) == 0) atomicAdd(&take[i & 1023], 1);
    __syncthreads();
    g.sync();
  }
}
int main() {
  int* d; cudaMalloc(&d, 4096 * 4); cudaMemset(d, 0, 4096 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 2000;
  for (int threads : {256, 512}) for (int per : {1, 2}) {
    for (int variant = 0; variant < 2; ++variant) {
      int blocks = sms * per;
      void* args1[] = {&iters, &d};
      int* t = d + 1024;
      void* args2[] = {&iters, &d, &t};
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e = variant == 0 ? cudaLaunchCooperativeKernel((void*)k, blocks, threads, args1, 0, 0)
                                   : cudaLaunchCooperativeKernel((void*)k2, blocks, threads, args2, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("variant %d threads %d blocks %d: %s  %.2f us per barrier\n", variant, threads, blocks,
             cudaGetErrorString(e), 1000.0 * ms / iters);
    }
  }
  return 0;
}
