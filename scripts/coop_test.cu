// bring-up probe: does cooperative grid.sync work with this toolchain/driver?
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int* ctr, int iters) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) atomicAdd(&ctr[i], 1);
    g.sync();
  }
}
int main() {
  int* d; cudaMalloc(&d, 1000 * 4); cudaMemset(d, 0, 4000);
  int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * occ; if (blocks > 296) blocks = 296;
  int iters = 10; void* args[] = {&d, &iters};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)k, blocks, 256, args, 0, 0);
  printf("launch %s occ=%d blocks=%d\n", cudaGetErrorString(e), occ, blocks); fflush(stdout);
  e = cudaDeviceSynchronize();
  int h[10]; cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("sync %s ctr0=%d ctr9=%d\n", cudaGetErrorString(e), h[0], h[9]);
  return 0;
}
