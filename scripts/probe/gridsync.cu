// Probe: cooperative-groups grid.sync() across one 1024-thread CTA per SM,
// compiled like libgpic (no -rdc). Each round every CTA publishes a value,
// syncs, and checks every other CTA's value (L2 loads).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void __launch_bounds__(1024, 1) k(long long* slots, int* errors, int rounds) {
  cg::grid_group grid = cg::this_grid();
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) slots[(r & 1) * 1024 + blockIdx.x] = (long long)r * 100000 + blockIdx.x;
    grid.sync();
    if (threadIdx.x == 0)
      for (int q = 0; q < (int)gridDim.x; ++q)
        if (__ldcg(slots + (r & 1) * 1024 + q) != (long long)r * 100000 + q) atomicAdd(errors, 1);
  }
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* slots;
  int* err;
  cudaMalloc(&slots, 2048 * 8);
  cudaMalloc(&err, 4);
  cudaMemset(err, 0, 4);
  int rounds = 200;
  void* args[] = {&slots, &err, &rounds};
  cudaError_t e = cudaLaunchCooperativeKernel((const void*)k, sms, 1024, args, 0, 0);
  cudaError_t e2 = cudaDeviceSynchronize();
  int h;
  cudaMemcpy(&h, err, 4, cudaMemcpyDeviceToHost);
  printf("launch %s sync %s errors %d (grid %d)\n", cudaGetErrorString(e), cudaGetErrorString(e2), h, sms);
  return 0;
}
