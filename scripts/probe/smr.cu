// Probe: setmaxnreg with 5 warpgroups (warpgroup 0 dec, 1-4 inc), 1 CTA/SM.
//   usage: smr DEC INC   (exit 0 = completed)
#include <cstdio>
#include <cstdlib>
template <int D, int I>
__global__ void __launch_bounds__(640, 1) k(float* out) {
  const int warp = threadIdx.x >> 5;
  float acc = threadIdx.x;
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(D));
    acc += 1.f;
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(I));
    for (int i = 0; i < 100; ++i) acc = acc * 1.0001f + 0.5f;
  }
  asm volatile("bar.sync 15, 640;" ::: "memory");
  out[blockIdx.x * 640 + threadIdx.x] = acc;
}
int main(int argc, char** argv) {
  float* o;
  cudaMalloc(&o, 148 * 640 * 4);
  const int d = atoi(argv[1]), i = atoi(argv[2]);
  if (d == 88 && i == 104) k<88, 104><<<148, 640>>>(o);
  else if (d == 40 && i == 112) k<40, 112><<<148, 640>>>(o);
  else if (d == 24 && i == 120) k<24, 120><<<148, 640>>>(o);
  else if (d == 56 && i == 104) k<56, 104><<<148, 640>>>(o);
  else if (d == 96 && i == 96) k<96, 96><<<148, 640>>>(o);
  printf("dec %d inc %d: %s\n", d, i, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
