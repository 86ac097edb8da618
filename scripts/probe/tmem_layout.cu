// Probe: the register layout of tcgen05.ld.16x256b (vs the known 32x32b).
// Writes value lane*1000+col into TMEM with 32x32b stores, reads back with
// 16x256b.x1 at lane bases 0 and 16 of warp 0's quadrant, prints the map.
#include <cstdio>
#include <cstdint>
__global__ void probe(int* out) {
  __shared__ uint32_t slot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot;
  if (warp == 0) {
    uint32_t v[8];
    for (int c = 0; c < 8; ++c) v[c] = lane * 1000 + c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(base),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    for (int half = 0; half < 2; ++half) {
      uint32_t r0, r1, r2, r3;
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                   : "r"(base + ((uint32_t)(half * 16) << 16)));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      int* o = out + (half * 32 + lane) * 4;
      o[0] = r0; o[1] = r1; o[2] = r2; o[3] = r3;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(base));
}
int main() {
  int* d; cudaMalloc(&d, 64 * 4 * 4);
  probe<<<1, 128>>>(d);
  int h[256]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  for (int half = 0; half < 2; ++half)
    for (int t = 0; t < 32; ++t) {
      int* o = h + (half * 32 + t) * 4;
      printf("base%2d t%2d:", half * 16, t);
      for (int k = 0; k < 4; ++k) printf(" (r%d c%d)", o[k] / 1000, o[k] % 1000);
      printf("\n");
    }
}
