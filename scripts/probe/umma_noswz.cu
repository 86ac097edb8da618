// Probe: tcgen05.mma kind::f16 with SWIZZLE_NONE K-major operands (K = 16),
// the layout of the affinity engine's 16-wide norm block. Core matrices are
// 8 rows x 16 B; the tile is [8-row group g][k group c][row r][8 fp16] and the
// probe tries both readings of (LBO, SBO) against a host product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1604_02700_b200/csrc \
//        scripts/probe/umma_noswz.cu -o scripts/probe/umma_noswz -lcuda
#include <cuda_fp16.h>

#include <cstdio>

#include "sm100.cuh"

using namespace gpic;

__global__ void probe(const __half* a, const __half* b, float* d, uint32_t lbo, uint32_t sbo,
                      uint32_t kgrp_stride, uint32_t grp_stride, int sw32) {
  __shared__ __align__(1024) uint8_t sA[128 * 32];
  __shared__ __align__(1024) uint8_t sB[128 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  // element (i, k) -> byte offset g*grp_stride + c*kgrp_stride + r*16 + e*2
  for (int idx = t; idx < 128 * 16; idx += blockDim.x) {
    const int i = idx / 16, k = idx % 16;
    // sw32: rows of 32 B, 16-byte chunk index XOR address bit 7 ((row >> 2) & 1)
    const uint32_t off = sw32 ? i * 32 + (((k / 8) ^ ((i >> 2) & 1)) * 16) + (k % 8) * 2
                              : (i / 8) * grp_stride + (k / 8) * kgrp_stride + (i % 8) * 16 + (k % 8) * 2;
    *reinterpret_cast<__half*>(sA + off) = a[i * 16 + k];
    *reinterpret_cast<__half*>(sB + off) = b[i * 16 + k];
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  auto desc = [&](const void* p) {
    uint64_t x = (uint64_t)((su32(p) >> 4) & 0x3FFFu);
    x |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    x |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    x |= (uint64_t)1u << 46;
    if (sw32) x |= (uint64_t)6u << 61;  // SWIZZLE_32B
    return x;  // else swizzle bits 61-63 = 0: SWIZZLE_NONE
  };
  if (t == 0) {
    mma_f16(tm, desc(sA), desc(sB), idesc_f16(128, 128), 0u);
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int cb = 0; cb < 4; ++cb) {
    uint32_t r[32];
    tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + cb * 32, r);
    for (int c = 0; c < 32; ++c) d[(warp * 32 + lane) * 128 + cb * 32 + c] = __uint_as_float(r[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

int main() {
  __half ha[128 * 16], hb[128 * 16];
  float fa[128 * 16], fb[128 * 16];
  for (int i = 0; i < 128; ++i)
    for (int k = 0; k < 16; ++k) {
      fa[i * 16 + k] = (float)((i * 3 + k * 7) % 13 - 6);
      fb[i * 16 + k] = (float)((i * 5 + k * 11) % 9 - 4);
      ha[i * 16 + k] = __float2half(fa[i * 16 + k]);
      hb[i * 16 + k] = __float2half(fb[i * 16 + k]);
    }
  __half *da, *db;
  float* dd;
  cudaMalloc(&da, sizeof ha);
  cudaMalloc(&db, sizeof hb);
  cudaMalloc(&dd, 128 * 128 * 4);
  cudaMemcpy(da, ha, sizeof ha, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, sizeof hb, cudaMemcpyHostToDevice);
  static float out[128 * 128];
  // layout [g][c][r][8]: k-group stride 128 B, 8-row-group stride 256 B
  const uint32_t variants[4][3] = {{128, 256, 0}, {256, 128, 0}, {16, 256, 1}, {256, 256, 1}};
  for (auto& v : variants) {
    cudaMemset(dd, 0, 128 * 128 * 4);
    probe<<<1, 128>>>(da, db, dd, v[0], v[1], 128, 256, (int)v[2]);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(out, dd, sizeof out, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < 128; ++j) {
        float s = 0.f;
        for (int k = 0; k < 16; ++k) s += fa[i * 16 + k] * fb[j * 16 + k];
        if (out[i * 128 + j] != s) ++bad;
      }
    printf("%s LBO=%u SBO=%u: %s, %d of 16384 wrong\n", v[2] ? "SW32" : "NONE", v[0], v[1],
           cudaGetErrorString(e), bad);
  }
  return 0;
}
