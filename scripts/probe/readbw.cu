// Read-only streaming bandwidth probe (what a GEMV over 20 GB can reach).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1604_02700_b200/csrc \
//        scripts/probe/readbw.cu -o scripts/probe/readbw && scripts/probe/readbw [GB]
// kernels: ldg   float4 grid-stride loads, 8 in flight per thread
//          bulk  one CTA per SM, cp.async.bulk ring (stages x bytes), no compute
#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace gpic;

__global__ void ldg_kernel(const float4* __restrict__ a, size_t n4, float* out) {
  float s = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldcs(a + i + k * stride);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  for (; i < n4; i += stride) { float4 v = a[i]; s += v.x + v.y + v.z + v.w; }
  if (s == 12345.f) *out = s;
}

template <int STAGES>
__global__ void bulk_kernel(const char* __restrict__ a, size_t bytes, uint32_t chunk, int split,
                            float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* st = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(st + STAGES * chunk);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nw); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t nchunks = bytes / chunk;
  const size_t c0 = nchunks * blockIdx.x / gridDim.x, c1 = nchunks * (blockIdx.x + 1) / gridDim.x;
  if (warp == nw) {
    if (lane) return;
    int s = 0; uint32_t ph = 0;
    const uint64_t once = policy_evict_first();
    const uint32_t piece = chunk / split;
    for (size_t c = c0; c < c1; ++c) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], chunk);
      for (int p = 0; p < split; ++p)
        bulk_load(st + s * chunk + p * piece, a + c * chunk + p * piece, piece, &full[s], once);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    return;
  }
  int s = 0; uint32_t ph = 0;
  float acc = 0.f;
  for (size_t c = c0; c < c1; ++c) {
    mbar_wait(&full[s], ph);
    acc += reinterpret_cast<const float*>(st + s * chunk)[warp * 32 + lane];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == STAGES) { s = 0; ph ^= 1; }
  }
  if (acc == 12345.f) *out = acc;
}

int main(int argc, char** argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 20.0;
  const size_t bytes = (size_t)(gb * 1e9) / (1 << 16) * (1 << 16);
  char* a;
  float* out;
  cudaMalloc(&a, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(a, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-40s %8.3f ms  %7.1f GB/s\n", name, best, bytes / (best * 1e-3) / 1e9);
  };
  for (int bpsm : {1, 2, 4, 8})
    for (int th : {256, 512, 1024}) {
      char nm[64];
      snprintf(nm, sizeof nm, "ldg grid=%dx%d th=%d", bpsm, sms, th);
      timeit(nm, [&] { ldg_kernel<<<bpsm * sms, th>>>((const float4*)a, bytes / 16, out); });
    }
  auto bulk = [&](auto kern, int stages, uint32_t chunk, int split, int warps) {
    const int smem = stages * chunk + 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    char nm[64];
    snprintf(nm, sizeof nm, "bulk %dx%uKB split=%d warps=%d", stages, chunk >> 10, split, warps);
    timeit(nm, [&] { kern<<<sms, (warps + 1) * 32, smem>>>(a, bytes, chunk, split, out); });
  };
  for (int split : {1, 4, 16}) bulk(bulk_kernel<3>, 3, 65536, split, 8);
  bulk(bulk_kernel<6>, 6, 32768, 1, 8);
  bulk(bulk_kernel<12>, 12, 16384, 1, 8);
  bulk(bulk_kernel<4>, 4, 49152, 1, 8);
  bulk(bulk_kernel<2>, 2, 65536, 1, 8);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
