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
                            float* out, float* side = nullptr, int side_floats = 0) {
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
    // optional side stream: side_floats floats written per chunk (the GEMV's
    // per-tile partials), spread over the consumer warps
    for (int f = warp * 32 + lane; f < side_floats; f += nw * 32) side[c * side_floats + f] = acc;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == STAGES) { s = 0; ph ^= 1; }
  }
  if (acc == 12345.f) *out = acc;
}

__global__ void stg_kernel(float4* __restrict__ a, size_t n4) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const float4 z = make_float4(1.f, 2.f, 3.f, (float)threadIdx.x);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) __stcs(a + i, z);
}

// smem -> global bulk stores (cp.async.bulk.global.shared::cta), chunk bytes
// per store, `depth` stores in flight per CTA
__global__ void bulk_store_kernel(char* __restrict__ a, size_t bytes, uint32_t chunk, int depth) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* st = smem_align<128>(smem_raw);
  for (int i = threadIdx.x; i < (int)chunk; i += blockDim.x) st[i] = (uint8_t)i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = bytes / chunk;
  const size_t c0 = nchunks * blockIdx.x / gridDim.x, c1 = nchunks * (blockIdx.x + 1) / gridDim.x;
  int inflight = 0;
  for (size_t c = c0; c < c1; ++c) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(a + c * chunk),
                 "r"(su32(st)), "r"(chunk)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++inflight >= depth) {
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
      inflight = 8;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// 4 KB "boxes" written as 32 rows x 128 B with a 512 B row pitch (the packed
// tile's 32 x 32 fp32 box layout), 16 boxes per 64 KB tile, by 128 threads
// with 8-byte stores; or contiguous 4 KB per box (box-major layout)
__global__ void box_store_kernel(float* __restrict__ a, size_t tiles, int strided) {
  const int t = threadIdx.x;
  const float val = (float)t;
  for (size_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    float* base = a + tile * 16384;
    for (int box = 0; box < 16; ++box) {
      const int q = box >> 2, ch = box & 3;
      // 1024 floats per box, 8 per thread (two float4)
      for (int k = 0; k < 2; ++k) {
        const int e = (k * 128 + t) * 4;  // element within the box
        const int r = e >> 5, c = e & 31;
        float* dst = strided ? base + (q * 32 + r) * 128 + ch * 32 + c : base + box * 1024 + e;
        __stcs(reinterpret_cast<float4*>(dst), make_float4(val, val, val, val));
      }
    }
  }
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
    timeit(nm, [&] { kern<<<sms, (warps + 1) * 32, smem>>>(a, bytes, chunk, split, out, nullptr, 0); });
  };
  for (int split : {1, 4, 16}) bulk(bulk_kernel<3>, 3, 65536, split, 8);
  bulk(bulk_kernel<6>, 6, 32768, 1, 8);
  bulk(bulk_kernel<12>, 12, 16384, 1, 8);
  bulk(bulk_kernel<4>, 4, 49152, 1, 8);
  bulk(bulk_kernel<2>, 2, 65536, 1, 8);
  {
    float* side;
    cudaMalloc(&side, (bytes / 65536) * 256 * 4 + 4096);
    for (int sf : {128, 256}) {
      cudaFuncSetAttribute(bulk_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536 + 256);
      char nm[64];
      snprintf(nm, sizeof nm, "bulk 3x64KB + %d B written per tile", sf * 4);
      timeit(nm, [&] { bulk_kernel<3><<<sms, 9 * 32, 3 * 65536 + 256>>>(a, bytes, 65536, 1, out, side, sf); });
    }
    cudaFree(side);
  }
  for (int th : {256, 1024})
    for (int bpsm : {1, 4}) {
      char nm[64];
      snprintf(nm, sizeof nm, "stg grid=%dx%d th=%d (write)", bpsm, sms, th);
      timeit(nm, [&] { stg_kernel<<<bpsm * sms, th>>>((float4*)a, bytes / 16); });
    }
  for (uint32_t chunk : {4096u, 16384u, 65536u}) {
    cudaFuncSetAttribute(bulk_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk + 256);
    char nm[64];
    snprintf(nm, sizeof nm, "bulk store %uKB depth 16 (write)", chunk >> 10);
    timeit(nm, [&] { bulk_store_kernel<<<sms, 128, chunk + 256>>>(a, bytes, chunk, 16); });
  }
  timeit("cudaMemsetAsync (write)", [&] { cudaMemsetAsync(a, 1, bytes); });
  for (int strided : {1, 0}) {
    char nm[64];
    snprintf(nm, sizeof nm, "box stores %s (write)", strided ? "32x128B pitch 512B" : "contiguous 4KB");
    timeit(nm, [&] { box_store_kernel<<<sms * 8, 128>>>((float*)a, bytes / 65536, strided); });
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
