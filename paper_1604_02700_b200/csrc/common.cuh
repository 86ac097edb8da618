// Shared device helpers for libgpic (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gpic.h"

namespace gpic {

constexpr int kWarp = 32;

// Count of kernels this library launched (bench gpu_launches claim).
extern unsigned long long g_launches;
inline void count_launch(unsigned long long k = 1) { g_launches += k; }

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Record the first error of a kind. `order` picks the smallest offending
// index (atomicMin) so the reported index is deterministic.
__device__ __forceinline__ void raise_status(gpic_ctl* ctl, int code, long long idx, long long idx2,
                                             double value) {
  // status: first writer wins per code class; index: min over writers.
  atomicCAS(&ctl->status, GPIC_OK, code);
  if (ctl->status == code) {
    atomicMin(reinterpret_cast<unsigned long long*>(&ctl->err_index),
              static_cast<unsigned long long>(idx));
    if (idx2 >= 0) ctl->err_index2 = idx2;
    ctl->err_value = value;
  }
  ctl->stop = 1;
}

// Streaming 128-bit load that bypasses L1 allocation (A is read once per
// iteration; keep L1 for v).
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream_f4(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// Streaming 8-byte store (a quad of lanes fills one 32-byte sector).
__device__ __forceinline__ void st_stream_f2(float* p, float a, float b) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

// Round fp32 to TF32 (10 explicit mantissa bits), round-to-nearest-away.
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Last-CTA-done election: returns true in exactly one CTA (all threads),
// after every CTA called it once. `counter` must start at 0; it is reset
// by the winner.
__device__ __forceinline__ bool last_block_done(unsigned int* counter) {
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    s_last = (prev == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

}  // namespace gpic

#define GPIC_CUDA_TRY(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return gpic::fail_cuda(_e, #expr); \
  } while (0)

namespace gpic {
int fail_cuda(cudaError_t e, const char* what);
int fail(int code, const char* msg);
}  // namespace gpic
