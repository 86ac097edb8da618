// Fixed-shape reductions of the iteration tail (power.cu) and the tail
// itself as device functions, shared with the fused iteration kernel
// (sym.cu): tau = the fixed-shape sum of y, v' = y / tau, delta =
// max|v' - v|, history and stop rule — bitwise the same in both.
#pragma once

#include "common.cuh"
#include "ops.h"

namespace gpic {
namespace tail {

constexpr int kRedThreads = 256;
constexpr int kRedPer = kRedBlock / kRedThreads;  // 8 elements per thread

// ------------------------------------------------- fixed-shape reductions
// Block b sums y[b*2048, (b+1)*2048) in a fixed pattern; the last block
// combines the per-block partials in a fixed pattern.
__device__ __forceinline__ double block_sum_fixed(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
#pragma unroll
  for (int s = kRedThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double block_max(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
#pragma unroll
  for (int s = kRedThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// Grid barrier of the iteration kernels (every CTA resident: tail grids are
// at most one CTA per SM, the fused kernel's is sized from the occupancy): arrive on ctl->bar_count, the last CTA
// resets it and bumps ctl->bar_gen (read as gen0 before arriving).
__device__ __forceinline__ void grid_barrier(gpic_ctl* ctl, unsigned gen0) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctl->bar_count, 1u) == gridDim.x - 1) {
      ctl->bar_count = 0u;
      __threadfence();
      atomicAdd(&ctl->bar_gen, 1u);
    } else {
      unsigned g;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&ctl->bar_gen) : "memory");
        if (g != gen0) break;
        __nanosleep(32);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// Phase 1: CTA-strided fixed 2048-element chunks of y -> part[b].
// kCG: y was written earlier in the same kernel by other CTAs (L2 loads).
// The tail's CTAs are blockIdx.x < ncta (all of them in tail_kernel).
// ready != null: chunk b is summed once ready[b] counts all its 128-row
// tiles (published by the CTAs that wrote them, same kernel); reset here.
template <bool kCG>
__device__ __forceinline__ void chunk_sums(const double* __restrict__ y, int64_t n,
                                           double* __restrict__ part, double* sh,
                                           unsigned ncta, unsigned* ready = nullptr) {
  const int64_t nb = (n + kRedBlock - 1) / kRedBlock;
  for (int64_t b = blockIdx.x; b < nb; b += ncta) {
    const int64_t b0 = b * kRedBlock;
    if (ready != nullptr) {
      if (threadIdx.x == 0) {
        const int64_t rows = n - b0 < kRedBlock ? n - b0 : kRedBlock;
        const unsigned want = (unsigned)((rows + 127) / 128);
        unsigned g;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(ready + b) : "memory");
          if (g >= want) break;
          __nanosleep(20);
        }
        ready[b] = 0u;
      }
      __syncthreads();
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kRedPer; ++q) {
      const int64_t i = b0 + threadIdx.x + q * kRedThreads;
      if (i < n) s += kCG ? __ldcg(y + i) : y[i];
    }
    s = block_sum_fixed(s, sh);
    if (threadIdx.x == 0) part[b] = s;
  }
}

// v' = y / tau, delta = max|v' - v| (order-free), the last CTA done records
// delta and applies the stop rule.
template <bool kCG>
__device__ __forceinline__ void normalise(const double* __restrict__ y, int64_t n,
                                          double* __restrict__ v64, float* __restrict__ v32,
                                          double* __restrict__ hist, gpic_ctl* ctl, int t,
                                          double tau, double* sh, unsigned ncta) {
  __shared__ bool s_last;
  const int64_t nb = (n + kRedBlock - 1) / kRedBlock;
  const double* __restrict__ vold = v64 + (int64_t)(t & 1) * n;
  double* __restrict__ vnew = v64 + (int64_t)((t + 1) & 1) * n;
  double m = 0.0;
  for (int64_t b = blockIdx.x; b < nb; b += ncta) {
    const int64_t b0 = b * kRedBlock;
#pragma unroll
    for (int q = 0; q < kRedPer; ++q) {
      const int64_t i = b0 + threadIdx.x + q * kRedThreads;
      if (i < n) {
        const double vn = (kCG ? __ldcg(y + i) : y[i]) / tau;
        m = fmax(m, fabs(vn - vold[i]));
        vnew[i] = vn;
        v32[i] = (float)vn;
      }
    }
  }
  m = block_max(m, sh);
  if (threadIdx.x == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(&ctl->delta_bits),
              (unsigned long long)__double_as_longlong(m));
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&ctl->arrive[1], 1u) == ncta - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    const double delta = __longlong_as_double((long long)ctl->delta_bits);
    hist[t] = delta;
    ctl->delta_bits = 0ull;
    ctl->arrive[1] = 0u;
    const int done = t + 1;
    ctl->iter = done;
    if (done >= 2 && fabs(delta - hist[t - 1]) <= ctl->eps) {
      ctl->converged = 1;
      ctl->stop = 1;
    } else if (done >= ctl->max_iter) {
      ctl->stop = 1;
    }
  }
}

// Phase 2: the last CTA to arrive combines the partials (tau_kernel's
// pattern) and publishes tau by bumping ctl->tau_gen (read as gen0 by every
// CTA before it arrived); the others spin on it (every CTA resident), then
// all normalise their chunks; the last CTA done records delta and applies
// the stop rule.
template <bool kCG>
__device__ __forceinline__ void finish(const double* __restrict__ y, int64_t n,
                                       double* __restrict__ part, double* __restrict__ v64,
                                       float* __restrict__ v32, double* __restrict__ hist,
                                       gpic_ctl* ctl, int t, unsigned gen0, double* sh,
                                       unsigned ncta) {
  __shared__ bool s_last;
  __shared__ double s_tau;
  const int64_t nb = (n + kRedBlock - 1) / kRedBlock;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&ctl->arrive[0], 1u) == ncta - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    double tt = 0.0;  // tau_kernel's last-block pattern
    for (int64_t i = threadIdx.x; i < nb; i += kRedThreads) tt += __ldcg(part + i);
    tt = block_sum_fixed(tt, sh);
    if (threadIdx.x == 0) {
      ctl->arrive[0] = 0u;
      ctl->tau = tt;
      s_tau = tt;
      if (!(tt > 0.0)) raise_status(ctl, GPIC_E_NONPOS_TAU, 0, -1, tt);
      __threadfence();
      atomicAdd(&ctl->tau_gen, 1u);
    }
  } else if (threadIdx.x == 0) {
    unsigned g;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&ctl->tau_gen) : "memory");
      if (g != gen0) break;
      __nanosleep(32);
    }
    s_tau = *(volatile double*)&ctl->tau;
  }
  __syncthreads();
  if (*(volatile int32_t*)&ctl->stop) return;  // NonPositiveTau
  normalise<kCG>(y, n, v64, v32, hist, ctl, t, s_tau, sh, ncta);
}

// tau inside the list reduce (sym.cu; one CTA per 128-row tile, 128
// threads): the CTA that completes a 2048-row chunk (ready[b] counts its
// tiles) forms the chunk's partial with chunk_sums' exact shape — each
// thread plays threads u and u + 128 of the 256-thread pattern, then the
// same tree — and the CTA that completes the last chunk (ctl->bar_count)
// combines the partials with finish's pattern and stores ctl->tau: bitwise
// the tail's tau, with no tail-side barrier. Call after the CTA wrote y.
__device__ __forceinline__ void tau_in_reduce(const double* y, int64_t n, int64_t R, int64_t nt,
                                              double* __restrict__ part, unsigned* ready,
                                              gpic_ctl* ctl) {
  __shared__ double sh[kRedThreads];
  __shared__ bool s_last;
  constexpr int64_t kChunkTiles = kRedBlock / 128;
  const int u = threadIdx.x;
  const int64_t b = R / kChunkTiles, nb = (n + kRedBlock - 1) / kRedBlock;
  __syncthreads();
  if (u == 0) {
    __threadfence();
    const int64_t r0 = b * kChunkTiles;
    const unsigned want = (unsigned)(nt - r0 < kChunkTiles ? nt - r0 : kChunkTiles);
    s_last = atomicAdd(ready + b, 1u) == want - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t b0 = b * kRedBlock;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int vt = u + 128 * h;
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kRedPer; ++q) {
      const int64_t i = b0 + vt + q * kRedThreads;
      if (i < n) s += __ldcg(y + i);
    }
    sh[vt] = s;
  }
  __syncthreads();
#pragma unroll
  for (int st = kRedThreads / 2; st > 0; st >>= 1) {
    if (u < st) sh[u] += sh[u + st];
    __syncthreads();
  }
  if (u == 0) {
    ready[b] = 0u;
    part[b] = sh[0];
    __threadfence();
    s_last = atomicAdd(&ctl->bar_count, 1u) == nb - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int vt = u + 128 * h;
    double tt = 0.0;
    for (int64_t i = vt; i < nb; i += kRedThreads) tt += __ldcg(part + i);
    sh[vt] = tt;
  }
  __syncthreads();
#pragma unroll
  for (int st = kRedThreads / 2; st > 0; st >>= 1) {
    if (u < st) sh[u] += sh[u + st];
    __syncthreads();
  }
  if (u == 0) {
    const double tt = sh[0];
    ctl->bar_count = 0u;
    ctl->tau = tt;
    if (!(tt > 0.0)) raise_status(ctl, GPIC_E_NONPOS_TAU, 0, -1, tt);
  }
}

}  // namespace tail
}  // namespace gpic
