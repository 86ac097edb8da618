// Device arithmetic of the low-degree rows (lowdeg.cu), shared with the
// fused iteration kernel (sym.cu) so both compute a listed row's y_i with
// the same operations and the same 256-thread summation shape.
#pragma once

#include "common.cuh"

namespace gpic {
namespace lowdeg {

constexpr int kLowThreads = 256;
constexpr int32_t kSmemD = 4096;  // x_i staged in shared memory up to 32 KB

// a_ij in fp64, the reference's operation order (affinity.py:89-101)
__device__ __forceinline__ double affinity_f64(const double* xi,
                                               const double* __restrict__ xj, int32_t d,
                                               int kind, double scale, double ni, double nj) {
  double acc = 0.0;
  if (kind == GPIC_KIND_COSINE) {
    for (int32_t f = 0; f < d; ++f) acc = __dadd_rn(acc, __dmul_rn(xi[f], xj[f]));
    const double c = __ddiv_rn(acc, __dmul_rn(ni, nj));
    return c > 0.0 ? c : 0.0;
  }
  for (int32_t f = 0; f < d; ++f) {
    const double df = __dsub_rn(xi[f], xj[f]);
    acc = __dadd_rn(acc, __dmul_rn(df, df));
  }
  return exp(__dmul_rn(acc, scale));
}

__device__ __forceinline__ double norm_f64(const double* __restrict__ x, int32_t d) {
  double s = 0.0;
  for (int32_t f = 0; f < d; ++f) s = __dadd_rn(s, __dmul_rn(x[f], x[f]));
  return sqrt(s);
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  v = warp_sum_f64(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int q = 0; q < kLowThreads / 32; ++q) t += sh[q];
  __syncthreads();
  return t;
}

// y_i = sum_j (a_ij / d_i) v_j of listed row i (j != i), thread-strided
// partials then the fixed warp / CTA tree; the result is in thread 0.
// `xs`: d doubles of shared memory when d <= kSmemD; `sh`: kLowThreads / 32.
__device__ __forceinline__ double matvec_row(const double* __restrict__ x, int64_t n, int32_t d,
                                             int kind, double scale, int64_t i, double di,
                                             const double* __restrict__ v, double* xs,
                                             double* sh) {
  __syncthreads();  // xs of the previous row is consumed
  const double* xi = d <= kSmemD ? xs : x + i * d;
  if (d <= kSmemD)
    for (int32_t f = threadIdx.x; f < d; f += blockDim.x) xs[f] = x[i * d + f];
  __syncthreads();
  const double ni = kind == GPIC_KIND_COSINE ? norm_f64(xi, d) : 1.0;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    if (j == i) continue;  // affinity.py:102-103
    const double* xj = x + j * d;
    const double nj = kind == GPIC_KIND_COSINE ? norm_f64(xj, d) : 1.0;
    const double a = affinity_f64(xi, xj, d, kind, scale, ni, nj);
    s += __ddiv_rn(a, di) * v[j];  // W = A / d (affinity.py:126), W v
  }
  return block_sum(s, sh);
}

}  // namespace lowdeg
}  // namespace gpic
