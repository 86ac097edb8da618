// Low-degree rows: isolated points whose fp32 affinities underflow
// (SURVEY.md §7 H4).
//
// The reference computes A in fp64 (affinity.py:96-101): exp underflows only
// below -745, so a point ~13 sigma from every other point keeps a tiny but
// positive degree (6e-85 for a point 20 sigma out) and a perfectly
// well-defined W row (affinity.py:122-127); ZeroDegree fires only when the
// fp64 row sum is exactly 0 (affinity.py:113-119). The stored engines
// compute A in fp32 with ex2.approx.ftz: every entry of such a row flushes
// to 0 and entries below ~1e-38 are lost in any row whose degree is tiny.
//
// Rows whose engine degree is below kLowDegree (kind-specific) are therefore
// redone in fp64 from the caller's original X, with the reference's own
// arithmetic (per-feature differences, rounded product then add, exp of
// d2 * (-1 / (2 sigma^2)); the cosine kind: feature-ordered dots and norms,
// max(0, .)):
//   * lowdeg_scan    lists them (device counter; the host reads it once);
//   * lowdeg_exact   their exact fp64 degrees (overwriting the engine's), and
//                    ZeroDegree(first row) only when that degree is 0;
//   * lowdeg_matvec  every iteration, y_i = sum_j (a_ij / d_i) v_j for those
//                    rows from the fp64 v, after the engine's GEMV wrote y.
// Their columns need no fix: a_ji <= d_i < kLowDegree is below the fp32
// resolution of any normal row's degree, as in the reference's fp64 sums.
// No row below the threshold: nothing is launched beyond the scan.
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "lowdeg.cuh"
#include "ops.h"

namespace gpic {

namespace {

using lowdeg::kLowThreads;
using lowdeg::kSmemD;
using lowdeg::affinity_f64;
using lowdeg::norm_f64;
using lowdeg::block_sum;

__global__ void lowdeg_scan_kernel(const double* __restrict__ deg, int64_t n, double thresh,
                                   int64_t* __restrict__ list, unsigned long long* count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = deg[i];
  if (!(d >= thresh)) {  // also catches NaN
    const unsigned long long slot = atomicAdd(count, 1ull);
    list[slot] = i;
  }
}

// One CTA per listed row: sum_j a_ij * (v_j [/ d_i]) in a fixed order
// (thread-strided partials, then warp / CTA trees) -> out.
template <bool kMatvec>
__global__ void __launch_bounds__(kLowThreads)
    lowdeg_row_kernel(const double* __restrict__ x, int64_t n, int32_t d, int kind, double scale,
                      const int64_t* __restrict__ list, const unsigned long long* count,
                      double* __restrict__ deg, const double* __restrict__ v64,
                      double* __restrict__ y0, double* __restrict__ y1, gpic_ctl* ctl) {
  __shared__ double sh[kLowThreads / 32];
  extern __shared__ double xs[];
  if (kMatvec && *(volatile int32_t*)&ctl->stop) return;
  const unsigned long long cnt = *count;  // the grid strides over the listed rows
  for (unsigned long long r = blockIdx.x; r < cnt; r += gridDim.x) {
    const int64_t i = list[r];
    if (kMatvec) {
      const int t = ctl->iter;
      const double s = lowdeg::matvec_row(x, n, d, kind, scale, i, deg[i],
                                          v64 + (int64_t)(t & 1) * n, xs, sh);
      if (threadIdx.x == 0) ((t & 1) ? y1 : y0)[i] = s;
      continue;
    }
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
      s += affinity_f64(xi, xj, d, kind, scale, ni, nj);
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) {
      deg[i] = s;
      if (!(s > 0.0)) raise_status(ctl, GPIC_E_ZERO_DEGREE, i, -1, s);
    }
  }
}

}  // namespace

double low_degree_threshold(int kind, int64_t n) {
  // RBF: the engines flush entries below 2^-64 (sm100.cuh kFlushLog2); n of
  // them stay below 2^-24 of any degree above n 2^-40 (and below 1e-20 the
  // fp32 row is gone anyway); cosine: the fp32 Gram's ~1e-7 absolute error
  // per entry dominates a degree < 1e-2
  if (kind == GPIC_KIND_COSINE) return 1e-2;
  const double t = (double)n * 0x1p-40;
  return t > 1e-20 ? t : 1e-20;
}

void launch_lowdeg_scan(const double* deg, int64_t n, int kind, int64_t* list,
                        unsigned long long* count, cudaStream_t s) {
  cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
  lowdeg_scan_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(
      deg, n, low_degree_threshold(kind, n), list, count);
  count_launch();
}

int read_low_count(const unsigned long long* d_count, int64_t* out, cudaStream_t s) {
  unsigned long long h = 0;
  GPIC_CUDA_TRY(cudaMemcpyAsync(&h, d_count, sizeof h, cudaMemcpyDeviceToHost, s));
  GPIC_CUDA_TRY(cudaStreamSynchronize(s));
  *out = (int64_t)h;
  return GPIC_OK;
}

static double rbf_scale(const LowRows& L) { return -1.0 / (2.0 * L.sigma * L.sigma); }
static size_t smem_bytes(int32_t d) { return (size_t)(d <= kSmemD ? d : 0) * sizeof(double); }

// grid: one CTA per listed row up to kLowGrid; count < 0 = not read back
// (the kernel strides over the device-side count, no host sync)
constexpr int64_t kLowGrid = 296;
static unsigned low_grid(int64_t count) {
  return (unsigned)(count < 0 || count > kLowGrid ? kLowGrid : count);
}

void launch_lowdeg_exact(const LowRows& L, double* deg, gpic_ctl* ctl, cudaStream_t s) {
  if (L.count == 0) return;
  lowdeg_row_kernel<false><<<low_grid(L.count), kLowThreads, smem_bytes(L.d), s>>>(
      L.x, L.n, L.d, L.kind, rbf_scale(L), L.list, L.d_count, deg, nullptr, nullptr, nullptr, ctl);
  count_launch();
}

void launch_lowdeg_matvec(const LowRows& L, const double* deg, const double* v64, double* y0,
                          double* y1, gpic_ctl* ctl, cudaStream_t s) {
  if (L.count == 0) return;
  lowdeg_row_kernel<true><<<low_grid(L.count), kLowThreads, smem_bytes(L.d), s>>>(
      L.x, L.n, L.d, L.kind, rbf_scale(L), L.list, L.d_count, const_cast<double*>(deg), v64, y0,
      y1, ctl);
  count_launch();
}

}  // namespace gpic
