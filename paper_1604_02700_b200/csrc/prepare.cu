// Stage 0: validate, centre, cast and split the points.
//
// Replaces the finiteness scan of validate_dataset (data.py:61-78) and
// builds the Gram-engine operands. RBF affinities are translation
// invariant, so X is centred in fp64 first (centring cuts
// the fp32 Gram cancellation error by ~5x); the centred rows are cast to
// fp32 and split into a TF32 head and an exact fp32 tail
// (xc = hi + lo exactly) for the 3xTF32 tcgen05 engine.
#include <cfloat>

#include "common.cuh"
#include "ops.h"

namespace gpic {

namespace {

constexpr int kColRows = 256;  // rows per column-sum partial

__global__ void ctl_init_kernel(gpic_ctl* ctl, double eps, int32_t max_iter) {
  if (threadIdx.x == 0) {
    ctl->iter = 0;
    ctl->stop = 0;
    ctl->converged = 0;
    ctl->status = GPIC_OK;
    ctl->err_index = -1;  // all ones: atomicMin identity
    ctl->err_index2 = -1;
    ctl->err_value = 0.0;
    ctl->eps = eps;
    ctl->max_iter = max_iter;
    ctl->nranks = 1;
    ctl->delta_bits = 0ull;
    for (int i = 0; i < 4; ++i) ctl->arrive[i] = 0u;
    ctl->tau = 0.0;
    ctl->sync_epoch = 0ull;
  }
}

// Partial column sums over a fixed block of kColRows rows, plus the
// non-finite scan (first offending element in row-major order wins).
__global__ void colsum_kernel(const double* __restrict__ x, int64_t n, int32_t d,
                              double* __restrict__ colpart, gpic_ctl* ctl) {
  const int64_t r0 = (int64_t)blockIdx.x * kColRows;
  const int64_t r1 = min(r0 + kColRows, n);
  for (int f = threadIdx.x; f < d; f += blockDim.x) {
    double s = 0.0;
    for (int64_t i = r0; i < r1; ++i) {
      double v = x[i * d + f];
      if (!isfinite(v)) {
        raise_status(ctl, GPIC_E_NONFINITE, i * d + f, -1, v);
        v = 0.0;
      }
      s += v;
    }
    colpart[(int64_t)blockIdx.x * d + f] = s;
  }
}

__global__ void mean_kernel(const double* __restrict__ colpart, int64_t nblk, int64_t n, int32_t d,
                            double* __restrict__ mean) {
  for (int f = threadIdx.x; f < d; f += blockDim.x) {
    double s = 0.0;
    for (int64_t b = 0; b < nblk; ++b) s += colpart[b * d + f];
    mean[f] = s / (double)n;
  }
}

// One warp per (padded) row: centre in fp64, cast to fp32, split into
// TF32 hi + fp32 lo, and the fp64-accumulated squared norm of the fp32 row.
__global__ void center_split_kernel(const double* __restrict__ x, int64_t n, int32_t d, int32_t dp,
                                    int64_t n_pad, const double* __restrict__ mean,
                                    float* __restrict__ xhi, float* __restrict__ xlo,
                                    float* __restrict__ sqn) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= n_pad) return;
  double sq = 0.0;
  for (int f = lane; f < dp; f += 32) {
    float xc = 0.f;
    if (row < n && f < d) {
      double v = x[row * d + f];
      if (!isfinite(v)) v = mean[f];
      xc = (float)(v - mean[f]);
    }
    const float hi = to_tf32(xc);
    const float lo = xc - hi;
    xhi[row * dp + f] = hi;
    xlo[row * dp + f] = lo;
    sq += (double)xc * (double)xc;
  }
  sq = warp_sum_f64(sq);
  if (lane == 0) sqn[row] = (float)sq;
}

// Cosine kind (affinity.py:41-53, 88-95): one warp per (padded) row, fp64
// norm, ZeroVector(first row) for a zero row, unit row cast to fp32 and
// split; the Gram engine then yields cos(x_i, x_j) directly.
__global__ void normalize_split_kernel(const double* __restrict__ x, int64_t n, int32_t d,
                                       int32_t dp, int64_t n_pad, float* __restrict__ xhi,
                                       float* __restrict__ xlo, float* __restrict__ sqn,
                                       gpic_ctl* ctl) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= n_pad) return;
  double sq = 0.0;
  if (row < n)
    for (int f = lane; f < d; f += 32) {
      double v = x[row * d + f];
      if (!isfinite(v)) v = 0.0;
      sq += v * v;
    }
  sq = warp_sum_f64(sq);
  if (row < n && sq == 0.0) {
    if (lane == 0) raise_status(ctl, GPIC_E_ZERO_VECTOR, row, -1, 0.0);
  }
  const double inv = sq > 0.0 ? 1.0 / sqrt(sq) : 0.0;
  for (int f = lane; f < dp; f += 32) {
    float xc = 0.f;
    if (row < n && f < d) {
      const double v = x[row * d + f];
      xc = isfinite(v) ? (float)(v * inv) : 0.f;
    }
    const float hi = to_tf32(xc);
    xhi[row * dp + f] = hi;
    xlo[row * dp + f] = xc - hi;
  }
  if (lane == 0) sqn[row] = 1.f;
}

}  // namespace

void launch_ctl_init(gpic_ctl* ctl, double eps, int32_t max_iter, cudaStream_t s) {
  ctl_init_kernel<<<1, 32, 0, s>>>(ctl, eps, max_iter);
  count_launch();
}

void launch_prepare(const double* x, int64_t n, int32_t d, float* xhi, float* xlo, float* sqn,
                    double* colpart, double* mean, gpic_ctl* ctl, cudaStream_t s, int kind) {
  const int64_t nblk = ceil_div(n, kColRows);
  const int threads = d >= 256 ? 256 : (int)round_up(d, 32);
  const int32_t dp = feature_pitch(d);
  const int64_t n_pad = row_pad(n);
  colsum_kernel<<<(unsigned)nblk, threads, 0, s>>>(x, n, d, colpart, ctl);  // + finiteness scan
  if (kind == GPIC_KIND_COSINE) {
    normalize_split_kernel<<<(unsigned)ceil_div(n_pad, 8), 256, 0, s>>>(x, n, d, dp, n_pad, xhi,
                                                                        xlo, sqn, ctl);
    count_launch(2);
    return;
  }
  mean_kernel<<<1, threads, 0, s>>>(colpart, nblk, n, d, mean);
  center_split_kernel<<<(unsigned)ceil_div(n_pad, 8), 256, 0, s>>>(x, n, d, dp, n_pad, mean, xhi,
                                                                  xlo, sqn);
  count_launch(3);
}

}  // namespace gpic
