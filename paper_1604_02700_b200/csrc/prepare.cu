// Stage 0: validate, centre, cast and split the points.
//
// Replaces the finiteness scan of validate_dataset (data.py:61-78) and
// builds the Gram-engine operands. RBF affinities are translation
// invariant, so X is centred in fp64 first (centring cuts
// the fp32 Gram cancellation error by ~5x). Two operand forms come out:
//
//   xc   (d_xlo buffer)  fp32 centred rows, pitch dp — the FFMA engine
//   hi/lo planes (d_xhi buffer, fp16, pitch dp, hi plane then lo plane)
//        xs = xc * s with s = 2^e chosen so max|xs| < 2^8 (exact scaling),
//        hi = fp16(xs), lo = fp16(xs - hi): the 3-term split of the
//        tcgen05 kind::f16 engine (hi.hi + hi.lo + lo.hi, fp32 accumulate);
//        1/s^2 is stored in the padding slot sqn[n_pad - 1]
//   norm block (after the planes; RBF): a 16-wide K extension that makes
//        the MMA accumulate -(s^2/2)|x_i - x_j|^2 directly:
//            row operand    [2^10, M_i, 0 ...]   (hi / lo planes)
//            column operand [M_j, 2^10, 0 ...]   M = -(s^2/2)|x~|^2 / 2^10
//        so acc = s^2 x_i.x_j + 2^10 M_j + 2^10 M_i, with |x~|^2 taken from
//        the split operands themselves (x~ = (hi + lo) / s), which keeps the
//        distance of a point to itself at the accumulator's rounding level.
//        Four planes [row hi][row lo][column hi][column lo], each n_pad rows
//        x 16 fp16 (32 B rows), loaded by TMA with the 32-byte swizzle.
//
// fp16 and TF32 both carry 11 significant bits, so the 3-term fp16 split
// is as accurate as 3xTF32 (the fp32 accumulation dominates both), with
// half the operand bytes per MMA and twice the tensor-pipe rate.
#include <cuda_fp16.h>

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
    ctl->bar_count = 0u;
  }
}

// Partial column sums over a fixed block of kColRows rows, plus the
// non-finite scan (first offending element in row-major order wins).
// blockDim = kGroups x (d rounded up to 32, <= 256): group g sums rows
// r0 + g, r0 + g + kGroups, ... (8 loads in flight), the groups are added
// in order through shared memory — a fixed order.
constexpr int kGroups = 4;
__global__ void colsum_kernel(const double* __restrict__ x, int64_t n, int32_t d,
                              double* __restrict__ colpart, gpic_ctl* ctl) {
  __shared__ double part[kGroups][256];
  const int64_t r0 = (int64_t)blockIdx.x * kColRows;
  const int64_t r1 = min(r0 + kColRows, n);
  const int width = blockDim.x / kGroups;
  const int g = threadIdx.x / width, t = threadIdx.x % width;
  for (int f0 = 0; f0 < d; f0 += width) {
    const int f = f0 + t;
    double s = 0.0;
    if (f < d) {
      int64_t i = r0 + g;
      for (; i + 7 * kGroups < r1; i += 8 * kGroups) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = x[(i + u * kGroups) * d + f];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (!isfinite(v[u])) {
            raise_status(ctl, GPIC_E_NONFINITE, (i + u * kGroups) * d + f, -1, v[u]);
            v[u] = 0.0;
          }
          s += v[u];
        }
      }
      for (; i < r1; i += kGroups) {
        double v = x[i * d + f];
        if (!isfinite(v)) {
          raise_status(ctl, GPIC_E_NONFINITE, i * d + f, -1, v);
          v = 0.0;
        }
        s += v;
      }
    }
    part[g][t] = s;
    __syncthreads();
    if (g == 0 && f < d) {
      double tot = part[0][t];
#pragma unroll
      for (int q = 1; q < kGroups; ++q) tot += part[q][t];
      colpart[(int64_t)blockIdx.x * d + f] = tot;
    }
    __syncthreads();
  }
}

// mean[f] = sum of the block partials / n: 8 segments per feature (a warp
// of 32 threads covers 4 features), segment sums added in order
__global__ void mean_kernel(const double* __restrict__ colpart, int64_t nblk, int64_t n, int32_t d,
                            double* __restrict__ mean) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int f = (blockIdx.x * (blockDim.x >> 5) + w) * 4 + (lane >> 3);
  const int sg = lane & 7;
  double s = 0.0;
  if (f < d) {
    const int64_t b0 = nblk * sg / 8, b1 = nblk * (sg + 1) / 8;
    for (int64_t b = b0; b < b1; ++b) s += colpart[b * d + f];
  }
  // segments 0..7 of a feature sit in consecutive lanes: add them in order
  double tot = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) tot += __shfl_sync(0xffffffffu, s, (lane & ~7) + q);
  if (sg == 0 && f < d) mean[f] = tot / (double)n;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    mean[d] = 0.0;      // max |x - mean| (maxabs_kernel)
    mean[d + 1] = 0.0;  // max_i |x_i - mean|^2 (center_split_kernel): the spread R^2
  }
}

// max |x - mean| over all finite entries -> mean[d] (non-negative doubles
// order like their bit patterns, so an integer atomicMax is exact)
// A warp per row (lanes over the features, no index division), four rows
// of loads in flight per warp.
__global__ void __launch_bounds__(256)
    maxabs_kernel(const double* __restrict__ x, int64_t n, int32_t d,
                  double* __restrict__ mean) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t stride = (int64_t)gridDim.x * 8;
  double m = 0.0;
  for (int64_t r0 = (int64_t)blockIdx.x * 8 + warp; r0 < n; r0 += 4 * stride) {
    for (int f = lane; f < d; f += 32) {
      const double mf = mean[f];
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t row = r0 + u * stride;
        v[u] = row < n ? x[row * d + f] : mf;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (isfinite(v[u])) m = fmax(m, fabs(v[u] - mf));
    }
  }
  m = warp_max_f64(m);
  if ((threadIdx.x & 31) == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(mean + d), (unsigned long long)__double_as_longlong(m));
}

// s = 2^e with max|x| * s < 2^8 (1 when every row is the mean); 2^8 keeps
// the norm block's M = (s^2/2)|x|^2 / 2^10 <= 32 d inside fp16 range
__device__ __forceinline__ double operand_scale(double maxabs) {
  if (!(maxabs > 0.0)) return 1.0;
  int e;
  frexp(maxabs, &e);  // maxabs < 2^e
  const int sh = 8 - e;  // clamped so 1/s^2 stays a normal fp32
  return ldexp(1.0, sh < -60 ? -60 : (sh > 60 ? 60 : sh));
}

// returns (double)(hi + lo), the split operand's value
__device__ __forceinline__ double split16(double xs, __half* hi, __half* lo, int64_t at) {
  const float x32 = (float)xs;
  const __half h = __float2half_rn(x32);
  const __half l = __float2half_rn(x32 - __half2float(h));
  hi[at] = h;
  lo[at] = l;
  return (double)__half2float(h) + (double)__half2float(l);
}

// Warps stride over the (padded) rows: centre in fp64, fp32 row for the
// FFMA engine, scaled fp16 hi/lo planes for the tensor engine,
// fp64-accumulated squared norm of the fp32 row, and the row's entries of
// the norm block. The spread max_i |x_i - mean|^2 is reduced per CTA and
// published with one atomic per CTA (a per-row atomic on one address
// serialised the kernel).
__global__ void __launch_bounds__(256)
    center_split_kernel(const double* __restrict__ x, int64_t n, int32_t d, int32_t dp,
                        int64_t n_pad, double* __restrict__ mean, __half* __restrict__ hi,
                        float* __restrict__ xc_out, float* __restrict__ sqn) {
  __shared__ double wmax[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __half* lo = hi + n_pad * dp;
  const double s = operand_scale(mean[d]);
  const int64_t plane = n_pad * 16;
  double spread = 0.0;
  // two rows per warp pass (both rows' loads in flight together)
  constexpr int kR = 2;
  const int64_t step = (int64_t)gridDim.x * 8 * kR;
  for (int64_t row0 = ((int64_t)blockIdx.x * 8 + warp) * kR; row0 < n_pad; row0 += step) {
    double sq[kR], sqs[kR];
#pragma unroll
    for (int u = 0; u < kR; ++u) sq[u] = sqs[u] = 0.0;
    for (int f = lane; f < dp; f += 32) {
      double c[kR];
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        const int64_t row = row0 + u;
        c[u] = 0.0;
        if (row < n && f < d) {
          double v = x[row * d + f];
          if (!isfinite(v)) v = mean[f];
          c[u] = v - mean[f];
        }
      }
#pragma unroll
      for (int u = 0; u < kR; ++u) {
        const int64_t row = row0 + u;
        if (row >= n_pad) break;
        const float xc = (float)c[u];
        xc_out[row * dp + f] = xc;
        const double t = split16(c[u] * s, hi, lo, row * dp + f);
        sq[u] += (double)xc * (double)xc;
        sqs[u] += t * t;  // |x~ s|^2 of the split operands
      }
    }
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      sq[u] = warp_sum_f64(sq[u]);
      sqs[u] = warp_sum_f64(sqs[u]);
    }
#pragma unroll
    for (int u = 0; u < kR; ++u) {
      const int64_t row = row0 + u;
      if (row >= n_pad) break;
      if (lane == 0) sqn[row] = row == n_pad - 1 ? (float)(1.0 / (s * s)) : (float)sq[u];
      if (row < n) spread = fmax(spread, sq[u]);  // spread R^2 for the engine routing
      // norm block: lanes 0-15 write k = lane of the row / column operands
      __half* nb = lo + n_pad * dp + row * 16 + lane;
      if (lane < 16) {
        const double m = row < n ? -0.5 * sqs[u] / 1024.0 : 0.0;
        const __half mh = __float2half_rn((float)m);
        const __half ml = __float2half_rn((float)(m - (double)__half2float(mh)));
        const __half one = __float2half_rn(1024.f), zero = __float2half_rn(0.f);
        nb[0] = lane == 0 ? one : (lane == 1 ? mh : zero);          // row operand hi
        nb[plane] = lane == 1 ? ml : zero;                           // row operand lo
        nb[2 * plane] = lane == 0 ? mh : (lane == 1 ? one : zero);   // column operand hi
        nb[3 * plane] = lane == 0 ? ml : zero;                       // column operand lo
      }
    }
  }
  if (lane == 0) wmax[warp] = spread;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = wmax[0];
    for (int w = 1; w < 8; ++w) m = fmax(m, wmax[w]);
    if (m > 0.0)  // non-negative doubles order like their bit patterns
      atomicMax(reinterpret_cast<unsigned long long*>(mean + d + 1),
                (unsigned long long)__double_as_longlong(m));
  }
}

// Cosine kind (affinity.py:41-53, 88-95): one warp per (padded) row, fp64
// norm, ZeroVector(first row) for a zero row, unit row cast to fp32 and
// split (s = 2^14: unit components); the Gram engines then yield
// cos(x_i, x_j) directly.
__global__ void normalize_split_kernel(const double* __restrict__ x, int64_t n, int32_t d,
                                       int32_t dp, int64_t n_pad, __half* __restrict__ hi,
                                       float* __restrict__ xc_out, float* __restrict__ sqn,
                                       gpic_ctl* ctl) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= n_pad) return;
  __half* lo = hi + n_pad * dp;
  constexpr double s = 16384.0;
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
    double u = 0.0;
    if (row < n && f < d) {
      const double v = x[row * d + f];
      u = isfinite(v) ? v * inv : 0.0;
    }
    xc_out[row * dp + f] = (float)u;
    split16(u * s, hi, lo, row * dp + f);
  }
  if (lane == 0) sqn[row] = row == n_pad - 1 ? (float)(1.0 / (s * s)) : 1.f;
  // the norm block is unused by the cosine kind: keep it zero
  if (lane < 16)
    for (int p = 0; p < 4; ++p) lo[n_pad * dp + p * n_pad * 16 + row * 16 + lane] = __float2half_rn(0.f);
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
  __half* planes = reinterpret_cast<__half*>(xhi);
  colsum_kernel<<<(unsigned)nblk, kGroups * threads, 0, s>>>(x, n, d, colpart, ctl);  // + finiteness scan
  if (kind == GPIC_KIND_COSINE) {
    normalize_split_kernel<<<(unsigned)ceil_div(n_pad, 8), 256, 0, s>>>(x, n, d, dp, n_pad, planes,
                                                                        xlo, sqn, ctl);
    count_launch(2);
    return;
  }
  mean_kernel<<<(unsigned)ceil_div(d, 32), 256, 0, s>>>(colpart, nblk, n, d, mean);
  const int64_t mblk = ceil_div(n * d, 256);
  (void)mblk;
  const int64_t xblk = ceil_div(n, 32);  // 8 warps x 4 rows per CTA pass
  maxabs_kernel<<<(unsigned)(xblk < 1184 ? xblk : 1184), 256, 0, s>>>(x, n, d, mean);
  const int64_t cblk = ceil_div(n_pad, 16);
  center_split_kernel<<<(unsigned)(cblk < 148 * 8 ? cblk : 148 * 8), 256, 0, s>>>(
      x, n, d, dp, n_pad, mean, planes, xlo, sqn);
  count_launch(4);
}

}  // namespace gpic
