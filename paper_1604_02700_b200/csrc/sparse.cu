// Block sparsity of A: tiles that are exactly zero in fp32, proved before
// they are computed.
//
// A_ij = exp(-|x_i - x_j|^2 / 2 sigma^2) is an fp32 zero whenever the
// exponent is below the smallest normal float (ex2.approx.ftz flushes:
// |x_i - x_j|^2 / 2 sigma^2 > 87.3). Well-separated clusters make most of
// A such zeros (config 3: the ~90 % of tile pairs that join two different
// blobs, e^-104). For every 128-row tile I a bounding sphere (centre c_I,
// radius r_I, over the centred rows the engines read) gives, for every pair
// (I, J), the lower bound dist >= |c_I - c_J| - r_I - r_J; a tile whose
// bound puts every exponent beyond kZeroExponent (100, i.e. 13 units of
// margin in the exponent over the fp32 flush, far above the engines'
// rounding) holds only zeros, so
//   * the affinity engines skip it (no operand load, MMA, exp or store),
//   * the GEMV skips it (no HBM read) and the degree combine adds nothing,
// and every stored value, degree and product is bit-identical to the dense
// computation (adding an exact zero changes no fp32 / fp64 sum).
//
// Work balance: the engines walk their packed work units in order; with most
// units skipped, each CTA's range is cut by the prefix count of NON-zero
// units (sparse_item_prefix) and the GEMV's by a per-super-block weight
// prefix, so CTAs get equal real work.
#include <cmath>

#include "common.cuh"
#include "ops.h"

namespace gpic {

namespace {

constexpr int kT = 128;            // rows per tile
constexpr double kZeroExponent = 100.0;
constexpr int kScanThreads = 1024;

// One CTA per row tile: centre (fp64 mean of the valid rows) and radius
// (max distance to it, rounded up by a relative 1e-6) of the centred fp32
// rows xc (pitch dp).
__global__ void tile_sphere_kernel(const float* __restrict__ xc, int64_t n, int32_t d, int32_t dp,
                                   double* __restrict__ centre, double* __restrict__ radius) {
  __shared__ double red[32];
  const int64_t I = blockIdx.x;
  const int64_t r0 = I * kT;
  const int rows = (int)(n - r0 < kT ? n - r0 : kT);
  double* c = centre + I * d;
  for (int f = threadIdx.x; f < d; f += blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < rows; ++r) s += (double)xc[(r0 + r) * dp + f];
    c[f] = s / rows;
  }
  __syncthreads();
  double mx = 0.0;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) {
    double s = 0.0;
    for (int f = 0; f < d; ++f) {
      const double t = (double)xc[(r0 + r) * dp + f] - c[f];
      s += t * t;
    }
    mx = fmax(mx, sqrt(s));
  }
  mx = warp_max_f64(mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, red[w]);
    radius[I] = m * (1.0 + 1e-6) + 1e-30;
  }
}

// zero[tile_index(I, J)] for the packed upper triangle (J >= I)
__global__ void tile_mask_kernel(const double* __restrict__ centre, const double* __restrict__ radius,
                                 int64_t nt, int32_t d, double inv2s2, uint8_t* __restrict__ zero) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = nt * (nt + 1) / 2;
  if (t >= total) return;
  // packed index -> (I, J): I = largest with I nt - I (I - 1) / 2 <= t
  int64_t lo = 0, hi = nt - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (mid * nt - mid * (mid - 1) / 2 <= t) lo = mid; else hi = mid - 1;
  }
  const int64_t I = lo, J = I + (t - (I * nt - I * (I - 1) / 2));
  const double* a = centre + I * d;
  const double* b = centre + J * d;
  double s = 0.0;
  for (int f = 0; f < d; ++f) {
    const double q = a[f] - b[f];
    s += q * q;
  }
  const double lb = sqrt(s) * (1.0 - 1e-9) - radius[I] - radius[J];
  zero[t] = (lb > 0.0 && lb * lb * inv2s2 > kZeroExponent) ? 1 : 0;
}

__device__ __forceinline__ bool tile_zero(const uint8_t* zero, int64_t I, int64_t J, int64_t nt) {
  if (I >= nt || J >= nt) return true;  // past the matrix: nothing to compute
  if (J < I) {
    const int64_t t = I;
    I = J;
    J = t;
  }
  return zero[I * nt - I * (I - 1) / 2 + (J - I)] != 0;
}

// Inclusive prefix (int64) of per-element weights produced by `weight(i)`,
// one CTA: each thread sums a contiguous segment, the segment totals are
// scanned, then each thread writes its segment's prefixes. out[0] = 0,
// out[i + 1] = sum of weights [0, i].
template <typename W>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(int64_t count, W weight,
                                                            int64_t* __restrict__ out) {
  __shared__ int64_t sh[kScanThreads];
  const int t = threadIdx.x;
  const int64_t seg = (count + kScanThreads - 1) / kScanThreads;
  const int64_t a = t * seg, b = min(count, a + seg);
  int64_t s = 0;
  for (int64_t i = a; i < b; ++i) s += weight(i);
  sh[t] = s;
  __syncthreads();
  for (int o = 1; o < kScanThreads; o <<= 1) {  // Hillis-Steele inclusive scan
    const int64_t v = t >= o ? sh[t - o] : 0;
    __syncthreads();
    sh[t] += v;
    __syncthreads();
  }
  int64_t run = t > 0 ? sh[t - 1] : 0;
  if (t == 0) out[0] = 0;
  for (int64_t i = a; i < b; ++i) {
    run += weight(i);
    out[i + 1] = run;
  }
}

// packed work unit u of the affinity engine (row block rb of MB tile rows,
// column tile cb >= rb * MB) is real work unless all its MB tiles are zero
struct ItemWeight {
  const uint8_t* zero;
  int64_t nt, n_ctiles;
  int mb;
  __device__ int64_t operator()(int64_t u) const {
    int64_t lo = 0, hi = (nt + mb - 1) / mb - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (mid * n_ctiles - (int64_t)mb * mid * (mid - 1) / 2 <= u) lo = mid; else hi = mid - 1;
    }
    const int64_t rb = lo, cb = rb * mb + (u - (rb * n_ctiles - (int64_t)mb * rb * (rb - 1) / 2));
    for (int m = 0; m < mb; ++m)
      if (!tile_zero(zero, rb * mb + m, cb, nt)) return 1;
    return 0;
  }
};

// GEMV super-block (P, Q >= P) of 4 x 4 tiles: weight = 8 x its non-zero
// tiles + 1 (the records it writes either way)
struct SbWeight {
  const uint8_t* zero;
  int64_t nt, ns;
  __device__ int64_t operator()(int64_t s) const {
    int64_t lo = 0, hi = ns - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (mid * ns - mid * (mid - 1) / 2 <= s) lo = mid; else hi = mid - 1;
    }
    const int64_t P = lo, Q = P + (s - (P * ns - P * (P - 1) / 2));
    int64_t w = 1;
    for (int64_t I = 4 * P; I < min(4 * P + 4, nt); ++I)
      for (int64_t J = max(I, 4 * Q); J < min(4 * Q + 4, nt); ++J)
        if (!tile_zero(zero, I, J, nt)) w += 8;
    return w;
  }
};

}  // namespace

int64_t sparse_mask_bytes(int64_t n, int32_t d) {
  const int64_t nt = ceil_div(n, kT);
  const int64_t ns = ceil_div(nt, 4);
  auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  return al(nt * d * 8) + al(nt * 8) + al(nt * (nt + 1) / 2) +
         al((packed_items_mb(n, 1) + 1) * 8) + al((packed_items_mb(n, 2) + 1) * 8) +
         al((ns * (ns + 1) / 2 + 1) * 8);
}

int64_t packed_items_mb(int64_t n, int mb) {
  const int64_t nrt = ceil_div(n, (int64_t)kT * mb), nct = ceil_div(n, kT);
  return nrt * nct - (int64_t)mb * nrt * (nrt - 1) / 2;
}

SparseMask carve_sparse(void* base, int64_t n, int32_t d) {
  auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  const int64_t nt = ceil_div(n, kT);
  const int64_t ns = ceil_div(nt, 4);
  uint8_t* p = static_cast<uint8_t*>(base);
  SparseMask m;
  m.nt = nt;
  m.centre = reinterpret_cast<double*>(p); p += al(nt * d * 8);
  m.radius = reinterpret_cast<double*>(p); p += al(nt * 8);
  m.zero = p; p += al(nt * (nt + 1) / 2);
  m.item_prefix1 = reinterpret_cast<int64_t*>(p); p += al((packed_items_mb(n, 1) + 1) * 8);
  m.item_prefix2 = reinterpret_cast<int64_t*>(p); p += al((packed_items_mb(n, 2) + 1) * 8);
  m.sb_prefix = reinterpret_cast<int64_t*>(p);
  m.n_sb = ns * (ns + 1) / 2;
  return m;
}

void launch_sparse_mask(const SparseMask& m, const float* xc, int64_t n, int32_t d, int32_t dp,
                        double sigma, cudaStream_t s) {
  const int64_t nt = m.nt;
  tile_sphere_kernel<<<(unsigned)nt, 128, 0, s>>>(xc, n, d, dp, m.centre, m.radius);
  const int64_t tiles = nt * (nt + 1) / 2;
  tile_mask_kernel<<<(unsigned)ceil_div(tiles, 256), 256, 0, s>>>(
      m.centre, m.radius, nt, d, 1.0 / (2.0 * sigma * sigma), m.zero);
  const int64_t nct = nt;
  scan_kernel<<<1, kScanThreads, 0, s>>>(packed_items_mb(n, 1), ItemWeight{m.zero, nt, nct, 1},
                                         m.item_prefix1);
  scan_kernel<<<1, kScanThreads, 0, s>>>(packed_items_mb(n, 2), ItemWeight{m.zero, nt, nct, 2},
                                         m.item_prefix2);
  scan_kernel<<<1, kScanThreads, 0, s>>>(m.n_sb, SbWeight{m.zero, nt, ceil_div(nt, 4)},
                                         m.sb_prefix);
  count_launch(5);
}

}  // namespace gpic
