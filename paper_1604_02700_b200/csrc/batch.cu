// Batched small-n PIC: the Experiment-II engine.
//
// Experiment II (cli.py:230-256) clusters 18 balanced
// subsamples x 10 repetitions of a dataset: 180 independent PIC runs of
// 2..~400 points each. One launch of the tiled engines per run would spend
// its time in launch latency and host syncs, and a 400-point problem fills
// one SM at most. Here one CTA owns one whole problem, start to finish,
// and a single grid runs the batch:
//
//   pic_small_kernel   finiteness scan (data.py:69-72), cosine norms +
//                      ZeroVector (affinity.py:41-53), fp64 affinity rows in
//                      the reference's feature-by-feature order with the
//                      zero diagonal (affinity.py:88-104), degrees +
//                      ZeroDegree (:113-119), W = A / d (:122-127), v0 =
//                      d / sum(d) (serial.py:90), and the power iteration
//                      with the acceleration stop (serial.py:117-128)
//   k-means            the same lloyd / polish / choose / finish kernels as
//                      the single-problem path, one CTA per problem
//
// Small problems are computed in fp64 with the reference's operation order
// (products and sums rounded separately: no FMA contraction in the affinity),
// so the embedding matches the reference to ~1e-15 and the k-means sees the
// same values. W lives in the workspace (n^2 doubles per problem; 1.3 MB at
// n = 405, L2-resident across the power iteration).
#include <algorithm>
#include <climits>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "ops.h"

namespace gpic {
namespace {

constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;
constexpr int64_t kSmallMaxN = 4096;

struct SmallProblem {
  const double* x;  // n x d, row-major
  int64_t n;
  double* w;        // n x n: A, then W = A / d in place
  double* deg;      // n
  double* v;        // n   result embedding
  double* y;        // n   W v
  double* nrm;      // n   cosine norms
  double* hist;     // max_iter deltas
  double eps;
  gpic_ctl* ctl;
};

__device__ double cta_sum(double v, double* red) {
  v = warp_sum_f64(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < kSmallWarps; ++i) t += red[i];
  return t;
}

__device__ double cta_max(double v, double* red) {
  v = warp_max_f64(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = red[0];
  for (int i = 1; i < kSmallWarps; ++i) t = fmax(t, red[i]);
  return t;
}

__device__ long long cta_min_ll(long long v, long long* red) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  long long t = red[0];
  for (int i = 1; i < kSmallWarps; ++i) t = min(t, red[i]);
  return t;
}

__global__ void __launch_bounds__(kSmallThreads)
    pic_small_kernel(const SmallProblem* __restrict__ probs, int d, int kind, double scale,
                     int max_iter) {
  const SmallProblem P = probs[blockIdx.x];
  __shared__ double red[kSmallWarps];
  __shared__ long long redi[kSmallWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = P.n;
  gpic_ctl* ctl = P.ctl;
  if (tid == 0) {
    ctl->iter = 0;
    ctl->stop = 0;
    ctl->converged = 0;
    ctl->status = GPIC_OK;
    ctl->err_index = -1;
    ctl->err_index2 = -1;
    ctl->err_value = 0.0;
    ctl->eps = P.eps;
    ctl->max_iter = max_iter;
    ctl->nranks = 1;
  }
  __syncthreads();
  const double* __restrict__ x = P.x;

  // 1. first non-finite entry in row-major order
  long long bad = LLONG_MAX;
  for (int64_t i = tid; i < n * d; i += kSmallThreads)
    if (!isfinite(x[i])) { bad = i; break; }
  bad = cta_min_ll(bad, redi);
  if (bad != LLONG_MAX) {
    if (tid == 0) raise_status(ctl, GPIC_E_NONFINITE, bad, -1, 0.0);
    return;
  }

  // 2. cosine norms, accumulated feature by feature
  if (kind == GPIC_KIND_COSINE) {
    long long zero = LLONG_MAX;
    for (int64_t i = tid; i < n; i += kSmallThreads) {
      double sq = 0.0;
      for (int f = 0; f < d; ++f) sq = __dadd_rn(sq, __dmul_rn(x[i * d + f], x[i * d + f]));
      if (sq == 0.0 && zero == LLONG_MAX) zero = i;
      P.nrm[i] = sqrt(sq);
    }
    zero = cta_min_ll(zero, redi);
    if (zero != LLONG_MAX) {
      if (tid == 0) raise_status(ctl, GPIC_E_ZERO_VECTOR, zero, -1, 0.0);
      return;
    }
  }

  // 3. affinity rows (one warp per row) + degrees
  for (int64_t i = warp; i < n; i += kSmallWarps) {
    double part = 0.0;
    for (int64_t j = lane; j < n; j += 32) {
      double a = 0.0;
      if (j != i) {
        if (kind == GPIC_KIND_COSINE) {
          double dots = 0.0;
          for (int f = 0; f < d; ++f) dots = __dadd_rn(dots, __dmul_rn(x[i * d + f], x[j * d + f]));
          a = fmax(__ddiv_rn(dots, __dmul_rn(P.nrm[i], P.nrm[j])), 0.0);
        } else {
          double d2 = 0.0;
          for (int f = 0; f < d; ++f) {
            const double diff = __dsub_rn(x[i * d + f], x[j * d + f]);
            d2 = __dadd_rn(d2, __dmul_rn(diff, diff));
          }
          a = exp(__dmul_rn(d2, scale));
        }
      }
      P.w[i * n + j] = a;
      part += a;
    }
    part = warp_sum_f64(part);
    if (lane == 0) P.deg[i] = part;
  }
  __syncthreads();
  long long zdeg = LLONG_MAX;
  for (int64_t i = tid; i < n; i += kSmallThreads)
    if (!(P.deg[i] > 0.0)) { zdeg = i; break; }
  zdeg = cta_min_ll(zdeg, redi);
  if (zdeg != LLONG_MAX) {
    if (tid == 0) raise_status(ctl, GPIC_E_ZERO_DEGREE, zdeg, -1, P.deg[zdeg]);
    return;
  }

  // 4. W = A / d (row-stochastic), 5. v0 = d / sum(d)
  for (int64_t e = tid; e < n * n; e += kSmallThreads) P.w[e] = __ddiv_rn(P.w[e], P.deg[e / n]);
  double part = 0.0;
  for (int64_t i = tid; i < n; i += kSmallThreads) part += P.deg[i];
  const double total = cta_sum(part, red);
  for (int64_t i = tid; i < n; i += kSmallThreads) P.v[i] = __ddiv_rn(P.deg[i], total);
  __syncthreads();

  // 6. power iteration with the acceleration stop
  double prev = 0.0;
  int t = 0, converged = 0;
  while (t < max_iter) {
    for (int64_t i = warp; i < n; i += kSmallWarps) {
      double acc = 0.0;
      const double* row = P.w + i * n;
      for (int64_t j = lane; j < n; j += 32) acc = fma(row[j], P.v[j], acc);
      acc = warp_sum_f64(acc);
      if (lane == 0) P.y[i] = acc;
    }
    __syncthreads();
    double l1 = 0.0;
    for (int64_t i = tid; i < n; i += kSmallThreads) l1 += fabs(P.y[i]);
    const double tau = cta_sum(l1, red);
    if (!(tau > 0.0)) {
      if (tid == 0) raise_status(ctl, GPIC_E_NONPOS_TAU, 0, -1, tau);
      return;
    }
    double dm = 0.0;
    for (int64_t i = tid; i < n; i += kSmallThreads) {
      const double vn = __ddiv_rn(P.y[i], tau);
      dm = fmax(dm, fabs(vn - P.v[i]));
      P.v[i] = vn;
    }
    const double delta = cta_max(dm, red);
    if (tid == 0) P.hist[t] = delta;
    ++t;
    if (t >= 2 && fabs(delta - prev) <= P.eps) {
      converged = 1;
      break;
    }
    prev = delta;
  }
  if (tid == 0) {
    ctl->iter = t;
    ctl->converged = converged;
    ctl->stop = 1;
  }
}

inline int64_t al(int64_t b) { return (b + 255) & ~int64_t(255); }

int64_t problem_bytes(int64_t n, int32_t k) {
  return al(n * n * 8) + 3 * al(n * 8) + al(kmeans_batch_scratch_bytes(n, k));
}

int64_t header_bytes(int32_t count, int32_t k) {
  return al((int64_t)count * 256) + al((int64_t)count * sizeof(SmallProblem)) +
         al((int64_t)count * kmeans_problem_bytes()) + al((int64_t)count * (k > 1 ? k - 1 : 1) * 8);
}

}  // namespace
}  // namespace gpic

using namespace gpic;

extern "C" {

int64_t gpic_batch_workspace_bytes(const int64_t* h_offsets, int32_t count, int32_t d, int32_t k,
                                   int32_t max_iter) {
  (void)max_iter;
  if (count < 1 || d < 1 || !h_offsets) return -1;
  int64_t total = header_bytes(count, k);
  for (int32_t b = 0; b < count; ++b) {
    const int64_t n = h_offsets[b + 1] - h_offsets[b];
    if (n < 1) return -1;
    total += problem_bytes(n, k);
  }
  return total;
}

int gpic_cluster_batch(const double* d_x, const int64_t* h_offsets, int32_t count, int32_t d,
                       double sigma, int32_t kind, int32_t k, const double* h_eps,
                       int32_t max_iter, const int64_t* h_first, const double* h_uniforms,
                       int64_t* d_labels, double* d_v, double* d_hist, gpic_ctl* h_ctl,
                       void* d_work, int64_t work_bytes, void* stream) {
  if (count < 1 || d < 1 || !h_offsets || !h_eps || !h_first || !h_ctl)
    return fail(GPIC_E_INVALID, "batch needs count >= 1, d >= 1 and every host array");
  if (kind != GPIC_KIND_RBF && kind != GPIC_KIND_COSINE) return fail(GPIC_E_INVALID, "unknown kind");
  if (kind == GPIC_KIND_RBF && !(sigma > 0)) return fail(GPIC_E_INVALID, "sigma must be positive");
  if (k < 2 || k > 64) return fail(GPIC_E_UNSUPPORTED, "k must lie in [2, 64] on the GPU path");
  if (max_iter < 1) return fail(GPIC_E_INVALID, "max_iterations must be at least 1");
  for (int32_t b = 0; b < count; ++b) {
    const int64_t n = h_offsets[b + 1] - h_offsets[b];
    if (n < 1) return fail(GPIC_E_EMPTY, "every problem needs at least one point");
    if (n > kSmallMaxN) return fail(GPIC_E_UNSUPPORTED, "batched problems hold at most 4096 points");
    if (k > n) return fail(GPIC_E_K_TOO_LARGE, "k exceeds the number of points of a problem");
    if (h_first[b] < 0 || h_first[b] >= n) return fail(GPIC_E_INVALID, "first_index out of range");
  }
  const int64_t need = gpic_batch_workspace_bytes(h_offsets, count, d, k, max_iter);
  if (work_bytes < need) return fail(GPIC_E_INVALID, "batch workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int km1 = k - 1;

  uint8_t* p = static_cast<uint8_t*>(d_work);
  gpic_ctl* ctls = reinterpret_cast<gpic_ctl*>(p); p += al((int64_t)count * 256);
  uint8_t* d_small = p; p += al((int64_t)count * sizeof(SmallProblem));
  uint8_t* d_kprob = p; p += al((int64_t)count * kmeans_problem_bytes());
  double* d_unif = reinterpret_cast<double*>(p); p += al((int64_t)count * (km1 > 0 ? km1 : 1) * 8);

  // largest problems first: the CTA scheduler takes blocks in index order
  std::vector<int32_t> order(count);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return h_offsets[a + 1] - h_offsets[a] > h_offsets[b + 1] - h_offsets[b];
  });
  std::vector<SmallProblem> small(count);
  std::vector<uint8_t> kprob((size_t)count * kmeans_problem_bytes());
  for (int32_t slot = 0; slot < count; ++slot) {
    const int32_t b = order[slot];
    const int64_t off = h_offsets[b], n = h_offsets[b + 1] - off;
    SmallProblem& q = small[slot];
    q.x = d_x + off * d;
    q.n = n;
    q.w = reinterpret_cast<double*>(p); p += al(n * n * 8);
    q.deg = reinterpret_cast<double*>(p); p += al(n * 8);
    q.y = reinterpret_cast<double*>(p); p += al(n * 8);
    q.nrm = reinterpret_cast<double*>(p); p += al(n * 8);
    q.v = d_v + off;
    q.hist = d_hist + (int64_t)b * max_iter;
    q.eps = h_eps[b];
    q.ctl = ctls + b;
    fill_kmeans_problem(kprob.data() + (size_t)slot * kmeans_problem_bytes(), d_v + off, n,
                        h_first[b], p, k, d_unif + (int64_t)b * km1, d_labels + off, ctls + b);
    p += al(kmeans_batch_scratch_bytes(n, k));
  }
  GPIC_CUDA_TRY(cudaMemcpyAsync(d_small, small.data(), sizeof(SmallProblem) * count,
                                cudaMemcpyHostToDevice, s));
  GPIC_CUDA_TRY(cudaMemcpyAsync(d_kprob, kprob.data(), kprob.size(), cudaMemcpyHostToDevice, s));
  if (km1 > 0)
    GPIC_CUDA_TRY(cudaMemcpyAsync(d_unif, h_uniforms, sizeof(double) * km1 * count,
                                  cudaMemcpyHostToDevice, s));
  const double scale = kind == GPIC_KIND_RBF ? -1.0 / (2.0 * sigma * sigma) : 0.0;
  pic_small_kernel<<<count, kSmallThreads, 0, s>>>(reinterpret_cast<const SmallProblem*>(d_small),
                                                   d, kind, scale, max_iter);
  count_launch();
  GPIC_CUDA_TRY(cudaGetLastError());
  int rc = launch_kmeans1d_batch(d_kprob, count, k, 100, 1e-12, true, s);
  if (rc) return rc;
  GPIC_CUDA_TRY(cudaMemcpyAsync(h_ctl, ctls, sizeof(gpic_ctl) * count, cudaMemcpyDeviceToHost, s));
  GPIC_CUDA_TRY(cudaStreamSynchronize(s));
  return GPIC_OK;
}

}  // extern "C"
