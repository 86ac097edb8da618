// Stage 4: 1-D k-means of the embedding on the GPU (kmeans.py:178-196).
//
//   lloyd_kernel   k-means++ seeding (kmeans.py:39-55) from host-drawn PCG64
//                  numbers, Lloyd rounds with lowest-index ties and
//                  empty-cluster reseeding (kmeans.py:58-94)
//   polish_kernel  n <= 4096 only: exact DP over the stable sorted order,
//                  earliest split on ties (kmeans.py:97-130), replacing the
//                  Lloyd labels when its WCSS is strictly lower (kmeans.py:190-193)
//   finish_kernel  contiguity check (kmeans.py:149-160, 194-195) and the
//                  canonical relabel by ascending centroid (kmeans.py:163-175)
//
// All three are single-CTA (1024 threads) kernels: the embedding is at most
// a few MB and every step is a full-vector reduction, so one SM streaming
// from L2 beats a grid-wide barrier per step. Every reduction has a fixed
// order, so labels are deterministic.
//
// Deviation, by construction unreachable: the reference's gap-split repair
// (kmeans.py:133-146) only runs when the labels are not contiguous in value
// order; both Lloyd's final nearest-centre assignment and the DP partition
// are always contiguous (1-D Voronoi cells are intervals), so the device
// path reports GPIC_E_UNSUPPORTED instead of silently diverging if that
// invariant is ever violated.
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdlib>
#include <cstdint>

#include "common.cuh"
#include "ops.h"

namespace gpic {

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxK = 64;
constexpr int kPolishLimit = 4096;  // kmeans.py:22 POLISH_LIMIT
constexpr int64_t kGridMin = 32768;  // single problems this large run on the whole GPU
constexpr int kGridMaxCtas = 256;

struct KScratch {
  int32_t* lab;     // n   Lloyd labels
  int32_t* alt;     // n   DP labels
  double* dist2;    // n
  double* unif;     // kMaxK
  int32_t* order;   // m = min(n, kPolishLimit): stable sorted order
  double* best;     // m + 1
  int32_t* split;   // (kcap + 1) x split_ld, split_ld = m + 1
  double* stats;    // small: [0] = wcss(lloyd), [1] = wcss(dp)
  double* gpart;    // grid path: per-CTA partials [kGridMaxCtas][kMaxK][4] (8-byte words)
  int64_t split_ld;
};

// One k-means problem; the batched launch (Experiment II) runs one per CTA.
struct KProblem {
  const double* v;
  int64_t n;
  int64_t first;     // k-means++ first centre (host PCG64 draw)
  KScratch s;
  int64_t* out;      // canonical labels
  gpic_ctl* ctl;
};

__host__ __device__ inline int64_t al(int64_t b) { return (b + 255) & ~int64_t(255); }

__host__ __device__ inline int64_t polish_len(int64_t n) { return n < kPolishLimit ? n : kPolishLimit; }

// grid path scratch (8-byte words): seeding chunk totals + the draw's index,
// empty-cluster candidates, and two alternating per-CTA record buffers
// [CTA][cluster][4] (alternation makes one barrier per pass enough)
constexpr int64_t kGSeed = 0, kGPick = kGridMaxCtas, kGRepair = kGridMaxCtas + 8,
                  kGRec = kGRepair + 2 * kGridMaxCtas, kGRecWords = (int64_t)kGridMaxCtas * kMaxK * 4;
__host__ __device__ constexpr int64_t grid_words() { return kGRec + 2 * kGRecWords; }

__host__ __device__ inline int64_t scratch_size(int64_t n, int kcap) {
  const int64_t m = polish_len(n);
  return al(n * 4) * 2 + al(n * 8) + al(kMaxK * 8) + al(m * 4) + al((m + 1) * 8) +
         al((int64_t)(kcap + 1) * (m + 1) * 4) + al(64 * 8) +
         (n >= kGridMin ? al(grid_words() * 8) : 0);
}

__host__ __device__ inline KScratch carve_k(void* base, int64_t n, int kcap) {
  const int64_t m = polish_len(n);
  uint8_t* p = static_cast<uint8_t*>(base);
  KScratch s;
  s.lab = reinterpret_cast<int32_t*>(p); p += al(n * 4);
  s.alt = reinterpret_cast<int32_t*>(p); p += al(n * 4);
  s.dist2 = reinterpret_cast<double*>(p); p += al(n * 8);
  s.unif = reinterpret_cast<double*>(p); p += al(kMaxK * 8);
  s.order = reinterpret_cast<int32_t*>(p); p += al(m * 4);
  s.best = reinterpret_cast<double*>(p); p += al((m + 1) * 8);
  s.split = reinterpret_cast<int32_t*>(p); p += al((int64_t)(kcap + 1) * (m + 1) * 4);
  s.stats = reinterpret_cast<double*>(p); p += al(64 * 8);
  s.gpart = n >= kGridMin ? reinterpret_cast<double*>(p) : nullptr;
  s.split_ld = m + 1;
  return s;
}

// the CTA's problem: `many[blockIdx.x]` in a batch, else the by-value one
__device__ __forceinline__ KProblem problem(const KProblem& one, const KProblem* many) {
  return many ? many[blockIdx.x] : one;
}

// ------------------------------------------------------- block primitives
constexpr int kStageRecs = 2048;
struct Shared {
  double wsum[kWarps][kMaxK];
  int wcnt[kWarps][kMaxK];
  double centers[kMaxK];
  double red_d[kWarps];
  long long red_i[kWarps];
  double scan[kThreads];
  double gstage[kGridMaxCtas];  // grid path: the CTAs' seeding totals, staged in parallel
  // grid path: the CTAs' Lloyd records (sums, counts) staged in parallel
  // when G x k fits (else read in place)
  double gsum[kStageRecs];
  long long gcnt[kStageRecs];
  int flag;
};

// argmax of val with lowest index on ties (np.argmax semantics).
__device__ long long block_argmax(double val, long long idx, Shared& sh) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, val, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > val || (ov == val && oi < idx)) { val = ov; idx = oi; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) { sh.red_d[w] = val; sh.red_i[w] = idx; }
  __syncthreads();
  double bv = sh.red_d[0];
  long long bi = sh.red_i[0];
  for (int i = 1; i < kWarps; ++i)
    if (sh.red_d[i] > bv || (sh.red_d[i] == bv && sh.red_i[i] < bi)) { bv = sh.red_d[i]; bi = sh.red_i[i]; }
  return bi;
}

__device__ long long block_min_i(long long v, Shared& sh) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh.red_i[w] = v;
  __syncthreads();
  long long b = sh.red_i[0];
  for (int i = 1; i < kWarps; ++i) b = min(b, sh.red_i[i]);
  return b;
}

// nearest centre, lowest index on ties (kmeans.py:58-60: argmin |v - c|)
__device__ __forceinline__ int nearest(double x, const double* c, int k) {
  int best = 0;
  double bd = fabs(x - c[0]);
  for (int j = 1; j < k; ++j) {
    const double d = fabs(x - c[j]);
    if (d < bd) { bd = d; best = j; }
  }
  return best;
}

__device__ void assign_all(const double* v, int64_t n, int k, int32_t* lab, Shared& sh) {
  for (int64_t i = threadIdx.x; i < n; i += kThreads) lab[i] = nearest(v[i], sh.centers, k);
  __syncthreads();
}

// per-cluster sums and counts (fixed order: per thread, then warp
// butterfly, then warps in order).
__device__ void cluster_stats(const double* v, int64_t n, int k, const int32_t* lab, Shared& sh,
                              double* sums, int64_t* cnts) {
  double ls[kMaxK];
  int lc[kMaxK];
  for (int j = 0; j < k; ++j) { ls[j] = 0.0; lc[j] = 0; }
  for (int64_t i = threadIdx.x; i < n; i += kThreads) {
    const int j = lab[i];
    ls[j] += v[i];
    lc[j] += 1;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int j = 0; j < k; ++j) {
    double s = warp_sum_f64(ls[j]);
    int c = lc[j];
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (l == 0) { sh.wsum[w][j] = s; sh.wcnt[w][j] = c; }
  }
  __syncthreads();
  if (threadIdx.x < k) {
    const int j = threadIdx.x;
    double s = 0.0;
    int64_t c = 0;
    for (int q = 0; q < kWarps; ++q) { s += sh.wsum[q][j]; c += sh.wcnt[q][j]; }
    sums[j] = s;
    cnts[j] = c;
  }
  __syncthreads();
}

// WCSS of a labelling (kmeans.py:63-69): per-cluster mean, then squared
// deviations; clusters added in id order.
__device__ double wcss(const double* v, int64_t n, int k, const int32_t* lab, Shared& sh) {
  __shared__ double sums[kMaxK];
  __shared__ int64_t cnts[kMaxK];
  __shared__ double mean[kMaxK];
  cluster_stats(v, n, k, lab, sh, sums, cnts);
  if (threadIdx.x < k) mean[threadIdx.x] = cnts[threadIdx.x] ? sums[threadIdx.x] / (double)cnts[threadIdx.x] : 0.0;
  __syncthreads();
  double ls[kMaxK];
  for (int j = 0; j < k; ++j) ls[j] = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += kThreads) {
    const int j = lab[i];
    const double d = v[i] - mean[j];
    ls[j] += d * d;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  for (int j = 0; j < k; ++j) {
    const double s = warp_sum_f64(ls[j]);
    if (l == 0) sh.wsum[w][j] = s;
  }
  __syncthreads();
  double total = 0.0;
  for (int j = 0; j < k; ++j) {
    if (!cnts[j]) continue;
    double s = 0.0;
    for (int q = 0; q < kWarps; ++q) s += sh.wsum[q][j];
    total += s;
  }
  __syncthreads();
  return total;
}

// ----------------------------------------------------------- Lloyd kernel
__global__ void __launch_bounds__(kThreads, 1)
    lloyd_kernel(KProblem one, const KProblem* __restrict__ many, int k, int max_rounds,
                 double tol) {
  const KProblem P = problem(one, many);
  if (P.ctl->status != GPIC_OK) return;  // failed upstream (batched PIC)
  const double* __restrict__ v = P.v;
  const int64_t n = P.n;
  const int64_t first_index = P.first;
  const KScratch s = P.s;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
  __shared__ double sums[kMaxK];
  __shared__ int64_t cnts[kMaxK];
  const int tid = threadIdx.x;

  // ---- k-means++ seeding (kmeans.py:39-55)
  if (tid == 0) sh.centers[0] = v[first_index];
  __syncthreads();
  for (int64_t i = tid; i < n; i += kThreads) {
    const double d = v[i] - sh.centers[0];
    s.dist2[i] = d * d;
  }
  __syncthreads();
  // contiguous chunk per thread so the running prefix follows index order
  const int64_t chunk = (n + kThreads - 1) / kThreads;
  const int64_t lo = min(n, (int64_t)tid * chunk), hi = min(n, lo + chunk);
  for (int j = 1; j < k; ++j) {
    // sequential sum of the thread's chunk, 8 loads in flight (same order)
    double part = 0.0;
    {
      int64_t i = lo;
      for (; i + 8 <= hi; i += 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = s.dist2[i + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) part += x[u];
      }
      for (; i < hi; ++i) part += s.dist2[i];
    }
    sh.scan[tid] = part;
    __syncthreads();
    // inclusive Hillis-Steele scan of the chunk totals (fixed pattern)
    for (int off = 1; off < kThreads; off <<= 1) {
      const double add = tid >= off ? sh.scan[tid - off] : 0.0;
      __syncthreads();
      sh.scan[tid] += add;
      __syncthreads();
    }
    const double total = sh.scan[kThreads - 1];
    if (!(total > 0.0)) {  // all mass on existing centres: duplicate the first
      if (tid == 0)
        for (int q = j; q < k; ++q) sh.centers[q] = sh.centers[0];
      __syncthreads();
      break;
    }
    const double r = s.unif[j - 1] * total;
    // searchsorted(cumsum(d2), r, side="right") = first i with cumsum_i > r
    double run = tid ? sh.scan[tid - 1] : 0.0;
    long long found = n;
    if (run + part > r || tid == kThreads - 1) {
      int64_t i = lo;
      for (; i + 8 <= hi && found == n; i += 8) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = s.dist2[i + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (found != n) break;
          run += x[u];
          if (run > r) found = i + u;
        }
      }
      for (; i < hi && found == n; ++i) {
        run += s.dist2[i];
        if (run > r) found = i;
      }
    }
    long long pick = block_min_i(found, sh);
    if (pick > n - 1) pick = n - 1;
    if (tid == 0) sh.centers[j] = v[pick];
    __syncthreads();
    const double cj = sh.centers[j];
    for (int64_t i = tid; i < n; i += kThreads) {
      const double d = v[i] - cj;
      s.dist2[i] = fmin(s.dist2[i], d * d);
    }
    __syncthreads();
  }

  // ---- Lloyd rounds (kmeans.py:75-94)
  assign_all(v, n, k, s.lab, sh);
  for (int round = 0; round < max_rounds; ++round) {
    cluster_stats(v, n, k, s.lab, sh, sums, cnts);
    // empty-cluster repair: reseed at the point farthest from its centre
    // (stats are refreshed after every reseed, as the reference reassigns)
    for (int j = 0; j < k; ++j) {
      if (cnts[j] != 0) continue;
      double bv = -1.0;
      long long bi = n;
      for (int64_t i = tid; i < n; i += kThreads) {
        const double d = fabs(v[i] - sh.centers[s.lab[i]]);
        if (d > bv) { bv = d; bi = i; }  // ascending i per thread: first max kept
      }
      const long long far = block_argmax(bv, bi, sh);
      if (tid == 0) sh.centers[j] = v[far];
      __syncthreads();
      assign_all(v, n, k, s.lab, sh);
      cluster_stats(v, n, k, s.lab, sh, sums, cnts);
    }
    if (tid == 0) {
      double moved = 0.0;
      for (int j = 0; j < k; ++j) {
        if (cnts[j]) {
          const double c = sums[j] / (double)cnts[j];
          moved = fmax(moved, fabs(c - sh.centers[j]));
          sh.centers[j] = c;
        }
      }
      sh.flag = moved < tol;
    }
    __syncthreads();
    assign_all(v, n, k, s.lab, sh);
    if (sh.flag) break;
    __syncthreads();
  }
  if (n > kPolishLimit) return;
  const double w = wcss(v, n, k, s.lab, sh);
  if (tid == 0) s.stats[0] = w;
}

// --------------------------------------------------- DP polish (n <= 4096)
__global__ void __launch_bounds__(kThreads, 1)
    polish_kernel(KProblem one, const KProblem* __restrict__ many, int k) {
  const KProblem P = problem(one, many);
  if (P.ctl->status != GPIC_OK || P.n > kPolishLimit) return;
  const double* __restrict__ v = P.v;
  const int64_t n = P.n;
  const KScratch s = P.s;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // [0, 4096) sort keys/values, then reused: ps (n+1), ps2 (n+1), prev (n+1)
  double* key = reinterpret_cast<double*>(smem_raw);                       // 4096
  int* idx = reinterpret_cast<int*>(key + kPolishLimit);                   // 4096
  double* ps = reinterpret_cast<double*>(idx + kPolishLimit);              // 4097
  double* ps2 = ps + (kPolishLimit + 1);                                   // 4097
  double* prev = ps2 + (kPolishLimit + 1);                                 // 4097
  const int tid = threadIdx.x;
  for (int i = tid; i < kPolishLimit; i += kThreads) {
    key[i] = i < n ? v[i] : __longlong_as_double(0x7ff0000000000000ll);
    idx[i] = i < n ? i : 0x7fffffff;
  }
  __syncthreads();
  // bitonic sort by (value, index): equals np.argsort(kind="stable")
  for (int size = 2; size <= kPolishLimit; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < kPolishLimit; i += kThreads) {
        const int jx = i ^ stride;
        if (jx > i) {
          const bool up = (i & size) == 0;
          const double ki = key[i], kj = key[jx];
          const int ii = idx[i], ij = idx[jx];
          const bool gt = ki > kj || (ki == kj && ii > ij);
          if (gt == up) { key[i] = kj; key[jx] = ki; idx[i] = ij; idx[jx] = ii; }
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < n; i += kThreads) s.order[i] = idx[i];
  // prefix sums exactly as np.cumsum (sequential, x*x rounded first)
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    ps[0] = 0.0;
    ps2[0] = 0.0;
    for (int i = 0; i < n; ++i) {
      const double x = key[i];
      a = __dadd_rn(a, x);
      b = __dadd_rn(b, __dmul_rn(x, x));
      ps[i + 1] = a;
      ps2[i + 1] = b;
    }
  }
  __syncthreads();
  // best[0][0] = 0, best[0][j>0] = inf
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  for (int j = tid; j <= n; j += kThreads) prev[j] = j == 0 ? 0.0 : inf;
  __syncthreads();
  double* cur = s.best;  // global row buffer (n + 1)
  for (int q = 1; q <= k; ++q) {
    for (int j = q + tid; j <= n; j += kThreads) {
      double bc = inf;
      int bi = q - 1;
      const double pj = ps[j], p2j = ps2[j];
      for (int i = q - 1; i < j; ++i) {
        const double sg = __dsub_rn(pj, ps[i]);
        const double c = __dsub_rn(__dadd_rn(prev[i], __dsub_rn(p2j, ps2[i])),
                                   __ddiv_rn(__dmul_rn(sg, sg), (double)(j - i)));
        if (c < bc) { bc = c; bi = i; }  // strict: earliest i on ties (np.argmin)
      }
      cur[j] = bc;
      s.split[(int64_t)q * s.split_ld + j] = bi;
    }
    __syncthreads();
    for (int j = tid; j <= n; j += kThreads) prev[j] = j < q ? inf : cur[j];
    __syncthreads();
  }
  if (tid == 0) {
    int j = (int)n;
    for (int q = k; q >= 1; --q) {
      const int i = s.split[(int64_t)q * s.split_ld + j];
      for (int p = i; p < j; ++p) s.alt[idx[p]] = q - 1;
      j = i;
    }
  }
}

// WCSS of the DP labelling, then choose (kmeans.py:190-193).
__global__ void __launch_bounds__(kThreads, 1)
    choose_kernel(KProblem one, const KProblem* __restrict__ many, int k) {
  const KProblem P = problem(one, many);
  if (P.ctl->status != GPIC_OK || P.n > kPolishLimit) return;
  const double* __restrict__ v = P.v;
  const int64_t n = P.n;
  const KScratch s = P.s;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
  const double w_dp = wcss(v, n, k, s.alt, sh);
  const bool take = w_dp < s.stats[0];
  if (threadIdx.x == 0) s.stats[1] = w_dp;
  if (take)
    for (int64_t i = threadIdx.x; i < n; i += kThreads) s.lab[i] = s.alt[i];
}

// Contiguity check + canonical relabel (kmeans.py:149-175).
__global__ void __launch_bounds__(kThreads, 1)
    finish_kernel(KProblem one, const KProblem* __restrict__ many, int k) {
  const KProblem P = problem(one, many);
  if (P.ctl->status != GPIC_OK) return;
  const double* __restrict__ v = P.v;
  const int64_t n = P.n;
  const KScratch s = P.s;
  int64_t* __restrict__ out = P.out;
  gpic_ctl* ctl = P.ctl;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
  __shared__ double sums[kMaxK];
  __shared__ int64_t cnts[kMaxK];
  __shared__ double lo_v[kMaxK], hi_v[kMaxK];
  __shared__ long long lo_i[kMaxK], hi_i[kMaxK];
  __shared__ int remap[kMaxK];
  const int tid = threadIdx.x;
  cluster_stats(v, n, k, s.lab, sh, sums, cnts);
  // lexicographic (value, index) extent of every cluster
  for (int j = 0; j < k; ++j) {
    double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
    long long mni = LLONG_MAX, mxi = -1;
    // 4 strided elements per step: labels loaded together, then values
    int64_t i = tid;
    for (; i + 3 * kThreads < n; i += 4 * kThreads) {
      int lb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) lb[u] = s.lab[i + u * kThreads];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (lb[u] != j) continue;
        const int64_t ii = i + u * kThreads;
        const double x = v[ii];
        if (x < mn || (x == mn && ii < mni)) { mn = x; mni = ii; }
        if (x > mx || (x == mx && ii > mxi)) { mx = x; mxi = ii; }
      }
    }
    for (; i < n; i += kThreads) {
      if (s.lab[i] != j) continue;
      const double x = v[i];
      if (x < mn || (x == mn && i < mni)) { mn = x; mni = i; }
      if (x > mx || (x == mx && i > mxi)) { mx = x; mxi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double a = __shfl_xor_sync(0xffffffffu, mn, o);
      const long long ai = __shfl_xor_sync(0xffffffffu, mni, o);
      if (a < mn || (a == mn && ai < mni)) { mn = a; mni = ai; }
      const double b = __shfl_xor_sync(0xffffffffu, mx, o);
      const long long bi = __shfl_xor_sync(0xffffffffu, mxi, o);
      if (b > mx || (b == mx && bi > mxi)) { mx = b; mxi = bi; }
    }
    const int w = tid >> 5, l = tid & 31;
    if (l == 0) { sh.red_d[w] = mn; sh.red_i[w] = mni; sh.wsum[w][0] = mx; sh.wcnt[w][0] = 0; }
    __shared__ long long s_mxi[kWarps];
    if (l == 0) s_mxi[w] = mxi;
    __syncthreads();
    if (tid == 0) {
      double bmn = sh.red_d[0], bmx = sh.wsum[0][0];
      long long bmni = sh.red_i[0], bmxi = s_mxi[0];
      for (int q = 1; q < kWarps; ++q) {
        if (sh.red_d[q] < bmn || (sh.red_d[q] == bmn && sh.red_i[q] < bmni)) { bmn = sh.red_d[q]; bmni = sh.red_i[q]; }
        if (sh.wsum[q][0] > bmx || (sh.wsum[q][0] == bmx && s_mxi[q] > bmxi)) { bmx = sh.wsum[q][0]; bmxi = s_mxi[q]; }
      }
      lo_v[j] = bmn; lo_i[j] = bmni; hi_v[j] = bmx; hi_i[j] = bmxi;
    }
    __syncthreads();
  }
  if (tid == 0) {
    // rank occupied clusters by centroid (stable on id), check that their
    // (value, index) extents do not interleave.
    int ids[kMaxK];
    double cen[kMaxK];
    int m = 0;
    for (int j = 0; j < k; ++j)
      if (cnts[j]) { ids[m] = j; cen[m] = sums[j] / (double)cnts[j]; ++m; }
    for (int a = 1; a < m; ++a) {  // insertion sort, stable
      const int id = ids[a];
      const double c = cen[a];
      int b = a - 1;
      while (b >= 0 && cen[b] > c) { ids[b + 1] = ids[b]; cen[b + 1] = cen[b]; --b; }
      ids[b + 1] = id;
      cen[b + 1] = c;
    }
    for (int j = 0; j < k; ++j) remap[j] = 0;
    for (int r = 0; r < m; ++r) remap[ids[r]] = r;
    // contiguity: sort extents by start, require end(prev) < start(next)
    int by[kMaxK];
    for (int r = 0; r < m; ++r) by[r] = ids[r];
    for (int a = 1; a < m; ++a) {
      const int id = by[a];
      int b = a - 1;
      while (b >= 0 && (lo_v[by[b]] > lo_v[id] || (lo_v[by[b]] == lo_v[id] && lo_i[by[b]] > lo_i[id]))) {
        by[b + 1] = by[b];
        --b;
      }
      by[b + 1] = id;
    }
    int ok = 1;
    for (int r = 1; r < m; ++r) {
      const int p = by[r - 1], q = by[r];
      if (!(hi_v[p] < lo_v[q] || (hi_v[p] == lo_v[q] && hi_i[p] < lo_i[q]))) ok = 0;
    }
    sh.flag = ok;
    if (!ok) raise_status(ctl, GPIC_E_UNSUPPORTED, 0, -1, 0.0);
  }
  __syncthreads();
  for (int64_t i = tid; i < n; i += kThreads) out[i] = remap[s.lab[i]];
}

// ------------------------------------------------ whole-GPU path (n large)
// The same algorithm as lloyd_kernel + finish_kernel, one cooperative grid
// (one 1024-thread CTA per SM): a single SM streaming v from L2 is what
// bounded the one-CTA kernels (~0.85 ms at n = 100k). CTA b owns the
// contiguous range [n b / G, n (b+1) / G); every cross-CTA reduction writes
// per-CTA partials and is combined in CTA order by every CTA identically
// after a grid barrier, so the result is deterministic for a given grid.
// Lloyd's assignment and the next round's statistics share one pass.
// Cross-CTA values are read with ld.global.cg (L2): the SMs' L1 caches are
// not coherent, and a barrier does not invalidate lines read earlier.
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(kThreads, 1)
    kmeans_grid_kernel(KProblem P, int k, int max_rounds, double tol) {
  cg::grid_group grid = cg::this_grid();
  if (P.ctl->status != GPIC_OK) return;  // uniform across the grid
  const double* __restrict__ v = P.v;
  const int64_t n = P.n;
  const KScratch s = P.s;
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const int w = tid >> 5, l = tid & 31;
  const int64_t blo = n * b / G, bhi = n * (b + 1) / G;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
  __shared__ double sums[kMaxK];
  __shared__ int64_t cnts[kMaxK];
  __shared__ double sb_tot, sb_r;
  __shared__ int sb_star;
  double* gp = s.gpart;  // [G][kMaxK][4]
  long long* gpi = reinterpret_cast<long long*>(s.gpart);

  // ---- k-means++ seeding (kmeans.py:39-55)
  if (tid == 0) sh.centers[0] = v[P.first];
  __syncthreads();
  for (int64_t i = blo + tid; i < bhi; i += kThreads) {
    const double d = v[i] - sh.centers[0];
    s.dist2[i] = d * d;
  }
  __syncthreads();
  const int64_t chunk = (bhi - blo + kThreads - 1) / kThreads;
  const int64_t lo = min(bhi, blo + (int64_t)tid * chunk), hi = min(bhi, lo + chunk);
  for (int j = 1; j < k; ++j) {
    double part = 0.0;
    for (int64_t i = lo; i < hi; ++i) part += s.dist2[i];
    sh.scan[tid] = part;
    __syncthreads();
    for (int off = 1; off < kThreads; off <<= 1) {
      const double add = tid >= off ? sh.scan[tid - off] : 0.0;
      __syncthreads();
      sh.scan[tid] += add;
      __syncthreads();
    }
    if (tid == 0) gp[kGSeed + b] = sh.scan[kThreads - 1];
    grid.sync();
    // the G totals: one L2 load per thread, then thread 0 walks them in
    // shared memory (a serial walk over L2 cost a round trip per CTA)
    if (tid < G) sh.gstage[tid] = __ldcg(gp + kGSeed + tid);
    __syncthreads();
    if (tid == 0) {
      // CTA prefix in order; the CTA holding the draw (last CTA if rounding
      // puts r past the end)
      double tot = 0.0;
      for (int q = 0; q < G; ++q) tot += sh.gstage[q];
      sb_tot = tot;
      const double r = s.unif[j - 1] * tot;
      double run = 0.0;
      int star = G - 1;
      for (int q = 0; q < G; ++q) {
        if (run + sh.gstage[q] > r) { star = q; break; }
        run += sh.gstage[q];
      }
      sb_star = star;
      sb_r = r - run;  // the draw relative to the start of CTA `star`
    }
    __syncthreads();
    if (!(sb_tot > 0.0)) {  // all mass on existing centres: duplicate the first
      if (tid == 0)
        for (int q = j; q < k; ++q) sh.centers[q] = sh.centers[0];
      __syncthreads();
      break;
    }
    if (b == sb_star) {
      const double r = sb_r;
      double run = tid ? sh.scan[tid - 1] : 0.0;
      long long found = n;
      if (run + part > r || tid == kThreads - 1) {
        for (int64_t i = lo; i < hi; ++i) {
          run += s.dist2[i];
          if (run > r) { found = i; break; }
        }
      }
      long long pick = block_min_i(found, sh);
      // rounding can keep this CTA's sequential sum at or below r although
      // its scanned total exceeds it: the crossing is then at the next
      // CTA's first index, as searchsorted would place it (clamped, as
      // kmeans.py:53 clamps to n - 1)
      if (pick > bhi - 1) pick = bhi < n ? bhi : n - 1;
      if (tid == 0) gpi[kGPick] = pick;
    }
    grid.sync();
    if (tid == 0) sh.centers[j] = v[__ldcg(gpi + kGPick)];
    __syncthreads();
    const double cj = sh.centers[j];
    for (int64_t i = blo + tid; i < bhi; i += kThreads) {
      const double d = v[i] - cj;
      s.dist2[i] = fmin(s.dist2[i], d * d);
    }
    __syncthreads();
  }

  // ---- assignment + statistics of the new assignment, one pass
  int ph = 0;  // record buffer of the next pass
  auto rec = [&](int buf, int q, int j, int slot) { return kGRec + buf * kGRecWords + (q * kMaxK + j) * 4 + slot; };
  auto assign_stats = [&]() {
    double ls[kMaxK];
    int lc[kMaxK];
    for (int j = 0; j < k; ++j) { ls[j] = 0.0; lc[j] = 0; }
    for (int64_t i = blo + tid; i < bhi; i += kThreads) {
      const double x = v[i];
      const int j = nearest(x, sh.centers, k);
      s.lab[i] = j;
      ls[j] += x;
      lc[j] += 1;
    }
    for (int j = 0; j < k; ++j) {
      const double sm = warp_sum_f64(ls[j]);
      int c = lc[j];
      for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (l == 0) { sh.wsum[w][j] = sm; sh.wcnt[w][j] = c; }
    }
    __syncthreads();
    if (tid < k) {
      double sm = 0.0;
      long long c = 0;
      for (int q = 0; q < kWarps; ++q) { sm += sh.wsum[q][tid]; c += sh.wcnt[q][tid]; }
      gp[rec(ph, b, tid, 0)] = sm;
      gpi[rec(ph, b, tid, 1)] = c;
    }
    grid.sync();
    if (G * k <= kStageRecs) {
      // every record loaded once, all in flight, then the in-order sums
      // from shared memory
      for (int e = tid; e < G * k; e += kThreads) {
        const int q = e / k, j = e - q * k;
        sh.gsum[e] = __ldcg(gp + rec(ph, q, j, 0));
        sh.gcnt[e] = __ldcg(gpi + rec(ph, q, j, 1));
      }
      __syncthreads();
      if (tid < k) {
        double sm = 0.0;
        int64_t c = 0;
        for (int q = 0; q < G; ++q) { sm += sh.gsum[q * k + tid]; c += sh.gcnt[q * k + tid]; }
        sums[tid] = sm;
        cnts[tid] = c;
      }
    } else if (tid < k) {
      double sm = 0.0;
      int64_t c = 0;
      int q = 0;
      for (; q + 8 <= G; q += 8) {  // 8 records' loads in flight, added in order
        double xs[8];
        long long xc[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          xs[u] = __ldcg(gp + rec(ph, q + u, tid, 0));
          xc[u] = __ldcg(gpi + rec(ph, q + u, tid, 1));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) { sm += xs[u]; c += xc[u]; }
      }
      for (; q < G; ++q) { sm += __ldcg(gp + rec(ph, q, tid, 0)); c += __ldcg(gpi + rec(ph, q, tid, 1)); }
      sums[tid] = sm;
      cnts[tid] = c;
    }
    ph ^= 1;
    __syncthreads();
  };

  // ---- Lloyd rounds (kmeans.py:75-94)
  assign_stats();
  for (int round = 0; round < max_rounds; ++round) {
    for (int j = 0; j < k; ++j) {
      if (cnts[j] != 0) continue;
      // empty cluster: reseed at the point farthest from its centre (first
      // index on ties), reassign, refresh the statistics
      double bv = -1.0;
      long long bi = n;
      for (int64_t i = blo + tid; i < bhi; i += kThreads) {
        const double d = fabs(v[i] - sh.centers[s.lab[i]]);
        if (d > bv) { bv = d; bi = i; }
      }
      const long long far = block_argmax(bv, bi, sh);
      if (tid == 0) {  // this CTA's candidate (value, index)
        gp[kGRepair + 2 * b] = far < bhi ? fabs(v[far] - sh.centers[s.lab[far]]) : -1.0;
        gpi[kGRepair + 2 * b + 1] = far;
      }
      grid.sync();
      if (tid == 0) {
        double best = -2.0;
        long long bidx = n;
        for (int q = 0; q < G; ++q) {
          const double d = __ldcg(gp + kGRepair + 2 * q);
          const long long ix = __ldcg(gpi + kGRepair + 2 * q + 1);
          if (d > best || (d == best && ix < bidx)) { best = d; bidx = ix; }
        }
        sh.centers[j] = v[bidx];
      }
      grid.sync();  // every CTA has read the candidates before they are reused
      assign_stats();
    }
    if (tid == 0) {
      double moved = 0.0;
      for (int j = 0; j < k; ++j) {
        if (cnts[j]) {
          const double c = sums[j] / (double)cnts[j];
          moved = fmax(moved, fabs(c - sh.centers[j]));
          sh.centers[j] = c;
        }
      }
      sh.flag = moved < tol;
    }
    __syncthreads();
    const int done = sh.flag;
    __syncthreads();
    assign_stats();
    if (done) break;
  }

  // ---- canonical labels (finish_kernel): cluster extents, contiguity, relabel
  for (int j = 0; j < k; ++j) {
    double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
    long long mni = LLONG_MAX, mxi = -1;
    for (int64_t i = blo + tid; i < bhi; i += kThreads) {
      if (s.lab[i] != j) continue;
      const double x = v[i];
      if (x < mn || (x == mn && i < mni)) { mn = x; mni = i; }
      if (x > mx || (x == mx && i > mxi)) { mx = x; mxi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double a = __shfl_xor_sync(0xffffffffu, mn, o);
      const long long ai = __shfl_xor_sync(0xffffffffu, mni, o);
      if (a < mn || (a == mn && ai < mni)) { mn = a; mni = ai; }
      const double c = __shfl_xor_sync(0xffffffffu, mx, o);
      const long long ci = __shfl_xor_sync(0xffffffffu, mxi, o);
      if (c > mx || (c == mx && ci > mxi)) { mx = c; mxi = ci; }
    }
    __shared__ double s_mn[kWarps], s_mx[kWarps];
    __shared__ long long s_mni[kWarps], s_mxi[kWarps];
    if (l == 0) { s_mn[w] = mn; s_mni[w] = mni; s_mx[w] = mx; s_mxi[w] = mxi; }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < kWarps; ++q) {
        if (s_mn[q] < mn || (s_mn[q] == mn && s_mni[q] < mni)) { mn = s_mn[q]; mni = s_mni[q]; }
        if (s_mx[q] > mx || (s_mx[q] == mx && s_mxi[q] > mxi)) { mx = s_mx[q]; mxi = s_mxi[q]; }
      }
      gp[rec(ph, b, j, 0)] = mn;  // the buffer the last pass did not use
      gpi[rec(ph, b, j, 1)] = mni;
      gp[rec(ph, b, j, 2)] = mx;
      gpi[rec(ph, b, j, 3)] = mxi;
    }
    __syncthreads();
  }
  grid.sync();
  __shared__ int remap[kMaxK];
  __shared__ double lo_v[kMaxK], hi_v[kMaxK];
  __shared__ long long lo_i[kMaxK], hi_i[kMaxK];
  if (tid < k) {  // cluster tid's extent over the CTAs' records
    const int j = tid;
    double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
    long long mni = LLONG_MAX, mxi = -1;
    for (int q = 0; q < G; ++q) {
      const double a = __ldcg(gp + rec(ph, q, j, 0)), c = __ldcg(gp + rec(ph, q, j, 2));
      const long long ai = __ldcg(gpi + rec(ph, q, j, 1)), ci = __ldcg(gpi + rec(ph, q, j, 3));
      if (a < mn || (a == mn && ai < mni)) { mn = a; mni = ai; }
      if (c > mx || (c == mx && ci > mxi)) { mx = c; mxi = ci; }
    }
    lo_v[j] = mn; lo_i[j] = mni; hi_v[j] = mx; hi_i[j] = mxi;
  }
  __syncthreads();
  if (tid == 0) {
    int ids[kMaxK];
    double cen[kMaxK];
    int m = 0;
    for (int j = 0; j < k; ++j)
      if (cnts[j]) { ids[m] = j; cen[m] = sums[j] / (double)cnts[j]; ++m; }
    for (int a = 1; a < m; ++a) {  // insertion sort, stable
      const int id = ids[a];
      const double c = cen[a];
      int q = a - 1;
      while (q >= 0 && cen[q] > c) { ids[q + 1] = ids[q]; cen[q + 1] = cen[q]; --q; }
      ids[q + 1] = id;
      cen[q + 1] = c;
    }
    for (int j = 0; j < k; ++j) remap[j] = 0;
    for (int r = 0; r < m; ++r) remap[ids[r]] = r;
    int by[kMaxK];
    for (int r = 0; r < m; ++r) by[r] = ids[r];
    for (int a = 1; a < m; ++a) {
      const int id = by[a];
      int q = a - 1;
      while (q >= 0 && (lo_v[by[q]] > lo_v[id] || (lo_v[by[q]] == lo_v[id] && lo_i[by[q]] > lo_i[id]))) {
        by[q + 1] = by[q];
        --q;
      }
      by[q + 1] = id;
    }
    int ok = 1;
    for (int r = 1; r < m; ++r) {
      const int p = by[r - 1], q = by[r];
      if (!(hi_v[p] < lo_v[q] || (hi_v[p] == lo_v[q] && hi_i[p] < lo_i[q]))) ok = 0;
    }
    if (!ok && b == 0) raise_status(P.ctl, GPIC_E_UNSUPPORTED, 0, -1, 0.0);
  }
  __syncthreads();
  for (int64_t i = blo + tid; i < bhi; i += kThreads) P.out[i] = remap[s.lab[i]];
}

int g_grid_ctas = 0;

int set_kmeans_attributes() {
  static bool done = false;
  if (done) return GPIC_OK;
  const int shm = (int)sizeof(Shared);
  const int pshm = kPolishLimit * (8 + 4) + 3 * (kPolishLimit + 1) * 8;
  GPIC_CUDA_TRY(cudaFuncSetAttribute(lloyd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
  GPIC_CUDA_TRY(cudaFuncSetAttribute(choose_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
  GPIC_CUDA_TRY(cudaFuncSetAttribute(finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
  GPIC_CUDA_TRY(cudaFuncSetAttribute(polish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pshm));
  GPIC_CUDA_TRY(cudaFuncSetAttribute(kmeans_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
  int dev = 0, sms = 0, per_sm = 0, coop = 0;
  GPIC_CUDA_TRY(cudaGetDevice(&dev));
  GPIC_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  GPIC_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  GPIC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kmeans_grid_kernel, kThreads, shm));
  // 64 CTAs: the grid barriers (2 per k-means++ centre, 1-2 per Lloyd round)
  // dominate, and they are cheaper on fewer CTAs while 64 still stream the
  // data fast enough (measured, scripts/km_time.py: n = 100k, k = 10 0.38 ms
  // vs 0.52 ms on all 148 SMs; n = 1M, k = 50 4.4 vs 4.6 ms)
  constexpr int kGridDefault = 64;
  const int cap = kGridDefault < kGridMaxCtas ? kGridDefault : kGridMaxCtas;
  g_grid_ctas = coop && per_sm > 0 ? (sms < cap ? sms : cap) : 0;
  if (const char* e = getenv("GPIC_KMEANS_CTAS"))  // measurement: grid size of the whole-GPU path
    if (g_grid_ctas > 0 && atoi(e) > 0)
      g_grid_ctas = atoi(e) < (sms < kGridMaxCtas ? sms : kGridMaxCtas) ? atoi(e)
                                                                      : (sms < kGridMaxCtas ? sms : kGridMaxCtas);
  done = true;
  return GPIC_OK;
}

// the four stages over `grid` problems (one = by-value problem when many == null)
int launch_stages(const KProblem& one, const KProblem* many, int grid, int k, int max_rounds,
                  double tol, bool polish, cudaStream_t st) {
  int rc = set_kmeans_attributes();
  if (rc) return rc;
  const size_t shm = sizeof(Shared);
  const int pshm = kPolishLimit * (8 + 4) + 3 * (kPolishLimit + 1) * 8;
  lloyd_kernel<<<grid, kThreads, shm, st>>>(one, many, k, max_rounds, tol);
  count_launch();
  if (polish) {
    polish_kernel<<<grid, kThreads, pshm, st>>>(one, many, k);
    choose_kernel<<<grid, kThreads, shm, st>>>(one, many, k);
    count_launch(2);
  }
  finish_kernel<<<grid, kThreads, shm, st>>>(one, many, k);
  count_launch();
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

}  // namespace

int64_t kmeans_scratch_bytes(int64_t n, int32_t k) {
  const int64_t small = scratch_size(n, kMaxK);
  const int64_t big = kmeans_big_scratch_bytes(n, k);  // 64 < k: kmeans_big.cu
  return big > small ? big : small;
}

int launch_kmeans1d(const double* v, int64_t n, int32_t k, int64_t first_index,
                    const double* h_uniforms, int32_t max_rounds, double tol, int64_t* labels,
                    void* scratch, gpic_ctl* ctl, cudaStream_t st) {
  if (k > n) return fail(GPIC_E_K_TOO_LARGE, "k exceeds the number of points");
  if (k < 2) return fail(GPIC_E_INVALID, "k must be at least 2");
  if (first_index < 0 || first_index >= n) return fail(GPIC_E_INVALID, "first_index out of range");
  // many clusters: the sorted-domain variant (kmeans_big.cu); GPIC_KMEANS_SORTED=1
  // routes every k there (measurement)
  const char* srt = getenv("GPIC_KMEANS_SORTED");
  if (k > kMaxK || (srt != nullptr && atoi(srt) != 0))
    return launch_kmeans1d_big(v, n, k, first_index, h_uniforms, max_rounds, tol, labels, scratch,
                               ctl, st);
  KProblem p;
  p.v = v;
  p.n = n;
  p.first = first_index;
  p.s = carve_k(scratch, n, kMaxK);
  p.out = labels;
  p.ctl = ctl;
  GPIC_CUDA_TRY(cudaMemcpyAsync(p.s.unif, h_uniforms, sizeof(double) * (k - 1),
                                cudaMemcpyHostToDevice, st));
  if (n >= kGridMin && getenv("GPIC_KMEANS_ONE_CTA") == nullptr) {
    int rc = set_kmeans_attributes();
    if (rc) return rc;
    if (g_grid_ctas > 0) {
      void* args[] = {&p, &k, &max_rounds, &tol};
      GPIC_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kmeans_grid_kernel, g_grid_ctas,
                                                kThreads, args, sizeof(Shared), st));
      count_launch();
      return GPIC_OK;
    }
  }
  return launch_stages(p, nullptr, 1, k, max_rounds, tol, n <= kPolishLimit, st);
}

// ---------------------------------------------------------------- batched
int64_t kmeans_batch_scratch_bytes(int64_t n, int32_t k) { return scratch_size(n, k); }

int64_t kmeans_problem_bytes() { return (int64_t)sizeof(KProblem); }

int fill_kmeans_problem(void* host_slot, const double* v, int64_t n, int64_t first, void* scratch,
                        int32_t k, const double* d_unif, int64_t* labels, gpic_ctl* ctl) {
  KProblem p;
  p.v = v;
  p.n = n;
  p.first = first;
  p.s = carve_k(scratch, n, k);
  p.s.unif = const_cast<double*>(d_unif);
  p.out = labels;
  p.ctl = ctl;
  *static_cast<KProblem*>(host_slot) = p;
  return GPIC_OK;
}

int launch_kmeans1d_batch(const void* d_problems, int32_t count, int32_t k, int32_t max_rounds,
                          double tol, bool polish, cudaStream_t st) {
  if (k < 2 || k > kMaxK) return fail(GPIC_E_UNSUPPORTED, "k must lie in [2, 64] on the GPU path");
  KProblem none{};
  return launch_stages(none, static_cast<const KProblem*>(d_problems), count, k, max_rounds, tol,
                       polish, st);
}

}  // namespace gpic
