// Stage 4 for many clusters (64 < k <= 4096): 1-D k-means in the sorted domain.
//
// Same algorithm and semantics as kmeans.cu (kmeans.py:39-196): seeded
// k-means++ (host PCG64 draws), Lloyd rounds with lowest-index ties and
// empty-cluster reseeding, the exact DP polish for n <= 4096, the canonical
// relabel by ascending centroid. kmeans.cu keeps one register / shared slot
// per cluster (k <= 64); here the per-round work is moved onto the values
// sorted once (stable, by value then index):
//
//   * 1-D nearest-centre cells are intervals, so with the centres ordered by
//     (value, index) every cluster is one contiguous run of the sorted
//     values. The boundary between two neighbouring owners a (c_a) < b (c_b)
//     is the first sorted value x with |x - c_b| < |x - c_a| (or equal and
//     b's index lower) — a monotone predicate, found by binary search.
//     Duplicate centres: the lowest index owns the run, the others are empty
//     (argmin's lowest-index tie rule, kmeans.py:58-60).
//   * cluster sums are differences of one fp64 prefix sum of the sorted
//     values, counts are run lengths: O(k log n) per round instead of O(n k).
//   * the empty-cluster reseed's farthest point (np.argmax of |v - c_label|,
//     lowest index on ties) is one of the two ends of a run: the first
//     element, or the first element of the last value group.
//
// Cluster means therefore round differently from the reference's
// sel.mean() (prefix differences instead of numpy's pairwise sum); labels
// agree except for points within an ulp of a cell boundary.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cfloat>
#include <cstdint>

#include "common.cuh"
#include "ops.h"

namespace gpic {

namespace {

constexpr int kT = 1024;
constexpr int kBigMaxK = 4096;
constexpr int kPolish = 4096;  // kmeans.py:22 POLISH_LIMIT

struct Big {
  const double* v;   // n values (original order)
  int64_t n;
  int k;
  int64_t first;     // k-means++ first centre
  const double* unif;  // k - 1 draws
  double* dist2;     // n
  double* sv;        // n sorted values
  int32_t* perm;     // n original index of each sorted position
  int32_t* iota;     // n
  double* keys;      // n sort keys (v with -0.0 -> +0.0)
  double* ps;        // n + 1 prefix sums of sv
  double* centers;   // k
  int32_t* lab;      // n labels by sorted position (Lloyd)
  int32_t* alt;      // n labels by sorted position (DP)
  int64_t* run_lo;   // k: run of cluster j in sorted order [run_lo, run_hi)
  int64_t* run_hi;
  double* stats;     // [0] wcss Lloyd, [1] wcss DP
  int32_t* split;    // (k + 1) x (m + 1), n <= kPolish
  double* best;      // m + 1
  int64_t* out;      // canonical labels (original order)
  gpic_ctl* ctl;
};

__device__ long long block_min_ll(long long v, long long* red) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  long long b = red[0];
  for (int i = 1; i < kT / 32; ++i) b = min(b, red[i]);
  __syncthreads();
  return b;
}

// k-means++ seeding (kmeans.py:39-55), one CTA: contiguous chunk per
// thread so the running prefix follows index order; searchsorted side=right
__global__ void __launch_bounds__(kT, 1) big_seed_kernel(Big B) {
  __shared__ double scan[kT];
  __shared__ long long red[kT / 32];
  if (B.ctl->status != GPIC_OK) return;
  const int tid = threadIdx.x;
  const int64_t n = B.n;
  const double* v = B.v;
  double c0 = v[B.first];
  if (tid == 0) B.centers[0] = c0;
  for (int64_t i = tid; i < n; i += kT) {
    const double d = v[i] - c0;
    B.dist2[i] = d * d;
  }
  __syncthreads();
  const int64_t chunk = (n + kT - 1) / kT;
  const int64_t lo = min(n, (int64_t)tid * chunk), hi = min(n, lo + chunk);
  for (int j = 1; j < B.k; ++j) {
    double part = 0.0;
    for (int64_t i = lo; i < hi; ++i) part += B.dist2[i];
    scan[tid] = part;
    __syncthreads();
    for (int off = 1; off < kT; off <<= 1) {
      const double add = tid >= off ? scan[tid - off] : 0.0;
      __syncthreads();
      scan[tid] += add;
      __syncthreads();
    }
    const double total = scan[kT - 1];
    if (!(total > 0.0)) {  // all mass on existing centres: duplicate the first
      for (int q = j + tid; q < B.k; q += kT) B.centers[q] = c0;
      break;
    }
    const double r = B.unif[j - 1] * total;
    double run = tid ? scan[tid - 1] : 0.0;
    long long found = n;
    if (run + part > r || tid == kT - 1) {
      for (int64_t i = lo; i < hi; ++i) {
        run += B.dist2[i];
        if (run > r) { found = i; break; }
      }
    }
    long long pick = block_min_ll(found, red);
    if (pick > n - 1) pick = n - 1;
    const double cj = v[pick];
    if (tid == 0) B.centers[j] = cj;
    for (int64_t i = tid; i < n; i += kT) {
      const double d = v[i] - cj;
      B.dist2[i] = fmin(B.dist2[i], d * d);
    }
    __syncthreads();
  }
}

__global__ void big_keys_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ keys,
                                int32_t* __restrict__ iota) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    keys[i] = v[i] + 0.0;  // -0.0 sorts with +0.0 (np.argsort compares them equal)
    iota[i] = (int32_t)i;
  }
}

// shared state of the Lloyd CTA
struct LSh {
  double cval[kBigMaxK];   // centres in (value, index) order
  int32_t cidx[kBigMaxK];
  double red_d[kT / 32];
  long long red_i[kT / 32];
  int flag;
};

// point at sorted position p goes to b (value cb, index ib) rather than a
__device__ __forceinline__ bool to_b(double x, double ca, int ia, double cb, int ib) {
  const double da = fabs(x - ca), db = fabs(x - cb);
  return db < da || (db == da && ib < ia);
}

// order the centres by (value, index) (bitonic over the next power of two)
__device__ void sort_centres(const double* centers, int k, LSh& sh) {
  int m = 1;
  while (m < k) m <<= 1;
  for (int i = threadIdx.x; i < m; i += kT) {
    sh.cval[i] = i < k ? centers[i] : DBL_MAX;
    sh.cidx[i] = i < k ? i : 0x7fffffff;
  }
  __syncthreads();
  for (int size = 2; size <= m; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < m; i += kT) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const double a = sh.cval[i], b = sh.cval[j];
          const int ia = sh.cidx[i], ib = sh.cidx[j];
          const bool gt = a > b || (a == b && ia > ib);
          if (gt == up) { sh.cval[i] = b; sh.cval[j] = a; sh.cidx[i] = ib; sh.cidx[j] = ia; }
        }
      }
      __syncthreads();
    }
}

// runs of every cluster for the current centres (empty: lo == hi)
__device__ void assign_runs(const Big& B, LSh& sh) {
  sort_centres(B.centers, B.k, sh);
  const int k = B.k;
  const int64_t n = B.n;
  for (int r = threadIdx.x; r < k; r += kT) {
    const int id = sh.cidx[r];
    const double c = sh.cval[r];
    if (r > 0 && sh.cval[r - 1] == c) {  // duplicate: the lowest index owns the run
      B.run_lo[id] = 0;
      B.run_hi[id] = 0;
      continue;
    }
    // previous / next owner (distinct values)
    int pr = r - 1;
    while (pr > 0 && sh.cval[pr - 1] == sh.cval[pr]) --pr;
    int nx = r + 1;
    while (nx < k && sh.cval[nx] == c) ++nx;
    int64_t lo = 0, hi = n;
    if (r > 0) {  // first position that prefers this centre over the previous owner
      const double ca = sh.cval[pr];
      const int ia = sh.cidx[pr];
      int64_t a = 0, b = n;
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (to_b(B.sv[mid], ca, ia, c, id)) b = mid; else a = mid + 1;
      }
      lo = a;
    }
    if (nx < k) {  // first position that prefers the next owner
      const double cb = sh.cval[nx];
      const int ib = sh.cidx[nx];
      int64_t a = 0, b = n;
      while (a < b) {
        const int64_t mid = (a + b) >> 1;
        if (to_b(B.sv[mid], c, id, cb, ib)) b = mid; else a = mid + 1;
      }
      hi = a;
    }
    B.run_lo[id] = lo;
    B.run_hi[id] = hi < lo ? lo : hi;
  }
  __syncthreads();
}

// farthest point from its centre (np.argmax: lowest index on ties): per
// run, the first element or the first element of the last value group
__device__ long long farthest(const Big& B, LSh& sh) {
  double bv = -1.0;
  long long bi = LLONG_MAX;
  for (int j = threadIdx.x; j < B.k; j += kT) {
    const int64_t lo = B.run_lo[j], hi = B.run_hi[j];
    if (lo >= hi) continue;
    const double c = B.centers[j];
    const double d0 = fabs(B.sv[lo] - c);
    const long long i0 = B.perm[lo];
    if (d0 > bv || (d0 == bv && i0 < bi)) { bv = d0; bi = i0; }
    const double xl = B.sv[hi - 1];
    int64_t a = lo, b = hi - 1;  // first position of the last value group
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (B.sv[mid] < xl) a = mid + 1; else b = mid;
    }
    // the lowest original index of that group (stable sort: its first)
    const double d1 = fabs(xl - c);
    const long long i1 = B.perm[a];
    if (d1 > bv || (d1 == bv && i1 < bi)) { bv = d1; bi = i1; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) { sh.red_d[w] = bv; sh.red_i[w] = bi; }
  __syncthreads();
  double v = sh.red_d[0];
  long long i = sh.red_i[0];
  for (int q = 1; q < kT / 32; ++q)
    if (sh.red_d[q] > v || (sh.red_d[q] == v && sh.red_i[q] < i)) { v = sh.red_d[q]; i = sh.red_i[q]; }
  __syncthreads();
  return i;
}

// Lloyd rounds (kmeans.py:72-94) on the sorted values, one CTA
__global__ void __launch_bounds__(kT, 1) big_lloyd_kernel(Big B, int max_rounds, double tol) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  LSh& sh = *reinterpret_cast<LSh*>(smem_raw);
  if (B.ctl->status != GPIC_OK) return;
  const int k = B.k;
  assign_runs(B, sh);
  for (int round = 0; round < max_rounds; ++round) {
    for (int j = 0; j < k; ++j) {  // empty-cluster repair, in id order
      if (B.run_lo[j] < B.run_hi[j]) continue;
      const long long far = farthest(B, sh);
      if (threadIdx.x == 0) B.centers[j] = B.v[far];
      __syncthreads();
      assign_runs(B, sh);
    }
    // new centres, and how far they moved
    double moved = 0.0;
    for (int j = threadIdx.x; j < k; j += kT) {
      const int64_t lo = B.run_lo[j], hi = B.run_hi[j];
      if (lo < hi) {
        const double c = (B.ps[hi] - B.ps[lo]) / (double)(hi - lo);
        moved = fmax(moved, fabs(c - B.centers[j]));
        B.centers[j] = c;
      }
    }
    moved = warp_max_f64(moved);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sh.red_d[w] = moved;
    __syncthreads();
    if (threadIdx.x == 0) {
      double m = sh.red_d[0];
      for (int q = 1; q < kT / 32; ++q) m = fmax(m, sh.red_d[q]);
      sh.flag = m < tol;
    }
    __syncthreads();
    assign_runs(B, sh);
    if (sh.flag) break;
    __syncthreads();
  }
  // labels by sorted position
  for (int j = threadIdx.x; j < k; j += kT)
    for (int64_t p = B.run_lo[j]; p < B.run_hi[j]; ++p) B.lab[p] = j;
}

// WCSS of a labelling given by sorted position (kmeans.py:63-69): every
// cluster is one run, mean then squared deviations, clusters in id order
__device__ double runs_wcss(const Big& B, const int32_t* lab, double* tmp, LSh& sh) {
  // per cluster: first / last position of its run (runs are contiguous)
  const int64_t n = B.n;
  for (int j = threadIdx.x; j < B.k; j += kT) { B.run_lo[j] = 0; B.run_hi[j] = 0; }
  __syncthreads();
  for (int64_t p = threadIdx.x; p < n; p += kT) {
    const int j = lab[p];
    if (p == 0 || lab[p - 1] != j) B.run_lo[j] = p;
    if (p == n - 1 || lab[p + 1] != j) B.run_hi[j] = p + 1;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < B.k; j += kT) {
    const int64_t lo = B.run_lo[j], hi = B.run_hi[j];
    double s = 0.0;
    if (lo < hi) {
      double m = 0.0;
      for (int64_t p = lo; p < hi; ++p) m += B.sv[p];
      m /= (double)(hi - lo);
      for (int64_t p = lo; p < hi; ++p) {
        const double d = B.sv[p] - m;
        s += d * d;
      }
    }
    tmp[j] = s;
  }
  __syncthreads();
  double total = 0.0;
  if (threadIdx.x == 0)
    for (int j = 0; j < B.k; ++j) total += tmp[j];
  (void)sh;
  return total;
}

// DP polish (kmeans.py:97-130, 190-193) over the sorted values (n <= 4096):
// optimal contiguous partition, earliest split on ties; replaces the Lloyd
// labels when its WCSS is strictly lower
__global__ void __launch_bounds__(kT, 1) big_polish_kernel(Big B) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  LSh& sh = *reinterpret_cast<LSh*>(smem_raw);
  double* ps2 = B.dist2;  // n + 1 (the seeding's scratch is free now)
  if (B.ctl->status != GPIC_OK || B.n > kPolish) return;
  const int64_t n = B.n;
  const int k = B.k;
  if (threadIdx.x == 0) {  // prefix sums exactly as np.cumsum (sequential, x*x rounded first)
    double a = 0.0, b = 0.0;
    B.ps[0] = 0.0;
    ps2[0] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      a = __dadd_rn(a, B.sv[i]);
      b = __dadd_rn(b, __dmul_rn(B.sv[i], B.sv[i]));
      B.ps[i + 1] = a;
      ps2[i + 1] = b;
    }
  }
  __syncthreads();
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const int64_t ld = n + 1;
  double* prev = B.best;             // n + 1
  double* cur = B.best + (n + 1);    // n + 1
  for (int64_t j = threadIdx.x; j <= n; j += kT) prev[j] = j == 0 ? 0.0 : inf;
  __syncthreads();
  for (int q = 1; q <= k; ++q) {
    for (int64_t j = q + threadIdx.x; j <= n; j += kT) {
      double bc = inf;
      int bi = q - 1;
      const double pj = B.ps[j], p2j = ps2[j];
      for (int64_t i = q - 1; i < j; ++i) {
        const double sg = __dsub_rn(pj, B.ps[i]);
        const double c = __dsub_rn(__dadd_rn(prev[i], __dsub_rn(p2j, ps2[i])),
                                   __ddiv_rn(__dmul_rn(sg, sg), (double)(j - i)));
        if (c < bc) { bc = c; bi = (int)i; }
      }
      cur[j] = bc;
      B.split[(int64_t)q * ld + j] = bi;
    }
    __syncthreads();
    for (int64_t j = threadIdx.x; j <= n; j += kT) prev[j] = j < q ? inf : cur[j];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int64_t j = n;
    for (int q = k; q >= 1; --q) {
      const int64_t i = B.split[(int64_t)q * ld + j];
      for (int64_t p = i; p < j; ++p) B.alt[p] = q - 1;
      j = i;
    }
  }
  __syncthreads();
  double* tmp = cur;  // k doubles (n + 1 >= k)
  const double w_l = runs_wcss(B, B.lab, tmp, sh);
  __syncthreads();
  const double w_d = runs_wcss(B, B.alt, tmp, sh);
  __shared__ int take;
  if (threadIdx.x == 0) {
    B.stats[0] = w_l;
    B.stats[1] = w_d;
    take = w_d < w_l;
  }
  __syncthreads();
  if (take)
    for (int64_t p = threadIdx.x; p < n; p += kT) B.lab[p] = B.alt[p];
}

// canonical relabel (kmeans.py:163-175): occupied clusters ranked by
// centroid (stable on id), written back in original order
__global__ void __launch_bounds__(kT, 1) big_finish_kernel(Big B) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  LSh& sh = *reinterpret_cast<LSh*>(smem_raw);
  if (B.ctl->status != GPIC_OK) return;
  const int64_t n = B.n;
  const int k = B.k;
  for (int j = threadIdx.x; j < k; j += kT) { B.run_lo[j] = 0; B.run_hi[j] = 0; }
  __syncthreads();
  for (int64_t p = threadIdx.x; p < n; p += kT) {
    const int j = B.lab[p];
    if (p == 0 || B.lab[p - 1] != j) B.run_lo[j] = p;
    if (p == n - 1 || B.lab[p + 1] != j) B.run_hi[j] = p + 1;
  }
  __syncthreads();
  // centroids (empty clusters: +inf, ranked last and never used)
  for (int j = threadIdx.x; j < k; j += kT) {
    const int64_t lo = B.run_lo[j], hi = B.run_hi[j];
    double m = DBL_MAX;
    if (lo < hi) {
      m = 0.0;
      for (int64_t p = lo; p < hi; ++p) m += B.sv[p];
      m /= (double)(hi - lo);
    }
    B.centers[j] = m;
  }
  __syncthreads();
  sort_centres(B.centers, k, sh);  // (centroid, id) order = the canonical ranks
  for (int r = threadIdx.x; r < k; r += kT) B.dist2[sh.cidx[r]] = (double)r;  // id -> rank
  __syncthreads();
  for (int64_t p = threadIdx.x; p < n; p += kT) B.out[B.perm[p]] = (int64_t)B.dist2[B.lab[p]];
}

int64_t al(int64_t b) { return (b + 255) & ~int64_t(255); }

size_t cub_bytes(int64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const double*)nullptr, (double*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const double*)nullptr, (double*)nullptr, (int)n + 1);
  return a > b ? a : b;
}

}  // namespace

int kmeans_big_max_k() { return kBigMaxK; }

int64_t kmeans_big_scratch_bytes(int64_t n, int32_t k) {
  const int64_t m = n < kPolish ? n : kPolish;
  return al((n + 1) * 8) * 4 + al(n * 4) * 4 + al((int64_t)k * 8) * 4 + al(64) +
         (n <= kPolish ? al((int64_t)(k + 1) * (m + 1) * 4) + al(2 * (m + 1) * 8) : 0) +
         al((int64_t)cub_bytes(n));
}

int launch_kmeans1d_big(const double* v, int64_t n, int32_t k, int64_t first_index,
                        const double* h_uniforms, int32_t max_rounds, double tol, int64_t* labels,
                        void* scratch, gpic_ctl* ctl, cudaStream_t st) {
  if (k > kBigMaxK) return fail(GPIC_E_UNSUPPORTED, "k must be at most 4096 on the GPU path");
  const int64_t m = n < kPolish ? n : kPolish;
  uint8_t* p = static_cast<uint8_t*>(scratch);
  auto take = [&](int64_t b) { uint8_t* q = p; p += al(b); return q; };
  Big B;
  B.v = v;
  B.n = n;
  B.k = k;
  B.first = first_index;
  B.dist2 = reinterpret_cast<double*>(take((n + 1) * 8));
  B.sv = reinterpret_cast<double*>(take((n + 1) * 8));
  B.keys = reinterpret_cast<double*>(take((n + 1) * 8));
  B.ps = reinterpret_cast<double*>(take((n + 1) * 8));
  B.perm = reinterpret_cast<int32_t*>(take(n * 4));
  B.iota = reinterpret_cast<int32_t*>(take(n * 4));
  B.lab = reinterpret_cast<int32_t*>(take(n * 4));
  B.alt = reinterpret_cast<int32_t*>(take(n * 4));
  double* unif = reinterpret_cast<double*>(take((int64_t)k * 8));
  B.unif = unif;
  B.centers = reinterpret_cast<double*>(take((int64_t)k * 8));
  B.run_lo = reinterpret_cast<int64_t*>(take((int64_t)k * 8));
  B.run_hi = reinterpret_cast<int64_t*>(take((int64_t)k * 8));
  B.stats = reinterpret_cast<double*>(take(64));
  B.split = nullptr;
  B.best = nullptr;
  if (n <= kPolish) {
    B.split = reinterpret_cast<int32_t*>(take((int64_t)(k + 1) * (m + 1) * 4));
    B.best = reinterpret_cast<double*>(take(2 * (m + 1) * 8));
  }
  void* tmp = p;
  size_t tmp_bytes = cub_bytes(n);
  B.out = labels;
  B.ctl = ctl;
  GPIC_CUDA_TRY(cudaMemcpyAsync(unif, h_uniforms, sizeof(double) * (k - 1), cudaMemcpyHostToDevice, st));
  static bool attr = false;
  if (!attr) {
    const int shm = (int)sizeof(LSh);
    GPIC_CUDA_TRY(cudaFuncSetAttribute(big_lloyd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
    GPIC_CUDA_TRY(cudaFuncSetAttribute(big_polish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
    GPIC_CUDA_TRY(cudaFuncSetAttribute(big_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
    attr = true;
  }
  big_seed_kernel<<<1, kT, 0, st>>>(B);
  big_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(v, n, B.keys, B.iota);
  GPIC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, B.keys, B.sv, B.iota, B.perm,
                                                (int)n, 0, 64, st));
  // ps[0] = 0, ps[i + 1] = sv[0] + ... + sv[i] (sv[n] is scratch: set 0)
  GPIC_CUDA_TRY(cudaMemsetAsync(B.sv + n, 0, 8, st));
  tmp_bytes = cub_bytes(n);
  GPIC_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, B.sv, B.ps, (int)n + 1, st));
  big_lloyd_kernel<<<1, kT, sizeof(LSh), st>>>(B, max_rounds, tol);
  if (n <= kPolish) big_polish_kernel<<<1, kT, sizeof(LSh), st>>>(B);
  big_finish_kernel<<<1, kT, sizeof(LSh), st>>>(B);
  count_launch(n <= kPolish ? 7 : 6);
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

}  // namespace gpic
