// Locality order: block sparsity and tile pruning for inputs in any order.
//
// Tile pruning (prune.cu) and the zero boxes (sparse.cu) need rows that are
// close in space to be close in index — true for data stored cluster by
// cluster, false for shuffled data, where every 512-row block holds every
// cluster and nothing can be pruned (the full 20 GB triangle at config 3).
// When the order looks random (order_metric below), gpic_cluster permutes
// the points first:
//
//   * m = n / 256 seeds (points at evenly spaced indices) and m2 <= 96
//     super-seeds (every (m / m2)-th seed); each seed takes its nearest
//     super-seed, each point its nearest seed (fp32 SIMT GEMM, argmin with
//     the lowest index on ties): Voronoi cells of ~256 points, cells of one
//     super-seed region adjacent;
//   * the points are stably sorted by (super-seed, seed) (CUB radix sort of
//     the cell rank, index order inside a cell) — perm[p] = original index
//     of position p — and X is gathered into that order.
//
// PIC is permutation-equivariant: the run proceeds on the permuted points
// and v is scattered back to the original order before the k-means, whose
// seeding therefore sees the reference's index order. The embedding differs
// from the unpermuted run only by summation order (fp32 / fp64 rounding),
// labels are the same on separated data (tests/test_gpu_locality.py).
#include <cub/device/device_radix_sort.cuh>

#include <cfloat>

#include "common.cuh"
#include "ops.h"

namespace gpic {

namespace {

constexpr int kRows = 128;   // points per CTA of the assignment
constexpr int kSeeds = 64;   // seeds per smem chunk
constexpr int kK = 32;       // features per smem stage
constexpr int kCell = 256;   // points per seed (target cell size)
constexpr int kMaxSuper = 96;  // the chain kernel keeps a kMaxSuper^2 distance matrix in static smem

// order metric: sum over sampled i of |x_i - x_(i+1)|^2 and of |x_i|^2
// (centred rows): about 1/2 of the ratio for random order, near 0 when
// neighbours in index are neighbours in space
__global__ void order_metric_kernel(const float* __restrict__ xc, int64_t n, int32_t dp,
                                    int64_t stride, double* __restrict__ out) {
  __shared__ double red[2][32];
  double a = 0.0, b = 0.0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t i = ((int64_t)blockIdx.x * (blockDim.x >> 5) + w) * stride; i + 1 < n;
       i += (int64_t)gridDim.x * (blockDim.x >> 5) * stride) {
    for (int f = lane; f < dp; f += 32) {
      const float u = xc[i * dp + f], v = xc[(i + 1) * dp + f];
      a += (double)(u - v) * (double)(u - v);
      b += (double)u * (double)u;
    }
  }
  a = warp_sum_f64(a);
  b = warp_sum_f64(b);
  if (lane == 0) {
    red[0][w] = a;
    red[1][w] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      sa += red[0][q];
      sb += red[1][q];
    }
    atomicAdd(out, sa);  // a heuristic's input: fp64 atomics' order is irrelevant
    atomicAdd(out + 1, sb);
  }
}

// |s_c|^2 of the seeds (rows seed_idx[c] of x)
__global__ void seed_norm_kernel(const float* __restrict__ x, int32_t dp,
                                 const int32_t* __restrict__ seed_idx, int64_t m,
                                 float* __restrict__ snorm) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= m) return;
  const float* s = x + (int64_t)seed_idx[c] * dp;
  float t = 0.f;
  for (int f = 0; f < dp; ++f) t = fmaf(s[f], s[f], t);
  snorm[c] = t;
}

// cell[i] = argmin_c (|s_c|^2 - 2 x_i . s_c) over the m seeds, lowest c on
// ties; CTA = 128 points, seeds streamed through smem 64 at a time.
// Thread (tr, tc): points tr * 8 .. + 8, seeds tc * 4 .. + 4 of a chunk.
__global__ void __launch_bounds__(256)
    nearest_seed_kernel(const float* __restrict__ x, int64_t n, int32_t dp,
                        const float* __restrict__ sx, const int32_t* __restrict__ seed_idx,
                        const float* __restrict__ snorm, int64_t m, int32_t* __restrict__ cell) {
  __shared__ float px[kK][kRows + 4];
  __shared__ float ps[kK][kSeeds + 4];
  __shared__ float bd[16][kRows];
  __shared__ int bi[16][kRows];
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int tid = threadIdx.x, tr = tid >> 4, tcl = tid & 15;
  float best[8];
  int besti[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    best[a] = FLT_MAX;
    besti[a] = 0x7fffffff;
  }
  for (int64_t c0 = 0; c0 < m; c0 += kSeeds) {
    float acc[8][4];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
    for (int k0 = 0; k0 < dp; k0 += kK) {
      __syncthreads();
      for (int e = tid; e < kRows * kK; e += 256) {
        const int r = e / kK, f = e % kK;
        const int64_t row = r0 + r;
        px[f][r] = (row < n && k0 + f < dp) ? x[row * dp + k0 + f] : 0.f;
      }
      for (int e = tid; e < kSeeds * kK; e += 256) {
        const int c = e / kK, f = e % kK;
        const int64_t sc = c0 + c;
        ps[f][c] = (sc < m && k0 + f < dp) ? sx[(int64_t)seed_idx[sc] * dp + k0 + f] : 0.f;
      }
      __syncthreads();
#pragma unroll 8
      for (int f = 0; f < kK; ++f) {
        float xv[8], sv[4];
#pragma unroll
        for (int a = 0; a < 8; ++a) xv[a] = px[f][tr * 8 + a];
#pragma unroll
        for (int b = 0; b < 4; ++b) sv[b] = ps[f][tcl * 4 + b];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xv[a], sv[b], acc[a][b]);
      }
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t sc = c0 + tcl * 4 + b;
      if (sc >= m) continue;
      const float sn = snorm[sc];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        const float dd = fmaf(-2.f, acc[a][b], sn);
        if (dd < best[a]) {  // ascending seed order per thread: first minimum kept
          best[a] = dd;
          besti[a] = (int)sc;
        }
      }
    }
  }
  // combine the 16 seed groups per point: smallest distance, lowest index
#pragma unroll
  for (int a = 0; a < 8; ++a) {
    bd[tcl][tr * 8 + a] = best[a];
    bi[tcl][tr * 8 + a] = besti[a];
  }
  __syncthreads();
  if (tid < kRows && r0 + tid < n) {
    float v = bd[0][tid];
    int c = bi[0][tid];
    for (int g = 1; g < 16; ++g)
      if (bd[g][tid] < v || (bd[g][tid] == v && bi[g][tid] < c)) {
        v = bd[g][tid];
        c = bi[g][tid];
      }
    cell[r0 + tid] = c;
  }
}

// Greedy nearest-neighbour chain over the m2 super-seeds (start at 0, go to
// the closest unvisited one, lowest index on ties): super-seeds of one
// cluster end up adjacent, so the cells of a cluster form one run.
// pos[a] = position of super-seed a in the chain. One CTA: the m2 x m2
// distance matrix in smem, then one warp walks the chain.
__global__ void __launch_bounds__(1024)
    super_chain_kernel(const float* __restrict__ xc, int32_t dp, const int32_t* __restrict__ super_idx,
                       int64_t m2, int32_t* __restrict__ pos) {
  __shared__ float dist[kMaxSuper][kMaxSuper + 1];
  __shared__ int visited[kMaxSuper];
  for (int e = threadIdx.x; e < m2 * m2; e += blockDim.x) {
    const int a = e / (int)m2, b = e % (int)m2;
    const float* xa = xc + (int64_t)super_idx[a] * dp;
    const float* xb = xc + (int64_t)super_idx[b] * dp;
    float t = 0.f;
    for (int f = 0; f < dp; ++f) {
      const float q = xa[f] - xb[f];
      t = fmaf(q, q, t);
    }
    dist[a][b] = t;
  }
  for (int a = threadIdx.x; a < kMaxSuper; a += blockDim.x) visited[a] = a >= m2;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  int cur = 0;
  if (lane == 0) {
    visited[0] = 1;
    pos[0] = 0;
  }
  __syncwarp();
  for (int step = 1; step < m2; ++step) {
    float bv = FLT_MAX;
    int bi = 0x7fffffff;
    for (int b = lane; b < m2; b += 32)
      if (!visited[b] && (dist[cur][b] < bv || (dist[cur][b] == bv && b < bi))) {
        bv = dist[cur][b];
        bi = b;
      }
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    cur = bi;
    if (lane == 0) {
      visited[cur] = 1;
      pos[cur] = step;
    }
    __syncwarp();
  }
}

// seed c -> rank of (chain position of its super-seed, c) among the m
// seeds: one CTA, bitonic over the next power of two of m (m <= 8192)
__global__ void __launch_bounds__(1024)
    cell_rank_kernel(const int32_t* __restrict__ seed_super, const int32_t* __restrict__ super_pos,
                     int64_t m, int32_t* __restrict__ rank) {
  extern __shared__ int64_t key[];
  int mm = 1;
  while (mm < m) mm <<= 1;
  for (int i = threadIdx.x; i < mm; i += blockDim.x)
    key[i] = i < m ? ((int64_t)super_pos[seed_super[i]] << 32) | i : INT64_MAX;
  __syncthreads();
  for (int size = 2; size <= mm; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < mm; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const int64_t a = key[i], b = key[j];
          if ((a > b) == up) { key[i] = b; key[j] = a; }
        }
      }
      __syncthreads();
    }
  for (int r = threadIdx.x; r < m; r += blockDim.x) rank[key[r] & 0xffffffffll] = r;
}

__global__ void point_keys_kernel(const int32_t* __restrict__ cell, const int32_t* __restrict__ rank,
                                  int64_t n, int32_t* __restrict__ keys, int32_t* __restrict__ iota) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    keys[i] = rank[cell[i]];
    iota[i] = (int32_t)i;
  }
}

__global__ void seeds_kernel(int64_t n, int64_t m, int64_t m2, int32_t* __restrict__ seed_idx,
                             int32_t* __restrict__ super_idx) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < m) seed_idx[c] = (int32_t)(c * n / m);
  if (c < m2) super_idx[c] = (int32_t)((c * m / m2) * n / m);
}

// Xp[p, :] = X[perm[p], :] (fp64, one warp per row)
__global__ void gather_rows_kernel(const double* __restrict__ x, int64_t n, int32_t d,
                                   const int32_t* __restrict__ perm, double* __restrict__ xp) {
  const int lane = threadIdx.x & 31;
  for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < n;
       p += (int64_t)gridDim.x * (blockDim.x >> 5)) {
    const double* src = x + (int64_t)perm[p] * d;
    double* dst = xp + p * d;
    for (int f = lane; f < d; f += 32) dst[f] = src[f];
  }
}

// out[perm[p]] = v[p] (the embedding back in the caller's order)
__global__ void scatter_kernel(const double* __restrict__ v, const int32_t* __restrict__ perm,
                               int64_t n, double* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) out[perm[p]] = v[p];
}

int64_t al(int64_t b) { return (b + 255) & ~int64_t(255); }

int64_t seeds_for(int64_t n) { return (n + kCell - 1) / kCell; }

size_t cub_sort_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  return b;
}

}  // namespace

int64_t locality_bytes(int64_t n, int32_t d) {
  const int64_t m = seeds_for(n);
  return al(n * d * 8) + 5 * al(n * 4) + 4 * al(m * 4) + al(m * 4) + al(64) +
         al(kMaxSuper * 4) + al((int64_t)cub_sort_bytes(n));
}

Locality carve_locality(void* base, int64_t n, int32_t d) {
  const int64_t m = seeds_for(n);
  uint8_t* p = static_cast<uint8_t*>(base);
  auto take = [&](int64_t b) { uint8_t* q = p; p += al(b); return q; };
  Locality L;
  L.xp = reinterpret_cast<double*>(take(n * d * 8));
  L.perm = reinterpret_cast<int32_t*>(take(n * 4));
  L.cell = reinterpret_cast<int32_t*>(take(n * 4));
  L.keys = reinterpret_cast<int32_t*>(take(n * 4));
  L.keys_out = reinterpret_cast<int32_t*>(take(n * 4));
  L.iota = reinterpret_cast<int32_t*>(take(n * 4));
  L.seed_idx = reinterpret_cast<int32_t*>(take(m * 4));
  L.super_idx = reinterpret_cast<int32_t*>(take(m * 4));
  L.seed_super = reinterpret_cast<int32_t*>(take(m * 4));
  L.rank = reinterpret_cast<int32_t*>(take(m * 4));
  L.snorm = reinterpret_cast<float*>(take(m * 4));
  L.metric = reinterpret_cast<double*>(take(64));
  L.super_pos = reinterpret_cast<int32_t*>(take(kMaxSuper * 4));
  L.tmp = p;
  L.tmp_bytes = cub_sort_bytes(n);
  L.m = m;
  return L;
}

bool locality_enabled() {
  const char* e = getenv("GPIC_REORDER");
  return e == nullptr || atoi(e) != 0;
}

bool locality_forced() {
  const char* e = getenv("GPIC_REORDER");
  return e != nullptr && atoi(e) == 2;
}

void launch_order_metric(const Locality& L, const float* xc, int64_t n, int32_t dp, cudaStream_t s) {
  cudaMemsetAsync(L.metric, 0, 16, s);
  const int64_t stride = n > 16384 ? n / 16384 : 1;  // ~16k sampled rows
  order_metric_kernel<<<148, 256, 0, s>>>(xc, n, dp, stride, L.metric);
  count_launch();
}

int launch_locality_order(const Locality& L, const float* xc, const double* x, int64_t n, int32_t d,
                          int32_t dp, cudaStream_t s) {
  const int64_t m = L.m;
  const int64_t m2 = m < kMaxSuper ? m : kMaxSuper;
  seeds_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, s>>>(n, m, m2, L.seed_idx, L.super_idx);
  // super-seeds: nearest super-seed of every seed (the seeds' rows as points)
  seed_norm_kernel<<<(unsigned)ceil_div(m2, 256), 256, 0, s>>>(xc, dp, L.super_idx, m2, L.snorm);
  // the seeds as a point set: gather their rows into cell-sized scratch (xp's fp32 view)
  float* sx = reinterpret_cast<float*>(L.xp);
  {
    // rows seed_idx[c] -> sx[c] (one warp per seed, through gather_rows on fp32 pairs)
    const int64_t words = (int64_t)dp / 2;  // dp is a multiple of 32: fp32 pairs as doubles
    gather_rows_kernel<<<(unsigned)ceil_div(m, 8), 256, 0, s>>>(
        reinterpret_cast<const double*>(xc), m, (int32_t)words, L.seed_idx,
        reinterpret_cast<double*>(sx));
  }
  nearest_seed_kernel<<<(unsigned)ceil_div(m, kRows), 256, 0, s>>>(sx, m, dp, xc, L.super_idx,
                                                                   L.snorm, m2, L.seed_super);
  const size_t shm = (size_t)8 * [&] { int64_t q = 1; while (q < m) q <<= 1; return q; }();
  if (shm > 48 * 1024)
    GPIC_CUDA_TRY(cudaFuncSetAttribute(cell_rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)shm));
  super_chain_kernel<<<1, 1024, 0, s>>>(xc, dp, L.super_idx, m2, L.super_pos);
  cell_rank_kernel<<<1, 1024, shm, s>>>(L.seed_super, L.super_pos, m, L.rank);
  // every point: its nearest seed
  seed_norm_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, s>>>(xc, dp, L.seed_idx, m, L.snorm);
  nearest_seed_kernel<<<(unsigned)ceil_div(n, kRows), 256, 0, s>>>(xc, n, dp, xc, L.seed_idx,
                                                                   L.snorm, m, L.cell);
  point_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(L.cell, L.rank, n, L.keys, L.iota);
  size_t tb = L.tmp_bytes;
  int bits = 1;
  while ((int64_t(1) << bits) < m) ++bits;
  GPIC_CUDA_TRY(cub::DeviceRadixSort::SortPairs(L.tmp, tb, L.keys, L.keys_out, L.iota, L.perm,
                                                (int)n, 0, bits, s));
  gather_rows_kernel<<<(unsigned)ceil_div(n, 8) < 1184 ? (unsigned)ceil_div(n, 8) : 1184, 256, 0, s>>>(
      x, n, d, L.perm, L.xp);
  count_launch(12);
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

void launch_unpermute(const double* v, const int32_t* perm, int64_t n, double* out, cudaStream_t s) {
  scatter_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(v, perm, n, out);
  count_launch();
}

}  // namespace gpic
