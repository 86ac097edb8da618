// Provably-zero block pairs: affinity tiles that are never computed.
//
// The engines store an RBF entry as an exact zero when its exponent is
// below 2^-64 (sm100.cuh kFlushLog2), and a 32 x 32 box of such zeros is
// neither stored nor read (sparse.cu). This file proves, BEFORE the tcgen05
// pass, that whole 128 x 128 tiles can only produce such zeros, so their
// operand loads, MMAs, TMEM reads and epilogue never run.
//
// Rows are grouped into blocks S of B consecutive rows (B a multiple of 256,
// one affinity work unit never straddles two blocks). With c_S the centroid
// of block S and u = c_S' - c_S, every pair i in S, j in S' satisfies
//
//     |x_i - x_j| >= u.(x_j - x_i) / |u| >= (min_{j in S'} u.x_j - max_{i in S} u.x_i) / |u|
//
// (Cauchy-Schwarz; the projection onto the line joining the two centroids).
// For well-separated clusters the projected spread of a block is a few
// noise units while |u| is the cluster separation, so the bound is tight
// where the sphere bound |c_S - c_S'| - r_S - r_S' is not (in d dimensions a
// block's radius grows like sqrt(d); its extent along one line does not).
//
// Both extremes come from one product P = Xc C^T (n x nb, fp32 SIMT GEMM):
//     max_{i in S} u.x_i = max_{i in S} (P[i, S'] - P[i, S]) = M[S][S']
//     min_{j in S'} u.x_j = -M[S'][S]
// so gap(S, S') = -(M[S][S'] + M[S'][S]), reduced with an order-free max
// (atomicMax on order-preserving integer images: deterministic).
//
// The pair (S, S') is skipped when (gap - err) / |u| >= D with
//     D^2 = kSkipLog2 * 2 sigma^2 / log2(e),   kSkipLog2 = 66,
// two units of margin in the exponent over the flush (a factor 4 in value,
// far above the engines' 2^-22 R^2 / 2sigma^2 Gram rounding, which the
// spread-driven engine routing bounds), and err a rigorous bound on the fp32
// rounding of the four dot products (4 (2d + 2) 2^-24 |x|max |c|max).
// Every value, flag, degree and product is then bit-identical to the run
// that computes those tiles (their entries all flush to zero there).
//
// Output: the list of affinity work units (packed enumeration of
// affinity_tc.cu, row blocks of 128 MB rows x column tiles J >= MB rb) that
// are NOT skipped, ascending, and its length — the engine's CTAs split the
// list evenly.
#include <mma.h>

#include <cstdlib>

#include "common.cuh"
#include "ops.h"

namespace gpic {

namespace {

constexpr double kSkipLog2 = 66.0;
constexpr int kItemW = 0;  // per-item balance overhead (quarter tiles)
constexpr int kGemmRows = 128;  // rows per GEMM CTA (within one block)
constexpr int kGemmCols = 64;   // centroids per GEMM CTA
constexpr int kGemmK = 32;      // features per smem stage

// order-preserving image of a float in uint32 (for atomicMax)
__device__ __forceinline__ unsigned f2ord(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// centroid of block S, relative to the centring mean, from the prepare
// pass's fp64 column sums of 256-row groups (colpart): c_S = sum / count -
// mean (any c_S gives a valid bound; own_i and P use this same array).
// Padded to dp with zeros; |c|max as float bits.
__global__ void block_centroid_kernel(const double* __restrict__ colpart,
                                      const double* __restrict__ mean, int64_t n, int32_t d,
                                      int32_t dp, int64_t B, float* __restrict__ cent,
                                      unsigned* __restrict__ scal) {
  __shared__ float red[8];
  const int64_t S = blockIdx.x;
  const int64_t r0 = S * B, r1 = min(n, r0 + B);
  const int64_t g0 = r0 / 256, g1 = (r1 + 255) / 256;
  float c2 = 0.f;
  for (int f = threadIdx.x; f < dp; f += blockDim.x) {
    float c = 0.f;
    if (f < d) {
      double s = 0.0;
      for (int64_t g = g0; g < g1; ++g) s += colpart[g * d + f];
      c = (float)(s / (double)(r1 - r0) - mean[f]);
    }
    cent[S * dp + f] = c;
    c2 = fmaf(c, c, c2);
  }
  c2 = warp_sum_f32(c2);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c2;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    atomicMax(scal + 0, __float_as_uint(sqrtf(t) * 1.0001f));  // nonnegative: bits order
  }
}

// own_i = x_i . c_{S(i)} and |x|max
__global__ void own_kernel(const float* __restrict__ xc, int64_t n, int32_t dp, int64_t B,
                           const float* __restrict__ cent, float* __restrict__ own,
                           unsigned* __restrict__ scal) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float x2 = 0.f;
  if (i < n) {
    const float* x = xc + i * dp;
    const float* c = cent + (i / B) * dp;
    float s = 0.f;
    for (int f = 0; f < dp; ++f) {
      s = fmaf(x[f], c[f], s);
      x2 = fmaf(x[f], x[f], x2);
    }
    own[i] = s;
  }
  float m = sqrtf(x2) * 1.0001f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(scal + 1, __float_as_uint(m));
}

// M[S][S'] = max over the CTA's 128 rows (all in block S) of
// x_i . c_S' - own_i, for 64 centroids S'; fp32 FMA, smem-staged operands.
// 256 threads: thread (tr, tc) holds rows tr*8..+8 x centroids tc*4..+4.
__global__ void __launch_bounds__(256)
    proj_max_kernel(const float* __restrict__ xc, int64_t n, int32_t dp, int64_t B, int64_t nb,
                    const float* __restrict__ cent, const float* __restrict__ own,
                    unsigned* __restrict__ mmax) {
  __shared__ float sx[kGemmK][kGemmRows + 4];
  __shared__ float sc[kGemmK][kGemmCols + 4];
  __shared__ unsigned cmax[16][kGemmCols];
  const int64_t r0 = (int64_t)blockIdx.x * kGemmRows;
  const int64_t c0 = (int64_t)blockIdx.y * kGemmCols;
  const int tid = threadIdx.x;
  const int tr = tid >> 4, tcl = tid & 15;
  float acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
  for (int k0 = 0; k0 < dp; k0 += kGemmK) {
    // stage 128 rows x 32 features (transposed) and 64 centroids x 32
    for (int e = tid; e < kGemmRows * kGemmK; e += 256) {
      const int r = e / kGemmK, f = e % kGemmK;
      const int64_t row = r0 + r;
      sx[f][r] = (row < n && k0 + f < dp) ? xc[row * dp + k0 + f] : 0.f;
    }
    for (int e = tid; e < kGemmCols * kGemmK; e += 256) {
      const int c = e / kGemmK, f = e % kGemmK;
      const int64_t col = c0 + c;
      sc[f][c] = (col < nb && k0 + f < dp) ? cent[col * dp + k0 + f] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int f = 0; f < kGemmK; ++f) {
      float xv[8], cv[4];
#pragma unroll
      for (int a = 0; a < 8; ++a) xv[a] = sx[f][tr * 8 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) cv[b] = sc[f][tcl * 4 + b];
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fmaf(xv[a], cv[b], acc[a][b]);
    }
    __syncthreads();
  }
  // column max over this thread's 8 rows, then over the 16 row groups
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    float m = -INFINITY;
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int64_t row = r0 + tr * 8 + a;
      if (row < n) m = fmaxf(m, acc[a][b] - own[row]);
    }
    cmax[tr][tcl * 4 + b] = f2ord(m);
  }
  __syncthreads();
  if (tid < kGemmCols && c0 + tid < nb) {
    unsigned m = cmax[0][tid];
    for (int g = 1; g < 16; ++g) m = max(m, cmax[g][tid]);
    atomicMax(mmax + (r0 / B) * nb + c0 + tid, m);
  }
}

// One pass per 128 rows (all in one block S): the X tile stays in shared
// memory, own_i = x_i . c_S and |x_i| are formed there, then every chunk of
// 64 centroids goes through TF32 tensor-core products (wmma m16n16k8, fp32
// accumulate; the operand rounding is in the pair test's bound) and the
// column maxima of P - own. Dynamic smem: X tile [128][dp + 4], then a
// buffer shared by the centroid chunk [64][dp + 4] and the products
// [128][68].
__global__ void __launch_bounds__(256)
    proj_fused_kernel(const float* __restrict__ xc, int64_t n, int32_t dp, int64_t B, int64_t nb,
                      const float* __restrict__ cent, unsigned* __restrict__ mmax,
                      unsigned* __restrict__ scal) {
  using namespace nvcuda;
  extern __shared__ __align__(128) float fsm[];
  const int ldx = dp + 4, ldc = kGemmCols + 4;
  float* sX = fsm;
  float* sU = fsm + kGemmRows * ldx;  // centroid chunk / products
  __shared__ float own[kGemmRows];
  __shared__ unsigned cmax[4][kGemmCols];
  __shared__ float xmax[8];
  const int64_t r0 = (int64_t)blockIdx.x * kGemmRows;
  const int64_t S = r0 / B;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // float4 copies, a warp per row (dp is a multiple of 64: no index division)
  for (int r = warp; r < kGemmRows; r += 8) {
    const int64_t row = r0 + r;
    for (int f = lane * 4; f < dp; f += 128) {
      const float4 v = row < n ? *reinterpret_cast<const float4*>(xc + row * dp + f)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
      *reinterpret_cast<float4*>(sX + r * ldx + f) = v;
    }
  }
  __syncthreads();
  // own products and norms: a warp per 16 rows, lanes over the features
  {
    const float* c = cent + S * dp;
    float xm = 0.f;
    for (int r = warp * 16; r < warp * 16 + 16; ++r) {
      float a = 0.f, b = 0.f;
      for (int f = lane; f < dp; f += 32) {
        const float x = sX[r * ldx + f];
        a = fmaf(x, __ldg(c + f), a);
        b = fmaf(x, x, b);
      }
      a = warp_sum_f32(a);
      b = warp_sum_f32(b);
      if (lane == 0) own[r] = a;
      if (r0 + r < n) xm = fmaxf(xm, sqrtf(b) * 1.0001f);
    }
    if (lane == 0) xmax[warp] = xm;
  }
  __syncthreads();
  if (tid == 0) {
    float m = xmax[0];
    for (int w = 1; w < 8; ++w) m = fmaxf(m, xmax[w]);
    atomicMax(scal + 1, __float_as_uint(m));
  }
  for (int64_t c0 = 0; c0 < nb; c0 += kGemmCols) {
    __syncthreads();  // the previous chunk's products are consumed
    for (int c = warp; c < kGemmCols; c += 8) {
      const int64_t col = c0 + c;
      for (int f = lane * 4; f < dp; f += 128) {
        float4 v = col < nb ? *reinterpret_cast<const float4*>(cent + col * dp + f)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        // rounded to TF32 once here, not in every warp's fragments
        v.x = wmma::__float_to_tf32(v.x);
        v.y = wmma::__float_to_tf32(v.y);
        v.z = wmma::__float_to_tf32(v.z);
        v.w = wmma::__float_to_tf32(v.w);
        *reinterpret_cast<float4*>(sU + c * ldx + f) = v;
      }
    }
    __syncthreads();
    wmma::fragment<wmma::accumulator, 16, 16, 8, float> acc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) wmma::fill_fragment(acc[j], 0.f);
    for (int kk = 0; kk < dp; kk += 8) {
      wmma::fragment<wmma::matrix_a, 16, 16, 8, wmma::precision::tf32, wmma::row_major> a;
      wmma::load_matrix_sync(a, sX + warp * 16 * ldx + kk, ldx);
#pragma unroll
      for (int t = 0; t < a.num_elements; ++t) a.x[t] = wmma::__float_to_tf32(a.x[t]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        wmma::fragment<wmma::matrix_b, 16, 16, 8, wmma::precision::tf32, wmma::col_major> b;
        wmma::load_matrix_sync(b, sU + j * 16 * ldx + kk, ldx);  // already TF32
        wmma::mma_sync(acc[j], a, b, acc[j]);
      }
    }
    __syncthreads();  // every warp is done with the chunk: reuse its buffer
#pragma unroll
    for (int j = 0; j < 4; ++j)
      wmma::store_matrix_sync(sU + warp * 16 * ldc + j * 16, acc[j], ldc, wmma::mem_row_major);
    __syncthreads();
    {
      const int c = tid & (kGemmCols - 1), g = tid >> 6;
      float m = -INFINITY;
      for (int r = g * 32; r < g * 32 + 32; ++r)
        if (r0 + r < n) m = fmaxf(m, sU[r * ldc + c] - own[r]);
      cmax[g][c] = f2ord(m);
    }
    __syncthreads();
    if (tid < kGemmCols && c0 + tid < nb) {
      unsigned m = cmax[0][tid];
      for (int g = 1; g < 4; ++g) m = max(m, cmax[g][tid]);
      atomicMax(mmax + S * nb + c0 + tid, m);
    }
  }
}

// The same products on raw mma.sync m16n8k8 TF32 with the column maxima
// taken on the accumulator fragments (no product tile through shared
// memory, no wmma address arithmetic): warp w owns rows 16w..16w+15 of the
// CTA's 128 and all 64 centroid columns of a chunk (8 n-tiles); thread
// (g = lane / 4, t = lane % 4) holds P[g][2t, 2t+1] and P[g+8][2t, 2t+1] of
// each n-tile. Rows are padded with own = +inf so they never win a max.
// Row operands are rounded to TF32 per fragment (sX keeps fp32 for own /
// |x|), centroid chunks once when staged.
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

__global__ void __launch_bounds__(256)
    proj_mma_kernel(const float* __restrict__ xc, int64_t n, int32_t dp, int64_t B, int64_t nb,
                    const float* __restrict__ cent, unsigned* __restrict__ mmax,
                    unsigned* __restrict__ scal) {
  extern __shared__ __align__(128) float fsm[];
  const int ldx = dp + 4;  // conflict-free fragment loads: bank = 4 g + t
  float* sX = fsm;                      // [128][ldx]
  float* sU = fsm + kGemmRows * ldx;    // [64][ldx], TF32-rounded
  __shared__ float sOwn[kGemmRows];
  __shared__ unsigned wmx[8][kGemmCols];
  __shared__ float xmax[8];
  const int64_t r0 = (int64_t)blockIdx.x * kGemmRows;
  const int64_t S = r0 / B;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  // stage the rows; own products and norms in fp32 on the way
  {
    const float* cS = cent + S * dp;
    float xm = 0.f;
    for (int r = warp; r < kGemmRows; r += 8) {
      const int64_t row = r0 + r;
      float a = 0.f, b = 0.f;
      for (int f = lane * 4; f < dp; f += 128) {
        const float4 v = row < n ? *reinterpret_cast<const float4*>(xc + row * dp + f)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4*>(sX + r * ldx + f) = v;
        const float4 c = *reinterpret_cast<const float4*>(cS + f);
        a = fmaf(v.x, c.x, a);
        a = fmaf(v.y, c.y, a);
        a = fmaf(v.z, c.z, a);
        a = fmaf(v.w, c.w, a);
        b = fmaf(v.x, v.x, b);
        b = fmaf(v.y, v.y, b);
        b = fmaf(v.z, v.z, b);
        b = fmaf(v.w, v.w, b);
      }
      a = warp_sum_f32(a);
      b = warp_sum_f32(b);
      if (lane == 0) sOwn[r] = row < n ? a : INFINITY;
      if (row < n) xm = fmaxf(xm, sqrtf(b) * 1.0001f);
    }
    if (lane == 0) xmax[warp] = xm;
  }
  __syncthreads();
  if (tid == 0) {
    float m = xmax[0];
    for (int w = 1; w < 8; ++w) m = fmaxf(m, xmax[w]);
    atomicMax(scal + 1, __float_as_uint(m));
  }
  const float own0 = sOwn[warp * 16 + g], own1 = sOwn[warp * 16 + g + 8];
  const float* a_lo = sX + (warp * 16 + g) * ldx + t;
  const float* a_hi = a_lo + 8 * ldx;
  for (int64_t c0 = 0; c0 < nb; c0 += kGemmCols) {
    __syncthreads();  // the previous chunk is consumed
    for (int c = warp; c < kGemmCols; c += 8) {
      const int64_t col = c0 + c;
      for (int f = lane * 4; f < dp; f += 128) {
        float4 v = col < nb ? *reinterpret_cast<const float4*>(cent + col * dp + f)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        v.x = __uint_as_float(to_tf32(v.x));
        v.y = __uint_as_float(to_tf32(v.y));
        v.z = __uint_as_float(to_tf32(v.z));
        v.w = __uint_as_float(to_tf32(v.w));
        *reinterpret_cast<float4*>(sU + c * ldx + f) = v;
      }
    }
    __syncthreads();
    float acc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    for (int k0 = 0; k0 < dp; k0 += 8) {
      const uint32_t a0 = to_tf32(a_lo[k0]), a1 = to_tf32(a_hi[k0]);
      const uint32_t a2 = to_tf32(a_lo[k0 + 4]), a3 = to_tf32(a_hi[k0 + 4]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float* bp = sU + (j * 8 + g) * ldx + k0 + t;
        const uint32_t b0 = __float_as_uint(bp[0]), b1 = __float_as_uint(bp[4]);
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, "
            "{%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
            : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
            : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      }
    }
    // max over the warp's 16 rows of P[i][c] - own_i, per column
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float m0 = fmaxf(acc[j][0] - own0, acc[j][2] - own1);
      float m1 = fmaxf(acc[j][1] - own0, acc[j][3] - own1);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
      }
      if (g == 0) {
        wmx[warp][j * 8 + 2 * t] = f2ord(m0);
        wmx[warp][j * 8 + 2 * t + 1] = f2ord(m1);
      }
    }
    __syncthreads();
    if (tid < kGemmCols && c0 + tid < nb) {
      unsigned m = wmx[0][tid];
#pragma unroll
      for (int w = 1; w < 8; ++w) m = max(m, wmx[w][tid]);
      atomicMax(mmax + S * nb + c0 + tid, m);
    }
  }
}

__global__ void fill_u32_kernel(unsigned* p, int64_t count, unsigned v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) p[i] = v;
}

// skip[S][S'] for every block pair (symmetric, diagonal 0)
__global__ void pair_skip_kernel(const float* __restrict__ cent, const unsigned* __restrict__ mmax,
                                 const unsigned* __restrict__ scal, int64_t nb, int32_t dp,
                                 int32_t d, double d2_thr, int tf32, uint8_t* __restrict__ skip) {
  // a warp per block pair, lanes over the features (coalesced rows);
  // the summation order of |u|^2 only moves the bound by ~1e-16 relative,
  // far inside its (1 - 1e-6) margin — and a skip is safe either way
  const int lane = threadIdx.x & 31;
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (t >= nb * nb) return;
  const int64_t S = t / nb, T = t - S * nb;
  if (S == T) {
    if (lane == 0) skip[t] = 0;
    return;
  }
  const float* a = cent + S * dp;
  const float* b = cent + T * dp;
  double u2 = 0.0;
  for (int f = lane; f < dp; f += 32) {
    const double q = (double)b[f] - (double)a[f];
    u2 += q * q;
  }
  u2 = warp_sum_f64(u2);
  if (lane != 0) return;
  const double gap = -((double)ord2f(mmax[S * nb + T]) + (double)ord2f(mmax[T * nb + S]));
  const double xm = (double)__uint_as_float(scal[1]), cm = (double)__uint_as_float(scal[0]);
  // |dot error| <= (operand rounding + d fp32 adds) |x| |c| per product,
  // four products per gap, doubled for safety: fp32 operands (SIMT) or TF32
  // (tensor cores, 2^-10 relative per operand)
  const double per = (tf32 ? 2.0 * 0x1p-11 : 0.0) + (d + 2.0) * 0x1p-24;
  const double err = 8.0 * per * xm * cm;
  const double lb = (gap - err) / sqrt(u2) * (1.0 - 1e-6);
  skip[t] = (u2 > 0.0 && lb > 0.0 && lb * lb >= d2_thr) ? 1 : 0;
}

// affinity work unit u (row block rb of MB tile rows, column tile
// cb >= MB rb) -> kept unless its block pair is skipped
struct UnitGeom {
  int64_t nrt, nct, nb, B;
  int mb;
  __device__ void decode(int64_t u, int64_t& rb, int64_t& cb) const {
    int64_t lo = 0, hi = nrt - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (mid * nct - (int64_t)mb * mid * (mid - 1) / 2 <= u) lo = mid; else hi = mid - 1;
    }
    rb = lo;
    cb = lo * mb + (u - (lo * nct - (int64_t)mb * lo * (lo - 1) / 2));
  }
  __device__ bool kept(const uint8_t* skip, int64_t rb, int64_t cb) const {
    const int64_t S = rb * mb * 128 / B, T = cb * 128 / B;
    return skip[S * nb + T] == 0;
  }
  __device__ void step(int64_t& rb, int64_t& cb) const {
    if (++cb == nct) {
      ++rb;
      cb = rb * mb;
    }
  }
};

// kept units per row block (one warp per row block rb >= rb0)
__global__ void unit_count_kernel(const uint8_t* __restrict__ skip, UnitGeom g, int64_t rb0,
                                  int32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t rb = rb0 + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (rb >= g.nrt) return;
  int c = 0;
  for (int64_t cb = rb * g.mb + lane; cb < g.nct; cb += 32) c += g.kept(skip, rb, cb);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[rb - rb0] = c;
}

// ascending list of kept unit ids: each CTA adds the counts of the row
// blocks before its own, then warp per row block writes its ids in order
__global__ void unit_write_kernel(const uint8_t* __restrict__ skip, UnitGeom g, int64_t rb0,
                                  const int32_t* __restrict__ cnt, int32_t* __restrict__ list,
                                  int64_t* __restrict__ count) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t base_sh;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t first = (int64_t)blockIdx.x * nw;  // first row block (relative to rb0)
  int64_t part = 0;
  for (int64_t q = threadIdx.x; q < first; q += blockDim.x) part += cnt[q];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) wsum[w] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t b = 0;
    for (int q = 0; q < nw; ++q) b += wsum[q];
    base_sh = b;
  }
  __syncthreads();
  const int64_t rel = first + w;
  const int64_t rb = rb0 + rel;
  if (rb >= g.nrt) return;
  int64_t pos = base_sh;
  for (int64_t q = first; q < rel; ++q) pos += cnt[q];
  const int64_t ubase = rb * g.nct - (int64_t)g.mb * rb * (rb - 1) / 2 - rb * g.mb;
  for (int64_t c0 = rb * g.mb; c0 < g.nct; c0 += 32) {
    const int64_t cb = c0 + lane;
    const bool k = cb < g.nct && g.kept(skip, rb, cb);
    const unsigned m = __ballot_sync(0xffffffffu, k);
    if (k) list[pos + __popc(m & ((1u << lane) - 1u))] = (int32_t)(ubase + cb);
    pos += __popc(m);
  }
  if (rb == g.nrt - 1 && lane == 0) *count = pos;
}

// Matrix-free sym pass items: (row block rb, chunk c) over column tiles
// [32 c, 32 c + 32) from the row block's diagonal tile on. An item is kept
// when one of its tiles is in a non-pruned block pair. One warp per row
// block: lane = tile within the chunk.
struct ItemGeom {
  int64_t nrt, nct, nch, nb, B;
  int mb;
  int item_w;  // per-item CTA-balance overhead in quarter tiles (item_weight)
  __device__ bool tile_kept(const uint8_t* skip, int64_t rb, int64_t cb) const {
    return skip[(rb * mb * 128 / B) * nb + cb * 128 / B] == 0;
  }
};

// CTA-balance weight of a kept item with kt kept tiles: 4 per tile plus a
// fixed per-item cost (item set-up, its partial-row stores), in quarter tiles
__device__ __forceinline__ int item_weight(int kt, int item_w) {
  return kt > 0 ? 4 * kt + item_w : 0;
}

// kept[rb][ch] = number of kept tiles of item (rb, ch) (0: the item is
// pruned); cnt[rb] = kept items, tiles[rb] = the row block's item weights

__global__ void item_count_kernel(const uint8_t* __restrict__ skip, ItemGeom g,
                                  uint8_t* __restrict__ kept, int32_t* __restrict__ cnt,
                                  int32_t* __restrict__ tiles) {
  const int lane = threadIdx.x & 31;
  const int64_t rb = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (rb >= g.nrt) return;
  int c = 0, t = 0;
  for (int64_t ch = 0; ch < g.nch; ++ch) {
    const int64_t cb = ch * 32 + lane;
    const bool k = cb >= rb * g.mb && cb < g.nct && g.tile_kept(skip, rb, cb);
    const int m = __popc(__ballot_sync(0xffffffffu, k));
    if (lane == 0) kept[rb * g.nch + ch] = (uint8_t)m;
    c += m > 0;
    t += item_weight(m, g.item_w);
  }
  if (lane == 0) {
    cnt[rb] = c;
    tiles[rb] = t;
  }
}

// ascending kept items + wpre[u] = kept tiles of the items before list
// entry u (wpre[count] = all): the engine's CTAs split the tiles evenly
__global__ void item_write_kernel(const uint8_t* __restrict__ kept, ItemGeom g,
                                  const int32_t* __restrict__ cnt, const int32_t* __restrict__ tiles,
                                  int32_t* __restrict__ list, int64_t* __restrict__ wpre,
                                  int64_t* __restrict__ count) {
  __shared__ int64_t wsum[32], tsum[32];
  __shared__ int64_t base_sh, tbase_sh;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t first = (int64_t)blockIdx.x * nw;
  int64_t part = 0, tpart = 0;
  for (int64_t q = threadIdx.x; q < first; q += blockDim.x) {
    part += cnt[q];
    tpart += tiles[q];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    part += __shfl_xor_sync(0xffffffffu, part, o);
    tpart += __shfl_xor_sync(0xffffffffu, tpart, o);
  }
  if (lane == 0) {
    wsum[w] = part;
    tsum[w] = tpart;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t b = 0, tb = 0;
    for (int q = 0; q < nw; ++q) {
      b += wsum[q];
      tb += tsum[q];
    }
    base_sh = b;
    tbase_sh = tb;
  }
  __syncthreads();
  const int64_t rb = first + w;
  if (rb >= g.nrt) return;
  int64_t pos = base_sh, tpos = tbase_sh;
  for (int64_t q = first; q < rb; ++q) {
    pos += cnt[q];
    tpos += tiles[q];
  }
  for (int64_t c0 = 0; c0 < g.nch; c0 += 32) {
    const int64_t ch = c0 + lane;
    const int kt = ch < g.nch ? item_weight(kept[rb * g.nch + ch], g.item_w) : 0;
    const bool k = kt > 0;
    const unsigned m = __ballot_sync(0xffffffffu, k);
    // inclusive scan of the kept-tile counts over the lanes
    int sc = kt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) sc += y;
    }
    if (k) {
      const int64_t at = pos + __popc(m & ((1u << lane) - 1u));
      list[at] = (int32_t)(rb * g.nch + ch);
      wpre[at] = tpos + sc - kt;
    }
    pos += __popc(m);
    tpos += __shfl_sync(0xffffffffu, sc, 31);
  }
  if (rb == g.nrt - 1 && lane == 0) {
    *count = pos;
    wpre[pos] = tpos;
  }
}

int64_t al256(int64_t b) { return (b + 255) & ~int64_t(255); }

// matrix-free items: row blocks of 128 rows at most (MB = 1) x 32-tile chunks
int64_t max_items(int64_t n) { return ceil_div(n, 128) * ceil_div(ceil_div(n, 128), 32); }

}  // namespace

// per-item CTA-balance overhead of the matrix-free item list, in quarter
// tiles (GPIC_MF_ITEM_W: measurement knob); item_wpre[count] =
// 4 * kept tiles + count * this
int prune_item_weight() {
  const char* iw = getenv("GPIC_MF_ITEM_W");
  return iw != nullptr ? atoi(iw) : kItemW;
}

bool prune_enabled() {
  const char* e = getenv("GPIC_PRUNE");
  return e == nullptr || atoi(e) != 0;
}

int64_t prune_block_rows(int64_t n) {
  // finer blocks prune more (config 5: 17 % of the work kept at B = 2048,
  // 10 % at 1024); the one-off GEMM costs n^2 d / B and the pair mask
  // (n / B)^2: 512-row blocks up to n = 2M, doubling after
  int64_t B = 512;
  while (B < 8192 && n / B > 4096) B <<= 1;
  return B;
}

int64_t prune_bytes(int64_t n, int32_t dp) {
  const int64_t B = prune_block_rows(n), nb = ceil_div(n, B);
  const int64_t nt = ceil_div(n, 128);
  return al256(nb * dp * 4) + al256(n * 4) + al256(nb * nb * 4) + al256(nb * nb) +
         al256(nt * (nt + 1) / 2 * 4) + al256(64) + al256(nt * 4) + al256(max_items(n) * 4) +
         al256(max_items(n)) + al256(nt * 4) + al256((max_items(n) + 1) * 8) +
         al256((3 + 257) * 8) + al256(256 * 8);
}

// count slot: [0] unit count, [8] item count, [16] scal, [32] sched; c is
// the unit count (the slot start)
unsigned* prune_sched(const int64_t* c) {
  return reinterpret_cast<unsigned*>(reinterpret_cast<uintptr_t>(c) + 32);
}

PruneMask carve_prune(void* base, int64_t n, int32_t dp) {
  PruneMask m;
  m.B = prune_block_rows(n);
  m.nb = ceil_div(n, m.B);
  const int64_t nt = ceil_div(n, 128);
  uint8_t* p = static_cast<uint8_t*>(base);
  m.cent = reinterpret_cast<float*>(p); p += al256(m.nb * dp * 4);
  m.own = reinterpret_cast<float*>(p); p += al256(n * 4);
  m.mmax = reinterpret_cast<unsigned*>(p); p += al256(m.nb * m.nb * 4);
  m.skip = p; p += al256(m.nb * m.nb);
  m.units = reinterpret_cast<int32_t*>(p); p += al256(nt * (nt + 1) / 2 * 4);
  m.count = reinterpret_cast<int64_t*>(p);
  m.scal = reinterpret_cast<unsigned*>(p + 16);
  m.sched = reinterpret_cast<unsigned*>(p + 32);  // zeroed with scal by launch_prune
  p += al256(64);
  m.rbcount = reinterpret_cast<int32_t*>(p); p += al256(nt * 4);
  m.items = reinterpret_cast<int32_t*>(p); p += al256(max_items(n) * 4);
  m.item_kept = p; p += al256(max_items(n));
  m.rbtiles = reinterpret_cast<int32_t*>(p); p += al256(nt * 4);
  m.item_wpre = reinterpret_cast<int64_t*>(p); p += al256((max_items(n) + 1) * 8);
  m.cta_cuts = reinterpret_cast<int64_t*>(p); p += al256((3 + 257) * 8);
  m.cta_ns = reinterpret_cast<uint64_t*>(p);
  m.item_count = m.count + 1;
  return m;
}

void launch_prune(const PruneMask& m, const float* xc, const double* colpart, const double* mean,
                  int64_t n, int32_t d, int32_t dp, double sigma, int mb, int64_t row_lo,
                  cudaStream_t s, int64_t row_hi) {
  if (row_hi <= 0) row_hi = n;
  const int64_t nb = m.nb, B = m.B;
  fill_u32_kernel<<<(unsigned)ceil_div(nb * nb + 2, 256), 256, 0, s>>>(m.mmax, nb * nb, 0u);
  fill_u32_kernel<<<1, 32, 0, s>>>(m.scal, 6, 0u);  // scal[2], pad, sched[2]
  fill_u32_kernel<<<1, 32, 0, s>>>(reinterpret_cast<unsigned*>(m.cta_cuts), 2, 0u);  // no cuts yet
  block_centroid_kernel<<<(unsigned)nb, 128, 0, s>>>(colpart, mean, n, d, dp, B, m.cent, m.scal);
  // GPIC_PRUNE_TF32=0: the fp32 SIMT products, =1: wmma, =2 (default):
  // mma.sync with the maxima on the fragments (measurement knob)
  const char* tfe = getenv("GPIC_PRUNE_TF32");
  const int tfm = tfe == nullptr ? 2 : atoi(tfe);
  const int tf32 = tfm != 0;
  if (!tf32) own_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(xc, n, dp, B, m.cent, m.own, m.scal);
  if (tfm == 2) {
    const size_t shm = (size_t)(kGemmRows + kGemmCols) * (dp + 4) * 4;
    static size_t shm_mma = 0;
    if (shm > 48 * 1024 && shm > shm_mma) {
      cudaFuncSetAttribute(proj_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
      shm_mma = shm;
    }
    proj_mma_kernel<<<(unsigned)ceil_div(n, kGemmRows), 256, shm, s>>>(xc, n, dp, B, nb, m.cent,
                                                                      m.mmax, m.scal);
  } else if (tf32) {
    const int ldx = dp + 4;
    const int ubuf = kGemmCols * ldx > kGemmRows * (kGemmCols + 4) ? kGemmCols * ldx
                                                                     : kGemmRows * (kGemmCols + 4);
    const size_t shm = (size_t)(kGemmRows * ldx + ubuf) * 4;
    static size_t shm_set = 0;
    if (shm > 48 * 1024 && shm > shm_set) {
      cudaFuncSetAttribute(proj_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
      shm_set = shm;
    }
    proj_fused_kernel<<<(unsigned)ceil_div(n, kGemmRows), 256, shm, s>>>(xc, n, dp, B, nb, m.cent,
                                                                        m.mmax, m.scal);
  } else {
    const dim3 pg((unsigned)ceil_div(n, kGemmRows), (unsigned)ceil_div(nb, kGemmCols));
    proj_max_kernel<<<pg, 256, 0, s>>>(xc, n, dp, B, nb, m.cent, m.own, m.mmax);
  }
  const double d2_thr = kSkipLog2 * 2.0 * sigma * sigma / 1.4426950408889634 * (1.0 + 1e-6);
  pair_skip_kernel<<<(unsigned)ceil_div(nb * nb, 8), 256, 0, s>>>(m.cent, m.mmax, m.scal, nb, dp,
                                                                    d, d2_thr, tf32, m.skip);
  if (mb <= 0) {  // matrix-free: the item list instead of the unit list
    ItemGeom g;
    g.mb = -mb;
    g.item_w = prune_item_weight();
    g.nct = ceil_div(n, 128);
    g.nrt = ceil_div(n, 128 * g.mb);
    g.nch = ceil_div(g.nct, 32);
    g.nb = nb;
    g.B = B;
    item_count_kernel<<<(unsigned)ceil_div(g.nrt, 8), 256, 0, s>>>(m.skip, g, m.item_kept,
                                                                   m.rbcount, m.rbtiles);
    item_write_kernel<<<(unsigned)ceil_div(g.nrt, 8), 256, 0, s>>>(
        m.item_kept, g, m.rbcount, m.rbtiles, m.items, m.item_wpre, m.item_count);
    count_launch(8);
    return;
  }
  UnitGeom g;
  g.nct = ceil_div(n, 128);
  g.nrt = ceil_div(row_hi, 128 * mb);  // a packed shard's units end at its last row block
  g.nb = nb;
  g.B = B;
  g.mb = mb;
  const int64_t rb0 = row_lo / (128 * mb);
  const int64_t u_lo = rb0 * g.nct - (int64_t)mb * rb0 * (rb0 - 1) / 2;
  const int64_t u_hi = g.nrt * g.nct - (int64_t)mb * g.nrt * (g.nrt - 1) / 2;
  (void)u_lo;
  (void)u_hi;
  const int64_t nrb = g.nrt - rb0;
  unit_count_kernel<<<(unsigned)ceil_div(nrb, 8), 256, 0, s>>>(m.skip, g, rb0, m.rbcount);
  unit_write_kernel<<<(unsigned)ceil_div(nrb, 8), 256, 0, s>>>(m.skip, g, rb0, m.rbcount, m.units,
                                                               m.count);
  count_launch(8);
}

}  // namespace gpic
