// Stage 1 (FP32 FFMA engine): affinity tile + fused epilogue.
//
// One CTA computes a 128x128 tile of the Gram matrix G = Xc Xc^T on the
// CUDA cores (fp32 FFMA, 8x8 outputs per thread), then in registers:
//     d2 = |x_i|^2 + |x_j|^2 - 2 G_ij   (clamped at 0)
//     a  = exp2(d2 * (-log2(e) / (2 sigma^2)))      == exp(-d2 / (2 sigma^2))
//     a  = 0 on the diagonal and in padding columns  (affinity.py:102-103)
// stores A once (fp32, streaming stores) and writes the tile's fp32 row
// partial sums; gpic_degree combines them in fixed order (fp64).
// It reads the fp32 centred rows (the d_xlo operand of gpic_prepare_points).
// This is the measured-error comparator of the tcgen05 3-term fp16 engine
// (affinity_tc.cu) and the engine used when tcgen05 is unavailable for a
// shape.
#include "common.cuh"
#include "ops.h"
#include "sm100.cuh"

namespace gpic {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, PADS = 4;

// DIFF (RBF): accumulate sum_f (x_if - x_jf)^2 directly instead of the Gram
// form |x_i|^2 + |x_j|^2 - 2 x_i.x_j: the fp32 rounding of the coordinates
// then costs ~2^-24 |x_i - x_j| |x| in d2 instead of ~2^-23 |x|^2, which is
// what keeps near pairs exact when the spread is large against sigma.
// PACKED: one CTA per upper-triangle tile (I <= J) of the packed layout,
// writing the tile plus its per-tile degree partials (row sums; column sums
// per 32-row quadrant off the diagonal) for launch_sym_degree.
// KD > 0: the data has at most KD (<= 16) non-zero features: one K chunk
// whose inner loop stops at KD (the padding columns are zero either way).
template <bool DIFF, bool PACKED, int KD>
__global__ void __launch_bounds__(256, KD == 2 ? 3 : 2)
    affinity_simt_kernel(const float* __restrict__ xc, const float* __restrict__ sqn, int64_t n, int32_t dp, int64_t row_lo,
                         int64_t row_hi, float neg_scale_log2, float* __restrict__ a, int64_t lda,
                         float* __restrict__ rowpart, int64_t rows_pad, int kind,
                         float* __restrict__ degcol) {
  __shared__ __align__(16) float As[BK][BM + PADS];
  __shared__ __align__(16) float Bs[BK][BN + PADS];

  const int tid = threadIdx.x;
  const int tx = tid & 15;   // column group
  const int ty = tid >> 4;   // row group
  int64_t tI = blockIdx.y, tJ = blockIdx.x;
  const int64_t nt = (n + BN - 1) / BN;
  if (PACKED) {  // packed tile index -> (I, J), row-major upper triangle
    // row I starts at S(I) = I nt - I (I - 1) / 2: invert the quadratic,
    // then correct the floating-point estimate by one step either way
    const int64_t t = blockIdx.x;
    const double b = 2.0 * (double)nt + 1.0;
    int64_t I = (int64_t)((b - sqrt(b * b - 8.0 * (double)t)) * 0.5);
    auto start = [&](int64_t r) { return r * nt - r * (r - 1) / 2; };
    if (I < 0) I = 0;
    while (I > 0 && start(I) > t) --I;
    while (start(I + 1) <= t) ++I;
    tI = I;
    tJ = I + (t - start(I));
  }
  const int64_t col0 = tJ * BN;
  const int64_t lrow0 = tI * BM;         // local (shard) row of the tile
  const int64_t grow0 = row_lo + lrow0;  // global row

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  // loader mapping: 128 rows x 16 features = 512 float4; 256 threads x 2
  const int kend = KD > 0 ? BK : dp;
  for (int k0 = 0; k0 < kend; k0 += BK) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int e = tid + q * 256;       // 0..511
      const int r = e >> 2;              // 0..127
      const int c = (e & 3) * 4;         // 0,4,8,12
      const int64_t ra = grow0 + r;      // rows are padded to 128 (zero rows)
      const int64_t rb = col0 + r;
      const float4 av = *reinterpret_cast<const float4*>(xc + ra * dp + k0 + c);
      const float4 bv = *reinterpret_cast<const float4*>(xc + rb * dp + k0 + c);
      As[c + 0][r] = av.x;
      As[c + 1][r] = av.y;
      As[c + 2][r] = av.z;
      As[c + 3][r] = av.w;
      Bs[c + 0][r] = bv.x;
      Bs[c + 1][r] = bv.y;
      Bs[c + 2][r] = bv.z;
      Bs[c + 3][r] = bv.w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < (KD > 0 ? KD : BK); ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[k][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[k][ty * 8 + 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[k][64 + tx * 4]);
      const float ar[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float br[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (DIFF) {
            const float t = ar[i] - br[j];
            acc[i][j] = fmaf(t, t, acc[i][j]);
          } else {
            acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
          }
        }
    }
    __syncthreads();
  }

  // fused epilogue
  __shared__ float csum[PACKED ? 16 : 1][PACKED ? BN : 1];  // packed: per-ty column sums
  float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  float sqb[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t cj = col0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
    sqb[j] = sqn[cj];
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t lr = lrow0 + ty * 8 + i;
    const int64_t gr = row_lo + lr;
    const float sqa = sqn[gr];
    float vals[8];
    float rs = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t cj = col0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      float e;
      if (kind == GPIC_KIND_COSINE) {
        e = fmaxf(acc[i][j], 0.f);  // unit rows: the Gram entry is the cosine
      } else if (DIFF) {
        e = ex2_flush(acc[i][j] * neg_scale_log2);
      } else {
        const float d2 = fmaxf(sqa + sqb[j] - 2.f * acc[i][j], 0.f);
        e = ex2_flush(d2 * neg_scale_log2);
      }
      if (cj == gr || cj >= n || (PACKED && gr >= n)) e = 0.f;
      vals[j] = e;
      rs += e;
      cs[j] += e;
    }
    // 16 column-group lanes share this row: fixed butterfly
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
    if (PACKED) {
      const int64_t tile = tI * nt - tI * (tI - 1) / 2 + (tJ - tI);
      float* trow = a + tile * (BM * BN) + (ty * 8 + i) * BN;
      st_stream_f4(reinterpret_cast<float4*>(trow + tx * 4),
                   make_float4(vals[0], vals[1], vals[2], vals[3]));
      st_stream_f4(reinterpret_cast<float4*>(trow + 64 + tx * 4),
                   make_float4(vals[4], vals[5], vals[6], vals[7]));
      if (tx == 0) rowpart[tile * BM + ty * 8 + i] = rs;  // degrow
    } else if (gr < row_hi) {
      float* arow = a + lr * lda;
      const int64_t c0 = col0 + tx * 4;
      const int64_t c1 = col0 + 64 + tx * 4;
      if (c0 < lda) st_stream_f4(reinterpret_cast<float4*>(arow + c0),
                                 make_float4(vals[0], vals[1], vals[2], vals[3]));
      if (c1 < lda) st_stream_f4(reinterpret_cast<float4*>(arow + c1),
                                 make_float4(vals[4], vals[5], vals[6], vals[7]));
      if (tx == 0) rowpart[(int64_t)blockIdx.x * rows_pad + lr] = rs;
    }
  }
  if (PACKED && tI < tJ) {
    // column sums per 32-row quadrant q (row groups ty = 4q..4q+3, in order)
#pragma unroll
    for (int j = 0; j < 8; ++j) csum[ty][j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4)] = cs[j];
    __syncthreads();
    const int64_t tile = tI * nt - tI * (tI - 1) / 2 + (tJ - tI);
    for (int e = tid; e < 4 * BN; e += 256) {
      const int q = e / BN, c = e % BN;
      degcol[(tile * 4 + q) * BN + c] =
          ((csum[4 * q][c] + csum[4 * q + 1][c]) + csum[4 * q + 2][c]) + csum[4 * q + 3][c];
    }
  }
}

// deg_i = sum over column tiles (fixed order, fp64) of the fp32 row partials.
__global__ void degree_kernel(const float* __restrict__ rowpart, int64_t rows, int64_t rows_pad,
                              int64_t n_ctiles, int64_t row_lo, double* __restrict__ deg,
                              gpic_ctl* ctl) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  double s = 0.0;
  for (int64_t t = 0; t < n_ctiles; ++t) s += (double)rowpart[t * rows_pad + i];
  deg[i] = s;
  if (ctl != nullptr && s <= 0.0) raise_status(ctl, GPIC_E_ZERO_DEGREE, row_lo + i, -1, s);
}

}  // namespace

void launch_affinity_simt(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                          int32_t d, int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2,
                          float* a, int64_t lda, float* rowpart, int64_t rows_pad,
                          cudaStream_t s, int kind) {
  const int64_t rows = row_hi - row_lo;
  dim3 grid((unsigned)ceil_div(n, BN), (unsigned)ceil_div(rows, BM));
#define GPIC_SIMT_LAUNCH(DIFF, PACKED, KD) \
  affinity_simt_kernel<DIFF, PACKED, KD><<<grid, 256, 0, s>>>( \
      xlo, sqn, n, dp, row_lo, row_hi, neg_scale_log2, a, lda, rowpart, rows_pad, kind, nullptr)
  if (kind == GPIC_KIND_COSINE) GPIC_SIMT_LAUNCH(false, false, 0);
  else if (d <= 2) GPIC_SIMT_LAUNCH(true, false, 2);
  else if (d <= 4) GPIC_SIMT_LAUNCH(true, false, 4);
  else if (d <= 8) GPIC_SIMT_LAUNCH(true, false, 8);
  else GPIC_SIMT_LAUNCH(true, false, 0);
#undef GPIC_SIMT_LAUNCH
  count_launch();
}

void launch_affinity_simt_packed(const float* xlo, const float* sqn, int64_t n, int32_t d,
                                 int32_t dp, float neg_scale_log2, float* a_packed, float* degrow,
                                 float* degcol, cudaStream_t s, int kind) {
  const unsigned grid = (unsigned)packed_tiles(n);
#define GPIC_SIMT_LAUNCH(DIFF, KD) \
  affinity_simt_kernel<DIFF, true, KD><<<grid, 256, 0, s>>>( \
      xlo, sqn, n, dp, 0, n, neg_scale_log2, a_packed, 0, degrow, 0, kind, degcol)
  if (kind == GPIC_KIND_COSINE) GPIC_SIMT_LAUNCH(false, 0);
  else if (d <= 2) GPIC_SIMT_LAUNCH(true, 2);
  else if (d <= 4) GPIC_SIMT_LAUNCH(true, 4);
  else if (d <= 8) GPIC_SIMT_LAUNCH(true, 8);
  else GPIC_SIMT_LAUNCH(true, 0);
#undef GPIC_SIMT_LAUNCH
  count_launch();
}

void launch_degree(const float* rowpart, int64_t rows, int64_t rows_pad, int64_t n_ctiles,
                   int64_t row_lo, double* deg, gpic_ctl* ctl, cudaStream_t s) {
  degree_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, s>>>(rowpart, rows, rows_pad, n_ctiles,
                                                              row_lo, deg, ctl);
  count_launch();
}

}  // namespace gpic
