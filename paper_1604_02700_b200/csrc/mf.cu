// Matrix-free power iteration: when 4n^2 bytes of A do not
// fit in HBM (config 5: n = 1M -> 4 TB), every product A v is recomputed
// from X: the tcgen05 affinity engine in matvec mode multiplies each fresh
// exp2 entry by v_j in registers and leaves one fp64 row partial per
// 32-tile column chunk (affinity_tc.cu); this reduce combines the chunk
// partials in fixed order, applies 1/deg and stores the row of y into every
// rank's y buffer (same epilogue contract as the dense GEMV, so the
// tau / normalise / stop tail and the multi-rank exchange are unchanged).
// Degrees are the same pass with v = 1.
//
// Whole matrix on one rank (the sym pass): only tiles J >= I are computed;
// y_i = (row partials of row i's chunks from its own diagonal tile on) +
// (column partials of the tiles (I', J(i)), I' < J(i), i.e. the transposed
// upper triangle), combined by mf_sym_reduce_kernel in a fixed order.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "ops.h"
#include "sm100.cuh"

namespace gpic {

namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(256)
    mf_reduce_kernel(const double* __restrict__ ypart, int64_t nparts, int64_t rows_pad,
                     int64_t rows, int64_t row_lo, const double* __restrict__ deg,
                     const PeerTable pt, gpic_ctl* ctl) {
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows) {
    double s = 0.0;
    for (int64_t p = 0; p < nparts; ++p) s += ypart[p * rows_pad + i];
    const double val = deg != nullptr ? s / deg[i] : s;
    const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
    for (int p = 0; p < pt.nranks; ++p) pt.y[p][parity][row_lo + i] = val;
  }
  if (pt.flags[0] == nullptr) return;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&ctl->arrive[2], 1u);
    if (prev == gridDim.x - 1) {
      ctl->arrive[2] = 0u;
      __threadfence_system();
      const uint64_t epoch = ctl->sync_epoch + (uint64_t)ctl->iter + 1;
      for (int p = 0; p < pt.nranks; ++p) st_release_sys(pt.flags[p] + pt.self, epoch);
    }
  }
}

// Difference-form pass for RBF with d <= 8 (the tensor Gram's fp32
// cancellation exceeds the embedding gate there; capi.cu effective_engine):
// CTA (chunk c, row block) sums a_ij v_j over the chunk's 4096 columns for
// 128 rows, a_ij = exp2(ns * sum_k (x_ik - x_jk)^2), a_ii = 0. Thread
// (row r, half h) takes columns h*64 .. h*64+63 of each 128-column tile
// (the warp reads one column at a time: shared-memory broadcast); fp32 per
// tile, fp64 across tiles and halves, fixed order. Writes the chunk's row
// partial in the tensor pass's layout (ypart[c * rows_pad + r]).
template <int KD>
__global__ void __launch_bounds__(256)
    mf_simt_kernel(const float* __restrict__ xc, int32_t dp, int64_t n, int64_t row_lo,
                   int64_t rows, int64_t rows_pad, float ns, const float* __restrict__ v32,
                   double* __restrict__ ypart, gpic_ctl* ctl) {
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  __shared__ float cx[128][KD];
  __shared__ float cv[128];
  __shared__ double half1[128];
  const int t = threadIdx.x, r = t & 127, h = t >> 7;
  const int64_t lr = (int64_t)blockIdx.y * 128 + r;
  const int64_t gi = row_lo + lr;
  float xi[KD];
#pragma unroll
  for (int k = 0; k < KD; ++k) xi[k] = gi < n ? xc[gi * dp + k] : 0.f;
  const int64_t c0 = (int64_t)blockIdx.x * 4096;
  double acc = 0.0;
  for (int tile = 0; tile < 32; ++tile) {
    const int64_t j0 = c0 + tile * 128;
    if (j0 >= n) break;
    __syncthreads();
    for (int e = t; e < 128 * KD; e += 256) {
      const int jj = e / KD, k = e % KD;
      const int64_t j = j0 + jj;
      cx[jj][k] = j < n ? xc[j * dp + k] : 0.f;
    }
    if (t < 128) cv[t] = j0 + t < n ? v32[j0 + t] : 0.f;
    __syncthreads();
    float s = 0.f;
#pragma unroll 4
    for (int jj = h * 64; jj < h * 64 + 64; ++jj) {
      float d2 = 0.f;
#pragma unroll
      for (int k = 0; k < KD; ++k) {
        const float df = xi[k] - cx[jj][k];
        d2 = fmaf(df, df, d2);
      }
      float a = ex2_flush(d2 * ns);
      if (j0 + jj == gi) a = 0.f;
      s = fmaf(a, cv[jj], s);
    }
    acc += (double)s;
  }
  if (h == 1) half1[r] = acc;
  __syncthreads();
  if (h == 0 && lr < rows) ypart[(int64_t)blockIdx.x * rows_pad + lr] = acc + half1[r];
}

// The item ids [lo, hi) a rank owns in a pruned sym pass shared by
// share_n ranks (the same tile-balanced split as the engine's, prune.cu
// list order); everything when unshared.
struct ItemShare {
  const int32_t* items;
  const int64_t* count;
  const int64_t* wpre;
  int r, nr;
  __device__ void range(int64_t* out) const {
    out[0] = 0;
    out[1] = INT64_MAX;
    if (items == nullptr || nr <= 1) return;
    const int64_t total = *count, W = wpre[total];
    auto lb = [&](int64_t target) {
      int64_t lo = 0, hi = total;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (wpre[mid] >= target) hi = mid; else lo = mid + 1;
      }
      return lo;
    };
    const int64_t ua = lb(W * r / nr), ub = r + 1 == nr ? total : lb(W * (r + 1) / nr);
    out[0] = ua < total ? items[ua] : INT64_MAX;
    out[1] = ub < total ? items[ub] : INT64_MAX;
  }
};

// One CTA per column tile J (128 rows of y), kSeg segments: segment s sums
// its share of row i's chunk partials (chunks from the row block's first
// tile on) and of the column records (row blocks I' = 0 .. J / MB), then the
// segment sums are added in order. The shape depends on (n, MB) only.
constexpr int kSeg = 8;

__global__ void __launch_bounds__(128 * kSeg)
    mf_sym_reduce_kernel(const double* __restrict__ ypart, const float* __restrict__ colpart,
                         int64_t nparts, int64_t rows_pad, int64_t n, int64_t nct, int mb,
                         const double* __restrict__ deg, const PeerTable pt, gpic_ctl* ctl,
                         const uint8_t* __restrict__ item_kept, const uint8_t* __restrict__ pskip,
                         int64_t pB, int64_t pnb, ItemShare sh) {
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  __shared__ double part[kSeg][128];
  __shared__ int64_t id_rng[2];
  if (threadIdx.x == 0) sh.range(id_rng);
  __syncthreads();
  const int64_t id_lo = id_rng[0], id_hi = id_rng[1];  // this rank's item ids
  const int64_t J = blockIdx.x;
  const int o = threadIdx.x % 128, sg = threadIdx.x / 128;
  const int64_t i = J * 128 + o;
  const int64_t rb = J / mb;  // row block of row i (128 * mb rows)
  const int64_t c0 = rb * mb / 32;  // first chunk written for this row block (kChunkTiles = 32)
  const int64_t p0 = c0 + (nparts - c0) * sg / kSeg, p1 = c0 + (nparts - c0) * (sg + 1) / kSeg;
  double s = 0.0;
  // pruned pass: chunk partials of kept items and records of kept tiles
  // only (the others are exact zeros and never written)
  if (i < n)
    for (int64_t p = p0; p < p1; ++p) {
      const int64_t id = rb * nparts + p;
      if ((item_kept == nullptr || item_kept[id] != 0) && id >= id_lo && id < id_hi)
        s += ypart[p * rows_pad + i];
    }
  const int64_t nrec = rb + 1;  // row blocks 0 .. rb hold tiles (I', J) with I' <= J
  const int64_t r0 = nrec * sg / kSeg, r1 = nrec * (sg + 1) / kSeg;
  const int64_t TJ = pskip != nullptr ? J * 128 / pB : 0;
#pragma unroll 4
  for (int64_t r = r0; r < r1; ++r) {
    if (pskip != nullptr && pskip[(r * mb * 128 / pB) * pnb + TJ]) continue;
    const int64_t id = r * nparts + J / 32;  // the item that wrote this record
    if (id < id_lo || id >= id_hi) continue;
    const int64_t rec = r * nct - (int64_t)mb * r * (r - 1) / 2 + (J - r * mb);
    s += (double)colpart[rec * 128 + o];
  }
  part[sg][o] = s;
  __syncthreads();
  if (sg == 0 && i < n) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kSeg; ++q) t += part[q][o];
    const double val = deg != nullptr ? t / deg[i] : t;
    const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
    const int own = pt.scatter ? slice_owner(i, n, pt.nranks) : -1;
    for (int p = 0; p < pt.nranks; ++p)
      if (own < 0 || own == p) pt.y[p][parity][i] = val;
  }
  if (pt.flags[0] == nullptr) return;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&ctl->arrive[2], 1u);
    if (prev == gridDim.x - 1) {
      ctl->arrive[2] = 0u;
      __threadfence_system();
      const uint64_t epoch = ctl->sync_epoch + (uint64_t)ctl->iter + 1;
      for (int p = 0; p < pt.nranks; ++p) st_release_sys(pt.flags[p] + pt.self, epoch);
    }
  }
}

__global__ void fill_ones_kernel(float* v, int64_t n, int64_t len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < len) v[i] = i < n ? 1.f : 0.f;
}

}  // namespace

// scratch of one pass: the chunk row partials, plus (whole matrix on one
// rank: the sym pass) the column-partial records behind them
bool mf_sym_default() {
  const char* e = getenv("GPIC_MF_SYM");  // tests / ablation: 0 forces the full-square pass
  return e == nullptr || atoi(e) != 0;
}
static bool mf_sym(const MfOperands& op, int64_t row_lo, int64_t rows) {
  return op.sym && row_lo == 0 && rows == op.n;
}

int64_t mf_ypart_doubles(int64_t n, int32_t dp, int64_t rows) {
  const int64_t rp = mf_parts(n, dp) * round_up(rows, kTileM);
  return rows == n ? rp + ceil_div(mf_colpart_floats(n, dp), 2) : rp;
}

int launch_mf_matvec(const MfOperands& op, int64_t row_lo, int64_t rows, const float* v32,
                     double* ypart, const double* deg, const PeerTable& pt, gpic_ctl* ctl,
                     cudaStream_t s) {
  const int64_t rows_pad = round_up(rows, kTileM);
  if (op.kind == GPIC_KIND_RBF && op.d > 0 && op.d <= 8) {
    const dim3 grid((unsigned)mf_parts(op.n, op.dp), (unsigned)ceil_div(rows, 128));
    if (op.d <= 2)
      mf_simt_kernel<2><<<grid, 256, 0, s>>>(op.xlo, op.dp, op.n, row_lo, rows, rows_pad, op.ns,
                                             v32, ypart, ctl);
    else if (op.d <= 4)
      mf_simt_kernel<4><<<grid, 256, 0, s>>>(op.xlo, op.dp, op.n, row_lo, rows, rows_pad, op.ns,
                                             v32, ypart, ctl);
    else
      mf_simt_kernel<8><<<grid, 256, 0, s>>>(op.xlo, op.dp, op.n, row_lo, rows, rows_pad, op.ns,
                                             v32, ypart, ctl);
    count_launch();
    mf_reduce_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, s>>>(
        ypart, mf_parts(op.n, op.dp), rows_pad, rows, row_lo, deg, pt, ctl);
    count_launch();
    GPIC_CUDA_TRY(cudaGetLastError());
    return GPIC_OK;
  }
  if (mf_sym(op, row_lo, rows)) {
    float* colpart = reinterpret_cast<float*>(ypart + mf_parts(op.n, op.dp) * rows_pad);
    const PruneMask* pm = op.pruned ? &op.prune : nullptr;
    int rc = launch_affinity_tc_matvec(op.xhi, op.xlo, op.sqn, op.n, op.dp, 0, op.n, op.ns, v32,
                                       ypart, rows_pad, ctl, s, op.kind, colpart, pm, op.share_r,
                                       op.share_n);
    if (rc) return rc;
    const int64_t nct = ceil_div(op.n, kTileN);
    const ItemShare sh{pm ? pm->items : nullptr, pm ? pm->item_count : nullptr,
                       pm ? pm->item_wpre : nullptr, op.share_r, op.share_n};
    mf_sym_reduce_kernel<<<(unsigned)nct, 128 * kSeg, 0, s>>>(
        ypart, colpart, mf_parts(op.n, op.dp), rows_pad, op.n, nct,
        mf_rows_per_block(op.dp) / 128, deg, pt, ctl, pm ? pm->item_kept : nullptr,
        pm ? pm->skip : nullptr, pm ? pm->B : 1, pm ? pm->nb : 0, sh);
    count_launch();
    if (pm != nullptr && mf_rebalance_enabled()) {
      rc = launch_mf_rebalance(pm, op.share_r, op.share_n, ctl, s);
      if (rc) return rc;
    }
    GPIC_CUDA_TRY(cudaGetLastError());
    return GPIC_OK;
  }
  int rc = launch_affinity_tc_matvec(op.xhi, op.xlo, op.sqn, op.n, op.dp, row_lo, row_lo + rows,
                                     op.ns, v32, ypart, rows_pad, ctl, s, op.kind);
  if (rc) return rc;
  mf_reduce_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, s>>>(
      ypart, mf_parts(op.n, op.dp), rows_pad, rows, row_lo, deg, pt, ctl);
  count_launch();
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int64_t mf_shard_scratch_bytes(int64_t n, int32_t d) {
  const int32_t dp = feature_pitch(d);
  return round_up(mf_ypart_doubles(n, dp, n) * 8, 256) + round_up(prune_bytes(n, dp), 256) +
         round_up(vector_pitch(n) * 4, 256);
}

PruneMask mf_shard_prune(double* ypart, int64_t n, int32_t d) {
  const int32_t dp = feature_pitch(d);
  uint8_t* p = reinterpret_cast<uint8_t*>(ypart) + round_up(mf_ypart_doubles(n, dp, n) * 8, 256);
  return carve_prune(p, n, dp);
}

// deg[i] = sum_j a_ij for the shard's rows (v = 1 through the same pass).
int launch_mf_degrees(const MfOperands& op, int64_t row_lo, int64_t rows, float* ones,
                      double* ypart, double* deg, cudaStream_t s) {
  const int64_t len = vector_pitch(op.n);
  fill_ones_kernel<<<(unsigned)ceil_div(len, 256), 256, 0, s>>>(ones, op.n, len);
  count_launch();
  PeerTable pt;
  std::memset(&pt, 0, sizeof pt);
  pt.y[0][0] = pt.y[0][1] = deg - row_lo;  // rows land at deg[i - row_lo]
  pt.nranks = 1;
  return launch_mf_matvec(op, row_lo, rows, ones, ypart, nullptr, pt, nullptr, s);
}

}  // namespace gpic
