// Matrix-free power iteration: when 4n^2 bytes of A do not
// fit in HBM (config 5: n = 1M -> 4 TB), every product A v is recomputed
// from X: the tcgen05 affinity engine in matvec mode multiplies each fresh
// exp2 entry by v_j in registers and leaves one fp64 row partial per
// 32-tile column chunk (affinity_tc.cu); this reduce combines the chunk
// partials in fixed order, applies 1/deg and stores the row of y into every
// rank's y buffer (same epilogue contract as the dense GEMV, so the
// tau / normalise / stop tail and the multi-rank exchange are unchanged).
// Degrees are the same pass with v = 1.
#include <cstring>

#include "common.cuh"
#include "ops.h"

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

__global__ void fill_ones_kernel(float* v, int64_t n, int64_t len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < len) v[i] = i < n ? 1.f : 0.f;
}

}  // namespace

int64_t mf_ypart_doubles(int64_t n, int32_t dp, int64_t rows) {
  return mf_parts(n, dp) * round_up(rows, kTileM);
}

int launch_mf_matvec(const MfOperands& op, int64_t row_lo, int64_t rows, const float* v32,
                     double* ypart, const double* deg, const PeerTable& pt, gpic_ctl* ctl,
                     cudaStream_t s) {
  const int64_t rows_pad = round_up(rows, kTileM);
  int rc = launch_affinity_tc_matvec(op.xhi, op.xlo, op.sqn, op.n, op.dp, row_lo, row_lo + rows,
                                     op.ns, v32, ypart, rows_pad, ctl, s, op.kind);
  if (rc) return rc;
  mf_reduce_kernel<<<(unsigned)ceil_div(rows, 256), 256, 0, s>>>(
      ypart, mf_parts(op.n, op.dp), rows_pad, rows, row_lo, deg, pt, ctl);
  count_launch();
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
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
