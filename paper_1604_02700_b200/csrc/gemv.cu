// Power-iteration GEMV: y_i = (sum_j A_ij v_j) / deg_i  (k_multiply,
// parallel.py:196-207, with k_normalize's D^-1 folded into the epilogue).
//
// HBM-bound: every iteration streams the whole fp32 A block (4 * rows * n
// bytes) once. Persistent CTAs (one per SM); a producer lane feeds a 3-stage
// smem ring with 1-D bulk copies (cp.async.bulk, completion on mbarriers):
// per stage, a 1024-column chunk of 16 rows plus the matching chunk of v
// (68 KB). ~200 KB per SM are in flight without tying up registers, which is
// what keeps HBM saturated; 8 consumer warps (2 rows each) read the stage
// with conflict-free 128-bit shared loads. Per-row sums are accumulated in
// fp32 within a chunk and in fp64 across chunks, then reduced across lanes
// by a fixed butterfly: the result for a row depends only on that row, not
// on the shard plan.
#include "common.cuh"
#include "ops.h"
#include "sm100.cuh"

namespace gpic {

namespace {

constexpr int kRG = 16;          // rows per group
constexpr int kCW = 1024;        // columns per chunk
constexpr int kStages = 3;
constexpr int kConsumers = 8;    // warps, kRG / kConsumers rows each
constexpr int kRowsPerWarp = kRG / kConsumers;
constexpr int kThreads = (kConsumers + 1) * 32;
constexpr int kStageFloats = (kRG + 1) * kCW;
constexpr int kSmem = kStages * kStageFloats * 4 + 64 + 128;

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    gemv_bulk_kernel(const float* __restrict__ a, int64_t lda, int64_t rows, int64_t row_lo,
                     const float* __restrict__ v32, const double* __restrict__ deg,
                     const PeerTable pt, gpic_ctl* ctl) {
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
  extern __shared__ uint8_t smem_raw[];
  float* st = reinterpret_cast<float*>(smem_align<128>(smem_raw));
  uint64_t* full = reinterpret_cast<uint64_t*>(st + kStages * kStageFloats);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t groups = (rows + kRG - 1) / kRG;
  const int64_t nchunks = (lda + kCW - 1) / kCW;

  if (warp == kConsumers) {
    if (lane != 0) return;
    int s = 0;
    uint32_t ph = 0;
    const uint64_t once = policy_evict_first(), keep = policy_evict_last();
    for (int64_t g = blockIdx.x; g < groups; g += gridDim.x) {
      const int64_t r0 = g * kRG;
      const int nr = (int)min((int64_t)kRG, rows - r0);
      for (int64_t ch = 0; ch < nchunks; ++ch) {
        const int64_t c0 = ch * kCW;
        const uint32_t cw = (uint32_t)min((int64_t)kCW, lda - c0);
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], (uint32_t)(nr + 1) * cw * 4u);
        float* dst = st + s * kStageFloats;
        bulk_load(dst + kRG * kCW, v32 + c0, cw * 4u, &full[s], keep);
        for (int r = 0; r < nr; ++r)
          bulk_load(dst + r * kCW, a + (r0 + r) * lda + c0, cw * 4u, &full[s], once);
        if (++s == kStages) { s = 0; ph ^= 1; }
      }
    }
    return;
  }

  int s = 0;
  uint32_t ph = 0;
  for (int64_t g = blockIdx.x; g < groups; g += gridDim.x) {
    const int64_t r0 = g * kRG;
    double acc64[kRowsPerWarp];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) acc64[r] = 0.0;
    for (int64_t ch = 0; ch < nchunks; ++ch) {
      const int cw4 = (int)(min((int64_t)kCW, lda - ch * kCW) >> 2);
      mbar_wait(&full[s], ph);
      const float* base = st + s * kStageFloats;
      const float4* vv = reinterpret_cast<const float4*>(base + kRG * kCW);
      float acc[kRowsPerWarp];
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) acc[r] = 0.f;
#pragma unroll 4
      for (int f = lane; f < cw4; f += 32) {
        const float4 x = vv[f];
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; ++r) {
          const float4 w =
              reinterpret_cast<const float4*>(base + (warp * kRowsPerWarp + r) * kCW)[f];
          acc[r] = fmaf(w.x, x.x, acc[r]);
          acc[r] = fmaf(w.y, x.y, acc[r]);
          acc[r] = fmaf(w.z, x.z, acc[r]);
          acc[r] = fmaf(w.w, x.w, acc[r]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == kStages) { s = 0; ph ^= 1; }
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) acc64[r] += (double)acc[r];
    }
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) {
      const double sum = warp_sum_f64(acc64[r]);
      const int64_t li = r0 + warp * kRowsPerWarp + r;
      if (lane == 0 && li < rows) {
        const double val = deg != nullptr ? sum / deg[li] : sum;
        // fused all-gather: the row lands in every rank's y (P2P over NVLink)
        for (int p = 0; p < pt.nranks; ++p) pt.y[p][parity][row_lo + li] = val;
      }
    }
  }
  if (pt.flags[0] == nullptr) return;
  // publish: after every consumer of every CTA stored its rows, release the
  // epoch into each rank's flag slot for this shard
  __threadfence_system();
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers * 32) : "memory");
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

// check_row_stochastic (serial.py:63-74) on an fp64 matrix: per-row sum,
// min and max, one warp per row (coalesced lane-strided reads, fixed
// butterfly, so a row's result depends only on that row). NaN propagates
// into all three, as numpy's sum/min/max would.
__global__ void __launch_bounds__(256) row_stats_kernel(const double* __restrict__ w,
                                                        int64_t rows, int64_t n, int64_t ldw,
                                                        double* sum, double* mn, double* mx) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const double* r = w + row * ldw;
  double s = 0.0, lo = INFINITY, hi = -INFINITY;
  for (int64_t j = lane; j < n; j += 32) {
    const double x = __ldcs(r + j);
    s += x;
    lo = (x < lo || x != x) ? x : lo;
    hi = (x > hi || x != x) ? x : hi;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = (l2 < lo || l2 != l2) ? l2 : lo;
    hi = (h2 > hi || h2 != h2) ? h2 : hi;
  }
  if (lane == 0) {
    sum[row] = s;
    mn[row] = lo;
    mx[row] = hi;
  }
}

}  // namespace

static int g_num_sms = 0;

// One-time attribute setup; called before any stream capture.
void gemv_prepare() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(gemv_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  }
}

void launch_gemv(const float* a, int64_t lda, int64_t rows, int64_t row_lo, const float* v32,
                 const double* deg, const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s) {
  gemv_prepare();
  const int num_sms = g_num_sms;
  const int64_t groups = (rows + kRG - 1) / kRG;
  const int grid = (int)(groups < num_sms ? groups : num_sms);
  gemv_bulk_kernel<<<grid, kThreads, kSmem, s>>>(a, lda, rows, row_lo, v32, deg, pt, ctl);
  count_launch();
}

void launch_row_stats(const double* w, int64_t rows, int64_t n, int64_t ldw, double* sum,
                      double* mn, double* mx, cudaStream_t s) {
  const int64_t grid = (rows + 7) / 8;
  row_stats_kernel<<<(unsigned)grid, 256, 0, s>>>(w, rows, n, ldw, sum, mn, mx);
  count_launch();
}

}  // namespace gpic
