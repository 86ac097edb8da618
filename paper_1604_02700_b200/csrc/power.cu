// Stage 2/3: start vector and the device-resident power iteration.
//
// Reference loop (serial.py:120-127, parallel.py:374-382):
//     wv = W v ; v' = wv / sum(wv) ; delta = max|v' - v| ;
//     stop when len(deltas) >= 2 and |delta_t - delta_(t-1)| <= eps
//
// Per iteration, three kernels, all no-ops once ctl->stop is set so a whole
// max_iterations loop can be replayed from one CUDA graph with no host
// synchronisation:
//   gemv (gemv.cu) y_i = (sum_j A_ij v_j) / deg_i       HBM-bound, 4n^2 bytes
//   tau_kernel    tau = fixed-shape sum of y             (k_reduce, parallel.py:161-178)
//   norm_kernel   v' = y / tau, delta = max|v' - v|, history, stop test
// (in the loop both run as one tail_kernel with an in-kernel grid barrier)
// Every reduction has a fixed shape over GLOBAL indices, so results are
// bitwise independent of how rows are sharded across ranks.
#include <cfloat>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ops.h"
#include "lowdeg.cuh"
#include "tail.cuh"

namespace gpic {

namespace {

using tail::kRedThreads;
using tail::kRedPer;
using tail::block_sum_fixed;
using tail::block_max;

// Sum of v[0, n) into *out (and ctl->tau when ctl != null). `guarded` skips
// when ctl->stop is set (loop mode).
__global__ void __launch_bounds__(kRedThreads)
    tau_kernel(const double* __restrict__ v0, const double* __restrict__ v1, int64_t n,
               double* __restrict__ part, double* __restrict__ out, gpic_ctl* ctl, int guarded) {
  __shared__ double sh[kRedThreads];
  if (guarded && *(volatile int32_t*)&ctl->stop) return;
  // loop mode: the y buffer of this iteration (parity ping-pong)
  const double* __restrict__ v = (guarded && (ctl->iter & 1)) ? v1 : v0;
  const int64_t b0 = (int64_t)blockIdx.x * kRedBlock;
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < kRedPer; ++q) {
    const int64_t i = b0 + threadIdx.x + q * kRedThreads;
    if (i < n) s += v[i];
  }
  s = block_sum_fixed(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (!last_block_done(&ctl->arrive[0])) return;
  // last block: fixed pattern over the partials
  const int64_t nb = gridDim.x;
  double t = 0.0;
  for (int64_t i = threadIdx.x; i < nb; i += kRedThreads) t += part[i];
  t = block_sum_fixed(t, sh);
  if (threadIdx.x == 0) {
    ctl->arrive[0] = 0u;
    if (out) *out = t;
    ctl->tau = t;
    if (guarded && !(t > 0.0)) raise_status(ctl, GPIC_E_NONPOS_TAU, 0, -1, t);
  }
}

// v' = y / tau ; delta = max|v' - v| ; last block records the history and
// applies the stop rule.
__global__ void __launch_bounds__(kRedThreads)
    norm_kernel(const double* __restrict__ y0, const double* __restrict__ y1, int64_t n,
                double* __restrict__ v64, float* __restrict__ v32, double* __restrict__ hist,
                gpic_ctl* ctl) {
  __shared__ double sh[kRedThreads];
  if (*(volatile int32_t*)&ctl->stop) return;
  const int t = ctl->iter;
  const double* __restrict__ y = (t & 1) ? y1 : y0;
  const double tau = ctl->tau;
  const double* __restrict__ vold = v64 + (int64_t)(t & 1) * n;
  double* __restrict__ vnew = v64 + (int64_t)((t + 1) & 1) * n;
  const int64_t b0 = (int64_t)blockIdx.x * kRedBlock;
  double m = 0.0;
#pragma unroll
  for (int q = 0; q < kRedPer; ++q) {
    const int64_t i = b0 + threadIdx.x + q * kRedThreads;
    if (i < n) {
      const double vn = y[i] / tau;
      m = fmax(m, fabs(vn - vold[i]));
      vnew[i] = vn;
      v32[i] = (float)vn;
    }
  }
  m = block_max(m, sh);
  if (threadIdx.x == 0)
    atomicMax(reinterpret_cast<unsigned long long*>(&ctl->delta_bits),
              (unsigned long long)__double_as_longlong(m));
  if (!last_block_done(&ctl->arrive[1])) return;
  if (threadIdx.x == 0) {
    const double delta = __longlong_as_double((long long)ctl->delta_bits);
    hist[t] = delta;
    ctl->delta_bits = 0ull;
    ctl->arrive[1] = 0u;
    const int done = t + 1;
    ctl->iter = done;
    if (done >= 2 && fabs(delta - hist[t - 1]) <= ctl->eps) {
      ctl->converged = 1;
      ctl->stop = 1;
    } else if (done >= ctl->max_iter) {
      ctl->stop = 1;
    }
  }
}

// tau_kernel + norm_kernel in one launch (loop mode): tail.cuh.
// Low-degree rows (lowdeg.cuh; listed by the device-side count low.d_count,
// null: none): their fp64 y_i are computed here first, one CTA per listed
// row as lowdeg_row_kernel does (bitwise the same), then a grid barrier.
__global__ void __launch_bounds__(kRedThreads)
    tail_kernel(double* y0, double* y1, int64_t n, double* __restrict__ part,
                double* __restrict__ v64, float* __restrict__ v32, double* __restrict__ hist,
                gpic_ctl* ctl, int tau_mode, LowRows low, const double* __restrict__ low_deg,
                double low_scale) {
  __shared__ double sh[kRedThreads];
  extern __shared__ double xs[];
  if (*(volatile int32_t*)&ctl->stop) return;
  const int t = ctl->iter;
  double* y = (t & 1) ? y1 : y0;
  const unsigned long long cnt = low.d_count != nullptr ? *low.d_count : 0ull;
  if (tau_mode == kTailTauAlways || (tau_mode == kTailTauIfNoLow && cnt == 0ull)) {
    // the reduce stored this iteration's tau (tail.cuh tau_in_reduce)
    tail::normalise<false>(y, n, v64, v32, hist, ctl, t, *(volatile double*)&ctl->tau, sh,
                           gridDim.x);
    return;
  }
  const unsigned gen0 = *(volatile unsigned*)&ctl->tau_gen;  // read before arriving
  if (cnt == 0ull) {
    tail::chunk_sums<false>(y, n, part, sh, gridDim.x);
    tail::finish<false>(y, n, part, v64, v32, hist, ctl, t, gen0, sh, gridDim.x);
    return;
  }
  const unsigned bgen = *(volatile unsigned*)&ctl->bar_gen;
  const double* v = v64 + (int64_t)(t & 1) * n;
  for (unsigned long long r = blockIdx.x; r < cnt; r += gridDim.x) {
    const int64_t i = low.list[r];
    const double s = lowdeg::matvec_row(low.x, n, low.d, low.kind, low_scale, i, low_deg[i], v, xs,
                                        sh);
    if (threadIdx.x == 0) y[i] = s;
  }
  tail::grid_barrier(ctl, bgen);
  tail::chunk_sums<true>(y, n, part, sh, gridDim.x);
  tail::finish<true>(y, n, part, v64, v32, hist, ctl, t, gen0, sh, gridDim.x);
}

// src / tau[0] -> fp64 + fp32 copies (start vector: k_norm(deg, k_reduce(deg))).
__global__ void scale_kernel(const double* __restrict__ src, int64_t n,
                             const double* __restrict__ tau, double* __restrict__ v64,
                             float* __restrict__ v32, int64_t v32_len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v32_len) return;
  if (i < n) {
    const double v = src[i] / tau[0];
    v64[i] = v;
    v32[i] = (float)v;
  } else {
    v32[i] = 0.f;
  }
}

__global__ void scale_by_kernel(const double* __restrict__ src, int64_t n, double tau,
                                double* __restrict__ dst, float* __restrict__ dst32,
                                int64_t f32_len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const double v = src[i] / tau;
    dst[i] = v;
    if (dst32) dst32[i] = (float)v;
  } else if (dst32 && i < f32_len) {
    dst32[i] = 0.f;
  }
}

// Acquire-spin until flags[slot0 .. slot0+count) all reach base (+ iter + 1
// when add_iter). A peer that never arrives (dead rank) trips the timeout
// (launch_peer_wait): the run stops with GPIC_E_COMM instead of hanging.
__global__ void peer_wait_kernel(const uint64_t* flags, int slot0, int count, uint64_t base,
                                 int add_iter, gpic_ctl* ctl, uint64_t timeout_ns) {
  if (threadIdx.x != 0) return;
  if (add_iter && *(volatile int32_t*)&ctl->stop) return;
  // loop mode: the epoch base lives in the control block so one captured
  // graph serves every run; gather mode: an explicit target
  const uint64_t target = add_iter ? ctl->sync_epoch + (uint64_t)ctl->iter + 1 : base;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int s = 0; s < count; ++s) {
    for (;;) {
      uint64_t v;
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + slot0 + s) : "memory");
      if (v >= target) break;
      uint64_t now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > timeout_ns) {
        raise_status(ctl, GPIC_E_COMM, slot0 + s, -1, 0.0);
        return;
      }
      __nanosleep(64);
    }
  }
  __threadfence_system();
}

__global__ void copy_result_kernel(const double* __restrict__ v64, int64_t n,
                                   double* __restrict__ out, const gpic_ctl* __restrict__ ctl) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = v64[(int64_t)(ctl->iter & 1) * n + i];
}

}  // namespace

void launch_tree_sum(const double* v, int64_t n, double* part, double* out, gpic_ctl* ctl,
                     cudaStream_t s) {
  tau_kernel<<<(unsigned)ceil_div(n, kRedBlock), kRedThreads, 0, s>>>(v, v, n, part, out, ctl, 0);
  count_launch();
}

void launch_scale_vector(const double* src, int64_t n, const double* tau, double* v64,
                         float* v32, int64_t v32_len, cudaStream_t s) {
  scale_kernel<<<(unsigned)ceil_div(v32_len, 256), 256, 0, s>>>(src, n, tau, v64, v32, v32_len);
  count_launch();
}

void launch_scale_by(const double* src, int64_t n, double tau, double* dst, float* dst32,
                     int64_t f32_len, cudaStream_t s) {
  const int64_t m = dst32 ? (f32_len > n ? f32_len : n) : n;
  scale_by_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, s>>>(src, n, tau, dst, dst32, f32_len);
  count_launch();
}

namespace {
__global__ void slot_combine_kernel(const double* __restrict__ slots, int64_t stride, int nranks,
                                    int64_t n, const double* __restrict__ deg, double* y0,
                                    double* y1, gpic_ctl* ctl) {
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double t = 0.0;
  for (int r = 0; r < nranks; ++r) t += slots[(2 * r + parity) * stride + i];
  (parity ? y1 : y0)[i] = deg != nullptr ? t / deg[i] : t;
}
}  // namespace

namespace {
__device__ __forceinline__ void st_release_sys64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// reduce-scatter exchange, second half: this rank's slice of y from the P
// partial slots (rank order, as slot_combine) stored into every rank's y;
// the last CTA publishes the all-gather epoch (flag slots [2P, 3P))
__global__ void slice_combine_kernel(const double* __restrict__ slots, int64_t stride, int64_t n,
                                     const double* __restrict__ deg, const PeerTable pt,
                                     gpic_ctl* ctl) {
  if (*(volatile const int32_t*)&ctl->stop) return;
  const int parity = ctl->iter & 1;
  const int64_t lo = slice_lo(n, pt.self, pt.nranks), hi = slice_lo(n, pt.self + 1, pt.nranks);
  const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < hi) {
    double t = 0.0;
    for (int r = 0; r < pt.nranks; ++r) t += slots[(2 * r + parity) * stride + i];
    const double val = deg != nullptr ? t / deg[i] : t;
    for (int r = 0; r < pt.nranks; ++r) pt.y[r][parity][i] = val;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&ctl->arrive[3], 1u);
    if (prev == gridDim.x - 1) {
      ctl->arrive[3] = 0u;
      __threadfence_system();
      const uint64_t epoch = ctl->sync_epoch + (uint64_t)ctl->iter + 1;
      for (int r = 0; r < pt.nranks; ++r)
        st_release_sys64(pt.flags[r] + 2 * kMaxRanks + pt.self, epoch);
    }
  }
}
}  // namespace

void launch_slice_combine(const double* slots, int64_t stride, int64_t n, const double* deg,
                          const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s) {
  const int64_t rows = slice_lo(n, pt.self + 1, pt.nranks) - slice_lo(n, pt.self, pt.nranks);
  const unsigned grid = (unsigned)(rows > 0 ? ceil_div(rows, 256) : 1);
  slice_combine_kernel<<<grid, 256, 0, s>>>(slots, stride, n, deg, pt, ctl);
  count_launch();
}

void launch_slot_combine(const double* slots, int64_t stride, int nranks, int64_t n,
                         const double* deg, double* y0, double* y1, gpic_ctl* ctl, cudaStream_t s) {
  slot_combine_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(slots, stride, nranks, n, deg, y0,
                                                                 y1, ctl);
  count_launch();
}

void launch_iteration_tail(double* y0, double* y1, int64_t n, double* redpart, double* v64,
                           float* v32, double* hist, gpic_ctl* ctl, cudaStream_t s, int tau_mode,
                           const LowRows& low, const double* low_deg) {
  const unsigned nb = (unsigned)ceil_div(n, kRedBlock);
  static const bool split = [] {
    const char* e = getenv("GPIC_TAIL_SPLIT");  // 1: the two-kernel tail (A/B)
    return e != nullptr && atoi(e) != 0;
  }();
  if (split) {
    if (low.count != 0) launch_lowdeg_matvec(low, low_deg, v64, y0, y1, ctl, s);
    tau_kernel<<<nb, kRedThreads, 0, s>>>(y0, y1, n, redpart, nullptr, ctl, 1);
    norm_kernel<<<nb, kRedThreads, 0, s>>>(y0, y1, n, v64, v32, hist, ctl);
    count_launch(2);
    return;
  }
  static const unsigned sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return (unsigned)v;
  }();
  LowRows lr = low;
  if (low.count == 0) lr.d_count = nullptr;  // no listed row
  const size_t dyn = lr.d_count != nullptr && low.d <= lowdeg::kSmemD ? (size_t)low.d * 8 : 0;
  tail_kernel<<<nb < sms ? nb : sms, kRedThreads, dyn, s>>>(
      y0, y1, n, redpart, v64, v32, hist, ctl, tau_mode, lr, low_deg,
      -1.0 / (2.0 * low.sigma * low.sigma));
  count_launch();
}

// Timeouts: a per-iteration wait (add_iter) covers one GEMV of the slowest
// rank, GPIC_PEER_TIMEOUT_S (default 10 s); barrier / gather waits also cover
// skew between ranks (graph instantiation, a slow host, a large shard
// build): 12x that (default 120 s).
void launch_peer_wait(const uint64_t* flags_self, int slot0, int count, uint64_t base,
                      int add_iter, gpic_ctl* ctl, cudaStream_t s) {
  double secs = 10.0;
  if (const char* e = getenv("GPIC_PEER_TIMEOUT_S"))
    if (atof(e) > 0.0) secs = atof(e);
  if (!add_iter) secs *= 12.0;
  peer_wait_kernel<<<1, 32, 0, s>>>(flags_self, slot0, count, base, add_iter, ctl,
                                    (uint64_t)(secs * 1e9));
  count_launch();
}

void launch_copy_result(const double* v64, int64_t n, double* out, const gpic_ctl* ctl,
                        cudaStream_t s) {
  copy_result_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(v64, n, out, ctl);
  count_launch();
}

namespace {

// Instantiated loop graphs, keyed by everything that is baked into them.
struct GraphKey {
  ShardLoop shards[kMaxRanks];
  int nlocal;
  int64_t n;
  int32_t max_iter;
  int device;
  bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof(GraphKey)) == 0; }
};
struct GraphEntry {
  GraphKey key;
  cudaGraphExec_t exec;
  unsigned long long launches;
  bool unrolled;
};
std::vector<GraphEntry> g_graphs;
constexpr size_t kGraphCache = 8;

}  // namespace

namespace {
// WHILE-node condition: another iteration unless the stop rule fired
__global__ void loop_cond_kernel(cudaGraphConditionalHandle h, const gpic_ctl* ctl) {
  cudaGraphSetConditional(h, *(volatile const int32_t*)&ctl->stop ? 0u : 1u);
}
}  // namespace

unsigned long long g_loop_per_iter = 0;  // kernels of one iteration of the last loop graph
void note_loop_iterations(int32_t iters) { g_launches += (unsigned long long)iters * g_loop_per_iter; }

// The whole loop as one CUDA graph: a conditional WHILE node whose body is
// one iteration — every local shard's GEMV (+ fused peer stores / epoch
// publish), then every local shard's [peer wait] + tau + normalise — and a
// one-thread kernel that sets the condition from the stop flag. The device
// decides when to stop; the graph replays no idle iterations (before:
// max_iter unrolled copies whose kernels exited at once, ~14 us per
// iteration of launch overhead after convergence).
int run_power_loops(ShardLoop* shards, int nlocal, int64_t n, int32_t max_iter, cudaStream_t s) {
  if (nlocal < 1 || nlocal > kMaxRanks) return fail(GPIC_E_INVALID, "bad local shard count");
  GraphKey key;
  std::memset(&key, 0, sizeof key);
  for (int i = 0; i < nlocal; ++i) key.shards[i] = shards[i];
  key.nlocal = nlocal;
  key.n = n;
  key.max_iter = max_iter;
  GPIC_CUDA_TRY(cudaGetDevice(&key.device));
  cudaStream_t cs = s;
  bool own = false;
  if (cs == nullptr || cs == cudaStreamLegacy || cs == cudaStreamPerThread) {
    GPIC_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    own = true;
    cudaEvent_t ev;  // order the private stream after the caller's work
    GPIC_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    GPIC_CUDA_TRY(cudaEventRecord(ev, s));
    GPIC_CUDA_TRY(cudaStreamWaitEvent(cs, ev, 0));
    GPIC_CUDA_TRY(cudaEventDestroy(ev));
  }
  GraphEntry* hit = nullptr;
  for (auto& e : g_graphs)
    if (e.key == key) hit = &e;
  if (hit == nullptr) {
    gemv_prepare();
    sym_prepare();
    cudaGraph_t graph;
    GraphEntry ent;
    ent.key = key;
    const unsigned long long before = g_launches;
    // GPIC_LOOP_UNROLLED=1: max_iter unrolled copies instead of the WHILE
    // node (Nsight Compute does not trace kernels inside conditional graph
    // bodies; the profiling scripts use this for the launch list)
    const bool unrolled = getenv("GPIC_LOOP_UNROLLED") != nullptr;
    GPIC_CUDA_TRY(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond{};
    cudaGraph_t body = graph;
    if (!unrolled) {
      GPIC_CUDA_TRY(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
      cudaGraphNodeParams cp = {};
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = cond;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      cudaGraphNode_t loop_node;
      GPIC_CUDA_TRY(cudaGraphAddNode(&loop_node, graph, nullptr, 0, &cp));
      body = cp.conditional.phGraph_out[0];
    }
    GPIC_CUDA_TRY(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                                cudaStreamCaptureModeThreadLocal));
    for (int t = 0; t < (unrolled ? max_iter : 1); ++t) {
      // packed whole-matrix rank: reduce + low rows + tail fused into one
      // kernel after the GEMV (sym.cu sym_iter_tail_kernel)
      int took[kMaxRanks] = {};  // what the GEMV launch took over (ops.h kTail*)
      for (int i = 0; i < nlocal; ++i) {
        const ShardLoop& L = shards[i];
        IterTail it;
        it.y0 = L.pt.y[L.pt.self][0];
        it.y1 = L.pt.y[L.pt.self][1];
        it.redpart = L.redpart;
        it.v64 = L.v64;
        it.v32 = L.v32;
        it.hist = L.hist;
        it.low = L.low;
        if (L.low.count == 0) it.low.d_count = nullptr;
        it.low_deg = L.low_deg;
        const IterTail* itp = nlocal == 1 ? &it : nullptr;
        if (L.mode == kLoopPacked) {
          took[i] = launch_sym_gemv(L.a, n, L.v32, L.rowp, L.colp, L.deg, L.pt, L.ctl, cs,
                                     ShardRange(), L.boxnz, L.sb_prefix, itp);
        } else if (L.mode == kLoopPacked16) {
          took[i] = launch_sym_gemv16(L.a, n, L.v32, L.rowp, L.colp, L.deg, L.pt, L.ctl, cs,
                                       L.boxnz, L.sb_prefix, itp);
        } else if (L.mode == kLoopPackedShard) {
          // partial y over the shard's tiles into every rank's slot of this shard
          launch_sym_gemv(L.a, n, L.v32, L.rowp, L.colp, nullptr, L.pt_slots, L.ctl, cs, L.sr,
                          L.boxnz, L.sb_prefix);
        } else if (L.mode == kLoopMatrixFree || L.mode == kLoopMfShard) {
          // item shard: partial y (no 1/deg) into every rank's slot of this shard
          const bool item = L.mode == kLoopMfShard;
          const int rc = launch_mf_matvec(L.mf, L.row_lo, L.rows, L.v32, L.ypart,
                                          item ? nullptr : L.deg, item ? L.pt_slots : L.pt,
                                          L.ctl, cs);
          if (rc) {
            cudaGraph_t junk;
            cudaStreamEndCapture(cs, &junk);
            cudaGraphDestroy(graph);
            return rc;
          }
        } else {
          launch_gemv(L.a, L.lda, L.rows, L.row_lo, L.v32, L.deg, L.pt, L.ctl, cs);
        }
      }
      // reduce-scatter shards: every local shard's slice combine (and its
      // all-gather stores) before any shard waits for the all-gather —
      // virtual ranks share one stream
      for (int i = 0; i < nlocal; ++i) {
        const ShardLoop& L = shards[i];
        const PeerTable& pt = L.pt;
        if (!(L.mode == kLoopPackedShard || L.mode == kLoopMfShard) || !L.pt_slots.scatter)
          continue;
        launch_peer_wait(pt.flags[pt.self], 0, pt.nranks, 0, 1, L.ctl, cs);
        launch_slice_combine(L.slots, L.slot_stride, n, L.deg_full, pt, L.ctl, cs);
      }
      for (int i = 0; i < nlocal; ++i) {
        if (took[i] == kTailFused) continue;
        const ShardLoop& L = shards[i];
        const PeerTable& pt = L.pt;
        const bool slotted = L.mode == kLoopPackedShard || L.mode == kLoopMfShard;
        if (slotted && L.pt_slots.scatter) {
          launch_peer_wait(pt.flags[pt.self], 2 * kMaxRanks, pt.nranks, 0, 1, L.ctl, cs);
        } else {
          if (pt.flags[0] != nullptr)
            launch_peer_wait(pt.flags[pt.self], 0, pt.nranks, 0, 1, L.ctl, cs);
          if (slotted)
            launch_slot_combine(L.slots, L.slot_stride, pt.nranks, n, L.deg_full,
                                pt.y[pt.self][0], pt.y[pt.self][1], L.ctl, cs);
        }
        // the low-degree rows' y (count < 0: on the device) inside the tail
        launch_iteration_tail(pt.y[pt.self][0], pt.y[pt.self][1], n, L.redpart, L.v64, L.v32,
                              L.hist, L.ctl, cs, took[i], L.low, L.low_deg);
      }
    }
    if (!unrolled) {
      loop_cond_kernel<<<1, 1, 0, cs>>>(cond, shards[nlocal - 1].ctl);
      count_launch();
    }
    cudaGraph_t captured;
    GPIC_CUDA_TRY(cudaStreamEndCapture(cs, &captured));
    GPIC_CUDA_TRY(cudaGraphInstantiate(&ent.exec, graph, 0));
    GPIC_CUDA_TRY(cudaGraphDestroy(graph));
    ent.launches = g_launches - before;
    ent.unrolled = unrolled;
    g_launches = before;
    if (g_graphs.size() >= kGraphCache) {
      cudaGraphExecDestroy(g_graphs.front().exec);
      g_graphs.erase(g_graphs.begin());
    }
    g_graphs.push_back(ent);
    hit = &g_graphs.back();
  }
  GPIC_CUDA_TRY(cudaGraphLaunch(hit->exec, cs));
  if (hit->unrolled) {
    g_launches += hit->launches;
    g_loop_per_iter = 0;
  } else {
    g_loop_per_iter = hit->launches;  // callers add iterations x this once they know the count
  }
  if (own) {
    cudaEvent_t ev;
    GPIC_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    GPIC_CUDA_TRY(cudaEventRecord(ev, cs));
    GPIC_CUDA_TRY(cudaStreamWaitEvent(s, ev, 0));
    GPIC_CUDA_TRY(cudaEventDestroy(ev));
    GPIC_CUDA_TRY(cudaStreamDestroy(cs));
  }
  return GPIC_OK;
}

int run_power_loop(const float* a, int64_t lda, const double* deg, int64_t n, double* y,
                   double* redpart, double* v64, float* v32, double* hist, gpic_ctl* ctl,
                   int32_t max_iter, cudaStream_t s) {
  ShardLoop L;
  std::memset(&L, 0, sizeof L);
  L.a = a;
  L.lda = lda;
  L.rows = n;
  L.row_lo = 0;
  L.deg = deg;
  L.redpart = redpart;
  L.v64 = v64;
  L.v32 = v32;
  L.hist = hist;
  L.ctl = ctl;
  L.pt.y[0][0] = y;
  L.pt.y[0][1] = y;
  L.pt.nranks = 1;
  L.pt.self = 0;
  return run_power_loops(&L, 1, n, max_iter, s);
}

}  // namespace gpic
