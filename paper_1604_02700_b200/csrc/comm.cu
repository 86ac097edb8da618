// Multi-rank power iteration, two shard storages.
//
// Packed symmetric shards (GPIC_STORAGE_PACKED): rank r owns 512-row
// super-rows and stores the upper-triangle tiles of its rows; its GEMV
// yields a PARTIAL y (and, once, partial degrees) that it P2P-stores into its
// slot of every rank's region; each rank sums the P slots in rank order
// (slot_combine) before the tail. Deterministic for a given P.
//
// Dense row shards: rank r owns rows [row_lo_r, row_lo_r + rows_r) of A
// (built by gpic_affinity_rbf with that row range; no communication). The
// only exchanges are (1) the degree slices, once, for v0 = d / sum(d), and
// (2) the y slices every iteration. Both are FUSED into the producing kernel: the
// GEMV's epilogue stores each finished row straight into every rank's y
// buffer (NVLink P2P stores through CUDA-IPC mappings of the peers' buffers),
// then its last CTA release-stores an epoch into every rank's flag slot; the
// consumer side is a one-thread acquire-spin kernel in front of the
// (redundant, bitwise-identical on every rank) tau / normalise / stop tail.
// There is no NCCL launch and no host synchronisation per iteration; the
// whole loop is one CUDA graph per rank.
//
// Virtual ranks: the same code with all P shards in one process on one
// device (peer pointers are ordinary device pointers), which is how the
// multi-rank path is exercised on a single GPU: with dense row shards the
// results are bitwise equal to the single-rank run for any P (every
// reduction has a fixed global shape).
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "ops.h"

namespace gpic {
struct gpic_local_t {
  gpic_ctl* ctl;
  double* v64;      // 2n
  float* v32;       // pitch(n)
  double* redpart;  // ceil(n/2048) + 1
  int64_t* lowlist;  // n: isolated rows (lowdeg.cu)
  unsigned long long* lowcount;
};
}  // namespace gpic

struct gpic_comm {
  int nranks = 0;
  int nlocal = 0;
  int rank0 = 0;  // global rank of local shard 0
  int64_t n = 0;
  int32_t max_iter = 0;
  uint8_t* region[gpic::kMaxRanks] = {};  // per rank: y0 | y1 | degf | flags
  bool opened[gpic::kMaxRanks] = {};      // IPC mapping (close) vs own allocation (free)
  uint8_t* priv = nullptr;                // private per-local-shard state
  gpic::gpic_local_t* loc = nullptr;
  uint64_t iter_epoch = 0;
  uint64_t gather_epoch = 0;
  int64_t low_count = 0;  // isolated rows found by the last degree gather
};

namespace gpic {

namespace {

inline int64_t al(int64_t b) { return (b + 255) & ~int64_t(255); }
// per rank: y0 | y1 | degf | flags | slots[kMaxRanks][2] (packed shards'
// y / degree partials, written by their owners, summed by this rank)
inline int64_t region_bytes(int64_t n) {
  return 3 * al(n * 8) + al(kFlagSlots * 8) + 2 * kMaxRanks * al(n * 8);
}
inline double* r_slot(uint8_t* r, int64_t n, int rank, int parity) {
  return reinterpret_cast<double*>(r + 3 * al(n * 8) + al(kFlagSlots * 8) +
                                   (2 * rank + parity) * al(n * 8));
}
inline double* r_y(uint8_t* r, int64_t n, int p) { return reinterpret_cast<double*>(r + p * al(n * 8)); }
inline double* r_deg(uint8_t* r, int64_t n) { return reinterpret_cast<double*>(r + 2 * al(n * 8)); }
inline uint64_t* r_flags(uint8_t* r, int64_t n) {
  return reinterpret_cast<uint64_t*>(r + 3 * al(n * 8));
}
inline int64_t local_bytes(int64_t n) {
  return al(sizeof(gpic_ctl)) + al(2 * n * 8) + al(vector_pitch(n) * 4) +
         al((ceil_div(n, kRedBlock) + 1) * 8) + al(n * 8) + al(8);
}

// Partial-y exchange of the slotted shards: all-to-all (every rank gets
// every partial: P n doubles out per rank per iteration) or reduce-scatter +
// all-gather of the y slices (2 n, one more epoch wait). Same sums in the
// same order either way. GPIC_EXCHANGE=bcast / rs overrides the default
// (reduce-scatter from P = 3, where it moves less).
int reduce_scatter(int nranks) {
  if (const char* e = getenv("GPIC_EXCHANGE")) return strcmp(e, "rs") == 0 ? 1 : 0;
  return nranks >= 3 ? 1 : 0;
}

PeerTable table(const gpic_comm* c, int self) {
  PeerTable pt;
  std::memset(&pt, 0, sizeof pt);
  for (int p = 0; p < c->nranks; ++p) {
    pt.y[p][0] = r_y(c->region[p], c->n, 0);
    pt.y[p][1] = r_y(c->region[p], c->n, 1);
    pt.flags[p] = r_flags(c->region[p], c->n);
  }
  pt.nranks = c->nranks;
  pt.self = self;
  return pt;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Copy this shard's values into every rank's buffer at [row_lo, row_lo +
// rows), then release `epoch` into flag slot kMaxRanks + self of every rank.
// rows may be 0 (pure barrier).
struct PubArgs {
  double* dsts[kMaxRanks];
  uint64_t* flags[kMaxRanks];
};

__global__ void publish_entry(const double* __restrict__ src, int64_t rows, int64_t row_lo,
                              const PubArgs args, int nranks, int self, uint64_t epoch,
                              unsigned int* counter) {
  // thin wrapper so the pointer tables travel by value in the kernel params
  __shared__ double* d[kMaxRanks];
  __shared__ uint64_t* f[kMaxRanks];
  if (threadIdx.x < kMaxRanks) {
    d[threadIdx.x] = args.dsts[threadIdx.x];
    f[threadIdx.x] = args.flags[threadIdx.x];
  }
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = src[i];
    for (int p = 0; p < nranks; ++p) d[p][row_lo + i] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(counter, 1u);
    if (prev == gridDim.x - 1) {
      *counter = 0u;
      __threadfence_system();
      for (int p = 0; p < nranks; ++p) st_release_sys(f[p] + kMaxRanks + self, epoch);
    }
  }
}

__global__ void set_epoch_kernel(gpic_ctl* ctl, uint64_t epoch) {
  if (threadIdx.x == 0) ctl->sync_epoch = epoch;
}

// a matrix-free shard over all rows marked lda = 1: an item shard of the
// pruned sym pass (gpic_mf_shard_build)
bool mf_item_shard(const gpic_shard& sh, int64_t n) {
  return sh.storage == GPIC_STORAGE_NONE && sh.row_lo == 0 && sh.rows == n && sh.lda == 1;
}

LowRows low_rows(const gpic_comm* c, const gpic_shard& sh, int li, int64_t count) {
  LowRows L;
  L.x = sh.x;
  L.n = c->n;
  L.d = sh.d;
  L.kind = sh.kind;
  L.sigma = sh.kind == GPIC_KIND_COSINE ? 1.0 : sh.sigma;
  L.list = c->loc[li].lowlist;
  L.d_count = c->loc[li].lowcount;
  L.count = count;
  return L;
}

int publish(gpic_comm* c, int li, const double* src, int64_t rows, int64_t row_lo,
            uint64_t epoch, cudaStream_t s) {
  PubArgs pa;
  std::memset(&pa, 0, sizeof pa);
  for (int p = 0; p < c->nranks; ++p) {
    pa.dsts[p] = r_deg(c->region[p], c->n);
    pa.flags[p] = r_flags(c->region[p], c->n);
  }
  const int self = c->rank0 + li;
  const int grid = rows > 0 ? (int)std::min<int64_t>(ceil_div(rows, 256), 148) : 1;
  publish_entry<<<grid, 256, 0, s>>>(src, rows, row_lo, pa, c->nranks, self, epoch,
                                     &c->loc[li].ctl->arrive[3]);
  count_launch();
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

// Every local shard publishes (data or a pure barrier), then every local
// shard waits for all P gather epochs.
int gather(gpic_comm* c, const gpic_shard* shards, bool with_data, cudaStream_t s) {
  const uint64_t epoch = ++c->gather_epoch;
  for (int li = 0; li < c->nlocal; ++li) {
    const int64_t rows = with_data ? shards[li].rows : 0;
    int rc = publish(c, li, with_data ? shards[li].deg : nullptr, rows,
                     with_data ? shards[li].row_lo : 0, epoch, s);
    if (rc) return rc;
  }
  for (int li = 0; li < c->nlocal; ++li) {
    const int self = c->rank0 + li;
    launch_peer_wait(r_flags(c->region[self], c->n), kMaxRanks, c->nranks, epoch, 0,
                     c->loc[li].ctl, s);
  }
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

// Packed shards: every local shard publishes its partial degrees (rows
// [row_lo, n)) into its slot (parity 0) of every rank, waits for all P, then
// each rank sums the P partials in rank order into its degf.
int gather_sum(gpic_comm* c, const gpic_shard* shards, cudaStream_t s) {
  const uint64_t epoch = ++c->gather_epoch;
  for (int li = 0; li < c->nlocal; ++li) {
    const int self = c->rank0 + li;
    PubArgs pa;
    std::memset(&pa, 0, sizeof pa);
    for (int p = 0; p < c->nranks; ++p) {
      pa.dsts[p] = r_slot(c->region[p], c->n, self, 0);
      pa.flags[p] = r_flags(c->region[p], c->n);
    }
    const int64_t rows = c->n - shards[li].row_lo;
    const int grid = rows > 0 ? (int)std::min<int64_t>(ceil_div(rows, 256), 148) : 1;
    publish_entry<<<grid, 256, 0, s>>>(shards[li].deg + shards[li].row_lo, rows, shards[li].row_lo,
                                       pa, c->nranks, self, epoch, &c->loc[li].ctl->arrive[3]);
    count_launch();
  }
  for (int li = 0; li < c->nlocal; ++li) {
    const int self = c->rank0 + li;
    launch_peer_wait(r_flags(c->region[self], c->n), kMaxRanks, c->nranks, epoch, 0,
                     c->loc[li].ctl, s);
    const int64_t stride = al(c->n * 8) / 8;
    launch_slot_combine(r_slot(c->region[self], c->n, 0, 0), stride, c->nranks, c->n, nullptr,
                        r_deg(c->region[self], c->n), r_deg(c->region[self], c->n), nullptr, s);
  }
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int alloc_locals(gpic_comm* c) {
  const int64_t lb = local_bytes(c->n);
  GPIC_CUDA_TRY(cudaMalloc(&c->priv, lb * c->nlocal));
  GPIC_CUDA_TRY(cudaMemset(c->priv, 0, lb * c->nlocal));
  c->loc = new gpic_local_t[c->nlocal];
  for (int li = 0; li < c->nlocal; ++li) {
    uint8_t* p = c->priv + li * lb;
    c->loc[li].ctl = reinterpret_cast<gpic_ctl*>(p);
    p += al(sizeof(gpic_ctl));
    c->loc[li].v64 = reinterpret_cast<double*>(p);
    p += al(2 * c->n * 8);
    c->loc[li].v32 = reinterpret_cast<float*>(p);
    p += al(vector_pitch(c->n) * 4);
    c->loc[li].redpart = reinterpret_cast<double*>(p);
    p += al((ceil_div(c->n, kRedBlock) + 1) * 8);
    c->loc[li].lowlist = reinterpret_cast<int64_t*>(p);
    p += al(c->n * 8);
    c->loc[li].lowcount = reinterpret_cast<unsigned long long*>(p);
  }
  return GPIC_OK;
}

}  // namespace
}  // namespace gpic

using namespace gpic;

extern "C" {

int gpic_comm_create(int32_t nranks, int32_t rank, int64_t n, gpic_comm** out,
                     uint8_t* h_ipc_handle) {
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || n < 1 || !out)
    return fail(GPIC_E_INVALID, "bad comm parameters (1 <= nranks <= 8)");
  gpic_comm* c = new gpic_comm;
  c->nranks = nranks;
  c->nlocal = 1;
  c->rank0 = rank;
  c->n = n;
  uint8_t* mine = nullptr;
  cudaError_t e = cudaMalloc(&mine, region_bytes(n));
  if (e != cudaSuccess) {
    delete c;
    return fail_cuda(e, "cudaMalloc(comm region)");
  }
  GPIC_CUDA_TRY(cudaMemset(mine, 0, region_bytes(n)));
  c->region[rank] = mine;
  if (nranks > 1) {
    cudaIpcMemHandle_t h;
    GPIC_CUDA_TRY(cudaIpcGetMemHandle(&h, mine));
    std::memcpy(h_ipc_handle, &h, sizeof h);
  }
  int rc = alloc_locals(c);
  if (rc) return rc;
  GPIC_CUDA_TRY(cudaDeviceSynchronize());
  *out = c;
  return GPIC_OK;
}

int gpic_comm_open(gpic_comm* c, const uint8_t* h_all_handles) {
  for (int p = 0; p < c->nranks; ++p) {
    if (p == c->rank0) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, h_all_handles + p * GPIC_IPC_HANDLE_BYTES, sizeof h);
    void* ptr = nullptr;
    GPIC_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    c->region[p] = static_cast<uint8_t*>(ptr);
    c->opened[p] = true;
  }
  return GPIC_OK;
}

int gpic_comm_create_virtual(int32_t nranks, int64_t n, gpic_comm** out) {
  if (nranks < 1 || nranks > kMaxRanks || n < 1 || !out)
    return fail(GPIC_E_INVALID, "bad comm parameters (1 <= nranks <= 8)");
  gpic_comm* c = new gpic_comm;
  c->nranks = nranks;
  c->nlocal = nranks;
  c->rank0 = 0;
  c->n = n;
  for (int p = 0; p < nranks; ++p) {
    GPIC_CUDA_TRY(cudaMalloc(&c->region[p], region_bytes(n)));
    GPIC_CUDA_TRY(cudaMemset(c->region[p], 0, region_bytes(n)));
  }
  int rc = alloc_locals(c);
  if (rc) return rc;
  GPIC_CUDA_TRY(cudaDeviceSynchronize());
  *out = c;
  return GPIC_OK;
}

int gpic_comm_destroy(gpic_comm* c) {
  if (!c) return GPIC_OK;
  cudaDeviceSynchronize();
  for (int p = 0; p < c->nranks; ++p) {
    if (!c->region[p]) continue;
    if (c->opened[p])
      cudaIpcCloseMemHandle(c->region[p]);
    else
      cudaFree(c->region[p]);
  }
  if (c->priv) cudaFree(c->priv);
  delete[] c->loc;
  delete c;
  return GPIC_OK;
}

int gpic_comm_gather_degrees(gpic_comm* c, const gpic_shard* shards, int32_t nlocal,
                             double* d_deg_full_out, void* stream) {
  if (!c || nlocal != c->nlocal) return fail(GPIC_E_INVALID, "shard count does not match the comm");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int li = 0; li < nlocal; ++li) launch_ctl_init(c->loc[li].ctl, 0.0, 1, s);
  // packed shards and matrix-free item shards hold partial degrees of all
  // rows (summed across ranks); row shards hold complete degrees of theirs
  auto partial = [&](const gpic_shard& sh) {
    return sh.storage == GPIC_STORAGE_PACKED || mf_item_shard(sh, c->n);
  };
  const bool packed = partial(shards[0]);
  for (int li = 1; li < nlocal; ++li)
    if (partial(shards[li]) != packed)
      return fail(GPIC_E_INVALID, "all shards of a comm use the same storage");
  int rc = packed ? gather_sum(c, shards, s) : gather(c, shards, true, s);
  if (rc) return rc;
  // every rank now holds all n degrees: isolated rows (fp32 degree ~ 0) are
  // redone in fp64 from X on every rank (identical results), and ZeroDegree
  // fires only for an exact fp64 zero (lowdeg.cu, affinity.py:113-119)
  for (int li = 0; li < nlocal; ++li)
    launch_lowdeg_scan(r_deg(c->region[c->rank0 + li], c->n), c->n, shards[li].kind,
                       c->loc[li].lowlist, c->loc[li].lowcount, s);
  gpic_ctl h;
  GPIC_CUDA_TRY(cudaMemcpyAsync(&h, c->loc[0].ctl, sizeof h, cudaMemcpyDeviceToHost, s));
  rc = read_low_count(c->loc[0].lowcount, &c->low_count, s);
  if (rc) return rc;
  if (h.status != GPIC_OK) return fail(h.status, "degree gather failed (peer timeout?)");
  if (c->low_count > 0) {
    for (int li = 0; li < nlocal; ++li) {
      if (shards[li].x == nullptr)
        return fail(GPIC_E_INVALID, "isolated rows need the shard's fp64 points (gpic_shard.x)");
      launch_lowdeg_exact(low_rows(c, shards[li], li, c->low_count),
                          r_deg(c->region[c->rank0 + li], c->n), c->loc[li].ctl, s);
    }
    GPIC_CUDA_TRY(cudaMemcpyAsync(&h, c->loc[0].ctl, sizeof h, cudaMemcpyDeviceToHost, s));
    GPIC_CUDA_TRY(cudaStreamSynchronize(s));
    if (h.status == GPIC_E_ZERO_DEGREE) {
      char buf[96];
      snprintf(buf, sizeof buf, "row %lld has zero degree", (long long)h.err_index);
      return fail(GPIC_E_ZERO_DEGREE, buf);
    }
    if (h.status != GPIC_OK) return fail(h.status, "isolated-row degrees failed");
  }
  const double* degf = r_deg(c->region[c->rank0], c->n);
  if (d_deg_full_out)
    GPIC_CUDA_TRY(cudaMemcpyAsync(d_deg_full_out, degf, c->n * 8, cudaMemcpyDeviceToDevice, s));
  return GPIC_OK;
}

int gpic_comm_iterate(gpic_comm* c, const gpic_shard* shards, int32_t nlocal, double eps,
                      int32_t max_iter, const double* d_v0, double* d_hist, double* d_vout,
                      gpic_ctl* h_ctl, void* stream) {
  if (!c || nlocal != c->nlocal) return fail(GPIC_E_INVALID, "shard count does not match the comm");
  if (max_iter < 1) return fail(GPIC_E_INVALID, "max_iterations must be at least 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t n = c->n;
  // start barrier: every rank has finished its previous loop before any
  // rank's GEMV writes into the shared y buffers again
  for (int li = 0; li < nlocal; ++li) launch_ctl_init(c->loc[li].ctl, eps, max_iter, s);
  int rc = gather(c, shards, false, s);
  if (rc) return rc;
  const uint64_t base = c->iter_epoch;
  c->iter_epoch += (uint64_t)max_iter + 1;
  ShardLoop loops[kMaxRanks];
  for (int li = 0; li < nlocal; ++li) {
    const int self = c->rank0 + li;
    gpic_local_t& L = c->loc[li];
    set_epoch_kernel<<<1, 32, 0, s>>>(L.ctl, base);
    count_launch();
    if (d_v0 != nullptr) {
      // explicit start vector (initial_vector, serial.py:77-101), same on every rank
      launch_scale_by(d_v0, n, 1.0, L.v64, L.v32, vector_pitch(n), s);
    } else {
      // v0 = d / tree_sum(d) from the gathered degrees (identical on every rank)
      const double* degf = r_deg(c->region[self], n);
      double* tau = L.redpart + ceil_div(n, kRedBlock);
      launch_tree_sum(degf, n, L.redpart, tau, L.ctl, s);
      launch_scale_vector(degf, n, tau, L.v64, L.v32, vector_pitch(n), s);
    }
    ShardLoop& S = loops[li];
    std::memset(&S, 0, sizeof S);
    S.a = shards[li].a;
    S.lda = shards[li].lda;
    if (shards[li].storage == GPIC_STORAGE_PACKED) {
      // packed shard: its super-rows' tiles; y partials go to every rank's
      // slot of this shard, each rank sums the slots in rank order
      const gpic_shard& sh = shards[li];
      S.mode = kLoopPackedShard;
      const int64_t nt = ceil_div(n, kTileN);
      S.sr.p_lo = sh.row_lo / 512;
      S.sr.p_hi = ceil_div(sh.row_lo + sh.rows, 512);
      S.sr.tile_base = 4 * S.sr.p_lo * nt - 4 * S.sr.p_lo * (4 * S.sr.p_lo - 1) / 2;
      const int64_t ns = ceil_div(nt, 4);
      const int64_t recs = (S.sr.sb_hi(ns) - S.sr.sb_lo(ns)) * 4 * 128;
      S.rowp = reinterpret_cast<float*>(sh.ypart);
      S.colp = S.rowp + ((recs * 4 + 255) / 256) * 64;
      S.pt_slots = table(c, self);
      for (int p = 0; p < c->nranks; ++p)
        for (int par = 0; par < 2; ++par) S.pt_slots.y[p][par] = r_slot(c->region[p], n, self, par);
      S.pt_slots.scatter = reduce_scatter(c->nranks);
      S.slots = r_slot(c->region[self], n, 0, 0);
      S.slot_stride = al(n * 8) / 8;
      S.deg_full = r_deg(c->region[self], n);
      if (sparse_enabled()) {  // the build's box flags and GEMV weights (gpic_packed_shard_build)
        const SparseMask sm = packed_shard_sparse(sh.ypart, n, sh.row_lo, sh.row_lo + sh.rows, sh.d);
        S.boxnz = sm.boxnz;
        S.sb_prefix = sm.sb_prefix;
      }
    }
    if (shards[li].storage == GPIC_STORAGE_NONE) {
      const gpic_shard& sh = shards[li];
      S.mode = kLoopMatrixFree;
      S.mf = MfOperands{sh.xhi, sh.xlo, sh.sqn, n, feature_pitch(sh.d),
                        (float)(-1.4426950408889634 / (2.0 * sh.sigma * sh.sigma)), sh.kind};
      S.mf.d = sh.d;
      S.ypart = sh.ypart;
      if (mf_item_shard(sh, n)) {
        // item shard: this rank's share of the pruned sym pass; partial y
        // over all rows into every rank's slot, summed in rank order
        S.mode = kLoopMfShard;
        S.mf.sym = 1;
        S.mf.pruned = 1;
        S.mf.prune = mf_shard_prune(sh.ypart, n, sh.d);
        S.mf.share_r = self;
        S.mf.share_n = c->nranks;
        S.pt_slots = table(c, self);
        for (int p = 0; p < c->nranks; ++p)
          for (int par = 0; par < 2; ++par) S.pt_slots.y[p][par] = r_slot(c->region[p], n, self, par);
        S.pt_slots.scatter = reduce_scatter(c->nranks);
        S.slots = r_slot(c->region[self], n, 0, 0);
        S.slot_stride = al(n * 8) / 8;
        S.deg_full = r_deg(c->region[self], n);
      }
    }
    S.rows = shards[li].rows;
    S.row_lo = shards[li].row_lo;
    S.deg = shards[li].deg;
    S.redpart = L.redpart;
    S.v64 = L.v64;
    S.v32 = L.v32;
    S.hist = d_hist + (int64_t)li * max_iter;
    S.ctl = L.ctl;
    S.pt = table(c, self);
    S.low = low_rows(c, shards[li], li, c->low_count);
    S.low_deg = r_deg(c->region[self], n);
  }
  rc = run_power_loops(loops, nlocal, n, max_iter, s);
  if (rc) return rc;
  for (int li = 0; li < nlocal; ++li) {
    launch_copy_result(c->loc[li].v64, n, d_vout + (int64_t)li * n, c->loc[li].ctl, s);
    GPIC_CUDA_TRY(cudaMemcpyAsync(h_ctl + li, c->loc[li].ctl, sizeof(gpic_ctl),
                                  cudaMemcpyDeviceToHost, s));
  }
  GPIC_CUDA_TRY(cudaStreamSynchronize(s));
  note_loop_iterations(h_ctl[0].iter);
  for (int li = 0; li < nlocal; ++li)
    if (h_ctl[li].status != GPIC_OK) return h_ctl[li].status;
  return GPIC_OK;
}

}  // extern "C"
