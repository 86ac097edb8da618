// Internal host-side launchers shared between the translation units of
// libgpic. Everything here is asynchronous on `stream`.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gpic.h"

namespace gpic {

// A packed shard (sym.cu): super-rows [p_lo, p_hi) of 4 x 128 rows, its
// tiles stored from global tile index tile_base. Default: the whole matrix.
struct ShardRange {
  int64_t p_lo = 0;
  int64_t p_hi = INT64_MAX / 4;
  int64_t tile_base = 0;
  __host__ __device__ int64_t sb_lo(int64_t ns) const;
  __host__ __device__ int64_t sb_hi(int64_t ns) const;
};


constexpr int kTileM = 128;  // affinity row tile
constexpr int kTileN = 128;  // affinity column tile
constexpr int kRedBlock = 2048;  // fixed block of the tau / delta reductions

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

int32_t feature_pitch(int32_t d);
int64_t row_pad(int64_t n);
int64_t operand_floats(int64_t n, int32_t d);
int64_t affinity_pitch(int64_t n);
// fp32 vector copies of v are zero-padded to whole 128-element tiles
inline int64_t vector_pitch(int64_t n) { return round_up(n, 128); }

// ---- symmetric packed storage (affinity_tc.cu, sym.cu) -------------------
int64_t packed_tiles(int64_t n);        // nt (nt + 1) / 2, nt = ceil(n / 128)
int64_t sym_partial_floats(int64_t n);  // packed_tiles(n) * 128
// Packed affinity; the epilogue also leaves per-tile degree partials:
// degrow [tile][packed_row_halves(dp)][128] (row sums of the stored tile)
// and degcol [tile][4][128] (column sums per 32-row quadrant, off-diagonal
// tiles), combined by launch_sym_degree.
int packed_row_halves(int32_t dp);
// SIMT engine, packed upper-triangle tiles + per-tile degree partials
void launch_affinity_simt_packed(const float* xlo, const float* sqn, int64_t n, int32_t d, int32_t dp,
                                 float neg_scale_log2, float* a_packed, float* degrow,
                                 float* degcol, cudaStream_t s, int kind);
// feature pitches the tcgen05 engine runs (store modes / matrix-free)
bool tc_supports_pitch(int32_t dp, bool matvec);
// boxnz: non-null -> zero boxes are not stored and flagged there (sparse.cu)
int launch_affinity_tc_packed(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                              int32_t dp, float neg_scale_log2, void* a_packed, float* degrow,
                              float* degcol, cudaStream_t s, int kind = GPIC_KIND_RBF,
                              bool half_out = false, int64_t row_lo = 0, int64_t row_hi = 0,
                              uint8_t* boxnz = nullptr, const int32_t* unit_list = nullptr,
                              const int64_t* unit_count = nullptr);
// M blocks (128-row tiles) per tcgen05 work unit at feature pitch dp
int tc_mblocks(int32_t dp);     // packed store modes
int tc_mblocks_mf(int32_t dp);  // the matrix-free pass
// boxnz non-null: tiles without a stored box contribute zero (not read);
// pm non-null: pruned block pairs are not even looked at (prune.cu)
struct PruneMask;
void launch_sym_degree(const float* degrow, const float* degcol, int64_t n, int nhalf,
                       double* deg, gpic_ctl* ctl, cudaStream_t s,
                       const ShardRange& sr = ShardRange(), const uint8_t* boxnz = nullptr,
                       const PruneMask* pm = nullptr, const int64_t* sb_prefix = nullptr);
void sym_prepare();

// Workspace carve-up (see capi.cu).
struct Workspace {
  gpic_ctl* ctl;
  float* xhi;          // n_pad x dp
  float* xlo;          // n_pad x dp
  float* sqn;          // n_pad
  double* colpart;     // ceil(n/256) x d
  double* mean;        // d
  float* rowpart;      // n_ctiles x rows_pad
  double* redpart;     // ceil(n/2048) partials
  double* y;           // n (fp64 GEMV result, full vector)
  double* deg;         // n row degrees (fp64)
  double* v64;         // 2 x n ping-pong
  float* v32;          // lda floats (fp32 copy of v, zero padded)
  double* kscratch;    // k-means scratch (see kmeans.cu)
  int64_t* lowlist;    // n low-degree row indices (lowdeg.cu)
  unsigned long long* lowcount;
  uint8_t* sparse;     // SparseMask storage (sparse.cu)
  uint8_t* prune;      // PruneMask storage (prune.cu)
  uint8_t* locality;   // Locality storage (locality.cu)
  int64_t kscratch_bytes;
  uint8_t* end;
};

int64_t workspace_bytes(int64_t n, int32_t d, int32_t k, int64_t rows, int32_t max_iter);
int carve(void* base, int64_t bytes, int64_t n, int32_t d, int32_t k, int64_t rows,
          int32_t max_iter, Workspace* ws);

// prepare.cu
void launch_ctl_init(gpic_ctl* ctl, double eps, int32_t max_iter, cudaStream_t s);
void launch_prepare(const double* x, int64_t n, int32_t d, float* xhi, float* xlo, float* sqn,
                    double* colpart, double* mean, gpic_ctl* ctl, cudaStream_t s,
                    int kind = GPIC_KIND_RBF);

// affinity_simt.cu / affinity_tc.cu
void launch_affinity_simt(const float* xhi, const float* xlo, const float* sqn, int64_t n, int32_t d,
                          int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2,
                          float* a, int64_t lda, float* rowpart, int64_t rows_pad,
                          cudaStream_t s, int kind = GPIC_KIND_RBF);
int launch_affinity_tc(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                       int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2, float* a,
                       int64_t lda, float* rowpart, int64_t rows_pad, cudaStream_t s,
                       int kind = GPIC_KIND_RBF);
void launch_degree(const float* rowpart, int64_t rows, int64_t rows_pad, int64_t n_ctiles,
                   int64_t row_lo, double* deg, gpic_ctl* ctl, cudaStream_t s);

// ---- rank exchange (comm.cu) -----------------------------------------
// Every rank owns rows [row_lo, row_lo + rows) of A. Each iteration, the
// GEMV of rank s stores its y rows straight into the y buffer of EVERY rank
// (peer pointers: CUDA IPC mappings over NVLink, or plain device pointers
// for virtual ranks on one GPU), then its last CTA release-stores the epoch
// into flags_p[s] on every rank p. A rank's tail waits (acquire) until all P
// epochs have arrived. y is double-buffered by iteration parity, so a fast
// rank writing iteration t+1 never races a slow rank still reading t.
constexpr int kMaxRanks = 8;
// [0,P): iteration epochs, [P,2P): gather epochs, [2P,3P): the y slices'
// all-gather epochs of a reduce-scatter exchange
constexpr int kFlagSlots = 3 * kMaxRanks;

struct PeerTable {
  double* y[kMaxRanks][2];     // y ping-pong of every rank, as seen from this process
  uint64_t* flags[kMaxRanks];  // kFlagSlots epochs per rank (nullptr: single rank)
  int nranks;
  int self;                    // global rank index of the local shard
  // partial-y slots (packed / matrix-free item shards): 0 = every rank gets
  // the whole partial (all-to-all), 1 = row i goes to its slice owner only
  // (reduce-scatter; the owners all-gather the finished y slices)
  int scatter;
  // the epoch base of a loop is ctl->sync_epoch (device-side, so one
  // captured graph is replayed for every run)
};

// power.cu
void launch_tree_sum(const double* v, int64_t n, double* part, double* out, gpic_ctl* ctl,
                     cudaStream_t s);
void launch_scale_vector(const double* src, int64_t n, const double* tau, double* v64,
                         float* v32, int64_t v32_len, cudaStream_t s);
void launch_scale_by(const double* src, int64_t n, double tau, double* dst, float* dst32,
                     int64_t f32_len, cudaStream_t s);
void gemv_prepare();
void launch_row_stats(const double* w, int64_t rows, int64_t n, int64_t ldw, double* sum,
                      double* mn, double* mx, cudaStream_t s);
void launch_gemv(const float* a, int64_t lda, int64_t rows, int64_t row_lo, const float* v32,
                 const double* deg, const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s);
void launch_peer_wait(const uint64_t* flags_self, int slot0, int count, uint64_t base,
                      int add_iter, gpic_ctl* ctl, cudaStream_t s);
// y = (sum over ranks of the packed shards' y partials, rank order) / deg
// reduce-scatter exchange: the owner's rows [n r / P, n (r+1) / P)
__host__ __device__ inline int64_t slice_lo(int64_t n, int r, int nranks) {
  return n * r / nranks;
}
__host__ __device__ inline int slice_owner(int64_t i, int64_t n, int nranks) {
  int r = (int)((i * nranks) / n);
  while (r + 1 < nranks && slice_lo(n, r + 1, nranks) <= i) ++r;
  while (r > 0 && slice_lo(n, r, nranks) > i) --r;
  return r;
}
// sum of the P slots for this rank's slice (rank order) / deg, stored into
// every rank's y, then the all-gather epoch published
void launch_slice_combine(const double* slots, int64_t stride, int64_t n, const double* deg,
                          const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s);
void launch_slot_combine(const double* slots, int64_t stride, int nranks, int64_t n,
                         const double* deg, double* y0, double* y1, gpic_ctl* ctl, cudaStream_t s);
// tau_mode: kTailTauAlways / kTailTauIfNoLow (*lowcnt == 0): ctl->tau was
// computed by the reduce, the tail only normalises
// low / low_deg: the low-degree rows, whose fp64 y_i the tail computes
// first (low.count == 0: none; < 0: the device-side count decides)
struct LowRows;
void launch_iteration_tail(double* y0, double* y1, int64_t n, double* redpart, double* v64,
                           float* v32, double* hist, gpic_ctl* ctl, cudaStream_t s, int tau_mode,
                           const LowRows& low, const double* low_deg);
void launch_copy_result(const double* v64, int64_t n, double* out, const gpic_ctl* ctl,
                        cudaStream_t s);

struct PeerTable;
// boxnz / sb_prefix: block sparsity (SparseMask), null = every box stored
struct IterTail;  // below
// what the GEMV launch took over from the iteration tail (IterTail given):
// kTailSeparate nothing; kTailTauAlways tau computed in the reduce;
// kTailTauIfNoLow tau in the reduce when the device-side low-row count is
// 0; kTailFused reduce + low rows + tau + normalise (GPIC_FUSED_TAIL=1)
enum : int { kTailSeparate = 0, kTailTauAlways = 1, kTailTauIfNoLow = 2, kTailFused = 3 };
int launch_sym_gemv(const float* tiles, int64_t n, const float* v32, float* rowp, float* colp,
                     const double* deg, const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s,
                     const ShardRange& sr = ShardRange(), const uint8_t* boxnz = nullptr,
                     const int64_t* sb_prefix = nullptr, const IterTail* it = nullptr);
// fp16 packed tiles (GPIC_STORAGE_PACKED16): same partials / reduce
int launch_sym_gemv16(const void* tiles, int64_t n, const float* v32, float* rowp, float* colp,
                       const double* deg, const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s,
                       const uint8_t* boxnz = nullptr, const int64_t* sb_prefix = nullptr,
                       const IterTail* it = nullptr);

// ---- provably-zero block pairs (prune.cu) -------------------------------
// Row blocks of B rows; skip[S * nb + T] = 1 when every entry between
// blocks S and T is proved to flush to zero; units = ascending list of the
// tcgen05 packed work units that are not skipped, *count of them.
struct PruneMask {
  int64_t B = 0, nb = 0;
  float* cent = nullptr;    // nb x dp block centroids
  float* own = nullptr;     // n: x_i . c_{S(i)}
  unsigned* mmax = nullptr; // nb x nb order-preserving max images
  uint8_t* skip = nullptr;  // nb x nb
  int32_t* units = nullptr;
  int64_t* count = nullptr;
  unsigned* scal = nullptr; // |c|max, |x|max (float bits)
  int32_t* rbcount = nullptr;  // kept units (items) per row block
  // matrix-free sym pass: kept (row block, chunk) items, id rb * chunks + c
  int32_t* items = nullptr;
  int64_t* item_count = nullptr;
  uint8_t* item_kept = nullptr;  // [row block][chunk] kept tiles of the item (0: pruned)
  int32_t* rbtiles = nullptr;    // kept tiles per row block
  int64_t* item_wpre = nullptr;  // kept tiles before list entry u (count + 1 entries)
  unsigned* sched = nullptr;     // affinity_tc's dynamic schedule counters (2 words)
  // matrix-free passes: CTA cuts re-balanced from the last pass's measured
  // per-CTA times (header: grid, ua, ub; then grid + 1 cuts) and those times
  int64_t* cta_cuts = nullptr;
  uint64_t* cta_ns = nullptr;
};
// after a pruned matrix-free pass: the next pass's CTA cuts from its times
int launch_mf_rebalance(const PruneMask* pm, int share_r, int share_n, const gpic_ctl* ctl,
                        cudaStream_t s);
bool mf_rebalance_enabled();
// the schedule counters in the count slot of a mask (from its unit count)
unsigned* prune_sched(const int64_t* unit_count);
bool prune_enabled();  // GPIC_PRUNE=0 computes every tile (comparisons)
int prune_item_weight();  // matrix-free items: item_wpre = 4 tiles + this per item
int64_t prune_block_rows(int64_t n);
int64_t prune_bytes(int64_t n, int32_t dp);
PruneMask carve_prune(void* base, int64_t n, int32_t dp);
// xc: the centred fp32 rows (pitch dp); colpart / mean: the prepare pass's
// 256-row column sums and centring mean; mb: tc_mblocks(dp) for the packed
// unit list, -tc_mblocks(dp) for the matrix-free item list
// row_lo / row_hi: a packed shard's rows (the unit list covers its row
// blocks only); row_hi <= 0: n
void launch_prune(const PruneMask& m, const float* xc, const double* colpart, const double* mean,
                  int64_t n, int32_t d, int32_t dp, double sigma, int mb, int64_t row_lo,
                  cudaStream_t s, int64_t row_hi = 0);

// ---- matrix-free (affinity_tc.cu matvec mode + mf.cu) --------------------
struct MfOperands {
  const float* xhi;
  const float* xlo;
  const float* sqn;
  int64_t n;
  int32_t dp;
  float ns;  // -log2(e) / (2 sigma^2)
  int kind = GPIC_KIND_RBF;
  int sym = 0;  // whole matrix on one rank: upper-triangle pass (mf.cu)
  int32_t d = 0;  // features (RBF with d <= 8: the difference-form SIMT pass)
  int pruned = 0;  // sym pass over the kept items of `prune` only (prune.cu)
  PruneMask prune;
  // pruned sym pass split across ranks: this rank computes the tile-balanced
  // share share_r of share_n of the kept items; its reduce yields a partial y
  int share_r = 0, share_n = 1;
};
// workspace of a matrix-free item shard: full-matrix partial buffers, the
// pruning mask, one fp32 vector
int64_t mf_shard_scratch_bytes(int64_t n, int32_t d);
PruneMask mf_shard_prune(double* ypart, int64_t n, int32_t d);
bool mf_sym_default();
int64_t mf_parts(int64_t n, int32_t dp);
int mf_rows_per_block(int32_t dp);
int64_t mf_colpart_floats(int64_t n, int32_t dp);
int64_t mf_ypart_doubles(int64_t n, int32_t dp, int64_t rows);
int launch_affinity_tc_matvec(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                              int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2,
                              const float* v32, double* ypart, int64_t rows_pad,
                              const gpic_ctl* ctl, cudaStream_t s, int kind = GPIC_KIND_RBF,
                              float* colpart = nullptr, const PruneMask* pm = nullptr,
                              int share_r = 0, int share_n = 1);
int launch_mf_matvec(const MfOperands& op, int64_t row_lo, int64_t rows, const float* v32,
                     double* ypart, const double* deg, const PeerTable& pt, gpic_ctl* ctl,
                     cudaStream_t s);
int launch_mf_degrees(const MfOperands& op, int64_t row_lo, int64_t rows, float* ones,
                      double* ypart, double* deg, cudaStream_t s);

// ---- block sparsity (sparse.cu) ------------------------------------------
// boxnz[tile * 16 + quadrant * 4 + chunk] = 1 when the affinity epilogue
// stored that 32 x 32 box of packed tile `tile`, 0 when every value of it was
// an exact fp32 zero (not stored); sb_prefix[s] = GEMV super-block weight
// (8 per stored tile + 1) before super-block s.
struct SparseMask {
  int64_t nt = 0;
  uint8_t* boxnz = nullptr;
  int64_t* sb_prefix = nullptr;
  int64_t n_sb = 0;
};
int64_t sparse_mask_bytes(int64_t n, int32_t d);
// per super-block box bits (16 tiles x 16 boxes), stored behind sb_prefix
const uint16_t* sb_bits(const int64_t* sb_prefix, int64_t n);
// the non-empty super-blocks (ascending ids, weight prefix per entry, count)
struct SbList {
  const int32_t* list;
  const int64_t* lpre;
  const int64_t* count;
  // ranges[0] = the grid they were cut for, ranges[1 + b] = first entry of
  // CTA b (ranges[1 + grid] = count)
  const int64_t* ranges = nullptr;
  // the reduce's per-super-row lists of non-empty record terms (sym.cu)
  const int32_t* tlist = nullptr;
  const int32_t* tcount = nullptr;
  int64_t tld = 0;
  // the GEMV's dynamic schedule counters (2 words, zeroed by sb_list_kernel)
  unsigned* sched = nullptr;
};
void launch_reduce_terms(const int64_t* sb_prefix, int64_t nt, int32_t* tlist, int32_t* tcount,
                         int64_t tld, cudaStream_t s);
SbList sb_list(const int64_t* sb_prefix, int64_t n);
SparseMask carve_sparse(void* base, int64_t n, int32_t d);
// the GEMV weights from the box flags the affinity engine wrote
void launch_sparse_prefix(const SparseMask& m, cudaStream_t s);
// every box flag = v (engines that store every box)
void launch_box_fill(const SparseMask& m, uint8_t v, cudaStream_t s);
// GPIC_SPARSE=0 turns the zero-box skipping off (dense packed runs, for comparisons)
bool sparse_enabled();
// a packed shard's block-sparsity region inside its build scratch (capi.cu)
SparseMask packed_shard_sparse(void* d_scratch, int64_t n, int64_t row_lo, int64_t row_hi,
                               int32_t d);

// ---- locality order (locality.cu) -----------------------------------------
// Points of a randomly ordered input permuted so that index neighbours are
// space neighbours (seed Voronoi cells, ordered by super-seed); the run
// proceeds on xp and v is scattered back through perm.
struct Locality {
  double* xp = nullptr;      // n x d fp64, the permuted points
  int32_t* perm = nullptr;   // perm[p] = original index at position p
  int32_t *cell = nullptr, *keys = nullptr, *keys_out = nullptr, *iota = nullptr;
  int32_t *seed_idx = nullptr, *super_idx = nullptr, *seed_super = nullptr, *rank = nullptr;
  int32_t* super_pos = nullptr;  // chain position of each super-seed
  float* snorm = nullptr;
  double* metric = nullptr;  // [0] sum |x_i - x_(i+1)|^2, [1] sum |x_i|^2 (sampled)
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int64_t m = 0;
};
int64_t locality_bytes(int64_t n, int32_t d);
Locality carve_locality(void* base, int64_t n, int32_t d);
bool locality_enabled();  // GPIC_REORDER=0: never; 2: always (tests)
bool locality_forced();
void launch_order_metric(const Locality& L, const float* xc, int64_t n, int32_t dp, cudaStream_t s);
int launch_locality_order(const Locality& L, const float* xc, const double* x, int64_t n, int32_t d,
                          int32_t dp, cudaStream_t s);
void launch_unpermute(const double* v, const int32_t* perm, int64_t n, double* out, cudaStream_t s);

// ---- low-degree (isolated) rows, lowdeg.cu -----------------------------
// Rows whose engine degree is below low_degree_threshold(kind): recomputed
// in fp64 from the caller's original X (n x d row-major) like the reference.
struct LowRows {
  const double* x = nullptr;
  int64_t n = 0;
  int32_t d = 0;
  int kind = GPIC_KIND_RBF;
  double sigma = 1.0;
  const int64_t* list = nullptr;              // row indices (device)
  const unsigned long long* d_count = nullptr;  // device count of list
  int64_t count = 0;  // host copy (0: nothing to do; < 0: unknown, kernels read d_count)
};
// What the fused iteration kernel (sym.cu) needs beyond the GEMV's operands:
// the y ping-pong, the tail's buffers and the low-degree rows. The launch
// returns true when it replaced reduce + low rows + tail (one whole-matrix
// rank, list reduce; opt-in: GPIC_FUSED_TAIL=1).
struct IterTail {
  double* y0 = nullptr;
  double* y1 = nullptr;
  double* redpart = nullptr;
  double* v64 = nullptr;
  float* v32 = nullptr;
  double* hist = nullptr;
  LowRows low;               // low.count == 0: no listed rows (d_count may be null)
  const double* low_deg = nullptr;
};
double low_degree_threshold(int kind, int64_t n);
void launch_lowdeg_scan(const double* deg, int64_t n, int kind, int64_t* list,
                        unsigned long long* count, cudaStream_t s);
int read_low_count(const unsigned long long* d_count, int64_t* out, cudaStream_t s);
// exact fp64 degrees of the listed rows into deg (ZeroDegree if one is 0)
void launch_lowdeg_exact(const LowRows& L, double* deg, gpic_ctl* ctl, cudaStream_t s);
// loop body: y_i = sum_j (a_ij / deg_i) v_j for the listed rows (fp64 v)
void launch_lowdeg_matvec(const LowRows& L, const double* deg, const double* v64, double* y0,
                          double* y1, gpic_ctl* ctl, cudaStream_t s);

enum { kLoopDense = 0, kLoopPacked = 1, kLoopMatrixFree = 2, kLoopPacked16 = 3, kLoopPackedShard = 4,
       kLoopMfShard = 5 };

// One shard's loop state (a single-rank run is one shard with nranks = 1).
struct ShardLoop {
  const float* a;     // dense row block, or the packed tiles when packed
  int mode;           // kLoopDense / kLoopPacked (whole matrix) / kLoopMatrixFree
  float* rowp;        // packed: per-tile row / column partials
  float* colp;
  MfOperands mf;      // matrix-free operands
  double* ypart;      // matrix-free row partials
  int64_t lda;
  int64_t rows;
  int64_t row_lo;
  const double* deg;  // degrees of the shard's rows
  double* redpart;
  double* v64;        // 2 x n ping-pong
  float* v32;         // pitch(n) floats
  double* hist;
  gpic_ctl* ctl;
  PeerTable pt;
  // packed shards (kLoopPackedShard): super-row range, the y-partial table
  // (every rank's slot of this shard), this rank's slots and full degrees
  ShardRange sr;
  PeerTable pt_slots;
  const double* slots;   // this rank's slot [0][0]; (rank, parity) at (2 rank + parity) * stride
  int64_t slot_stride;
  const double* deg_full;
  // packed modes: stored-box flags + GEMV super-block weights (null: dense)
  const uint8_t* boxnz;
  const int64_t* sb_prefix;
  // isolated rows redone in fp64 after the y exchange (count 0: none)
  LowRows low;
  const double* low_deg;  // full n-vector of degrees (exact for listed rows)
};
// Capture max_iter iterations of every local shard into one CUDA graph
// (virtual ranks: all GEMVs of an iteration precede all tails) and launch it.
int run_power_loops(ShardLoop* shards, int nlocal, int64_t n, int32_t max_iter, cudaStream_t s);
// launch accounting for the conditional loop graph: iterations x kernels
void note_loop_iterations(int32_t iters);
int run_power_loop(const float* a, int64_t lda, const double* deg, int64_t n, double* y,
                   double* redpart, double* v64, float* v32, double* hist, gpic_ctl* ctl,
                   int32_t max_iter, cudaStream_t s);

// kmeans.cu
int64_t kmeans_scratch_bytes(int64_t n, int32_t k);
// Device App-B generator (generate.cu): X row-major n x d fp64, labels int64
int launch_generate_blobs(const double* centers, const int64_t* offsets, int64_t n, int d, int k,
                          uint64_t seed, double noise, double offset, double* x, int64_t* labels,
                          cudaStream_t s);
// 64 < k <= kmeans_big_max_k(): sorted-domain Lloyd (kmeans_big.cu)
int kmeans_big_max_k();
int64_t kmeans_big_scratch_bytes(int64_t n, int32_t k);
int launch_kmeans1d_big(const double* v, int64_t n, int32_t k, int64_t first_index,
                        const double* h_uniforms, int32_t max_rounds, double tol, int64_t* labels,
                        void* scratch, gpic_ctl* ctl, cudaStream_t st);
int launch_kmeans1d(const double* v, int64_t n, int32_t k, int64_t first_index,
                    const double* h_uniforms, int32_t max_rounds, double tol, int64_t* labels,
                    void* scratch, gpic_ctl* ctl, cudaStream_t s);
// batched k-means (batch.cu): one CTA per problem, problems described by
// opaque KProblem records filled on the host and copied to the device
int64_t kmeans_batch_scratch_bytes(int64_t n, int32_t k);
int64_t kmeans_problem_bytes();
int fill_kmeans_problem(void* host_slot, const double* v, int64_t n, int64_t first, void* scratch,
                        int32_t k, const double* d_unif, int64_t* labels, gpic_ctl* ctl);
int launch_kmeans1d_batch(const void* d_problems, int32_t count, int32_t k, int32_t max_rounds,
                          double tol, bool polish, cudaStream_t s);

}  // namespace gpic
