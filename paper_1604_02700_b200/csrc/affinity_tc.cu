// Stage 1 (tensor-core engine): affinity tiles on tcgen05 with a fused
// exp / diagonal / row-sum epilogue, in three output modes.
//
//   G = Xc_I Xc_J^T via a 3-term fp16 split: s^2 G ~= hi_I.lo_J + lo_I.hi_J +
//   hi_I.hi_J, where xc s ~= hi + lo (hi = fp16(xc s), lo = fp16(xc s - hi),
//   s = 2^e from the data range, prepare.cu), each term a
//   tcgen05.mma.kind::f16 (M=128, N=128, K=16) accumulating in TMEM (fp32).
//   fp16 and TF32 both keep 11 significant bits, so this matches 3xTF32's
//   accuracy at half the smem operand bytes per MMA and twice the rate.
//   a_ij = exp2(min(ns*(|x_i|^2 + |x_j|^2 - 2 G_ij), 0)),  ns = -log2(e)/(2 sigma^2)
//   a_ii = 0, a_ij = 0 for padding rows / columns          (affinity.py:96-103)
//
// Modes (epilogue):
//   dense   store rows [row_lo, row_hi) x all columns, fp32 pitch lda, plus
//           fp32 row partials per 128-column tile for the degree combine
//   packed  store only tiles J >= I of the (exactly symmetric) matrix, each
//           128x128 tile contiguous (sym.cu streams them)
//   matvec  matrix-free: nothing is stored; each element is
//           multiplied by v_j in registers and row sums are accumulated per
//           32-tile column chunk (fp64) -> ypart; A v is recomputed every
//           iteration when n^2 does not fit HBM.
//           sym (whole matrix on one rank): only tiles J >= I are computed
//           (A is exactly symmetric); each off-diagonal tile also yields the
//           column partials sum_i a_ij v_i (its transpose's row partials),
//           combined across the CTA's warps in fixed order -> colpart, one
//           128-float record per (row block, column tile). Half the work.
//
// Persistent warp-specialised kernel, one CTA per SM (576 threads):
//   warp 0      TMA producer: the CTA's row block (MB x 128 rows, hi + lo,
//               all K) stays resident in smem while the CTA walks its
//               contiguous range of column tiles; B tiles (128 columns,
//               hi + lo, one 64-wide K block per stage) stream through a
//               ring of smem stages.
//   warp 1      TMEM owner + single-thread MMA issuer: 3 x 4 x KB MMAs per
//               M block into one of two TMEM accumulators (double buffer,
//               so the next tile's MMAs overlap this tile's epilogue).
//   warps 2-17  epilogue: tcgen05.ld 32 columns at a time, exp2 + masks +
//               row sums in registers; store modes go through swizzled
//               st.shared and TMA bulk-tensor stores of 32x32 fp32 boxes.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "ops.h"
#include "sm100.cuh"

namespace gpic {

namespace {

enum { kModeDense = 0, kModePacked = 1, kModeMatvec = 2, kModePacked16 = 3 };
// packed symmetric tiles, fp32 (kModePacked) or fp16 (kModePacked16) values
__host__ __device__ constexpr bool is_packed(int MODE) {
  return MODE == kModePacked || MODE == kModePacked16;
}

constexpr int kBN = 128;           // columns per tile (one MMA N)
constexpr int kKBlk = 64;          // fp16 per 128-byte swizzle row
constexpr int kTileBytes = 128 * kKBlk * 2;  // 16 KB: 128 rows x 64 fp16
constexpr int kEpiWarps = 16;      // 4 per SM sub-partition: latency hiding for the epilogue
// warpgroup 0: TMA producer (warp 0), MMA issuer (warp 1), two idle warps;
// warpgroups 1-4: epilogue. setmaxnreg moves registers from warpgroup 0
// (kCtlRegs) to the epilogue (kEpiRegs, room for the next chunk's TMEM load
// in flight). Launch: 96 per thread; an increase is served only from what
// warpgroup 0 releases (measured, scripts/probe/smr.cu: 56 -> 104 runs,
// 88 -> 104 waits forever), so 128 (96 - kCtlRegs) >= 512 (kEpiRegs - 96).
constexpr int kThreads = 128 + kEpiWarps * 32;  // with the register split (matrix-free)
constexpr int kCtlRegs = 64;
constexpr int kEpiRegs = 104;
static_assert(128 * (96 - kCtlRegs) >= kEpiWarps * 32 * (kEpiRegs - 96),
              "setmaxnreg.inc would wait for registers nobody releases");
// Matrix-free (compute-bound): registers rebalanced and the next chunk's
// TMEM load overlapped with this chunk's work (config 5 pass 273 -> 244 ms).
// Store modes keep 96 each and one chunk in flight (measured faster: the
// producer / MMA code spills at 64 registers and the stores bound them).
template <int MODE>
constexpr bool kSplitRegs = MODE == kModeMatvec;
// first epilogue warp: 4 with the split (warpgroup 0 = producer, MMA, two
// idle warps), else 2 (producer, MMA); CTA size follows
template <int MODE>
constexpr int kEpiBase = kSplitRegs<MODE> ? 4 : 2;
template <int MODE>
constexpr int kCtaThreads = 32 * kEpiBase<MODE> + kEpiWarps * 32;
constexpr int kSmemBudget = 232448 - 1024 - 256;  // 227 KB opt-in minus alignment + barriers
constexpr int kChunkTiles = 32;              // matvec: column tiles per work item
constexpr int kMaxRebalanceGrid = 256;       // matvec re-balance: CTAs per pass at most

// rows per CTA block: 256 (two M blocks sharing every B stage) while the
// operands fit, else 128
// packed store modes: M blocks per unit at KB = 1 (GPIC_TC_PACKED_MB build knob)
#ifndef GPIC_TC_PACKED_MB
#define GPIC_TC_PACKED_MB 2
#endif
__host__ __device__ constexpr int mblocks(int KB, int MODE) {
  return KB == 1 ? (is_packed(MODE) ? GPIC_TC_PACKED_MB : 2) : 1;
}
// norm block (prepare.cu): per 128-row tile, hi + lo planes of 128 x 16 fp16
// (32-byte swizzle), one extra K = 16 step that adds -(s^2/2)(|x_i|^2+|x_j|^2)
constexpr int kNrmPlane = 128 * 16 * 2;   // 4 KB
constexpr int kNrmBytes = 2 * kNrmPlane;  // hi + lo
__host__ __device__ constexpr int a_main_bytes(int KB, int MODE) { return 2 * mblocks(KB, MODE) * KB * kTileBytes; }
__host__ __device__ constexpr int a_bytes(int KB, int MODE) { return a_main_bytes(KB, MODE) + mblocks(KB, MODE) * kNrmBytes; }
constexpr int kStageBytes = 2 * kTileBytes + kNrmBytes;  // B hi, B lo, B norm block
// store modes: one 4 KB staging buffer (a swizzled 32 x 32 fp32 box) per
// epilogue warp, also used for the row-sum combine; matvec: a fp64
// [warp][32 rows] combine scratch + the sym column-partial exchange
// [tile parity][m][quadrant][128 columns] fp32
constexpr int kStageOutBytes = 32 * 128;
__host__ __device__ constexpr int colx_bytes(int KB) { return 2 * mblocks(KB, kModeMatvec) * 4 * 128 * 4; }
__host__ __device__ constexpr int out_bytes(int KB, int MODE) {
  return MODE == kModeMatvec ? kEpiWarps * 32 * 8 + colx_bytes(KB) : kEpiWarps * kStageOutBytes;
}
// matvec: per epilogue warp, double-buffered by tile, the 64 columns' v_j
__host__ __device__ constexpr int col_bytes(int MODE) {
  return MODE == kModeMatvec ? kEpiWarps * 2 * 64 * 4 : 0;
}
__host__ __device__ constexpr int stages_raw(int KB, int MODE) {
  return (kSmemBudget - a_bytes(KB, MODE) - out_bytes(KB, MODE) - col_bytes(MODE)) / kStageBytes;
}
__host__ __device__ constexpr int stages(int KB, int MODE) {
  return stages_raw(KB, MODE) > 4 ? 4 : (stages_raw(KB, MODE) < 1 ? 1 : stages_raw(KB, MODE));
}
__host__ __device__ constexpr int smem_bytes(int KB, int MODE) {
  return a_bytes(KB, MODE) + stages(KB, MODE) * kStageBytes + out_bytes(KB, MODE) + col_bytes(MODE) +
         256 + 1024;
}

constexpr uint32_t kIdesc = idesc_f16(128, kBN);

struct TcArgs {
  const float* sqn;
  int64_t n;
  int64_t row_lo;
  int64_t rows;
  float ns;  // -log2(e) / (2 sigma^2)
  float* rowpart;    // dense: [n_ctiles][rows_pad] fp32 row partials
  int64_t rows_pad;
  int64_t n_rtiles;  // row blocks of 128*MB rows (packed shards: global end)
  int64_t rb_base;   // packed shards: first row block (global); else 0
  int64_t u_lo;      // packed shards: units before rb_base (contiguous order)
  int64_t tile_base; // packed shards: global index of the shard's first stored tile
  int64_t n_ctiles;  // column tiles of 128
  const float* v32;  // matvec: vector_pitch(n) floats
  double* ypart;     // matvec: [n_chunks * parts][rows_pad] fp64 row partials
  int64_t n_chunks;  // matvec: column chunks (kChunkTiles tiles) per row block
  const gpic_ctl* ctl;  // matvec in a loop: exit at once when ctl->stop is set
  float* out;        // stored A: dense rows (pitch lda) or packed 128 x 128 tiles
  int64_t lda;
  float* degrow;     // packed: [tile][128] row partials of each stored tile
  float* degcol;     // packed: [tile][4 row quadrants][128] column partials
  int kind;          // GPIC_KIND_RBF: exp2 epilogue; GPIC_KIND_COSINE: max(0, G) on unit rows
  const float* gscale;  // 1 / s^2 of the fp16 operand planes (sqn[n_pad - 1], prepare.cu)
  int strided;          // dense / packed: row-block-strided work order (see Cursor)
  int64_t n_pad;        // rows per operand plane (the norm block's plane stride)
  int sym;              // matvec: upper-triangle tiles only, column partials -> colpart
  int store_hint;       // store modes: L2 evict-first hint on the output stream
  float* colpart;       // matvec sym: [packed (row block, column tile)][128] fp32
  // packed store modes: non-null -> a 32 x 32 box whose values are all exact
  // zeros is not stored; boxnz[(tile) * 16 + quadrant * 4 + chunk] records
  // which boxes were (sparse.cu). Indexed by the global packed tile.
  uint8_t* boxnz;
  // packed store modes: non-null -> only the listed work units (ascending
  // packed unit ids, *unit_count of them) are computed; the others are
  // provably zero block pairs (prune.cu) and the CTAs split the list
  const int32_t* unit_list;
  const int64_t* unit_count;
  // matvec sym: non-null -> unit_list holds the kept (row block, chunk)
  // items (id = rb * n_chunks + chunk) and a tile cb of an item is computed
  // only if pskip[S(rb) * pnb + T(cb)] == 0 (blocks of pB rows, prune.cu)
  const uint8_t* pskip;
  int64_t pB, pnb;
  const int64_t* wpre;  // matvec listed: kept tiles before each item (CTA balance)
  int share_r, share_n;  // matvec listed across ranks: this rank's tile-balanced share
  // listed runs: [0] claim counter, [1] CTAs done claiming (the last resets
  // both) — list ranges are claimed at run time instead of split in advance;
  // null: the static split
  unsigned* sched;
  // matvec listed: CTA cuts measured by the previous pass (mf.cu rebalance:
  // [0] grid, [1] ua, [2] ub, then grid + 1 list positions; used when the
  // header matches this launch) and this pass's per-CTA time in ns
  const int64_t* cuts;
  uint64_t* cta_ns;
};

// Claim k of a dynamic run over list entries [lo, hi) on G CTAs: G claims
// of 5/8 of an equal share, 2G of 1/8, then 1/64-share claims to the end
// (large first claims keep row blocks contiguous, small last ones even out
// the finish). false: nothing left.
__device__ inline bool claim_range(int64_t k, int64_t lo, int64_t hi, int64_t G, int64_t& e0,
                                   int64_t& e1) {
  const int64_t n = hi - lo;
  const int64_t s1 = max((int64_t)1, n * 5 / (8 * G)), s2 = max((int64_t)1, n / (8 * G));
  const int64_t s3 = max((int64_t)1, n / (64 * G));
  int64_t off, sz;
  if (k < G) {
    off = k * s1;
    sz = s1;
  } else if (k < 3 * G) {
    off = G * s1 + (k - G) * s2;
    sz = s2;
  } else {
    off = G * s1 + 2 * G * s2 + (k - 3 * G) * s3;
    sz = s3;
  }
  e0 = lo + off;
  if (e0 >= hi) return false;
  e1 = min(e0 + sz, hi);
  return true;
}

// The producer's claims reach the MMA issuer and the epilogue warps through
// a 4-slot ring in the barrier area: [0] = first entry (-1: no more), [1] = end.
constexpr int kFeedSlots = 4;
struct Feed {
  // one base: full [kFeedSlots] (count 1, the producer), empty [kFeedSlots]
  // (count 1 + kEpiWarps: MMA issuer + epilogue warps), then the ranges
  // [kFeedSlots][2] as int32 — the epilogue's registers are tight
  uint64_t* full;
  int q = 0;
  uint32_t ph = 0;
  __device__ uint64_t* empty_bar(int i) const { return full + kFeedSlots + i; }
  __device__ int32_t* rng() const { return reinterpret_cast<int32_t*>(full + 2 * kFeedSlots); }
  // reader: the next range (false: the run is over); `arrive`: this thread
  // releases the slot (lane 0 of a reading warp)
  __device__ bool read(int64_t& e0, int64_t& e1, bool arrive) {
    mbar_wait(&full[q], ph);
    const int32_t a = rng()[2 * q], b = rng()[2 * q + 1];
    __syncwarp(__activemask());
    if (arrive) mbar_arrive(empty_bar(q));
    if (++q == kFeedSlots) { q = 0; ph ^= 1; }
    e0 = a;
    e1 = b;
    return a >= 0;
  }
  __device__ void write(int64_t e0, int64_t e1) {
    mbar_wait(empty_bar(q), ph ^ 1);
    rng()[2 * q] = (int32_t)e0;
    rng()[2 * q + 1] = (int32_t)e1;
    mbar_arrive(&full[q]);
    if (++q == kFeedSlots) { q = 0; ph ^= 1; }
  }
};

// [ua, ub): the list entries of rank share_r of share_n, tile-balanced
__device__ inline void item_share(const TcArgs& a, int64_t total, int64_t& ua, int64_t& ub);

// first u in [lo, hi] with a[u] >= target (a non-decreasing)
__device__ inline int64_t lower_bound_w(const int64_t* a, int64_t lo, int64_t hi, int64_t target) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] >= target) hi = mid; else lo = mid + 1;
  }
  return lo;
}

__device__ inline void item_share(const TcArgs& a, int64_t total, int64_t& ua, int64_t& ub) {
  ua = 0;
  ub = total;
  if (a.share_n > 1) {
    const int64_t W = a.wpre[total];
    ua = lower_bound_w(a.wpre, 0, total, W * a.share_r / a.share_n);
    ub = a.share_r + 1 == a.share_n ? total
                                    : lower_bound_w(a.wpre, 0, total, W * (a.share_r + 1) / a.share_n);
  }
}

// the work list of a listed run (packed units or matrix-free items)
template <int MODE>
__host__ __device__ inline bool run_listed(const TcArgs& a) {
  return a.unit_list != nullptr && (is_packed(MODE) || (MODE == kModeMatvec && a.sym));
}

__host__ __device__ inline int64_t packed_items(int64_t nrt, int64_t nct, int mb) {
  return nrt * nct - (int64_t)mb * nrt * (nrt - 1) / 2;
}

// Packed index of tile (I, J), J >= I, row-major over the upper triangle.
__host__ __device__ inline int64_t tile_index(int64_t I, int64_t J, int64_t nt) {
  return I * nt - I * (I - 1) / 2 + (J - I);
}

// Work sequence of one CTA, identical for all three roles. Two orders:
//   contiguous (a.strided == 0; dense / packed with L2-resident operands):
//           a balanced contiguous range of tiles (rb, cb) in row-major order
//           (packed keeps cb >= rb*MB only)
//   strided (matvec always; dense / packed when the operands exceed ~L2/4):
//           wave w gives CTA k the row block w*G + k (G = gridDim.x; packed /
//           dense reverse odd waves, which balances the packed triangle),
//           walked from its first column tile to the last. The CTAs of a
//           wave read the same B tiles at about the same time, so operands
//           larger than the L2 stream from DRAM about once per wave instead
//           of once per CTA. A matvec chunk's row partial is produced by
//           one CTA (fixed shape).
template <int MB, int MODE>
struct Cursor {
  int64_t u, u_end;    // contiguous: unit counter; strided: 0 while running, 1 when done
  int rb, cb;          // current tile (tile counts stay far below 2^31)
  int cb_end;          // matvec: end of the current item's columns
  int chunk;           // matvec: chunk index of the current item
  int wave;            // strided: current wave
  bool strided;
  bool listed;         // unit list (prune.cu): u indexes the list
  int64_t uid;         // listed: current unit id

  __device__ void decode_unit(const TcArgs& a) { decode_id(a, u); }
  __device__ void decode_id(const TcArgs& a, int64_t id) {
    if (MODE == kModeDense) {
      rb = (int)(id / a.n_ctiles);
      cb = (int)(id % a.n_ctiles);
    } else {
      int64_t lo = 0, hi = a.n_rtiles - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        const int64_t s = mid * a.n_ctiles - (int64_t)MB * mid * (mid - 1) / 2;
        if (s <= id) lo = mid; else hi = mid - 1;
      }
      rb = (int)lo;
      cb = (int)(lo * MB + (id - (lo * a.n_ctiles - (int64_t)MB * lo * (lo - 1) / 2)));
    }
  }
  // strided: first row block at or after `wave`; false when none is left
  __device__ bool start_row(const TcArgs& a) {
    const int G = gridDim.x, k = blockIdx.x;
    for (;; ++wave) {
      if ((int64_t)wave * G >= a.n_rtiles - a.rb_base) return false;
      rb = (int)a.rb_base + wave * G + ((wave & 1) && (MODE != kModeMatvec || a.sym) ? G - 1 - k : k);
      if (rb < a.n_rtiles) break;
    }
    if (MODE == kModeMatvec) {
      cb = a.sym ? rb * MB : 0;  // sym: the upper triangle J >= I only
      chunk = cb / kChunkTiles;
      cb_end = (int)min((int64_t)(chunk + 1) * kChunkTiles, a.n_ctiles);
    } else {
      cb = is_packed(MODE) ? rb * MB : 0;
    }
    return true;
  }
  // matvec listed: first kept tile of the current item at or after x
  // (cb_end if none); pruned blocks are jumped over whole
  int ncb;  // next kept tile of the item after cb (cb_end: cb is its last)
  __device__ int find_kept(const TcArgs& a, int x) const {
    const uint8_t* row = a.pskip + ((int64_t)rb * MB * 128 / a.pB) * a.pnb;
    while (x < cb_end) {
      const int64_t T = (int64_t)x * 128 / a.pB;
      if (row[T] == 0) return x;
      x = (int)((T + 1) * a.pB / 128);
    }
    return cb_end;
  }
  __device__ void load_item(const TcArgs& a) {
    uid = a.unit_list[u];
    rb = (int)(uid / a.n_chunks);
    chunk = (int)(uid - (int64_t)rb * a.n_chunks);
    cb_end = (int)min((int64_t)(chunk + 1) * kChunkTiles, a.n_ctiles);
    const int first = max(chunk * kChunkTiles, rb * MB);
    cb = find_kept(a, first);
    ncb = find_kept(a, cb + 1);
  }
  __device__ void begin(const TcArgs& a, int64_t u0, int64_t u1) {
    listed = run_listed<MODE>(a);
    if (listed) {
      strided = false;
      u = u0;
      u_end = u1;
      if (u < u_end) {
        if constexpr (MODE == kModeMatvec) {
          load_item(a);
        } else {
          uid = a.unit_list[u];
          decode_id(a, uid);
        }
      }
      return;
    }
    strided = MODE == kModeMatvec || a.strided;
    if (strided) {
      wave = 0;
      u_end = 1;
      u = start_row(a) ? 0 : 1;
      return;
    }
    u = u0;
    u_end = u1;
    if (u < u_end) decode_unit(a);
  }
  __device__ bool valid() const { return u < u_end; }
  __device__ bool item_last() const {
    if (MODE != kModeMatvec) return true;
    return listed ? ncb >= cb_end : cb + 1 == cb_end;
  }
  // units are walked in order, so the successor is found without the
  // division / search of decode_unit (which runs once, in begin())
  __device__ void next(const TcArgs& a) {
    if (MODE == kModeMatvec && listed) {
      if (ncb < cb_end) {
        cb = ncb;
        ncb = find_kept(a, cb + 1);
      } else if (++u < u_end) {
        load_item(a);
      }
      return;
    }
    if (MODE == kModeMatvec) {
      if (cb + 1 < cb_end) {
        ++cb;
      } else if (++chunk < a.n_chunks) {
        cb = chunk * kChunkTiles;
        cb_end = (int)min((int64_t)cb + kChunkTiles, a.n_ctiles);
      } else {
        ++wave;
        if (!start_row(a)) u = 1;
      }
      return;
    }
    if (listed) {  // packed units
      if (++u >= u_end) return;
      const int64_t id = a.unit_list[u];
      if (id == uid + 1 && cb + 1 < a.n_ctiles) {
        ++cb;
      } else {
        decode_id(a, id);
      }
      uid = id;
      return;
    }
    if (strided) {
      if (++cb == a.n_ctiles) {
        ++wave;
        if (!start_row(a)) u = 1;
      }
      return;
    }
    ++u;
    if (u >= u_end) return;
    if (++cb == a.n_ctiles) {
      ++rb;
      cb = is_packed(MODE) ? rb * MB : 0;
    }
  }
};

// the feed ring sits behind the pipeline barriers and the TMEM slot word
// (2 ST + 8 words; with ST <= 4 it ends within the 256-byte barrier area)
__device__ inline uint64_t* tmem_slot_bars(uint64_t* bars, int st) { return bars + 2 * st + 8; }

template <int MB, int MODE>
__host__ __device__ inline int64_t total_units(const TcArgs& a) {
  if (is_packed(MODE)) return packed_items(a.n_rtiles, a.n_ctiles, MB);
  if (MODE == kModeMatvec) return a.n_rtiles * a.n_chunks;  // (strided: unused)
  return a.n_rtiles * a.n_ctiles;
}

template <int KB, int MODE, int KIND>
__global__ void __launch_bounds__(kCtaThreads<MODE>, 1)
    affinity_tc_kernel(const __grid_constant__ CUtensorMap map_hi,
                       const __grid_constant__ CUtensorMap map_lo,
                       const __grid_constant__ CUtensorMap map_out,
                       const __grid_constant__ CUtensorMap map_nrm, const TcArgs args) {
  constexpr bool kNorm = KIND == GPIC_KIND_RBF;  // the distance comes out of the MMA
  constexpr int MB = mblocks(KB, MODE);
  constexpr int ST = stages(KB, MODE);
  constexpr int kTmemCols = 2 * MB * kBN;  // 2 accumulators
  if (MODE == kModeMatvec && args.ctl != nullptr && *(volatile const int32_t*)&args.ctl->stop)
    return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = smem_align<1024>(smem_raw);
  uint8_t* sA = base;                                     // [hl][m][kb] 16 KB tiles
  uint8_t* sAn = sA + a_main_bytes(KB, MODE);                   // [m][hl] 4 KB norm planes
  uint8_t* sB = sA + a_bytes(KB, MODE);                         // [stage]{hi, lo, norm hi, norm lo}
  uint8_t* sOut = sB + ST * kStageBytes;                  // [epi warp] staging / combine
  float* sCol = reinterpret_cast<float*>(sOut + out_bytes(KB, MODE));  // matvec: [warp][buf][v][64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sCol) + col_bytes(MODE));
  uint64_t* full = bars;                 // [ST]
  uint64_t* empty = bars + ST;           // [ST]
  uint64_t* a_full = bars + 2 * ST;
  uint64_t* a_empty = a_full + 1;
  uint64_t* t_full = a_full + 2;         // [2]
  uint64_t* t_empty = a_full + 4;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 6);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // listed (pruned) runs split the list of kept units, else the unit range
  const bool listed = run_listed<MODE>(args);
  const int64_t total = listed ? *args.unit_count : total_units<MB, MODE>(args) - args.u_lo;
  const int64_t u0 = listed ? 0 : args.u_lo;
  int64_t u_begin = u0 + total * blockIdx.x / gridDim.x;
  int64_t u_end = u0 + total * (blockIdx.x + 1) / gridDim.x;
  if (listed && args.wpre != nullptr) {  // equal shares of kept tiles, not of items
    int64_t ua, ub;  // this rank's share of the list (all of it on one rank)
    item_share(args, total, ua, ub);
    if (args.cuts != nullptr && args.cuts[0] == gridDim.x && args.cuts[1] == ua &&
        args.cuts[2] == ub) {
      // cuts re-balanced by the previous pass's measured CTA times
      u_begin = args.cuts[3 + blockIdx.x];
      u_end = args.cuts[4 + blockIdx.x];
    } else {
      const int64_t Wa = args.wpre[ua], W = args.wpre[ub] - Wa;
      u_begin = lower_bound_w(args.wpre, ua, ub, Wa + W * blockIdx.x / gridDim.x);
      u_end = blockIdx.x + 1 == gridDim.x ? ub
                                          : lower_bound_w(args.wpre, ua, ub, Wa + W * (blockIdx.x + 1) / gridDim.x);
    }
  }

  // dynamic claims (listed runs): the range is this rank's share
  static_assert(2 * ST + 8 + 2 * kFeedSlots + kFeedSlots <= 32, "feed ring outside the barrier area");
  // packed store modes only: in the matrix-free pass the claims measured
  // slower at config 5 (its tile-balanced static split keeps the column
  // operands' L2 reuse; 162 -> 198 ms per run), and the feed's registers
  // cost the register-tight matvec epilogue even when unused
  constexpr bool kDynMode = MODE != kModeMatvec;
  const bool dyn = kDynMode && listed && args.sched != nullptr;
  int64_t d_lo = 0, d_hi = total;
  if (dyn && args.wpre != nullptr) item_share(args, total, d_lo, d_hi);
  Feed feed;
  feed.full = tmem_slot_bars(bars, ST);
  if (threadIdx.x == 0) {
    if (dyn)
      for (int q = 0; q < kFeedSlots; ++q) {
        mbar_init(&feed.full[q], 1);
        mbar_init(feed.empty_bar(q), 1 + kEpiWarps);
      }
    for (int s = 0; s < ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&t_full[b], 1);
      mbar_init(&t_empty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_hi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_lo)) : "memory");
    if (MODE != kModeMatvec)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_out)) : "memory");
    if (kNorm)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_nrm)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // every role ends here (no code after the role branches: the warpgroups
  // run with different register budgets after setmaxnreg)
  // the CTA's span (thread 0): the matrix-free rebalance reads it
  uint64_t trace_t0 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(trace_t0));
  auto teardown = [&]() {
    tc_fence_before();
    asm volatile("barrier.sync 15, %0;" ::"n"(kCtaThreads<MODE>) : "memory");
    if (MODE == kModeMatvec && args.cta_ns != nullptr && threadIdx.x == 0) {
      uint64_t t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      args.cta_ns[blockIdx.x] = t1 - trace_t0;
    }
#ifdef GPIC_TC_TRACE
    if (threadIdx.x == 0) {
      uint64_t t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      const int64_t tiles = args.wpre != nullptr ? args.wpre[u_end] - args.wpre[u_begin] : -1;
      int64_t rbs = 0, prev = -1;
      if (listed && MODE == kModeMatvec)
        for (int64_t u = u_begin; u < u_end; ++u) {
          const int64_t rb = args.unit_list[u] / args.n_chunks;
          rbs += rb != prev;
          prev = rb;
        }
      printf("TCTRACE %d %llu %lld %lld %lld %lld\n", (int)blockIdx.x,
             (unsigned long long)(t1 - trace_t0), (long long)(u_end - u_begin), (long long)tiles,
             (long long)rbs, (long long)u_begin);
    }
#endif
    if (warp == 1) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(kTmemCols)
                   : "memory");
    }
  };

  if (warp < kEpiBase<MODE>) {
  // warpgroup 0 gives registers back in one instruction all its warps share
  if constexpr (kSplitRegs<MODE>) setmaxnreg_dec<kCtlRegs>();
  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      int64_t cur_rb = -1;
      uint32_t a_par = 1;
      int s = 0;
      uint32_t ph = 0;
      // the operands (MBs) are re-read by every CTA: keep them in L2 against
      // the GB-scale output stream
      const uint64_t keep = policy_evict_last();
      Cursor<MB, MODE> c;
      // dynamic: claim the next range, hand it to the other roles; at the
      // end the last CTA to finish claiming resets the counters
      auto claim = [&]() {
        int64_t e0, e1;
        const int64_t k = (int64_t)atomicAdd(args.sched, 1u);
        if (claim_range(k, d_lo, d_hi, gridDim.x, e0, e1)) {
          feed.write(e0, e1);
          c.begin(args, e0, e1);
        } else {
          feed.write(-1, -1);
          c.u = c.u_end = 0;
          if (atomicAdd(args.sched + 1, 1u) == gridDim.x - 1) {
            atomicExch(args.sched, 0u);
            atomicExch(args.sched + 1, 0u);
          }
        }
      };
      if (dyn) claim(); else c.begin(args, u_begin, u_end);
      for (; c.valid(); ) {
        if (c.rb != cur_rb) {
          mbar_wait_sleep(a_empty, a_par);
          a_par ^= 1;
          mbar_expect_tx(a_full, kNorm ? a_bytes(KB, MODE) : a_main_bytes(KB, MODE));
          for (int hl = 0; hl < 2; ++hl)
            for (int m = 0; m < MB; ++m) {
              const int row0 = (int)(args.row_lo + (c.rb * MB + m) * 128);
              for (int kb = 0; kb < KB; ++kb)
                tma_load_2d(sA + ((hl * MB + m) * KB + kb) * kTileBytes, hl ? &map_lo : &map_hi,
                            kb * kKBlk, row0, a_full, keep);
              if (kNorm)  // row-operand norm planes 0 (hi) / 1 (lo)
                tma_load_2d(sAn + (m * 2 + hl) * kNrmPlane, &map_nrm, 0,
                            (int)(hl * args.n_pad) + row0, a_full, keep);
            }
          cur_rb = c.rb;
        }
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait_sleep(&empty[s], ph ^ 1);
          const bool nrm = kNorm && kb == KB - 1;
          mbar_expect_tx(&full[s], 2 * kTileBytes + (nrm ? kNrmBytes : 0));
          uint8_t* stg = sB + s * kStageBytes;
          tma_load_2d(stg, &map_hi, kb * kKBlk, (int)(c.cb * kBN), &full[s], keep);
          tma_load_2d(stg + kTileBytes, &map_lo, kb * kKBlk, (int)(c.cb * kBN), &full[s], keep);
          if (nrm)  // column-operand norm planes 2 (hi) / 3 (lo)
            for (int hl = 0; hl < 2; ++hl)
              tma_load_2d(stg + 2 * kTileBytes + hl * kNrmPlane, &map_nrm, 0,
                          (int)((2 + hl) * args.n_pad + c.cb * kBN), &full[s], keep);
          if (++s == ST) { s = 0; ph ^= 1; }
        }
        c.next(args);
        if (dyn && !c.valid()) claim();
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
      int64_t cur_rb = -1;
      uint32_t a_par = 0;
      uint32_t te_bits = 3u;  // TMEM-empty parity per accumulator buffer
      int s = 0;
      uint32_t ph = 0;
      int i = 0;
      Cursor<MB, MODE> c;
      auto pull = [&]() {
        int64_t e0, e1;
        if (feed.read(e0, e1, true)) c.begin(args, e0, e1); else c.u = c.u_end = 0;
      };
      if (dyn) pull(); else c.begin(args, u_begin, u_end);
      for (; c.valid(); ++i) {
        const int64_t rb = c.rb;
        if (rb != cur_rb) {
          mbar_wait_sleep(a_full, a_par);
          a_par ^= 1;
          cur_rb = rb;
        }
        const int buf = i & 1;
        mbar_wait_sleep(&t_empty[buf], (te_bits >> buf) & 1u);
        te_bits ^= 1u << buf;
        tc_fence_after();
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait_sleep(&full[s], ph);
          tc_fence_after();
          uint8_t* stg = sB + s * kStageBytes;
          const uint64_t bh = sw128_desc(su32(stg));
          const uint64_t bl = sw128_desc(su32(stg + kTileBytes));
#pragma unroll
          for (int m = 0; m < MB; ++m) {
            const uint32_t d = tmem_base + (uint32_t)((buf * MB + m) * kBN);
            const uint64_t ah = sw128_desc(su32(sA + ((0 * MB + m) * KB + kb) * kTileBytes));
            const uint64_t al = sw128_desc(su32(sA + ((1 * MB + m) * KB + kb) * kTileBytes));
#pragma unroll
            for (int k = 0; k < kKBlk / 16; ++k) {
              const uint64_t off = (uint64_t)(k * 16 * 2 >> 4);  // 32 bytes along K
              mma_f16(d, ah + off, bl + off, kIdesc, (kb | k) != 0);
              mma_f16(d, al + off, bh + off, kIdesc, 1u);
              mma_f16(d, ah + off, bh + off, kIdesc, 1u);
            }
            if (kNorm && kb == KB - 1) {  // + the norm block: acc = -(s^2/2)|x_i - x_j|^2
              const uint64_t nah = sw32_desc(su32(sAn + (m * 2 + 0) * kNrmPlane));
              const uint64_t nal = sw32_desc(su32(sAn + (m * 2 + 1) * kNrmPlane));
              const uint64_t nbh = sw32_desc(su32(stg + 2 * kTileBytes));
              const uint64_t nbl = sw32_desc(su32(stg + 2 * kTileBytes + kNrmPlane));
              mma_f16(d, nah, nbl, kIdesc, 1u);
              mma_f16(d, nal, nbh, kIdesc, 1u);
              mma_f16(d, nah, nbh, kIdesc, 1u);
            }
          }
          tc_commit(&empty[s]);  // frees the B stage once these MMAs retire
          if (++s == ST) { s = 0; ph ^= 1; }
        }
        tc_commit(&t_full[buf]);
        c.next(args);
        if (dyn && !c.valid()) pull();
        if (!c.valid() || c.rb != rb) tc_commit(a_empty);  // last tile of this row block
      }
    }
  }  // split mode: warps 2-3 are idle, they only complete warpgroup 0
  teardown();
  } else {
    // --------------------------------------------------------- epilogue
    if constexpr (kSplitRegs<MODE>) setmaxnreg_inc<kEpiRegs>();
    // Warp w may only read TMEM lanes 32*(w%4)..+31: q = w & 3 picks this
    // warp's 32 rows; the 4 warps of a quadrant (h = e >> 2) split the
    // tile's MB x 4 chunks of 32 columns, MB chunks each. The GW = 4 / MB
    // warps that cover the same rows combine their row sums in fixed order.
    //
    // Accumulators are read with tcgen05.ld.16x256b (two 16-lane halves x4):
    // thread t holds rows hf*16 + t/4 (+8) and, per 8-column block b, the
    // two columns 8b + 2(t%4) + {0,1}. So every thread owns just 4 rows and
    // 8 columns: row / column terms stay in registers (no per-element
    // broadcasts) and the column-degree partials are a 7-shuffle
    // reduce-scatter instead of a re-read of the staged tile. Values go out
    // through a swizzled 32 x 32 staging box (8-byte st.shared, conflict-free)
    // and a TMA bulk-tensor store (direct 8-byte global stores were measured
    // slower: one L1 wavefront per row segment).
    constexpr int UPW = MB;
    constexpr int GW = 4 / MB;
    const int e = warp - kEpiBase<MODE>;
    const int q = warp & 3;
    const int h = e >> 2;
    const int m = (h * UPW) >> 2;
    const int c_lo = (h * UPW) & 3;
    const int gi = h % GW;                   // position in the row group
    const uint32_t bar_id = 1 + q * MB + m;  // named barrier of the row group
    const int tq = lane >> 2;                // row within a 16-lane half (and +8)
    const int tc = (lane & 3) * 2;           // first of this thread's 2 columns per block
    double* comb = reinterpret_cast<double*>(sOut);  // matvec: [warp][32 rows] row-sum combine
    uint8_t* stage = sOut + e * kStageOutBytes;       // store modes: this warp's staging box
    const uint64_t stream_pol = policy_evict_first();  // A is written once here
    int stores = 0;
    const float gs = __ldg(args.gscale);  // accumulator units -> G (1 / s^2)
    const float m2ns = -2.f * args.ns * gs;
    uint32_t tf_bits = 0;  // TMEM-full parity per accumulator buffer
    int i = 0;
    // matvec: the 4 rows' partials over an item as unevaluated fp32 pairs
    // (hi + lo, TwoSum per tile: ~46 significant bits, FMA pipe only) and
    // converted to fp64 once per item — an fp64 add per tile waits on a
    // f32 -> f64 conversion queued behind the saturated ex2 pipe
    float acc_hi[4] = {0.f, 0.f, 0.f, 0.f}, acc_lo[4] = {0.f, 0.f, 0.f, 0.f};
    auto group_sync = [&]() {
      asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(GW * 32) : "memory");
    };
    float vrow[4] = {0.f, 0.f, 0.f, 0.f};  // matvec sym: v_i of the 4 rows (column partials)
    int grow[4] = {0, 0, 0, 0};  // row / column indices fit 32 bits (n < 2^31)
    const int n32 = (int)args.n, row_lo32 = (int)args.row_lo;
    // matvec sym: the warps holding the same columns (all quadrants, both M
    // blocks) exchange column partials through smem; one writer per group
    float* colx = reinterpret_cast<float*>(sOut + kEpiWarps * 32 * 8);
    const uint32_t colbar = 9 + c_lo / UPW;
    const bool col_writer = q == 0 && m == 0;
    int cur_rb = -1;
    // matvec: v_j of a tile arrives one tile ahead by cp.async into this
    // warp's double buffer: lane l copies column l of each of its chunks
    float* colw = sCol + e * (2 * 64);
    auto fetch_cols = [&](int64_t cbn, int slot) {
      if constexpr (MODE == kModeMatvec) {
        float* dst = colw + slot * 64;
#pragma unroll
        for (int cc = 0; cc < UPW; ++cc)
          cp_async4(dst + cc * 32 + lane, args.v32 + cbn * kBN + (c_lo + cc) * 32 + lane);
        cp_async_commit();
      }
    };
    Cursor<MB, MODE> c;
    auto pull = [&]() {
      int64_t e0, e1;
      if (feed.read(e0, e1, lane == 0)) c.begin(args, e0, e1); else c.u = c.u_end = 0;
    };
    if (dyn) pull(); else c.begin(args, u_begin, u_end);
    if (c.valid()) fetch_cols(c.cb, 0);
    for (; c.valid(); ++i) {
      const int rb = c.rb, cb = c.cb;
      const bool item_last = c.item_last();
      const int chunk = c.chunk;
      const int buf = i & 1;
      const int tI = rb * MB + m;  // tile row of this warp's rows
      // packed: the lower-triangle half of a diagonal row block is not stored
      const bool store_ok = !is_packed(MODE) || tI <= cb;
      // packed: this warp's tile, global (flags) and shard-relative (values,
      // degree partials) — once per unit, not per chunk
      const int64_t tg = is_packed(MODE) && store_ok ? tile_index(tI, cb, args.n_ctiles) : 0;
      const int64_t tl = tg - args.tile_base;
      // matvec sym: row partials from tiles J >= I, column partials from J > I
      const bool row_ok = MODE != kModeMatvec || !args.sym || tI <= cb;
      const bool col_ok = MODE == kModeMatvec && args.sym && tI < cb;
      const int lr0 = (rb * MB + m) * 128 + q * 32;  // shard-local first row of this warp
      if (rb != cur_rb) {
        // this thread's 4 rows: rr = 2*half + {0: tq, 1: tq + 8}
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          grow[rr] = row_lo32 + lr0 + (rr >> 1) * 16 + tq + (rr & 1) * 8;
          if (MODE == kModeMatvec) vrow[rr] = grow[rr] < n32 ? __ldg(args.v32 + grow[rr]) : 0.f;
        }
        cur_rb = rb;
      }
      c.next(args);
      if (dyn && !c.valid()) pull();
      if constexpr (MODE == kModeMatvec) {
        if (c.valid()) {
          fetch_cols(c.cb, (i + 1) & 1);
          cp_async_wait<1>();  // this tile's group has landed
        } else {
          cp_async_wait<0>();
        }
        __syncwarp();
      }
      const float* colt = colw + (i & 1) * 64;
      mbar_wait_sleep(&t_full[buf], (tf_bits >> buf) & 1u);
      tf_bits ^= 1u << buf;
      tc_fence_after();
      float rsum[4] = {0.f, 0.f, 0.f, 0.f};  // this thread's 4 rows, its 8 columns per chunk
      // chunk cc's 32 values per thread, [hf][block b][4]: (row tq, c),
      // (row tq, c+1), (row tq+8, c), (row tq+8, c+1); the next chunk's
      // TMEM load is in flight while this one is processed
      uint32_t rbuf[2][32];
      auto tmem_chunk = [&](int cc, uint32_t* r) {
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) +
                               (uint32_t)((buf * MB + m) * kBN + (c_lo + cc) * 32);
        tmem_ld16x256_x4(taddr, r);
        tmem_ld16x256_x4(taddr + (16u << 16), r + 16);
      };
      auto tmem_done = [&]() {  // accumulator fully read: hand it back to the MMA warp
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&t_empty[buf]);
      };
      // one 32-column chunk of this warp's rows: exp, masks, sums, stores
      auto process_chunk = [&](const int cc, const uint32_t* r) {
        const int ch = c_lo + cc;
        const int col0 = cb * kBN + ch * 32;
        // matvec: this thread's 8 columns' v_j from the staged copy
        float vcol[8];
        if constexpr (MODE == kModeMatvec) {
#pragma unroll
          for (int b2 = 0; b2 < 4; ++b2) {
            const float2 v2 = *reinterpret_cast<const float2*>(colt + cc * 32 + 8 * b2 + tc);
            vcol[2 * b2] = v2.x;
            vcol[2 * b2 + 1] = v2.y;
          }
        }
        // RBF, stored-tile / matrix-free modes: the flush to exact zeros is
        // decided per 32 x 32 box — a box whose every entry is below 2^-64
        // is zero (skipped: no exp, no sums, no store; flags 0 in boxnz, zero
        // column partials); a box with one entry above keeps all its entries
        // (ex2.approx.ftz still flushes below 2^-126). The dropped mass of a
        // row stays below n 2^-64, as with a per-element flush, and every
        // storage and pass sees the same boxes, so runs agree bit for bit.
        bool box_big = true;
        if constexpr (KIND == GPIC_KIND_RBF && MODE != kModeDense) {
          float gm = __uint_as_float(r[0]);
#pragma unroll
          for (int x = 1; x < 32; ++x) gm = fmaxf(gm, __uint_as_float(r[x]));
          box_big = __any_sync(0xffffffffu, gm * m2ns >= kFlushLog2);
          if (!box_big) {
            if constexpr (MODE == kModeMatvec) {
              if (args.sym) colx[((buf * MB + m) * 4 + q) * 128 + ch * 32 + lane] = 0.f;
              return;
            } else {
              if (args.boxnz != nullptr) {
                if (lane == 0 && store_ok)
                  args.boxnz[tg * 16 + q * 4 + ch] = 0;
                if (store_ok && tI != cb)
                  args.degcol[(tl * 4 + q) * 128 +
                              ch * 32 + lane] = 0.f;
                return;
              }
            }
          }
        }
        const bool diag = (col0 < row_lo32 + lr0 + 32) && (row_lo32 + lr0 < col0 + 32);
        const bool pad = col0 + 32 > n32 || row_lo32 + lr0 + 32 > n32;
        float vals[32];
#pragma unroll
        for (int x = 0; x < 32; ++x) {
          const float g = __uint_as_float(r[x]);
          if constexpr (KIND == GPIC_KIND_COSINE)
            vals[x] = fmaxf(g * gs, 0.f);  // unit rows: G = cos, clamped (affinity.py:93-94)
          else if constexpr (MODE == kModeDense)
            // g = -(s^2/2)|x_i - x_j|^2 from the MMA (norm block); no clamp:
            // a near-duplicate's distance^2 rounding below 0 gives
            // exp2(+ulp-scale) = 1 + O(1e-6), the Gram's own rounding order
            vals[x] = ex2_flush(g * m2ns);
          else
            vals[x] = box_big ? ex2(g * m2ns) : 0.f;  // box-level flush (above)
        }
        if (diag || pad) {
#pragma unroll
          for (int x = 0; x < 32; ++x) {
            const int rr = (x >> 4) * 2 + ((x >> 1) & 1);
            const int col = col0 + ((x >> 2) & 3) * 8 + tc + (x & 1);
            if (col == grow[rr] || col >= n32 || grow[rr] >= n32) vals[x] = 0.f;
          }
        }
        if constexpr (MODE == kModePacked16) {
          // degrees from the stored (rounded) values: W = D^-1 A stays
          // exactly row-stochastic in the stored precision
#pragma unroll
          for (int x = 0; x < 32; x += 2) {
            const float2 f = __half22float2(__floats2half2_rn(vals[x], vals[x + 1]));
            vals[x] = f.x;
            vals[x + 1] = f.y;
          }
        }
        if constexpr (MODE == kModeMatvec) {
          if (row_ok) {
#pragma unroll
            for (int x = 0; x < 32; ++x) {
              const int rr = (x >> 4) * 2 + ((x >> 1) & 1);
              const int k = ((x >> 2) & 3) * 2 + (x & 1);
              rsum[rr] = fmaf(vals[x], vcol[k], rsum[rr]);
            }
          }
          if (args.sym) {
            // column partials sum_i a_ij v_i over this warp's 32 rows (same
            // fixed reduce-scatter as the packed degree partials)
            float cs[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int x0 = (k >> 1) * 4 + (k & 1);
              cs[k] = col_ok ? fmaf(vals[x0], vrow[0], vals[x0 + 2] * vrow[1]) +
                                   fmaf(vals[x0 + 16], vrow[2], vals[x0 + 18] * vrow[3])
                             : 0.f;
            }
            const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float send = b4 ? cs[k] : cs[k + 4];
              const float keep = b4 ? cs[k + 4] : cs[k];
              cs[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const float send = b3 ? cs[k] : cs[k + 2];
              const float keep = b3 ? cs[k + 2] : cs[k];
              cs[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
            {
              const float send = b2 ? cs[0] : cs[1];
              const float keep = b2 ? cs[1] : cs[0];
              cs[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
            }
            const int k = (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0);
            const int col = 8 * (k >> 1) + tc + (k & 1);
            colx[((buf * MB + m) * 4 + q) * 128 + ch * 32 + col] = cs[0];
          }
        } else {
#pragma unroll
          for (int x = 0; x < 32; ++x) rsum[(x >> 4) * 2 + ((x >> 1) & 1)] += vals[x];
          // sparse: a box of exact zeros is not stored, only flagged
          bool box_nz = true;
          if (is_packed(MODE) && args.boxnz != nullptr) {
            bool any = false;
#pragma unroll
            for (int x = 0; x < 32; ++x) any |= vals[x] != 0.f;
            box_nz = __any_sync(0xffffffffu, any);
            if (lane == 0 && store_ok)
              args.boxnz[tg * 16 + q * 4 + ch] = box_nz ? 1 : 0;
          }
          // full 32-byte sectors straight from registers: each quad writes 8
          // consecutive floats of one row per (block, row)
          // stage the 32 x 32 box (row R at R*128, 16-byte chunk c/4 ^ (R&7))
          if (box_nz) {
          if (stores > 0) {  // the previous TMA store must have read the box
            if (lane == 0) tma_store_wait_read<0>();
            __syncwarp();
          }
          if constexpr (MODE == kModePacked16) {
            // fp16 box: 32 rows x 64 B, 64-byte swizzle (16-byte chunk ^
            // (R >> 1) & 3); 4-byte stores, conflict-free
#pragma unroll
            for (int x = 0; x < 32; x += 2) {
              const int R = (x >> 4) * 16 + tq + ((x >> 1) & 1) * 8;
              const int blk = (x >> 2) & 3;
              const uint32_t addr = su32(stage) + R * 64 + ((blk ^ ((R >> 1) & 3)) << 4) + tc * 2;
              const __half2 h = __floats2half2_rn(vals[x], vals[x + 1]);
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr),
                           "r"(*reinterpret_cast<const uint32_t*>(&h))
                           : "memory");
            }
          } else {
            // a 64-bit store is served 16 lanes at a time: with every lane on
            // the same column block, lanes (tq, upper pair) and (tq ^ 1,
            // lower pair) hit one 16-byte chunk (2-way conflict). The upper
            // column pair of each quad stores block blk ^ 2 in the same
            // instruction instead, which moves it to the other 64 bytes.
            const bool up = tc & 4;
#pragma unroll
            for (int x = 0; x < 32; x += 2) {
              const int xs = x ^ 8;
              const int R = (x >> 4) * 16 + tq + ((x >> 1) & 1) * 8;
              const int blk = ((x >> 2) & 3) ^ (up ? 2 : 0);
              const int cq = blk * 2 + (tc >> 2);  // 16-byte chunk of the columns
              const uint32_t addr = su32(stage) + R * 128 + ((cq ^ (R & 7)) << 4) + (tc & 3) * 4;
              const float v0 = up ? vals[xs] : vals[x];
              const float v1 = up ? vals[xs + 1] : vals[x + 1];
              asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v0), "f"(v1)
                           : "memory");
            }
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0 && store_ok) {
            const int64_t out_row0 = is_packed(MODE)
                                         ? tl * 128 + q * 32
                                         : lr0;
            if (args.store_hint)
              tma_store_2d(&map_out, is_packed(MODE) ? ch * 32 : (int)col0, (int)out_row0, stage,
                           stream_pol);
            else
              tma_store_2d(&map_out, is_packed(MODE) ? ch * 32 : (int)col0, (int)out_row0, stage);
          }
          ++stores;
          }  // box_nz
          if (is_packed(MODE) && store_ok && tI != cb) {
            // degrees of the tile's COLUMN rows (A is symmetric): per column
            // slot k, this thread's 4 rows, then a reduce-scatter over the 8
            // threads sharing the slot (xor 16, 8, 4): thread (tq, quad) ends
            // with the 32-row total of slot k = tq. Fixed order.
            float cs[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int x0 = (k >> 1) * 4 + (k & 1);  // half 0, row tq
              cs[k] = (vals[x0] + vals[x0 + 2]) + (vals[x0 + 16] + vals[x0 + 18]);
            }
            const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // slots k | 4 go up when lane bit 4 is set
              const float send = b4 ? cs[k] : cs[k + 4];
              const float keep = b4 ? cs[k + 4] : cs[k];
              cs[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const float send = b3 ? cs[k] : cs[k + 2];
              const float keep = b3 ? cs[k + 2] : cs[k];
              cs[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
            }
            {
              const float send = b2 ? cs[0] : cs[1];
              const float keep = b2 ? cs[1] : cs[0];
              cs[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
            }
            const int k = (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2 ? 1 : 0);  // = tq
            const int col = 8 * (k >> 1) + tc + (k & 1);
            args.degcol[(tl * 4 + q) * 128 + ch * 32 + col] = cs[0];
          }
        }
      };
      if constexpr (kSplitRegs<MODE>) {
        tmem_chunk(0, rbuf[0]);
        tmem_wait_ld(rbuf[0]);
        if (UPW == 1) tmem_done();
#pragma unroll
        for (int cc = 0; cc < UPW; ++cc) {
          if (cc + 1 < UPW) tmem_chunk(cc + 1, rbuf[(cc + 1) & 1]);
          process_chunk(cc, rbuf[cc & 1]);
          if (cc + 1 < UPW) {
            tmem_wait_ld(rbuf[(cc + 1) & 1]);
            if (cc + 1 == UPW - 1) tmem_done();
          }
        }
      } else {
#pragma unroll 1
        for (int cc = 0; cc < UPW; ++cc) {
          tmem_chunk(cc, rbuf[0]);
          tmem_wait_ld(rbuf[0]);
          if (cc == UPW - 1) tmem_done();
          process_chunk(cc, rbuf[0]);
        }
      }
      // this thread's row partials -> the quad's row totals (xor 1, 2)
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        rsum[rr] += __shfl_xor_sync(0xffffffffu, rsum[rr], 1);
        rsum[rr] += __shfl_xor_sync(0xffffffffu, rsum[rr], 2);
      }
      const bool quad_lead = (lane & 3) == 0;
      if constexpr (MODE == kModeMatvec) {
        if (args.sym) {
          // combine the column partials of the 4 * MB warps sharing these
          // columns (M block, then quadrant order) into one record
          asm volatile("bar.sync %0, %1;" ::"r"(colbar), "r"(4 * MB * 32) : "memory");
          if (col_writer) {
            const int64_t rec = (int64_t)rb * args.n_ctiles - (int64_t)MB * rb * (rb - 1) / 2 +
                                (cb - (int64_t)rb * MB);
#pragma unroll
            for (int cc = 0; cc < UPW; ++cc) {
              const int cidx = (c_lo + cc) * 32 + lane;
              float t = 0.f;
#pragma unroll
              for (int mm = 0; mm < MB; ++mm)
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) t += colx[((buf * MB + mm) * 4 + qq) * 128 + cidx];
              args.colpart[rec * 128 + cidx] = t;
            }
          }
        }
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const float t = acc_hi[rr] + rsum[rr];
          const float bb = t - acc_hi[rr];
          acc_lo[rr] += (acc_hi[rr] - (t - bb)) + (rsum[rr] - bb);
          acc_hi[rr] = t;
        }
        if (item_last) {
          double acc64[4];
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) acc64[rr] = (double)acc_hi[rr] + (double)acc_lo[rr];
          double tot[4] = {acc64[0], acc64[1], acc64[2], acc64[3]};
          if (GW > 1) {
            if (quad_lead)
#pragma unroll
              for (int rr = 0; rr < 4; ++rr)
                comb[e * 32 + (rr >> 1) * 16 + tq + (rr & 1) * 8] = acc64[rr];
            group_sync();
            if (gi == 0 && quad_lead)
              for (int g2 = 1; g2 < GW; ++g2)
#pragma unroll
                for (int rr = 0; rr < 4; ++rr)
                  tot[rr] += comb[(e + 4 * g2) * 32 + (rr >> 1) * 16 + tq + (rr & 1) * 8];
            group_sync();
          }
          if (gi == 0 && quad_lead)
#pragma unroll
            for (int rr = 0; rr < 4; ++rr) {
              const int64_t lrow = lr0 + (rr >> 1) * 16 + tq + (rr & 1) * 8;
              if (lrow < args.rows) args.ypart[(int64_t)chunk * args.rows_pad + lrow] = tot[rr];
            }
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) acc_hi[rr] = acc_lo[rr] = 0.f;
        }
      } else if (MODE == kModeDense || store_ok) {
        // row sums of the tile's rows: the group's warps combine in order
        float tot[4] = {rsum[0], rsum[1], rsum[2], rsum[3]};
        if (GW > 1) {
          // partials go through each writer's staging box once it is drained
          if (gi > 0) {
            if (lane == 0) tma_store_wait_read<0>();
            __syncwarp();
            if (quad_lead) {
              float* cf = reinterpret_cast<float*>(stage);
#pragma unroll
              for (int rr = 0; rr < 4; ++rr) cf[(rr >> 1) * 16 + tq + (rr & 1) * 8] = rsum[rr];
            }
          }
          group_sync();
          if (gi == 0 && quad_lead)
            for (int g2 = 1; g2 < GW; ++g2) {
              const float* cf = reinterpret_cast<const float*>(sOut + (e + 4 * g2) * kStageOutBytes);
#pragma unroll
              for (int rr = 0; rr < 4; ++rr) tot[rr] += cf[(rr >> 1) * 16 + tq + (rr & 1) * 8];
            }
          group_sync();
        }
        if (gi == 0 && quad_lead)
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const int rloc = (rr >> 1) * 16 + tq + (rr & 1) * 8;  // row within the warp's 32
            if constexpr (is_packed(MODE)) {
              args.degrow[tl * 128 + q * 32 + rloc] = tot[rr];
            } else {
              const int64_t lrow = lr0 + rloc;
              if (lrow < args.rows) args.rowpart[cb * args.rows_pad + lrow] = tot[rr];
            }
          }
      }
    }
    if (MODE != kModeMatvec && lane == 0) tma_store_wait_all();
    __syncwarp();
    teardown();
  }
}

// ---------------------------------------------------------- host side
}  // namespace
bool tc_supports_pitch(int32_t dp, bool matvec);
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer,
              uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer,
              CUtensorMapDataType dtype = CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
              CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dtype, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_num_sms = 0;

template <int KB, int MODE>
int launch_kb(const CUtensorMap& mh, const CUtensorMap& ml, const CUtensorMap& mo,
              const CUtensorMap& mn, const TcArgs& a0, cudaStream_t s) {
  constexpr int MB = mblocks(KB, MODE);
  if (!tc_supports_pitch(KB * kKBlk, MODE == kModeMatvec))
    return fail(GPIC_E_UNSUPPORTED,
                "tcgen05 affinity engine: d too wide for this storage mode (SIMT engine: any d)");
  TcArgs a = a0;
  a.n_rtiles = ceil_div(a.rows, 128 * MB);
  a.n_chunks = ceil_div(a.n_ctiles, kChunkTiles);
  if (is_packed(MODE)) {  // shard = row blocks [row_lo / (128 MB), n_rtiles), rows stay global
    a.rb_base = a.row_lo / (128 * MB);
    a.u_lo = packed_items(a.rb_base, a.n_ctiles, MB);
    a.row_lo = 0;
  }
  static bool attr = false;
  if (!attr) {
    GPIC_CUDA_TRY(cudaFuncSetAttribute(affinity_tc_kernel<KB, MODE, GPIC_KIND_RBF>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_bytes(KB, MODE)));
    GPIC_CUDA_TRY(cudaFuncSetAttribute(affinity_tc_kernel<KB, MODE, GPIC_KIND_COSINE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_bytes(KB, MODE)));
    attr = true;
  }
  if (g_num_sms == 0) {
    int dev;
    GPIC_CUDA_TRY(cudaGetDevice(&dev));
    GPIC_CUDA_TRY(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  // strided order once there is at least one full wave of row blocks: the
  // CTAs of a wave stream the same B tiles together, so operand tiles come
  // from L2 instead of DRAM even next to a GB-scale output stream (config 3
  // packed: 745 -> 54 MB of DRAM reads, 4.01 -> 3.55 ms); small problems
  // keep the contiguous split, which uses every SM. The fp16 store mode is
  // epilogue-bound rather than store-bound and prefers the contiguous split's
  // balance (3.1 vs 3.4 ms) while its operands fit in ~L2/4.
  a.strided = MODE == kModePacked16
                  ? (int64_t)row_pad(a.n) * kKBlk * KB * 4 > (32ll << 20)
                  : a.n_rtiles - a.rb_base >= g_num_sms;
  if (const char* o = getenv("GPIC_TC_ORDER")) a.strided = atoi(o) != 0;  // tests: force an order
  a.store_hint = 1;
  if (const char* o = getenv("GPIC_TC_STORE_HINT")) a.store_hint = atoi(o) != 0;  // measurement
  if (run_listed<MODE>(a)) a.strided = 0;  // the list's order
  const int64_t total = run_listed<MODE>(a) ? g_num_sms
                        : (MODE == kModeMatvec || a.strided) ? a.n_rtiles - a.rb_base
                                                              : total_units<MB, MODE>(a) - a.u_lo;
  // listed: the kept-unit count is on the device; every SM gets a share
  const int grid = (int)(total < g_num_sms ? total : g_num_sms);
  if (grid < 1) return GPIC_OK;
  // the similarity kind is a template parameter: a runtime select would
  // evaluate both epilogues per element
  if (a.kind == GPIC_KIND_COSINE)
    affinity_tc_kernel<KB, MODE, GPIC_KIND_COSINE><<<grid, kCtaThreads<MODE>, smem_bytes(KB, MODE), s>>>(
        mh, ml, mo, mn, a);
  else
    affinity_tc_kernel<KB, MODE, GPIC_KIND_RBF><<<grid, kCtaThreads<MODE>, smem_bytes(KB, MODE), s>>>(
        mh, ml, mo, mn, a);
  count_launch();
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

struct Maps {
  CUtensorMap hi, lo, out, nrm;
};

template <int MODE>
int dispatch_kb(int KB, const Maps& mp, const TcArgs& args, cudaStream_t s) {
  switch (KB) {
    case 1: return launch_kb<1, MODE>(mp.hi, mp.lo, mp.out, mp.nrm, args, s);
    case 2: return launch_kb<2, MODE>(mp.hi, mp.lo, mp.out, mp.nrm, args, s);
    case 3: return launch_kb<3, MODE>(mp.hi, mp.lo, mp.out, mp.nrm, args, s);
    default: return launch_kb<4, MODE>(mp.hi, mp.lo, mp.out, mp.nrm, args, s);
  }
}

// The fp16 hi / lo planes live back to back in the d_xhi buffer, followed
// by the norm block's four 16-wide planes (prepare.cu).
int operand_maps(const float* xhi, int64_t n, int32_t dp, Maps* mp) {
  const int KB = dp / kKBlk;
  if (dp % kKBlk || KB < 1 || KB > 4)
    return fail(GPIC_E_UNSUPPORTED, "tcgen05 affinity engine supports d <= 256");
  const int64_t npad = row_pad(n);
  const uint16_t* hi = reinterpret_cast<const uint16_t*>(xhi);
  const uint16_t* lo = hi + npad * dp;
  const uint16_t* nrm = lo + npad * dp;
  if (!make_map(&mp->hi, hi, (uint64_t)dp, (uint64_t)npad, (uint64_t)dp * 2, kKBlk, 128,
                CU_TENSOR_MAP_DATA_TYPE_FLOAT16) ||
      !make_map(&mp->lo, lo, (uint64_t)dp, (uint64_t)npad, (uint64_t)dp * 2, kKBlk, 128,
                CU_TENSOR_MAP_DATA_TYPE_FLOAT16) ||
      !make_map(&mp->nrm, nrm, 16, (uint64_t)(4 * npad), 32, 16, 128,
                CU_TENSOR_MAP_DATA_TYPE_FLOAT16, CU_TENSOR_MAP_SWIZZLE_32B))
    return fail(GPIC_E_CUDA, "cuTensorMapEncodeTiled failed");
  mp->out = mp->hi;  // placeholder for the matvec mode (no stores)
  return GPIC_OK;
}

}  // namespace

int64_t packed_tiles(int64_t n) {
  const int64_t nt = ceil_div(n, kBN);
  return nt * (nt + 1) / 2;
}

// Symmetric packed output: tile (I, J), J >= I, stored as a contiguous
// 128 x 128 fp32 block at tile_index(I, J) (row-major over the triangle).
int packed_row_halves(int32_t /*dp*/) { return 1; }  // the epilogue combines a row's warps

// GPIC_TC_DYN=0: the static split of a listed run over the CTAs (A/B;
// measured at config 3: SM busy time max / mean 1.27 with it)
static bool tc_dynamic() {
  const char* e = getenv("GPIC_TC_DYN");
  return e == nullptr || atoi(e) != 0;
}

int launch_affinity_tc_packed(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                              int32_t dp, float neg_scale_log2, void* a_packed, float* degrow,
                              float* degcol, cudaStream_t s, int kind, bool half_out,
                              int64_t row_lo, int64_t row_hi, uint8_t* boxnz,
                              const int32_t* unit_list, const int64_t* unit_count) {
  if (row_hi <= 0) row_hi = n;
  const int64_t nt = ceil_div(n, kBN);
  const int64_t t_lo = tile_index(row_lo / 128, row_lo / 128, nt);
  const int64_t t_hi = row_hi >= n ? packed_tiles(n) : tile_index(row_hi / 128, row_hi / 128, nt);
  Maps mp;
  int rc = operand_maps(xhi, n, dp, &mp);
  if (rc) return rc;
  const bool ok = half_out ? make_map(&mp.out, a_packed, 128, (uint64_t)(t_hi - t_lo) * 128, 256,
                                      32, 32, CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                                      CU_TENSOR_MAP_SWIZZLE_64B)
                           : make_map(&mp.out, a_packed, 128, (uint64_t)(t_hi - t_lo) * 128, 512,
                                      32, 32);
  if (!ok) return fail(GPIC_E_CUDA, "cuTensorMapEncodeTiled failed");
  TcArgs args{};
  args.n_pad = row_pad(n);
  args.sqn = sqn;
  args.gscale = sqn + row_pad(n) - 1;
  args.n = n;
  args.row_lo = row_lo;  // launch_kb turns the row range into row blocks
  args.rows = row_hi;
  args.tile_base = t_lo;
  args.ns = neg_scale_log2;
  args.n_ctiles = ceil_div(n, kBN);
  args.out = static_cast<float*>(a_packed);
  args.degrow = degrow;
  args.degcol = degcol;
  args.kind = kind;
  args.boxnz = boxnz;
  args.unit_list = unit_list;
  args.unit_count = unit_count;
  // the prune mask's count slot holds the schedule counters too (prune.cu)
  if (unit_list != nullptr && tc_dynamic()) args.sched = prune_sched(unit_count);
  if (half_out) return dispatch_kb<kModePacked16>(dp / kKBlk, mp, args, s);
  return dispatch_kb<kModePacked>(dp / kKBlk, mp, args, s);
}

int launch_affinity_tc(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                       int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2, float* a,
                       int64_t lda, float* rowpart, int64_t rows_pad, cudaStream_t s, int kind) {
  const int64_t rows = row_hi - row_lo;
  Maps mp;
  int rc = operand_maps(xhi, n, dp, &mp);
  if (rc) return rc;
  if (!make_map(&mp.out, a, (uint64_t)lda, (uint64_t)rows, (uint64_t)lda * 4, 32, 32))
    return fail(GPIC_E_CUDA, "cuTensorMapEncodeTiled failed");
  TcArgs args{};
  args.n_pad = row_pad(n);
  args.sqn = sqn;
  args.gscale = sqn + row_pad(n) - 1;
  args.n = n;
  args.row_lo = row_lo;
  args.rows = rows;
  args.ns = neg_scale_log2;
  args.rowpart = rowpart;
  args.rows_pad = rows_pad;
  args.n_ctiles = ceil_div(n, kBN);
  args.out = a;
  args.lda = lda;
  args.kind = kind;
  return dispatch_kb<kModeDense>(dp / kKBlk, mp, args, s);
}

int64_t mf_parts(int64_t n, int32_t dp) {
  const int64_t chunks = ceil_div(ceil_div(n, kBN), kChunkTiles);
  (void)dp;
  return chunks;  // one fp64 partial per (chunk item, row): the row's warps combine in-CTA
}

int mf_rows_per_block(int32_t dp) { return 128 * mblocks(dp / kKBlk, kModeMatvec); }

int tc_mblocks(int32_t dp) { return mblocks(dp / kKBlk, kModePacked); }
int tc_mblocks_mf(int32_t dp) { return mblocks(dp / kKBlk, kModeMatvec); }

// sym column-partial records: one per (row block of 128 * MB rows, column
// tile J >= MB * row block)
int64_t mf_colpart_floats(int64_t n, int32_t dp) {
  const int mb = mblocks(dp / kKBlk, kModeMatvec);
  return packed_items(ceil_div(n, 128 * mb), ceil_div(n, kBN), mb) * 128;
}

// Matrix-free row block: ypart[p][i - row_lo] = sum over chunk p of
// a_ij v_j (fp64 across tiles); gpic's mf_reduce combines the parts.
// ---- matrix-free CTA re-balance from measured times -------------------
// After a listed pass: the CTAs' measured times over their list ranges give
// a piecewise-constant cost density over the kept tiles; the next pass cuts
// the same range at equal predicted cost (alpha: step toward that target).
// Which CTA computes an item never changes a value, so results stay
// bitwise identical; only the finish time moves.
__global__ void __launch_bounds__(kMaxRebalanceGrid + 1)
    mf_rebalance_kernel(const TcArgs a, int G, int64_t* __restrict__ cuts,
                        const uint64_t* __restrict__ ns, float alpha) {
  __shared__ double xpos[kMaxRebalanceGrid + 1];
  __shared__ double cpre[kMaxRebalanceGrid + 1];  // measured cost before CTA b
  __shared__ int64_t newc[kMaxRebalanceGrid + 1];
  __shared__ bool have;
  if (a.ctl != nullptr && *(volatile const int32_t*)&a.ctl->stop) return;
  const int t = threadIdx.x;
  const int64_t total = *a.unit_count;
  int64_t ua, ub;
  item_share(a, total, ua, ub);
  const int64_t Wa = a.wpre[ua], W = a.wpre[ub] - Wa;
  if (t == 0) have = cuts[0] == G && cuts[1] == ua && cuts[2] == ub;
  __syncthreads();
  // the cuts the pass used (one thread per cut, each its own search)
  if (t <= G) {
    int64_t c;
    if (have) c = cuts[3 + t];
    else if (t == G) c = ub;
    else c = lower_bound_w(a.wpre, ua, ub, Wa + W * t / G);
    xpos[t] = (double)(a.wpre[c] - Wa);
  }
  if (t == 0) {
    double acc = 0.0;
    for (int b = 0; b < G; ++b) {
      cpre[b] = acc;
      acc += (double)ns[b];
    }
    cpre[G] = acc;
  }
  __syncthreads();
  const double T = cpre[G];
  if (!(T > 0.0) || W <= 0) return;
  // cut k: where the piecewise-linear measured cost reaches k T / G
  if (t >= 1 && t < G) {
    const double target = T * t / G;
    int lo = 0, hi = G - 1;  // last segment with cpre[seg] <= target
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cpre[mid] <= target) lo = mid; else hi = mid - 1;
    }
    const double len = cpre[lo + 1] - cpre[lo];
    const double frac = len > 0.0 ? (target - cpre[lo]) / len : 0.0;
    const double xt = xpos[lo] + fmin(fmax(frac, 0.0), 1.0) * (xpos[lo + 1] - xpos[lo]);
    const double x = xpos[t] + alpha * (xt - xpos[t]);
    newc[t] = lower_bound_w(a.wpre, ua, ub, Wa + (int64_t)(x + 0.5));
  }
  if (t == 0) {
    newc[0] = ua;
    newc[G] = ub;
  }
  __syncthreads();
  if (t == 0) {  // monotone, then the header last
    for (int k = 1; k <= G; ++k)
      if (newc[k] < newc[k - 1]) newc[k] = newc[k - 1];
    for (int k = 0; k <= G; ++k) cuts[3 + k] = newc[k];
    cuts[1] = ua;
    cuts[2] = ub;
    __threadfence();
    cuts[0] = G;
  }
}

int launch_mf_rebalance(const PruneMask* pm, int share_r, int share_n, const gpic_ctl* ctl,
                        cudaStream_t s) {
  if (g_num_sms == 0) {
    int dev;
    GPIC_CUDA_TRY(cudaGetDevice(&dev));
    GPIC_CUDA_TRY(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  if (g_num_sms > kMaxRebalanceGrid) return GPIC_OK;
  TcArgs a{};
  a.unit_list = pm->items;
  a.unit_count = pm->item_count;
  a.wpre = pm->item_wpre;
  a.share_r = share_r;
  a.share_n = share_n;
  a.ctl = ctl;
  const char* e = getenv("GPIC_MF_REBALANCE_ALPHA");
  const float alpha = e != nullptr ? (float)atof(e) : 1.0f;
  mf_rebalance_kernel<<<1, kMaxRebalanceGrid + 1, 0, s>>>(a, g_num_sms, pm->cta_cuts, pm->cta_ns,
                                                         alpha);
  count_launch();
  return GPIC_OK;
}

bool mf_rebalance_enabled() {
  const char* e = getenv("GPIC_MF_REBALANCE");
  return e == nullptr || atoi(e) != 0;
}

int launch_affinity_tc_matvec(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                              int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2,
                              const float* v32, double* ypart, int64_t rows_pad,
                              const gpic_ctl* ctl, cudaStream_t s, int kind, float* colpart,
                              const PruneMask* pm, int share_r, int share_n) {
  Maps mp;
  int rc = operand_maps(xhi, n, dp, &mp);
  if (rc) return rc;
  TcArgs args{};
  args.n_pad = row_pad(n);
  args.sqn = sqn;
  args.gscale = sqn + row_pad(n) - 1;
  args.n = n;
  args.row_lo = row_lo;
  args.rows = row_hi - row_lo;
  args.ns = neg_scale_log2;
  args.rows_pad = rows_pad;
  args.n_ctiles = ceil_div(n, kBN);
  args.v32 = v32;
  args.ypart = ypart;
  args.ctl = ctl;
  args.kind = kind;
  args.sym = colpart != nullptr && row_lo == 0 && row_hi == n;
  args.colpart = colpart;
  if (pm != nullptr && args.sym) {  // pruned sym pass: the kept items only
    args.unit_list = pm->items;
    args.unit_count = pm->item_count;
    args.pskip = pm->skip;
    args.pB = pm->B;
    args.pnb = pm->nb;
    args.wpre = pm->item_wpre;
    args.share_r = share_r;
    args.share_n = share_n;
    if (mf_rebalance_enabled()) {
      args.cuts = pm->cta_cuts;
      args.cta_ns = pm->cta_ns;
    }
  }
  return dispatch_kb<kModeMatvec>(dp / kKBlk, mp, args, s);
}

// Feature pitches the engine runs: 64 * KB with the CTA's shared memory
// (resident row operands + at least one B stage + the epilogue buffers)
// within the 227 KB opt-in. Store modes stop at KB = 3 (d <= 192): their
// 64 KB of per-warp staging leaves no room for a KB = 4 stage.
bool tc_supports_pitch(int32_t dp, bool matvec) {
  if (dp % kKBlk) return false;
  const int KB = dp / kKBlk;
  constexpr int kLimit = kSmemBudget + 256 + 1024;
  auto fits = [&](int kb, int mode) {
    return stages_raw(kb, mode) >= 1 && smem_bytes(kb, mode) <= kLimit;
  };
  switch (KB) {
    case 1: return matvec ? fits(1, kModeMatvec) : fits(1, kModePacked) && fits(1, kModeDense);
    case 2: return matvec ? fits(2, kModeMatvec) : fits(2, kModePacked) && fits(2, kModeDense);
    case 3: return matvec ? fits(3, kModeMatvec) : fits(3, kModePacked) && fits(3, kModeDense);
    case 4: return matvec ? fits(4, kModeMatvec) : fits(4, kModePacked) && fits(4, kModeDense);
    default: return false;
  }
}

}  // namespace gpic
