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
//           iteration when n^2 does not fit HBM
//
// Persistent warp-specialised kernel, one CTA per SM (320 threads):
//   warp 0      TMA producer: the CTA's row block (MB x 128 rows, hi + lo,
//               all K) stays resident in smem while the CTA walks its
//               contiguous range of column tiles; B tiles (128 columns,
//               hi + lo, one 64-wide K block per stage) stream through a
//               ring of smem stages.
//   warp 1      TMEM owner + single-thread MMA issuer: 3 x 4 x KB MMAs per
//               M block into one of two TMEM accumulators (double buffer,
//               so the next tile's MMAs overlap this tile's epilogue).
//   warps 2-9   epilogue: tcgen05.ld 32 columns at a time, exp2 + masks +
//               row sums in registers; store modes go through swizzled
//               st.shared and TMA bulk-tensor stores of 32x32 fp32 boxes.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "ops.h"
#include "sm100.cuh"

namespace gpic {

namespace {

enum { kModeDense = 0, kModePacked = 1, kModeMatvec = 2 };

constexpr int kBN = 128;           // columns per tile (one MMA N)
constexpr int kKBlk = 64;          // fp16 per 128-byte swizzle row
constexpr int kTileBytes = 128 * kKBlk * 2;  // 16 KB: 128 rows x 64 fp16
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + kEpiWarps * 32;
constexpr int kStageOutBytes = 32 * 128;     // 32 rows x 32 fp32 per epilogue warp
constexpr int kSmemBudget = 224 * 1024;
constexpr int kChunkTiles = 32;              // matvec: column tiles per work item

__host__ __device__ constexpr int mblocks(int KB) { return KB <= 2 ? 2 : 1; }
__host__ __device__ constexpr int a_bytes(int KB) { return 2 * mblocks(KB) * KB * kTileBytes; }
// output staging buffers per epilogue warp (double-buffered where smem allows)
// DIRECT: the epilogue stores straight from registers (no smem staging)
__host__ __device__ constexpr int out_bufs(int KB, int MODE, bool DIRECT) {
  return (MODE == kModeMatvec || DIRECT) ? 0 : ((KB == 1 || KB == 3) ? 2 : 1);
}
__host__ __device__ constexpr int out_bytes(int KB, int MODE, bool DIRECT) {
  return kEpiWarps * out_bufs(KB, MODE, DIRECT) * kStageOutBytes;
}
__host__ __device__ constexpr int stages(int KB, int MODE, bool DIRECT) {
  return (kSmemBudget - a_bytes(KB) - out_bytes(KB, MODE, DIRECT)) / (2 * kTileBytes) > 4
             ? 4
             : (kSmemBudget - a_bytes(KB) - out_bytes(KB, MODE, DIRECT)) / (2 * kTileBytes);
}
__host__ __device__ constexpr int smem_bytes(int KB, int MODE, bool DIRECT) {
  return a_bytes(KB) + stages(KB, MODE, DIRECT) * 2 * kTileBytes + out_bytes(KB, MODE, DIRECT) +
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
  int64_t n_rtiles;  // row blocks of 128*MB rows
  int64_t n_ctiles;  // column tiles of 128
  const float* v32;  // matvec: vector_pitch(n) floats
  double* ypart;     // matvec: [n_chunks * parts][rows_pad] fp64 row partials
  int64_t n_chunks;  // matvec: column chunks (kChunkTiles tiles) per row block
  const gpic_ctl* ctl;  // matvec in a loop: exit at once when ctl->stop is set
  float* out;        // DIRECT stores: dense A rows (pitch lda) or packed tiles
  int64_t lda;
  float* degrow;     // packed: [tile][halves][128] row partials of each stored tile
  float* degcol;     // packed: [tile][4 row quadrants][128] column partials
  int kind;          // GPIC_KIND_RBF: exp2 epilogue; GPIC_KIND_COSINE: max(0, G) on unit rows
  const float* gscale;  // 1 / s^2 of the fp16 operand planes (sqn[n_pad - 1], prepare.cu)
};

__host__ __device__ inline int64_t packed_items(int64_t nrt, int64_t nct, int mb) {
  return nrt * nct - (int64_t)mb * nrt * (nrt - 1) / 2;
}

// Packed index of tile (I, J), J >= I, row-major over the upper triangle.
__host__ __device__ inline int64_t tile_index(int64_t I, int64_t J, int64_t nt) {
  return I * nt - I * (I - 1) / 2 + (J - I);
}

// Work sequence of one CTA, identical for all three roles.
//   dense / packed: units are tiles (rb, cb); packed keeps cb >= rb*MB only
//   matvec: units are items (rb, chunk) of up to kChunkTiles column tiles, so
//           a chunk's row partial is always produced by one CTA (fixed shape)
template <int MB, int MODE>
struct Cursor {
  int64_t u, u_end;    // unit counter
  int64_t rb, cb;      // current tile
  int64_t cb_end;      // matvec: end of the current item's columns
  int64_t chunk;       // matvec: chunk index of the current item

  __device__ void decode_unit(const TcArgs& a) {
    if (MODE == kModeDense) {
      rb = u / a.n_ctiles;
      cb = u % a.n_ctiles;
    } else if (MODE == kModePacked) {
      int64_t lo = 0, hi = a.n_rtiles - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        const int64_t s = mid * a.n_ctiles - (int64_t)MB * mid * (mid - 1) / 2;
        if (s <= u) lo = mid; else hi = mid - 1;
      }
      rb = lo;
      cb = rb * MB + (u - (lo * a.n_ctiles - (int64_t)MB * lo * (lo - 1) / 2));
    } else {
      rb = u / a.n_chunks;
      chunk = u % a.n_chunks;
      cb = chunk * kChunkTiles;
      cb_end = min(cb + kChunkTiles, a.n_ctiles);
    }
  }
  __device__ void begin(const TcArgs& a, int64_t u0, int64_t u1) {
    u = u0;
    u_end = u1;
    if (u < u_end) decode_unit(a);
  }
  __device__ bool valid() const { return u < u_end; }
  __device__ bool item_last() const { return MODE != kModeMatvec || cb + 1 == cb_end; }
  __device__ void next(const TcArgs& a) {
    if (MODE == kModeMatvec && cb + 1 < cb_end) {
      ++cb;
      return;
    }
    ++u;
    if (u < u_end) decode_unit(a);
  }
};

template <int MB, int MODE>
__host__ __device__ inline int64_t total_units(const TcArgs& a) {
  if (MODE == kModePacked) return packed_items(a.n_rtiles, a.n_ctiles, MB);
  if (MODE == kModeMatvec) return a.n_rtiles * a.n_chunks;
  return a.n_rtiles * a.n_ctiles;
}

template <int KB, int MODE, bool DIRECT>
__global__ void __launch_bounds__(kThreads, 1)
    affinity_tc_kernel(const __grid_constant__ CUtensorMap map_hi,
                       const __grid_constant__ CUtensorMap map_lo,
                       const __grid_constant__ CUtensorMap map_out, const TcArgs args) {
  constexpr int MB = mblocks(KB);
  constexpr int ST = stages(KB, MODE, DIRECT);
  constexpr int kTmemCols = 2 * MB * kBN;  // 2 accumulators
  if (MODE == kModeMatvec && args.ctl != nullptr && *(volatile const int32_t*)&args.ctl->stop)
    return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = base;                                     // [hl][m][kb] 16 KB tiles
  uint8_t* sB = sA + a_bytes(KB);                         // [stage][hl] 16 KB tiles
  uint8_t* sOut = sB + ST * 2 * kTileBytes;               // [epi warp][buf] 4 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sOut + out_bytes(KB, MODE, DIRECT));
  uint64_t* full = bars;                 // [ST]
  uint64_t* empty = bars + ST;           // [ST]
  uint64_t* a_full = bars + 2 * ST;
  uint64_t* a_empty = a_full + 1;
  uint64_t* t_full = a_full + 2;         // [2]
  uint64_t* t_empty = a_full + 4;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 6);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t total = total_units<MB, MODE>(args);
  const int64_t u_begin = total * blockIdx.x / gridDim.x;
  const int64_t u_end = total * (blockIdx.x + 1) / gridDim.x;

  if (threadIdx.x == 0) {
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
    if (MODE != kModeMatvec && !DIRECT)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_out)) : "memory");
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
      for (c.begin(args, u_begin, u_end); c.valid(); c.next(args)) {
        if (c.rb != cur_rb) {
          mbar_wait(a_empty, a_par);
          a_par ^= 1;
          mbar_expect_tx(a_full, a_bytes(KB));
          for (int hl = 0; hl < 2; ++hl)
            for (int m = 0; m < MB; ++m)
              for (int kb = 0; kb < KB; ++kb)
                tma_load_2d(sA + ((hl * MB + m) * KB + kb) * kTileBytes, hl ? &map_lo : &map_hi,
                            kb * kKBlk, (int)(args.row_lo + (c.rb * MB + m) * 128), a_full, keep);
          cur_rb = c.rb;
        }
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], 2 * kTileBytes);
          tma_load_2d(sB + (s * 2 + 0) * kTileBytes, &map_hi, kb * kKBlk, (int)(c.cb * kBN), &full[s],
                      keep);
          tma_load_2d(sB + (s * 2 + 1) * kTileBytes, &map_lo, kb * kKBlk, (int)(c.cb * kBN), &full[s],
                      keep);
          if (++s == ST) { s = 0; ph ^= 1; }
        }
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
      for (c.begin(args, u_begin, u_end); c.valid(); ++i) {
        const int64_t rb = c.rb;
        if (rb != cur_rb) {
          mbar_wait(a_full, a_par);
          a_par ^= 1;
          cur_rb = rb;
        }
        const int buf = i & 1;
        mbar_wait(&t_empty[buf], (te_bits >> buf) & 1u);
        te_bits ^= 1u << buf;
        tc_fence_after();
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint64_t bh = sw128_desc(su32(sB + (s * 2 + 0) * kTileBytes));
          const uint64_t bl = sw128_desc(su32(sB + (s * 2 + 1) * kTileBytes));
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
          }
          tc_commit(&empty[s]);  // frees the B stage once these MMAs retire
          if (++s == ST) { s = 0; ph ^= 1; }
        }
        tc_commit(&t_full[buf]);
        c.next(args);
        if (!c.valid() || c.rb != rb) tc_commit(a_empty);  // last tile of this row block
      }
    }
  } else {
    // --------------------------------------------------------- epilogue
    constexpr int NC = MB == 2 ? 4 : 2;  // 32-column chunks per warp per tile
    constexpr int NBUF = out_bufs(KB, MODE, DIRECT);
    const int e = warp - 2;
    const int q = warp & 3;          // TMEM lane quadrant this warp may access
    const int g = e >> 2;            // group: M block (MB=2) or column half (MB=1)
    const int m = MB == 2 ? g : 0;
    const int c_lo = MB == 2 ? 0 : 2 * g;
    uint8_t* stage0 = sOut + e * (NBUF > 0 ? NBUF : 1) * kStageOutBytes;
    const float ns = args.ns;
    const float gs = __ldg(args.gscale);  // accumulator units -> G
    const float m2ns = -2.f * ns * gs;
    const uint64_t stream_pol = policy_evict_first();  // A is written once here
    uint32_t tf_bits = 0;  // TMEM-full parity per accumulator buffer
    int i = 0;
    int stores = 0;
    double acc64 = 0.0;  // matvec: row partial over the current item
    // column norms (and matvec v) of the next tile are fetched one tile ahead
    // so the L2 latency hides behind the TMEM-full wait
    float nx_cb[NC], nx_v[NC], nx_ra = 0.f;
    auto prefetch = [&](const Cursor<MB, MODE>& c) {
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const int64_t col = c.cb * kBN + (c_lo + cc) * 32 + lane;
        nx_cb[cc] = ns * __ldg(args.sqn + col);
        if (MODE == kModeMatvec) nx_v[cc] = __ldg(args.v32 + col);
      }
      const int64_t gr = args.row_lo + (c.rb * MB + m) * 128 + q * 32 + lane;
      nx_ra = gr < args.n ? ns * __ldg(args.sqn + gr) : 0.f;
    };
    Cursor<MB, MODE> c;
    c.begin(args, u_begin, u_end);
    if (c.valid()) prefetch(c);
    for (; c.valid(); ++i) {
      const int64_t rb = c.rb, cb = c.cb;
      const bool item_last = c.item_last();
      const int64_t chunk = c.chunk;
      const int buf = i & 1;
      const int64_t tI = rb * MB + m;  // tile row of this warp's rows
      // packed: the lower-triangle half of a diagonal row block is not stored
      const bool store_ok = MODE != kModePacked || tI <= cb;
      const int64_t out_row0 = MODE == kModePacked ? tile_index(tI, cb, args.n_ctiles) * 128 + q * 32
                                                   : (rb * MB + m) * 128 + q * 32;
      const int64_t lr0 = (rb * MB + m) * 128 + q * 32;  // shard-local first row of this warp
      const int64_t lr = lr0 + lane;
      const int64_t gr = args.row_lo + lr;
      float cbv[NC], vv[NC];
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        cbv[cc] = nx_cb[cc];
        vv[cc] = nx_v[cc];
      }
      const float ra = nx_ra;
      c.next(args);
      if (c.valid()) prefetch(c);
      mbar_wait(&t_full[buf], (tf_bits >> buf) & 1u);
      tf_bits ^= 1u << buf;
      tc_fence_after();
      float rsum = 0.f;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const int ch = c_lo + cc;
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)((buf * MB + m) * kBN + ch * 32),
                  r);
        if (cc == NC - 1) {  // accumulator fully read: hand it back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&t_empty[buf]);
        }
        const int64_t col0 = cb * kBN + ch * 32;
        const bool diag = (col0 < args.row_lo + lr0 + 32) && (args.row_lo + lr0 < col0 + 32);
        const bool pad = col0 + 32 > args.n || args.row_lo + lr0 + 32 > args.n;
        float vals[32];
        if (args.kind == GPIC_KIND_COSINE) {
          // rows are unit vectors: G_ij = cos(x_i, x_j), clamped at 0 (affinity.py:93-94)
#pragma unroll
          for (int j = 0; j < 32; ++j) vals[j] = fmaxf(__uint_as_float(r[j]) * gs, 0.f);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float cj = __shfl_sync(0xffffffffu, cbv[cc], j);
            const float arg = fmaf(__uint_as_float(r[j]), m2ns, ra + cj);
            vals[j] = ex2(fminf(arg, 0.f));
          }
        }
        if (diag || pad) {
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j == gr || col0 + j >= args.n || gr >= args.n) vals[j] = 0.f;
        }
        if constexpr (MODE == kModeMatvec) {
#pragma unroll
          for (int j = 0; j < 32; ++j) rsum = fmaf(vals[j], __shfl_sync(0xffffffffu, vv[cc], j), rsum);
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) rsum += vals[j];
          // the store issued NBUF chunks ago must have finished reading this buffer
          uint8_t* stage = stage0 + (stores % NBUF) * kStageOutBytes;
          if (stores >= NBUF) {
            if (lane == 0) tma_store_wait_read<NBUF - 1>();
            __syncwarp();
          }
          const uint32_t srow = su32(stage) + lane * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint32_t addr = srow + ((j ^ (lane & 7)) << 4);
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(vals[4 * j]),
                         "f"(vals[4 * j + 1]), "f"(vals[4 * j + 2]), "f"(vals[4 * j + 3])
                         : "memory");
          }
          fence_async_smem();
          __syncwarp();
          if (lane == 0 && store_ok)
            tma_store_2d(&map_out, MODE == kModePacked ? ch * 32 : (int)col0, (int)out_row0, stage,
                         stream_pol);
          ++stores;
          if (MODE == kModePacked && store_ok && tI != cb) {
            // degrees of the tile's COLUMN rows (A is symmetric): lane l sums
            // column l of the staged 32x32 chunk over this warp's 32 rows
            // (row r of the swizzled stage: chunk (l/4) ^ (r & 7)), fixed order
            const uint32_t sb = su32(stage) + (lane & 3) * 4;
            float cs[4] = {0.f, 0.f, 0.f, 0.f};  // 4 chains: rows r2 = 4u + w
#pragma unroll
            for (int r2 = 0; r2 < 32; ++r2) {
              float x;
              asm volatile("ld.shared.f32 %0, [%1];"
                           : "=f"(x)
                           : "r"(sb + r2 * 128 + ((((lane >> 2) ^ (r2 & 7))) << 4)));
              cs[r2 & 3] += x;
            }
            args.degcol[(tile_index(tI, cb, args.n_ctiles) * 4 + q) * 128 + ch * 32 + lane] =
                (cs[0] + cs[1]) + (cs[2] + cs[3]);
          }
        }
      }
      if constexpr (MODE == kModePacked) {
        // degrees of the tile's ROW rows: this warp's partial over its chunks
        if (store_ok) {
          constexpr int NH = MB == 2 ? 1 : 2;  // column halves per row
          args.degrow[(tile_index(tI, cb, args.n_ctiles) * NH + (MB == 2 ? 0 : g)) * 128 + q * 32 +
                      lane] = rsum;
        }
      } else if constexpr (MODE == kModeMatvec) {
        acc64 += (double)rsum;
        if (item_last) {
          // MB=2: one partial per (chunk, row); MB=1: one per (chunk, half, row)
          const int64_t slot = MB == 2 ? chunk : chunk * 2 + g;
          if (lr < args.rows) args.ypart[slot * args.rows_pad + lr] = acc64;
          acc64 = 0.0;
        }
      } else if constexpr (MODE == kModeDense) {
        if constexpr (MB == 2) {
          if (lr < args.rows) args.rowpart[cb * args.rows_pad + lr] = rsum;
        } else {
          // two warps (column halves) share each row: half 1 parks its sum in
          // smem, half 0 adds it (fixed order) after a 64-thread named barrier.
          __shared__ float half1[4][32];
          if (g == 1) half1[q][lane] = rsum;
          asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(64) : "memory");
          if (g == 0 && lr < args.rows) args.rowpart[cb * args.rows_pad + lr] = rsum + half1[q][lane];
          asm volatile("bar.sync %0, %1;" ::"r"(1 + q), "r"(64) : "memory");
        }
      }
    }
    if (MODE != kModeMatvec && !DIRECT && lane == 0) tma_store_wait_all();
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols)
                 : "memory");
  }
}

// ---------------------------------------------------------- host side
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
              CUtensorMapDataType dtype = CU_TENSOR_MAP_DATA_TYPE_FLOAT32) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dtype, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int g_num_sms = 0;

template <int KB, int MODE, bool DIRECT>
int launch_kb(const CUtensorMap& mh, const CUtensorMap& ml, const CUtensorMap& mo,
              const TcArgs& a0, cudaStream_t s) {
  constexpr int MB = mblocks(KB);
  TcArgs a = a0;
  a.n_rtiles = ceil_div(a.rows, 128 * MB);
  a.n_chunks = ceil_div(a.n_ctiles, kChunkTiles);
  static bool attr = false;
  if (!attr) {
    GPIC_CUDA_TRY(cudaFuncSetAttribute(affinity_tc_kernel<KB, MODE, DIRECT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_bytes(KB, MODE, DIRECT)));
    attr = true;
  }
  if (g_num_sms == 0) {
    int dev;
    GPIC_CUDA_TRY(cudaGetDevice(&dev));
    GPIC_CUDA_TRY(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int64_t total = total_units<MB, MODE>(a);
  const int grid = (int)(total < g_num_sms ? total : g_num_sms);
  if (grid < 1) return GPIC_OK;
  affinity_tc_kernel<KB, MODE, DIRECT><<<grid, kThreads, smem_bytes(KB, MODE, DIRECT), s>>>(
      mh, ml, mo, a);
  count_launch();
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

// The epilogue stores through swizzled smem staging + TMA bulk-tensor
// stores (measured 2x faster on config 3 than direct 128-bit st.global from
// registers, which left partially written lines to the L2). The DIRECT
// template flag only removes the staging smem (matvec mode stores nothing).
template <int MODE>
int dispatch_kb(int KB, const CUtensorMap& mh, const CUtensorMap& ml, const CUtensorMap& mo,
                const TcArgs& args, cudaStream_t s) {
  constexpr bool kNoStage = MODE == kModeMatvec;
  switch (KB) {
    case 1: return launch_kb<1, MODE, kNoStage>(mh, ml, mo, args, s);
    case 2: return launch_kb<2, MODE, kNoStage>(mh, ml, mo, args, s);
    case 3: return launch_kb<3, MODE, kNoStage>(mh, ml, mo, args, s);
    default: return launch_kb<4, MODE, kNoStage>(mh, ml, mo, args, s);
  }
}

// The fp16 hi / lo planes live back to back in the d_xhi buffer (prepare.cu).
int operand_maps(const float* xhi, int64_t n, int32_t dp, CUtensorMap* mh, CUtensorMap* ml) {
  const int KB = dp / kKBlk;
  if (dp % kKBlk || KB < 1 || KB > 4)
    return fail(GPIC_E_UNSUPPORTED, "tcgen05 affinity engine supports d <= 256");
  const int64_t npad = row_pad(n);
  const uint16_t* hi = reinterpret_cast<const uint16_t*>(xhi);
  const uint16_t* lo = hi + npad * dp;
  if (!make_map(mh, hi, (uint64_t)dp, (uint64_t)npad, (uint64_t)dp * 2, kKBlk, 128,
                CU_TENSOR_MAP_DATA_TYPE_FLOAT16) ||
      !make_map(ml, lo, (uint64_t)dp, (uint64_t)npad, (uint64_t)dp * 2, kKBlk, 128,
                CU_TENSOR_MAP_DATA_TYPE_FLOAT16))
    return fail(GPIC_E_CUDA, "cuTensorMapEncodeTiled failed");
  return GPIC_OK;
}

}  // namespace

int64_t packed_tiles(int64_t n) {
  const int64_t nt = ceil_div(n, kBN);
  return nt * (nt + 1) / 2;
}

// Symmetric packed output: tile (I, J), J >= I, stored as a contiguous
// 128 x 128 fp32 block at tile_index(I, J) (row-major over the triangle).
int packed_row_halves(int32_t dp) { return mblocks(dp / kKBlk) == 2 ? 1 : 2; }

int launch_affinity_tc_packed(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                              int32_t dp, float neg_scale_log2, float* a_packed, float* degrow,
                              float* degcol, cudaStream_t s, int kind) {
  CUtensorMap mh, ml, mo;
  int rc = operand_maps(xhi, n, dp, &mh, &ml);
  if (rc) return rc;
  if (!make_map(&mo, a_packed, 128, (uint64_t)packed_tiles(n) * 128, 512, 32, 32))
    return fail(GPIC_E_CUDA, "cuTensorMapEncodeTiled failed");
  TcArgs args{};
  args.sqn = sqn;
  args.gscale = sqn + row_pad(n) - 1;
  args.n = n;
  args.rows = n;
  args.ns = neg_scale_log2;
  args.n_ctiles = ceil_div(n, kBN);
  args.out = a_packed;
  args.degrow = degrow;
  args.degcol = degcol;
  args.kind = kind;
  return dispatch_kb<kModePacked>(dp / kKBlk, mh, ml, mo, args, s);
}

int launch_affinity_tc(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                       int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2, float* a,
                       int64_t lda, float* rowpart, int64_t rows_pad, cudaStream_t s, int kind) {
  const int64_t rows = row_hi - row_lo;
  CUtensorMap mh, ml, mo;
  int rc = operand_maps(xhi, n, dp, &mh, &ml);
  if (rc) return rc;
  if (!make_map(&mo, a, (uint64_t)lda, (uint64_t)rows, (uint64_t)lda * 4, 32, 32))
    return fail(GPIC_E_CUDA, "cuTensorMapEncodeTiled failed");
  TcArgs args{};
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
  return dispatch_kb<kModeDense>(dp / kKBlk, mh, ml, mo, args, s);
}

int64_t mf_parts(int64_t n, int32_t dp) {
  const int64_t chunks = ceil_div(ceil_div(n, kBN), kChunkTiles);
  return mblocks(dp / kKBlk) == 2 ? chunks : 2 * chunks;
}

// Matrix-free row block: ypart[p][i - row_lo] = sum over chunk p of
// a_ij v_j (fp64 across tiles); gpic's mf_reduce combines the parts.
int launch_affinity_tc_matvec(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                              int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2,
                              const float* v32, double* ypart, int64_t rows_pad,
                              const gpic_ctl* ctl, cudaStream_t s, int kind) {
  CUtensorMap mh, ml;
  int rc = operand_maps(xhi, n, dp, &mh, &ml);
  if (rc) return rc;
  TcArgs args{};
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
  return dispatch_kb<kModeMatvec>(dp / kKBlk, mh, ml, mh, args, s);
}

}  // namespace gpic
