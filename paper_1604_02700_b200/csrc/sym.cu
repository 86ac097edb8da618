// Symmetric packed storage: A is exactly symmetric (affinity.py:96-103;
// test_affinity.py:81-87), so only the upper triangle of 128 x 128 tiles is
// stored (tile (I, J), J >= I, contiguous 64 KB at tile_index(I, J)). That
// halves the bytes of the two HBM-bound stages: the affinity store and the
// per-iteration GEMV read (2n^2 instead of 4n^2 bytes).
//
//   sym_gemv_kernel   streams every stored tile once (1-D bulk copies into a
//                     smem ring), walking 4 x 4-tile super-blocks, and
//                     produces per super-block the 128 row partials
//                     sum_j T[i][j] v_J[j] of each of its tile rows (for y_I)
//                     and, off the diagonal, the 128 column partials
//                     sum_i T[i][j] v_I[i] of each tile column (for
//                     y_J = (T^T v_I)_J). fp32 within a super-block.
//   sym_reduce_kernel y_i = sum over the row's super-block records (fp64):
//                     column records of (P', Q(i)), P' <= Q(i), then row
//                     records of (Q(i), Q'), Q' >= Q(i); / deg_i; stored into
//                     every rank's y (same epilogue as the dense GEMV).
// Degrees come from the affinity epilogue's per-tile partials (sums of the
// stored values). Every sum has a fixed order, so results are deterministic.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "ops.h"
#include "sm100.cuh"
#include "lowdeg.cuh"
#include "tail.cuh"

namespace gpic {

namespace {

constexpr int kTS = 128;
constexpr int kTileFloats = kTS * kTS;
constexpr int kStages = 3;  // fp32 tiles (64 KB); fp16 tiles (32 KB) use 2x the stages
constexpr int kWarps = 8;                   // consumers; 16 rows each
constexpr int kRowsPerWarp = kTS / kWarps;  // 16
constexpr int kThreads = (kWarps + 1) * 32;
constexpr int kSmem = kStages * kTileFloats * 4 + 2 * kWarps * 4 * kTS * 4 + 64 + 128;
template <typename T>
struct TileTraits;  // element type of the stored tiles
template <>
struct TileTraits<float> {
  static constexpr int kStg = kStages;
  // 4 consecutive values of row i at this lane's columns
  __device__ static float4 load4(const uint8_t* row, int lane) {
    return reinterpret_cast<const float4*>(row)[lane];
  }
};
template <>
struct TileTraits<__half> {
  static constexpr int kStg = 2 * kStages;
  __device__ static float4 load4(const uint8_t* row, int lane) {
    const uint2 u = reinterpret_cast<const uint2*>(row)[lane];
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
};

__host__ __device__ inline int64_t tile_index(int64_t I, int64_t J, int64_t nt) {
  return I * nt - I * (I - 1) / 2 + (J - I);
}

// tile index -> (I, J) by the row prefix P(I) = I*nt - I*(I-1)/2
__device__ inline void tile_coords(int64_t t, int64_t nt, int64_t& I, int64_t& J) {
  int64_t lo = 0, hi = nt - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (mid * nt - mid * (mid - 1) / 2 <= t) lo = mid; else hi = mid - 1;
  }
  I = lo;
  J = I + (t - (I * nt - I * (I - 1) / 2));
}

// Super-blocks of kSB x kSB tiles, (P, Q >= P) row-major over the
// NS x NS triangle (NS = ceil(NT / kSB)), same index formula as the tiles.
constexpr int kSB = 4;

// Block sparsity (sparse.cu): boxnz[t * 16 + quadrant * 4 + chunk] flags the
// 32 x 32 boxes of packed tile t the affinity engine stored (the others are
// exact zeros, never written); a tile with no stored box is never read.
// sbp[s] = weight prefix of the GEMV super-blocks (8 per stored tile + 1),
// so a super-block of weight 1 holds no stored tile. Both null: dense.
struct Sparse {
  const uint8_t* boxnz;
  const int64_t* sbp;
  const uint16_t* bits;  // [super-block][16 tiles] box masks (sb_bits), or null
  int prefetch;          // producer: tiles prefetched into L2 ahead of the smem ring
  int bits_consumer;     // consumers read the super-block records too (else per-tile flags)
  int evict_first;       // tile loads with the L2 evict-first policy
  const int32_t* list;   // non-empty super-blocks (sb_list), or null: walk the id range
  const int64_t* lpre;
  const int64_t* lcount;
  const int64_t* ranges;  // precomputed CTA ranges over the list (sb_list), or null
  // reduce: per super-row Q the ascending term indices of its non-empty
  // records (column records of (P', Q) as P', then row records of (Q, Q')
  // as Q + 1 + Q' - Q), tlist[Q * tld ...], tcount[Q] of them; or null
  const int32_t* tlist;
  const int32_t* tcount;
  int64_t tld;
  // dynamic GEMV schedule (list mode): [0] next list entry to claim, [1]
  // CTAs past their last claim (the last one resets both); or null: the
  // static weight ranges
  unsigned* sched;
  // the 16 tile masks of super-block s (two 16-byte loads), kept in
  // registers: selected by comparisons, never indexed (an indexed array
  // went to local memory)
  struct Rec {
    uint4 a, b;
  };
  __device__ Rec record(int64_t s) const {
    const uint4* p = reinterpret_cast<const uint4*>(bits + s * kSB * kSB);
    return Rec{__ldg(p), __ldg(p + 1)};
  }
  __device__ static bool empty(const Rec& r) {
    return ((r.a.x | r.a.y | r.a.z | r.a.w) | (r.b.x | r.b.y | r.b.z | r.b.w)) == 0u;
  }
  __device__ static uint32_t mask_of(const Rec& r, int idx) {
    const int q = idx >> 1;
    const uint4 h = q < 4 ? r.a : r.b;
    const int c = q & 3;
    const uint32_t w = c < 2 ? (c == 0 ? h.x : h.y) : (c == 2 ? h.z : h.w);
    return (idx & 1) ? (w >> 16) : (w & 0xffffu);
  }
  __device__ uint4 flags(int64_t I, int64_t J, int64_t nt) const {
    return *reinterpret_cast<const uint4*>(boxnz + tile_index(I, J, nt) * 16);
  }
  __device__ bool skip_tile(int64_t I, int64_t J, int64_t nt) const {
    if (boxnz == nullptr) return false;
    const uint4 f = flags(I, J, nt);
    return (f.x | f.y | f.z | f.w) == 0u;
  }
  __device__ bool empty_sb(int64_t s) const { return sbp != nullptr && sbp[s + 1] - sbp[s] == 1; }
};

// first s in [lo, hi] with sbp[s] >= target (sbp strictly increasing)
__device__ inline int64_t lower_bound64(const int64_t* a, int64_t lo, int64_t hi, int64_t target) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] >= target) hi = mid; else lo = mid + 1;
  }
  return lo;
}

}  // namespace

// A packed shard: super-rows [p_lo, p_hi) of the super-block triangle (tile
// rows [kSB p_lo, kSB p_hi)), stored from global tile index tile_base.
// Whole matrix: {0, huge, 0}.
__host__ __device__ int64_t ShardRange::sb_lo(int64_t ns) const {
  return p_lo * ns - p_lo * (p_lo - 1) / 2;
}
__host__ __device__ int64_t ShardRange::sb_hi(int64_t ns) const {
  const int64_t p = p_hi < ns ? p_hi : ns;
  return p * ns - p * (p - 1) / 2;
}

namespace {

// The tiles of one super-block, in the order both roles walk them: rows
// I = kSB P .. (< NT), then columns J = max(I, kSB Q) .. (< NT).
struct SbWalk {
  int64_t nt, ns;
  int64_t P, Q, I, J;
  int64_t i_end, j_end;
  __device__ void open(int64_t p, int64_t q) {
    P = p;
    Q = q;
    I = kSB * P;
    i_end = min(I + kSB, nt);
    j_end = min(kSB * Q + kSB, nt);
    J = max(I, kSB * Q);
  }
  // advance to the next tile of the super-block; false at its end
  __device__ bool next() {
    if (++J < j_end) return true;
    if (++I >= i_end) return false;
    J = max(I, kSB * Q);
    return J < j_end;
  }
  __device__ void next_sb() {
    if (++Q == ns) {
      ++P;
      Q = P;
    }
  }
};

// The CTA's super-blocks, in order: either the id range [sb, s1) (every
// super-block, empty ones skipped by their weight) or, with a list of the
// non-empty ones (sparse.cu sb_list_kernel), the entries [e, e1) of it.
// (P, Q) follow the current super-block.
struct SbCursor {
  const int32_t* list;
  int64_t e, e1;    // list mode
  int64_t sb, s1;   // current id (both modes); range end
  int64_t P, Q, ns;
  __device__ void begin_range(int64_t s0, int64_t s_end, int64_t ns_) {
    list = nullptr;
    ns = ns_;
    sb = s0;
    s1 = s_end;
    if (sb < s1) tile_coords(sb, ns, P, Q);
  }
  __device__ void begin_list(const int32_t* l, int64_t e0, int64_t e_end, int64_t ns_) {
    list = l;
    ns = ns_;
    e = e0;
    e1 = e_end;
    if (e < e1) {
      sb = list[e];
      tile_coords(sb, ns, P, Q);
    }
  }
  __device__ bool valid() const { return list ? e < e1 : sb < s1; }
  __device__ void step() {
    if (list) {
      if (++e < e1) {
        sb = list[e];
        tile_coords(sb, ns, P, Q);
      }
      return;
    }
    ++sb;
    if (++Q == ns) {
      ++P;
      Q = P;
    }
  }
  // range mode: a super-block without a stored tile is skipped
  __device__ bool skip(const Sparse& sp) const { return list == nullptr && sp.empty_sb(sb); }
};

// Enumerates the stored tiles (global packed index) of the CTA's
// super-blocks in the walk order; -1 at the end.
struct TileEnum {
  SbWalk w;
  SbCursor c;
  Sparse::Rec rec;
  bool open, fresh;
  __device__ void begin(const SbCursor& c0, int64_t nt) {
    c = c0;
    w.nt = nt;
    w.ns = c.ns;
    open = false;
  }
  __device__ int64_t next(const Sparse& sp) {
    for (;;) {
      if (!open) {
        if (!c.valid()) return -1;
        if (sp.bits != nullptr) {
          rec = sp.record(c.sb);
          if (Sparse::empty(rec)) { c.step(); continue; }
        } else if (c.skip(sp)) {
          c.step();
          continue;
        }
        w.open(c.P, c.Q);
        open = true;
        fresh = true;
      }
      if (!fresh && !w.next()) {
        open = false;
        c.step();
        continue;
      }
      fresh = false;
      const bool stored = sp.bits != nullptr
                              ? Sparse::mask_of(rec, (int)((w.I - kSB * w.P) * kSB + (w.J - kSB * w.Q))) != 0u
                              : !sp.skip_tile(w.I, w.J, w.nt);
      if (stored) return tile_index(w.I, w.J, w.nt);
    }
  }
};

// Packed GEMV with super-block aggregation. Per stored tile (I, J) the 8
// consumer warps (16 rows each) form the row products sum_j T[i][j] v_J[j]
// (kept per lane across the row's tiles of the super-block) and, off the
// diagonal, the column products sum_i T[i][j] v_I[i] (combined across warps
// in smem and accumulated per column tile in I order). One 128-float record
// per (super-block, tile row) and per (super-block, tile column) goes to
// HBM: ~2 KB of partials per 16 tiles (1 MB) instead of 1 KB per 64 KB tile
// (measured: 1 KB of writes per 64 KB read costs a read stream ~7 %,
// scripts/probe/readbw.cu). Every sum has a fixed shape independent of the
// grid, so results are deterministic and grid-invariant.
template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
    sym_gemv_kernel(const T* __restrict__ tiles, int64_t nt, const float* __restrict__ v32,
                    float* __restrict__ rowp, float* __restrict__ colp,
                    const gpic_ctl* __restrict__ ctl, ShardRange sr, Sparse sp) {
  constexpr int kStages = TileTraits<T>::kStg;
  constexpr int kTileBytes = kTileFloats * (int)sizeof(T);
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* st = smem_align<128>(smem_raw);
  // [2 (super-block parity)][kWarps][kSB columns][128] column products
  float* red = reinterpret_cast<float*>(st + kStages * kTileBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * kWarps * kSB * kTS);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ns = (nt + kSB - 1) / kSB;
  // the shard's super-blocks [sb_lo, sb_hi) (whole matrix: all of them);
  // records are indexed from sb_lo, tiles from the shard's first tile
  const int64_t sb_lo = sr.sb_lo(ns), total = sr.sb_hi(ns) - sb_lo;
  SbCursor cur0;
  // dynamic schedule: super-blocks are claimed one at a time from the list
  // (atomic counter); the producer passes each claim to the consumers
  // through a small ring in shared memory. A super-block's records are
  // the same whichever CTA computes it, so results stay bitwise identical.
  const bool dyn = sp.list != nullptr && sp.sched != nullptr;
  constexpr int kQ = 4;
  __shared__ int32_t q_entry[kQ];
  __shared__ __align__(8) uint64_t q_full[kQ], q_empty[kQ];
  if (dyn) {
    if (threadIdx.x == 0) {
      for (int q = 0; q < kQ; ++q) {
        mbar_init(&q_full[q], 1);
        mbar_init(&q_empty[q], kWarps);
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  } else if (sp.list != nullptr) {
    // the non-empty super-blocks only, equal shares of their weight (cut
    // in advance by sb_list_kernel when it used this grid size)
    int64_t e0, e1;
    if (sp.ranges != nullptr && sp.ranges[0] == gridDim.x) {
      e0 = sp.ranges[1 + blockIdx.x];
      e1 = sp.ranges[2 + blockIdx.x];
    } else {
      const int64_t cnt = *sp.lcount;
      const int64_t w0 = sp.lpre[0], W = sp.lpre[cnt] - w0;
      e0 = lower_bound64(sp.lpre, 0, cnt, w0 + W * blockIdx.x / gridDim.x);
      e1 = blockIdx.x + 1 == gridDim.x
               ? cnt
               : lower_bound64(sp.lpre, 0, cnt, w0 + W * (blockIdx.x + 1) / gridDim.x);
    }
    if (e0 >= e1) return;
    cur0.begin_list(sp.list, e0, e1, ns);
  } else {
    int64_t s0 = sb_lo + total * blockIdx.x / gridDim.x;
    int64_t s1 = sb_lo + total * (blockIdx.x + 1) / gridDim.x;
    if (sp.sbp != nullptr) {  // equal shares of real work (non-zero tiles), not of super-blocks
      const int64_t sb_hi = sb_lo + total;
      const int64_t w0 = sp.sbp[sb_lo], W = sp.sbp[sb_hi] - w0;
      s0 = lower_bound64(sp.sbp, sb_lo, sb_hi, w0 + W * blockIdx.x / gridDim.x);
      s1 = blockIdx.x + 1 == gridDim.x
               ? sb_hi
               : lower_bound64(sp.sbp, sb_lo, sb_hi, w0 + W * (blockIdx.x + 1) / gridDim.x);
    }
    if (s0 >= s1) return;
    cur0.begin_range(s0, s1, ns);
  }
  SbWalk w;
  w.nt = nt;
  w.ns = ns;

  if (warp == kWarps && dyn) {  // producer, dynamic schedule
    if (lane != 0) return;
    int s = 0, q = 0;
    uint32_t ph = 0, qph = 0;
    const uint8_t* src0 = reinterpret_cast<const uint8_t*>(tiles);
    const uint64_t stream_pol = policy_evict_first();
    const int64_t cnt = *sp.lcount;
    for (;;) {
      const int64_t e = (int64_t)atomicAdd(sp.sched, 1u);
      const bool end = e >= cnt;
      mbar_wait(&q_empty[q], qph ^ 1);
      q_entry[q] = end ? -1 : (int32_t)e;
      mbar_arrive(&q_full[q]);
      if (++q == kQ) { q = 0; qph ^= 1; }
      if (end) break;
      SbCursor c1;
      c1.begin_list(sp.list, e, e + 1, ns);
      TileEnum cur;
      cur.begin(c1, nt);
      for (;;) {
        const int64_t t = cur.next(sp);
        if (t < 0) break;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], kTileBytes);
        if (sp.evict_first)
          bulk_load(st + s * kTileBytes, src0 + (t - sr.tile_base) * kTileBytes, kTileBytes,
                    &full[s], stream_pol);
        else
          bulk_load(st + s * kTileBytes, src0 + (t - sr.tile_base) * kTileBytes, kTileBytes,
                    &full[s]);
        if (++s == kStages) { s = 0; ph ^= 1; }
      }
    }
    // every CTA has made its last claim once all have counted in: the last
    // one resets the schedule for the next launch
    if (atomicAdd(sp.sched + 1, 1u) == gridDim.x - 1) {
      atomicExch(sp.sched, 0u);
      atomicExch(sp.sched + 1, 0u);
    }
    return;
  }
  if (warp == kWarps) {  // producer
    if (lane != 0) return;
    int s = 0;
    uint32_t ph = 0;
    const uint8_t* src0 = reinterpret_cast<const uint8_t*>(tiles);
    // the stored tiles of the CTA's super-blocks, in the consumers' order;
    // a second enumerator runs `ahead` tiles in front and prefetches them
    // into L2 (more bytes in flight than the smem ring holds)
    const uint64_t stream_pol = policy_evict_first();
    TileEnum cur, pre;
    cur.begin(cur0, nt);
    pre.begin(cur0, nt);
    const int ahead = sp.prefetch;
    for (int d = 0; d < ahead; ++d) {
      const int64_t t = pre.next(sp);
      if (t < 0) break;
      bulk_prefetch_l2(src0 + (t - sr.tile_base) * kTileBytes, kTileBytes);
    }
    for (;;) {
      const int64_t t = cur.next(sp);
      if (t < 0) break;
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], kTileBytes);
      if (sp.evict_first)  // the tile stream must not push the flags / v out of L2
        bulk_load(st + s * kTileBytes, src0 + (t - sr.tile_base) * kTileBytes, kTileBytes, &full[s],
                  stream_pol);
      else
        bulk_load(st + s * kTileBytes, src0 + (t - sr.tile_base) * kTileBytes, kTileBytes, &full[s]);
      if (++s == kStages) { s = 0; ph ^= 1; }
      if (ahead > 0) {
        const int64_t ta = pre.next(sp);
        if (ta >= 0) bulk_prefetch_l2(src0 + (ta - sr.tile_base) * kTileBytes, kTileBytes);
      }
    }
    return;
  }

  int s = 0;
  uint32_t ph = 0;
  int rb = 0;
  const int t = threadIdx.x;
  Sparse::Rec rec{};
  Sparse cs = sp;  // the consumers' view
  if (!sp.bits_consumer) cs.bits = nullptr;
  int q = 0;
  uint32_t qph = 0;
  for (;;) {
  if (dyn) {  // the producer's next claim
    mbar_wait(&q_full[q], qph);
    const int32_t e = q_entry[q];
    __syncwarp();
    if (lane == 0) mbar_arrive(&q_empty[q]);
    if (++q == kQ) { q = 0; qph ^= 1; }
    if (e < 0) break;
    cur0.begin_list(sp.list, e, e + 1, ns);
  }
  for (SbCursor cur = cur0; cur.valid(); cur.step()) {
    const int64_t sb = cur.sb;
    // no stored tile: its records are never read
    if (cs.bits != nullptr) {
      rec = cs.record(sb);
      if (Sparse::empty(rec)) continue;
    } else if (cur.skip(cs)) {
      continue;
    }
    w.open(cur.P, cur.Q);
    // per lane: the column products of the super-block's kSB tile columns,
    // accumulated over its tile rows (one cross-warp combine per super-block)
    float4 cpa[kSB];
#pragma unroll
    for (int c = 0; c < kSB; ++c) cpa[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    float acc[kRowsPerWarp];
#pragma unroll
    for (int i = 0; i < kRowsPerWarp; ++i) acc[i] = 0.f;
    float vi_l = lane < kRowsPerWarp ? __ldg(v32 + w.I * kTS + warp * kRowsPerWarp + lane) : 0.f;
    float4 vj = __ldg(reinterpret_cast<const float4*>(v32 + w.J * kTS) + lane);
    for (;;) {
      const int64_t I = w.I, J = w.J;
      bool zt, box_ok = true;
      if (cs.bits != nullptr) {
        const uint32_t m = Sparse::mask_of(rec, (int)((I - kSB * w.P) * kSB + (J - kSB * w.Q)));
        zt = m == 0u;
        // this lane's box (rows of this warp, columns 4 lane .. +3): stored?
        box_ok = (m >> ((warp >> 1) * 4 + (lane >> 3))) & 1u;
      } else {
        zt = cs.skip_tile(I, J, nt);
        if (cs.boxnz != nullptr && !zt)
          box_ok = cs.boxnz[tile_index(I, J, nt) * 16 + (warp >> 1) * 4 + (lane >> 3)] != 0;
      }
      const bool more = w.next();
      const bool row_end = !more || w.I != I;
      // next tile's v slices, one tile ahead
      float4 vj_n = vj;
      float vi_n = vi_l;
      if (more) {
        vj_n = __ldg(reinterpret_cast<const float4*>(v32 + w.J * kTS) + lane);
        if (row_end && lane < kRowsPerWarp) vi_n = __ldg(v32 + w.I * kTS + warp * kRowsPerWarp + lane);
      }
      if (!zt) {
      mbar_wait(&full[s], ph);
      const uint8_t* tile = st + s * kTileBytes + warp * kRowsPerWarp * kTS * (int)sizeof(T);
      // row products into acc; off the diagonal, column products into the
      // accumulator of tile column J (static index: one case per column)
      auto tile_products = [&](float4& cp, bool col) {
#pragma unroll
        for (int i = 0; i < kRowsPerWarp; ++i) {
          float4 a = TileTraits<T>::load4(tile + i * kTS * (int)sizeof(T), lane);
          if (!box_ok) a = make_float4(0.f, 0.f, 0.f, 0.f);  // unstored box: exact zeros
          float r = fmaf(a.x, vj.x, acc[i]);
          r = fmaf(a.y, vj.y, r);
          r = fmaf(a.z, vj.z, r);
          acc[i] = fmaf(a.w, vj.w, r);
          if (col) {
            const float vi = __shfl_sync(0xffffffffu, vi_l, i);
            cp.x = fmaf(a.x, vi, cp.x);
            cp.y = fmaf(a.y, vi, cp.y);
            cp.z = fmaf(a.z, vi, cp.z);
            cp.w = fmaf(a.w, vi, cp.w);
          }
        }
      };
      if (I == J) {
        tile_products(cpa[0], false);
      } else {
        switch ((int)(J - kSB * w.Q)) {
          case 0: tile_products(cpa[0], true); break;
          case 1: tile_products(cpa[1], true); break;
          case 2: tile_products(cpa[2], true); break;
          default: tile_products(cpa[3], true); break;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == kStages) { s = 0; ph ^= 1; }
      }
      if (row_end) {
        // transpose-reduce the 16 row accumulators across the 32 lanes
        // (fixed pattern): after 4 halving steps lane l holds row f(l) over
        // 16 lanes, the last xor-1 step completes it
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const bool up = lane & 16;
          const float send = up ? acc[k] : acc[k + 8];
          const float keep = up ? acc[k + 8] : acc[k];
          acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool up = lane & 8;
          const float send = up ? acc[k] : acc[k + 4];
          const float keep = up ? acc[k + 4] : acc[k];
          acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const bool up = lane & 4;
          const float send = up ? acc[k] : acc[k + 2];
          const float keep = up ? acc[k + 2] : acc[k];
          acc[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        {
          const bool up = lane & 2;
          const float send = up ? acc[0] : acc[1];
          const float keep = up ? acc[1] : acc[0];
          acc[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
        }
        acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
        const int row = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                        ((lane >> 1) & 1);
        if ((lane & 1) == 0)
          rowp[((sb - sb_lo) * kSB + (I - kSB * w.P)) * kTS + warp * kRowsPerWarp + row] = acc[0];
#pragma unroll
        for (int i = 0; i < kRowsPerWarp; ++i) acc[i] = 0.f;
      }
      vj = vj_n;
      vi_l = vi_n;
      if (!more) break;
    }
    // the super-block's column records: the 8 warps combine in order
    // (double-buffered by super-block, one barrier)
    float* rw = red + rb * kWarps * kSB * kTS;
#pragma unroll
    for (int c = 0; c < kSB; ++c) reinterpret_cast<float4*>(rw + (warp * kSB + c) * kTS)[lane] = cpa[c];
    asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
    if (t < kTS)
#pragma unroll
      for (int c = 0; c < kSB; ++c) {
        float sum = 0.f;
#pragma unroll
        for (int w8 = 0; w8 < kWarps; ++w8) sum += rw[(w8 * kSB + c) * kTS + t];
        colp[((sb - sb_lo) * kSB + c) * kTS + t] = sum;
      }
    rb ^= 1;
  }
  if (!dyn) break;
  }
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One CTA per tile row R (128 rows of y), kSeg segments over the row's
// ns + 1 super-block records in a fixed order: column records of the
// super-blocks (P', Q) for P' = 0 .. Q (Q = R / kSB; tiles (I, R) with I < R),
// then row records of (Q, Q') for Q' = Q .. ns - 1 (tiles (R, J >= R)); the
// segment sums are added in order. The shape depends on NT only.
constexpr int kSeg = 8;

__global__ void __launch_bounds__(kTS * kSeg)
    sym_reduce_kernel(const float* __restrict__ rowp, const float* __restrict__ colp, int64_t n,
                      int64_t nt, const double* __restrict__ deg, const PeerTable pt,
                      gpic_ctl* ctl, ShardRange sr, Sparse sp) {
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  __shared__ double part[kSeg][kTS];
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t p_hi = sr.p_hi < ns ? sr.p_hi : ns;
  const int64_t R = kSB * sr.p_lo + blockIdx.x;  // rows above the shard get nothing from it
  const int o = threadIdx.x % kTS, sg = threadIdx.x / kTS;
  const int64_t Q = R / kSB, k = R - kSB * Q;
  const int64_t sb0 = sr.sb_lo(ns);
  // the shard's records of row R: column records of (P', Q), P' in
  // [p_lo, min(Q, p_hi - 1)], then row records of (Q, Q') if Q is its own
  const int64_t ncol = (Q < p_hi - 1 ? Q : p_hi - 1) - sr.p_lo + 1;
  const int64_t nrow = Q < p_hi ? ns - Q : 0;
  const int64_t terms = ncol + nrow;
  const int64_t p0 = terms * sg / kSeg, p1 = terms * (sg + 1) / kSeg;
  if (sp.tlist != nullptr) {
    // only the non-empty records, in the same order and segments: the sum
    // is the one below bit for bit (the skipped terms are exact zeros)
    const int32_t* tl = sp.tlist + Q * sp.tld;
    const int L = sp.tcount[Q];
    double s2 = 0.0;
    for (int e = 0; e < L; ++e) {
      const int64_t p = tl[e];
      if (p < p0) continue;
      if (p >= p1) break;
      const int64_t sbi = p < ncol ? tile_index(sr.p_lo + p, Q, ns) : tile_index(Q, Q + (p - ncol), ns);
      s2 += (double)(p < ncol ? colp[((sbi - sb0) * kSB + k) * kTS + o]
                              : rowp[((sbi - sb0) * kSB + k) * kTS + o]);
    }
    part[sg][o] = s2;
  } else {
  auto load = [&](int64_t p) {
    const int64_t sbi = p < ncol ? tile_index(sr.p_lo + p, Q, ns) : tile_index(Q, Q + (p - ncol), ns);
    if (sp.empty_sb(sbi)) return 0.f;  // no records: a super-block of zero tiles
    return p < ncol ? colp[((sbi - sb0) * kSB + k) * kTS + o]
                    : rowp[((sbi - sb0) * kSB + k) * kTS + o];
  };
  double s = 0.0;
  int64_t p = p0;
  for (; p + 4 <= p1; p += 4) {  // independent loads in flight, added in order
    float x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = load(p + u);
#pragma unroll
    for (int u = 0; u < 4; ++u) s += (double)x[u];
  }
  for (; p < p1; ++p) s += (double)load(p);
  part[sg][o] = s;
  }
  __syncthreads();
  const int64_t i = R * kTS + o;
  if (sg == 0 && i < n) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kSeg; ++q) t += part[q][o];
    const double val = deg != nullptr ? t / deg[i] : t;
    const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
    const int own = pt.scatter ? slice_owner(i, n, pt.nranks) : -1;
    for (int r = 0; r < pt.nranks; ++r)
      if (own < 0 || own == r) pt.y[r][parity][i] = val;
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
      for (int r = 0; r < pt.nranks; ++r) st_release_sys(pt.flags[r] + pt.self, epoch);
    }
  }
}

// The reduce over the per-super-row term lists (whole matrix, sparse): one
// thread per row, all kSeg segments in turn — the same per-segment sums and
// the same in-order combine as sym_reduce_kernel (bit for bit), without the
// 8 threads per row that each walked the list, and small CTAs that all fit
// on the GPU at once. Row i = R kTS + o; returns sum / deg_i (deg != null).
__device__ __forceinline__ double reduce_list_row(const float* __restrict__ rowp,
                                                  const float* __restrict__ colp, int64_t n,
                                                  int64_t nt, const double* __restrict__ deg,
                                                  const Sparse& sp, int64_t R, int o) {
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t Q = R / kSB, k = R - kSB * Q;
  const int64_t ncol = Q + 1, terms = ncol + (ns - Q);
  const int32_t* tl = sp.tlist + Q * sp.tld;
  const int L = sp.tcount[Q];
  const int64_t i = R * kTS + o;
  const double di = deg != nullptr && i < n ? deg[i] : 1.0;  // in flight with the partials
  double t = 0.0, seg_sum = 0.0;
  int sg = 0;
  int64_t p1 = terms / kSeg;  // end of segment 0
  // kBatch independent loads in flight per thread, then the in-order adds
  // (the loads, not the adds, are the latency: ~40 records per row)
  constexpr int kBatch = 16;
  for (int e0 = 0; e0 < L; e0 += kBatch) {
    // unconditional (clamped) loads: a guarded load becomes a branch that
    // serialises load and use
    float val[kBatch];
    int32_t pp[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) pp[j] = tl[min(e0 + j, L - 1)];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int64_t p = pp[j];
      const int64_t sbi = p < ncol ? tile_index(p, Q, ns) : tile_index(Q, Q + (p - ncol), ns);
      const float* src = p < ncol ? colp : rowp;
      val[j] = __ldcs(src + (sbi * kSB + k) * kTS + o);
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      if (e0 + j >= L) break;
      while (pp[j] >= p1) {  // close the segments before p, in order
        t += seg_sum;
        seg_sum = 0.0;
        ++sg;
        p1 = terms * (sg + 1) / kSeg;
      }
      seg_sum += (double)val[j];
    }
  }
  for (; sg < kSeg; ++sg) {
    t += seg_sum;
    seg_sum = 0.0;
  }
  return deg != nullptr ? t / di : t;
}

// The stop / flag epilogue is sym_reduce_kernel's.
__global__ void __launch_bounds__(kTS)
    sym_reduce_list_kernel(const float* __restrict__ rowp, const float* __restrict__ colp,
                           int64_t n, int64_t nt, const double* __restrict__ deg,
                           const PeerTable pt, gpic_ctl* ctl, Sparse sp, double* tau_part,
                           unsigned* tau_ready, int tau_mode,
                           const unsigned long long* lowcnt) {
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  const int64_t R = blockIdx.x;
  const int o = threadIdx.x;
  const int64_t i = R * kTS + o;
  const double val = reduce_list_row(rowp, colp, n, nt, deg, sp, R, o);
  const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
  if (i < n) {
    const int own = pt.scatter ? slice_owner(i, n, pt.nranks) : -1;
    for (int r = 0; r < pt.nranks; ++r)
      if (own < 0 || own == r) pt.y[r][parity][i] = val;
  }
  // one whole-matrix rank: tau right here (kTailTauAlways), or when no
  // low-degree row will still rewrite y (kTailTauIfNoLow, device count)
  if (tau_mode == kTailTauAlways || (tau_mode == kTailTauIfNoLow && *lowcnt == 0ull))
    tail::tau_in_reduce(pt.y[0][parity], n, R, nt, tau_part, tau_ready, ctl);
  if (pt.flags[0] == nullptr) return;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&ctl->arrive[2], 1u);
    if (prev == gridDim.x - 1) {
      ctl->arrive[2] = 0u;
      __threadfence_system();
      const uint64_t epoch = ctl->sync_epoch + (uint64_t)ctl->iter + 1;
      for (int r = 0; r < pt.nranks; ++r) st_release_sys(pt.flags[r] + pt.self, epoch);
    }
  }
}

// One iteration's tail in one launch (whole matrix, one rank, list reduce):
// y = the list reduce (two tile rows per 256-thread CTA) -> grid barrier ->
// the low-degree rows' fp64 y (lowdeg.cuh, only when the device-side count
// is non-zero; one more barrier) -> tau, v' = y / tau, delta, stop
// (tail.cuh). Every value is computed by the same device code, with the
// same shapes, as sym_reduce_list_kernel + lowdeg_row_kernel + tail_kernel:
// results are bitwise those of the three-kernel sequence.
__global__ void __launch_bounds__(tail::kRedThreads, 3)
    sym_iter_tail_kernel(const float* __restrict__ rowp, const float* __restrict__ colp,
                         int64_t n, int64_t nt, const double* __restrict__ deg, double* y0,
                         double* y1, Sparse sp, LowRows low, const double* low_deg,
                         double low_scale, double* __restrict__ part, double* __restrict__ v64,
                         float* __restrict__ v32, double* __restrict__ hist, gpic_ctl* ctl,
                         unsigned tail_ctas, unsigned* ready) {
  __shared__ double sh[tail::kRedThreads];
  extern __shared__ double xs[];
  if (*(volatile int32_t*)&ctl->stop) return;
  const int t = ctl->iter;
  double* y = (t & 1) ? y1 : y0;
  const unsigned tgen0 = *(volatile unsigned*)&ctl->tau_gen;  // read before arriving
  unsigned bgen = *(volatile unsigned*)&ctl->bar_gen;
  constexpr int kRows = tail::kRedThreads / kTS;  // tile rows per CTA pass
  const int o = threadIdx.x % kTS;
  const unsigned long long cnt = low.d_count != nullptr ? *low.d_count : 0ull;
  constexpr int64_t kChunkTiles = kRedBlock / kTS;  // 16 tile rows per tail chunk
  static_assert(kChunkTiles % kRows == 0, "a CTA pass stays inside one chunk");
  for (int64_t R0 = (int64_t)blockIdx.x * kRows; R0 < nt; R0 += (int64_t)gridDim.x * kRows) {
    const int64_t R = R0 + threadIdx.x / kTS;
    if (R < nt) {
      const double val = reduce_list_row(rowp, colp, n, nt, deg, sp, R, o);
      const int64_t i = R * kTS + o;
      if (i < n) y[i] = val;
    }
    if (cnt == 0ull) {  // publish the pass's tile rows to the chunk's owner
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ready + R0 / kChunkTiles, (unsigned)(nt - R0 < kRows ? nt - R0 : kRows));
      }
    }
  }
  if (cnt != 0ull) {
    tail::grid_barrier(ctl, bgen);
    bgen = *(volatile unsigned*)&ctl->bar_gen;  // stable: nobody arrives before this CTA
    const double* v = v64 + (int64_t)(t & 1) * n;
    for (unsigned long long r = blockIdx.x; r < cnt; r += gridDim.x) {
      const int64_t i = low.list[r];
      const double s = lowdeg::matvec_row(low.x, n, low.d, low.kind, low_scale, i, low_deg[i], v,
                                          xs, sh);
      if (threadIdx.x == 0) y[i] = s;
    }
    tail::grid_barrier(ctl, bgen);
  }
  // the tail on as many CTAs as tail_kernel's grid (one per 2048-row chunk,
  // at most one per SM): fewer CTAs arriving at and spinning on its barrier
  const int64_t nb = (n + kRedBlock - 1) / kRedBlock;
  const unsigned ncta = (unsigned)min(nb, (int64_t)min(gridDim.x, tail_ctas));
  if (blockIdx.x >= ncta) return;
  tail::chunk_sums<true>(y, n, part, sh, ncta, cnt == 0ull ? ready : nullptr);
  tail::finish<true>(y, n, part, v64, v32, hist, ctl, t, tgen0, sh, ncta);
}

// Degrees over the same per-super-row term lists (whole matrix, sparse):
// one thread per row; the live tiles of row tile R come, in ascending p,
// from the non-empty super-blocks of its column (tiles (p, R), p < R) and
// row (tiles (R, p), p >= R) with their 32-byte box records; the segment
// sums and their in-order combine are sym_degree_kernel's, bit for bit.
__global__ void __launch_bounds__(kTS)
    sym_degree_list_kernel(const float* __restrict__ degrow, const float* __restrict__ degcol,
                           int64_t n, int64_t nt, int nhalf, double* __restrict__ deg,
                           gpic_ctl* ctl, Sparse sp) {
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t R = blockIdx.x;
  const int o = threadIdx.x;
  const int64_t Q = R / kSB, k = R - kSB * Q;
  const int64_t ncol = Q + 1;
  const int32_t* tl = sp.tlist + Q * sp.tld;
  const int L = sp.tcount[Q];
  double t = 0.0, seg = 0.0;
  int sg = 0;
  int64_t p1 = nt / kSeg;
  auto to_segment = [&](int64_t p) {
    while (p >= p1) {
      t += seg;
      seg = 0.0;
      ++sg;
      p1 = nt * (sg + 1) / kSeg;
    }
  };
  // per term: every live tile's partials loaded first (up to 4 tiles x 4
  // values in flight), then added in the order of the one-at-a-time walk;
  // the next term's index and box record are loaded a term ahead (a deeper
  // pipeline holding the next term's partials too measured slower: 97 vs
  // 66 us, registers)
  auto term_sb = [&](int64_t term) {
    return term < ncol ? tile_index(term, Q, ns) : tile_index(Q, Q + (term - ncol), ns);
  };
  int64_t term_next = L > 0 ? tl[0] : 0;
  Sparse::Rec rec_next = L > 0 ? sp.record(term_sb(term_next)) : Sparse::Rec{};
  for (int e = 0; e < L; ++e) {
    const int64_t term = term_next;
    const Sparse::Rec rec = rec_next;
    if (e + 1 < L) {
      term_next = tl[e + 1];
      rec_next = sp.record(term_sb(term_next));
    }
    float c[kSB][4];
    bool live[kSB];
    int64_t p0;
    const bool col = term < ncol;
    if (col) {  // super-block (term, Q): tiles (p, R), p < R
      const int64_t P = term;
      const int64_t pe = min(min(kSB * P + kSB, R), nt);
      p0 = kSB * P;
#pragma unroll
      for (int j = 0; j < kSB; ++j) {
        const int64_t p = p0 + j;
        live[j] = p < pe && Sparse::mask_of(rec, (int)(j * kSB + k)) != 0u;
        // unconditional loads (a dead slot reads a valid dummy address):
        // guarded loads compile to branches that serialise load and use
        const float* src = degcol + (live[j] ? tile_index(p, R, nt) * 4 * kTS : 0) + o;
#pragma unroll
        for (int q = 0; q < 4; ++q) c[j][q] = src[q * kTS];
      }
    } else {  // super-block (Q, Q'): tiles (R, p), p >= R
      const int64_t Qp = Q + (term - ncol);
      const int64_t pe = min(kSB * Qp + kSB, nt);
      p0 = kSB * Qp;
#pragma unroll
      for (int j = 0; j < kSB; ++j) {
        const int64_t p = p0 + j;
        live[j] = p >= R && p < pe && Sparse::mask_of(rec, (int)(k * kSB + j)) != 0u;
        const float* src = degrow + (live[j] ? tile_index(R, p, nt) * nhalf * kTS : 0) + o;
        c[j][0] = src[0];
        c[j][1] = src[(nhalf - 1) * kTS];
      }
    }
#pragma unroll
    for (int j = 0; j < kSB; ++j) {
      if (!live[j]) continue;
      to_segment(p0 + j);
      if (col) {
        seg += (double)c[j][0] + (double)c[j][1] + (double)c[j][2] + (double)c[j][3];
      } else {
        seg += (double)c[j][0];
        if (nhalf == 2) seg += (double)c[j][1];
      }
    }
  }
  for (; sg < kSeg; ++sg) {
    t += seg;
    seg = 0.0;
  }
  const int64_t i = R * kTS + o;
  if (i < n) {
    deg[i] = t;
    if (ctl != nullptr && t <= 0.0) raise_status(ctl, GPIC_E_ZERO_DEGREE, i, -1, t);
  }
}

// Per super-row Q (one warp each): the term indices of its non-empty
// records in ascending order — column records (P', Q), P' <= Q, as P', then
// row records (Q, Q'), Q' >= Q, as Q + 1 + (Q' - Q) — from the super-block
// weights (weight 1: no stored tile, no record). Whole matrix only.
__global__ void reduce_terms_kernel(const int64_t* __restrict__ sbp, int64_t ns,
                                    int32_t* __restrict__ tlist, int32_t* __restrict__ tcount,
                                    int64_t tld) {
  const int lane = threadIdx.x & 31;
  const int64_t Q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (Q >= ns) return;
  int32_t* out = tlist + Q * tld;
  int cnt = 0;
  const int64_t ncol = Q + 1, terms = ncol + (ns - Q);
  for (int64_t c0 = 0; c0 < terms; c0 += 32) {
    const int64_t p = c0 + lane;
    bool nz = false;
    if (p < terms) {
      const int64_t sbi = p < ncol ? tile_index(p, Q, ns) : tile_index(Q, Q + (p - ncol), ns);
      nz = sbp[sbi + 1] - sbp[sbi] > 1;
    }
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    if (nz) out[cnt + __popc(m & ((1u << lane) - 1u))] = (int32_t)p;
    cnt += __popc(m);
  }
  if (lane == 0) tcount[Q] = cnt;
}

// deg_i from the affinity epilogue's partials (same segmented fixed shape as
// sym_reduce): column partials (4 row quadrants) of tiles (p, R), p < R,
// then row partials (nhalf column halves) of tiles (R, p), p >= R.
__global__ void __launch_bounds__(kTS * kSeg)
    sym_degree_kernel(const float* __restrict__ degrow, const float* __restrict__ degcol,
                      int64_t n, int64_t nt, int nhalf, double* __restrict__ deg, gpic_ctl* ctl,
                      ShardRange sr, Sparse sp, const uint8_t* __restrict__ pskip, int64_t pB,
                      int64_t pnb) {
  extern __shared__ int32_t live[];  // sparse: the row's tiles that hold a stored box, ascending
  __shared__ double part[kSeg][kTS];
  __shared__ int32_t wcount[kSeg * kTS / 32];
  __shared__ int32_t nlive;
  // shard: tile rows [tr_lo, tr_hi) are stored (from tile_base); row R gets
  // the column partials of its stored tiles (p, R) and, if R is its own,
  // the row partials of (R, p >= R). deg is then the shard's partial.
  const int64_t tr_lo = kSB * sr.p_lo, tr_hi = kSB * sr.p_hi < nt ? kSB * sr.p_hi : nt;
  const int64_t R = tr_lo + blockIdx.x;
  const int o = threadIdx.x % kTS, sg = threadIdx.x / kTS;
  const int64_t p0 = nt * sg / kSeg, p1 = nt * (sg + 1) / kSeg;
  double s = 0.0;
  // 4 tiles' partials in flight per step, then added in order
  auto load4 = [&](int64_t p, float (&x)[4]) {
    x[0] = x[1] = x[2] = x[3] = 0.f;
    if (p < R) {
      if (p < tr_lo || p >= tr_hi) return;  // tile (p, R) lives on another shard
      const float* c = degcol + (tile_index(p, R, nt) - sr.tile_base) * 4 * kTS + o;
      x[0] = c[0]; x[1] = c[kTS]; x[2] = c[2 * kTS]; x[3] = c[3 * kTS];
    } else {
      if (R >= tr_hi) return;
      const float* r = degrow + (tile_index(R, p, nt) - sr.tile_base) * nhalf * kTS + o;
      x[0] = r[0]; x[1] = nhalf == 2 ? r[kTS] : 0.f;
    }
  };
  auto add4 = [&](int64_t p, const float (&x)[4]) {
    if (p < R) {
      s += (double)x[0] + (double)x[1] + (double)x[2] + (double)x[3];
    } else {
      s += (double)x[0];
      if (nhalf == 2) s += (double)x[1];
    }
  };
  if (sp.boxnz != nullptr) {
    // sparse: first the ordered list of tiles with a stored box (pruned
    // block pairs and all-zero tiles are exact zeros: skipping them leaves
    // every fp64 sum bit-identical), then the same segments over it
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (t == 0) nlive = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < nt; c0 += kSeg * kTS) {
      const int64_t p = c0 + t;
      bool k = p < nt;
      if (k && pskip != nullptr) k = pskip[(R * kTS / pB) * pnb + p * kTS / pB] == 0;
      if (k) k = !sp.skip_tile(p < R ? p : R, p < R ? R : p, nt);
      const unsigned m = __ballot_sync(0xffffffffu, k);
      if (lane == 0) wcount[w] = __popc(m);
      __syncthreads();
      if (k) {
        int pos = nlive + __popc(m & ((1u << lane) - 1u));
        for (int q = 0; q < w; ++q) pos += wcount[q];
        live[pos] = (int32_t)p;
      }
      __syncthreads();
      if (t == 0) {
        int tot = 0;
        for (int q = 0; q < kSeg * kTS / 32; ++q) tot += wcount[q];
        nlive += tot;
      }
      __syncthreads();
    }
    const int L = nlive;
    int a = 0;
    while (a < L && live[a] < p0) ++a;
    int b = a;
    while (b < L && live[b] < p1) ++b;
    for (; a + 4 <= b; a += 4) {
      float x[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) load4(live[a + u], x[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) add4(live[a + u], x[u]);
    }
    for (; a < b; ++a) {
      float x[4];
      load4(live[a], x);
      add4(live[a], x);
    }
  } else {
    int64_t p = p0;
    for (; p + 4 <= p1; p += 4) {
      float x[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) load4(p + u, x[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) add4(p + u, x[u]);
    }
    for (; p < p1; ++p) {
      float x[4];
      load4(p, x);
      add4(p, x);
    }
  }
  part[sg][o] = s;
  __syncthreads();
  const int64_t i = R * kTS + o;
  if (sg == 0 && i < n) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kSeg; ++q) t += part[q][o];
    deg[i] = t;
    if (ctl != nullptr && t <= 0.0) raise_status(ctl, GPIC_E_ZERO_DEGREE, i, -1, t);
  }
}

int g_sms = 0;

// tiles each GEMV producer prefetches into L2 ahead of its smem ring
// (GPIC_GEMV_PREFETCH, default 0: measured slower at config 3)
// GPIC_GEMV_LIST=0: walk every super-block id (A/B against the list)
int gemv_use_list() {
  const char* e = getenv("GPIC_GEMV_LIST");
  return e != nullptr ? atoi(e) : 1;
}

// GPIC_GEMV_DYN=0: static CTA ranges by super-block weight instead of the
// dynamic claims (A/B; measured at config 3: SM busy time max / mean 1.28
// with the static ranges)
int gemv_dynamic() {
  const char* e = getenv("GPIC_GEMV_DYN");
  return e != nullptr ? atoi(e) : 1;
}

// GPIC_GEMV_SHARD_LIST=0: packed shards walk their super-block id range with
// static weight ranges (A/B)
int gemv_shard_list() {
  const char* e = getenv("GPIC_GEMV_SHARD_LIST");
  return e == nullptr || atoi(e) != 0;
}

int gemv_evict_first() {
  const char* e = getenv("GPIC_GEMV_EVICT");
  return e != nullptr ? atoi(e) : 1;
}

int gemv_prefetch() {
  const char* e = getenv("GPIC_GEMV_PREFETCH");
  return e != nullptr ? atoi(e) : 0;
}

// GPIC_FUSED_TAIL=1: the fused iteration kernel instead of the three-kernel
// tail. Off by default: bitwise the same results, but measured no faster at
// config 3 (ncu: 33.0 us fused vs 14.2 + 3.2 + 16.0 us; in the graph
// 2.055 vs 2.038 ms per 6 iterations): the tail's time is the latency
// chain of its fixed-shape reductions, not the launches.
int fused_tail_enabled() {
  const char* e = getenv("GPIC_FUSED_TAIL");
  return e != nullptr && atoi(e) != 0;
}

// The fused iteration kernel in place of reduce + low rows + tail when the
// list reduce applies to one whole-matrix rank (no peer stores); false:
// nothing launched. Grid: the CTAs that are resident at once (its grid
// barriers spin), at most one per two tile rows.
bool launch_iter_tail(const IterTail* it, const float* rowp, const float* colp, int64_t n,
                      int64_t nt, const double* deg, const PeerTable& pt, gpic_ctl* ctl,
                      const Sparse& sp, cudaStream_t s) {
  if (it == nullptr || ctl == nullptr || sp.tlist == nullptr || pt.flags[0] != nullptr ||
      pt.nranks != 1 || pt.scatter || !fused_tail_enabled())
    return false;
  if (pt.y[0][0] != it->y0 || pt.y[0][1] != it->y1) return false;
  const size_t dyn = it->low.d <= lowdeg::kSmemD ? (size_t)it->low.d * sizeof(double) : 0;
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sym_iter_tail_kernel,
                                                    tail::kRedThreads, dyn) != cudaSuccess ||
      per_sm < 1)
    return false;
  const int64_t want = (nt + 1) / 2;
  const int64_t cap = (int64_t)per_sm * sms;
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  const double scale = -1.0 / (2.0 * it->low.sigma * it->low.sigma);
  sym_iter_tail_kernel<<<grid, tail::kRedThreads, dyn, s>>>(
      rowp, colp, n, nt, deg, it->y0, it->y1, sp, it->low, it->low_deg, scale, it->redpart,
      it->v64, it->v32, it->hist, ctl, (unsigned)sms,
      reinterpret_cast<unsigned*>(it->redpart + ceil_div(n, kRedBlock) + 1));
  return true;
}

// tau inside the list reduce (tail.cuh tau_in_reduce) for one whole-matrix
// rank without peer stores: opt-in, GPIC_TAU_IN_REDUCE=1 (not with
// GPIC_TAIL_SPLIT=1). Bitwise the tail's tau, but measured no faster at
// config 3 (2.002 vs 2.006 ms per 6 iterations): the chunk-completion chain
// at the end of the reduce costs what the tail's barrier did.
struct TauPlan {
  double* part = nullptr;
  unsigned* ready = nullptr;
  int mode = kTailSeparate;
  const unsigned long long* lowcnt = nullptr;
};
TauPlan tau_plan(const IterTail* it, const PeerTable& pt, const gpic_ctl* ctl, int64_t n) {
  static const bool on = [] {
    const char* e = getenv("GPIC_TAU_IN_REDUCE");
    const char* sp = getenv("GPIC_TAIL_SPLIT");
    return (e != nullptr && atoi(e) != 0) && !(sp != nullptr && atoi(sp) != 0);
  }();
  TauPlan tp;
  if (!on || it == nullptr || ctl == nullptr || pt.flags[0] != nullptr || pt.nranks != 1 ||
      pt.scatter || pt.y[0][0] != it->y0 || pt.y[0][1] != it->y1)
    return tp;
  if (it->low.count == 0) {
    tp.mode = kTailTauAlways;
  } else if (it->low.count < 0 && it->low.d_count != nullptr) {
    tp.mode = kTailTauIfNoLow;
    tp.lowcnt = it->low.d_count;
  } else {
    return tp;  // listed rows rewrite y after the reduce: the tail sums
  }
  tp.part = it->redpart;
  tp.ready = reinterpret_cast<unsigned*>(it->redpart + ceil_div(n, kRedBlock) + 1);
  return tp;
}

}  // namespace

void launch_sym_degree(const float* degrow, const float* degcol, int64_t n, int nhalf,
                       double* deg, gpic_ctl* ctl, cudaStream_t s, const ShardRange& sr,
                       const uint8_t* boxnz, const PruneMask* pm, const int64_t* sb_prefix) {
  const int64_t nt = ceil_div(n, kTS);
  const int64_t rows = nt - kSB * sr.p_lo;  // tile rows that can receive partials
  if (rows < 1) return;
  if (boxnz != nullptr && sb_prefix != nullptr && sr.p_lo == 0 && sr.tile_base == 0 &&
      gemv_use_list()) {
    // the per-super-row term lists and box records of the sparse prefix pass
    const SbList sl = sb_list(sb_prefix, n);
    const Sparse lp{boxnz, sb_prefix, sb_bits(sb_prefix, n), 0, 0, 0, sl.list, sl.lpre, sl.count,
                    sl.ranges, sl.tlist, sl.tcount, sl.tld, nullptr};
    sym_degree_list_kernel<<<(unsigned)nt, kTS, 0, s>>>(degrow, degcol, n, nt, nhalf, deg, ctl, lp);
    count_launch();
    return;
  }
  const Sparse sp{boxnz, nullptr, nullptr, 0, 0, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr};
  const size_t dyn = boxnz != nullptr ? (size_t)nt * 4 : 0;  // the live-tile list
  if (dyn > 48 * 1024)
    cudaFuncSetAttribute(sym_degree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  sym_degree_kernel<<<(unsigned)rows, kTS * kSeg, dyn, s>>>(
      degrow, degcol, n, nt, nhalf, deg, ctl, sr, sp, pm ? pm->skip : nullptr, pm ? pm->B : 1,
      pm ? pm->nb : 0);
  count_launch();
}

void sym_prepare() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(sym_gemv_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(sym_gemv_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
  }
}

void launch_reduce_terms(const int64_t* sb_prefix, int64_t nt, int32_t* tlist, int32_t* tcount,
                         int64_t tld, cudaStream_t s) {
  const int64_t ns = (nt + kSB - 1) / kSB;
  reduce_terms_kernel<<<(unsigned)ceil_div(ns, 8), 256, 0, s>>>(sb_prefix, ns, tlist, tcount, tld);
  count_launch();
}

// GEMV partial records (super-block rows / columns) or the affinity
// epilogue's per-tile degree partials, whichever is larger
int64_t sym_partial_floats(int64_t n) {
  const int64_t nt = ceil_div(n, kTS);
  const int64_t ns = ceil_div(nt, kSB);
  const int64_t tiles = nt * (nt + 1) / 2, recs = ns * (ns + 1) / 2 * kSB;
  return (tiles > recs ? tiles : recs) * kTS;
}

int launch_sym_gemv(const float* tiles, int64_t n, const float* v32, float* rowp, float* colp,
                     const double* deg, const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s,
                     const ShardRange& sr, const uint8_t* boxnz, const int64_t* sb_prefix,
                     const IterTail* it) {
  // packed shards: their box flags, super-block records and the list of
  // their non-empty super-blocks live in whole-triangle arrays (only the
  // shard's tiles flagged), so the list walk and its claims apply; the
  // per-super-row term lists of the list reduce are whole-matrix only
  const bool whole = sr.p_lo == 0 && sr.tile_base == 0 && sr.p_hi >= ceil_div(ceil_div(n, kTS), kSB);
  // GPIC_SB_BITS: 0 per-tile flags everywhere, 1 super-block records for
  // producer and consumers (default), 2 records for the producer only.
  // Measured at config 3 (scripts/gemv_ab.py, one box): id walk + flags
  // 0.500 ms, list + flags 0.465, list + records 0.424
  const int bits_mode = getenv("GPIC_SB_BITS") != nullptr ? atoi(getenv("GPIC_SB_BITS")) : 1;
  const bool lists = boxnz != nullptr && sb_prefix != nullptr && (whole || gemv_shard_list());
  const SbList sl = lists && gemv_use_list() ? sb_list(sb_prefix, n)
                                             : SbList{nullptr, nullptr, nullptr};
  Sparse sp{boxnz, boxnz != nullptr ? sb_prefix : nullptr,
            lists && bits_mode != 0 ? sb_bits(sb_prefix, n) : nullptr,
            gemv_prefetch(), bits_mode == 1, gemv_evict_first(), sl.list, sl.lpre, sl.count,
            whole ? sl.ranges : nullptr, whole ? sl.tlist : nullptr, whole ? sl.tcount : nullptr,
            sl.tld, nullptr};
  if (sl.list != nullptr && gemv_dynamic() && gemv_prefetch() == 0) sp.sched = sl.sched;
  sym_prepare();
  const int64_t nt = ceil_div(n, kTS);
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t total = sr.sb_hi(ns) - sr.sb_lo(ns);  // the shard's super-blocks
  const int grid = (int)(total < g_sms ? total : g_sms);
  const int64_t rows = nt - kSB * sr.p_lo;
  if (grid < 1 || rows < 1) return kTailSeparate;
  sym_gemv_kernel<float><<<grid, kThreads, kSmem, s>>>(tiles, nt, v32, rowp, colp, ctl, sr, sp);
  if (launch_iter_tail(it, rowp, colp, n, nt, deg, pt, ctl, sp, s)) {
    count_launch(2);
    return kTailFused;
  }
  if (sp.tlist != nullptr) {
    const TauPlan tp = tau_plan(it, pt, ctl, n);
    sym_reduce_list_kernel<<<(unsigned)nt, kTS, 0, s>>>(rowp, colp, n, nt, deg, pt, ctl, sp,
                                                        tp.part, tp.ready, tp.mode, tp.lowcnt);
    count_launch(2);
    return tp.mode;
  }
  else
    sym_reduce_kernel<<<(unsigned)rows, kTS * kSeg, 0, s>>>(rowp, colp, n, nt, deg, pt, ctl, sr, sp);
  count_launch(2);
  return kTailSeparate;
}

int launch_sym_gemv16(const void* tiles, int64_t n, const float* v32, float* rowp, float* colp,
                       const double* deg, const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s,
                       const uint8_t* boxnz, const int64_t* sb_prefix, const IterTail* it) {
  const SbList sl = boxnz != nullptr && gemv_use_list() ? sb_list(sb_prefix, n)
                                                        : SbList{nullptr, nullptr, nullptr};
  Sparse sp{boxnz, boxnz != nullptr ? sb_prefix : nullptr,
            boxnz != nullptr ? sb_bits(sb_prefix, n) : nullptr, gemv_prefetch(), 0,
            gemv_evict_first(), sl.list, sl.lpre, sl.count, sl.ranges, sl.tlist, sl.tcount,
            sl.tld, nullptr};
  if (sl.list != nullptr && gemv_dynamic() && gemv_prefetch() == 0) sp.sched = sl.sched;
  sym_prepare();
  const int64_t nt = ceil_div(n, kTS);
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t total = ns * (ns + 1) / 2;  // super-blocks
  const int grid = (int)(total < g_sms ? total : g_sms);
  const ShardRange all{};
  sym_gemv_kernel<__half><<<grid, kThreads, kSmem, s>>>(static_cast<const __half*>(tiles), nt, v32,
                                                            rowp, colp, ctl, all, sp);
  if (launch_iter_tail(it, rowp, colp, n, nt, deg, pt, ctl, sp, s)) {
    count_launch(2);
    return kTailFused;
  }
  if (sp.tlist != nullptr) {
    const TauPlan tp = tau_plan(it, pt, ctl, n);
    sym_reduce_list_kernel<<<(unsigned)nt, kTS, 0, s>>>(rowp, colp, n, nt, deg, pt, ctl, sp,
                                                        tp.part, tp.ready, tp.mode, tp.lowcnt);
    count_launch(2);
    return tp.mode;
  }
  else
    sym_reduce_kernel<<<(unsigned)nt, kTS * kSeg, 0, s>>>(rowp, colp, n, nt, deg, pt, ctl, all, sp);
  count_launch(2);
  return kTailSeparate;
}

}  // namespace gpic
