// Block sparsity of the stored affinity tiles: exact zero boxes.
//
// A_ij = exp(-|x_i - x_j|^2 / 2 sigma^2) is an fp32 zero whenever the
// exponent is below the smallest normal float (ex2.approx.ftz flushes at
// |x_i - x_j|^2 / 2 sigma^2 > 87.3). Well-separated clusters make most of A
// such zeros: at config 3 every tile pair joining two different blobs
// (e^-95 .. e^-110), ~90 % of the packed triangle.
//
// The affinity epilogue knows, per 32 x 32 box it produces, whether every
// value is exactly 0 (warp vote). It then skips that box's store and writes
// boxnz[tile][quadrant * 4 + chunk] = 0 (1 for a stored box); a tile with no
// stored box costs no HBM write at all. The packed GEMV loads only tiles with
// a stored box and treats the unstored boxes of a loaded tile as zeros, and
// the degree partials are sums of the same (zero) values — so every product,
// degree and embedding is bit-identical to the dense computation (an exact
// zero adds nothing to any fp32 / fp64 sum). No geometric bound is involved:
// the flags are the computed values' own.
//
// GEMV balance: sb_weight_scan turns the flags into a prefix of super-block
// weights (8 per stored tile + 1 per super-block) so every GEMV CTA gets an
// equal share of the tiles that are actually read.
#include <cstdlib>

#include "common.cuh"
#include "ops.h"

namespace gpic {

namespace {

constexpr int kT = 128;  // rows per tile
constexpr int kSB = 4;   // tiles per super-block side (sym.cu)
constexpr int kMaxGrid = 1024;  // GEMV CTAs the precomputed ranges cover
// host copies of the grid sizes (a stable source for the async H2D copy)
struct GridWords {
  int64_t v[kMaxGrid + 1];
  constexpr GridWords() : v() {
    for (int i = 0; i <= kMaxGrid; ++i) v[i] = i;
  }
  const int64_t& operator[](int i) const { return v[i]; }
};
constexpr GridWords kGridWords{};
constexpr int kScanThreads = 1024;

__device__ __forceinline__ bool tile_stored(const uint8_t* boxnz, int64_t t) {
  const uint4 f = *reinterpret_cast<const uint4*>(boxnz + t * 16);
  return (f.x | f.y | f.z | f.w) != 0u;
}

// weight of super-block s (packed triangle of kSB x kSB tile super-blocks):
// 8 x its stored tiles + 1, written to prefix[s + 1]; and its box bits:
// bits[s][(I - kSB P) * kSB + (J - kSB Q)] = the 16 box flags of tile (I, J)
// (bit quadrant * 4 + chunk), 0 for tiles below the diagonal / past nt —
// one 32-byte record the GEMV reads per super-block instead of a flag load
// per tile. One thread each.
__global__ void sb_weight_kernel(const uint8_t* __restrict__ boxnz, int64_t nt,
                                 int64_t* __restrict__ prefix, uint16_t* __restrict__ bits) {
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t count = ns * (ns + 1) / 2;
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s == 0) prefix[0] = 0;
  if (s >= count) return;
  int64_t lo = 0, hi = ns - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (mid * ns - mid * (mid - 1) / 2 <= s) lo = mid; else hi = mid - 1;
  }
  const int64_t P = lo, Q = P + (s - (P * ns - P * (P - 1) / 2));
  int64_t w = 1;
  uint16_t b[kSB * kSB];
#pragma unroll
  for (int q = 0; q < kSB * kSB; ++q) b[q] = 0;
  for (int64_t I = kSB * P; I < min(kSB * P + kSB, nt); ++I)
    for (int64_t J = max(I, kSB * Q); J < min(kSB * Q + kSB, nt); ++J) {
      const uint4 f = *reinterpret_cast<const uint4*>(boxnz + (I * nt - I * (I - 1) / 2 + (J - I)) * 16);
      const uint32_t wd[4] = {f.x, f.y, f.z, f.w};
      uint16_t m = 0;
#pragma unroll
      for (int q = 0; q < 16; ++q) m |= (uint16_t)(((wd[q >> 2] >> (8 * (q & 3))) & 0xffu) != 0u) << q;
      b[(I - kSB * P) * kSB + (J - kSB * Q)] = m;
      if (m) w += 8;
    }
  prefix[s + 1] = w;
  uint4* out = reinterpret_cast<uint4*>(bits + s * kSB * kSB);
  out[0] = make_uint4(b[0] | (uint32_t)b[1] << 16, b[2] | (uint32_t)b[3] << 16,
                      b[4] | (uint32_t)b[5] << 16, b[6] | (uint32_t)b[7] << 16);
  out[1] = make_uint4(b[8] | (uint32_t)b[9] << 16, b[10] | (uint32_t)b[11] << 16,
                      b[12] | (uint32_t)b[13] << 16, b[14] | (uint32_t)b[15] << 16);
}

// in-place inclusive scan of prefix[1 .. count]: one CTA walks the array in
// coalesced 1024-element chunks (block scan + running carry)
__global__ void __launch_bounds__(kScanThreads)
    sb_scan_kernel(int64_t nt, int64_t* __restrict__ prefix) {
  // each thread a contiguous segment: its sum, one warp-shuffle block scan of
  // the segment sums, then the segment rewritten from its offset
  __shared__ int64_t wsum[kScanThreads / 32];
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t count = ns * (ns + 1) / 2;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t seg = (count + kScanThreads - 1) / kScanThreads;
  const int64_t a = min(count, t * seg), b = min(count, a + seg);
  int64_t c = 0;
  for (int64_t i = a; i < b; ++i) c += prefix[i + 1];
  int64_t incl = c;  // inclusive scan within the warp
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    int64_t v = lane < kScanThreads / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    if (lane < kScanThreads / 32) wsum[lane] = v;  // inclusive over warps
  }
  __syncthreads();
  int64_t run = (w > 0 ? wsum[w - 1] : 0) + incl - c;  // exclusive offset of the segment
  for (int64_t i = a; i < b; ++i) {
    run += prefix[i + 1];
    prefix[i + 1] = run;
  }
}

// the ascending list of non-empty super-blocks (weight > 1) with the weight
// prefix at each entry (lpre[e] = prefix[list[e]], lpre[count] = total): the
// GEMV walks only these, so its CTAs never touch (and never load the
// weights of) the ~80 % empty ones. One CTA, contiguous segments.
__global__ void __launch_bounds__(kScanThreads)
    sb_list_kernel(int64_t nt, const int64_t* __restrict__ prefix, int32_t* __restrict__ list,
                   int64_t* __restrict__ lpre, int64_t* __restrict__ count, int grid,
                   int64_t* __restrict__ ranges) {
  __shared__ int64_t sh[kScanThreads];
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t total = ns * (ns + 1) / 2;
  const int t = threadIdx.x;
  const int64_t seg = (total + kScanThreads - 1) / kScanThreads;
  const int64_t a = min(total, t * seg), b = min(total, a + seg);
  int64_t c = 0;
  for (int64_t s = a; s < b; ++s) c += prefix[s + 1] - prefix[s] > 1;
  sh[t] = c;
  __syncthreads();
  for (int o = 1; o < kScanThreads; o <<= 1) {
    const int64_t add = t >= o ? sh[t - o] : 0;
    __syncthreads();
    sh[t] += add;
    __syncthreads();
  }
  int64_t w = t > 0 ? sh[t - 1] : 0;
  for (int64_t s = a; s < b; ++s)
    if (prefix[s + 1] - prefix[s] > 1) {
      list[w] = (int32_t)s;
      lpre[w] = prefix[s];
      ++w;
    }
  if (t == kScanThreads - 1) {
    *count = sh[t];
    lpre[sh[t]] = prefix[total];
    unsigned* sched = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(count) + 64);
    sched[0] = 0u;  // the GEMV's dynamic schedule (sym.cu)
    sched[1] = 0u;
  }
  // the GEMV's CTA ranges over the list for a grid of `grid` CTAs (equal
  // shares of weight, the kernel's own lower_bound), so its CTAs start
  // without a search: ranges[b] .. ranges[b + 1]
  __syncthreads();
  const int64_t cnt = sh[kScanThreads - 1];
  const int64_t w0 = lpre[0], W = lpre[cnt] - w0;
  for (int b = t; b <= grid; b += kScanThreads) {
    int64_t e;
    if (b == grid) {
      e = cnt;
    } else {
      const int64_t target = w0 + W * b / grid;
      int64_t lo = 0, hi = cnt;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (lpre[mid] >= target) hi = mid; else lo = mid + 1;
      }
      e = lo;
    }
    ranges[b] = e;
  }
}

// sb_scan_kernel + sb_list_kernel in one CTA with the weights staged in
// shared memory (config 3: 19,306 super-blocks, 154 KB): every global
// access is coalesced and the per-thread segment walks run on shared
// memory. The same segments, sums and entries: the same integers.
constexpr int64_t kScanSmemMax = 200 * 1024;
__global__ void __launch_bounds__(kScanThreads)
    sb_scan_list_smem_kernel(int64_t nt, int64_t* __restrict__ prefix, int32_t* __restrict__ list,
                             int64_t* __restrict__ lpre, int64_t* __restrict__ count_out,
                             int grid, int64_t* __restrict__ ranges) {
  extern __shared__ int64_t sp[];  // prefix[0 .. total]
  __shared__ int64_t wsum[kScanThreads / 32];
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t total = ns * (ns + 1) / 2;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int64_t i = t; i <= total; i += kScanThreads) sp[i] = prefix[i];
  __syncthreads();
  const int64_t seg = (total + kScanThreads - 1) / kScanThreads;
  const int64_t a = min(total, t * seg), b = min(total, a + seg);
  // block-wide exclusive scan of one value per thread (warp shuffles)
  auto block_excl = [&](int64_t c, int64_t* tot) {
    int64_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    if (w == 0) {
      int64_t v = lane < kScanThreads / 32 ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (lane < kScanThreads / 32) wsum[lane] = v;
    }
    __syncthreads();
    const int64_t r = (w > 0 ? wsum[w - 1] : 0) + incl - c;
    *tot = wsum[kScanThreads / 32 - 1];
    __syncthreads();  // wsum is reused
    return r;
  };
  // the weight prefix (sb_scan_kernel)
  int64_t c = 0;
  for (int64_t i = a; i < b; ++i) c += sp[i + 1];
  int64_t tot;
  int64_t run = block_excl(c, &tot);
  for (int64_t i = a; i < b; ++i) {
    run += sp[i + 1];
    sp[i + 1] = run;
  }
  __syncthreads();
  for (int64_t i = t + 1; i <= total; i += kScanThreads) prefix[i] = sp[i];
  // the non-empty list (sb_list_kernel)
  int64_t k = 0;
  for (int64_t q = a; q < b; ++q) k += sp[q + 1] - sp[q] > 1;
  int64_t cnt;
  int64_t e = block_excl(k, &cnt);
  for (int64_t q = a; q < b; ++q)
    if (sp[q + 1] - sp[q] > 1) {
      list[e] = (int32_t)q;
      lpre[e] = sp[q];
      ++e;
    }
  if (t == kScanThreads - 1) {
    *count_out = cnt;
    lpre[cnt] = sp[total];
    unsigned* sched = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(count_out) + 64);
    sched[0] = 0u;  // the GEMV's dynamic schedule (sym.cu)
    sched[1] = 0u;
  }
  __syncthreads();
  const int64_t w0 = lpre[0], W = lpre[cnt] - w0;
  for (int g = t; g <= grid; g += kScanThreads) {
    int64_t r;
    if (g == grid) {
      r = cnt;
    } else {
      const int64_t target = w0 + W * g / grid;
      int64_t lo = 0, hi = cnt;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (lpre[mid] >= target) hi = mid; else lo = mid + 1;
      }
      r = lo;
    }
    ranges[g] = r;
  }
}

__global__ void fill_kernel(uint8_t* p, int64_t n, uint8_t v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace

bool sparse_enabled() {
  const char* e = getenv("GPIC_SPARSE");
  return e == nullptr || atoi(e) != 0;
}

int64_t sparse_mask_bytes(int64_t n, int32_t /*d*/) {
  const int64_t nt = ceil_div(n, kT);
  const int64_t ns = ceil_div(nt, kSB);
  auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  const int64_t nsb = ns * (ns + 1) / 2;
  return al(nt * (nt + 1) / 2 * 16) + al((nsb + 1) * 8) + al(nsb * kSB * kSB * 2) + al(8) +
         al((nsb + 1) * 8) + al(nsb * 4) + al((kMaxGrid + 2) * 8) + al(ns * (ns + 2) * 4) +
         al(ns * 4);
}

// the non-empty super-block list behind the box bits (sb_list_kernel)
SbList sb_list(const int64_t* sb_prefix, int64_t n) {
  SbList L{nullptr, nullptr, nullptr};
  if (sb_prefix == nullptr) return L;
  auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  const int64_t ns = ceil_div(ceil_div(n, kT), kSB), nsb = ns * (ns + 1) / 2;
  const uint8_t* p = reinterpret_cast<const uint8_t*>(sb_prefix) + al((nsb + 1) * 8) +
                     al(nsb * kSB * kSB * 2);
  L.count = reinterpret_cast<const int64_t*>(p);
  L.sched = reinterpret_cast<unsigned*>(const_cast<uint8_t*>(p) + 64);  // same 256-byte slot
  p += al(8);
  L.lpre = reinterpret_cast<const int64_t*>(p);
  p += al((nsb + 1) * 8);
  L.list = reinterpret_cast<const int32_t*>(p);
  p += al(nsb * 4);
  L.ranges = reinterpret_cast<const int64_t*>(p);  // [0] = grid, then grid + 1 bounds
  p += al((kMaxGrid + 2) * 8);
  L.tld = ns + 2;
  L.tlist = reinterpret_cast<const int32_t*>(p);
  p += al(ns * (ns + 2) * 4);
  L.tcount = reinterpret_cast<const int32_t*>(p);
  return L;
}

// the per-super-block box bits live right behind the GEMV weights
const uint16_t* sb_bits(const int64_t* sb_prefix, int64_t n) {
  if (sb_prefix == nullptr) return nullptr;
  const int64_t ns = ceil_div(ceil_div(n, kT), kSB);
  const int64_t b = ((ns * (ns + 1) / 2 + 1) * 8 + 255) & ~int64_t(255);
  return reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(sb_prefix) + b);
}

SparseMask carve_sparse(void* base, int64_t n, int32_t /*d*/) {
  auto al = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  const int64_t nt = ceil_div(n, kT);
  const int64_t ns = ceil_div(nt, kSB);
  uint8_t* p = static_cast<uint8_t*>(base);
  SparseMask m;
  m.nt = nt;
  m.boxnz = p;
  p += al(nt * (nt + 1) / 2 * 16);
  m.sb_prefix = reinterpret_cast<int64_t*>(p);
  m.n_sb = ns * (ns + 1) / 2;
  return m;
}

void launch_sparse_prefix(const SparseMask& m, cudaStream_t s) {
  sb_weight_kernel<<<(unsigned)ceil_div(m.n_sb, 256), 256, 0, s>>>(
      m.boxnz, m.nt, m.sb_prefix, const_cast<uint16_t*>(sb_bits(m.sb_prefix, m.nt * kT)));
  const SbList L = sb_list(m.sb_prefix, m.nt * kT);
  const int64_t smem = (m.n_sb + 1) * 8;
  // GPIC_SB_SCAN_SMEM=0: the two global-memory kernels (A/B)
  const char* se = getenv("GPIC_SB_SCAN_SMEM");
  const bool staged = smem <= kScanSmemMax && (se == nullptr || atoi(se) != 0);
  if (!staged) sb_scan_kernel<<<1, kScanThreads, 0, s>>>(m.nt, m.sb_prefix);
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = sms < kMaxGrid ? sms : kMaxGrid;
  int64_t* ranges = const_cast<int64_t*>(L.ranges);
  cudaMemcpyAsync(ranges, &kGridWords[grid], 8, cudaMemcpyHostToDevice, s);
  if (staged) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(sb_scan_list_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kScanSmemMax);
      attr = true;
    }
    sb_scan_list_smem_kernel<<<1, kScanThreads, smem, s>>>(
        m.nt, m.sb_prefix, const_cast<int32_t*>(L.list), const_cast<int64_t*>(L.lpre),
        const_cast<int64_t*>(L.count), grid, ranges + 1);
  } else {
    sb_list_kernel<<<1, kScanThreads, 0, s>>>(m.nt, m.sb_prefix, const_cast<int32_t*>(L.list),
                                              const_cast<int64_t*>(L.lpre),
                                              const_cast<int64_t*>(L.count), grid, ranges + 1);
  }
  launch_reduce_terms(m.sb_prefix, m.nt, const_cast<int32_t*>(L.tlist),
                      const_cast<int32_t*>(L.tcount), L.tld, s);
  count_launch(staged ? 2 : 3);
}

void launch_box_fill(const SparseMask& m, uint8_t v, cudaStream_t s) {
  const int64_t bytes = m.nt * (m.nt + 1) / 2 * 16;
  fill_kernel<<<(unsigned)ceil_div(bytes, 256), 256, 0, s>>>(m.boxnz, bytes, v);
  count_launch();
}

}  // namespace gpic
