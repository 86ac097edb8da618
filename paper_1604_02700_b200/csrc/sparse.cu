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
constexpr int kScanThreads = 1024;

__device__ __forceinline__ bool tile_stored(const uint8_t* boxnz, int64_t t) {
  const uint4 f = *reinterpret_cast<const uint4*>(boxnz + t * 16);
  return (f.x | f.y | f.z | f.w) != 0u;
}

// prefix[s + 1] = prefix[s] + 8 x (stored tiles of super-block s) + 1 over
// the packed super-block triangle; one CTA, contiguous per-thread segments
// (super-block coordinates stepped, not searched), then a block scan.
__global__ void __launch_bounds__(kScanThreads)
    sb_weight_scan_kernel(const uint8_t* __restrict__ boxnz, int64_t nt,
                          int64_t* __restrict__ prefix) {
  __shared__ int64_t sh[kScanThreads];
  const int64_t ns = (nt + kSB - 1) / kSB;
  const int64_t count = ns * (ns + 1) / 2;
  const int t = threadIdx.x;
  const int64_t seg = (count + kScanThreads - 1) / kScanThreads;
  const int64_t a = min(count, t * seg), b = min(count, a + seg);
  auto coords = [&](int64_t s, int64_t& P, int64_t& Q) {
    int64_t lo = 0, hi = ns - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (mid * ns - mid * (mid - 1) / 2 <= s) lo = mid; else hi = mid - 1;
    }
    P = lo;
    Q = P + (s - (P * ns - P * (P - 1) / 2));
  };
  auto weight = [&](int64_t P, int64_t Q) {
    int64_t w = 1;
    for (int64_t I = kSB * P; I < min(kSB * P + kSB, nt); ++I)
      for (int64_t J = max(I, kSB * Q); J < min(kSB * Q + kSB, nt); ++J)
        if (tile_stored(boxnz, I * nt - I * (I - 1) / 2 + (J - I))) w += 8;
    return w;
  };
  auto step = [&](int64_t& P, int64_t& Q) {
    if (++Q == ns) Q = ++P;
  };
  int64_t s = 0, P = 0, Q = 0;
  if (a < b) coords(a, P, Q);
  for (int64_t i = a; i < b; ++i, step(P, Q)) s += weight(P, Q);
  sh[t] = s;
  __syncthreads();
  for (int o = 1; o < kScanThreads; o <<= 1) {  // Hillis-Steele inclusive scan
    const int64_t v = t >= o ? sh[t - o] : 0;
    __syncthreads();
    sh[t] += v;
    __syncthreads();
  }
  int64_t run = t > 0 ? sh[t - 1] : 0;
  if (t == 0) prefix[0] = 0;
  if (a < b) coords(a, P, Q);
  for (int64_t i = a; i < b; ++i, step(P, Q)) {
    run += weight(P, Q);
    prefix[i + 1] = run;
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
  return al(nt * (nt + 1) / 2 * 16) + al((ns * (ns + 1) / 2 + 1) * 8);
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
  sb_weight_scan_kernel<<<1, kScanThreads, 0, s>>>(m.boxnz, m.nt, m.sb_prefix);
  count_launch();
}

void launch_box_fill(const SparseMask& m, uint8_t v, cudaStream_t s) {
  const int64_t bytes = m.nt * (m.nt + 1) / 2 * 16;
  fill_kernel<<<(unsigned)ceil_div(bytes, 256), 256, 0, s>>>(m.boxnz, bytes, v);
  count_launch();
}

}  // namespace gpic
