// Symmetric packed storage: A is exactly symmetric (affinity.py:96-103;
// test_affinity.py:81-87), so only the upper triangle of 128 x 128 tiles is
// stored (tile (I, J), J >= I, contiguous 64 KB at tile_index(I, J)). That
// halves the bytes of the two HBM-bound stages: the affinity store and the
// per-iteration GEMV read (2n^2 instead of 4n^2 bytes).
//
//   sym_gemv_kernel   streams every stored tile once (1-D bulk copies into a
//                     3-stage smem ring) and produces, per tile, the 128 row
//                     partials  sum_j T[i][j] v_J[j]   (for y_I) and, off the
//                     diagonal, the 128 column partials  sum_i T[i][j] v_I[i]
//                     (for y_J = (T^T v_I)_J). fp32 within a tile.
//   sym_reduce_kernel y_i = sum over the row's tiles in column order (fp64):
//                     column partials of tiles (J', R), J' < R, then row
//                     partials of tiles (R, J), J >= R; / deg_i; stored into
//                     every rank's y (same epilogue as the dense GEMV).
// Degrees are the same GEMV with v = 1 (exactly consistent with the stored
// fp32 values). Every sum has a fixed order, so results are deterministic.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "ops.h"
#include "sm100.cuh"

namespace gpic {

namespace {

constexpr int kTS = 128;
constexpr int kTileFloats = kTS * kTS;
constexpr int kStages = 3;  // fp32 tiles (64 KB); fp16 tiles (32 KB) use 2x the stages
constexpr int kWarps = 8;                   // consumers; 16 rows each
constexpr int kRowsPerWarp = kTS / kWarps;  // 16
constexpr int kThreads = (kWarps + 1) * 32;
constexpr int kSmem = kStages * kTileFloats * 4 + 2 * kWarps * kTS * 4 + 64 + 128;
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

template <typename T>
__global__ void __launch_bounds__(kThreads, 1)
    sym_gemv_kernel(const T* __restrict__ tiles, int64_t nt, const float* __restrict__ v32,
                    float* __restrict__ rowp, float* __restrict__ colp,
                    const gpic_ctl* __restrict__ ctl, int split, int pol, int ablate) {
  constexpr int kStages = TileTraits<T>::kStg;
  constexpr int kTileBytes = kTileFloats * (int)sizeof(T);
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* st = smem_align<128>(smem_raw);
  float* red = reinterpret_cast<float*>(st + kStages * kTileBytes);  // [2][kWarps][128] column partials
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * kWarps * kTS);
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
  const int64_t total = nt * (nt + 1) / 2;
  const int64_t t0 = total * blockIdx.x / gridDim.x;
  const int64_t t1 = total * (blockIdx.x + 1) / gridDim.x;

  if (warp == kWarps) {  // producer
    if (lane != 0) return;
    int s = 0;
    uint32_t ph = 0;
    const uint64_t once = policy_evict_first();  // every tile is read once per pass
    const uint32_t piece = kTileBytes / split;
    const uint8_t* src0 = reinterpret_cast<const uint8_t*>(tiles);
    for (int64_t t = t0; t < t1; ++t) {
      mbar_wait(&empty[s], ph ^ 1);
      mbar_expect_tx(&full[s], kTileBytes);
      for (int p = 0; p < split; ++p) {
        uint8_t* dst = st + s * kTileBytes + p * piece;
        const uint8_t* src = src0 + t * kTileBytes + p * piece;
        if (pol) bulk_load(dst, src, piece, &full[s], once);
        else bulk_load(dst, src, piece, &full[s]);
      }
      if (++s == kStages) { s = 0; ph ^= 1; }
    }
    return;
  }

  int s = 0;
  uint32_t ph = 0;
  int rb = 0;
  int64_t I = 0, J = 0;
  if (t0 < t1) tile_coords(t0, nt, I, J);
  // v slices of the next tile are loaded one tile ahead (L2 latency off the
  // per-tile critical path)
  auto load_vj = [&](int64_t j) { return __ldg(reinterpret_cast<const float4*>(v32 + j * kTS) + lane); };
  auto load_vi = [&](int64_t i) {
    return lane < kRowsPerWarp ? __ldg(v32 + i * kTS + warp * kRowsPerWarp + lane) : 0.f;
  };
  float4 vj_next = make_float4(0.f, 0.f, 0.f, 0.f);
  float vi_next = 0.f;
  if (t0 < t1) {
    vj_next = load_vj(J);
    vi_next = load_vi(I);
  }
  for (int64_t t = t0; t < t1; ++t) {
    const float4 vj = vj_next;
    const float vi_l = vi_next;
    if (t + 1 < t1) {
      const int64_t In = J + 1 == nt ? I + 1 : I, Jn = J + 1 == nt ? I + 1 : J + 1;
      vj_next = load_vj(Jn);
      vi_next = load_vi(In);
    }
    mbar_wait(&full[s], ph);
    if (ablate == 1) {  // measurement only (GPIC_SYM_ABLATE=1): stream without compute
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == kStages) { s = 0; ph ^= 1; }
      if (++J == nt) { ++I; J = I; }
      continue;
    }
    const uint8_t* tile = st + s * kTileBytes + warp * kRowsPerWarp * kTS * (int)sizeof(T);
    float acc[kRowsPerWarp];
    float4 cp = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < kRowsPerWarp; ++i) {
      const float4 a = TileTraits<T>::load4(tile + i * kTS * (int)sizeof(T), lane);
      const float vi = __shfl_sync(0xffffffffu, vi_l, i);
      float r = a.x * vj.x;
      r = fmaf(a.y, vj.y, r);
      r = fmaf(a.z, vj.z, r);
      acc[i] = fmaf(a.w, vj.w, r);
      cp.x = fmaf(a.x, vi, cp.x);
      cp.y = fmaf(a.y, vi, cp.y);
      cp.z = fmaf(a.z, vi, cp.z);
      cp.w = fmaf(a.w, vi, cp.w);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == kStages) { s = 0; ph ^= 1; }
    // transpose-reduce the 16 row partials across the 32 lanes (fixed
    // pattern): after 4 halving steps lane l holds row f(l) over 16 lanes,
    // the last xor-1 step completes it.
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
    if ((lane & 1) == 0) rowp[t * kTS + warp * kRowsPerWarp + row] = acc[0];
    // column partials: combine the 8 warps in order
    float* rw = red + rb * kWarps * kTS;
    reinterpret_cast<float4*>(rw + warp * kTS)[lane] = cp;
    asm volatile("bar.sync 1, %0;" ::"n"(kWarps * 32) : "memory");
    if (I != J && threadIdx.x < kTS) {
      float c = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) c += rw[w * kTS + threadIdx.x];
      colp[t * kTS + threadIdx.x] = c;
    }
    rb ^= 1;  // double-buffered: the next tile writes the other half
    if (++J == nt) { ++I; J = I; }
  }
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One CTA per tile row R (128 rows), 8 segments of the row's NT tiles per
// row: segment s sums its contiguous column-tile range in order (column
// partials of tiles (p, R) for p < R, row partials of (R, p) for p >= R),
// then the 8 segment sums are added in order. The shape depends on NT only.
constexpr int kSeg = 8;

__global__ void __launch_bounds__(kTS * kSeg)
    sym_reduce_kernel(const float* __restrict__ rowp, const float* __restrict__ colp, int64_t n,
                      int64_t nt, const double* __restrict__ deg, const PeerTable pt,
                      gpic_ctl* ctl) {
  if (ctl != nullptr && *(volatile const int32_t*)&ctl->stop) return;
  __shared__ double part[kSeg][kTS];
  const int64_t R = blockIdx.x;
  const int o = threadIdx.x % kTS, sg = threadIdx.x / kTS;
  const int64_t p0 = nt * sg / kSeg, p1 = nt * (sg + 1) / kSeg;
  double s = 0.0;
  const int64_t diag = tile_index(R, R, nt);
  auto load = [&](int64_t p) {
    return p < R ? colp[tile_index(p, R, nt) * kTS + o] : rowp[(diag + (p - R)) * kTS + o];
  };
  // batches of 8 independent loads in flight, then added in order
  int64_t p = p0;
  for (; p + 8 <= p1; p += 8) {
    float x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = load(p + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += (double)x[u];
  }
  for (; p < p1; ++p) s += (double)load(p);
  part[sg][o] = s;
  __syncthreads();
  const int64_t i = R * kTS + o;
  if (sg == 0 && i < n) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kSeg; ++q) t += part[q][o];
    const double val = deg != nullptr ? t / deg[i] : t;
    const int parity = ctl != nullptr ? (ctl->iter & 1) : 0;
    for (int p = 0; p < pt.nranks; ++p) pt.y[p][parity][i] = val;
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

// deg_i from the affinity epilogue's partials (same segmented fixed shape as
// sym_reduce): column partials (4 row quadrants) of tiles (p, R), p < R,
// then row partials (nhalf column halves) of tiles (R, p), p >= R.
__global__ void __launch_bounds__(kTS * kSeg)
    sym_degree_kernel(const float* __restrict__ degrow, const float* __restrict__ degcol,
                      int64_t n, int64_t nt, int nhalf, double* __restrict__ deg, gpic_ctl* ctl) {
  __shared__ double part[kSeg][kTS];
  const int64_t R = blockIdx.x;
  const int o = threadIdx.x % kTS, sg = threadIdx.x / kTS;
  const int64_t p0 = nt * sg / kSeg, p1 = nt * (sg + 1) / kSeg;
  double s = 0.0;
  for (int64_t p = p0; p < p1; ++p) {
    if (p < R) {
      const float* c = degcol + tile_index(p, R, nt) * 4 * kTS + o;
      s += (double)c[0] + (double)c[kTS] + (double)c[2 * kTS] + (double)c[3 * kTS];
    } else {
      const float* r = degrow + tile_index(R, p, nt) * nhalf * kTS + o;
      s += (double)r[0];
      if (nhalf == 2) s += (double)r[kTS];
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
    if (t <= 0.0) raise_status(ctl, GPIC_E_ZERO_DEGREE, i, -1, t);
  }
}

int g_sms = 0;
int g_split = 1, g_pol = 0;  // evict_first on the tile stream measured 4% slower
int g_ablate = 0;  // GEMV copy shape (GPIC_SYM_SPLIT pieces per tile, GPIC_SYM_POL)

}  // namespace

void launch_sym_degree(const float* degrow, const float* degcol, int64_t n, int nhalf,
                       double* deg, gpic_ctl* ctl, cudaStream_t s) {
  const int64_t nt = ceil_div(n, kTS);
  sym_degree_kernel<<<(unsigned)nt, kTS * kSeg, 0, s>>>(degrow, degcol, n, nt, nhalf, deg, ctl);
  count_launch();
}

void sym_prepare() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(sym_gemv_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    cudaFuncSetAttribute(sym_gemv_kernel<__half>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (const char* e = getenv("GPIC_SYM_SPLIT")) {
      const int v = atoi(e);
      if (v == 1 || v == 2 || v == 4 || v == 8 || v == 16) g_split = v;
    }
    if (const char* e = getenv("GPIC_SYM_POL")) g_pol = atoi(e) != 0;
    if (const char* e = getenv("GPIC_SYM_ABLATE")) g_ablate = atoi(e);
  }
}

int64_t sym_partial_floats(int64_t n) {
  const int64_t nt = ceil_div(n, kTS);
  return nt * (nt + 1) / 2 * kTS;
}

void launch_sym_gemv(const float* tiles, int64_t n, const float* v32, float* rowp, float* colp,
                     const double* deg, const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s) {
  sym_prepare();
  const int64_t nt = ceil_div(n, kTS);
  const int64_t total = nt * (nt + 1) / 2;
  const int grid = (int)(total < g_sms ? total : g_sms);
  sym_gemv_kernel<float><<<grid, kThreads, kSmem, s>>>(tiles, nt, v32, rowp, colp, ctl, g_split,
                                                           g_pol, g_ablate);
  sym_reduce_kernel<<<(unsigned)nt, kTS * kSeg, 0, s>>>(rowp, colp, n, nt, deg, pt, ctl);
  count_launch(2);
}

void launch_sym_gemv16(const void* tiles, int64_t n, const float* v32, float* rowp, float* colp,
                       const double* deg, const PeerTable& pt, gpic_ctl* ctl, cudaStream_t s) {
  sym_prepare();
  const int64_t nt = ceil_div(n, kTS);
  const int64_t total = nt * (nt + 1) / 2;
  const int grid = (int)(total < g_sms ? total : g_sms);
  sym_gemv_kernel<__half><<<grid, kThreads, kSmem, s>>>(static_cast<const __half*>(tiles), nt, v32,
                                                            rowp, colp, ctl, g_split, g_pol,
                                                            g_ablate);
  sym_reduce_kernel<<<(unsigned)nt, kTS * kSeg, 0, s>>>(rowp, colp, n, nt, deg, pt, ctl);
  count_launch(2);
}

}  // namespace gpic
