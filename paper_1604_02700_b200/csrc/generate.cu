// Device-side App-B data generation: the d-dimensional
// Gaussian blobs of datasets.gaussian_blobs written straight into HBM, so an
// n = 1M run (512 MB of fp64 X) needs neither a host generator pass nor an
// H2D copy.
//
// Row i belongs to blob c with offsets[c] <= i < offsets[c+1] (the caller's
// graded or balanced counts); x_if = centers[c][f] + noise * z_if + offset.
// z comes from a counter-based Philox4x32-10 stream keyed by the seed: the
// pair of elements (2p, 2p+1) of the row-major n x d array uses counter
// (p_lo, p_hi, 0, 0), whose four words form two 53-bit uniforms for one
// Box-Muller draw. The output therefore depends only on (seed, n, d, centres,
// counts), not on the launch shape; oracle/pic_oracle.py restates it in numpy.
// HBM-write-bound: 8 n d bytes (+ 8 n for labels), one store per element.
#include "common.cuh"
#include "ops.h"

namespace gpic {

namespace {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__global__ void __launch_bounds__(256) blobs_kernel(const double* __restrict__ centers,
                                                    const int64_t* __restrict__ offsets, int64_t n,
                                                    int d, int k, uint64_t seed, double noise,
                                                    double offset, double* __restrict__ x,
                                                    int64_t* __restrict__ labels) {
  const int64_t total = n * (int64_t)d;
  const int64_t pairs = (total + 1) / 2;
  const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < pairs;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint4 w = philox4x32_10(make_uint4((uint32_t)p, (uint32_t)((uint64_t)p >> 32), 0u, 0u),
                                  key);
    const uint64_t a = ((uint64_t)w.x << 21) | (w.y >> 11);
    const uint64_t b = ((uint64_t)w.z << 21) | (w.w >> 11);
    const double u1 = 1.0 - (double)a * 0x1.0p-53;  // (0, 1]
    const double u2 = (double)b * 0x1.0p-53;        // [0, 1)
    const double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincospi(2.0 * u2, &sn, &cs);
    const double z[2] = {r * cs, r * sn};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t e = 2 * p + h;
      if (e >= total) break;
      const int64_t i = e / d;
      const int f = (int)(e - i * d);
      int c = 0;
      while (c + 1 < k && offsets[c + 1] <= i) ++c;
      x[e] = centers[(int64_t)c * d + f] + noise * z[h] + offset;
      if (f == 0 && labels) labels[i] = c;
    }
  }
}

}  // namespace

int launch_generate_blobs(const double* centers, const int64_t* offsets, int64_t n, int d, int k,
                          uint64_t seed, double noise, double offset, double* x, int64_t* labels,
                          cudaStream_t s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t pairs = (n * (int64_t)d + 1) / 2;
  int64_t grid = (pairs + 255) / 256;
  if (grid > (int64_t)sms * 8) grid = (int64_t)sms * 8;
  blobs_kernel<<<(unsigned)grid, 256, 0, s>>>(centers, offsets, n, d, k, seed, noise, offset, x,
                                              labels);
  count_launch();
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

}  // namespace gpic
