// Internal host-side launchers shared between the translation units of
// libgpic. Everything here is asynchronous on `stream`.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gpic.h"

namespace gpic {

constexpr int kTileM = 128;  // affinity row tile
constexpr int kTileN = 128;  // affinity column tile
constexpr int kRedBlock = 2048;  // fixed block of the tau / delta reductions

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

int32_t feature_pitch(int32_t d);
int64_t row_pad(int64_t n);
int64_t affinity_pitch(int64_t n);

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
  int64_t kscratch_bytes;
  uint8_t* end;
};

int64_t workspace_bytes(int64_t n, int32_t d, int32_t k, int64_t rows, int32_t max_iter);
int carve(void* base, int64_t bytes, int64_t n, int32_t d, int32_t k, int64_t rows,
          int32_t max_iter, Workspace* ws);

// prepare.cu
void launch_ctl_init(gpic_ctl* ctl, double eps, int32_t max_iter, cudaStream_t s);
void launch_prepare(const double* x, int64_t n, int32_t d, float* xhi, float* xlo, float* sqn,
                    double* colpart, double* mean, gpic_ctl* ctl, cudaStream_t s);

// affinity_simt.cu / affinity_tc.cu
void launch_affinity_simt(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                          int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2,
                          float* a, int64_t lda, float* rowpart, int64_t rows_pad,
                          cudaStream_t s);
int launch_affinity_tc(const float* xhi, const float* xlo, const float* sqn, int64_t n,
                       int32_t dp, int64_t row_lo, int64_t row_hi, float neg_scale_log2, float* a,
                       int64_t lda, float* rowpart, int64_t rows_pad, cudaStream_t s);
void launch_degree(const float* rowpart, int64_t rows, int64_t rows_pad, int64_t n_ctiles,
                   int64_t row_lo, double* deg, gpic_ctl* ctl, cudaStream_t s);

// power.cu
void launch_tree_sum(const double* v, int64_t n, double* part, double* out, gpic_ctl* ctl,
                     cudaStream_t s);
void launch_scale_vector(const double* src, int64_t n, const double* tau, double* v64,
                         float* v32, int64_t v32_len, cudaStream_t s);
void launch_scale_by(const double* src, int64_t n, double tau, double* dst, float* dst32,
                     int64_t f32_len, cudaStream_t s);
void gemv_prepare();
void launch_gemv(const float* a, int64_t lda, int64_t rows, int64_t row_lo, const float* v32,
                 const double* deg, double* y, const gpic_ctl* ctl, cudaStream_t s);
void launch_iteration_tail(const double* y, int64_t n, double* redpart, double* v64,
                           float* v32, double* hist, gpic_ctl* ctl, cudaStream_t s);
void launch_copy_result(const double* v64, int64_t n, double* out, const gpic_ctl* ctl,
                        cudaStream_t s);
int run_power_loop(const float* a, int64_t lda, const double* deg, int64_t n, double* y,
                   double* redpart, double* v64, float* v32, double* hist, gpic_ctl* ctl,
                   int32_t max_iter, cudaStream_t s);

// kmeans.cu
int64_t kmeans_scratch_bytes(int64_t n, int32_t k);
int launch_kmeans1d(const double* v, int64_t n, int32_t k, int64_t first_index,
                    const double* h_uniforms, int32_t max_rounds, double tol, int64_t* labels,
                    void* scratch, gpic_ctl* ctl, cudaStream_t s);

}  // namespace gpic
