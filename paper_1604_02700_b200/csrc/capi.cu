// extern "C" entry points of libgpic.so (declared in include/gpic.h).
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <vector>
#include <string>

#include "common.cuh"
#include "ops.h"

static_assert(sizeof(gpic_ctl) == 256, "gpic_ctl must stay 256 bytes");

namespace gpic {

unsigned long long g_launches = 0;
static thread_local std::string g_err;
// detail of the last failure (gpic_last_detail): status, index / (row, col), value
struct LastDetail {
  int status = GPIC_OK;
  int64_t index = -1, index2 = -1;
  double value = 0.0;
};
static thread_local LastDetail g_detail;

int fail_cuda(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
          ") at " + what;
  return GPIC_E_CUDA;
}

int fail(int code, const char* msg) {
  g_err = msg;
  g_detail = LastDetail();
  g_detail.status = code;
  return code;
}

// 64 features = one 128-byte swizzle row of the fp16 tensor operands
int32_t feature_pitch(int32_t d) { return (int32_t)round_up(d, 64); }
// rows padded to the tile plus one spare tile: shard row tiles may start
// at any row, so a tile can overhang n by up to 127 rows.
int64_t row_pad(int64_t n) { return round_up(n, kTileM) + kTileM; }
int64_t affinity_pitch(int64_t n) { return round_up(n, 32); }
// d_xhi: hi + lo fp16 planes (n_pad x dp each) + the norm block (4 planes of
// n_pad x 16 fp16) = n_pad x (dp + 32) floats
int64_t operand_floats(int64_t n, int32_t d) { return row_pad(n) * (feature_pitch(d) + 32); }

static inline int64_t al(int64_t b) { return (b + 255) & ~int64_t(255); }

// Page-locked readback slots of the routing decision (one set per host
// thread): a pageable destination would make the copy itself the sync.
static double* routing_probe() {
  static thread_local double* p = nullptr;
  if (p == nullptr && cudaMallocHost(reinterpret_cast<void**>(&p), 64) != cudaSuccess) p = nullptr;
  return p;
}

int64_t workspace_bytes(int64_t n, int32_t d, int32_t k, int64_t rows, int32_t /*max_iter*/) {
  const int64_t dp = feature_pitch(d), npad = row_pad(n);
  const int64_t rows_pad = round_up(rows, kTileM);
  const int64_t n_ctiles = ceil_div(n, kTileN);
  int64_t b = al(sizeof(gpic_ctl));
  b += al(operand_floats(n, d) * 4);          // xhi: fp16 planes + norm block
  b += al(npad * dp * 4);                     // xlo
  b += al(npad * 4);                          // sqn
  b += al(ceil_div(n, 256) * d * 8);          // colpart
  b += al((int64_t)(d + 2) * 8);              // mean + max|x - mean| + spread R^2
  b += al(n_ctiles * rows_pad * 4);           // rowpart
  b += al((ceil_div(n, kRedBlock) + 1) * 8 + ceil_div(n, kRedBlock) * 4);  // redpart + chunk counters
  b += al(n * 8);                             // y
  b += al(n * 8);                             // deg
  b += al(2 * n * 8);                         // v64
  b += al(vector_pitch(n) * 4);               // v32
  b += al(kmeans_scratch_bytes(n, k));        // kmeans
  b += al(n * 8) + al(8);                     // low-degree row list + count
  b += al(sparse_mask_bytes(n, d));           // block-sparsity mask (sparse.cu)
  b += al(prune_bytes(n, dp));                // provably-zero block pairs (prune.cu)
  b += al(locality_bytes(n, d));              // locality order (locality.cu)
  return b;
}

int carve(void* base, int64_t bytes, int64_t n, int32_t d, int32_t k, int64_t rows,
          int32_t max_iter, Workspace* ws) {
  if (base == nullptr) return fail(GPIC_E_INVALID, "workspace is null");
  if ((reinterpret_cast<uintptr_t>(base) & 255) != 0)
    return fail(GPIC_E_INVALID, "workspace must be 256-byte aligned");
  const int64_t need = workspace_bytes(n, d, k, rows, max_iter);
  if (bytes < need) return fail(GPIC_E_INVALID, "workspace too small");
  const int64_t dp = feature_pitch(d), npad = row_pad(n);
  const int64_t rows_pad = round_up(rows, kTileM);
  const int64_t n_ctiles = ceil_div(n, kTileN);
  uint8_t* p = static_cast<uint8_t*>(base);
  auto take = [&](int64_t sz) { uint8_t* q = p; p += al(sz); return q; };
  ws->ctl = reinterpret_cast<gpic_ctl*>(take(sizeof(gpic_ctl)));
  ws->xhi = reinterpret_cast<float*>(take(operand_floats(n, d) * 4));
  ws->xlo = reinterpret_cast<float*>(take(npad * dp * 4));
  ws->sqn = reinterpret_cast<float*>(take(npad * 4));
  ws->colpart = reinterpret_cast<double*>(take(ceil_div(n, 256) * d * 8));
  ws->mean = reinterpret_cast<double*>(take((int64_t)(d + 2) * 8));
  ws->rowpart = reinterpret_cast<float*>(take(n_ctiles * rows_pad * 4));
  ws->redpart = reinterpret_cast<double*>(
      take((ceil_div(n, kRedBlock) + 1) * 8 + ceil_div(n, kRedBlock) * 4));
  ws->y = reinterpret_cast<double*>(take(n * 8));
  ws->deg = reinterpret_cast<double*>(take(n * 8));
  ws->v64 = reinterpret_cast<double*>(take(2 * n * 8));
  ws->v32 = reinterpret_cast<float*>(take(vector_pitch(n) * 4));
  ws->kscratch_bytes = kmeans_scratch_bytes(n, k);
  ws->kscratch = reinterpret_cast<double*>(take(ws->kscratch_bytes));
  ws->lowlist = reinterpret_cast<int64_t*>(take(n * 8));
  ws->lowcount = reinterpret_cast<unsigned long long*>(take(8));
  ws->sparse = take(sparse_mask_bytes(n, d));
  ws->prune = take(prune_bytes(n, dp));
  ws->locality = take(locality_bytes(n, d));
  ws->end = p;
  return GPIC_OK;
}

static int status_text(const gpic_ctl& h, int32_t d, char* buf, size_t cap);

static int status_from_ctl(const gpic_ctl& h, int32_t d) {
  char buf[256];
  const int rc = status_text(h, d, buf, sizeof buf);
  if (rc != GPIC_OK) {
    g_detail.status = rc;
    g_detail.index = h.err_index;
    g_detail.index2 = -1;
    g_detail.value = h.err_value;
    if (rc == GPIC_E_NONFINITE) {
      g_detail.index = h.err_index / (d > 0 ? d : 1);
      g_detail.index2 = h.err_index % (d > 0 ? d : 1);
    }
  }
  return rc;
}

static int status_text(const gpic_ctl& h, int32_t d, char* buf, size_t cap) {
  switch (h.status) {
    case GPIC_OK:
      return GPIC_OK;
    case GPIC_E_ZERO_DEGREE:
      snprintf(buf, cap, "row %lld has zero degree", (long long)h.err_index);
      return fail(h.status, buf);
    case GPIC_E_NONFINITE:
      snprintf(buf, cap, "non-finite value at row %lld column %lld",
               (long long)(h.err_index / (d > 0 ? d : 1)), (long long)(h.err_index % (d > 0 ? d : 1)));
      return fail(h.status, buf);
    case GPIC_E_NONPOS_TAU:
      snprintf(buf, cap, "non-positive normaliser %g", h.err_value);
      return fail(h.status, buf);
    case GPIC_E_ZERO_VECTOR:
      snprintf(buf, cap, "point %lld has zero norm", (long long)h.err_index);
      return fail(h.status, buf);
    case GPIC_E_UNSUPPORTED:
      return fail(h.status, "k-means produced non-contiguous clusters (gap repair not on device)");
    default:
      snprintf(buf, cap, "device status %d", h.status);
      return fail(h.status, buf);
  }
}

}  // namespace gpic

using namespace gpic;

extern "C" {

const char* gpic_version(void) { return "gpic 0.1.0 sm_100a"; }
const char* gpic_last_error(void) { return g_err.c_str(); }
int gpic_last_detail(int64_t* index, int64_t* index2, double* value) {
  if (index) *index = g_detail.index;
  if (index2) *index2 = g_detail.index2;
  if (value) *value = g_detail.value;
  return g_detail.status;
}
int gpic_malloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return fail(GPIC_E_INVALID, "gpic_malloc needs an output pointer");
  GPIC_CUDA_TRY(cudaMalloc(out, (size_t)(bytes > 0 ? bytes : 1)));
  return GPIC_OK;
}
int gpic_free(void* p) {
  GPIC_CUDA_TRY(cudaFree(p));
  return GPIC_OK;
}
int64_t gpic_launch_count(void) { return (int64_t)g_launches; }

int64_t gpic_workspace_bytes(int64_t n, int32_t d, int32_t k, int64_t rows, int32_t max_iter) {
  if (n < 1 || d < 1 || rows < 0 || rows > n) return -1;
  return workspace_bytes(n, d, k, rows, max_iter);
}
int64_t gpic_affinity_pitch(int64_t n) { return affinity_pitch(n); }
int32_t gpic_feature_pitch(int32_t d) { return feature_pitch(d); }
int64_t gpic_row_pad(int64_t n) { return row_pad(n); }
int64_t gpic_operand_floats(int64_t n, int32_t d) { return n < 1 || d < 1 ? -1 : operand_floats(n, d); }

int gpic_ctl_read(const gpic_ctl* d_ctl, gpic_ctl* h_out, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  GPIC_CUDA_TRY(cudaMemcpyAsync(h_out, d_ctl, sizeof(gpic_ctl), cudaMemcpyDeviceToHost, s));
  GPIC_CUDA_TRY(cudaStreamSynchronize(s));
  return GPIC_OK;
}

int gpic_ctl_init(gpic_ctl* d_ctl, double eps, int32_t max_iter, void* stream) {
  launch_ctl_init(d_ctl, eps, max_iter, static_cast<cudaStream_t>(stream));
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int gpic_prepare_points(const double* d_x, int64_t n, int32_t d, int32_t kind, float* d_xhi,
                        float* d_xlo, float* d_sqn, void* d_work, gpic_ctl* d_ctl, void* stream) {
  if (n < 1 || d < 1) return fail(GPIC_E_EMPTY, "dataset must contain at least one point and one feature");
  if (kind != GPIC_KIND_RBF && kind != GPIC_KIND_COSINE) return fail(GPIC_E_INVALID, "unknown kind");
  // d_work: colpart (ceil(n/256) * d doubles) followed by mean (d + 2 doubles)
  double* colpart = static_cast<double*>(d_work);
  double* mean = colpart + ceil_div(n, 256) * d;
  launch_prepare(d_x, n, d, d_xhi, d_xlo, d_sqn, colpart, mean, d_ctl,
                 static_cast<cudaStream_t>(stream), kind);
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

// Engine routing, applied the same way by the workspace query, the cluster
// entry points and the stage-wise affinity calls:
//  * the tcgen05 engine keeps a row block's operands resident in shared
//    memory: d <= 192 with stored A, d <= 256 matrix-free (tc_supports_pitch);
//    wider stored-A runs go to the SIMT engine with dense rows (any d);
//  * RBF with d <= kSimtDiffMaxD stored-A runs on the SIMT engine, which
//    forms |x_i - x_j|^2 from coordinate differences: the Gram form's
//    cancellation error (~2^-22 |x|^2 / 2 sigma^2 relative in A) exceeds the
//    1e-4 embedding gate when the spread is large against sigma, which is
//    typical at low d (sigma = sqrt(d)/2); there the tensor Gram also runs
//    at <= 8/64 of its K width, so the difference form costs nothing.
//  * matrix-free stays on tcgen05 (an error beyond d = 256).
//  * RBF whose spread is large against sigma also runs the SIMT difference
//    form: the Gram form's error is ~2^-24 R^2 / (2 sigma^2) relative per
//    entry (measured embedding error: 2.8e-6 at config 3, R^2/2s^2 = 64;
//    4e-7 at config 2, 121), so above R^2/2s^2 = 167.8 (1e-5, a tenth of the
//    gate) the tensor engine is not used for stored A. Matrix-free and fp16
//    tiles exist on the tensor engine only and keep it.
constexpr int32_t kSimtDiffMaxD = 8;
constexpr double kTcMaxSpread = 167.77216;  // 2^24 x 1e-5
static void effective_engine(int kind, int32_t d, int32_t* impl, int32_t* storage,
                             double spread2 = 0.0, double sigma = 1.0) {
  if (storage && *storage == GPIC_STORAGE_NONE) return;
  if (!tc_supports_pitch(feature_pitch(d), false)) {
    if (*impl == GPIC_AFFINITY_TC) *impl = GPIC_AFFINITY_SIMT;
    if (storage && (*storage == GPIC_STORAGE_PACKED || *storage == GPIC_STORAGE_PACKED16))
      *storage = GPIC_STORAGE_DENSE;
    return;
  }
  if (kind == GPIC_KIND_RBF && *impl == GPIC_AFFINITY_TC &&
      (d <= kSimtDiffMaxD || spread2 / (2.0 * sigma * sigma) > kTcMaxSpread)) {
    // the SIMT difference form; it stores fp32, so requested fp16 tiles
    // become fp32 packed tiles (their workspace is sized for that)
    *impl = GPIC_AFFINITY_SIMT;
    if (storage && *storage == GPIC_STORAGE_PACKED16) *storage = GPIC_STORAGE_PACKED;
  }
}

static int affinity_rows(int kind, const float* d_xhi, const float* d_xlo, const float* d_sqn,
                         int64_t n, int32_t d, int64_t row_lo, int64_t row_hi, double sigma,
                         int32_t impl, float* d_a, int64_t lda, double* d_deg, void* d_work,
                         gpic_ctl* d_ctl, void* stream);

int32_t gpic_engine_for(int32_t kind, int32_t d, double sigma, double spread2, int32_t impl,
                        int32_t storage) {
  if (kind == GPIC_KIND_COSINE) sigma = 1.0;
  effective_engine(kind, d, &impl, &storage, spread2, sigma);
  return impl;
}

int gpic_affinity_rbf(const float* d_xhi, const float* d_xlo, const float* d_sqn, int64_t n,
                      int32_t d, int64_t row_lo, int64_t row_hi, double sigma, int32_t impl,
                      float* d_a, int64_t lda, double* d_deg, void* d_work, gpic_ctl* d_ctl,
                      void* stream) {
  if (!(sigma > 0)) return fail(GPIC_E_INVALID, "sigma must be positive");
  return affinity_rows(GPIC_KIND_RBF, d_xhi, d_xlo, d_sqn, n, d, row_lo, row_hi, sigma, impl,
                       d_a, lda, d_deg, d_work, d_ctl, stream);
}

int gpic_affinity_cosine(const float* d_xhi, const float* d_xlo, const float* d_sqn, int64_t n,
                         int32_t d, int64_t row_lo, int64_t row_hi, int32_t impl, float* d_a,
                         int64_t lda, double* d_deg, void* d_work, gpic_ctl* d_ctl, void* stream) {
  return affinity_rows(GPIC_KIND_COSINE, d_xhi, d_xlo, d_sqn, n, d, row_lo, row_hi, 1.0, impl,
                       d_a, lda, d_deg, d_work, d_ctl, stream);
}

static int affinity_rows(int kind, const float* d_xhi, const float* d_xlo, const float* d_sqn,
                         int64_t n, int32_t d, int64_t row_lo, int64_t row_hi, double sigma,
                         int32_t impl, float* d_a, int64_t lda, double* d_deg, void* d_work,
                         gpic_ctl* d_ctl, void* stream) {
  if (row_lo < 0 || row_hi > n || row_lo >= row_hi) return fail(GPIC_E_INVALID, "bad row range");
  if (lda < affinity_pitch(n) || lda % 32) return fail(GPIC_E_INVALID, "lda must be >= pitch(n) and a multiple of 32");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t rows = row_hi - row_lo;
  const int64_t rows_pad = round_up(rows, kTileM);
  const int32_t dp = feature_pitch(d);
  const float neg_scale_log2 = (float)(-1.4426950408889634 / (2.0 * sigma * sigma));
  float* rowpart = static_cast<float*>(d_work);  // n_ctiles x rows_pad
  effective_engine(kind, d, &impl, nullptr);
  if (impl == GPIC_AFFINITY_TC) {
    int rc = launch_affinity_tc(d_xhi, d_xlo, d_sqn, n, dp, row_lo, row_hi, neg_scale_log2, d_a,
                                lda, rowpart, rows_pad, s, kind);
    if (rc != GPIC_OK) return rc;
  } else if (impl == GPIC_AFFINITY_SIMT) {
    launch_affinity_simt(d_xhi, d_xlo, d_sqn, n, d, dp, row_lo, row_hi, neg_scale_log2, d_a, lda,
                         rowpart, rows_pad, s, kind);
  } else {
    return fail(GPIC_E_INVALID, "unknown affinity engine");
  }
  launch_degree(rowpart, rows, rows_pad, ceil_div(n, kTileN), row_lo, d_deg, d_ctl, s);
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int gpic_initial_vector(const double* d_deg, int64_t n, double* d_v64, float* d_v32,
                        void* d_work, gpic_ctl* d_ctl, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(d_work);
  double* tau = part + ceil_div(n, kRedBlock);
  launch_tree_sum(d_deg, n, part, tau, d_ctl, s);
  launch_scale_vector(d_deg, n, tau, d_v64, d_v32, vector_pitch(n), s);
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int gpic_power_iterate(const float* d_a, int64_t lda, const double* d_deg, int64_t n,
                       double* d_v64, float* d_v32, double eps, int32_t max_iter,
                       double* d_delta_hist, double* d_v64_out, void* d_work, gpic_ctl* d_ctl,
                       void* stream) {
  if (max_iter < 1) return fail(GPIC_E_INVALID, "max_iterations must be at least 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // d_work: y (n doubles) then the reduction partials
  double* y = static_cast<double*>(d_work);
  double* part = y + n;
  int rc = run_power_loop(d_a, lda, d_deg, n, y, part, d_v64, d_v32, d_delta_hist, d_ctl,
                          max_iter, s);
  if (rc != GPIC_OK) return rc;
  note_loop_iterations(1);  // asynchronous: at least one iteration ran
  launch_copy_result(d_v64, n, d_v64_out, d_ctl, s);
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int gpic_kmeans1d(const double* d_v, int64_t n, int32_t k, int64_t first_index,
                  const double* h_uniforms, int32_t max_rounds, double tol, int64_t* d_labels,
                  void* d_work, gpic_ctl* d_ctl, void* stream) {
  return launch_kmeans1d(d_v, n, k, first_index, h_uniforms, max_rounds, tol, d_labels, d_work,
                         d_ctl, static_cast<cudaStream_t>(stream));
}

int gpic_reduce_sum(const double* d_v, int64_t n, double* d_out, void* d_work, void* stream) {
  if (n < 1) return fail(GPIC_E_EMPTY, "cannot reduce an empty vector");
  // d_work: a gpic_ctl followed by the partials
  gpic_ctl* ctl = static_cast<gpic_ctl*>(d_work);
  double* part = reinterpret_cast<double*>(static_cast<uint8_t*>(d_work) + sizeof(gpic_ctl));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  launch_ctl_init(ctl, 0.0, 1, s);
  launch_tree_sum(d_v, n, part, d_out, ctl, s);
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int gpic_scale(const double* d_src, int64_t n, double tau, double* d_dst, float* d_dst32,
               int64_t f32_len, void* stream) {
  if (!(tau > 0.0)) return fail(GPIC_E_NONPOS_TAU, "normalisation constant must be positive");
  launch_scale_by(d_src, n, tau, d_dst, d_dst32, f32_len, static_cast<cudaStream_t>(stream));
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int64_t gpic_kmeans_scratch_bytes(int64_t n, int32_t k) { return kmeans_scratch_bytes(n, k); }

int gpic_sym_matvec16(const void* d_tiles, int64_t n, const float* d_v, float* d_rowp,
                      float* d_colp, const double* d_row_scale, double* d_y, void* stream) {
  if (n < 1) return fail(GPIC_E_EMPTY, "empty matrix");
  PeerTable pt;
  std::memset(&pt, 0, sizeof pt);
  pt.y[0][0] = pt.y[0][1] = d_y;
  pt.nranks = 1;
  launch_sym_gemv16(d_tiles, n, d_v, d_rowp, d_colp, d_row_scale, pt, nullptr,
                    static_cast<cudaStream_t>(stream));
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int gpic_sym_matvec(const float* d_tiles, int64_t n, const float* d_v, float* d_rowp,
                    float* d_colp, const double* d_row_scale, double* d_y, void* stream) {
  if (n < 1) return fail(GPIC_E_EMPTY, "empty matrix");
  PeerTable pt;
  std::memset(&pt, 0, sizeof pt);
  pt.y[0][0] = pt.y[0][1] = d_y;
  pt.nranks = 1;
  launch_sym_gemv(d_tiles, n, d_v, d_rowp, d_colp, d_row_scale, pt, nullptr,
                  static_cast<cudaStream_t>(stream));
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int gpic_sym_matvec_sparse(const void* d_tiles, int32_t half, int64_t n, const float* d_v,
                           float* d_rowp, float* d_colp, const double* d_row_scale, double* d_y,
                           const uint8_t* d_boxnz, const int64_t* d_sb_prefix, void* stream) {
  if (n < 1) return fail(GPIC_E_EMPTY, "empty matrix");
  PeerTable pt;
  std::memset(&pt, 0, sizeof pt);
  pt.y[0][0] = pt.y[0][1] = d_y;
  pt.nranks = 1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (half)
    launch_sym_gemv16(d_tiles, n, d_v, d_rowp, d_colp, d_row_scale, pt, nullptr, s, d_boxnz,
                      d_sb_prefix);
  else
    launch_sym_gemv(static_cast<const float*>(d_tiles), n, d_v, d_rowp, d_colp, d_row_scale, pt,
                    nullptr, s, ShardRange(), d_boxnz, d_sb_prefix);
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int64_t gpic_vector_pitch(int64_t n) { return vector_pitch(n); }

int64_t gpic_mf_ypart_doubles(int64_t n, int32_t d, int64_t rows) {
  if (n < 1 || d < 1 || rows < 1) return -1;
  return mf_ypart_doubles(n, feature_pitch(d), rows);
}

int gpic_mf_degrees(const float* d_xhi, const float* d_xlo, const float* d_sqn, int64_t n,
                    int32_t d, int64_t row_lo, int64_t row_hi, double sigma, int32_t kind,
                    float* d_ones, double* d_ypart, double* d_deg, void* stream) {
  if (kind == GPIC_KIND_RBF && !(sigma > 0)) return fail(GPIC_E_INVALID, "sigma must be positive");
  if (row_lo < 0 || row_hi > n || row_lo >= row_hi) return fail(GPIC_E_INVALID, "bad row range");
  MfOperands op{d_xhi, d_xlo, d_sqn, n, feature_pitch(d),
                (float)(-1.4426950408889634 / (2.0 * sigma * sigma)), kind};
  op.sym = mf_sym_default();
  op.d = d;
  return launch_mf_degrees(op, row_lo, row_hi - row_lo, d_ones, d_ypart, d_deg,
                           static_cast<cudaStream_t>(stream));
}

// One matrix-free A v pass (y = A v, no 1/deg) over the operands, pruning
// mask and partial buffers a gpic_cluster(storage = NONE) run left in its
// workspace: the loop's own pass, for kernel-level timing.
int gpic_cluster_mf_pass(void* d_work, int64_t n, int32_t d, int32_t k, int32_t max_iter,
                         double sigma, int32_t kind, int32_t pruned, const float* d_v32,
                         double* d_y, void* stream) {
  if (n < 1 || d < 1) return fail(GPIC_E_INVALID, "bad shape");
  Workspace ws;
  const int64_t scratch = workspace_bytes(n, d, k, n, max_iter);
  int rc = carve(d_work, scratch, n, d, k, n, max_iter, &ws);
  if (rc) return rc;
  const int32_t dp = feature_pitch(d);
  MfOperands op{ws.xhi, ws.xlo, ws.sqn, n, dp,
                (float)(-1.4426950408889634 / (2.0 * sigma * sigma)), kind};
  op.sym = mf_sym_default();
  op.d = d;
  if (pruned) {
    op.prune = carve_prune(ws.prune, n, dp);
    op.pruned = 1;
  }
  PeerTable pt;
  std::memset(&pt, 0, sizeof pt);
  pt.y[0][0] = pt.y[0][1] = d_y;
  pt.nranks = 1;
  double* ypart = reinterpret_cast<double*>(static_cast<uint8_t*>(d_work) + scratch);
  return launch_mf_matvec(op, 0, n, d_v32, ypart, nullptr, pt, nullptr,
                          static_cast<cudaStream_t>(stream));
}

// The locality permutation of the last gpic_cluster run on this workspace
// (locality.cu): *reordered = 1 and perm[p] = original index of position p,
// or *reordered = 0 (the input order was kept). Synchronizes `stream`.
int gpic_cluster_permutation(const void* d_work, int64_t n, int32_t d, int32_t k, int32_t max_iter,
                             int32_t* d_perm, int32_t* reordered, void* stream) {
  if (n < 1 || d < 1 || !reordered) return fail(GPIC_E_INVALID, "bad query");
  Workspace ws;
  int rc = carve(const_cast<void*>(d_work), workspace_bytes(n, d, k, n, max_iter), n, d, k, n,
                 max_iter, &ws);
  if (rc) return rc;
  const Locality loc = carve_locality(ws.locality, n, d);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double flag = 0.0;
  GPIC_CUDA_TRY(cudaMemcpyAsync(&flag, loc.metric + 2, 8, cudaMemcpyDeviceToHost, s));
  GPIC_CUDA_TRY(cudaStreamSynchronize(s));
  *reordered = flag == 1.0;
  if (*reordered && d_perm)
    GPIC_CUDA_TRY(cudaMemcpyAsync(d_perm, loc.perm, n * 4, cudaMemcpyDeviceToDevice, s));
  GPIC_CUDA_TRY(cudaStreamSynchronize(s));
  return GPIC_OK;
}

// Work the tensor engine did in a gpic_cluster run after tile pruning:
// packed storages -> kept / all work units (128 MB x 128 tiles); matrix-free
// -> kept / all tile units of one sym pass. Synchronizes `stream`.
int gpic_cluster_pruned_work(const void* d_work, int64_t n, int32_t d, int32_t k,
                             int32_t max_iter, int32_t storage, int64_t* kept, int64_t* total,
                             void* stream) {
  if (n < 1 || d < 1 || !kept || !total) return fail(GPIC_E_INVALID, "bad query");
  Workspace ws;
  const int64_t scratch = workspace_bytes(n, d, k, n, max_iter);
  int rc = carve(const_cast<void*>(d_work), scratch, n, d, k, n, max_iter, &ws);
  if (rc) return rc;
  const int32_t dp = feature_pitch(d);
  const PruneMask pm = carve_prune(ws.prune, n, dp);
  const int64_t mb = storage == GPIC_STORAGE_NONE ? tc_mblocks_mf(dp) : tc_mblocks(dp);
  const int64_t nrt = ceil_div(n, 128 * mb), nct = ceil_div(n, 128);
  *total = nrt * nct - mb * nrt * (nrt - 1) / 2;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (storage == GPIC_STORAGE_NONE) {
    int64_t cnt = 0;
    GPIC_CUDA_TRY(cudaMemcpyAsync(&cnt, pm.item_count, 8, cudaMemcpyDeviceToHost, s));
    GPIC_CUDA_TRY(cudaStreamSynchronize(s));
    int64_t w = 0;
    GPIC_CUDA_TRY(cudaMemcpyAsync(&w, pm.item_wpre + cnt, 8, cudaMemcpyDeviceToHost, s));
    GPIC_CUDA_TRY(cudaStreamSynchronize(s));
    *kept = (w - cnt * prune_item_weight()) / 4;  // the weights count quarter tiles
  } else {
    GPIC_CUDA_TRY(cudaMemcpyAsync(kept, pm.count, 8, cudaMemcpyDeviceToHost, s));
  }
  GPIC_CUDA_TRY(cudaStreamSynchronize(s));
  return GPIC_OK;
}

int64_t gpic_mf_shard_scratch_bytes(int64_t n, int32_t d) { return mf_shard_scratch_bytes(n, d); }

int gpic_mf_shard_build(const float* d_xhi, const float* d_xlo, const float* d_sqn,
                        const double* d_prep_work, int64_t n, int32_t d, double sigma,
                        int32_t nranks, int32_t rank, double* d_deg_partial, void* d_scratch,
                        void* stream) {
  if (n < 1 || d < 1 || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(GPIC_E_INVALID, "bad matrix-free shard parameters");
  if (!(sigma > 0)) return fail(GPIC_E_INVALID, "sigma must be positive");
  const int32_t dp = feature_pitch(d);
  if (d <= 8 || !tc_supports_pitch(dp, true) || !mf_sym_default() || !sparse_enabled() ||
      !prune_enabled())
    return fail(GPIC_E_UNSUPPORTED, "matrix-free item shards need the pruned tcgen05 sym pass");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* ypart = static_cast<double*>(d_scratch);
  MfOperands op{d_xhi, d_xlo, d_sqn, n, dp, (float)(-1.4426950408889634 / (2.0 * sigma * sigma)),
                GPIC_KIND_RBF};
  op.d = d;
  op.sym = 1;
  op.pruned = 1;
  op.prune = mf_shard_prune(ypart, n, d);
  op.share_r = rank;
  op.share_n = nranks;
  const double* colpart = d_prep_work;  // gpic_prepare_points: column sums, then the mean
  const double* mean = d_prep_work + ceil_div(n, 256) * d;
  launch_prune(op.prune, d_xlo, colpart, mean, n, d, dp, sigma, -tc_mblocks_mf(dp), 0, s);
  float* ones = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ypart) +
                                         round_up(mf_ypart_doubles(n, dp, n) * 8, 256) +
                                         round_up(prune_bytes(n, dp), 256));
  return launch_mf_degrees(op, 0, n, ones, ypart, d_deg_partial, s);
}

int gpic_matvec(const float* d_a, int64_t lda, int64_t rows, int64_t n, const float* d_v,
                const double* d_row_scale, double* d_y, void* stream) {
  if (lda % 4 || lda < n) return fail(GPIC_E_INVALID, "lda must be >= n and a multiple of 4");
  PeerTable pt;
  std::memset(&pt, 0, sizeof pt);
  pt.y[0][0] = pt.y[0][1] = d_y;
  pt.nranks = 1;
  launch_gemv(d_a, lda, rows, 0, d_v, d_row_scale, pt, nullptr, static_cast<cudaStream_t>(stream));
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int gpic_generate_blobs(const double* d_centers, const int64_t* d_offsets, int64_t n, int32_t d,
                        int32_t k, uint64_t seed, double noise, double offset, double* d_x,
                        int64_t* d_labels, void* stream) {
  if (n < 1 || d < 1 || k < 1 || k > n) return fail(GPIC_E_INVALID, "need n >= k >= 1, d >= 1");
  if (!(noise >= 0.0)) return fail(GPIC_E_INVALID, "noise must be >= 0");
  return launch_generate_blobs(d_centers, d_offsets, n, d, k, seed, noise, offset, d_x, d_labels,
                               static_cast<cudaStream_t>(stream));
}

int gpic_row_stats(const double* d_w, int64_t rows, int64_t n, int64_t ldw, double* d_sum,
                   double* d_min, double* d_max, void* stream) {
  if (rows < 1 || n < 1) return fail(GPIC_E_EMPTY, "empty matrix");
  if (ldw < n) return fail(GPIC_E_INVALID, "ldw must be >= n");
  launch_row_stats(d_w, rows, n, ldw, d_sum, d_min, d_max, static_cast<cudaStream_t>(stream));
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int64_t gpic_packed_tiles(int64_t n) { return n < 1 ? -1 : packed_tiles(n); }
int64_t gpic_sym_partial_floats(int64_t n) { return n < 1 ? -1 : sym_partial_floats(n); }

// ---- packed shards (multi-rank symmetric storage) ----------------------
// Rank r of P owns super-rows (512 rows) [P_r, P_r+1), balanced by stored
// tile count; its tiles are the contiguous packed range of those rows.
static int64_t super_rows(int64_t n) { return ceil_div(ceil_div(n, kTileN), 4); }
static int64_t tiles_before_row(int64_t n, int64_t tile_row) {
  const int64_t nt = ceil_div(n, kTileN);
  const int64_t I = tile_row < nt ? tile_row : nt;
  return I * nt - I * (I - 1) / 2;
}

int gpic_packed_shard_range(int64_t n, int32_t nranks, int32_t rank, int64_t* row_lo,
                            int64_t* row_hi) {
  if (n < 1 || nranks < 1 || rank < 0 || rank >= nranks || !row_lo || !row_hi)
    return fail(GPIC_E_INVALID, "bad packed shard parameters");
  const int64_t ns = super_rows(n);
  if (ns < nranks) return fail(GPIC_E_INVALID, "too few 512-row super-rows for the rank count");
  const int64_t total = tiles_before_row(n, 4 * ns);
  auto cut = [&](int64_t r) {  // first super-row whose tile prefix reaches r / P of the total
    if (r <= 0) return (int64_t)0;
    if (r >= nranks) return ns;
    const int64_t want = total * r / nranks;
    int64_t lo = 0, hi = ns;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (tiles_before_row(n, 4 * mid) >= want) hi = mid; else lo = mid + 1;
    }
    // every rank keeps at least one super-row
    if (lo < r) lo = r;
    if (lo > ns - (nranks - r)) lo = ns - (nranks - r);
    return lo;
  };
  const int64_t p0 = cut(rank), p1 = cut(rank + 1);
  *row_lo = 512 * p0;
  *row_hi = 512 * p1 < n ? 512 * p1 : n;
  return GPIC_OK;
}

int64_t gpic_prune_scratch_bytes(int64_t n, int32_t d) {
  if (n < 1 || d < 1) return -1;
  return prune_bytes(n, feature_pitch(d));
}

int gpic_packed_shard_ranges_pruned(const float* d_xlo, const double* d_prep_work, int64_t n,
                                    int32_t d, double sigma, int32_t nranks, void* d_scratch,
                                    int64_t* bounds, void* stream) {
  if (n < 1 || d < 1 || nranks < 1 || !d_xlo || !d_prep_work || !d_scratch || !bounds)
    return fail(GPIC_E_INVALID, "bad packed shard parameters");
  if (!(sigma > 0)) return fail(GPIC_E_INVALID, "sigma must be positive");
  const int64_t ns = super_rows(n);
  if (ns < nranks) return fail(GPIC_E_INVALID, "too few 512-row super-rows for the rank count");
  const int32_t dp = feature_pitch(d);
  const int mb = tc_mblocks(dp);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // the whole matrix's pruning mask: kept tensor units per row block
  const PruneMask pm = carve_prune(d_scratch, n, dp);
  launch_prune(pm, d_xlo, d_prep_work, d_prep_work + ceil_div(n, 256) * d, n, d, dp, sigma, mb, 0,
               s);
  const int64_t nrt = ceil_div(n, 128 * mb);
  std::vector<int32_t> cnt(nrt);
  GPIC_CUDA_TRY(cudaMemcpyAsync(cnt.data(), pm.rbcount, nrt * 4, cudaMemcpyDeviceToHost, s));
  GPIC_CUDA_TRY(cudaStreamSynchronize(s));
  // super-row weights: its row blocks' kept units (+1: a super-row is never free)
  std::vector<int64_t> pre(ns + 1, 0);
  for (int64_t q = 0; q < ns; ++q) {
    int64_t w = 1;
    for (int64_t rb = q * 512 / (128 * mb); rb < (q + 1) * 512 / (128 * mb) && rb < nrt; ++rb)
      w += cnt[rb];
    pre[q + 1] = pre[q] + w;
  }
  bounds[0] = 0;
  for (int32_t r = 1; r < nranks; ++r) {
    const int64_t want = pre[ns] * r / nranks;
    int64_t q = std::lower_bound(pre.begin(), pre.end(), want) - pre.begin();
    const int64_t prev = bounds[r - 1] / 512;
    if (q < prev + 1) q = prev + 1;                  // every rank keeps a super-row
    if (q > ns - (nranks - r)) q = ns - (nranks - r);
    bounds[r] = 512 * q;
  }
  bounds[nranks] = n;
  return GPIC_OK;
}

int64_t gpic_packed_shard_tiles(int64_t n, int64_t row_lo, int64_t row_hi) {
  if (n < 1 || row_lo % 512 || row_hi <= row_lo) return -1;
  return tiles_before_row(n, ceil_div(row_hi, kTileN)) - tiles_before_row(n, row_lo / kTileN);
}

// scratch: [GEMV row records][GEMV column records][degree row partials]
// [degree column partials (4 quadrants)], each 256-byte aligned
static int64_t shard_records(int64_t n, int64_t row_lo, int64_t row_hi) {
  const int64_t ns = super_rows(n);
  const int64_t p0 = row_lo / 512, p1 = ceil_div(row_hi, 512);
  const int64_t a = p0 * ns - p0 * (p0 - 1) / 2, b = p1 * ns - p1 * (p1 - 1) / 2;
  return (b - a) * 4 * 128;
}
// [records][records][degree partials][degree partials][block sparsity of the
// whole triangle (sparse.cu; flags of other shards' tiles stay 0)][pruning
// mask (prune.cu), sized for the widest pitch]
int64_t gpic_packed_shard_scratch_bytes(int64_t n, int64_t row_lo, int64_t row_hi) {
  const int64_t t = gpic_packed_shard_tiles(n, row_lo, row_hi);
  if (t < 0) return -1;
  const int64_t r = shard_records(n, row_lo, row_hi);
  return 2 * al(r * 4) + al(t * 128 * 4) + al(t * 4 * 128 * 4) + al(sparse_mask_bytes(n, 256)) +
         al(prune_bytes(n, 256));
}

// the shard scratch's block-sparsity and pruning regions
static void shard_sparse(void* d_scratch, int64_t n, int64_t row_lo, int64_t row_hi, int32_t d,
                         SparseMask* sm, PruneMask* pm) {
  const int64_t t = gpic_packed_shard_tiles(n, row_lo, row_hi);
  const int64_t r = shard_records(n, row_lo, row_hi);
  uint8_t* p = static_cast<uint8_t*>(d_scratch) + 2 * al(r * 4) + al(t * 128 * 4) +
               al(t * 4 * 128 * 4);
  *sm = carve_sparse(p, n, d);
  *pm = carve_prune(p + al(sparse_mask_bytes(n, 256)), n, feature_pitch(d));
}

}  // extern "C"
namespace gpic {
SparseMask packed_shard_sparse(void* d_scratch, int64_t n, int64_t row_lo, int64_t row_hi,
                               int32_t d) {
  SparseMask sm;
  PruneMask pm;
  shard_sparse(d_scratch, n, row_lo, row_hi, d, &sm, &pm);
  return sm;
}
}  // namespace gpic
extern "C" {

int gpic_packed_shard_build(const float* d_xhi, const float* d_xlo, const float* d_sqn, int64_t n,
                            int32_t d, int64_t row_lo, int64_t row_hi, double sigma, int32_t kind,
                            float* d_tiles, double* d_deg_partial, void* d_scratch,
                            const double* d_prep_work, void* stream) {
  if (kind == GPIC_KIND_RBF && !(sigma > 0)) return fail(GPIC_E_INVALID, "sigma must be positive");
  if (kind == GPIC_KIND_COSINE) sigma = 1.0;
  const int64_t t = gpic_packed_shard_tiles(n, row_lo, row_hi);
  if (t < 0) return fail(GPIC_E_INVALID, "bad packed shard row range");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int32_t dp = feature_pitch(d);
  const int64_t r = shard_records(n, row_lo, row_hi);
  uint8_t* base = static_cast<uint8_t*>(d_scratch) + 2 * al(r * 4);
  float* degrow = reinterpret_cast<float*>(base);
  float* degcol = reinterpret_cast<float*>(base + al(t * 128 * 4));
  const float neg_scale_log2 = (float)(-1.4426950408889634 / (2.0 * sigma * sigma));
  // block sparsity of the shard's tiles (flags in a whole-triangle array) and,
  // with the prepare pass's column sums (RBF), tile pruning of its units
  SparseMask sm;
  PruneMask pm;
  shard_sparse(d_scratch, n, row_lo, row_hi, d, &sm, &pm);
  const bool sparse = sparse_enabled();
  const bool prune = sparse && kind == GPIC_KIND_RBF && prune_enabled() && d_prep_work != nullptr;
  if (sparse) GPIC_CUDA_TRY(cudaMemsetAsync(sm.boxnz, 0, packed_tiles(n) * 16, s));
  if (prune)
    launch_prune(pm, d_xlo, d_prep_work, d_prep_work + ceil_div(n, 256) * d, n, d, dp, sigma,
                 tc_mblocks(dp), row_lo, s, row_hi);
  int rc = launch_affinity_tc_packed(d_xhi, d_xlo, d_sqn, n, dp, neg_scale_log2, d_tiles, degrow,
                                     degcol, s, kind, false, row_lo, row_hi,
                                     sparse ? sm.boxnz : nullptr, prune ? pm.units : nullptr,
                                     prune ? pm.count : nullptr);
  if (rc) return rc;
  if (sparse) launch_sparse_prefix(sm, s);
  GPIC_CUDA_TRY(cudaMemsetAsync(d_deg_partial, 0, n * 8, s));
  ShardRange sr;
  sr.p_lo = row_lo / 512;
  sr.p_hi = ceil_div(row_hi, 512);
  sr.tile_base = tiles_before_row(n, row_lo / kTileN);
  launch_sym_degree(degrow, degcol, n, packed_row_halves(dp), d_deg_partial, nullptr, s, sr,
                    sparse ? sm.boxnz : nullptr, prune ? &pm : nullptr);
  GPIC_CUDA_TRY(cudaGetLastError());
  return GPIC_OK;
}

int gpic_cluster_workspace_layout(int64_t n, int32_t d, int32_t k, int32_t max_iter,
                                  int32_t storage, int64_t* offsets) {
  if (n < 1 || d < 1 || !offsets) return fail(GPIC_E_INVALID, "bad layout query");
  const int64_t scratch = workspace_bytes(n, d, k, n, max_iter);
  Workspace ws;
  uint8_t* base = reinterpret_cast<uint8_t*>(uintptr_t(1) << 20);  // arithmetic only
  int rc = carve(base, scratch, n, d, k, n, max_iter, &ws);
  if (rc) return rc;
  const bool half = storage == GPIC_STORAGE_PACKED16;
  const int64_t tiles = scratch;
  const int64_t rowp = tiles + packed_tiles(n) * 128 * 128 * (half ? 2 : 4);
  const int64_t colp = rowp + al(sym_partial_floats(n) * 4);
  const SparseMask sm = carve_sparse(ws.sparse, n, d);
  offsets[0] = tiles;
  offsets[1] = rowp;
  offsets[2] = colp;
  offsets[3] = reinterpret_cast<uint8_t*>(sm.boxnz) - base;
  offsets[4] = reinterpret_cast<uint8_t*>(sm.sb_prefix) - base;
  offsets[5] = reinterpret_cast<uint8_t*>(ws.deg) - base;
  const PruneMask pm = carve_prune(ws.prune, n, feature_pitch(d));
  offsets[6] = reinterpret_cast<uint8_t*>(pm.count) - base;
  const int64_t mb = tc_mblocks(feature_pitch(d));
  const int64_t nrt = ceil_div(n, 128 * mb), nct = ceil_div(n, 128);
  offsets[7] = nrt * nct - mb * nrt * (nrt - 1) / 2;
  return GPIC_OK;
}

int64_t gpic_cluster_workspace_bytes(int64_t n, int32_t d, int32_t k, int32_t max_iter,
                                     int32_t storage) {
  if (n < 1 || d < 1) return -1;
  int32_t impl = GPIC_AFFINITY_TC;
  effective_engine(GPIC_KIND_RBF, d, &impl, &storage);
  const int64_t scratch = workspace_bytes(n, d, k, n, max_iter);
  if (storage == GPIC_STORAGE_PACKED)  // tiles + GEMV partials (2) + degree partials (<= 2 + 4)
    return scratch + packed_tiles(n) * 128 * 128 * 4 + 8 * al(sym_partial_floats(n) * 4);
  if (storage == GPIC_STORAGE_PACKED16)  // fp32-sized: a large spread demotes to fp32 tiles
    return scratch + packed_tiles(n) * 128 * 128 * 4 + 8 * al(sym_partial_floats(n) * 4);
  if (storage == GPIC_STORAGE_NONE)
    return scratch + al(mf_ypart_doubles(n, feature_pitch(d), n) * 8);
  return scratch + n * affinity_pitch(n) * 4;
}

namespace {
__global__ void fill_ones_kernel(float* v, int64_t n, int64_t len) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < len) v[i] = i < n ? 1.f : 0.f;
}
}  // namespace

}  // extern "C"

namespace {
// Phase boundaries of one cluster() run (report.py:28 PHASES): prepare +
// affinity | degree | (normalize: folded into the GEMV) | start vector +
// power loop | k-means. `ev` is null or 5 recorded events.
inline void mark(cudaEvent_t* ev, int i, cudaStream_t s) {
  if (ev) cudaEventRecord(ev[i], s);
}

int cluster_impl(const double* d_x, int64_t n, int32_t d, double sigma, int32_t kind, int32_t k,
                 double eps, int32_t max_iter, int64_t first_index, const double* h_uniforms,
                 int32_t impl, int32_t storage, const double* d_v0, int64_t* d_labels, double* d_v,
                 double* d_delta_hist, int32_t* h_iters, int32_t* h_converged, void* d_work,
                 int64_t work_bytes, void* stream, cudaEvent_t* ev) {
  if (n < 1 || d < 1) return fail(GPIC_E_EMPTY, "dataset must contain at least one point and one feature");
  if (k > n) return fail(GPIC_E_K_TOO_LARGE, "k exceeds the number of points");
  if (kind != GPIC_KIND_RBF && kind != GPIC_KIND_COSINE) return fail(GPIC_E_INVALID, "unknown kind");
  if (kind == GPIC_KIND_RBF && !(sigma > 0)) return fail(GPIC_E_INVALID, "sigma must be positive");
  if (kind == GPIC_KIND_COSINE) sigma = 1.0;  // unused
  effective_engine(kind, d, &impl, &storage);
  if ((storage == GPIC_STORAGE_NONE || storage == GPIC_STORAGE_PACKED16) &&
      impl != GPIC_AFFINITY_TC)
    return fail(GPIC_E_UNSUPPORTED, "fp16 packed / matrix-free storage runs on the tcgen05 engine");
  if (storage < GPIC_STORAGE_DENSE || storage > GPIC_STORAGE_PACKED16)
    return fail(GPIC_E_INVALID, "unknown storage mode");
  Workspace ws;
  const int64_t scratch = workspace_bytes(n, d, k, n, max_iter);
  const int64_t need = gpic_cluster_workspace_bytes(n, d, k, max_iter, storage);
  if (work_bytes < need) return fail(GPIC_E_INVALID, "workspace too small for the affinity matrix");
  int rc = carve(d_work, scratch, n, d, k, n, max_iter, &ws);
  if (rc) return rc;
  float* a = reinterpret_cast<float*>(static_cast<uint8_t*>(d_work) + scratch);
  double* deg = ws.deg;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  mark(ev, 0, s);
  launch_ctl_init(ws.ctl, eps, max_iter, s);
  launch_prepare(d_x, n, d, ws.xhi, ws.xlo, ws.sqn, ws.colpart, ws.mean, ws.ctl, s, kind);
  const int32_t dp = feature_pitch(d);
  // locality order (locality.cu): randomly ordered inputs are permuted so
  // that block sparsity and tile pruning apply; the metric is read at the
  // engine-routing sync below
  const Locality loc = carve_locality(ws.locality, n, d);
  const bool packed_any = storage == GPIC_STORAGE_PACKED || storage == GPIC_STORAGE_PACKED16;
  // packed storage, or the pruned matrix-free symmetric pass (d > 8)
  const bool prunable = packed_any || (storage == GPIC_STORAGE_NONE && d > 8 && mf_sym_default());
  const bool may_reorder = kind == GPIC_KIND_RBF && impl == GPIC_AFFINITY_TC && prunable &&
                           n >= 16384 && locality_enabled() && sparse_enabled() && prune_enabled();
  if (may_reorder) launch_order_metric(loc, ws.xlo, n, dp, s);
  GPIC_CUDA_TRY(cudaMemsetAsync(loc.metric + 2, 0, 8, s));
  bool reordered = false;
  const double* x_run = d_x;  // the points the run works on (permuted when reordered)
  // packed storage, RBF, tensor engine: the tile pruning of the input order
  // is launched before the host waits for the routing decision below, so
  // the GPU runs it while the host wakes up and decides (kept when the
  // decision is the tensor engine on the input order, the common case;
  // otherwise redone / unused — it only writes the pruning scratch and
  // the box flags, both rewritten before use)
  const bool packed_rbf_tc = packed_any && kind == GPIC_KIND_RBF && impl == GPIC_AFFINITY_TC &&
                             sparse_enabled() && prune_enabled();
  bool pruned_early = false;
  if (kind == GPIC_KIND_RBF && impl == GPIC_AFFINITY_TC &&
      (storage != GPIC_STORAGE_NONE || may_reorder)) {
    // data-driven engine choice: the spread R^2 from the prepare pass
    double spread2 = 0.0, metric[2] = {0.0, 0.0};
    double* probe = routing_probe();
    if (probe != nullptr) {
      GPIC_CUDA_TRY(cudaMemcpyAsync(probe, ws.mean + d + 1, 8, cudaMemcpyDeviceToHost, s));
      if (may_reorder)
        GPIC_CUDA_TRY(cudaMemcpyAsync(probe + 1, loc.metric, 16, cudaMemcpyDeviceToHost, s));
      cudaEvent_t ev;
      GPIC_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      GPIC_CUDA_TRY(cudaEventRecord(ev, s));
      if (packed_rbf_tc) {
        const SparseMask sm0 = carve_sparse(ws.sparse, n, d);
        const PruneMask pm0 = carve_prune(ws.prune, n, dp);
        GPIC_CUDA_TRY(cudaMemsetAsync(sm0.boxnz, 0, packed_tiles(n) * 16, s));
        launch_prune(pm0, ws.xlo, ws.colpart, ws.mean, n, d, dp, sigma, tc_mblocks(dp), 0, s);
        pruned_early = true;
      }
      const cudaError_t e = cudaEventSynchronize(ev);
      cudaEventDestroy(ev);
      GPIC_CUDA_TRY(e);
      spread2 = probe[0];
      if (may_reorder) {
        metric[0] = probe[1];
        metric[1] = probe[2];
      }
    } else {
      GPIC_CUDA_TRY(cudaMemcpyAsync(&spread2, ws.mean + d + 1, 8, cudaMemcpyDeviceToHost, s));
      if (may_reorder)
        GPIC_CUDA_TRY(cudaMemcpyAsync(metric, loc.metric, 16, cudaMemcpyDeviceToHost, s));
      GPIC_CUDA_TRY(cudaStreamSynchronize(s));
    }
    effective_engine(kind, d, &impl, &storage, spread2, sigma);
    if (impl != GPIC_AFFINITY_TC) pruned_early = false;
    // index neighbours about as far apart as random pairs (E|x_i - x_j|^2 =
    // 2 E|x|^2 for centred data): reorder; cluster-ordered data sit near 0
    if (may_reorder && impl == GPIC_AFFINITY_TC &&
        (locality_forced() || metric[0] > 1.0 * metric[1])) {
      int rc2 = launch_locality_order(loc, ws.xlo, d_x, n, d, dp, s);
      if (rc2) return rc2;
      x_run = loc.xp;
      reordered = true;
      pruned_early = false;  // the order changed: prune again below
      static const double one = 1.0;  // recorded for gpic_cluster_permutation
      GPIC_CUDA_TRY(cudaMemcpyAsync(loc.metric + 2, &one, 8, cudaMemcpyHostToDevice, s));
      launch_prepare(x_run, n, d, ws.xhi, ws.xlo, ws.sqn, ws.colpart, ws.mean, ws.ctl, s, kind);
    }
  }
  const float neg_scale_log2 = (float)(-1.4426950408889634 / (2.0 * sigma * sigma));
  const int64_t lda = affinity_pitch(n);
  ShardLoop L;
  std::memset(&L, 0, sizeof L);
  if (storage == GPIC_STORAGE_PACKED || storage == GPIC_STORAGE_PACKED16) {
    const bool half = storage == GPIC_STORAGE_PACKED16;
    float* rowp = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(a) +
                                           packed_tiles(n) * 128 * 128 * (half ? 2 : 4));
    float* colp = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(rowp) + al(sym_partial_floats(n) * 4));
    // degree partials from the affinity epilogue (row sums + column sums of
    // every stored tile, consistent with the stored fp32 values)
    const int64_t pf = al(sym_partial_floats(n) * 4) / 4;
    float* degrow = colp + pf;
    float* degcol = degrow + 2 * pf;
    // block sparsity: the tensor engine does not store 32 x 32 boxes whose
    // values are all exact fp32 zeros and flags the ones it stores; the GEMV
    // reads only those (sparse.cu; bit-identical to the dense run)
    const SparseMask sm = carve_sparse(ws.sparse, n, d);
    const bool sparse = sparse_enabled() && impl == GPIC_AFFINITY_TC;
    // tile pruning (RBF): block pairs proved to hold only flushed entries are
    // not computed at all (prune.cu); their box flags stay 0
    const bool prune = sparse && kind == GPIC_KIND_RBF && prune_enabled();
    const PruneMask pm = carve_prune(ws.prune, n, dp);
    if (prune && !pruned_early) {
      GPIC_CUDA_TRY(cudaMemsetAsync(sm.boxnz, 0, packed_tiles(n) * 16, s));
      launch_prune(pm, ws.xlo, ws.colpart, ws.mean, n, d, dp, sigma, tc_mblocks(dp), 0, s);
    }
    if (impl == GPIC_AFFINITY_SIMT) {
      launch_affinity_simt_packed(ws.xlo, ws.sqn, n, d, dp, neg_scale_log2, a, degrow, degcol, s,
                                  kind);
    } else {
      rc = launch_affinity_tc_packed(ws.xhi, ws.xlo, ws.sqn, n, dp, neg_scale_log2, a, degrow,
                                     degcol, s, kind, half, 0, 0, sparse ? sm.boxnz : nullptr,
                                     prune ? pm.units : nullptr, prune ? pm.count : nullptr);
      if (rc) return rc;
    }
    if (sparse) launch_sparse_prefix(sm, s);
    mark(ev, 1, s);
    launch_sym_degree(degrow, degcol, n, packed_row_halves(dp), deg, nullptr, s, ShardRange(),
                      sparse ? sm.boxnz : nullptr, prune ? &pm : nullptr,
                      sparse ? sm.sb_prefix : nullptr);
    L.mode = half ? kLoopPacked16 : kLoopPacked;
    L.rowp = rowp;
    L.colp = colp;
    L.boxnz = sparse ? sm.boxnz : nullptr;
    L.sb_prefix = sparse ? sm.sb_prefix : nullptr;
  } else if (storage == GPIC_STORAGE_NONE) {
    // matrix-free: A is recomputed from X for the degrees and every iteration
    double* ypart = reinterpret_cast<double*>(a);
    L.mode = kLoopMatrixFree;
    L.mf = MfOperands{ws.xhi, ws.xlo, ws.sqn, n, dp, neg_scale_log2, kind};
    L.mf.d = d;
    L.mf.sym = mf_sym_default();
    // tile pruning of the sym tensor pass (RBF, d > 8): the kept items only
    if (L.mf.sym && kind == GPIC_KIND_RBF && d > 8 && impl == GPIC_AFFINITY_TC &&
        sparse_enabled() && prune_enabled()) {
      L.mf.prune = carve_prune(ws.prune, n, dp);
      launch_prune(L.mf.prune, ws.xlo, ws.colpart, ws.mean, n, d, dp, sigma, -tc_mblocks_mf(dp), 0, s);
      L.mf.pruned = 1;
    }
    L.ypart = ypart;
    mark(ev, 1, s);  // matrix-free: the degree pass is the first A recompute
    rc = launch_mf_degrees(L.mf, 0, n, ws.v32, ypart, deg, s);
    if (rc) return rc;
  } else {
    const int64_t rows_pad = round_up(n, kTileM);
    if (impl == GPIC_AFFINITY_TC) {
      rc = launch_affinity_tc(ws.xhi, ws.xlo, ws.sqn, n, dp, 0, n, neg_scale_log2, a, lda,
                              ws.rowpart, rows_pad, s, kind);
      if (rc) return rc;
    } else {
      launch_affinity_simt(ws.xhi, ws.xlo, ws.sqn, n, d, dp, 0, n, neg_scale_log2, a, lda,
                           ws.rowpart, rows_pad, s, kind);
    }
    mark(ev, 1, s);
    launch_degree(ws.rowpart, n, rows_pad, ceil_div(n, kTileN), 0, deg, nullptr, s);
  }
  // isolated points (H4): rows whose fp32 degree is (nearly) 0 are redone
  // in fp64 from X; ZeroDegree only when the fp64 degree is 0 (lowdeg.cu)
  launch_lowdeg_scan(deg, n, kind, ws.lowlist, ws.lowcount, s);
  LowRows low;
  low.x = x_run;
  low.n = n;
  low.d = d;
  low.kind = kind;
  low.sigma = sigma;
  low.list = ws.lowlist;
  low.d_count = ws.lowcount;
  // the listed rows are handled by kernels striding over the device-side
  // count (no host read here); a failure so far (NonFiniteEntry, ...) has
  // set ctl->stop, so the loop and the k-means are no-ops and the final
  // control-block read reports it
  low.count = -1;
  launch_lowdeg_exact(low, deg, ws.ctl, s);
  mark(ev, 2, s);
  if (d_v0 != nullptr) {  // explicit start vector (initial_vector, serial.py:77-101)
    launch_scale_by(d_v0, n, 1.0, ws.v64, ws.v32, vector_pitch(n), s);
  } else {                // v0 = d / tree_sum(d) (initial_embedding, parallel.py:210-214)
    launch_tree_sum(deg, n, ws.redpart, ws.redpart + ceil_div(n, kRedBlock), ws.ctl, s);
    launch_scale_vector(deg, n, ws.redpart + ceil_div(n, kRedBlock), ws.v64, ws.v32,
                        vector_pitch(n), s);
  }
  L.a = a;
  L.lda = lda;
  L.rows = n;
  L.deg = deg;
  L.redpart = ws.redpart;
  // the fused iteration kernel's per-chunk ready counters (sym.cu), behind
  // the tail's partials; each chunk's owner resets its counter after use
  GPIC_CUDA_TRY(cudaMemsetAsync(ws.redpart + ceil_div(n, kRedBlock) + 1, 0,
                                ceil_div(n, kRedBlock) * 4, s));
  L.v64 = ws.v64;
  L.v32 = ws.v32;
  L.hist = d_delta_hist;
  L.ctl = ws.ctl;
  L.pt.y[0][0] = L.pt.y[0][1] = ws.y;
  L.pt.nranks = 1;
  L.low = low;
  L.low_deg = deg;
  rc = run_power_loops(&L, 1, n, max_iter, s);
  if (rc) return rc;
  if (reordered) {  // back to the caller's order before the k-means
    launch_copy_result(ws.v64, n, ws.y, ws.ctl, s);
    launch_unpermute(ws.y, loc.perm, n, d_v, s);
  } else {
    launch_copy_result(ws.v64, n, d_v, ws.ctl, s);
  }
  mark(ev, 3, s);
  GPIC_CUDA_TRY(cudaGetLastError());
  // the k-means kernels read the loop's status on the device (a failed loop
  // leaves them no-ops), so the control block is read once, at the end
  rc = launch_kmeans1d(d_v, n, k, first_index, h_uniforms, 100, 1e-12, d_labels, ws.kscratch,
                       ws.ctl, s);
  if (rc) return rc;
  mark(ev, 4, s);
  gpic_ctl h;
  rc = gpic_ctl_read(ws.ctl, &h, stream);
  if (rc) return rc;
  note_loop_iterations(h.iter);
  if (h_iters) *h_iters = h.iter;
  if (h_converged) *h_converged = h.converged;
  return status_from_ctl(h, d);
}
}  // namespace

extern "C" {

int gpic_cluster(const double* d_x, int64_t n, int32_t d, double sigma, int32_t kind, int32_t k,
                 double eps, int32_t max_iter, int64_t first_index, const double* h_uniforms,
                 int32_t impl, int32_t storage, const double* d_v0, int64_t* d_labels, double* d_v,
                 double* d_delta_hist, int32_t* h_iters, int32_t* h_converged, void* d_work,
                 int64_t work_bytes, void* stream) {
  return cluster_impl(d_x, n, d, sigma, kind, k, eps, max_iter, first_index, h_uniforms, impl,
                      storage, d_v0, d_labels, d_v, d_delta_hist, h_iters, h_converged, d_work,
                      work_bytes, stream, nullptr);
}

int gpic_cluster_timed(const double* d_x, int64_t n, int32_t d, double sigma, int32_t kind,
                       int32_t k, double eps, int32_t max_iter, int64_t first_index,
                       const double* h_uniforms, int32_t impl, int32_t storage,
                       const double* d_v0, int64_t* d_labels, double* d_v, double* d_delta_hist,
                       int32_t* h_iters, int32_t* h_converged, void* d_work, int64_t work_bytes,
                       void* stream, float* h_phase_ms) {
  if (!h_phase_ms) return fail(GPIC_E_INVALID, "h_phase_ms must point at 5 floats");
  cudaEvent_t ev[5];
  for (int i = 0; i < 5; ++i) GPIC_CUDA_TRY(cudaEventCreate(&ev[i]));
  int rc = cluster_impl(d_x, n, d, sigma, kind, k, eps, max_iter, first_index, h_uniforms, impl,
                        storage, d_v0, d_labels, d_v, d_delta_hist, h_iters, h_converged, d_work,
                        work_bytes, stream, ev);
  if (rc == GPIC_OK) {
    // the final gpic_ctl_read synchronised the stream: all 5 events are complete
    float t[4];
    for (int i = 0; i < 4; ++i) cudaEventElapsedTime(&t[i], ev[i], ev[i + 1]);
    h_phase_ms[0] = t[0];  // affinity (prepare + Gram + exp epilogue)
    h_phase_ms[1] = t[1];  // rowsum (degree combine)
    h_phase_ms[2] = 0.f;   // normalize: folded into the GEMV epilogue
    h_phase_ms[3] = t[2];  // iterate (start vector + device-resident loop)
    h_phase_ms[4] = t[3];  // kmeans
  }
  for (int i = 0; i < 5; ++i) cudaEventDestroy(ev[i]);
  return rc;
}

int64_t gpic_cluster_host_workspace_bytes(int64_t n, int32_t d, int32_t k, int32_t max_iter,
                                          int32_t storage) {
  const int64_t w = gpic_cluster_workspace_bytes(n, d, k, max_iter, storage);
  if (w < 0 || max_iter < 1) return -1;
  return al(w) + al(n * d * 8) + al(n * 8) * 3 + al((int64_t)max_iter * 8);
}

int gpic_cluster_host(const double* h_x, int64_t n, int32_t d, double sigma, int32_t kind,
                      int32_t k, double eps, int32_t max_iter, int64_t first_index,
                      const double* h_uniforms, int32_t impl, int32_t storage,
                      const double* h_v0, int64_t* h_labels, double* h_v, double* h_delta_hist,
                      int32_t* h_iters, int32_t* h_converged, void* d_work, int64_t work_bytes,
                      void* stream) {
  if (n < 1 || d < 1) return fail(GPIC_E_EMPTY, "dataset must contain at least one point and one feature");
  if (max_iter < 1) return fail(GPIC_E_INVALID, "max_iterations must be at least 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // device staging after the pipeline workspace: X, labels, v, v0, deltas
  const int64_t scratch = al(gpic_cluster_workspace_bytes(n, d, k, max_iter, storage));
  if (work_bytes < gpic_cluster_host_workspace_bytes(n, d, k, max_iter, storage))
    return fail(GPIC_E_INVALID, "workspace too small (gpic_cluster_host_workspace_bytes)");
  uint8_t* p = static_cast<uint8_t*>(d_work) + scratch;
  double* dx = reinterpret_cast<double*>(p); p += al(n * d * 8);
  int64_t* dl = reinterpret_cast<int64_t*>(p); p += al(n * 8);
  double* dv = reinterpret_cast<double*>(p); p += al(n * 8);
  double* dv0 = reinterpret_cast<double*>(p); p += al(n * 8);
  double* dh = reinterpret_cast<double*>(p);
  GPIC_CUDA_TRY(cudaMemcpyAsync(dx, h_x, n * d * 8, cudaMemcpyHostToDevice, s));
  if (h_v0) GPIC_CUDA_TRY(cudaMemcpyAsync(dv0, h_v0, n * 8, cudaMemcpyHostToDevice, s));
  int32_t iters = 0, conv = 0;
  int rc = gpic_cluster(dx, n, d, sigma, kind, k, eps, max_iter, first_index, h_uniforms, impl,
                        storage, h_v0 ? dv0 : nullptr, dl, dv, dh, &iters, &conv, d_work, scratch,
                        stream);
  if (rc) return rc;
  GPIC_CUDA_TRY(cudaMemcpyAsync(h_labels, dl, n * 8, cudaMemcpyDeviceToHost, s));
  GPIC_CUDA_TRY(cudaMemcpyAsync(h_v, dv, n * 8, cudaMemcpyDeviceToHost, s));
  GPIC_CUDA_TRY(cudaMemcpyAsync(h_delta_hist, dh, (int64_t)iters * 8, cudaMemcpyDeviceToHost, s));
  GPIC_CUDA_TRY(cudaStreamSynchronize(s));
  if (h_iters) *h_iters = iters;
  if (h_converged) *h_converged = conv;
  return GPIC_OK;
}

}  // extern "C"
