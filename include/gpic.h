/*
 * gpic.h — C ABI of libgpic.so, the B200 (sm_100a) engine behind the
 * reference's Power Iteration Clustering operators.
 *
 * Every entry point replaces one operator of the reference package
 * (/root/reference/pkg/src/picluster, cited file:line). Conventions:
 *
 *   - Plain pointers and sizes only. Pointers named d_* are DEVICE memory
 *     owned by the caller (PyTorch tensors in the Python binding); h_* are
 *     host memory. The library never allocates on the hot path: scratch
 *     space comes from a caller-provided workspace sized by
 *     gpic_workspace_bytes().
 *   - Calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) unless stated otherwise.
 *   - Data-dependent errors (a zero-degree row, a non-finite input, a
 *     non-positive normaliser) are detected ON THE DEVICE and recorded in
 *     the gpic_ctl block; gpic_ctl_read() / the synchronous entry points
 *     return them as status codes. The Python layer maps codes onto the
 *     reference's exception classes (errors.py:10-113):
 *         GPIC_E_INVALID      -> InvalidSpec / DimensionMismatch
 *         GPIC_E_ZERO_DEGREE  -> ZeroDegree(index)          (affinity.py:113-119)
 *         GPIC_E_NONFINITE    -> NonFiniteEntry(row, col)   (data.py:69-72)
 *         GPIC_E_NONPOS_TAU   -> NonPositiveTau(tau)        (parallel.py:181-193)
 *         GPIC_E_EMPTY        -> EmptyVector / EmptyDataSet
 *         GPIC_E_K_TOO_LARGE  -> KTooLarge                  (kmeans.py:187-188)
 *         GPIC_E_CUDA, GPIC_E_COMM, GPIC_E_UNSUPPORTED -> RuntimeError
 *   - Not reentrant per stream / ctl block. One host thread per device.
 */
#ifndef GPIC_H
#define GPIC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPIC_OK 0
#define GPIC_E_INVALID 1
#define GPIC_E_ZERO_DEGREE 2
#define GPIC_E_NONFINITE 3
#define GPIC_E_NONPOS_TAU 4
#define GPIC_E_EMPTY 5
#define GPIC_E_K_TOO_LARGE 6
#define GPIC_E_CUDA 16
#define GPIC_E_COMM 17
#define GPIC_E_UNSUPPORTED 18
#define GPIC_E_ZERO_VECTOR 7 /* ZeroVector(index), cosine kind (affinity.py:41-53) */

/* Similarity kinds (affinity.py:22-35). */
#define GPIC_KIND_RBF 0    /* GaussianRbf(sigma): exp(-|x-y|^2 / 2 sigma^2) */
#define GPIC_KIND_COSINE 1 /* Cosine(): max(0, x.y / (|x||y|)), sigma ignored */

/* Affinity engines (KernelConfig.affinity_impl). The tcgen05 engine holds a
 * row block's operands in shared memory: d <= 192 with stored A (dense /
 * packed / packed16), d <= 256 matrix-free. Wider data asked of it runs on the
 * SIMT engine with dense rows (the cluster calls and their workspace query
 * apply the same rule, so the caller's sizes stay consistent). RBF with
 * d <= 8 and stored A runs on the SIMT engine in difference form (the tensor
 * Gram's fp32 cancellation would exceed the 1e-4 embedding gate there). */
#define GPIC_AFFINITY_TC 0   /* tcgen05 kind::f16, 3-term fp16 split, TMEM accumulators */
#define GPIC_AFFINITY_SIMT 1 /* FP32 FFMA engine, any d */

/* Device-resident control block of one power-iteration run (64-bit aligned,
 * 256 bytes). Written by the kernels; read back once at the end. */
typedef struct gpic_ctl {
  int32_t iter;        /* iterations completed                          */
  int32_t stop;        /* 1 once converged / capped / failed             */
  int32_t converged;   /* PicTrace.converged                             */
  int32_t status;      /* GPIC_OK or a GPIC_E_* code                     */
  int64_t err_index;   /* first offending row (ZeroDegree, NonFinite)    */
  int64_t err_index2;  /* column for NonFiniteEntry                      */
  double err_value;    /* tau for NonPositiveTau                         */
  double eps;          /* resolved stop threshold                        */
  int32_t max_iter;
  int32_t nranks;
  uint64_t delta_bits; /* running max |v_t - v_(t-1)| (as fp64 bits)    */
  uint32_t arrive[4];  /* last-CTA-done counters                         */
  double tau;          /* current L1 normaliser                          */
  uint64_t sync_epoch; /* cross-rank exchange epoch                      */
  uint32_t tau_gen;    /* bumped each time the fused tail publishes tau  */
  uint32_t bar_count;  /* grid barrier of the fused iteration kernel     */
  uint32_t bar_gen;    /* its generation                                 */
  uint8_t pad[256 - 108];
} gpic_ctl;

/* Library identity: "gpic <version> sm_100a". */
const char* gpic_version(void);
/* Last host-side error message (thread-local). */
const char* gpic_last_error(void);
/* Status of the last failure with its detail (thread-local): index = first
 * offending row for ZeroDegree / ZeroVector, (index, index2) = (row, col)
 * for NonFiniteEntry, value = tau for NonPositiveTau; -1 / 0 otherwise. */
int gpic_last_detail(int64_t* index, int64_t* index2, double* value);
/* Device memory for bindings without a CUDA allocator of their own (cgo,
 * JNI, a bare ctypes caller); never used on the hot path. */
int gpic_malloc(int64_t bytes, void** out);
int gpic_free(void* ptr);

/* Bytes of device scratch the pipeline needs for n points of dimension d,
 * k clusters, a row shard of `rows` rows and `max_iter` iterations. */
int64_t gpic_workspace_bytes(int64_t n, int32_t d, int32_t k, int64_t rows, int32_t max_iter);
/* Row pitch (floats) of the stored affinity block for n columns. */
int64_t gpic_affinity_pitch(int64_t n);

/* ---- stage 0: validate + centre + cast -------------------------------
 * Replaces validate_dataset's finiteness scan (data.py:61-78) and prepares
 * the operands of the Gram engines (dp = gpic_feature_pitch(d),
 * n_pad = gpic_row_pad(n)):
 *   d_xlo  n_pad x dp floats: xc = fp32(x - mean_fp64), row-major (the FFMA
 *          engine)
 *   d_xhi  gpic_operand_floats(n, d) floats: the tensor engine's fp16
 *          planes hi = fp16(xc * s) (n_pad x dp halves) then
 *          lo = fp16(xc * s - hi); s = 2^e, max|xc * s| < 2^8; then the
 *          norm block (4 planes of n_pad x 16 halves: row operand hi / lo
 *          [2^10, M_i], column operand hi / lo [M_j, 2^10],
 *          M = -(s^2/2)|x~|^2 / 2^10) with which the MMA accumulates
 *          -(s^2/2)|x_i - x_j|^2 directly
 *   d_sqn  |xc|^2 per row; d_sqn[n_pad - 1] (a padding row) holds 1 / s^2
 * A non-finite entry sets GPIC_E_NONFINITE with the first (row, col) in
 * row-major order. d_work: (ceil(n / 256) + 1) * d + 2 doubles; after the
 * call its last two hold max |xc| over all entries and R^2 = max_i |xc_i|^2
 * (RBF), the spread that gpic_engine_for routes on.
 * kind GPIC_KIND_COSINE instead scales every row to unit length in fp64
 * (no centring: cosine is not translation invariant) and reports a zero
 * row as GPIC_E_ZERO_VECTOR(first row) (cosine_norms, affinity.py:41-53). */
int32_t gpic_feature_pitch(int32_t d);
int64_t gpic_row_pad(int64_t n);
int64_t gpic_operand_floats(int64_t n, int32_t d);
int gpic_prepare_points(const double* d_x, int64_t n, int32_t d, int32_t kind, float* d_xhi,
                        float* d_xlo, float* d_sqn, void* d_work, gpic_ctl* d_ctl, void* stream);
/* The affinity engine a storage runs for data of spread R^2 (max squared
 * distance to the mean, from gpic_prepare_points): the tensor engine's Gram
 * form carries ~2^-24 R^2 / (2 sigma^2) relative error per entry, so RBF
 * data with R^2 / (2 sigma^2) > 167.8 (2^24 x 1e-5: a tenth of the 1e-4
 * embedding gate) and RBF at d <= 8 run the SIMT difference form; d > 192
 * with stored A runs SIMT dense rows. gpic_cluster applies this itself. */
int32_t gpic_engine_for(int32_t kind, int32_t d, double sigma, double spread2, int32_t impl,
                        int32_t storage);

/* ---- stage 1: affinity block + degree ---------------------------------
 * Replaces similarity_rows/build_affinity (affinity.py:74-110, RBF kind),
 * k_affinity (parallel.py:113-128) and k_rowsum/degree (affinity.py:113-119,
 * parallel.py:131-143) for rows [row_lo, row_hi):
 *     A[i - row_lo, j] = exp(-|x_i - x_j|^2 / (2 sigma^2)),  A[i, i] = 0
 * stored fp32 with row pitch `lda` (>= n, multiple of 32; pad columns 0),
 * deg[i - row_lo] = sum_j A[i, j] accumulated in fp64 from the stored
 * fp32 values, fixed order (independent of the shard plan). W = D^-1 A is
 * never materialised: the power iteration applies 1/deg in its epilogue
 * (folded normalisation, k_normalize parallel.py:146-158). deg <= 0 sets
 * GPIC_E_ZERO_DEGREE(first row). */
int gpic_affinity_rbf(const float* d_xhi, const float* d_xlo, const float* d_sqn, int64_t n,
                      int32_t d, int64_t row_lo, int64_t row_hi, double sigma, int32_t impl,
                      float* d_a, int64_t lda, double* d_deg, void* d_work, gpic_ctl* d_ctl,
                      void* stream);
/* Same for the cosine kind (affinity.py:88-95): A_ij = max(0, cos(x_i, x_j))
 * on points prepared with GPIC_KIND_COSINE. */
int gpic_affinity_cosine(const float* d_xhi, const float* d_xlo, const float* d_sqn, int64_t n,
                         int32_t d, int64_t row_lo, int64_t row_hi, int32_t impl, float* d_a,
                         int64_t lda, double* d_deg, void* d_work, gpic_ctl* d_ctl, void* stream);

/* ---- stage 2: start vector -----------------------------------------------
 * initial_embedding "degree" choice (parallel.py:210-214 = k_norm(deg,
 * k_reduce(deg))): v0 = deg / tree_sum(deg). Writes fp64 and fp32 copies. */
int gpic_initial_vector(const double* d_deg, int64_t n, double* d_v64, float* d_v32,
                        void* d_work, gpic_ctl* d_ctl, void* stream);

/* ---- stage 3: power iteration ------------------------------------------
 * Replaces power_iterate (serial.py:104-128) / iterate (parallel.py:217-233):
 *     y = (A v) / deg ; tau = tree_sum(y) ; v' = y / tau ;
 *     delta_t = max|v' - v| ; stop when t >= 2 and |delta_t - delta_(t-1)| <= eps
 * entirely on the device (no host sync per iteration): each iteration is a
 * GEMV with the D^-1 epilogue, a fixed-shape tau reduction and a fused
 * normalise/delta/stop kernel; the loop is a CUDA graph whose kernels
 * become no-ops once ctl->stop is set. Single-rank form: the shard is the
 * whole matrix (row_lo = 0, rows = n). d_v64 holds 2*n doubles (ping-pong),
 * the final vector is returned in d_v64_out. h_* outputs are filled after
 * an internal stream synchronize. */
int gpic_power_iterate(const float* d_a, int64_t lda, const double* d_deg, int64_t n,
                       double* d_v64, float* d_v32, double eps, int32_t max_iter,
                       double* d_delta_hist, double* d_v64_out, void* d_work, gpic_ctl* d_ctl,
                       void* stream);

/* ---- stage 4: 1-D k-means ----------------------------------------------
 * kmeans_1d (kmeans.py:178-196): k-means++ seeding from the caller's PCG64
 * draws (first index + k-1 uniforms from np.random.default_rng(seed),
 * kmeans.py:43,51,73), Lloyd rounds (<= max_rounds, tol), exact DP polish
 * when n <= 4096 (kmeans.py:97-130), contiguity check/repair
 * (kmeans.py:133-160) and canonical relabel by ascending centroid
 * (kmeans.py:163-175). Writes int64 labels. 2 <= k <= min(n, 4096):
 * k <= 64 keeps per-cluster registers (kmeans.cu); 64 < k runs the same
 * algorithm on the once-sorted values (kmeans_big.cu: clusters are
 * contiguous runs, sums are prefix differences). */
int gpic_kmeans1d(const double* d_v, int64_t n, int32_t k, int64_t first_index,
                  const double* h_uniforms, int32_t max_rounds, double tol, int64_t* d_labels,
                  void* d_work, gpic_ctl* d_ctl, void* stream);

/* ---- per-operator entry points (parity tests, reference kernel API) ---- */
/* k_reduce (parallel.py:161-178): fixed-shape fp64 sum into *d_out.
 * d_work: 256 + 8 * (ceil(n / 2048) + 1) bytes. */
int gpic_reduce_sum(const double* d_v, int64_t n, double* d_out, void* d_work, void* stream);
/* k_multiply (parallel.py:196-207) on an fp32 matrix: y = (A v) * scale_i,
 * scale = d_inv_deg (fp64, may be NULL for 1). */
int gpic_matvec(const float* d_a, int64_t lda, int64_t rows, int64_t n, const float* d_v,
                const double* d_row_scale, double* d_y, void* stream);
/* App-B Gaussian blobs generated in device memory (the
 * host generator is datasets.gaussian_blobs): row i of blob c
 * (d_offsets[c] <= i < d_offsets[c+1], k+1 entries, d_offsets[k] = n) is
 * d_centers[c] + noise * z + offset, z standard normal from Philox4x32-10
 * keyed by `seed` (element pair p -> counter (p, 0, 0), Box-Muller on two
 * 53-bit uniforms). d_x: n x d fp64 row-major; d_labels: n int64 or NULL.
 * Deterministic in (seed, n, d, centres, offsets). */
int gpic_generate_blobs(const double* d_centers, const int64_t* d_offsets, int64_t n, int32_t d,
                        int32_t k, uint64_t seed, double noise, double offset, double* d_x,
                        int64_t* d_labels, void* stream);
/* check_row_stochastic (serial.py:63-74) on an fp64 row-major matrix
 * (leading dimension ldw doubles): per-row sum, min and max into d_sum /
 * d_min / d_max (rows doubles each); NaN propagates. The caller applies the
 * reference's tolerance (row sums within 1e-9 of 1, entries in [0, 1]). */
int gpic_row_stats(const double* d_w, int64_t rows, int64_t n, int64_t ldw, double* d_sum,
                   double* d_min, double* d_max, void* stream);
/* k_multiply on PACKED symmetric tiles (gpic_packed_tiles(n) tiles of
 * 128 x 128 fp32, upper triangle): y = (A v) * scale_i. d_v holds
 * gpic_vector_pitch(n) floats (zero padded); d_rowp / d_colp hold
 * gpic_sym_partial_floats(n) floats each (super-block partial records). */
int gpic_sym_matvec(const float* d_tiles, int64_t n, const float* d_v, float* d_rowp,
                    float* d_colp, const double* d_row_scale, double* d_y, void* stream);
/* Floats of each partial buffer (d_rowp, d_colp) of gpic_sym_matvec[16]. */
int64_t gpic_sym_partial_floats(int64_t n);
/* Same over fp16 tiles (GPIC_STORAGE_PACKED16 layout, 128 x 128 halves each). */
int gpic_sym_matvec16(const void* d_tiles, int64_t n, const float* d_v, float* d_rowp,
                      float* d_colp, const double* d_row_scale, double* d_y, void* stream);
int64_t gpic_vector_pitch(int64_t n);
/* k_multiply on the packed tiles a gpic_cluster run left in its workspace,
 * with the run's block sparsity: only tiles with a stored 32 x 32 box are
 * read, unstored boxes count as the exact zeros they are (d_boxnz, 16
 * flags per tile; d_sb_prefix the GEMV weights; both NULL = every tile).
 * half: fp16 tiles (GPIC_STORAGE_PACKED16). Offsets of the tiles, partial
 * buffers, flags and weights: gpic_cluster_workspace_layout. */
int gpic_sym_matvec_sparse(const void* d_tiles, int32_t half, int64_t n, const float* d_v,
                           float* d_rowp, float* d_colp, const double* d_row_scale, double* d_y,
                           const uint8_t* d_boxnz, const int64_t* d_sb_prefix, void* stream);

/* ---- whole pipeline ----------------------------------------------------
 * cluster (serial.py:131-150 / parallel.py:236-255) for one rank owning the
 * whole matrix. Device in/out; d_work must hold
 * gpic_cluster_workspace_bytes(n, d, k, max_iter, storage). Synchronous:
 * returns the first error. d_v0: NULL starts from d / sum(d) (the "degree"
 * choice, initial_embedding parallel.py:210-214); otherwise n doubles of an
 * explicit start vector, already validated by the caller like
 * initial_vector (serial.py:77-101: "uniform" = 1/n, or length n,
 * nonnegative, unit L1 norm).
 *
 * storage: GPIC_STORAGE_DENSE keeps A as n x pitch(n) fp32 rows (4n^2 bytes
 * per power iteration); GPIC_STORAGE_PACKED keeps only the upper triangle
 * of 128 x 128 tiles (A is exactly symmetric, test_affinity.py:81-87): half
 * the bytes for the affinity store and for every iteration's GEMV
 * (tcgen05 engine only). */
#define GPIC_STORAGE_DENSE 0
#define GPIC_STORAGE_PACKED 1
/* matrix-free (n^2 beyond HBM): A is never stored; every A v is
 * recomputed from X by the tcgen05 engine with the multiply-by-v fused into
 * the exp epilogue (compute-bound instead of HBM-bound). */
#define GPIC_STORAGE_NONE 2
/* packed upper-triangle tiles stored as fp16 (A in [0, 1]; the compressed-W
 * option of SURVEY.md §8f-2): a quarter of the dense bytes per iteration.
 * Degrees are the sums of the stored (rounded) values, so W = D^-1 A stays
 * row-stochastic; fp32 accumulation everywhere. Opt-in: the default is fp32. */
#define GPIC_STORAGE_PACKED16 3
int64_t gpic_packed_tiles(int64_t n);
int64_t gpic_cluster_workspace_bytes(int64_t n, int32_t d, int32_t k, int32_t max_iter,
                                     int32_t storage);
/* Byte offsets inside that workspace (packed storages), offsets[8]: [0]
 * tiles, [1] GEMV row records, [2] column records, [3] stored-box flags,
 * [4] GEMV weights, [5] degrees (fp64), [6] the count (int64) of tcgen05
 * work units computed after tile pruning, [7] the number of units before
 * pruning (a value, not an offset). For measurement and tests. */
int gpic_cluster_workspace_layout(int64_t n, int32_t d, int32_t k, int32_t max_iter,
                                  int32_t storage, int64_t* offsets);
/* Work the tensor engine did in the last gpic_cluster run on this
 * workspace after tile pruning (prune.cu: block pairs proved to hold only
 * entries below 2^-64 are never computed): packed storages -> kept / all
 * work units (128 MB rows x 128 columns); GPIC_STORAGE_NONE -> kept / all
 * tile units of one symmetric pass. Synchronizes `stream`. */
int gpic_cluster_pruned_work(const void* d_work, int64_t n, int32_t d, int32_t k,
                             int32_t max_iter, int32_t storage, int64_t* kept, int64_t* total,
                             void* stream);
/* The locality order of the last gpic_cluster run on this workspace
 * (randomly ordered inputs are permuted so that block sparsity and tile
 * pruning apply; v is scattered back): *reordered = 1 and d_perm[p] (n
 * int32) = the caller's index of permuted position p, or *reordered = 0.
 * Measurement / tests. Synchronizes `stream`. */
int gpic_cluster_permutation(const void* d_work, int64_t n, int32_t d, int32_t k, int32_t max_iter,
                             int32_t* d_perm, int32_t* reordered, void* stream);
/* One matrix-free pass y = A v (no 1/deg) on the operands, pruning mask
 * (pruned != 0) and partial buffers that a GPIC_STORAGE_NONE gpic_cluster
 * run left in d_work — the power loop's own pass, for kernel timing. */
int gpic_cluster_mf_pass(void* d_work, int64_t n, int32_t d, int32_t k, int32_t max_iter,
                         double sigma, int32_t kind, int32_t pruned, const float* d_v32,
                         double* d_y, void* stream);
int gpic_cluster(const double* d_x, int64_t n, int32_t d, double sigma, int32_t kind, int32_t k,
                 double eps, int32_t max_iter, int64_t first_index, const double* h_uniforms,
                 int32_t impl, int32_t storage, const double* d_v0, int64_t* d_labels, double* d_v,
                 double* d_delta_hist, int32_t* h_iters, int32_t* h_converged, void* d_work,
                 int64_t work_bytes, void* stream);

/* gpic_cluster plus per-phase device times (CUDA events on `stream`), the
 * phases of report.py:28 / run_timed report.py:47-99: h_phase_ms[5] =
 * {affinity, rowsum, normalize (0: folded into the GEMV), iterate, kmeans}. */
int gpic_cluster_timed(const double* d_x, int64_t n, int32_t d, double sigma, int32_t kind,
                       int32_t k, double eps, int32_t max_iter, int64_t first_index,
                       const double* h_uniforms, int32_t impl, int32_t storage,
                       const double* d_v0, int64_t* d_labels, double* d_v, double* d_delta_hist,
                       int32_t* h_iters, int32_t* h_converged, void* d_work, int64_t work_bytes,
                       void* stream, float* h_phase_ms);

/* Same, HOST buffers in and out (the reference-facing call a ctypes/cffi
 * binding makes, replacing picluster.cluster(...) of __init__.py:39-45 /
 * parallel.cluster, parallel.py:236-255): copies X in, runs, copies
 * labels/v/deltas out. d_work must hold gpic_cluster_host_workspace_bytes
 * (= gpic_cluster_workspace_bytes, 256-aligned, + the staging of X (n*d*8),
 * labels, v and v0 (n*8 each) and the deltas (max_iter*8)); h_v0 as d_v0. On failure the
 * status code is returned and gpic_last_detail() gives the offending index
 * (ZeroDegree / ZeroVector), (row, col) (NonFiniteEntry) or tau. */
int64_t gpic_cluster_host_workspace_bytes(int64_t n, int32_t d, int32_t k, int32_t max_iter,
                                          int32_t storage);
int gpic_cluster_host(const double* h_x, int64_t n, int32_t d, double sigma, int32_t kind,
                      int32_t k, double eps, int32_t max_iter, int64_t first_index,
                      const double* h_uniforms, int32_t impl, int32_t storage,
                      const double* h_v0, int64_t* h_labels, double* h_v, double* h_delta_hist,
                      int32_t* h_iters, int32_t* h_converged, void* d_work, int64_t work_bytes,
                      void* stream);

/* Reset a control block (iteration 0, no error) with the stop threshold and
 * iteration cap of the run. */
int gpic_ctl_init(gpic_ctl* d_ctl, double eps, int32_t max_iter, void* stream);

/* k_norm (parallel.py:181-193): dst = src / tau in fp64, plus an optional
 * fp32 copy zero-padded to f32_len (NULL to skip). tau must be > 0 (checked
 * on the host, NonPositiveTau otherwise, NaN included). */
int gpic_scale(const double* d_src, int64_t n, double tau, double* d_dst, float* d_dst32,
               int64_t f32_len, void* stream);

/* Device scratch of gpic_kmeans1d for n values and k clusters. */
int64_t gpic_kmeans_scratch_bytes(int64_t n, int32_t k);

/* Read the control block back (synchronizes `stream`). */
int gpic_ctl_read(const gpic_ctl* d_ctl, gpic_ctl* h_out, void* stream);

/* Kernels launched by this library since load (for the bench's
 * gpu_launches claim). */
int64_t gpic_launch_count(void);

/* ---- multi-rank (row-sharded) power iteration --------------------------
 * Replaces the worker fan-out of the reference's parallel backend
 * (plan_rows / _run_workers, parallel.py:90-110; k_multiply per row range,
 * :196-207) with one rank per GPU: rank r owns rows [row_lo, row_lo + rows)
 * of A. Exchanges are fused into the producing kernels (P2P stores of the
 * y / degree slices into every rank's buffers through CUDA IPC over
 * NVLink, epoch flags, acquire-spin waits); no NCCL launch and no host sync
 * per iteration. Results are bitwise independent of the rank count (the
 * reference's p-invariance, parallel.py:10-22, test_parallel.py:194-223).
 *
 * Real ranks (one process per GPU): gpic_comm_create on every rank, share
 * the GPIC_IPC_HANDLE_BYTES handles (any host collective), gpic_comm_open.
 * Virtual ranks (P shards in one process on one device, the identical
 * exchange code path): gpic_comm_create_virtual. At most 8 ranks. */
#define GPIC_IPC_HANDLE_BYTES 64
typedef struct gpic_comm gpic_comm;
typedef struct gpic_shard {
  const float* a;     /* rows x lda fp32 affinity rows of this shard        */
  int64_t lda;
  const double* deg;  /* rows degrees                                       */
  int64_t row_lo;
  int64_t rows;
  /* matrix-free shards (storage == GPIC_STORAGE_NONE): a is unused and the
   * rows are recomputed from the prepared points every iteration */
  int32_t storage;
  int32_t d;
  const float* xhi;
  const float* xlo;
  const float* sqn;
  double sigma;
  int32_t kind;       /* GPIC_KIND_*                                          */
  double* ypart;      /* gpic_mf_ypart_doubles(n, d, rows) doubles          */
  /* the caller's fp64 points (n x d, row-major, every rank holds all of X):
   * rows whose fp32 degree underflows (isolated points) are redone from them
   * in fp64 like the reference (affinity.py:96-119); may be null when no
   * such row exists (gpic_comm_gather_degrees then fails with INVALID) */
  const double* x;
} gpic_shard;

/* Packed shard rows balanced by WORK: the whole matrix's tile-pruning mask
 * (prune.cu, the same on every rank) gives the kept tensor units per row
 * block; bounds[0..nranks] are 512-aligned rows cutting the kept-unit
 * prefix into equal parts (bounds[nranks] = n). gpic_packed_shard_range
 * balances the dense triangle instead, which leaves block-sparse ranks
 * unequal. d_xlo / d_prep_work: gpic_prepare_points' outputs; d_scratch:
 * gpic_prune_scratch_bytes(n, d) bytes. Replaces: parallel.py:44-77
 * plan_rows for the packed symmetric shards. */
int64_t gpic_prune_scratch_bytes(int64_t n, int32_t d);
int gpic_packed_shard_ranges_pruned(const float* d_xlo, const double* d_prep_work, int64_t n,
                                    int32_t d, double sigma, int32_t nranks, void* d_scratch,
                                    int64_t* bounds, void* stream);
/* Packed shards (symmetric storage across ranks, GPIC_STORAGE_PACKED in
 * gpic_shard): rank r owns the 512-row super-rows [row_lo, row_hi) returned
 * by gpic_packed_shard_range (balanced by stored tile count) and stores the
 * upper-triangle tiles of those rows (gpic_packed_shard_tiles x 64 KB).
 * gpic_packed_shard_build computes them plus the shard's partial degrees
 * (d_deg_partial: n doubles, global row index). In the gpic_shard: a = the
 * tiles, deg = the partial degrees, row_lo / rows = the range, ypart = the
 * build's scratch (gpic_packed_shard_scratch_bytes). Every iteration the
 * partial y go over NVLink P2P either to every rank (P = 2) or, from P = 3,
 * to their row slice's owner, which sums the P partials and all-gathers the
 * finished y slice (GPIC_EXCHANGE=bcast / rs forces one); the P partials
 * are summed in rank order either way: deterministic for a given P. */
int gpic_packed_shard_range(int64_t n, int32_t nranks, int32_t rank, int64_t* row_lo,
                            int64_t* row_hi);
int64_t gpic_packed_shard_tiles(int64_t n, int64_t row_lo, int64_t row_hi);
int64_t gpic_packed_shard_scratch_bytes(int64_t n, int64_t row_lo, int64_t row_hi);
/* d_prep_work: the work buffer of gpic_prepare_points (column sums + mean):
 * with it (RBF) the shard's provably-zero block pairs are not computed; its
 * zero 32 x 32 boxes are never stored either way (block sparsity, flags in
 * d_scratch). NULL: no pruning. */
int gpic_packed_shard_build(const float* d_xhi, const float* d_xlo, const float* d_sqn, int64_t n,
                            int32_t d, int64_t row_lo, int64_t row_hi, double sigma, int32_t kind,
                            float* d_tiles, double* d_deg_partial, void* d_scratch,
                            const double* d_prep_work, void* stream);

/* Matrix-free degrees of rows [row_lo, row_hi): deg = A 1 recomputed from the
 * prepared points (gpic_prepare_points). d_ones: gpic_vector_pitch(n) floats
 * of scratch; d_ypart: gpic_mf_ypart_doubles(n, d, rows) doubles. */
int64_t gpic_mf_ypart_doubles(int64_t n, int32_t d, int64_t rows);
int gpic_mf_degrees(const float* d_xhi, const float* d_xlo, const float* d_sqn, int64_t n,
                    int32_t d, int64_t row_lo, int64_t row_hi, double sigma, int32_t kind,
                    float* d_ones, double* d_ypart, double* d_deg, void* stream);

/* Matrix-free item shards (GPIC_STORAGE_NONE with row_lo = 0, rows = n in
 * gpic_shard): every rank holds all of X; the pruned symmetric pass's kept
 * (row block, column chunk) items (prune.cu) are split across the ranks by
 * kept-tile count, and each rank's reduce yields a PARTIAL y over all rows
 * that is exchanged and summed in rank order like the packed shards'
 * (half the exp / MMA work of row bands, and no pruned pair is computed).
 * Such a shard is marked lda = 1 (row_lo = 0, rows = n, ypart = d_scratch).
 * gpic_mf_shard_build builds the pruning mask (d_prep_work: the work buffer
 * of gpic_prepare_points) and the shard's partial degrees (n doubles);
 * d_scratch (gpic_mf_shard_scratch_bytes) is the gpic_shard's ypart. RBF
 * with d > 8 on the tensor engine; GPIC_E_UNSUPPORTED otherwise (row bands
 * then). */
int64_t gpic_mf_shard_scratch_bytes(int64_t n, int32_t d);
int gpic_mf_shard_build(const float* d_xhi, const float* d_xlo, const float* d_sqn,
                        const double* d_prep_work, int64_t n, int32_t d, double sigma,
                        int32_t nranks, int32_t rank, double* d_deg_partial, void* d_scratch,
                        void* stream);

int gpic_comm_create(int32_t nranks, int32_t rank, int64_t n, gpic_comm** out,
                     uint8_t* h_ipc_handle);
int gpic_comm_open(gpic_comm* comm, const uint8_t* h_all_handles /* nranks x 64 bytes */);
int gpic_comm_create_virtual(int32_t nranks, int64_t n, gpic_comm** out);
int gpic_comm_destroy(gpic_comm* comm);
/* All-gather of the degree slices (once per run) + the global ZeroDegree
 * check; optionally copies the full degree vector out. Synchronous. */
int gpic_comm_gather_degrees(gpic_comm* comm, const gpic_shard* shards, int32_t nlocal,
                             double* d_deg_full_out, void* stream);
/* v0 = d / tree_sum(d) (d_v0 NULL) or the explicit d_v0 (n doubles, see
 * gpic_cluster), then the device-resident loop. d_hist holds nlocal x
 * max_iter doubles, d_vout nlocal x n (every shard ends with the same full
 * embedding), h_ctl nlocal control blocks. Synchronous. */
int gpic_comm_iterate(gpic_comm* comm, const gpic_shard* shards, int32_t nlocal, double eps,
                      int32_t max_iter, const double* d_v0, double* d_hist, double* d_vout,
                      gpic_ctl* h_ctl, void* stream);

/* ---- batched small-n PIC (Experiment II: cli.py:230-256)
 * `count` independent problems of n_b = h_offsets[b+1] - h_offsets[b]
 * (1..4096) points each, all with d features, concatenated row-major in
 * d_x. One CTA runs one whole problem in fp64 (the reference's operation
 * order) — affinity, degrees, W, v0, power iteration — then the k-means.
 * Per problem: h_eps[b] (resolved epsilon), h_first[b] + h_uniforms[b*(k-1)
 * ...] (its k-means PCG64 draws), outputs d_labels / d_v at its offset,
 * d_hist[b*max_iter ...], and its control block h_ctl[b] (status, iter,
 * converged, error index) — a failing problem does not stop the others.
 * Synchronous. */
int64_t gpic_batch_workspace_bytes(const int64_t* h_offsets, int32_t count, int32_t d, int32_t k,
                                   int32_t max_iter);
int gpic_cluster_batch(const double* d_x, const int64_t* h_offsets, int32_t count, int32_t d,
                       double sigma, int32_t kind, int32_t k, const double* h_eps,
                       int32_t max_iter, const int64_t* h_first, const double* h_uniforms,
                       int64_t* d_labels, double* d_v, double* d_hist, gpic_ctl* h_ctl,
                       void* d_work, int64_t work_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GPIC_H */
