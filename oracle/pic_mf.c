/*
 * pic_mf.c -- fp64 MATRIX-FREE restatement of the reference PIC pipeline.
 * TEST INFRASTRUCTURE ONLY: built into oracle/_build/libpicmf.so and called
 * by tests/, tests/golden/make_config_fixtures.py and bench.py's CPU legs as
 * the checker. The product path never links or loads it.
 *
 * Why it exists (BASELINE.md §2 "Parity oracle for config 5"):
 * the reference materialises A and W as dense fp64 n x n matrices
 * (affinity.py:107-127), 80 GB at n = 100k and 8 TB at n = 1M, so at the
 * benchmark configs it cannot run on any host here. This file recomputes
 * each affinity row on the fly instead, with the reference's arithmetic:
 *
 *   - affinity.py:96-101  d2_ij = sum over features f = 0..m-1, in that
 *     order, of (x_if - x_jf)^2 (each product rounded, then added: compiled
 *     with -ffp-contract=off so no FMA merges the two), then
 *     a_ij = exp(d2_ij * (-1 / (2 sigma^2))).  exp() is pic_exp below
 *     (<= 1 ulp from a correctly rounded exp; numpy's differs by <= 1 ulp).
 *   - affinity.py:102-103 the diagonal a_ii = 0.
 *   - affinity.py:41-53,88-95 the cosine kind: a_ij = max(0, x_i.x_j /
 *     (|x_i| |x_j|)), dots and norms accumulated feature by feature.
 *   - affinity.py:113-119 deg_i = sum_j a_ij (ZeroDegree is the caller's).
 *   - affinity.py:122-127 + serial.py:121 (W v)_i = sum_j (a_ij / deg_i) v_j.
 *
 * Each row is an independent task (pthreads pulling row chunks from an
 * atomic counter; no libgomp in this image); the sum over j runs in a fixed
 * order per row, so results do not depend on the thread count. The reference sums with numpy's pairwise summation and
 * OpenBLAS; differences are at the 1e-16 relative level per entry
 * (validated against the reference itself on configs 1-2 to <= 1e-12 in
 * tests/test_oracle_mf.py, fixtures made by tests/golden/make_golden.py).
 */
#include <math.h>
#include <pthread.h>
#include <unistd.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* exp(x) in fp64, branch-free so gcc vectorises the row loop.
 * Cody-Waite reduction x = k ln2 + r, |r| <= ln2/2, degree-13 Taylor
 * polynomial (truncation < 2^-60), scaled by 2^k in two steps so that
 * subnormal results (x in [-745.13, -708.4]) round like libm's. */
static inline double pic_exp(double x) {
  const double ln2_hi = 6.93147180369123816490e-01;
  const double ln2_lo = 1.90821492927058770002e-10;
  const double inv_ln2 = 1.44269504088896338700e+00;
  double xc = x < -746.0 ? -746.0 : (x > 709.0 ? 709.0 : x);
  /* round to nearest via the 1.5*2^52 shifter (vectorises; no -ffast-math) */
  const double shifter = 6755399441055744.0;
  double kf = (xc * inv_ln2 + shifter) - shifter;
  double r = (xc - kf * ln2_hi) - kf * ln2_lo;
  double p = 1.0 / 6227020800.0;           /* 1/13! */
  p = p * r + 1.0 / 479001600.0;           /* 1/12! */
  p = p * r + 1.0 / 39916800.0;
  p = p * r + 1.0 / 3628800.0;
  p = p * r + 1.0 / 362880.0;
  p = p * r + 1.0 / 40320.0;
  p = p * r + 1.0 / 5040.0;
  p = p * r + 1.0 / 720.0;
  p = p * r + 1.0 / 120.0;
  p = p * r + 1.0 / 24.0;
  p = p * r + 1.0 / 6.0;
  p = p * r + 0.5;
  p = p * r + 1.0;
  p = p * r + 1.0;
  /* 2^k = 2^k1 * 2^k2 with k1 = floor(k/2): each factor is a normal number.
   * Exponent bits are built from the shifter's mantissa (AVX2 has 64-bit
   * integer add/shift but no double -> int64 conversion). */
  const double k1f = __builtin_floor(kf * 0.5), k2f = kf - k1f;
  const double t1 = k1f + (shifter + 1023.0), t2 = k2f + (shifter + 1023.0);
  int64_t b1, b2, bs;
  __builtin_memcpy(&b1, &t1, 8);
  __builtin_memcpy(&b2, &t2, 8);
  __builtin_memcpy(&bs, &shifter, 8);
  b1 = (b1 - bs) << 52;
  b2 = (b2 - bs) << 52;
  double s1, s2;
  __builtin_memcpy(&s1, &b1, 8);
  __builtin_memcpy(&s2, &b2, 8);
  double out = (p * s1) * s2;
  return x < -746.0 ? 0.0 : out;
}

typedef double v4d __attribute__((vector_size(32), aligned(8)));
#define PW 16 /* columns per panel: 4 vectors of 4 doubles */

/* Column panels of X: xp[((j / PW) * m + f) * PW + j % PW] = x[j, f], zero
 * padded to a multiple of PW columns, so one row pair x one panel keeps its
 * 2 x 16 partial sums in registers across the whole feature loop. */
static double *pack_panels(const double *x, int64_t n, int32_t m) {
  const int64_t np = (n + PW - 1) / PW;
  double *xp = (double *)aligned_alloc(64, sizeof(double) * (size_t)(np * m * PW));
  memset(xp, 0, sizeof(double) * (size_t)(np * m * PW));
  for (int64_t j = 0; j < n; ++j)
    for (int32_t f = 0; f < m; ++f) xp[((j / PW) * m + f) * PW + j % PW] = x[(size_t)j * m + f];
  return xp;
}

/* cosine norms (affinity.py:41-53): sqrt of the feature-ordered sum of squares */
static void cos_norms(const double *x, int64_t n, int32_t m, double *nrm) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int32_t f = 0; f < m; ++f) s += x[(size_t)i * m + f] * x[(size_t)i * m + f];
    nrm[i] = sqrt(s);
  }
}

/* For rows xa, xb and panels [p0, p1): o[j] = sum_f (x_f - col_jf)^2 in
 * feature order (RBF, affinity.py:96-100) or sum_f x_f col_jf (cosine,
 * affinity.py:89-91). Products are rounded before the add (no FMA). */
static void pair_rbf(const double *xp, const double *xa, const double *xb, int32_t m,
                     int64_t p0, int64_t p1, double *oa, double *ob) {
  for (int64_t p = p0; p < p1; ++p) {
    const double *col = xp + (size_t)p * m * PW;
    v4d a0 = {0}, a1 = {0}, a2 = {0}, a3 = {0}, b0 = {0}, b1 = {0}, b2 = {0}, b3 = {0};
    for (int32_t f = 0; f < m; ++f) {
      const v4d c0 = *(const v4d *)(col + f * PW), c1 = *(const v4d *)(col + f * PW + 4);
      const v4d c2 = *(const v4d *)(col + f * PW + 8), c3 = *(const v4d *)(col + f * PW + 12);
      const double u = xa[f], w = xb[f];
      v4d d;
      d = u - c0; a0 += d * d;  d = u - c1; a1 += d * d;
      d = u - c2; a2 += d * d;  d = u - c3; a3 += d * d;
      d = w - c0; b0 += d * d;  d = w - c1; b1 += d * d;
      d = w - c2; b2 += d * d;  d = w - c3; b3 += d * d;
    }
    double *qa = oa + (p - p0) * PW, *qb = ob + (p - p0) * PW;
    *(v4d *)qa = a0; *(v4d *)(qa + 4) = a1; *(v4d *)(qa + 8) = a2; *(v4d *)(qa + 12) = a3;
    *(v4d *)qb = b0; *(v4d *)(qb + 4) = b1; *(v4d *)(qb + 8) = b2; *(v4d *)(qb + 12) = b3;
  }
}

static void pair_dot(const double *xp, const double *xa, const double *xb, int32_t m,
                     int64_t p0, int64_t p1, double *oa, double *ob) {
  for (int64_t p = p0; p < p1; ++p) {
    const double *col = xp + (size_t)p * m * PW;
    v4d a0 = {0}, a1 = {0}, a2 = {0}, a3 = {0}, b0 = {0}, b1 = {0}, b2 = {0}, b3 = {0};
    for (int32_t f = 0; f < m; ++f) {
      const v4d c0 = *(const v4d *)(col + f * PW), c1 = *(const v4d *)(col + f * PW + 4);
      const v4d c2 = *(const v4d *)(col + f * PW + 8), c3 = *(const v4d *)(col + f * PW + 12);
      const double u = xa[f], w = xb[f];
      a0 += u * c0; a1 += u * c1; a2 += u * c2; a3 += u * c3;
      b0 += w * c0; b1 += w * c1; b2 += w * c2; b3 += w * c3;
    }
    double *qa = oa + (p - p0) * PW, *qb = ob + (p - p0) * PW;
    *(v4d *)qa = a0; *(v4d *)(qa + 4) = a1; *(v4d *)(qa + 8) = a2; *(v4d *)(qa + 12) = a3;
    *(v4d *)qb = b0; *(v4d *)(qb + 4) = b1; *(v4d *)(qb + 8) = b2; *(v4d *)(qb + 12) = b3;
  }
}

/* accumulator -> affinity values in place, columns [j0, j0 + w) of row i */
static void finish_row(double *o, int64_t w, int64_t i, int64_t j0, double scale, int cosine,
                       const double *nrm) {
  if (cosine) {
    const double ni = nrm[i];
#pragma omp simd
    for (int64_t j = 0; j < w; ++j) {
      double c = o[j] / (ni * nrm[j0 + j]);
      o[j] = c > 0.0 ? c : 0.0; /* affinity.py:93-94 */
    }
  } else {
#pragma omp simd
    for (int64_t j = 0; j < w; ++j) o[j] = pic_exp(o[j] * scale); /* affinity.py:101 */
  }
  if (i >= j0 && i < j0 + w) o[i - j0] = 0.0; /* affinity.py:102-103 */
}

static double sum_seq(const double *a, int64_t w) {
  /* 4 interleaved partials, fixed order: deterministic and vectorisable */
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int64_t j = 0;
  for (; j + 4 <= w; j += 4) { s0 += a[j]; s1 += a[j + 1]; s2 += a[j + 2]; s3 += a[j + 3]; }
  for (; j < w; ++j) s0 += a[j];
  return (s0 + s1) + (s2 + s3);
}

static double dot_seq(const double *a, const double *b, int64_t w) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int64_t j = 0;
  for (; j + 4 <= w; j += 4) {
    s0 += a[j] * b[j]; s1 += a[j + 1] * b[j + 1];
    s2 += a[j + 2] * b[j + 2]; s3 += a[j + 3] * b[j + 3];
  }
  for (; j < w; ++j) s0 += a[j] * b[j];
  return (s0 + s1) + (s2 + s3);
}

/*
 * mode 0: out[i] = deg_i = sum_j a_ij                        (affinity.py:113-115)
 * mode 1: out[i] = sum_j (a_ij / deg_i) v_j                  (affinity.py:126, serial.py:121)
 * rows [lo, hi) only (the caller may sample rows); sigma <= 0 selects cosine.
 */
typedef struct {
  const double *x, *xp, *nrm, *deg, *v;
  int64_t n, lo, hi;
  int32_t m;
  int mode, cosine;
  double scale;
  double *out;
  int64_t next; /* atomic row cursor */
} job_t;

/*
 * Optional block skip (picmf_set_skip), for the n = 1M fixture only: skip[S *
 * nb + T] = 1 marks a pair of BLK-row / BLK-column blocks whose every entry
 * is proved (by the caller's fp64 projection bound, oracle/pic_mf.py) to be
 * below e^-70. Such a block's sum is <= BLK e^-70 ~ 4e-28 per row, far below
 * half an ulp of any row sum that contains a block with real neighbours
 * (>= 1e-8 here), so adding it or not leaves the fp64 row sum bit for bit
 * unchanged — whether it comes before or after the significant blocks (a
 * tiny prefix is absorbed by the first significant block sum). Checked
 * against the unskipped pass on config 3 (tests/test_oracle_mf.py).
 */
static const uint8_t *g_skip = NULL;
static int64_t g_skip_nb = 0;
void picmf_set_skip(const uint8_t *skip, int64_t nb) {
  g_skip = skip;
  g_skip_nb = nb;
}

static int n_threads(void) {
  const char *e = getenv("PICMF_THREADS");
  long t = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  return t < 1 ? 1 : (t > 512 ? 512 : (int)t);
}

#define BLK 1024 /* columns per block (64 panels): both rows' partials stay in L1 */

static void *worker(void *arg) {
  job_t *jb = (job_t *)arg;
  double *buf = (double *)aligned_alloc(64, sizeof(double) * 2 * BLK);
  const int64_t n = jb->n;
  for (;;) {
    const int64_t i0 = __atomic_fetch_add(&jb->next, 2, __ATOMIC_RELAXED);
    if (i0 >= jb->hi) break;
    const int64_t ia = i0, ib = i0 + 1 < jb->hi ? i0 + 1 : i0; /* odd tail: pair with itself */
    const double *xa = jb->x + (size_t)ia * jb->m, *xb = jb->x + (size_t)ib * jb->m;
    double acc[2] = {0.0, 0.0};
    for (int64_t j0 = 0; j0 < n; j0 += BLK) {
      const int64_t w = j0 + BLK < n ? BLK : n - j0;
      if (g_skip != NULL && jb->mode != 2 && g_skip[(ia / BLK) * g_skip_nb + j0 / BLK] &&
          g_skip[(ib / BLK) * g_skip_nb + j0 / BLK])
        continue; /* both rows' blocks proved negligible (see picmf_set_skip) */
      double *oa = buf, *ob = buf + BLK;
      if (jb->cosine)
        pair_dot(jb->xp, xa, xb, jb->m, j0 / PW, (j0 + w + PW - 1) / PW, oa, ob);
      else
        pair_rbf(jb->xp, xa, xb, jb->m, j0 / PW, (j0 + w + PW - 1) / PW, oa, ob);
      for (int r = 0; r < 2; ++r) {
        const int64_t i = r ? ib : ia;
        if (r && ib == ia) break;
        double *o = r ? ob : oa;
        finish_row(o, w, i, j0, jb->scale, jb->cosine, jb->nrm);
        if (jb->mode == 2) {
          memcpy(jb->out + (size_t)(i - jb->lo) * n + j0, o, sizeof(double) * (size_t)w);
        } else if (jb->mode == 0) {
          acc[r] += sum_seq(o, w);
        } else {
          const double di = jb->deg[i];
          for (int64_t j = 0; j < w; ++j) o[j] = o[j] / di; /* W = A / deg (affinity.py:126) */
          acc[r] += dot_seq(o, jb->v + j0, w);
        }
      }
    }
    if (jb->mode != 2) {
      jb->out[ia - jb->lo] = acc[0];
      if (ib != ia) jb->out[ib - jb->lo] = acc[1];
    }
  }
  free(buf);
  return NULL;
}

/*
 * mode 0: out[i] = deg_i = sum_j a_ij                        (affinity.py:113-115)
 * mode 1: out[i] = sum_j (a_ij / deg_i) v_j                  (affinity.py:126, serial.py:121)
 * mode 2: out[i, :] = a_i (row of A)                          (affinity.py:96-103)
 * rows [lo, hi) only (the caller may sample rows); sigma <= 0 selects cosine.
 */
static void pass(const double *x, int64_t n, int32_t m, double sigma, int64_t lo, int64_t hi,
                 int mode, const double *deg, const double *v, double *out) {
  job_t jb;
  memset(&jb, 0, sizeof jb);
  jb.cosine = !(sigma > 0.0);
  jb.scale = jb.cosine ? 0.0 : -1.0 / (2.0 * sigma * sigma); /* affinity.py:101 */
  jb.x = x; jb.n = n; jb.m = m; jb.lo = lo; jb.hi = hi; jb.mode = mode;
  jb.deg = deg; jb.v = v; jb.out = out; jb.next = lo;
  double *xp = pack_panels(x, n, m);
  double *nrm = NULL;
  if (jb.cosine) {
    nrm = (double *)malloc(sizeof(double) * (size_t)n);
    cos_norms(x, n, m, nrm);
  }
  jb.xp = xp; jb.nrm = nrm;
  int nt = n_threads();
  if ((hi - lo + 1) / 2 < nt) nt = (int)((hi - lo + 1) / 2) > 0 ? (int)((hi - lo + 1) / 2) : 1;
  pthread_t th[512];
  for (int t = 1; t < nt; ++t) pthread_create(&th[t], NULL, worker, &jb);
  worker(&jb);
  for (int t = 1; t < nt; ++t) pthread_join(th[t], NULL);
  free(nrm);
  free(xp);
}

/* deg[0 : hi-lo] = row sums of A for rows [lo, hi) */
void picmf_degree(const double *x, int64_t n, int32_t m, double sigma, int64_t lo, int64_t hi,
                  double *deg) {
  pass(x, n, m, sigma, lo, hi, 0, NULL, NULL, deg);
}

/* y[0 : hi-lo] = (W v)[lo:hi], W = D^-1 A, deg the full degree vector */
void picmf_matvec(const double *x, int64_t n, int32_t m, double sigma, int64_t lo, int64_t hi,
                  const double *deg, const double *v, double *y) {
  pass(x, n, m, sigma, lo, hi, 1, deg, v, y);
}

/* rows [lo, hi) of A itself, (hi-lo) x n, for small parity checks */
void picmf_rows(const double *x, int64_t n, int32_t m, double sigma, int64_t lo, int64_t hi,
                double *a) {
  pass(x, n, m, sigma, lo, hi, 2, NULL, NULL, a);
}

double picmf_exp(double x) { return pic_exp(x); }

int64_t picmf_block(void) { return BLK; }
