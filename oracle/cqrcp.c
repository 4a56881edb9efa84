/*
 * cqrcp.c — the oracle's rank-k column-pivoted Householder QR (O4a) as plain C,
 * parallel across columns with OpenMP.  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load it (through oracle/fast.py).  It shares no code, header or constant with the
 * CUDA path (paper_2012_00706_b200/) and is compiled by build() only so that the
 * checker exists.
 *
 * It is a line-by-line restatement of oracle/qrcp.py::qrcp_householder for one
 * shard (formation "fma", the right-looking form), written so that every column's
 * arithmetic happens in exactly the order the numpy oracle uses — the two are pinned
 * bit for bit against each other by tests/test_oracle_c.py — and so that the result
 * does not depend on the thread count (threads only split the set of columns).
 *
 * What is computed (PAPER.md, P:L = line L):
 *   Algorithm 2 line 4, Eq. (6)-(7): A_L Z = Q R, rank k,
 *   pivot = the largest remaining column norm (ties: lowest original index),
 *   in the paper's simulated low precision: fp16/fp32 storage, fp32
 *   arithmetic, the working matrix re-stored (rounded to the storage format) every
 *   nb steps (reading R4), R rows normalised to R_jj >= 0.
 *   update = 0 ("fma"):  W <- fl32(W - v f)        one rounding (emulated in fp64 as
 *                                                  the numpy oracle does)
 *   update = 1 ("rne"):  W <- fl32(W - fl32(v f))  every operation rounded
 *   acc = 0 ("chain8"):  8-row fp32 FMA chains, group partials added in fp64 (R5)
 *   acc = 1 ("seq64"):   exact products added in fp64 in increasing row order
 *   fmt = 64: the same algorithm in fp64 (Algorithm 1), no storage rounding.
 *   Tolerance stop (reading R8): before step j >= 1, stop when
 *   sqrt(sum_{i >= j} s_i) <= eps ||A_L||_F.
 *
 * Compile with -ffp-contract=off (no fused multiply-add anywhere): every operation is
 * the IEEE operation written.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <fenv.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* fl16(x): round-to-nearest-even of x to IEEE binary16 (Table 1; reading R1),
 * returned as a float.  The quantum of x's binade is 2^(e-11) with x = f 2^e,
 * f in [0.5, 1) (frexp), floored at the subnormal quantum 2^-24; x / q is then an exact
 * power-of-two scaling and nearbyint() rounds half to even (the default rounding mode). */
static float round_half(float xf) {
  const double x = (double)xf;
  if (x == 0.0 || isnan(x) || isinf(x)) return xf;
  int e;
  frexp(fabs(x), &e);
  int qe = e - 11;
  if (qe < -24) qe = -24;
  const double q = ldexp(1.0, qe);
  const double r = nearbyint(x / q) * q;
  if (fabs(r) > 65504.0) return x > 0 ? INFINITY : -INFINITY;
  return (float)r;
}

/* The working matrix, column-major with leading dimension m8; one of the two is set. */
typedef struct {
  float* f;
  double* d;
  int64_t ld;
} Work;

static inline double wget(const Work* W, int64_t r, int64_t c) {
  return W->f ? (double)W->f[c * W->ld + r] : W->d[c * W->ld + r];
}

/* column sums (s_i, w_i) of one column over rows [g0, m8): rows < jl count as 0 */
static void reduce_col(const Work* W, int64_t i, int64_t j, int64_t jl, int64_t g0, int64_t m8, int acc,
                       double* s_out, double* w_out) {
  if (acc == 1) {
    /* seq64: running fp64 sum of the exact products, first term first (np.add.accumulate) */
    double s = 0.0, w = 0.0;
    for (int64_t r = g0; r < m8; ++r) {
      const double x = r < jl ? 0.0 : wget(W, r, i);
      const double u = r < jl ? 0.0 : wget(W, r, j);
      const double ps = x * x, pw = x * u;
      if (r == g0) { s = ps; w = pw; }
      else { s = s + ps; w = w + pw; }
    }
    *s_out = s;
    *w_out = w;
    return;
  }
  /* chain8: per 8-row group a working-precision chain p = x0 y0; p = fl(xi yi + p),
   * then the group partials added in fp64 in group order */
  double s = 0.0, w = 0.0;
  for (int64_t g = g0; g < m8; g += 8) {
    double as, aw;
    if (W->f) {
      float cs = 0.f, cw = 0.f;
      for (int q = 0; q < 8; ++q) {
        const int64_t r = g + q;
        const double x = r < jl ? 0.0 : (double)W->f[i * W->ld + r];
        const double u = r < jl ? 0.0 : (double)W->f[j * W->ld + r];
        if (q == 0) { cs = (float)(x * x); cw = (float)(x * u); }
        else { cs = (float)(x * x + (double)cs); cw = (float)(x * u + (double)cw); }
      }
      as = (double)cs;
      aw = (double)cw;
    } else {
      double cs = 0.0, cw = 0.0;
      for (int q = 0; q < 8; ++q) {
        const int64_t r = g + q;
        const double x = r < jl ? 0.0 : W->d[i * W->ld + r];
        const double u = r < jl ? 0.0 : W->d[j * W->ld + r];
        if (q == 0) { cs = x * x; cw = x * u; }
        else { cs = x * x + cs; cw = x * u + cw; }
      }
      as = cs;
      aw = cw;
    }
    if (g == g0) { s = as; w = aw; }
    else { s = s + as; w = w + aw; }
  }
  *s_out = s;
  *w_out = w;
}

static void swap_cols(Work* W, int64_t a, int64_t b, int64_t m8) {
  if (W->f) {
    float* x = W->f + a * W->ld;
    float* y = W->f + b * W->ld;
    for (int64_t r = 0; r < m8; ++r) { float t = x[r]; x[r] = y[r]; y[r] = t; }
  } else {
    double* x = W->d + a * W->ld;
    double* y = W->d + b * W->ld;
    for (int64_t r = 0; r < m8; ++r) { double t = x[r]; x[r] = y[r]; y[r] = t; }
  }
}

static double seqsum(const double* x, int64_t n) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s = i == 0 ? x[0] : s + x[i];
  return s;
}

/*
 * AL: m x n column-major (ld = m) values already rounded to the storage format.
 * fmt: 16, 32 or 64.  Outputs: perm (n, 0-based original index per position),
 * R (k_max x n row-major, pivoted order; rows >= k_out untouched), top2 (k_max x 2),
 * resid (k_max + 1; resid_len = entries written), k_out, status (0 ok, 1 underflow),
 * normAL, maxnorm0.  Returns 0, or -1 on bad arguments / allocation failure.
 */
int oracle_qrcp(const double* AL, int64_t m, int64_t n, int32_t k_max, int32_t fmt, int32_t nb, double eps,
                int32_t update, int32_t acc, int32_t nthreads, int32_t* perm, double* R, double* top2,
                double* resid, int32_t* resid_len, int32_t* k_out, int32_t* status, double* normAL,
                double* maxnorm0) {
  if (m < 1 || n < 1 || k_max < 1 || k_max > n || k_max > m || nb < 1) return -1;
  if (fmt != 16 && fmt != 32 && fmt != 64) return -1;
  fesetround(FE_TONEAREST);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  const int64_t m8 = (m + 7) / 8 * 8;
  Work W = {0, 0, m8};
  if (fmt == 64) W.d = (double*)calloc((size_t)(m8 * n), sizeof(double));
  else W.f = (float*)calloc((size_t)(m8 * n), sizeof(float));
  double* vn = (double*)malloc(sizeof(double) * n);
  double* s = (double*)malloc(sizeof(double) * n);
  double* w = (double*)malloc(sizeof(double) * n);
  double* x = (double*)malloc(sizeof(double) * n);
  double* Rraw = (double*)malloc(sizeof(double) * n);
  double* fv = (double*)malloc(sizeof(double) * n);
  double* v = (double*)malloc(sizeof(double) * m8);
  if ((!W.f && !W.d) || !vn || !s || !w || !x || !Rraw || !fv || !v) {
    free(W.f); free(W.d); free(vn); free(s); free(w); free(x); free(Rraw); free(fv); free(v);
    return -1;
  }
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c)
    for (int64_t r = 0; r < m; ++r) {
      if (W.f) W.f[c * m8 + r] = (float)AL[c * m + r];
      else W.d[c * m8 + r] = AL[c * m + r];
    }
  for (int64_t c = 0; c < n; ++c) perm[c] = (int32_t)c;
  /* initial exact norms^2 (acc seq64: sequential fp64; chain8 model: numpy's np.sum
   * is replaced by the same sequential fp64 sum — fp16 squares add exactly in fp64) */
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < n; ++c) {
    double t = 0.0;
    for (int64_t r = 0; r < m; ++r) {
      const double a = AL[c * m + r];
      t = r == 0 ? a * a : t + a * a;
    }
    vn[c] = t;
  }
  *normAL = sqrt(seqsum(vn, n));
  double mx = vn[0];
  for (int64_t c = 1; c < n; ++c) mx = vn[c] > mx ? vn[c] : mx;
  *maxnorm0 = sqrt(mx);
  const double tiny = fmt == 64 ? 2.2250738585072014e-308 : 1.1754943508222875e-38;
  int32_t kk = k_max, st = 0, nres = 0;
  for (int64_t j = 0; j < k_max; ++j) {
    const int64_t jl = j, g0 = (j / 8) * 8;
    /* 1. pivot: max vn over i >= j, ties -> lowest original index */
    double best = vn[j];
    for (int64_t i = j + 1; i < n; ++i) best = vn[i] > best ? vn[i] : best;
    int64_t p = -1;
    for (int64_t i = j; i < n; ++i)
      if (vn[i] == best && (p < 0 || perm[i] < perm[p])) p = i;
    {
      double a1 = -INFINITY, a2 = -INFINITY;
      for (int64_t i = j; i < n; ++i) {
        if (vn[i] > a1) { a2 = a1; a1 = vn[i]; }
        else if (vn[i] > a2) a2 = vn[i];
      }
      top2[2 * j] = sqrt(a1 > 0.0 ? a1 : 0.0);
      top2[2 * j + 1] = (n - j > 1) ? sqrt(a2 > 0.0 ? a2 : 0.0) : 0.0;
    }
    if (p != j) {
      swap_cols(&W, j, p, m8);
      for (int64_t r = 0; r < j; ++r) { double t = R[r * n + j]; R[r * n + j] = R[r * n + p]; R[r * n + p] = t; }
      int32_t tp = perm[j]; perm[j] = perm[p]; perm[p] = tp;
      double tv = vn[j]; vn[j] = vn[p]; vn[p] = tv;
    }
    /* 2. store point: W(j:, j:) <- fl_L(W) every nb steps */
    if (j > 0 && j % nb == 0 && fmt == 16) {
#pragma omp parallel for schedule(static)
      for (int64_t c = j; c < n; ++c)
        for (int64_t r = jl; r < m8; ++r) W.f[c * m8 + r] = round_half(W.f[c * m8 + r]);
    }
    /* 3. s_i = ||W(j:, i)||^2, w_i = W(j:, i)^T u, u = W(j:, j) */
#pragma omp parallel for schedule(static)
    for (int64_t c = j; c < n; ++c) reduce_col(&W, c, j, jl, g0, m8, acc, &s[c], &w[c]);
    resid[nres++] = sqrt(seqsum(s + j, n - j));
    if (eps > 0.0 && j > 0 && resid[nres - 1] <= eps * *normAL) { kk = (int32_t)j; break; }
    for (int64_t c = j; c < n; ++c) x[c] = wget(&W, jl, c);
    const double sj = s[j];
    if (!(sj >= tiny)) { st = 1; kk = (int32_t)j; break; }
    /* 4. reflector */
    const double u0 = x[j];
    const double beta = -copysign(sqrt(sj), u0);
    const double cc = 1.0 / (u0 - beta);
    for (int64_t r = jl; r < m8; ++r) {
      const double vv = wget(&W, r, j) * cc;
      v[r] = fmt == 64 ? vv : (double)(float)vv;
    }
    v[jl] = 1.0;
    const double sgn = copysign(1.0, beta);
    for (int64_t c = j; c < n; ++c) {
      Rraw[c] = w[c] / beta;
      const double fx = x[c] - Rraw[c];
      fv[c] = fmt == 64 ? fx : (double)(float)fx;
      const double rr = Rraw[c] * sgn;
      R[j * n + c] = fmt == 64 ? rr : (double)(float)rr;
    }
    for (int64_t c = j + 1; c < n; ++c) vn[c] = s[c] - Rraw[c] * Rraw[c];
    /* 5. update W(j:, j:) <- fl(W - v f^T) */
#pragma omp parallel for schedule(static)
    for (int64_t c = j; c < n; ++c) {
      if (W.f) {
        float* col = W.f + c * m8;
        const float f = (float)fv[c];
        for (int64_t r = jl; r < m8; ++r) {
          const float vr = (float)v[r];
          if (update == 0) col[r] = (float)((double)(-vr) * (double)f + (double)col[r]);
          else {
            const float pr = vr * f;
            col[r] = col[r] - pr;
          }
        }
      } else {
        double* col = W.d + c * m8;
        const double f = fv[c];
        for (int64_t r = jl; r < m8; ++r) {
          if (update == 0) col[r] = (-v[r]) * f + col[r];
          else col[r] = col[r] - v[r] * f;
        }
      }
    }
  }
  if (st == 0 && kk == k_max && k_max < (m < n ? m : n)) {
    const int64_t j = k_max, jl = j, g0 = (j / 8) * 8;
#pragma omp parallel for schedule(static)
    for (int64_t c = j; c < n; ++c) reduce_col(&W, c, j, jl, g0, m8, acc, &s[c], &w[c]);
    resid[nres++] = sqrt(seqsum(s + j, n - j));
  }
  *k_out = kk;
  *status = st;
  *resid_len = nres;
  free(W.f); free(W.d); free(vn); free(s); free(w); free(x); free(Rraw); free(fv); free(v);
  return 0;
}
