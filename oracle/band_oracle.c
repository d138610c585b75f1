/*
 * band_oracle.c -- CPU restatement of the reference's band Cholesky, solve and
 * residual.  TEST INFRASTRUCTURE ONLY: this is the checker the CUDA path is
 * compared against.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path never
 * calls it and has no CPU fallback.
 *
 * Pinning: bco_factor_reference reproduces the reference's
 * factor_reference BIT FOR BIT (same products, exactly rounded sums, same sqrt and
 * division); tests/test_oracle.py checks it against SHA-256 fingerprints and
 * arrays produced by the reference itself (tests/golden/make_golden.py).
 *
 * Storage: LAPACK lower band, element (i,j) at data[j*ldab + (i-j)]
 * (pkg/src/bandchol/core.py:1-19, :34-44).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define AT(p, ld, i, j) (p)[(int64_t)(j) * (ld) + ((i) - (j))]

/* Exactly rounded sum of x[0..n) -- the published Shewchuk/"msum" algorithm with
 * the round-half-even fix-up, which is what math.fsum computes (the reference's
 * inner-product accumulator, reference.py:51).  Non-finite inputs fall back to
 * the plain sum (they never occur on SPD test inputs). */
double bco_fsum(const double* x, int64_t n) {
  double partials[256];
  int np = 0;
  double special = 0.0;
  int nonfinite = 0;
  for (int64_t t = 0; t < n; ++t) {
    double v = x[t];
    if (!isfinite(v)) { nonfinite = 1; special += v; continue; }
    int i = 0;
    for (int p = 0; p < np; ++p) {
      double y = partials[p];
      if (fabs(v) < fabs(y)) { double tmp = v; v = y; y = tmp; }
      double hi = v + y;
      double lo = y - (hi - v);
      if (lo != 0.0) partials[i++] = lo;
      v = hi;
    }
    np = i;
    partials[np++] = v;
    if (np >= 255) return NAN;  /* cannot happen for finite doubles */
  }
  if (nonfinite) return special;
  if (np == 0) return 0.0;
  int k = np;
  double hi = partials[--k];
  double lo = 0.0;
  while (k > 0) {
    double xx = hi;
    double y = partials[--k];
    hi = xx + y;
    double yr = hi - xx;
    lo = y - yr;
    if (lo != 0.0) break;
  }
  if (k > 0 && ((lo < 0.0 && partials[k - 1] < 0.0) || (lo > 0.0 && partials[k - 1] > 0.0))) {
    double y = lo * 2.0;
    double xx = hi + y;
    double yr = xx - hi;
    if (y == yr) hi = xx;
  }
  return hi;
}

/* Left-looking factorization, reference.py:32-63.  Row i, column j in
 * [max(0,i-k), i]: t = fsum_l L(i,l)*L(j,l) over l in [max(0,i-k), j-1];
 * pivot = A(i,i)-t must satisfy `pivot > 0` (NaN fails) else the global column i
 * is returned; L(i,i) = sqrt(pivot); L(i,j) = (A(i,j)-t)/L(j,j).
 * Returns -1 on success. */
int64_t bco_factor_reference(int64_t n, int64_t kd, int64_t ldab, double* a) {
  double* prod = (double*)malloc(sizeof(double) * (size_t)(kd + 1));
  if (!prod) return -2;
  for (int64_t i = 0; i < n; ++i) {
    int64_t lo = i - kd > 0 ? i - kd : 0;
    for (int64_t j = lo; j <= i; ++j) {
      int64_t cnt = j - lo;
      for (int64_t l = 0; l < cnt; ++l) prod[l] = AT(a, ldab, i, lo + l) * AT(a, ldab, j, lo + l);
      double t = cnt ? bco_fsum(prod, cnt) : 0.0;
      if (i == j) {
        double pivot = AT(a, ldab, i, i) - t;
        if (!(pivot > 0.0)) { free(prod); return i; }
        AT(a, ldab, i, i) = sqrt(pivot);
      } else {
        AT(a, ldab, i, j) = (AT(a, ldab, i, j) - t) / AT(a, ldab, j, j);
      }
    }
  }
  free(prod);
  return -1;
}

/* Fast plain-double right-looking variant for the large configs (C3/C4 sizes,
 * where the exactly-rounded oracle is too slow).  Same recurrence, ordinary
 * rounding; agrees with bco_factor_reference to ~1e-15 scaled.  Failure column
 * semantics identical.  Returns -1 on success. */
int64_t bco_factor_plain(int64_t n, int64_t kd, int64_t ldab, double* a) {
  for (int64_t j = 0; j < n; ++j) {
    double pivot = AT(a, ldab, j, j);
    if (!(pivot > 0.0)) return j;
    double d = sqrt(pivot);
    AT(a, ldab, j, j) = d;
    int64_t m = (n - 1 - j) < kd ? (n - 1 - j) : kd;
    double* col = &AT(a, ldab, j, j);
    for (int64_t r = 1; r <= m; ++r) col[r] /= d;
#pragma omp parallel for schedule(static) if (m > 256)
    for (int64_t c = 1; c <= m; ++c) {
      double lc = col[c];
      double* tgt = &AT(a, ldab, j + c, j + c);
      for (int64_t r = c; r <= m; ++r) tgt[r - c] -= col[r] * lc;
    }
  }
  return -1;
}

/* Band solve L L^T x = b, core.py:216-240: forward sweep over rows
 * y[i] = (b[i] - sum_l L(i,l) y[l]) / L(i,i), backward sweep over columns
 * x[j] = (y[j] - sum_r L(r,j) x[r]) / L(j,j).  Returns -1, or the first column
 * whose diagonal is <= 0 (SingularFactor, core.py:227-230), checked before any
 * arithmetic like the reference. */
int64_t bco_solve(int64_t n, int64_t kd, int64_t ldab, const double* l, const double* b, double* x) {
  for (int64_t j = 0; j < n; ++j)
    if (AT(l, ldab, j, j) <= 0.0) return j;
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  if (!y) return -2;
  for (int64_t i = 0; i < n; ++i) {
    int64_t lo = i - kd > 0 ? i - kd : 0;
    double t = 0.0;
    for (int64_t c = lo; c < i; ++c) t += AT(l, ldab, i, c) * y[c];
    y[i] = (b[i] - t) / AT(l, ldab, i, i);
  }
  for (int64_t j = n - 1; j >= 0; --j) {
    int64_t m = (n - 1 - j) < kd ? (n - 1 - j) : kd;
    double t = 0.0;
    for (int64_t r = 1; r <= m; ++r) t += AT(l, ldab, j + r, j) * x[j + r];
    x[j] = (y[j] - t) / AT(l, ldab, j, j);
  }
  free(y);
  return -1;
}

/* ||A - L L^T||_F / ||A||_F over the band, off-diagonals weighted twice
 * (core.py:186-213).  (L L^T)(j+d, j) = sum_s L(j+d, j-s) L(j, j-s). */
double bco_residual(int64_t n, int64_t kd, int64_t lda, const double* a, int64_t ldl, const double* l) {
  double num = 0.0, den = 0.0;
#pragma omp parallel for reduction(+ : num, den) schedule(static)
  for (int64_t j = 0; j < n; ++j) {
    int64_t m = (n - 1 - j) < kd ? (n - 1 - j) : kd;
    for (int64_t d = 0; d <= m; ++d) {
      double r = 0.0;
      int64_t smax = kd - d < j ? kd - d : j;
      for (int64_t s = 0; s <= smax; ++s) r += AT(l, ldl, j + d, j - s) * AT(l, ldl, j, j - s);
      double av = AT(a, lda, j + d, j);
      double w = d == 0 ? 1.0 : 2.0;
      double diff = av - r;
      num += w * diff * diff;
      den += w * av * av;
    }
  }
  if (den == 0.0) return num == 0.0 ? 0.0 : INFINITY;
  return sqrt(num / den);
}

/* max over in-band entries of |x - y| / max(|y|, 1): the reference's parity
 * scale (pkg/tests/test_acceptance.py:49). */
double bco_max_scaled_diff(int64_t n, int64_t kd, int64_t ldx, const double* x, int64_t ldy, const double* y) {
  double worst = 0.0;
  for (int64_t j = 0; j < n; ++j) {
    int64_t m = (n - 1 - j) < kd ? (n - 1 - j) : kd;
    for (int64_t d = 0; d <= m; ++d) {
      double yv = AT(y, ldy, j + d, j);
      double s = fabs(yv) > 1.0 ? fabs(yv) : 1.0;
      double e = fabs(AT(x, ldx, j + d, j) - yv) / s;
      if (!(e <= worst)) worst = e;  /* NaN propagates as the worst value */
    }
  }
  return worst;
}
