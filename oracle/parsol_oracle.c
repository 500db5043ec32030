/*
 * parsol_oracle.c -- TEST INFRASTRUCTURE ONLY (see parsol_oracle.h).
 *
 * CPU restatement of the reference `parsol` partition solver, in plain C.
 * Each routine cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  The operation order is kept identical so results
 * are bit-for-bit those of the reference (pinned by tests/test_oracle.py
 * against oracle/_ref and tests/golden/).  Compile with -ffp-contract=off.
 *
 * The only deliberate departures:
 *   - Abd/Babd entry addressing uses a prefix table of block-row offsets
 *     (O(1)) instead of the reference's O(b) rescan
 *     (src/structmat.cpp:47-54); the addresses are the same.
 *   - Babd accepts the s = m, r = 0 layout that make() rejects
 *     (src/structmat.cpp:173-174) -- the BASELINE config 4 BVP layout.
 */
#include "parsol_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* Errc numbering, include/parsol/errors.hpp:12-35 */
enum {
  E_DimensionMismatch = 0,
  E_InvalidBandwidth,
  E_CornerForbidden,
  E_TooLargeForDense,
  E_InvalidParameter,
  E_ParseError,
  E_UnsupportedVersion,
  E_TooManyPartitions,
  E_UnsupportedKind,
  E_UnsupportedStructure,
  E_IndexOutOfRange,
  E_ZeroPivot,
  E_SingularBlock,
  E_SingularFactor,
  E_SingularReducedSystem,
};

static int fail(char* err, size_t errlen, int code, const char* fmt, ...) {
  if (err && errlen) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, errlen, fmt, ap);
    va_end(ap);
  }
  return 1 + code;
}

static int imax(int a, int b) { return a > b ? a : b; }
static int imin(int a, int b) { return a < b ? a : b; }

/* ------------------------------------------------------------------------ */
/* structmat: src/structmat.cpp                                              */
/* ------------------------------------------------------------------------ */

static size_t band_offset(int n, int s, int d) { /* src/structmat.cpp:34-38 */
  size_t off = 0;
  for (int b = -s; b < d; ++b) off += (size_t)(n - abs(b));
  return off;
}

static void abd_span(int n, int m, int s, int r, int b, int* c0, int* c1) { /* :41-45 */
  *c0 = imax(0, b * m - s);
  *c1 = imin(n, b * m + m + r);
}

size_t or_body_entry_count(int kind, int n, int m, int s, int r) { /* :64-84 */
  switch (kind) {
    case OR_BANDED: {
      size_t c = 0;
      for (int d = -s; d <= r; ++d) c += (size_t)(n - abs(d));
      return c;
    }
    case OR_BLOCKTRI: {
      int nb = n / m;
      return (size_t)(3 * nb - 2) * m * m;
    }
    case OR_ABD:
    case OR_BABD: {
      int nb = n / m;
      size_t off = 0;
      for (int q = 0; q < nb; ++q) {
        int c0, c1;
        abd_span(n, m, s, r, q, &c0, &c1);
        off += (size_t)m * (c1 - c0);
      }
      return off;
    }
    case OR_CIRCULANT:
      return (size_t)(s + r + 1) * n;
  }
  return 0;
}

int or_mat_prepare(or_mat* A, char* err, size_t errlen) { /* make(): :153-207 */
  A->abd_off = NULL;
  const int n = A->n, m = A->m, s = A->s, r = A->r;
  if (n <= 0) return fail(err, errlen, E_DimensionMismatch, "n must be positive");
  if (m <= 0) return fail(err, errlen, E_DimensionMismatch, "m must be positive");
  if (s < 0 || r < 0) return fail(err, errlen, E_InvalidBandwidth, "bandwidths must be non-negative");
  switch (A->kind) {
    case OR_BANDED:
      if (m != 1) return fail(err, errlen, E_DimensionMismatch, "scalar kinds require m = 1");
      if (s + r + 1 > n) return fail(err, errlen, E_InvalidBandwidth, "band wider than matrix");
      break;
    case OR_BLOCKTRI:
      if (n % m != 0) return fail(err, errlen, E_DimensionMismatch, "n must be a multiple of m");
      if (s != 1 || r != 1)
        return fail(err, errlen, E_InvalidBandwidth, "block tridiagonal requires s = r = 1");
      break;
    case OR_ABD:
    case OR_BABD: {
      if (n % m != 0) return fail(err, errlen, E_DimensionMismatch, "n must be a multiple of m");
      if (m < 2) return fail(err, errlen, E_DimensionMismatch, "ABD requires m >= 2");
      int ok = (s >= 1 && r >= 1 && s + r == m) || (A->kind == OR_BABD && s == m && r == 0);
      if (!ok) return fail(err, errlen, E_InvalidBandwidth, "ABD requires s,r >= 1 with s + r = m");
      if (n / m < 2) return fail(err, errlen, E_DimensionMismatch, "ABD requires at least 2 block rows");
      break;
    }
    default:
      return fail(err, errlen, E_UnsupportedKind, "oracle supports banded/blocktri/abd/babd");
  }
  if (A->kind == OR_BABD) {
    if (!A->corner) return fail(err, errlen, E_DimensionMismatch, "BABD requires a corner block");
    if (A->corner_rows < 1 || A->corner_cols < 1 || A->corner_rows > m || A->corner_cols > m)
      return fail(err, errlen, E_DimensionMismatch, "corner block must fit inside the first/last block");
    if (m + r > n - A->corner_cols)
      return fail(err, errlen, E_DimensionMismatch, "corner overlaps the first block row span");
  } else if (A->corner_rows || A->corner_cols) {
    return fail(err, errlen, E_CornerForbidden, "corner block not allowed for this kind");
  }
  size_t want = or_body_entry_count(A->kind, n, m, s, r);
  if (A->data_len != want)
    return fail(err, errlen, E_DimensionMismatch, "expected %zu body entries, got %zu", want,
                A->data_len);
  if (A->kind == OR_ABD || A->kind == OR_BABD) {
    int nb = n / m;
    A->abd_off = (size_t*)malloc(sizeof(size_t) * (nb + 1));
    size_t off = 0;
    for (int q = 0; q <= nb; ++q) {
      A->abd_off[q] = off;
      if (q < nb) {
        int c0, c1;
        abd_span(n, m, s, r, q, &c0, &c1);
        off += (size_t)m * (c1 - c0);
      }
    }
  }
  return 0;
}

void or_mat_release(or_mat* A) {
  free(A->abd_off);
  A->abd_off = NULL;
}

static int in_structure(const or_mat* A, int i, int j) { /* :86-110 */
  const int n = A->n;
  if (i < 0 || j < 0 || i >= n || j >= n) return 0;
  switch (A->kind) {
    case OR_BANDED:
      return j - i <= A->r && i - j <= A->s;
    case OR_BLOCKTRI: {
      int bi = i / A->m, bj = j / A->m;
      return abs(bi - bj) <= 1;
    }
    case OR_ABD:
    case OR_BABD: {
      int b = i / A->m, c0, c1;
      abd_span(n, A->m, A->s, A->r, b, &c0, &c1);
      if (j >= c0 && j < c1) return 1;
      if (A->kind == OR_BABD && i < A->corner_rows && j >= n - A->corner_cols) return 1;
      return 0;
    }
  }
  return 0;
}

double or_at(const or_mat* A, int i, int j) { /* :112-145 */
  if (!in_structure(A, i, j)) return 0.0;
  const int n = A->n, m = A->m;
  switch (A->kind) {
    case OR_BANDED: {
      int d = j - i;
      int i0 = imax(0, -d);
      return A->data[band_offset(n, A->s, d) + (size_t)(i - i0)];
    }
    case OR_BLOCKTRI: {
      int bi = i / m, bj = j / m;
      size_t off = bi == 0 ? 0 : (size_t)(3 * bi - 1) * m * m;
      int blk = bi > 0 ? bj - bi + 1 : bj - bi;
      return A->data[off + (size_t)blk * m * m + (size_t)(i - bi * m) * m + (j - bj * m)];
    }
    case OR_ABD:
    case OR_BABD: {
      int b = i / m, c0, c1;
      abd_span(n, m, A->s, A->r, b, &c0, &c1);
      if (j >= c0 && j < c1)
        return A->data[A->abd_off[b] + (size_t)(i - b * m) * (c1 - c0) + (j - c0)];
      return A->corner[(size_t)i * A->corner_cols + (j - (n - A->corner_cols))];
    }
  }
  return 0.0;
}

void or_scalar_envelope(const or_mat* A, int* es, int* er) { /* :271-280 */
  switch (A->kind) {
    case OR_BANDED:
    case OR_CIRCULANT: *es = A->s; *er = A->r; return;
    case OR_BLOCKTRI: *es = 2 * A->m - 1; *er = 2 * A->m - 1; return;
    default: *es = A->m - 1 + A->s; *er = A->m - 1 + A->r; return;
  }
}

/* Per-row ascending structural walk (for_each_in_row, :211-248). */
static void row_columns(const or_mat* A, int i, int* j0, int* j1, int* k0, int* k1) {
  *k0 = *k1 = 0;
  switch (A->kind) {
    case OR_BANDED:
      *j0 = imax(0, i - A->s);
      *j1 = imin(A->n - 1, i + A->r) + 1;
      return;
    case OR_BLOCKTRI: {
      int bi = i / A->m;
      *j0 = imax(0, (bi - 1) * A->m);
      *j1 = imin(A->n, (bi + 2) * A->m);
      return;
    }
    default: {
      int b = i / A->m;
      abd_span(A->n, A->m, A->s, A->r, b, j0, j1);
      if (A->kind == OR_BABD && i < A->corner_rows) {
        *k0 = A->n - A->corner_cols;
        *k1 = A->n;
      }
      return;
    }
  }
}

void or_matvec(const or_mat* A, const double* x, double* y) { /* matvec :260-269 */
  for (int i = 0; i < A->n; ++i) {
    int j0, j1, k0, k1;
    row_columns(A, i, &j0, &j1, &k0, &k1);
    double acc = 0.0;
    for (int j = j0; j < j1; ++j) acc += or_at(A, i, j) * x[j];
    for (int j = k0; j < k1; ++j) acc += or_at(A, i, j) * x[j];
    y[i] = acc;
  }
}

double or_residual(const or_mat* A, const double* x, const double* f) { /* src/parfact.cpp:241-251 */
  double* Ax = (double*)malloc(sizeof(double) * (size_t)A->n);
  or_matvec(A, x, Ax);
  double num = 0.0, den = 0.0;
  for (int i = 0; i < A->n; ++i) {
    double v = fabs(Ax[i] - f[i]);
    if (num < v) num = v; /* std::max(num, v) */
    double w = fabs(f[i]);
    if (den < w) den = w;
  }
  free(Ax);
  return den > 0 ? num / den : num;
}

/* ------------------------------------------------------------------------ */
/* partition: src/partition.cpp                                              */
/* ------------------------------------------------------------------------ */

static int separator_size_for(const or_mat* A) { /* :39-48 */
  switch (A->kind) {
    case OR_BANDED:
    case OR_CIRCULANT: return imax(A->s, A->r);
    default: return A->m;
  }
}

int or_plan_partition(const or_mat* A, int p, or_plan* plan, char* err, size_t errlen) { /* :52-105 */
  memset(plan, 0, sizeof(*plan));
  if (p < 2) return fail(err, errlen, E_TooManyPartitions, "p must be >= 2");
  if (A->kind == OR_CIRCULANT) return fail(err, errlen, E_UnsupportedKind, "circulant not in oracle");
  plan->kind = A->kind;
  plan->n = A->n;
  plan->m = A->m;
  plan->p = p;
  plan->sep_size = separator_size_for(A);
  plan->has_corner = A->kind == OR_BABD;
  if (A->kind == OR_BABD) {
    plan->corner_rows = A->corner_rows;
    plan->corner_cols = A->corner_cols;
  }
  const int k = plan->sep_size;
  const int seps = plan->has_corner ? p + 1 : p - 1;
  const int unit = A->kind == OR_BANDED ? 1 : A->m;
  if (k % unit != 0) return fail(err, errlen, E_UnsupportedKind, "separator does not tile blocks");
  const int n_units = A->n / unit;
  const int k_units = k / unit;
  const long long body_units_total = (long long)n_units - (long long)seps * k_units;
  const int min_body_units = imax(1, k_units);
  if (body_units_total < (long long)p * min_body_units)
    return fail(err, errlen, E_TooManyPartitions, "n too small for p = %d partitions of this kind", p);
  const int base = (int)(body_units_total / p);
  const int rem = (int)(body_units_total % p);
  plan->body_begin = (int*)malloc(sizeof(int) * p);
  plan->body_end = (int*)malloc(sizeof(int) * p);
  plan->sep_start = (int*)malloc(sizeof(int) * (seps > 0 ? seps : 1));
  plan->sep_count = 0;
  int cursor = 0;
  if (plan->has_corner) {
    plan->sep_start[plan->sep_count++] = cursor * unit;
    cursor += k_units;
  }
  for (int i = 0; i < p; ++i) {
    int units = base + (i < rem ? 1 : 0);
    plan->body_begin[i] = cursor * unit;
    plan->body_end[i] = (cursor + units) * unit;
    cursor += units;
    if (i < p - 1 || plan->has_corner) {
      plan->sep_start[plan->sep_count++] = cursor * unit;
      cursor += k_units;
    }
  }
  return 0;
}

void or_plan_release(or_plan* plan) {
  free(plan->body_begin);
  free(plan->body_end);
  free(plan->sep_start);
  memset(plan, 0, sizeof(*plan));
}

/* ------------------------------------------------------------------------ */
/* localfact, banded core (LU / LUD): src/localfact.cpp:47-225               */
/* ------------------------------------------------------------------------ */

typedef struct {
  int L, k0, k1, es, er, lud;
  double* fac;  /* L x w */
  double* dvec; /* LUD */
  double *z, *w, *y, *v;                  /* L x k0, L x k0, L x k1, L x k1 (row-major) */
  double *alpha1, *alpha2, *beta, *gamma; /* k0xk0, k1xk1, k1xk0, k0xk1 */
  double* kept;                           /* (k0+k1)^2 */
} local_t;

static void local_free(local_t* lf) {
  free(lf->fac); free(lf->dvec);
  free(lf->z); free(lf->w); free(lf->y); free(lf->v);
  free(lf->alpha1); free(lf->alpha2); free(lf->beta); free(lf->gamma); free(lf->kept);
  memset(lf, 0, sizeof(*lf));
}

/* banded_eliminate, :84-100 */
static int banded_eliminate(local_t* c, char* err, size_t errlen) {
  const int w = c->es + 1 + c->er;
  for (int k = 0; k < c->L; ++k) {
    double d = c->fac[(size_t)k * w + c->es];
    if (d == 0.0) return fail(err, errlen, E_ZeroPivot, "zero pivot at body row %d", k);
    int ilim = imin(c->L - 1, k + c->es);
    for (int i = k + 1; i <= ilim; ++i) {
      double* e = &c->fac[(size_t)i * w + (k - i + c->es)];
      if (*e == 0.0) continue;
      double mu = *e / d;
      *e = mu;
      int jlim = imin(c->L - 1, k + c->er);
      for (int j = k + 1; j <= jlim; ++j)
        c->fac[(size_t)i * w + (j - i + c->es)] -= mu * c->fac[(size_t)k * w + (j - k + c->es)];
    }
  }
  return 0;
}

static void lsolve(const local_t* c, double* x) { /* :103-111 */
  const int w = c->es + 1 + c->er;
  for (int i = 0; i < c->L; ++i) {
    double acc = x[i];
    int dlim = imin(c->es, i);
    for (int d = 1; d <= dlim; ++d) acc -= c->fac[(size_t)i * w + (c->es - d)] * x[i - d];
    x[i] = acc;
  }
}

static void usolve(const local_t* c, double* x) { /* :114-122 */
  const int w = c->es + 1 + c->er;
  for (int i = c->L - 1; i >= 0; --i) {
    double acc = x[i];
    int dlim = imin(c->er, c->L - 1 - i);
    for (int d = 1; d <= dlim; ++d) acc -= c->fac[(size_t)i * w + (c->es + d)] * x[i + d];
    x[i] = acc / c->fac[(size_t)i * w + c->es];
  }
}

static void uprime_solve(const local_t* c, double* x) { /* :125-134 */
  const int w = c->es + 1 + c->er;
  for (int i = c->L - 1; i >= 0; --i) {
    double acc = x[i];
    int dlim = imin(c->er, c->L - 1 - i);
    for (int d = 1; d <= dlim; ++d)
      acc -= (c->fac[(size_t)i * w + (c->es + d)] / c->dvec[i + d]) * x[i + d];
    x[i] = acc;
  }
}

static void ut_solve(const local_t* c, double* x) { /* :137-145 */
  const int w = c->es + 1 + c->er;
  for (int i = 0; i < c->L; ++i) {
    double acc = x[i];
    int dlim = imin(c->er, i);
    for (int d = 1; d <= dlim; ++d) acc -= c->fac[(size_t)(i - d) * w + (c->es + d)] * x[i - d];
    x[i] = acc / c->fac[(size_t)i * w + c->es];
  }
}

static void n_inv(const local_t* c, double* x) { /* banded_N_inv :147-151 */
  lsolve(c, x);
  if (c->lud) uprime_solve(c, x);
}

static void s_inv(const local_t* c, double* x) { /* banded_S_inv :153-160 */
  if (c->lud) {
    for (int i = 0; i < c->L; ++i) x[i] /= c->dvec[i];
  } else {
    usolve(c, x);
  }
}

static void st_inv(const local_t* c, double* x) { /* banded_St_inv :162-169 */
  if (c->lud) {
    for (int i = 0; i < c->L; ++i) x[i] /= c->dvec[i];
  } else {
    ut_solve(c, x);
  }
}

/* solve_columns :171-180: X(:, j) = op(B(:, j)); B, X are L x k row-major. */
static double* solve_columns(const local_t* c, const double* B, int k,
                             void (*op)(const local_t*, double*)) {
  double* X = (double*)calloc((size_t)c->L * (k ? k : 1), sizeof(double));
  double* col = (double*)malloc(sizeof(double) * (size_t)(c->L ? c->L : 1));
  for (int j = 0; j < k; ++j) {
    for (int i = 0; i < c->L; ++i) col[i] = B[(size_t)i * k + j];
    op(c, col);
    for (int i = 0; i < c->L; ++i) X[(size_t)i * k + j] = col[i];
  }
  free(col);
  return X;
}

/* at_b :47-56: C(ca x cb) = A^T B, A is L x ca, B is L x cb. */
static double* at_b(const double* A, int L, int ca, const double* B, int cb) {
  double* C = (double*)calloc((size_t)(ca ? ca : 1) * (cb ? cb : 1), sizeof(double));
  for (int k = 0; k < L; ++k)
    for (int i = 0; i < ca; ++i) {
      double a = A[(size_t)k * ca + i];
      if (a == 0.0) continue;
      for (int j = 0; j < cb; ++j) C[(size_t)i * cb + j] += a * B[(size_t)k * cb + j];
    }
  return C;
}

/* extract_block (src/partition.cpp:107-173) fused with banded_factor
 * (src/localfact.cpp:182-225).  i is 1-based like the reference. */
static int factor_partition(const or_mat* A, const or_plan* plan, int i, int lud, local_t* lf,
                            double* corner_slice, char* err, size_t errlen) {
  memset(lf, 0, sizeof(*lf));
  const int b = plan->body_begin[i - 1], e = plan->body_end[i - 1];
  const int L = e - b;
  const int k = plan->sep_size;
  const int left_sep = plan->has_corner ? i - 1 : i - 2;
  const int right_sep = plan->has_corner ? i : i - 1;
  const int k0 = left_sep >= 0 ? k : 0;
  const int k1 = right_sep < plan->sep_count ? k : 0;
  int es, er;
  or_scalar_envelope(A, &es, &er);
  lf->L = L;
  lf->k0 = k0;
  lf->k1 = k1;
  lf->lud = lud;
  lf->es = imin(es, L - 1);
  lf->er = imin(er, L - 1);
  const int w = lf->es + 1 + lf->er;
  lf->fac = (double*)calloc((size_t)L * w, sizeof(double));
  for (int x = 0; x < L; ++x)
    for (int j = imax(0, x - lf->es); j <= imin(L - 1, x + lf->er); ++j)
      lf->fac[(size_t)x * w + (j - x + lf->es)] = or_at(A, b + x, b + j);

  double* b0 = (double*)calloc((size_t)L * (k0 ? k0 : 1), sizeof(double));
  double* c0 = (double*)calloc((size_t)L * (k0 ? k0 : 1), sizeof(double));
  double* b1 = (double*)calloc((size_t)L * (k1 ? k1 : 1), sizeof(double));
  double* c1 = (double*)calloc((size_t)L * (k1 ? k1 : 1), sizeof(double));
  double* a_right = (double*)calloc((size_t)(k1 ? k1 * k1 : 1), sizeof(double));
  if (k0 > 0) {
    int ls = plan->sep_start[left_sep];
    for (int x = 0; x < L; ++x)
      for (int t = 0; t < k; ++t) {
        b0[(size_t)x * k + t] = or_at(A, b + x, ls + t);
        c0[(size_t)x * k + t] = or_at(A, ls + t, b + x);
      }
  }
  if (k1 > 0) {
    int rs = plan->sep_start[right_sep];
    for (int x = 0; x < L; ++x)
      for (int t = 0; t < k; ++t) {
        c1[(size_t)x * k + t] = or_at(A, b + x, rs + t);
        b1[(size_t)x * k + t] = or_at(A, rs + t, b + x);
      }
    for (int t = 0; t < k; ++t)
      for (int u = 0; u < k; ++u) a_right[t * k + u] = or_at(A, rs + t, rs + u);
  }
  if (plan->has_corner && i == 1 && k > 0 && corner_slice) {
    int s0 = plan->sep_start[0], sp = plan->sep_start[plan->sep_count - 1];
    for (int t = 0; t < k; ++t)
      for (int u = 0; u < k; ++u) corner_slice[t * k + u] = or_at(A, s0 + t, sp + u);
  }

  int rc = banded_eliminate(lf, err, errlen);
  if (rc == 0) {
    if (lud) {
      lf->dvec = (double*)malloc(sizeof(double) * (size_t)L);
      for (int x = 0; x < L; ++x) lf->dvec[x] = lf->fac[(size_t)x * w + lf->es];
    }
    lf->z = solve_columns(lf, b0, k0, n_inv);
    lf->y = solve_columns(lf, c1, k1, n_inv);
    lf->w = solve_columns(lf, c0, k0, st_inv);
    lf->v = solve_columns(lf, b1, k1, st_inv);
    double* wz = at_b(lf->w, L, k0, lf->z, k0);
    double* vy = at_b(lf->v, L, k1, lf->y, k1);
    double* vz = at_b(lf->v, L, k1, lf->z, k0);
    double* wy = at_b(lf->w, L, k0, lf->y, k1);
    lf->alpha1 = wz;
    for (int t = 0; t < k0 * k0; ++t) lf->alpha1[t] = -lf->alpha1[t];
    lf->alpha2 = (double*)calloc((size_t)(k1 ? k1 * k1 : 1), sizeof(double));
    for (int t = 0; t < k1 * k1; ++t) lf->alpha2[t] = a_right[t] - vy[t];
    free(vy);
    lf->beta = vz;
    for (int t = 0; t < k1 * k0; ++t) lf->beta[t] = -lf->beta[t];
    lf->gamma = wy;
    for (int t = 0; t < k0 * k1; ++t) lf->gamma[t] = -lf->gamma[t];
    const int kd = k0 + k1;
    lf->kept = (double*)calloc((size_t)(kd ? kd * kd : 1), sizeof(double));
    for (int a = 0; a < k0; ++a)
      for (int c = 0; c < k0; ++c) lf->kept[a * kd + c] = lf->alpha1[a * k0 + c];
    for (int a = 0; a < k0; ++a)
      for (int c = 0; c < k1; ++c) lf->kept[a * kd + k0 + c] = lf->gamma[a * k1 + c];
    for (int a = 0; a < k1; ++a)
      for (int c = 0; c < k0; ++c) lf->kept[(k0 + a) * kd + c] = lf->beta[a * k0 + c];
    for (int a = 0; a < k1; ++a)
      for (int c = 0; c < k1; ++c) lf->kept[(k0 + a) * kd + k0 + c] = lf->alpha2[a * k1 + c];
  }
  free(b0); free(c0); free(b1); free(c1); free(a_right);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* parfact: src/parfact.cpp                                                  */
/* ------------------------------------------------------------------------ */

struct or_fact {
  or_mat A; /* borrowed arrays, own abd_off copy */
  or_plan plan;
  int strategy;
  local_t* locals;
  int q, dim, k;
  double* T; /* dim x dim */
  int* kept_map; /* p x (2k), -1 when absent */
};

int or_parallel_factor(const or_mat* A, int p, int strategy, or_fact** out, char* err,
                       size_t errlen) { /* :21-132 */
  *out = NULL;
  if (strategy != OR_LU && strategy != OR_LUD)
    return fail(err, errlen, E_UnsupportedStructure, "oracle implements lu and lud only");
  or_fact* F = (or_fact*)calloc(1, sizeof(or_fact));
  F->A = *A;
  F->A.abd_off = NULL;
  if (A->abd_off) {
    size_t nb = (size_t)(A->n / A->m) + 1;
    F->A.abd_off = (size_t*)malloc(sizeof(size_t) * nb);
    memcpy(F->A.abd_off, A->abd_off, sizeof(size_t) * nb);
  }
  F->strategy = strategy;
  int rc = or_plan_partition(A, p, &F->plan, err, errlen);
  if (rc) {
    or_fact_release(F);
    return rc;
  }
  const or_plan* plan = &F->plan;
  const int k = plan->sep_size;
  F->k = k;
  F->locals = (local_t*)calloc((size_t)p, sizeof(local_t));
  double* corner_slice = (double*)calloc((size_t)k * k, sizeof(double));
  /* The reference rethrows the lowest failing partition index (:61-68). */
  for (int i = 1; i <= p; ++i) {
    char sub[200] = {0};
    rc = factor_partition(A, plan, i, strategy == OR_LUD, &F->locals[i - 1], corner_slice, sub,
                          sizeof sub);
    if (rc) {
      fail(err, errlen, rc - 1, "partition %d: %s", i, sub);
      free(corner_slice);
      or_fact_release(F);
      return rc;
    }
  }
  F->q = plan->sep_count;
  F->dim = F->q * k;
  const int dim = F->dim;
  F->T = (double*)calloc((size_t)dim * (dim ? dim : 1), sizeof(double));
  if (plan->has_corner) { /* :94-104 */
    int s0 = plan->sep_start[0];
    int o0 = 0, op = (F->q - 1) * k;
    for (int t = 0; t < k; ++t)
      for (int u = 0; u < k; ++u) F->T[(size_t)(o0 + t) * dim + o0 + u] += or_at(A, s0 + t, s0 + u);
    for (int t = 0; t < k; ++t)
      for (int u = 0; u < k; ++u) F->T[(size_t)(o0 + t) * dim + op + u] += corner_slice[t * k + u];
  }
  free(corner_slice);
  F->kept_map = (int*)malloc(sizeof(int) * (size_t)p * 2 * k);
  for (int i = 0; i < p; ++i) { /* :106-127 */
    const local_t* lf = &F->locals[i];
    int* map = &F->kept_map[(size_t)i * 2 * k];
    int left_sep = plan->has_corner ? i : i - 1;
    int right_sep = plan->has_corner ? i + 1 : i;
    int cnt = 0;
    for (int t = 0; t < 2 * k; ++t) map[t] = -1;
    if (lf->k0 > 0)
      for (int t = 0; t < k; ++t) map[cnt++] = left_sep * k + t;
    if (lf->k1 > 0)
      for (int t = 0; t < k; ++t) map[cnt++] = right_sep * k + t;
    const int kd = lf->k0 + lf->k1;
    for (int a = 0; a < kd; ++a)
      for (int c = 0; c < kd; ++c) F->T[(size_t)map[a] * dim + map[c]] += lf->kept[a * kd + c];
  }
  *out = F;
  return 0;
}

void or_fact_release(or_fact* F) {
  if (!F) return;
  if (F->locals)
    for (int i = 0; i < F->plan.p; ++i) local_free(&F->locals[i]);
  free(F->locals);
  free(F->T);
  free(F->kept_map);
  free(F->A.abd_off);
  or_plan_release(&F->plan);
  free(F);
}

void or_fact_dims(const or_fact* F, int* q, int* dim, int* k) {
  if (q) *q = F->q;
  if (dim) *dim = F->dim;
  if (k) *k = F->k;
}

void or_fact_T(const or_fact* F, double* T) {
  memcpy(T, F->T, sizeof(double) * (size_t)F->dim * F->dim);
}

void or_fact_local(const or_fact* F, int i, int* k0, int* k1, double* alpha1, double* alpha2,
                   double* beta, double* gamma) {
  const local_t* lf = &F->locals[i];
  if (k0) *k0 = lf->k0;
  if (k1) *k1 = lf->k1;
  if (alpha1) memcpy(alpha1, lf->alpha1, sizeof(double) * lf->k0 * lf->k0);
  if (alpha2) memcpy(alpha2, lf->alpha2, sizeof(double) * lf->k1 * lf->k1);
  if (beta) memcpy(beta, lf->beta, sizeof(double) * lf->k1 * lf->k0);
  if (gamma) memcpy(gamma, lf->gamma, sizeof(double) * lf->k0 * lf->k1);
}

/* solve_reduced :134-184 (dense partial-pivot LU, refactored every call). */
static int solve_reduced(const double* T, int n, const double* rhs, double* x, long long* ops_out,
                         char* err, size_t errlen) {
  if (n == 0) return 0;
  long long ops = 0;
  double* lu = (double*)malloc(sizeof(double) * (size_t)n * n);
  memcpy(lu, T, sizeof(double) * (size_t)n * n);
  int* perm = (int*)malloc(sizeof(int) * n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    double best = fabs(lu[(size_t)c * n + c]);
    for (int i = c + 1; i < n; ++i) {
      double v = fabs(lu[(size_t)i * n + c]);
      if (v > best) {
        best = v;
        piv = i;
      }
    }
    if (best == 0.0) {
      free(lu); free(perm);
      return fail(err, errlen, E_SingularReducedSystem, "reduced system is singular");
    }
    if (piv != c) {
      for (int j = 0; j < n; ++j) {
        double t = lu[(size_t)c * n + j];
        lu[(size_t)c * n + j] = lu[(size_t)piv * n + j];
        lu[(size_t)piv * n + j] = t;
      }
      int t = perm[c];
      perm[c] = perm[piv];
      perm[piv] = t;
    }
    for (int i = c + 1; i < n; ++i) {
      double mu = lu[(size_t)i * n + c] / lu[(size_t)c * n + c];
      lu[(size_t)i * n + c] = mu;
      ++ops;
      for (int j = c + 1; j < n; ++j) {
        lu[(size_t)i * n + j] -= mu * lu[(size_t)c * n + j];
        ++ops;
      }
    }
  }
  for (int i = 0; i < n; ++i) x[i] = rhs[perm[i]];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) {
      x[i] -= lu[(size_t)i * n + j] * x[j];
      ++ops;
    }
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) {
      x[i] -= lu[(size_t)i * n + j] * x[j];
      ++ops;
    }
    x[i] /= lu[(size_t)i * n + i];
    ++ops;
  }
  if (ops_out) *ops_out += ops;
  free(lu);
  free(perm);
  return 0;
}

int or_solve(const or_fact* F, const double* f, double* x, long long* reduced_ops, char* err,
             size_t errlen) { /* :186-239 */
  const or_plan* plan = &F->plan;
  const int p = plan->p, k = F->k, dim = F->dim;
  double** ghat = (double**)calloc((size_t)p, sizeof(double*));
  double* kept_rhs = (double*)calloc((size_t)p * 2 * k, sizeof(double));
  for (int i = 0; i < p; ++i) { /* phase 1, condense :765-781 */
    const local_t* lf = &F->locals[i];
    const int b = plan->body_begin[i], L = lf->L;
    ghat[i] = (double*)malloc(sizeof(double) * (size_t)(L ? L : 1));
    memcpy(ghat[i], f + b, sizeof(double) * (size_t)L);
    n_inv(lf, ghat[i]);
    double* kr = &kept_rhs[(size_t)i * 2 * k];
    for (int t = 0; t < lf->k0; ++t) {
      double acc = 0.0;
      for (int xx = 0; xx < L; ++xx) acc += lf->w[(size_t)xx * lf->k0 + t] * ghat[i][xx];
      kr[t] = -acc;
    }
    for (int t = 0; t < lf->k1; ++t) {
      double acc = 0.0;
      for (int xx = 0; xx < L; ++xx) acc += lf->v[(size_t)xx * lf->k1 + t] * ghat[i][xx];
      kr[lf->k0 + t] = -acc;
    }
  }
  double* rrhs = (double*)calloc((size_t)(dim ? dim : 1), sizeof(double));
  for (int bidx = 0; bidx < F->q; ++bidx) /* :205-211 */
    for (int t = 0; t < k; ++t) rrhs[bidx * k + t] = f[plan->sep_start[bidx] + t];
  for (int i = 0; i < p; ++i) { /* :212-214 */
    const local_t* lf = &F->locals[i];
    const int kd = lf->k0 + lf->k1;
    for (int a = 0; a < kd; ++a) rrhs[F->kept_map[(size_t)i * 2 * k + a]] += kept_rhs[(size_t)i * 2 * k + a];
  }
  double* xk = (double*)calloc((size_t)(dim ? dim : 1), sizeof(double));
  int rc = solve_reduced(F->T, dim, rrhs, xk, reduced_ops, err, errlen);
  if (rc == 0) {
    for (int bidx = 0; bidx < F->q; ++bidx)
      for (int t = 0; t < k; ++t) x[plan->sep_start[bidx] + t] = xk[bidx * k + t];
    for (int i = 0; i < p; ++i) { /* phase 3, backsolve :809-818 */
      const local_t* lf = &F->locals[i];
      const int L = lf->L, b = plan->body_begin[i];
      double xkept[64];
      const int kd = lf->k0 + lf->k1;
      for (int a = 0; a < kd; ++a) xkept[a] = xk[F->kept_map[(size_t)i * 2 * k + a]];
      double* rhs = ghat[i];
      for (int xx = 0; xx < L; ++xx) {
        double acc = rhs[xx];
        for (int t = 0; t < lf->k0; ++t) acc -= lf->z[(size_t)xx * lf->k0 + t] * xkept[t];
        for (int t = 0; t < lf->k1; ++t) acc -= lf->y[(size_t)xx * lf->k1 + t] * xkept[lf->k0 + t];
        rhs[xx] = acc;
      }
      s_inv(lf, rhs);
      memcpy(x + b, rhs, sizeof(double) * (size_t)L);
    }
  }
  for (int i = 0; i < p; ++i) free(ghat[i]);
  free(ghat);
  free(kept_rhs);
  free(rrhs);
  free(xk);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* seqref: src/seqref.cpp:12-93                                              */
/* ------------------------------------------------------------------------ */

/* DenseLu + solve, src/dense.cpp:78-120 */
static int dense_lu_solve(double* lu, int n, const double* b, double* y, char* err, size_t errlen) {
  int* perm = (int*)malloc(sizeof(int) * (n ? n : 1));
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    double best = fabs(lu[(size_t)k * n + k]);
    for (int i = k + 1; i < n; ++i) {
      double v = fabs(lu[(size_t)i * n + k]);
      if (v > best) {
        best = v;
        piv = i;
      }
    }
    if (best == 0.0) {
      free(perm);
      return fail(err, errlen, E_SingularFactor, "zero pivot column in dense LU");
    }
    if (piv != k) {
      for (int j = 0; j < n; ++j) {
        double t = lu[(size_t)k * n + j];
        lu[(size_t)k * n + j] = lu[(size_t)piv * n + j];
        lu[(size_t)piv * n + j] = t;
      }
      int t = perm[k];
      perm[k] = perm[piv];
      perm[piv] = t;
    }
    double d = lu[(size_t)k * n + k];
    for (int i = k + 1; i < n; ++i) {
      double m = lu[(size_t)i * n + k] / d;
      lu[(size_t)i * n + k] = m;
      if (m == 0.0) continue;
      for (int j = k + 1; j < n; ++j) lu[(size_t)i * n + j] -= m * lu[(size_t)k * n + j];
    }
  }
  for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) y[i] -= lu[(size_t)i * n + j] * y[j];
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) y[i] -= lu[(size_t)i * n + j] * y[j];
    y[i] /= lu[(size_t)i * n + i];
  }
  free(perm);
  return 0;
}

int or_solve_sequential(const or_mat* A, const double* f, double* x, char* err, size_t errlen) {
  const int n = A->n;
  int es, er;
  or_scalar_envelope(A, &es, &er);
  int K = 0;
  if (A->kind == OR_BABD) K = A->corner_cols;
  if (K > 0) K = imin(K + er + es, n);
  const int nb = n - K;
  const int w = es + 1 + er;
  const size_t nbz = (size_t)(nb > 0 ? nb : 0);
  double* band = (double*)calloc(nbz * w + 1, sizeof(double));
  double* spike = (double*)calloc(nbz * (K ? K : 1) + 1, sizeof(double));
  double* rhs = (double*)malloc(sizeof(double) * (size_t)n);
  memcpy(rhs, f, sizeof(double) * (size_t)n);
  for (int i = 0; i < nb; ++i) {
    for (int j = imax(0, i - es); j <= imin(nb - 1, i + er); ++j)
      band[(size_t)i * w + (j - i + es)] = or_at(A, i, j);
    for (int j = nb; j < n; ++j) spike[(size_t)i * K + (j - nb)] = or_at(A, i, j);
  }
  int rc = 0;
  for (int k = 0; k < nb && rc == 0; ++k) {
    double d = band[(size_t)k * w + es];
    if (d == 0.0) {
      rc = fail(err, errlen, E_SingularFactor, "zero pivot in sequential reference");
      break;
    }
    for (int i = k + 1; i <= imin(nb - 1, k + es); ++i) {
      double e = band[(size_t)i * w + (k - i + es)];
      if (e == 0.0) continue;
      double mu = e / d;
      for (int j = k + 1; j <= imin(nb - 1, k + er); ++j)
        band[(size_t)i * w + (j - i + es)] -= mu * band[(size_t)k * w + (j - k + es)];
      for (int q = 0; q < K; ++q) spike[(size_t)i * K + q] -= mu * spike[(size_t)k * K + q];
      rhs[i] -= mu * rhs[k];
    }
  }
  double* tail = (double*)calloc((size_t)(K ? K * K : 1), sizeof(double));
  double* trhs = (double*)calloc((size_t)(K ? K : 1), sizeof(double));
  double* row = (double*)calloc((size_t)n, sizeof(double));
  for (int t = 0; t < K && rc == 0; ++t) {
    int i = nb + t;
    memset(row, 0, sizeof(double) * (size_t)n);
    int j0, j1, c0, c1;
    row_columns(A, i, &j0, &j1, &c0, &c1);
    for (int j = j0; j < j1; ++j) {
      double v = or_at(A, i, j);
      if (v != 0.0) row[j] = v;
    }
    for (int j = c0; j < c1; ++j) {
      double v = or_at(A, i, j);
      if (v != 0.0) row[j] = v;
    }
    double rv = f[i];
    for (int k = imax(0, i - es - K); k < nb; ++k) {
      double e = row[k];
      if (e == 0.0) continue;
      double mu = e / band[(size_t)k * w + es];
      row[k] = 0.0;
      for (int j = k + 1; j <= imin(nb - 1, k + er); ++j) row[j] -= mu * band[(size_t)k * w + (j - k + es)];
      for (int q = 0; q < K; ++q) row[nb + q] -= mu * spike[(size_t)k * K + q];
      rv -= mu * rhs[k];
    }
    for (int q = 0; q < K; ++q) tail[t * K + q] = row[nb + q];
    trhs[t] = rv;
  }
  free(row);
  if (rc == 0) {
    for (int i = 0; i < n; ++i) x[i] = 0.0;
    if (K > 0) {
      double* xt = (double*)malloc(sizeof(double) * K);
      rc = dense_lu_solve(tail, K, trhs, xt, err, errlen);
      if (rc == 0)
        for (int q = 0; q < K; ++q) x[nb + q] = xt[q];
      free(xt);
    }
    if (rc == 0)
      for (int k = nb - 1; k >= 0; --k) {
        double acc = rhs[k];
        for (int j = k + 1; j <= imin(nb - 1, k + er); ++j) acc -= band[(size_t)k * w + (j - k + es)] * x[j];
        for (int q = 0; q < K; ++q) acc -= spike[(size_t)k * K + q] * x[nb + q];
        x[k] = acc / band[(size_t)k * w + es];
      }
  }
  free(band); free(spike); free(rhs); free(tail); free(trhs);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* rng: include/parsol/rng.hpp:11-35, config generators     */
/* ------------------------------------------------------------------------ */

static uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t or_splitmix_u64(uint64_t seed, uint64_t stream, uint64_t k) {
  uint64_t base = sm_mix(seed + 0x9E3779B97F4A7C15ull * (stream + 1));
  return sm_mix(base + 0x9E3779B97F4A7C15ull * k);
}

double or_splitmix_unit(uint64_t seed, uint64_t stream, uint64_t k) {
  const uint64_t u = or_splitmix_u64(seed, stream, k) >> 11;
  return 2.0 * ((double)u / 9007199254740992.0) - 1.0 + 1.1102230246251565e-16;
}

/* U[-1,1] = next_unit(); U[0,1] = (next_unit()+1)/2; U[-1/2,1/2] = next_unit()/2.
 * Element e of a stream uses the (e+1)-th draw. */
#define UNIT(st, e) or_splitmix_unit(seed, (st), (uint64_t)(e) + 1)

int or_config_shape(int cfg, int size, int* kind, int* n, int* m, int* s, int* r,
                    size_t* data_len, int* corner_rows, int* corner_cols) {
  *corner_rows = *corner_cols = 0;
  switch (cfg) {
    case 0:
    case 1: *kind = OR_BANDED; *n = size; *m = 1; *s = 1; *r = 1; break;
    case 2: *kind = OR_BLOCKTRI; *n = 4 * size; *m = 4; *s = 1; *r = 1; break;
    case 3: *kind = OR_BANDED; *n = size; *m = 1; *s = 3; *r = 3; break;
    case 4:
      *kind = OR_BABD; *n = 8 * (size + 1); *m = 8; *s = 8; *r = 0;
      *corner_rows = *corner_cols = 8;
      break;
    default: return 1 + E_InvalidParameter;
  }
  *data_len = or_body_entry_count(*kind, *n, *m, *s, *r);
  return 0;
}

int or_generate_config(int cfg, int size, uint64_t seed, double* data, double* corner, double* f) {
  int kind, n, m, s, r, cr, cc;
  size_t len;
  if (or_config_shape(cfg, size, &kind, &n, &m, &s, &r, &len, &cr, &cc)) return 1 + E_InvalidParameter;
  if (cfg == 0 || cfg == 1) {
    /* data = [sub (n-1) | diag (n) | super (n-1)] */
    for (int e = 0; e < n - 1; ++e) data[e] = UNIT(0, e);
    for (int e = 0; e < n; ++e) data[(size_t)(n - 1) + e] = 4.0 + 0.5 * (UNIT(1, e) + 1.0);
    for (int e = 0; e < n - 1; ++e) data[(size_t)(2 * n - 1) + e] = UNIT(2, e);
    for (int e = 0; e < n; ++e) f[e] = UNIT(3, e);
  } else if (cfg == 2) {
    const int N = size;
    for (int b = 0; b < N; ++b) {
      size_t off = b == 0 ? 0 : (size_t)(3 * b - 1) * 16;
      int blk = 0;
      if (b > 0) { /* sub block of row b: stream 1, index (b-1)*16 */
        for (int t = 0; t < 16; ++t) data[off + t] = 0.5 * UNIT(1, (size_t)(b - 1) * 16 + t);
        blk = 1;
      }
      for (int t = 0; t < 16; ++t) /* diag block: stream 0 */
        data[off + (size_t)blk * 16 + t] = ((t / 4 == t % 4) ? 8.0 : 0.0) + 0.5 * UNIT(0, (size_t)b * 16 + t);
      if (b < N - 1)
        for (int t = 0; t < 16; ++t) data[off + (size_t)(blk + 1) * 16 + t] = 0.5 * UNIT(2, (size_t)b * 16 + t);
    }
    for (int e = 0; e < n; ++e) f[e] = UNIT(3, e);
  } else if (cfg == 3) {
    size_t pos = 0, offd = 0;
    for (int d = -s; d <= r; ++d) {
      int len_d = n - abs(d);
      for (int t = 0; t < len_d; ++t) {
        if (d == 0)
          data[pos + t] = 8.0 + 0.5 * (UNIT(1, t) + 1.0);
        else
          data[pos + t] = UNIT(0, offd + t);
      }
      if (d != 0) offd += (size_t)len_d;
      pos += (size_t)len_d;
    }
    for (int e = 0; e < n; ++e) f[e] = UNIT(2, e);
  } else {
    /* BABD, BC row first: block row 0 = B0 = I (span [0,8)), corner = B1;
     * block row k+1 = [-(I + h/2 M_k), I - h/2 M_{k+1}] over cols [8k, 8k+16). */
    const int N = size;
    const double h = 1.0 / (double)N, hh = 0.5 * h;
    for (int t = 0; t < 64; ++t) data[t] = (t / 8 == t % 8) ? 1.0 : 0.0;
    for (int t = 0; t < 64; ++t) corner[t] = 0.5 * UNIT(2, t);
    for (int k = 0; k < N; ++k) {
      double* row = data + 64 + (size_t)k * 128;
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          double mk = UNIT(0, (size_t)k * 64 + i * 8 + j) / 8.0;
          double mk1 = UNIT(0, (size_t)(k + 1) * 64 + i * 8 + j) / 8.0;
          double id = (i == j) ? 1.0 : 0.0;
          row[i * 16 + j] = -(id + hh * mk);
          row[i * 16 + 8 + j] = id - hh * mk1;
        }
    }
    for (int i = 0; i < 8; ++i) f[i] = UNIT(3, i);
    for (int k = 0; k < N; ++k)
      for (int i = 0; i < 8; ++i)
        f[8 + (size_t)k * 8 + i] = hh * (UNIT(1, (size_t)k * 8 + i) + UNIT(1, (size_t)(k + 1) * 8 + i));
  }
  return 0;
}

/* generate_random (src/structmat.cpp:282-333): draws in storage order from
 * SplitMix64(seed), Babd corner m x m, then diagonal rescaled to
 * +-dominance * max(off-row |sum|, 1).  Babd here also accepts s = m, r = 0. */
int or_generate_random(int kind, int n, int m, int s, int r, uint64_t seed, double dominance, double* data,
                       double* corner) {
  if (dominance < 0) return 1 + E_InvalidParameter;
  const size_t count = or_body_entry_count(kind, n, m, s, r);
  uint64_t ctr = 0;
  for (size_t e = 0; e < count; ++e) data[e] = or_splitmix_unit(seed, 0, ++ctr);
  if (kind == OR_BABD)
    for (int e = 0; e < m * m; ++e) corner[e] = or_splitmix_unit(seed, 0, ++ctr);
  or_mat A = {kind, n, m, s, r, data, count, kind == OR_BABD ? corner : NULL, kind == OR_BABD ? m : 0,
              kind == OR_BABD ? m : 0, NULL};
  char err[128];
  int rc = or_mat_prepare(&A, err, sizeof err);
  if (rc) return rc;
  if (dominance > 0.0) {
    for (int i = 0; i < n; ++i) {
      int j0, j1, k0, k1;
      row_columns(&A, i, &j0, &j1, &k0, &k1);
      double off = 0.0;
      for (int j = j0; j < j1; ++j)
        if (j != i) off += fabs(or_at(&A, i, j));
      for (int j = k0; j < k1; ++j)
        if (j != i) off += fabs(or_at(&A, i, j));
      double mag = dominance * (off > 1.0 ? off : 1.0);
      double old = or_at(&A, i, i);
      double val = old < 0 ? -mag : mag;
      size_t pos;
      switch (kind) {
        case OR_BANDED: pos = band_offset(n, s, 0) + (size_t)i; break;
        case OR_BLOCKTRI: {
          int b = i / m;
          size_t offr = b == 0 ? 0 : (size_t)(3 * b - 1) * m * m;
          int blk = b > 0 ? 1 : 0;
          pos = offr + (size_t)blk * m * m + (size_t)(i - b * m) * m + (i - b * m);
          break;
        }
        default: {
          int b = i / m, c0, c1;
          abd_span(n, m, s, r, b, &c0, &c1);
          pos = A.abd_off[b] + (size_t)(i - b * m) * (c1 - c0) + (i - c0);
          break;
        }
      }
      data[pos] = val;
    }
  }
  or_mat_release(&A);
  return 0;
}
