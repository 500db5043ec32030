/*
 * parsol_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference `parsol` hot path (parallel
 * factorization A = F T G, arXiv 0912.3678) used as the CPU oracle for the
 * B200 solver.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library, and only as the
 * checker or the CPU baseline -- never as the product path.
 *
 * Parity pin: every routine follows the reference operation order (file:line
 * cited in parsol_oracle.c) so that its results are bit-identical to the
 * unmodified reference compiled into oracle/_ref/libparsol_ref.so; the test
 * suite checks that (tests/test_oracle.py) and checks both against the
 * committed golden fixtures (tests/golden/).
 *
 * Supported kinds: Banded, BlockTridiagonal, Abd, Babd (CirculantLike is
 * rejected with UnsupportedKind).  Strategies: Lu and Lud.
 */
#ifndef PARSOL_ORACLE_H
#define PARSOL_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Kind / Strategy / Errc numbering follows the reference enums
 * (include/parsol/structmat.hpp:11, localfact.hpp:11, errors.hpp:12-35). */
enum { OR_BANDED = 0, OR_BLOCKTRI = 1, OR_ABD = 2, OR_BABD = 3, OR_CIRCULANT = 4 };
enum { OR_LU = 0, OR_LUD = 1 };

typedef struct {
  int kind, n, m, s, r;
  const double* data;
  size_t data_len;
  const double* corner;
  int corner_rows, corner_cols;
  size_t* abd_off; /* prepared: N+1 block-row offsets (Abd/Babd) */
} or_mat;

/* Returns 0 or 1+Errc.  Mirrors make() (src/structmat.cpp:153-207) except
 * that Babd additionally accepts the paper's s = m, r = 0 BVP layout. */
int or_mat_prepare(or_mat* A, char* err, size_t errlen);
void or_mat_release(or_mat* A);
size_t or_body_entry_count(int kind, int n, int m, int s, int r);
double or_at(const or_mat* A, int i, int j);
void or_scalar_envelope(const or_mat* A, int* es, int* er);

typedef struct {
  int kind, n, m, p, sep_size, has_corner, corner_rows, corner_cols, sep_count;
  int* body_begin; /* p */
  int* body_end;   /* p */
  int* sep_start;  /* sep_count */
} or_plan;

int or_plan_partition(const or_mat* A, int p, or_plan* plan, char* err, size_t errlen);
void or_plan_release(or_plan* plan);

typedef struct or_fact or_fact;

int or_parallel_factor(const or_mat* A, int p, int strategy, or_fact** out, char* err,
                       size_t errlen);
void or_fact_release(or_fact* F);
/* q (kept blocks), dim (scalar reduced dimension), sep_size k. */
void or_fact_dims(const or_fact* F, int* q, int* dim, int* k);
/* Dense reduced matrix T (dim x dim, row-major). */
void or_fact_T(const or_fact* F, double* T);
/* Partition i (0-based): alpha1 (k0 x k0), alpha2 (k1 x k1), beta (k1 x k0),
 * gamma (k0 x k1); returns k0 and k1 through pointers (arrays may be NULL). */
void or_fact_local(const or_fact* F, int i, int* k0, int* k1, double* alpha1, double* alpha2,
                   double* beta, double* gamma);
int or_solve(const or_fact* F, const double* f, double* x, long long* reduced_ops, char* err,
             size_t errlen);

int or_solve_sequential(const or_mat* A, const double* f, double* x, char* err, size_t errlen);
void or_matvec(const or_mat* A, const double* x, double* y);
double or_residual(const or_mat* A, const double* x, const double* f);

/* SplitMix64 draw k (1-based counter) of (seed, stream), include/parsol/rng.hpp:11-35. */
uint64_t or_splitmix_u64(uint64_t seed, uint64_t stream, uint64_t k);
double or_splitmix_unit(uint64_t seed, uint64_t stream, uint64_t k);

/* BASELINE config generators (SURVEY.md 8(d) stream mapping).  cfg 0/1:
 * tridiagonal; 2: block tridiagonal m=4; 3: banded s=r=3; 4: BABD m=8,
 * s=8, r=0 with an m x m corner.  size = n (cfg 0,1,3), N block rows
 * (cfg 2), or N intervals (cfg 4).  Fills data (body_entry_count entries),
 * corner (64 entries, cfg 4 only) and f (n entries). */
int or_config_shape(int cfg, int size, int* kind, int* n, int* m, int* s, int* r,
                    size_t* data_len, int* corner_rows, int* corner_cols);
int or_generate_config(int cfg, int size, uint64_t seed, double* data, double* corner,
                       double* f);

/* generate_random, src/structmat.cpp:282-333 (corner m x m for Babd). */
int or_generate_random(int kind, int n, int m, int s, int r, uint64_t seed, double dominance, double* data,
                       double* corner);

#ifdef __cplusplus
}
#endif
#endif
