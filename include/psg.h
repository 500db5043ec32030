/*
 * psg.h -- C ABI of the B200-native partition solver (parallel factorization
 * A = F T G of arXiv 0912.3678), the drop-in boundary under the reference's
 * C++ solver API.
 *
 * Every entry point is plain C: raw pointers, sizes and an opaque cudaStream_t
 * (passed as void*, NULL = legacy default stream).  Nothing here throws; each
 * returns 0 on success or 1 + Errc (the reference error enum,
 * proj/include/parsol/errors.hpp:12-35) and writes a message into err.  The
 * C++ host layer (include/parsol/parfact.hpp in this repo) turns that into
 * parsol::Error(code, detail) exactly like the reference.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   psg_factor          <- parallel_factor()      include/parsol/parfact.hpp:52-53
 *                                                  (impl src/parfact.cpp:21-132)
 *   psg_solve           <- solve()                include/parsol/parfact.hpp:60
 *                                                  (impl src/parfact.cpp:186-239)
 *   psg_solve_reduced   <- solve_reduced()        include/parsol/parfact.hpp:56
 *                                                  (impl src/parfact.cpp:134-184)
 *   psg_residual        <- residual()             include/parsol/parfact.hpp:63
 *                                                  (impl src/parfact.cpp:241-251)
 *   psg_matvec          <- matvec()               include/parsol/structmat.hpp:66
 *   psg_plan            <- plan_partition()       include/parsol/partition.hpp:82
 *   psg_reduced_*       <- ParallelFactorization::reduced (ReducedSystem,
 *                          include/parsol/parfact.hpp:14-22)
 *   psg_ode_trajectory  <- solve_ivp_parallel()   include/parsol/odeparallel.hpp (reference
 *                          proj/include/parsol/odeparallel.hpp; impl src/odeparallel.cpp:183-233)
 *   psg_pr_*            <- propagate / parareal_init / parareal_iterate / parareal_solve
 *                          include/parsol/parareal.hpp (reference proj/include/parsol/parareal.hpp;
 *                          impl src/parareal.cpp:56-117)
 *   psg_generate_config -- (new) device generator of the BASELINE configs,
 *                          bit-identical to SplitMix64 (include/parsol/rng.hpp)
 */
#ifndef PSG_H
#define PSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Kind numbering = parsol::Kind (structmat.hpp:11). */
enum psg_kind { PSG_BANDED = 0, PSG_BLOCKTRI = 1, PSG_ABD = 2, PSG_BABD = 3, PSG_CIRCULANT = 4 };
/* Strategy numbering = parsol::Strategy (localfact.hpp:11). */
enum psg_strategy { PSG_LU = 0, PSG_LUD = 1, PSG_CR = 2, PSG_ARCE = 3, PSG_LUPIVOT = 4, PSG_QR = 5 };
/* Errc numbering = parsol::Errc; functions return 1 + value on failure. */
enum psg_errc {
  PSG_E_DIMENSION_MISMATCH = 0, PSG_E_INVALID_BANDWIDTH, PSG_E_CORNER_FORBIDDEN,
  PSG_E_TOO_LARGE_FOR_DENSE, PSG_E_INVALID_PARAMETER, PSG_E_PARSE_ERROR,
  PSG_E_UNSUPPORTED_VERSION, PSG_E_TOO_MANY_PARTITIONS, PSG_E_UNSUPPORTED_KIND,
  PSG_E_UNSUPPORTED_STRUCTURE, PSG_E_INDEX_OUT_OF_RANGE, PSG_E_ZERO_PIVOT,
  PSG_E_SINGULAR_BLOCK, PSG_E_SINGULAR_FACTOR, PSG_E_SINGULAR_REDUCED_SYSTEM,
  PSG_E_SINGULAR_WINDOW, PSG_E_EXHAUSTED_BODY, PSG_E_STEP_TOO_LARGE,
  PSG_E_INVALID_INTERVAL, PSG_E_EXPM_FAILURE, PSG_E_NOT_CONVERGED, PSG_E_IO_ERROR,
  PSG_E_CUDA = 100 /* CUDA runtime failure (no reference equivalent) */
};

/* Structured matrix descriptor, storage exactly as parsol::StructuredMatrix
 * (structmat.hpp:16-31): data holds the kind's body entries, corner the
 * row-major Babd corner block.  on_device = 1: data/corner are device
 * pointers BORROWED by a handle (they must stay alive and unchanged until
 * psg_release); on_device = 0: host pointers, copied into the handle. */
typedef struct {
  int kind, n, m, s, r;
  const double* data;
  size_t data_len;
  const double* corner;
  int corner_rows, corner_cols;
  int on_device;
} psg_desc;

/* Mirrors parsol::SolveStats (parfact.hpp:24-30) plus the GPU certificate. */
typedef struct {
  double factor_seconds;
  double phase1_seconds; /* condense (speculative interface) */
  double phase2_seconds; /* reduced solve */
  double phase3_seconds; /* back-substitution + certificate */
  long long reduced_ops; /* multiply-adds of phase 2 (function of q only) */
  double certificate;    /* max componentwise backward error over separator rows */
  int speculative;       /* 1: the truncated interface was certified and used */
  int fallbacks;         /* exact re-solves triggered by a failed certificate */
} psg_stats;

typedef struct psg_handle psg_handle;

/* Factor A on p partitions (parallel_factor).  tol is accepted for API
 * parity (the reference uses it only for LuPivot/Qr).  Lu, Lud and (where the
 * reference allows it) CyclicReduction share the same GPU kernels;
 * LuPivot/Qr (and every strategy on the circulant-like kind) run the pivoting
 * engine; Arce returns UnsupportedStructure (no CPU fallback). */
int psg_factor(const psg_desc* A, int p, int strategy, double tol, void* stream,
               psg_handle** out, char* err, size_t errlen);

/* Three-phase solve (solve).  f and x are n-vectors, device pointers when
 * on_device = 1, else host pointers (copied through the handle's device
 * buffers; pinned host memory makes the copies fast and, for large
 * speculative tridiagonal solves without stats, lets f arrive and x leave in
 * overlapping row chunks).  Blocks until the result and its certificate are
 * known.  stats may be NULL. */
int psg_solve(const psg_handle* h, const double* f, double* x, int on_device, void* stream,
              psg_stats* stats, char* err, size_t errlen);

void psg_release(psg_handle* h);

/* Asynchronous solve (device pointers only; the tridiagonal path; other kinds
 * run blocking).  Enqueues the speculative solve on `stream` and returns; x is
 * final in stream order unless its certificate fails, in which case psg_sync
 * re-solves that right-hand side exactly.  Call psg_sync before reading x on
 * the host or reusing f.  timing != 0 records phase events for psg_sync's
 * stats.  Up to 64 solves may be pending; more drain the oldest. */
int psg_solve_async(const psg_handle* h, const double* f, double* x, int timing, void* stream, char* err,
                    size_t errlen);
/* Wait for every pending asynchronous solve, repair failed certificates, and
 * accumulate their statistics (SolveStats semantics: phases add up). */
int psg_sync(const psg_handle* h, psg_stats* stats, char* err, size_t errlen);

/* New matrix values with the structure the handle was factored for (kind, n,
 * m, s, r, corner shape, p): recompute the factorization in place, without
 * re-planning or re-allocating.  The equivalent of parallel_factor on a
 * matrix whose sparsity pattern is unchanged.
 * Pending asynchronous solves: when A comes in a different buffer than the
 * handle's current one (or as host memory, copied into the handle), they are
 * drained first -- certificates checked and failures repaired against the
 * matrix they were enqueued for -- and their statistics are reported by the
 * next psg_sync.  With the same device buffer they stay pending (stream order
 * runs them on the old factor data) and are certified at psg_sync against the
 * buffer's values then: call psg_sync before overwriting A's values in place.
 * Calls on one handle from different streams are ordered: each entry point
 * makes its stream wait for the work previously enqueued on the handle. */
int psg_refactor(psg_handle* h, const psg_desc* A, void* stream, char* err, size_t errlen);

/* Reduced system metadata (ReducedSystem, parfact.hpp:14-22): q kept blocks,
 * scalar dimension, block size k, corner flag. */
int psg_reduced_info(const psg_handle* h, int* q, int* dim, int* k, int* has_corner);
/* Reduced-system layout in position order (ReducedSystem::positions /
 * block_sizes, src/parfact.cpp:72-88): q entries, each a separator (size k)
 * or, for LuPivot / Qr, an adaptive extra (size 1). */
int psg_reduced_layout(const psg_handle* h, int* positions, int* sizes);
/* Dense dim x dim image of the reduced matrix T (ReducedSystem::T), row-major,
 * for every strategy; callers bound dim (the C++ layer: 4096). */
int psg_reduced_dense(const psg_handle* h, double* T, char* err, size_t errlen);
/* Host copies of the reduced matrix T in block form (k x k row-major
 * blocks): diag[q], sub[q] (coupling of block i to i-1; sub[0] = corner
 * coupling when has_corner), super[q] (coupling of block i to i+1).  Any
 * pointer may be NULL. */
int psg_reduced_blocks(const psg_handle* h, double* diag, double* sub, double* super, char* err,
                       size_t errlen);

/* The reduced right-hand side of f on the reference plan (the rrhs that
 * solve() hands to solve_reduced, src/parfact.cpp:205-214): f at the
 * separator rows plus every partition's condensed contribution kept_rhs
 * (LocalFactorization::condense, src/localfact.cpp:765-781), computed by the
 * exact phase-1 kernels; out has dim entries.  Not for LuPivot / Qr handles. */
int psg_reduced_rhs(const psg_handle* h, const double* f, double* out, int on_device, void* stream, char* err,
                    size_t errlen);

/* Solve T x = rhs for the handle's reduced system (solve_reduced), device
 * or host vectors of length dim. */
int psg_solve_reduced(const psg_handle* h, const double* rhs, double* x, int on_device,
                      void* stream, psg_stats* stats, char* err, size_t errlen);

/* plan_partition on the host: body_begin/body_end (p), sep_start (p+1
 * capacity); writes sep_count and sep_size. */
int psg_plan(const psg_desc* A, int p, int* body_begin, int* body_end, int* sep_start,
             int* sep_count, int* sep_size, char* err, size_t errlen);

/* Device residual ||A x - f||_inf / ||f||_inf with the reference's fixed
 * ascending-column summation and no FMA contraction (bit-identical to the
 * reference).  A->on_device must match on_device. */
int psg_residual(const psg_desc* A, const double* x, const double* f, int on_device,
                 void* stream, double* out, char* err, size_t errlen);
int psg_matvec(const psg_desc* A, const double* x, double* y, int on_device, void* stream,
               char* err, size_t errlen); /* host vectors (on_device = 0) are staged through the device */

/* Time-parallel linear IVP trajectory (solve_ivp_parallel): the one-step
 * recursion diag_w y_k = sub_w y_{k-1} + g_k over p windows of N steps,
 * closed by y_0 = y0, solved as one BVP-layout BABD on the device (the chain
 * path).  win: p x (diag_w, sub_w), each m x m row-major (host); g: host,
 * (p N + 1) m = y0 followed by the method right-hand sides g_1 .. g_pN;
 * out: host, (p N + 1) m trajectory.  1 <= m <= 8.  Blocks until done. */
int psg_ode_trajectory(int m, int p, int N, const double* win, const double* g, double* out, void* stream,
                       psg_stats* stats, char* err, size_t errlen);

/* Parareal for linear IVPs (src/parareal.cpp:56-117; the C++ layer
 * include/parsol/parareal.hpp builds the steppers).  Each propagator is a
 * per-window stepper y <- T y + Minv rhs_n, n = 1..S: T and Minv are nmat
 * distinct m x m matrices (row-major), mat[i] picks window i+1's; rhs is
 * p x S x m (host).  1 <= m <= 64.  inits are p x m (window initial values,
 * inits[0] = y0). */
typedef struct psg_pr psg_pr;
int psg_pr_create(int m, int p, const double* y0, int Sf, int nmat_f, const double* Tf, const double* Mf,
                  const int* matf, const double* rhsf, int Sc, int nmat_c, const double* Tc, const double* Mc,
                  const int* matc, const double* rhsc, psg_pr** out, char* err, size_t errlen);
int psg_pr_set_inits(psg_pr* h, const double* inits);
int psg_pr_get_inits(psg_pr* h, double* inits, double* fine); /* fine: (p-1) x m, F_i inits[i-1]; may be NULL */
int psg_pr_coarse_sweep(psg_pr* h, char* err, size_t errlen); /* parareal_init */
int psg_pr_iterate(psg_pr* h, double* update, double* scale, char* err, size_t errlen); /* parareal_iterate */
/* parareal_solve: coarse sweep, then iterations until update <= tol * max(scale, 1e-300); history[k-1] = update. */
int psg_pr_solve(psg_pr* h, double tol, int max_iter, int* iterations, double* history, int* converged,
                 char* err, size_t errlen);
/* propagate(): which = 0 fine, 1 coarse; window i in 1..p; y, out host m-vectors. */
int psg_pr_apply(psg_pr* h, int which, int i, const double* y, double* out, char* err, size_t errlen);
void psg_pr_release(psg_pr* h);

/* BASELINE config generator on the device (same stream mapping and values as
 * oracle/parsol_oracle.c or_generate_config).  Shapes via psg_config_shape. */
int psg_config_shape(int cfg, int size, int* kind, int* n, int* m, int* s, int* r,
                     size_t* data_len, int* corner_rows, int* corner_cols);
int psg_generate_config(int cfg, int size, uint64_t seed, double* data, double* corner,
                        double* f, void* stream, char* err, size_t errlen);

/* make() validation (src/structmat.cpp:153-207, plus the Babd s = m, r = 0
 * layout) and body_entry_count (:64-84) -- host-only, no device work. */
int psg_validate(const psg_desc* A, char* err, size_t errlen);
size_t psg_body_entry_count(int kind, int n, int m, int s, int r);

/* ---- Per-partition local factorization (the reference's LocalFactorization,
 * proj/include/parsol/localfact.hpp:24-125; src/localfact.cpp:84-225 banded
 * Lu/Lud, :266-384 cyclic reduction, :400-700 LuPivot/Qr, :765-875 member
 * operations).  One partition block is factored by one CTA on the device
 * (csrc/psg_local.cu); every field is bit-identical to the reference's.
 * Replaces factor() / factor_lu / factor_lud / factor_cyclic_reduction /
 * factor_lu_pivot / factor_qr (localfact.hpp:118-125).  ARCE returns
 * UnsupportedStructure. ---- */
typedef struct {
  int kind, m, s, r;      /* matrix kind fields the block was cut from (CR needs them) */
  int L, k0, k1;          /* body rows, left / right separator sizes */
  int env_s, env_r;       /* envelope half-bandwidths (PartitionBlock::env_s/env_r) */
  const double* env;      /* L x (env_s + 1 + env_r), diagonal-aligned rows (host) */
  const double* b0;       /* L x k0 row-major (host); NULL when k0 = 0 */
  const double* c0;       /* L x k0 */
  const double* b1;       /* L x k1 */
  const double* c1;       /* L x k1 */
  const double* a_right;  /* k1 x k1 */
} psg_block;

typedef struct psg_local psg_local;

typedef struct {
  int strategy, L, k0, k1, env_s, env_r;
  int core;        /* 1 banded (Lu/Lud), 2 cyclic reduction, 3 dense recorded (LuPivot/Qr) */
  int cr_levels;   /* CR: reduction levels */
  int g;           /* CR: block size */
  int n_elims;     /* CR: eliminations */
  int n_rem;       /* CR: remaining block rows (1 or 2) */
  int rem[2];      /* CR: their block indices */
  int dim;         /* k0 + L + k1 */
  int n_a_order;   /* dense: retired pivots */
  int n_extras;    /* dense: deferred pivots (adaptive extras) */
} psg_local_info;

/* Fields readable with psg_local_read (doubles unless noted int). */
enum psg_local_field {
  PSG_LF_FAC = 0,        /* banded: eliminated envelope L x w */
  PSG_LF_DVEC,           /* Lud: pivots (L) */
  PSG_LF_Z, PSG_LF_W,    /* L x k0 */
  PSG_LF_Y, PSG_LF_V,    /* L x k1 */
  PSG_LF_ALPHA1, PSG_LF_ALPHA2, PSG_LF_BETA, PSG_LF_GAMMA,
  PSG_LF_KEPT,           /* kept_dim x kept_dim */
  PSG_LF_CR_ELIM_IDX,    /* int, n_elims x (j, left, right) */
  PSG_LF_CR_ELIM_MAT,    /* n_elims x (ml, mr, a, c, dinv), each g x g */
  PSG_LF_CR_D2, PSG_LF_CR_D2INV,  /* (n_rem g)^2 */
  PSG_LF_CR_CMAT,        /* (n_rem g) x (k0 + k1) */
  PSG_LF_CR_RMAT_D2INV,  /* (k0 + k1) x (n_rem g) */
  PSG_LF_WMID, PSG_LF_LMAT, PSG_LF_LINV, /* dense frame, dim x dim */
  PSG_LF_A_ORDER,        /* int, n_a_order x (row, col) */
  PSG_LF_KEPT_ROWS, PSG_LF_KEPT_COLS,    /* int, kept_dim */
  PSG_LF_EXTRA_POS,      /* int, n_extras */
  PSG_LF_EXTRA_ALPHA     /* n_extras */
};

int psg_local_factor(const psg_block* blk, int strategy, double tol, void* stream, psg_local** out, char* err,
                     size_t errlen);
int psg_local_query(const psg_local* lf, psg_local_info* info);
/* Copy one field to host memory of `count` elements (returns DimensionMismatch if too small). */
int psg_local_read(const psg_local* lf, int field, void* out, size_t count, char* err, size_t errlen);
/* condense (phase 1): f_body (L) -> ghat (L), kept_rhs (kept_dim); host vectors. */
int psg_local_condense(const psg_local* lf, const double* f_body, double* ghat, double* kept_rhs, char* err,
                       size_t errlen);
/* backsolve (phase 3): ghat (L), x_kept (kept_dim) -> x (L). */
int psg_local_backsolve(const psg_local* lf, const double* ghat, const double* x_kept, double* x, char* err,
                        size_t errlen);
/* which = 0: apply_N_inv, 1: apply_S_inv (body vectors of length L). */
int psg_local_apply(const psg_local* lf, int which, const double* rhs, double* out, char* err, size_t errlen);
void psg_local_release(psg_local* lf);

/* Dense reduced solve of an explicit n x n matrix T (row-major, host) --
 * solve_reduced(const ReducedSystem&) for a ReducedSystem without a device
 * handle (src/parfact.cpp:134-184): LU with partial pivoting on the device,
 * bit-identical to the reference; *ops receives its multiply-add count.
 * SingularReducedSystem on a zero pivot column. */
int psg_dense_solve(int n, const double* T, const double* rhs, double* x, long long* ops, void* stream, char* err,
                    size_t errlen);

/* Options (per handle): */
enum psg_option {
  PSG_OPT_SPECULATIVE = 0, /* 1 (default): truncated interface + certificate; 0: exact */
  PSG_OPT_HALO = 1,        /* truncation depth H in rows (default 32) */
  PSG_OPT_CERT_TOL = 2,    /* certificate threshold (default 1e-14) */
  PSG_OPT_BODY_CERT = 3    /* 1: the tridiagonal certificate also covers every body row (componentwise
                              backward error from the rows K3 already holds; default 0: separator rows) */
};
int psg_set_option(psg_handle* h, int option, double value);

/* Wait until the factorization enqueued by psg_factor / psg_refactor is
 * complete; device_seconds (may be NULL) receives its device time. */
int psg_factor_wait(const psg_handle* h, double* device_seconds);

/* Number of kernels the last psg_factor / psg_solve on this handle launched. */
int psg_last_launches(const psg_handle* h, int* factor_launches, int* solve_launches);

/* Inspection of the speculative tridiagonal factor (tests / tools): copy an
 * internal device buffer to host memory of `cap` doubles.  what = 1: the
 * speculative reduced diagonal (nsep); other values: -1 (the separator
 * weights of earlier versions are no longer formed).  Returns the count
 * copied, -count if cap is too small, -1 on a CUDA error. */
long psg_debug_buffer(const psg_handle* h, int what, double* out, long cap);

/* Version string including the hash of the sources the library was built
 * from (paper_0912_3678_b200/build.py source_hash). */
const char* psg_version(void);

#ifdef __cplusplus
}
#endif
#endif
