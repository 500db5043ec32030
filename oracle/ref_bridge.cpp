// ref_bridge.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" bridge onto the UNMODIFIED reference `parsol` library, compiled
// from /root/reference/proj/src by oracle/Makefile with -Dparsol=parsol_ref
// into oracle/_ref/libparsol_ref.so.  Used (1) to pin the C restatement in
// parsol_oracle.c (tests/test_oracle.py), (2) to generate the golden fixtures
// (tests/golden/make_golden.py) and (3) as the CPU baseline timed by
// bench.py (`--impl reference`, `cpu_baseline.kind = "reference"`).
//
// No reference source is copied here: this file only calls the reference's
// public API (proj/include/parsol/*.hpp).  The StructuredMatrix is built by
// aggregate initialisation (its fields are public, structmat.hpp:33-43) so
// that the BASELINE config 4 BABD layout s = m, r = 0 -- which make()
// rejects at src/structmat.cpp:173-174 -- can be fed to the unmodified
// factor/solve path.
#include <omp.h>

#include <algorithm>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "parsol/errors.hpp"
#include "parsol/io.hpp"
#include "parsol/odeparallel.hpp"
#include "parsol/parareal.hpp"
#include "parsol/parfact.hpp"
#include "parsol/seqref.hpp"
#include "parsol/structmat.hpp"

using namespace parsol;  // expands to parsol_ref via -Dparsol=parsol_ref

namespace {

struct RefMat {
  StructuredMatrix A;
};

struct RefFact {
  ParallelFactorization F;
};

int report(const std::exception& e, char* err, size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
  if (auto* pe = dynamic_cast<const Error*>(&e)) return 1 + int(pe->code());
  return 1000;
}

}  // namespace

extern "C" {

void* ref_mat_create(int kind, int n, int m, int s, int r, const double* data, size_t len,
                     const double* corner, int corner_rows, int corner_cols) {
  auto* h = new RefMat;
  h->A.kind = Kind(kind);
  h->A.n = n;
  h->A.m = m;
  h->A.s = s;
  h->A.r = r;
  h->A.data.assign(data, data + len);
  if (corner) h->A.corner.assign(corner, corner + size_t(corner_rows) * corner_cols);
  h->A.corner_rows = corner_rows;
  h->A.corner_cols = corner_cols;
  return h;
}

void ref_mat_destroy(void* h) { delete static_cast<RefMat*>(h); }

int ref_set_threads(int t) {
  if (t > 0) omp_set_num_threads(t);
  return omp_get_max_threads();
}

int ref_factor(void* hm, int p, int strategy, void** out, double* seconds, char* err,
               size_t errlen) {
  try {
    auto* f = new RefFact;
    f->F = parallel_factor(static_cast<RefMat*>(hm)->A, p, Strategy(strategy));
    if (seconds) *seconds = f->F.factor_seconds;
    *out = f;
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

int ref_factor_tol(void* hm, int p, int strategy, double tol, void** out, char* err, size_t errlen) {
  try {
    auto* f = new RefFact;
    f->F = parallel_factor(static_cast<RefMat*>(hm)->A, p, Strategy(strategy), tol);
    *out = f;
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

// ReducedSystem positions / block sizes in position order (src/parfact.cpp:72-88)
int ref_fact_layout(void* hf, int* positions, int* sizes) {
  auto& R = static_cast<RefFact*>(hf)->F.reduced;
  for (int j = 0; j < R.q; ++j) {
    positions[j] = R.positions[j];
    sizes[j] = R.block_sizes[j];
  }
  return 0;
}

void ref_fact_destroy(void* h) { delete static_cast<RefFact*>(h); }

int ref_fact_dims(void* hf, int* q, int* dim) {
  auto& R = static_cast<RefFact*>(hf)->F.reduced;
  *q = R.q;
  *dim = R.dim;
  return 0;
}

int ref_fact_T(void* hf, double* T) {
  auto& R = static_cast<RefFact*>(hf)->F.reduced;
  std::memcpy(T, R.T.a.data(), sizeof(double) * R.T.a.size());
  return 0;
}

int ref_fact_local(void* hf, int i, double* alpha1, double* alpha2, double* beta, double* gamma) {
  auto& lf = static_cast<RefFact*>(hf)->F.locals[i];
  auto put = [](double* dst, const DenseMatrix& M) {
    if (dst && !M.a.empty()) std::memcpy(dst, M.a.data(), sizeof(double) * M.a.size());
  };
  put(alpha1, lf.alpha1);
  put(alpha2, lf.alpha2);
  put(beta, lf.beta);
  put(gamma, lf.gamma);
  return 0;
}

int ref_solve(void* hf, const double* f, double* x, size_t n, double* phase_seconds,
              long long* reduced_ops, char* err, size_t errlen) {
  try {
    SolveStats st;
    Vector fv(f, f + n);
    Vector xv = solve(static_cast<RefFact*>(hf)->F, fv, &st);
    std::memcpy(x, xv.data(), sizeof(double) * n);
    if (phase_seconds) {
      phase_seconds[0] = st.phase1_seconds;
      phase_seconds[1] = st.phase2_seconds;
      phase_seconds[2] = st.phase3_seconds;
    }
    if (reduced_ops) *reduced_ops = st.reduced_ops;
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

int ref_solve_sequential(void* hm, const double* f, double* x, size_t n, char* err,
                         size_t errlen) {
  try {
    Vector fv(f, f + n);
    Vector xv = solve_sequential(static_cast<RefMat*>(hm)->A, fv);
    std::memcpy(x, xv.data(), sizeof(double) * n);
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

double ref_residual(void* hm, const double* x, const double* f, size_t n) {
  Vector xv(x, x + n), fv(f, f + n);
  return residual(static_cast<RefMat*>(hm)->A, xv, fv);
}

// generate_random (src/structmat.cpp:282-333) through the reference itself.
int ref_generate_random(int kind, int n, int m, int s, int r, unsigned long long seed, double dominance,
                        double* data, double* corner, char* err, size_t errlen) {
  try {
    StructuredMatrix A = generate_random(Kind(kind), n, m, s, r, seed, dominance);
    std::memcpy(data, A.data.data(), sizeof(double) * A.data.size());
    if (!A.corner.empty() && corner) std::memcpy(corner, A.corner.data(), sizeof(double) * A.corner.size());
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

// STRUCTMAT / VEC text through the reference writer / parser (src/io.cpp):
// returns the byte length (writing at most cap bytes), or -1 - error code.
long ref_write_matrix(void* hm, const char* comment, char* out, size_t cap) {
  std::vector<std::string> c;
  if (comment) c.emplace_back(comment);
  const std::string s = write_matrix(static_cast<RefMat*>(hm)->A, c);
  std::memcpy(out, s.data(), std::min(cap, s.size()));
  return (long)s.size();
}

long ref_write_vector(const double* v, size_t n, const char* comment, char* out, size_t cap) {
  std::vector<std::string> c;
  if (comment) c.emplace_back(comment);
  const std::string s = write_vector(Vector(v, v + n), c);
  std::memcpy(out, s.data(), std::min(cap, s.size()));
  return (long)s.size();
}

// parse a STRUCTMAT text with the reference parser: 0 and a new matrix handle, or 1 + Errc
int ref_parse_matrix(const char* text, size_t len, void** out, char* err, size_t errlen) {
  try {
    auto* h = new RefMat;
    h->A = parse_matrix(std::string(text, len));
    *out = h;
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

int ref_mat_dims(void* hm, int* kind, int* n, int* m, int* s, int* r, size_t* len, double* data) {
  const auto& A = static_cast<RefMat*>(hm)->A;
  *kind = int(A.kind);
  *n = A.n;
  *m = A.m;
  *s = A.s;
  *r = A.r;
  *len = A.data.size();
  if (data) std::memcpy(data, A.data.data(), sizeof(double) * A.data.size());
  return 0;
}

// The reference's time-parallel IVP solver (src/odeparallel.cpp:184-252) with
// the forcing given as a C callback g(t, out[m], ctx); parallel = 0 runs
// solve_ivp_sequential.  out: (p N + 1) m trajectory values.
int ref_ode_solve(int m, const double* L, const double* y0, double t0, double T, int p, int N, int method,
                  void (*g)(double, double*, void*), void* ctx, int parallel, double* out, char* err,
                  size_t errlen) {
  try {
    IVProblem prob;
    prob.L = DenseMatrix(m, m);
    std::memcpy(prob.L.a.data(), L, sizeof(double) * m * m);
    prob.y0.assign(y0, y0 + m);
    prob.t0 = t0;
    prob.T = T;
    if (g)
      prob.g = [g, ctx, m](double t) {
        Vector v(m, 0.0);
        g(t, v.data(), ctx);
        return v;
      };
    TimeGrid grid = coarse_mesh(t0, T, p, N);
    OdeMethod meth = method == 0 ? OdeMethod::ImplicitEuler : OdeMethod::Trapezoidal;
    Trajectory tr = parallel ? solve_ivp_parallel(prob, grid, meth) : solve_ivp_sequential(prob, grid, meth);
    std::memcpy(out, tr.flat.data(), sizeof(double) * tr.flat.size());
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

int ref_plan(void* hm, int p, int* body_begin, int* body_end, int* sep_start, int* sep_count,
             int* sep_size, char* err, size_t errlen) {
  try {
    PartitionPlan plan = plan_partition(static_cast<RefMat*>(hm)->A, p);
    for (int i = 0; i < plan.p; ++i) {
      body_begin[i] = plan.body_ranges[i].first;
      body_end[i] = plan.body_ranges[i].second;
    }
    for (int j = 0; j < plan.sep_count(); ++j) sep_start[j] = plan.separator_starts[j];
    *sep_count = plan.sep_count();
    *sep_size = plan.sep_size;
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

// Parareal through the reference (src/parareal.cpp:94-120): same arguments as
// psg_parareal_solve in libparsol_b200.
int ref_parareal_solve(int m, const double* L, const double* y0, double t0, double T, int p, int N,
                       void (*g)(double, double*, void*), void* ctx, int fkind, int fmethod, int fsteps, int ckind,
                       int cmethod, int csteps, double tol, int max_iter, double* inits, double* history,
                       int history_cap, int* iterations, int* converged, char* err, size_t errlen) {
  try {
    IVProblem prob;
    prob.L = DenseMatrix(m, m);
    std::copy(L, L + size_t(m) * m, prob.L.a.begin());
    prob.y0.assign(y0, y0 + m);
    prob.t0 = t0;
    prob.T = T;
    if (g)
      prob.g = [g, ctx, m](double t) {
        Vector v(m, 0.0);
        g(t, v.data(), ctx);
        return v;
      };
    auto prop = [](int kind, int method, int steps) {
      Propagator P;
      P.kind = PropagatorKind(kind);
      P.method = method == 0 ? OdeMethod::ImplicitEuler : OdeMethod::Trapezoidal;
      P.steps = steps;
      return P;
    };
    const TimeGrid grid = coarse_mesh(t0, T, p, N);
    const PararealResult r = parareal_solve(prob, grid, prop(fkind, fmethod, fsteps), prop(ckind, cmethod, csteps),
                                            tol, max_iter);
    for (int i = 0; i < p; ++i) std::copy(r.inits[i].begin(), r.inits[i].end(), inits + size_t(i) * m);
    for (int k = 0; k < int(r.history.size()) && k < history_cap; ++k) history[k] = r.history[k];
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

int ref_expm(int m, const double* L, double t, double* out, char* err, size_t errlen) {
  try {
    DenseMatrix A(m, m);
    std::copy(L, L + size_t(m) * m, A.a.begin());
    const DenseMatrix E = matrix_exponential(A, t);
    std::copy(E.a.begin(), E.a.end(), out);
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

}  // extern "C"
