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
#include "parsol/localfact.hpp"
#include "parsol/partition.hpp"
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

struct RefBlock {
  PartitionBlock B;
};

struct RefLocal {
  LocalFactorization lf;
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

// ---- per-partition pieces (localfact.hpp public API) ----------------------

void* ref_block_extract(void* hm, int p, int i, int* dims, char* err, size_t errlen) {
  try {
    const StructuredMatrix& A = static_cast<RefMat*>(hm)->A;
    PartitionPlan plan = plan_partition(A, p);
    auto* b = new RefBlock{extract_block(A, plan, i)};
    dims[0] = b->B.L;
    dims[1] = b->B.k0;
    dims[2] = b->B.k1;
    dims[3] = b->B.env_s;
    dims[4] = b->B.env_r;
    return b;
  } catch (const std::exception& e) {
    report(e, err, errlen);
    return nullptr;
  }
}

void* ref_block_create(int kind, int m, int s, int r, int L, int k0, int k1, int es, int er, const double* env,
                       const double* b0, const double* c0, const double* b1, const double* c1, const double* ar) {
  auto* b = new RefBlock;
  PartitionBlock& B = b->B;
  B.index = 2;
  B.kind = Kind(kind);
  B.m = m;
  B.s = s;
  B.r = r;
  B.L = L;
  B.k0 = k0;
  B.k1 = k1;
  B.env_s = es;
  B.env_r = er;
  B.env.assign(env, env + size_t(L) * (es + 1 + er));
  auto mat = [](int rows, int cols, const double* src) {
    DenseMatrix M(rows, cols);
    if (src && rows * cols) std::memcpy(M.a.data(), src, sizeof(double) * rows * cols);
    return M;
  };
  B.b0 = mat(L, k0, b0);
  B.c0 = mat(L, k0, c0);
  B.b1 = mat(L, k1, b1);
  B.c1 = mat(L, k1, c1);
  if (k1) B.a_right = mat(k1, k1, ar);
  return b;
}

int ref_block_arrays(void* hb, double* env, double* b0, double* c0, double* b1, double* c1, double* ar) {
  const PartitionBlock& B = static_cast<RefBlock*>(hb)->B;
  auto put = [](double* dst, const std::vector<double>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(double) * v.size());
  };
  put(env, B.env);
  put(b0, B.b0.a);
  put(c0, B.c0.a);
  put(b1, B.b1.a);
  put(c1, B.c1.a);
  put(ar, B.a_right.a);
  return 0;
}

void ref_block_destroy(void* hb) { delete static_cast<RefBlock*>(hb); }

int ref_local_factor(void* hb, int strategy, double tol, void** out, char* err, size_t errlen) {
  try {
    *out = new RefLocal{factor(Strategy(strategy), static_cast<RefBlock*>(hb)->B, tol)};
    return 0;
  } catch (const std::exception& e) {
    *out = nullptr;
    return report(e, err, errlen);
  }
}

void ref_local_destroy(void* hl) { delete static_cast<RefLocal*>(hl); }

// dims: [kept_dim, n_extras, cr_levels, core(1 banded, 2 cyclic, 3 dense), dim, n_a_order, n_elims, g, n_rem]
int ref_local_dims(void* hl, int* d) {
  const LocalFactorization& lf = static_cast<RefLocal*>(hl)->lf;
  d[0] = lf.kept_dim();
  d[1] = int(lf.extras.size());
  d[2] = lf.cr_levels;
  d[3] = int(lf.core.index());
  d[4] = lf.k0 + lf.L + lf.k1;
  d[5] = d[6] = d[7] = d[8] = 0;
  if (auto* dc = std::get_if<LocalFactorization::DenseCore>(&lf.core)) d[5] = int(dc->a_order.size());
  if (auto* cc = std::get_if<LocalFactorization::CyclicCore>(&lf.core)) {
    d[6] = int(cc->elims.size());
    d[7] = cc->g;
    d[8] = int(cc->rem.size());
  }
  return 0;
}

// field numbering = enum psg_local_field (include/psg.h); returns the count written
long ref_local_field(void* hl, int field, void* out) {
  const LocalFactorization& lf = static_cast<RefLocal*>(hl)->lf;
  auto put = [out](const std::vector<double>& v) {
    if (!v.empty()) std::memcpy(out, v.data(), sizeof(double) * v.size());
    return long(v.size());
  };
  auto puti = [out](const std::vector<int>& v) {
    if (!v.empty()) std::memcpy(out, v.data(), sizeof(int) * v.size());
    return long(v.size());
  };
  const auto* bc = std::get_if<LocalFactorization::BandedCore>(&lf.core);
  const auto* cc = std::get_if<LocalFactorization::CyclicCore>(&lf.core);
  const auto* dc = std::get_if<LocalFactorization::DenseCore>(&lf.core);
  switch (field) {
    case 0: return bc ? put(bc->fac) : 0;
    case 1: return bc ? put(bc->dvec) : 0;
    case 2: return put(lf.z.a);
    case 3: return put(lf.w.a);
    case 4: return put(lf.y.a);
    case 5: return put(lf.v.a);
    case 6: return put(lf.alpha1.a);
    case 7: return put(lf.alpha2.a);
    case 8: return put(lf.beta.a);
    case 9: return put(lf.gamma.a);
    case 10: return put(lf.kept.a);
    case 11: {
      if (!cc) return 0;
      std::vector<int> v;
      for (auto& e : cc->elims) v.insert(v.end(), {e.j, e.lnb, e.rnb});
      return puti(v);
    }
    case 12: {
      if (!cc) return 0;
      std::vector<double> v;
      for (auto& e : cc->elims)
        for (const DenseMatrix* M : {&e.ml, &e.mr, &e.a, &e.c, &e.dinv}) v.insert(v.end(), M->a.begin(), M->a.end());
      return put(v);
    }
    case 13: return cc ? put(cc->d2.a) : 0;
    case 14: return cc ? put(cc->d2inv.a) : 0;
    case 15: return cc ? put(cc->cmat.a) : 0;
    case 16: return cc ? put(cc->rmat_d2inv.a) : 0;
    case 17: return dc ? put(dc->Wmid.a) : 0;
    case 18: return dc ? put(dc->Lmat.a) : 0;
    case 19: return dc ? put(dc->Linv.a) : 0;
    case 20: {
      if (!dc) return 0;
      std::vector<int> v;
      for (auto& [r, c] : dc->a_order) v.insert(v.end(), {r, c});
      return puti(v);
    }
    case 21: return dc ? puti(dc->kept_rows) : 0;
    case 22: return dc ? puti(dc->kept_cols) : 0;
    case 23: {
      std::vector<int> v;
      for (auto& x : lf.extras) v.push_back(x.position);
      return puti(v);
    }
    case 24: {
      std::vector<double> v;
      for (auto& x : lf.extras) v.push_back(x.alpha);
      return put(v);
    }
  }
  return -1;
}

// op 0 condense (ghat -> out, kept_rhs -> out2), 1 backsolve(in, in2) -> out,
// 2 apply_N_inv, 3 apply_S_inv
int ref_local_op(void* hl, int op, const double* in, const double* in2, double* out, double* out2, char* err,
                 size_t errlen) {
  try {
    const LocalFactorization& lf = static_cast<RefLocal*>(hl)->lf;
    const Vector v(in, in + lf.L);
    Vector r;
    if (op == 0) {
      Vector ghat, kr;
      lf.condense(v, ghat, kr);
      std::memcpy(out2, kr.data(), sizeof(double) * kr.size());
      r = ghat;
    } else if (op == 1) {
      r = lf.backsolve(v, Vector(in2, in2 + lf.kept_dim()));
    } else if (op == 2) {
      r = lf.apply_N_inv(v);
    } else {
      r = lf.apply_S_inv(v);
    }
    std::memcpy(out, r.data(), sizeof(double) * r.size());
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

// which 0: F_loc, 1: T_loc, 2: G_loc (dim x dim)
int ref_local_dense(void* hl, int which, double* out) {
  const LocalFactorization& lf = static_cast<RefLocal*>(hl)->lf;
  const DenseMatrix M = which == 0 ? lf.dense_F_loc() : which == 1 ? lf.dense_T_loc() : lf.dense_G_loc();
  std::memcpy(out, M.a.data(), sizeof(double) * M.a.size());
  return 0;
}

// solve_reduced on a hand-built ReducedSystem with a dense T
int ref_solve_reduced_dense(int n, const double* T, const double* rhs, double* x, long long* ops, char* err,
                            size_t errlen) {
  try {
    ReducedSystem R;
    R.q = n;
    R.dim = n;
    R.T = DenseMatrix(n, n);
    std::memcpy(R.T.a.data(), T, sizeof(double) * size_t(n) * n);
    SolveStats st;
    Vector xv = solve_reduced(R, Vector(rhs, rhs + n), &st);
    std::memcpy(x, xv.data(), sizeof(double) * n);
    *ops = st.reduced_ops;
    return 0;
  } catch (const std::exception& e) {
    return report(e, err, errlen);
  }
}

}  // extern "C"
