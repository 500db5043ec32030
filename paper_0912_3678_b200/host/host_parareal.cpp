// host_parareal.cpp -- Parareal (include/parsol/parareal.hpp; reference
// proj/src/parareal.cpp, paper §4).  The host builds each propagator's
// per-window stepper (the reference's window discretisation,
// src/odeparallel.cpp:69-110, with diag^{-1} formed once per distinct step
// size) and the forcing samples; every propagation, the coarse sweep and the
// stopping norms run on the GPU through the psg_pr_* C ABI.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <string>

#include "parsol/errors.hpp"
#include "parsol/parareal.hpp"
#include "psg.h"

namespace parsol {

namespace {

struct StepperHost {
  int S = 1;
  std::vector<double> T, M;  // distinct m x m matrices
  std::vector<int> mat;      // per window
  std::vector<double> rhs;   // p x S x m (empty: no forcing)
  int nmat() const { return int(mat.empty() ? 0 : *std::max_element(mat.begin(), mat.end()) + 1); }
};

std::uint64_t bits(double v) {
  std::uint64_t b;
  std::memcpy(&b, &v, sizeof b);
  return b;
}

void append(std::vector<double>& dst, const DenseMatrix& A) { dst.insert(dst.end(), A.a.begin(), A.a.end()); }

// One-step method over each window with `steps` steps (src/parareal.cpp:13-19:
// the window's own grid coarse_mesh({tau_{i-1}, tau_i}, steps)).
StepperHost discrete_stepper(const IVProblem& prob, const TimeGrid& grid, OdeMethod method, int steps) {
  const int p = grid.windows(), m = prob.dim();
  if (steps < 1) fail(Errc::InvalidParameter, "propagator steps must be >= 1");
  StepperHost st;
  st.S = steps;
  st.mat.resize(p);
  if (prob.g) st.rhs.assign(std::size_t(p) * steps * m, 0.0);
  std::map<std::uint64_t, int> by_h;
  std::vector<int> first;  // a window of each distinct step size
  for (int i = 1; i <= p; ++i) {
    const double h = (grid.tau[i] - grid.tau[i - 1]) / steps;  // coarse_mesh's h (src/odeparallel.cpp:39-41)
    auto it = by_h.find(bits(h));
    if (it == by_h.end()) {
      it = by_h.emplace(bits(h), int(first.size())).first;
      first.push_back(i);
    }
    st.mat[i - 1] = it->second;
  }
  std::vector<std::string> errs(p);
  std::vector<int> codes(p, -1);
#pragma omp parallel for schedule(static)
  for (int i = 1; i <= (prob.g ? p : 0); ++i) {
    try {
      const TimeGrid local = coarse_mesh({grid.tau[i - 1], grid.tau[i]}, steps);
      const WindowSystem W = discretize_window(prob, local, 1, method);
      std::copy(W.gvec.begin(), W.gvec.end(), st.rhs.begin() + std::size_t(i - 1) * steps * m);
    } catch (const Error& e) {
      codes[i - 1] = int(e.code());
      errs[i - 1] = e.detail();
    }
  }
  for (int i = 0; i < p; ++i)
    if (codes[i] >= 0) fail(Errc(codes[i]), errs[i]);
  for (int i : first) {
    const TimeGrid local = coarse_mesh({grid.tau[i - 1], grid.tau[i]}, steps);
    IVProblem hom = prob;
    hom.g = nullptr;
    const WindowSystem W = discretize_window(hom, local, 1, method);
    const DenseMatrix Minv = W.diag_lu.solve(DenseMatrix::identity(m));
    append(st.M, Minv);
    append(st.T, matmul(Minv, W.sub));
  }
  return st;
}

struct PrHandle {
  psg_pr* h = nullptr;
  ~PrHandle() { psg_pr_release(h); }
};

std::unique_ptr<PrHandle> make_pr(const IVProblem& prob, const StepperHost& F, const StepperHost& G, int p) {
  auto H = std::make_unique<PrHandle>();
  char err[256] = {0};
  const int rc = psg_pr_create(prob.dim(), p, prob.y0.data(), F.S, F.nmat(), F.T.data(), F.M.data(), F.mat.data(),
                               F.rhs.empty() ? nullptr : F.rhs.data(), G.S, G.nmat(), G.T.data(), G.M.data(),
                               G.mat.data(), G.rhs.empty() ? nullptr : G.rhs.data(), &H->h, err, sizeof err);
  if (rc) fail(Errc(rc - 1), err);
  return H;
}

void check(int rc, const char* err) {
  if (rc) fail(Errc(rc - 1), err);
}

// The propagator as a stepper.  MatrixExponential: one step with
// T = e^{delta L}, M = I and rhs = the forcing's particular solution by the
// discrete rule (src/parareal.cpp:33-43), computed on the GPU.
StepperHost stepper_of(const Propagator& P, const IVProblem& prob, const TimeGrid& grid) {
  if (P.kind != PropagatorKind::MatrixExponential) return discrete_stepper(prob, grid, P.method, P.steps);
  const int p = grid.windows(), m = prob.dim();
  StepperHost st;
  st.S = 1;
  st.mat.resize(p);
  std::map<std::uint64_t, int> by_d;
  for (int i = 1; i <= p; ++i) {
    const double delta = grid.tau[i] - grid.tau[i - 1];
    auto it = by_d.find(bits(delta));
    if (it == by_d.end()) {
      it = by_d.emplace(bits(delta), int(by_d.size())).first;
      append(st.T, matrix_exponential(prob.L, delta));
      append(st.M, DenseMatrix::identity(m));
    }
    st.mat[i - 1] = it->second;
  }
  if (prob.g) {
    st.rhs.assign(std::size_t(p) * m, 0.0);
    const StepperHost D = discrete_stepper(prob, grid, P.method, P.steps);
    auto H = make_pr(prob, D, D, p);
    char err[256] = {0};
    const Vector zero(m, 0.0);
    for (int i = 1; i <= p; ++i)
      check(psg_pr_apply(H->h, 0, i, zero.data(), st.rhs.data() + std::size_t(i - 1) * m, err, sizeof err), err);
  }
  return st;
}

void check_problem(const IVProblem& prob) {
  if (prob.L.rows != prob.L.cols) fail(Errc::DimensionMismatch, "L must be square");
  if (int(prob.y0.size()) != prob.dim()) fail(Errc::DimensionMismatch, "y0 length");
}

std::vector<Vector> unflatten(const std::vector<double>& flat, int rows, int m) {
  std::vector<Vector> out(rows);
  for (int i = 0; i < rows; ++i) out[i].assign(flat.begin() + std::size_t(i) * m, flat.begin() + std::size_t(i + 1) * m);
  return out;
}

}  // namespace

Vector propagate(const Propagator& P, const IVProblem& prob, const TimeGrid& grid, int i, const Vector& y) {
  if (i < 1 || i > grid.windows()) fail(Errc::IndexOutOfRange, "window index");
  if (int(y.size()) != prob.dim()) fail(Errc::DimensionMismatch, "initial value length");
  check_problem(prob);
  const TimeGrid one = coarse_mesh({grid.tau[i - 1], grid.tau[i]}, grid.N);
  const StepperHost st = stepper_of(P, prob, one);
  auto H = make_pr(prob, st, st, 1);
  Vector out(prob.dim());
  char err[256] = {0};
  check(psg_pr_apply(H->h, 0, 1, y.data(), out.data(), err, sizeof err), err);
  return out;
}

PararealState parareal_init(const IVProblem& prob, const TimeGrid& grid, const Propagator& coarse) {
  check_problem(prob);
  const int p = grid.windows(), m = prob.dim();
  const StepperHost G = stepper_of(coarse, prob, grid);
  auto H = make_pr(prob, G, G, p);
  char err[256] = {0};
  check(psg_pr_coarse_sweep(H->h, err, sizeof err), err);
  std::vector<double> flat(std::size_t(p) * m);
  check(psg_pr_get_inits(H->h, flat.data(), nullptr), "copy");
  PararealState st;
  st.k = 0;
  st.inits = unflatten(flat, p, m);
  return st;
}

PararealState parareal_iterate(const PararealState& state, const Propagator& fine, const Propagator& coarse,
                               const IVProblem& prob, const TimeGrid& grid) {
  check_problem(prob);
  const int p = int(state.inits.size()), m = prob.dim();
  if (p != grid.windows()) fail(Errc::DimensionMismatch, "state does not match the grid");
  auto H = make_pr(prob, stepper_of(fine, prob, grid), stepper_of(coarse, prob, grid), p);
  std::vector<double> flat(std::size_t(p) * m), fc(std::size_t(std::max(p - 1, 0)) * m);
  for (int i = 0; i < p; ++i) std::copy(state.inits[i].begin(), state.inits[i].end(), flat.begin() + std::size_t(i) * m);
  check(psg_pr_set_inits(H->h, flat.data()), "copy");
  char err[256] = {0};
  double upd = 0;
  check(psg_pr_iterate(H->h, &upd, nullptr, err, sizeof err), err);
  check(psg_pr_get_inits(H->h, flat.data(), fc.data()), "copy");
  PararealState next;
  next.k = state.k + 1;
  next.history = state.history;
  next.history.push_back(upd);
  next.inits = unflatten(flat, p, m);
  next.fine_cache = unflatten(fc, p - 1, m);
  return next;
}

PararealResult parareal_solve(const IVProblem& prob, const TimeGrid& grid, const Propagator& fine,
                              const Propagator& coarse, double tol, int max_iter) {
  if (tol <= 0) fail(Errc::InvalidParameter, "tol must be positive");
  check_problem(prob);
  const int p = grid.windows(), m = prob.dim();
  if (max_iter < 0) max_iter = 2 * p;
  auto H = make_pr(prob, stepper_of(fine, prob, grid), stepper_of(coarse, prob, grid), p);
  std::vector<double> hist(std::max(max_iter, 1)), flat(std::size_t(p) * m);
  int iters = 0, conv = 1;
  char err[256] = {0};
  check(psg_pr_solve(H->h, tol, max_iter, &iters, hist.data(), &conv, err, sizeof err), err);
  check(psg_pr_get_inits(H->h, flat.data(), nullptr), "copy");
  PararealResult res;
  res.inits = unflatten(flat, p, m);
  res.iterations = iters;
  res.history.assign(hist.begin(), hist.begin() + iters);
  res.converged = conv != 0;
  return res;
}

// e^{tL}: scale by 2^-s until ||tL|| <= 1/2, degree-7 diagonal Pade
// approximant (numerator U + V, denominator V - U with the even / odd parts of
// the Pade polynomial), then square s times.
DenseMatrix matrix_exponential(const DenseMatrix& L, double t) {
  if (L.rows != L.cols) fail(Errc::DimensionMismatch, "expm needs square input");
  const int m = L.rows;
  DenseMatrix B = scale(L, t);
  double nrm = inf_norm(B);
  if (!std::isfinite(nrm)) fail(Errc::ExpmFailure, "non-finite input");
  int s = 0;
  while (nrm > 0.5) {
    nrm /= 2;
    if (++s > 1070) fail(Errc::ExpmFailure, "scaling overflow");
  }
  B = scale(B, std::ldexp(1.0, -s));
  // Pade(7,7) coefficients: c_j = (14 - j)! 7! / (14! j! (7 - j)!) scaled by 14!/7!
  static const double c[8] = {17297280.0, 8648640.0, 1995840.0, 277200.0, 25200.0, 1512.0, 56.0, 1.0};
  const DenseMatrix I = DenseMatrix::identity(m);
  const DenseMatrix B2 = matmul(B, B), B4 = matmul(B2, B2), B6 = matmul(B4, B2);
  const DenseMatrix odd = add(add(scale(B6, c[7]), scale(B4, c[5])), add(scale(B2, c[3]), scale(I, c[1])));
  const DenseMatrix U = matmul(B, odd);
  const DenseMatrix V = add(add(scale(B6, c[6]), scale(B4, c[4])), add(scale(B2, c[2]), scale(I, c[0])));
  DenseMatrix X;
  try {
    X = lu_solve(sub(V, U), add(V, U));
  } catch (const Error&) {
    fail(Errc::ExpmFailure, "Pade denominator singular");
  }
  for (int q = 0; q < s; ++q) X = matmul(X, X);
  for (double v : X.a)
    if (!std::isfinite(v)) fail(Errc::ExpmFailure, "overflow while squaring");
  return X;
}

IVProblem heat_problem(int m, double t0, double T) {
  if (m < 1) fail(Errc::InvalidParameter, "need at least one interior point");
  IVProblem prob;
  prob.t0 = t0;
  prob.T = T;
  prob.L = DenseMatrix(m, m);
  const double inv_dx2 = double(m + 1) * double(m + 1);
  for (int i = 0; i < m; ++i) {
    prob.L.at(i, i) = -2.0 * inv_dx2;
    if (i > 0) prob.L.at(i, i - 1) = inv_dx2;
    if (i + 1 < m) prob.L.at(i, i + 1) = inv_dx2;
  }
  prob.y0.resize(m);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < m; ++i) prob.y0[i] = std::sin(pi * double(i + 1) / double(m + 1));
  return prob;
}

IVProblem decay_problem(double lambda, double t0, double T) {
  IVProblem prob;
  prob.t0 = t0;
  prob.T = T;
  prob.L = DenseMatrix(1, 1);
  prob.L.at(0, 0) = lambda;
  prob.y0 = {1.0};
  return prob;
}

}  // namespace parsol

// C entries (ctypes / other languages).  Propagators as (kind, method, steps);
// forcing as a C callback g(t, out[m], ctx) or NULL.
namespace {
parsol::Propagator prop_of(int kind, int method, int steps) {
  parsol::Propagator P;
  P.kind = parsol::PropagatorKind(kind);
  P.method = method == 0 ? parsol::OdeMethod::ImplicitEuler : parsol::OdeMethod::Trapezoidal;
  P.steps = steps;
  return P;
}
int c_error(const parsol::Error& e, char* err, size_t errlen) {
  if (err && errlen) {
    std::strncpy(err, e.what(), errlen - 1);
    err[errlen - 1] = 0;
  }
  return 1 + int(e.code());
}
}  // namespace

extern "C" int psg_parareal_solve(int m, const double* L, const double* y0, double t0, double T, int p, int N,
                                  void (*g)(double, double*, void*), void* ctx, int fkind, int fmethod, int fsteps,
                                  int ckind, int cmethod, int csteps, double tol, int max_iter, double* inits,
                                  double* history, int history_cap, int* iterations, int* converged, char* err,
                                  size_t errlen) {
  using namespace parsol;
  try {
    IVProblem prob;
    prob.L = DenseMatrix(m, m);
    std::copy(L, L + std::size_t(m) * m, prob.L.a.begin());
    prob.y0.assign(y0, y0 + m);
    prob.t0 = t0;
    prob.T = T;
    if (g)
      prob.g = [g, ctx, m](double t) {
        Vector v(m, 0.0);
        g(t, v.data(), ctx);
        return v;
      };
    const TimeGrid grid = coarse_mesh(t0, T, p, N);
    const PararealResult r = parareal_solve(prob, grid, prop_of(fkind, fmethod, fsteps), prop_of(ckind, cmethod, csteps),
                                            tol, max_iter);
    for (int i = 0; i < p; ++i) std::copy(r.inits[i].begin(), r.inits[i].end(), inits + std::size_t(i) * m);
    for (int k = 0; k < int(r.history.size()) && k < history_cap; ++k) history[k] = r.history[k];
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    return 0;
  } catch (const Error& e) {
    return c_error(e, err, errlen);
  }
}

extern "C" int psg_expm(int m, const double* L, double t, double* out, char* err, size_t errlen) {
  using namespace parsol;
  try {
    DenseMatrix A(m, m);
    std::copy(L, L + std::size_t(m) * m, A.a.begin());
    const DenseMatrix E = matrix_exponential(A, t);
    std::copy(E.a.begin(), E.a.end(), out);
    return 0;
  } catch (const Error& e) {
    return c_error(e, err, errlen);
  }
}
