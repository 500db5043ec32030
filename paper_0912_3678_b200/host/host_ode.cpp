// host_ode.cpp -- time-parallel linear IVP solver (include/parsol/odeparallel.hpp;
// reference proj/src/odeparallel.cpp, paper §3).
//
// The window-level pieces follow the reference's definitions
// (src/odeparallel.cpp:69-180): per window diag = I - h L (implicit Euler) or
// I - h/2 L (trapezoidal), sub = I or I + h/2 L, method right-hand side h g(t_n)
// or h/2 (g(t_{n-1}) + g(t_n)).  solve_ivp_parallel solves the whole discrete
// trajectory on the GPU as one BVP-layout BABD (see the header).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "parsol/errors.hpp"
#include "parsol/odeparallel.hpp"
#include "parsol/parfact.hpp"
#include "parsol/structmat.hpp"

namespace parsol {

const char* method_name(OdeMethod m) { return m == OdeMethod::ImplicitEuler ? "ie" : "trap"; }

OdeMethod method_from_name(const std::string& s) {
  if (s == "ie" || s == "euler") return OdeMethod::ImplicitEuler;
  if (s == "trap" || s == "trapezoidal") return OdeMethod::Trapezoidal;
  fail(Errc::InvalidParameter, "unknown method '" + s + "'");
}

TimeGrid coarse_mesh(double t0, double T, int p, int N) {
  if (!(T > t0)) fail(Errc::InvalidInterval, "T must exceed t0");
  if (p < 1 || N < 1) fail(Errc::InvalidInterval, "p and N must be >= 1");
  std::vector<double> tau(p + 1);
  for (int i = 0; i <= p; ++i) tau[i] = t0 + (T - t0) * double(i) / double(p);
  tau[0] = t0;
  tau[p] = T;
  return coarse_mesh(std::move(tau), N);
}

TimeGrid coarse_mesh(std::vector<double> tau, int N) {
  if (tau.size() < 2) fail(Errc::InvalidInterval, "need at least one window");
  if (N < 1) fail(Errc::InvalidInterval, "N must be >= 1");
  for (std::size_t i = 1; i < tau.size(); ++i)
    if (!(tau[i] > tau[i - 1])) fail(Errc::InvalidInterval, "mesh must be strictly increasing");
  TimeGrid g;
  g.tau = std::move(tau);
  g.N = N;
  for (std::size_t i = 1; i < g.tau.size(); ++i) g.h.push_back((g.tau[i] - g.tau[i - 1]) / N);
  return g;
}

DenseMatrix WindowSystem::v_dense() const {
  DenseMatrix V(m * N, m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) V.at(i, j) = sub.at(i, j);
  return V;
}

DenseMatrix WindowSystem::m_dense() const {
  DenseMatrix M(m * N, m * N);
  for (int s = 0; s < N; ++s)
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) {
        M.at(s * m + i, s * m + j) = diag.at(i, j);
        if (s > 0) M.at(s * m + i, (s - 1) * m + j) = -sub.at(i, j);
      }
  return M;
}

DenseMatrix WindowSolution::w_tail() const {
  DenseMatrix W(m, m);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) W.at(i, j) = w.at((N - 1) * m + i, j);
  return W;
}

WindowSystem discretize_window(const IVProblem& prob, const TimeGrid& grid, int i, OdeMethod method) {
  if (i < 1 || i > grid.windows()) fail(Errc::IndexOutOfRange, "window index");
  if ((int)prob.y0.size() != prob.dim()) fail(Errc::DimensionMismatch, "y0 length");
  WindowSystem W;
  W.index = i;
  W.method = method;
  W.m = prob.dim();
  W.N = grid.N;
  W.h = grid.h[i - 1];
  W.tstart = grid.tau[i - 1];
  const DenseMatrix I = DenseMatrix::identity(W.m);
  if (method == OdeMethod::ImplicitEuler) {
    W.diag = sub(I, scale(prob.L, W.h));
    W.sub = I;
  } else {
    W.diag = sub(I, scale(prob.L, W.h / 2));
    W.sub = add(I, scale(prob.L, W.h / 2));
  }
  try {
    W.diag_lu = DenseLu(W.diag);
  } catch (const Error&) {
    fail(Errc::StepTooLarge, "window matrix singular for h = " + std::to_string(W.h));
  }
  W.gvec.assign(std::size_t(W.m) * W.N, 0.0);
  for (int s = 1; s <= W.N; ++s) {
    const double tn = W.tstart + s * W.h;
    Vector gn = prob.forcing(tn);
    if (method == OdeMethod::ImplicitEuler) {
      for (double& v : gn) v *= W.h;
    } else {
      const Vector g0 = prob.forcing(tn - W.h);
      for (int q = 0; q < W.m; ++q) gn[q] = W.h / 2 * (g0[q] + gn[q]);
    }
    std::copy(gn.begin(), gn.end(), W.gvec.begin() + std::size_t(s - 1) * W.m);
  }
  return W;
}

Vector window_forward(const WindowSystem& W, const Vector& y_init) {
  Vector out(std::size_t(W.m) * W.N), prev = y_init, rhs(W.m);
  for (int s = 0; s < W.N; ++s) {
    for (int q = 0; q < W.m; ++q) {
      double acc = W.gvec[std::size_t(s) * W.m + q];
      for (int j = 0; j < W.m; ++j) acc += W.sub.at(q, j) * prev[j];
      rhs[q] = acc;
    }
    prev = W.diag_lu.solve(rhs);
    std::copy(prev.begin(), prev.end(), out.begin() + std::size_t(s) * W.m);
  }
  return out;
}

WindowSolution solve_window_homogeneous(const WindowSystem& W) {
  WindowSolution sol;
  sol.m = W.m;
  sol.N = W.N;
  sol.z = window_forward(W, Vector(W.m, 0.0));
  sol.w = DenseMatrix(W.m * W.N, W.m);
  WindowSystem hom = W;
  std::fill(hom.gvec.begin(), hom.gvec.end(), 0.0);
  for (int j = 0; j < W.m; ++j) {
    Vector e(W.m, 0.0);
    e[j] = 1.0;
    const Vector col = window_forward(hom, e);
    for (int q = 0; q < W.m * W.N; ++q) sol.w.at(q, j) = col[q];
  }
  return sol;
}

std::vector<Vector> reduced_recursion(const std::vector<WindowSolution>& sols, const Vector& y0) {
  std::vector<Vector> inits(sols.size());
  if (sols.empty()) return inits;
  inits[0] = y0;
  for (std::size_t i = 0; i + 1 < sols.size(); ++i) {
    Vector next = sols[i].z_tail();
    const DenseMatrix wN = sols[i].w_tail();
    for (int q = 0; q < sols[i].m; ++q)
      for (int j = 0; j < sols[i].m; ++j) next[q] += wN.at(q, j) * inits[i][j];
    inits[i + 1] = std::move(next);
  }
  return inits;
}

Trajectory parallel_update(const TimeGrid& grid, const std::vector<WindowSolution>& sols,
                           const std::vector<Vector>& inits) {
  (void)grid;
  Trajectory tr;
  tr.m = sols.at(0).m;
  tr.p = (int)sols.size();
  tr.N = sols[0].N;
  tr.flat.assign(std::size_t(tr.p * tr.N + 1) * tr.m, 0.0);
  std::copy(inits[0].begin(), inits[0].end(), tr.flat.begin());
  for (int i = 0; i < tr.p; ++i)
    for (int q = 0; q < tr.m * tr.N; ++q) {
      double acc = sols[i].z[q];
      for (int j = 0; j < tr.m; ++j) acc += sols[i].w.at(q, j) * inits[i][j];
      tr.flat[std::size_t(i) * tr.N * tr.m + tr.m + q] = acc;
    }
  return tr;
}

// ---------------------------------------------------------------------------
// the GPU trajectory solve
// ---------------------------------------------------------------------------
Trajectory solve_ivp_parallel(const IVProblem& prob, const TimeGrid& grid, OdeMethod method, SolveStats* stats) {
  const int m = prob.dim(), p = grid.windows(), N = grid.N;
  if (m < 1) fail(Errc::DimensionMismatch, "empty system");
  if ((int)prob.y0.size() != m) fail(Errc::DimensionMismatch, "y0 length");
  if (m > 8) fail(Errc::UnsupportedStructure, "the GPU trajectory solve supports systems of dimension <= 8");
  const int MB = m <= 2 ? 2 : (m <= 4 ? 4 : 8);  // padded block size: inert components
  const long steps = (long)p * N;
  const long nsteps = std::max<long>(steps, 64);  // short trajectories: identity steps appended
  const long nb = nsteps + 1;
  if ((long)MB * nb > 0x7fffffffL) fail(Errc::TooLargeForDense, "trajectory too long for one solve");
  const long BW = 2L * MB * MB;
  std::vector<double> data(std::size_t(MB) * MB + std::size_t(nsteps) * BW, 0.0);
  std::vector<double> f(std::size_t(MB) * nb, 0.0);
  for (int i = 0; i < MB; ++i) data[std::size_t(i) * MB + i] = 1.0;  // y_0 = y0
  std::copy(prob.y0.begin(), prob.y0.end(), f.begin());
  long k = 0;  // step index (block row k + 1)
  for (int w = 1; w <= p; ++w) {
    const WindowSystem W = discretize_window(prob, grid, w, method);
    // one block row per step: [ -sub | diag ], padding rows [ -I | I ]
    std::vector<double> row(BW, 0.0);
    for (int i = 0; i < MB; ++i)
      for (int j = 0; j < MB; ++j) {
        const bool real = i < m && j < m;
        row[std::size_t(i) * 2 * MB + j] = real ? -W.sub.at(i, j) : (i == j ? -1.0 : 0.0);
        row[std::size_t(i) * 2 * MB + MB + j] = real ? W.diag.at(i, j) : (i == j ? 1.0 : 0.0);
      }
    for (int s = 0; s < N; ++s, ++k) {
      std::copy(row.begin(), row.end(), data.begin() + MB * MB + k * BW);
      for (int q = 0; q < m; ++q) f[std::size_t(k + 1) * MB + q] = W.gvec[std::size_t(s) * m + q];
    }
  }
  for (; k < nsteps; ++k)  // appended identity steps: y_{k+1} = y_k
    for (int i = 0; i < MB; ++i) {
      data[MB * MB + k * BW + std::size_t(i) * 2 * MB + i] = -1.0;
      data[MB * MB + k * BW + std::size_t(i) * 2 * MB + MB + i] = 1.0;
    }
  StructuredMatrix A = make(Kind::Babd, (int)(MB * nb), MB, MB, 0, std::move(data),
                            std::vector<double>(std::size_t(MB) * MB, 0.0), MB, MB);
  const int pp = (int)std::max<long>(2, std::min<long>(4096, nb / 16));
  ParallelFactorization F = parallel_factor(A, pp, Strategy::Lu);
  const Vector x = solve(F, f, stats);
  Trajectory tr;
  tr.m = m;
  tr.p = p;
  tr.N = N;
  tr.flat.resize(std::size_t(steps + 1) * m);
  for (long b = 0; b <= steps; ++b)
    for (int q = 0; q < m; ++q) tr.flat[std::size_t(b) * m + q] = x[std::size_t(b) * MB + q];
  return tr;
}

Trajectory solve_ivp_parallel(const IVProblem& prob, const TimeGrid& grid, OdeMethod method) {
  return solve_ivp_parallel(prob, grid, method, nullptr);
}

Trajectory solve_ivp_sequential(const IVProblem& prob, const TimeGrid& grid, OdeMethod method) {
  return solve_ivp_parallel(prob, grid, method, nullptr);
}

}  // namespace parsol

// C entry (ctypes / other languages): forcing as a C callback g(t, out[m], ctx)
extern "C" int psg_ode_solve(int m, const double* L, const double* y0, double t0, double T, int p, int N, int method,
                             void (*g)(double, double*, void*), void* ctx, double* out, double* certificate,
                             char* err, size_t errlen) {
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
    SolveStats st;
    const Trajectory tr = solve_ivp_parallel(prob, grid, method == 0 ? OdeMethod::ImplicitEuler : OdeMethod::Trapezoidal,
                                             &st);
    std::copy(tr.flat.begin(), tr.flat.end(), out);
    if (certificate) *certificate = st.certificate;
    return 0;
  } catch (const Error& e) {
    if (err && errlen) {
      std::strncpy(err, e.what(), errlen - 1);
      err[errlen - 1] = 0;
    }
    return 1 + int(e.code());
  }
}
