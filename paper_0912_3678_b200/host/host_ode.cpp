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
#include <functional>
#include <string>

#include "parsol/errors.hpp"
#include "parsol/odeparallel.hpp"
#include "parsol/parfact.hpp"
#include "parsol/structmat.hpp"
#include "psg.h"

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
namespace {

// g(t) written straight into out[m] (no per-sample allocation).
using Sampler = std::function<void(double, double*)>;

// Window i's blocks and method right-hand sides, sampled at exactly the
// reference's points (src/odeparallel.cpp:96-109: t_n = tstart + n h, and
// t_n - h for the trapezoidal left end).  A trapezoidal left sample is
// taken from the previous step when t_n - h equals the previous t_n
// bitwise, so the values match the reference's two-calls-per-step loop.
void window_blocks(const DenseMatrix& L, const TimeGrid& grid, int i, OdeMethod method, const Sampler& g, double* win,
                   double* rhs) {
  const int m = L.rows, N = grid.N;
  const double h = grid.h[i - 1], tstart = grid.tau[i - 1];
  const std::size_t mm = std::size_t(m) * m;
  DenseMatrix D(m, m);
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < m; ++c) {
      const double id = r == c ? 1.0 : 0.0;
      const double l = L.at(r, c);
      if (method == OdeMethod::ImplicitEuler) {
        D.at(r, c) = id - l * h;
        win[mm + r * m + c] = id;
      } else {
        D.at(r, c) = id - l * (h / 2);
        win[mm + r * m + c] = id + l * (h / 2);
      }
    }
  try {
    DenseLu lu(D);
  } catch (const Error&) {
    fail(Errc::StepTooLarge, "window matrix singular for h = " + std::to_string(h));
  }
  std::copy(D.a.begin(), D.a.end(), win);
  std::vector<double> g0(m), gn(m);
  double prev_t = 0;
  for (int n = 1; n <= N; ++n) {
    const double tn = tstart + n * h;
    double* out = rhs + std::size_t(n - 1) * m;
    if (method == OdeMethod::ImplicitEuler) {
      g(tn, out);
      for (int q = 0; q < m; ++q) out[q] *= h;
      continue;
    }
    const double tl = tn - h;
    if (n > 1 && tl == prev_t)
      g0.swap(gn);
    else
      g(tl, g0.data());
    g(tn, gn.data());
    prev_t = tn;
    for (int q = 0; q < m; ++q) out[q] = h / 2 * (g0[q] + gn[q]);
  }
}

// The trajectory ((p N + 1) m, into out) of y' = L y + g on grid.
void trajectory_on_gpu(const DenseMatrix& L, const double* y0, const TimeGrid& grid, OdeMethod method,
                       const Sampler& g, double* out, psg_stats* st) {
  const int m = L.rows, p = grid.windows(), N = grid.N;
  if (m < 1) fail(Errc::DimensionMismatch, "empty system");
  if (L.cols != m) fail(Errc::DimensionMismatch, "L must be square");
  if (m > 8) fail(Errc::UnsupportedStructure, "the GPU trajectory solve supports systems of dimension <= 8");
  const std::size_t mm = std::size_t(m) * m, steps = std::size_t(p) * N;
  std::vector<double> win(std::size_t(p) * 2 * mm), rhs((steps + 1) * m);
  std::copy(y0, y0 + m, rhs.begin());
  // windows concurrently, as in the reference (src/odeparallel.cpp:199-209:
  // g is called from worker threads)
  std::vector<std::string> errs(p);
  std::vector<int> codes(p, -1);
#pragma omp parallel for schedule(static)
  for (int w = 1; w <= p; ++w) {
    try {
      window_blocks(L, grid, w, method, g, win.data() + std::size_t(w - 1) * 2 * mm,
                    rhs.data() + m + std::size_t(w - 1) * N * m);
    } catch (const Error& e) {
      codes[w - 1] = int(e.code());
      errs[w - 1] = e.detail();
    }
  }
  for (int w = 0; w < p; ++w)
    if (codes[w] >= 0) fail(Errc(codes[w]), errs[w]);
  char err[256] = {0};
  const int rc = psg_ode_trajectory(m, p, N, win.data(), rhs.data(), out, nullptr, st, err, sizeof err);
  if (rc) fail(Errc(rc - 1), err);
}

}  // namespace

Trajectory solve_ivp_parallel(const IVProblem& prob, const TimeGrid& grid, OdeMethod method, SolveStats* stats) {
  const int m = prob.dim();
  if ((int)prob.y0.size() != m) fail(Errc::DimensionMismatch, "y0 length");
  Sampler g = [&prob, m](double t, double* out) {
    if (!prob.g) {
      std::fill(out, out + m, 0.0);
      return;
    }
    const Vector v = prob.g(t);
    if ((int)v.size() != m) fail(Errc::DimensionMismatch, "g(t) length");
    std::copy(v.begin(), v.end(), out);
  };
  Trajectory tr;
  tr.m = m;
  tr.p = grid.windows();
  tr.N = grid.N;
  tr.flat.resize((std::size_t(tr.p) * tr.N + 1) * m);
  psg_stats st{};
  trajectory_on_gpu(prob.L, prob.y0.data(), grid, method, g, tr.flat.data(), &st);
  if (stats) {
    stats->factor_seconds = st.factor_seconds;
    stats->phase1_seconds = st.phase1_seconds;
    stats->phase2_seconds = st.phase2_seconds;
    stats->phase3_seconds = st.phase3_seconds;
    stats->reduced_ops = st.reduced_ops;
    stats->certificate = st.certificate;
    stats->fallbacks = st.fallbacks;
  }
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
    if (m < 1) fail(Errc::DimensionMismatch, "empty system");
    DenseMatrix Lm(m, m);
    std::copy(L, L + std::size_t(m) * m, Lm.a.begin());
    const TimeGrid grid = coarse_mesh(t0, T, p, N);
    Sampler sampler = [g, ctx, m](double t, double* o) {
      if (g)
        g(t, o, ctx);
      else
        std::fill(o, o + m, 0.0);
    };
    psg_stats st{};
    trajectory_on_gpu(Lm, y0, grid, method == 0 ? OdeMethod::ImplicitEuler : OdeMethod::Trapezoidal, sampler, out,
                      &st);
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
