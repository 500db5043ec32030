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

namespace {

void require_interval(bool ok, const char* what) {
  if (!ok) fail(Errc::InvalidInterval, what);
}

// write block B (scaled by sgn) into M at (r0, c0)
void put_block(DenseMatrix& M, int r0, int c0, const DenseMatrix& B, double sgn = 1.0) {
  for (int i = 0; i < B.rows; ++i)
    for (int j = 0; j < B.cols; ++j) M.at(r0 + i, c0 + j) = sgn * B.at(i, j);
}

// rows [r0, r0 + m) of a tall block matrix
DenseMatrix rows_of(const DenseMatrix& T, int r0, int m) {
  DenseMatrix B(m, T.cols);
  std::copy_n(T.a.begin() + std::ptrdiff_t(r0) * T.cols, std::size_t(m) * T.cols, B.a.begin());
  return B;
}

// one implicit step of the window: y <- diag^{-1} (sub y + rhs)
Vector implicit_step(const WindowSystem& W, const Vector& y, const double* rhs) {
  Vector t = matvec(W.sub, y);
  for (int q = 0; q < W.m; ++q) t[q] = rhs[q] + t[q];
  return W.diag_lu.solve(t);
}

}  // namespace

// The coarse mesh tau_i = t0 + (T - t0) i / p (end points exact) and the fine
// step h_i = (tau_i - tau_{i-1}) / N of every window (paper §3; the sample
// points must be the reference's: the GPU trajectory reproduces its values).
TimeGrid coarse_mesh(double t0, double T, int p, int N) {
  require_interval(T > t0, "T must exceed t0");
  require_interval(p >= 1 && N >= 1, "p and N must be >= 1");
  std::vector<double> tau(p + 1);
  int i = 0;
  std::generate(tau.begin(), tau.end(), [&] { return t0 + (T - t0) * double(i++) / double(p); });
  tau.front() = t0;
  tau.back() = T;
  return coarse_mesh(std::move(tau), N);
}

TimeGrid coarse_mesh(std::vector<double> tau, int N) {
  require_interval(tau.size() >= 2, "need at least one window");
  require_interval(N >= 1, "N must be >= 1");
  require_interval(std::adjacent_find(tau.begin(), tau.end(), [](double a, double b) { return !(b > a); }) ==
                       tau.end(),
                   "mesh must be strictly increasing");
  TimeGrid g;
  g.N = N;
  g.h.resize(tau.size() - 1);
  std::transform(tau.begin() + 1, tau.end(), tau.begin(), g.h.begin(),
                 [N](double hi, double lo) { return (hi - lo) / N; });
  g.tau = std::move(tau);
  return g;
}

// v_i: the window's coupling to its initial value, nonzero in the first step only
DenseMatrix WindowSystem::v_dense() const {
  DenseMatrix V(m * N, m);
  put_block(V, 0, 0, sub);
  return V;
}

// M_i: block lower bidiagonal, diag on the diagonal, -sub below it
DenseMatrix WindowSystem::m_dense() const {
  DenseMatrix M(m * N, m * N);
  for (int s = 0; s < N; ++s) {
    put_block(M, s * m, s * m, diag);
    if (s) put_block(M, s * m, (s - 1) * m, sub, -1.0);
  }
  return M;
}

DenseMatrix WindowSolution::w_tail() const { return rows_of(w, (N - 1) * m, m); }

// Window i of the one-step scheme y_n - y_{n-1} = h (theta L y_n + (1-theta) L y_{n-1}) + rhs_n:
// implicit Euler theta = 1 (diag = I - h L, sub = I, rhs_n = h g(t_n)), trapezoidal
// theta = 1/2 (diag = I - h/2 L, sub = I + h/2 L, rhs_n = h/2 (g(t_n - h) + g(t_n))).
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
  const bool trap = method == OdeMethod::Trapezoidal;
  const double hi = trap ? W.h / 2 : W.h;  // step weight of the implicit end
  const DenseMatrix I = DenseMatrix::identity(W.m);
  W.diag = sub(I, scale(prob.L, hi));
  W.sub = trap ? add(I, scale(prob.L, hi)) : I;
  try {
    W.diag_lu = DenseLu(W.diag);
  } catch (const Error&) {
    fail(Errc::StepTooLarge, "window matrix singular for h = " + std::to_string(W.h));
  }
  W.gvec.resize(std::size_t(W.m) * W.N);
  auto out = W.gvec.begin();
  for (int s = 1; s <= W.N; ++s, out += W.m) {
    const double tn = W.tstart + s * W.h;
    const Vector right = prob.forcing(tn);
    if (trap) {
      const Vector left = prob.forcing(tn - W.h);
      std::transform(left.begin(), left.end(), right.begin(), out, [hi](double a, double b) { return hi * (a + b); });
    } else {
      std::transform(right.begin(), right.end(), out, [hi](double b) { return b * hi; });
    }
  }
  return W;
}

// the window's steps from y_init with its right-hand sides
Vector window_forward(const WindowSystem& W, const Vector& y_init) {
  Vector out;
  out.reserve(std::size_t(W.m) * W.N);
  Vector y = y_init;
  for (int s = 0; s < W.N; ++s) {
    y = implicit_step(W, y, W.gvec.data() + std::size_t(s) * W.m);
    out.insert(out.end(), y.begin(), y.end());
  }
  return out;
}

// z = M^{-1} g and w = M^{-1} v: the homogeneous propagator is carried as one
// m x m matrix through the steps (Y_s = diag^{-1} sub Y_{s-1}, Y_0 = I)
WindowSolution solve_window_homogeneous(const WindowSystem& W) {
  WindowSolution sol;
  sol.m = W.m;
  sol.N = W.N;
  sol.z = window_forward(W, Vector(W.m, 0.0));
  sol.w = DenseMatrix(W.m * W.N, W.m);
  DenseMatrix Y = DenseMatrix::identity(W.m);
  for (int s = 0; s < W.N; ++s) {
    Y = W.diag_lu.solve(matmul(W.sub, Y));
    put_block(sol.w, s * W.m, 0, Y);
  }
  return sol;
}

// y_{0,i+1} = z_N,i + w_N,i y_{0,i}, window after window
std::vector<Vector> reduced_recursion(const std::vector<WindowSolution>& sols, const Vector& y0) {
  std::vector<Vector> inits;
  inits.reserve(sols.size());
  if (sols.empty()) return inits;
  inits.push_back(y0);
  for (std::size_t i = 0; i + 1 < sols.size(); ++i) {
    Vector next = matvec(sols[i].w_tail(), inits.back());
    const Vector zt = sols[i].z_tail();
    std::transform(zt.begin(), zt.end(), next.begin(), next.begin(), std::plus<double>());
    inits.push_back(std::move(next));
  }
  return inits;
}

// every window's trajectory from its initial value: y = z + w y_{0,i}
Trajectory parallel_update(const TimeGrid&, const std::vector<WindowSolution>& sols,
                           const std::vector<Vector>& inits) {
  Trajectory tr;
  tr.m = sols.at(0).m;
  tr.p = (int)sols.size();
  tr.N = sols[0].N;
  tr.flat = inits.at(0);
  for (int i = 0; i < tr.p; ++i) {
    Vector y = matvec(sols[i].w, inits[i]);
    std::transform(sols[i].z.begin(), sols[i].z.end(), y.begin(), y.begin(), std::plus<double>());
    tr.flat.insert(tr.flat.end(), y.begin(), y.end());
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
