// C++ API tests, written like the reference's doctest suites
// (proj/tests/test_structmat.cpp, test_partition.cpp, and the SPEC.md
// parfact examples that test_parfact.cpp leaves as placeholders).
//   test_host_api --cpu   host-only checks (no device work)
//   test_host_api --gpu   factor / solve / residual on the B200
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "parsol/errors.hpp"
#include "parsol/io.hpp"
#include "parsol/odeparallel.hpp"
#include "parsol/parfact.hpp"
#include "parsol/partition.hpp"
#include "parsol/rng.hpp"
#include "parsol/seqref.hpp"
#include "parsol/structmat.hpp"

using namespace parsol;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                                   \
  do {                                                                                \
    ++g_checks;                                                                       \
    if (!(cond)) {                                                                    \
      ++g_fail;                                                                       \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond);   \
    }                                                                                 \
  } while (0)
#define CHECK_THROWS_CODE(expr, errc)                                                 \
  do {                                                                                \
    ++g_checks;                                                                       \
    bool ok_ = false;                                                                 \
    try {                                                                             \
      (void)(expr);                                                                   \
    } catch (const Error& e_) {                                                       \
      ok_ = e_.code() == (errc);                                                      \
    }                                                                                 \
    if (!ok_) {                                                                       \
      ++g_fail;                                                                       \
      std::fprintf(stderr, "%s:%d: expected %s from %s\n", __FILE__, __LINE__, #errc, #expr); \
    }                                                                                 \
  } while (0)

static double rel_err(const Vector& got, const Vector& want) {  // tests/oracles.hpp:61-68
  double num = 0, den = 0;
  for (std::size_t i = 0; i < got.size(); ++i) {
    num = std::max(num, std::fabs(got[i] - want[i]));
    den = std::max(den, std::fabs(want[i]));
  }
  return den > 0 ? num / den : num;
}

static Vector random_vector(int n, std::uint64_t seed) {  // tests/oracles.hpp:42-47
  SplitMix64 rng(seed, 77);
  Vector v(n);
  for (auto& x : v) x = rng.next_unit();
  return v;
}

static StructuredMatrix toeplitz(int n) {
  std::vector<double> d;
  for (int i = 0; i < n - 1; ++i) d.push_back(-1);
  for (int i = 0; i < n; ++i) d.push_back(2);
  for (int i = 0; i < n - 1; ++i) d.push_back(-1);
  return make(Kind::Banded, n, 1, 1, 1, std::move(d));
}

// ---------------------------------------------------------------- host only
static void cpu_tests() {
  // layouts and structural access (test_structmat.cpp:10-34)
  StructuredMatrix T = toeplitz(5);
  CHECK(T.at(0, 0) == 2 && T.at(0, 1) == -1 && T.at(1, 0) == -1 && T.at(0, 2) == 0);
  DenseMatrix D = to_dense(T);
  CHECK(D.at(4, 4) == 2 && D.at(4, 3) == -1);
  StructuredMatrix B = generate_random(Kind::Babd, 24, 2, 1, 1, 3, 2.0);
  CHECK(B.in_structure(0, 23) && B.in_structure(1, 22) && !B.in_structure(2, 23));
  CHECK(B.at(0, 22) == B.corner[0]);
  // make() validation (test_structmat.cpp:97-108) + the Babd BVP relaxation
  CHECK_THROWS_CODE(make(Kind::Banded, 10, 1, 1, 1, std::vector<double>(27)), Errc::DimensionMismatch);
  CHECK_THROWS_CODE(make(Kind::Banded, 3, 1, 2, 1, std::vector<double>(7)), Errc::InvalidBandwidth);
  CHECK_THROWS_CODE(make(Kind::BlockTridiagonal, 12, 4, 2, 1, std::vector<double>(112)), Errc::InvalidBandwidth);
  CHECK_THROWS_CODE(make(Kind::Banded, 10, 1, 1, 1, std::vector<double>(28), {1.0}, 1, 1), Errc::CornerForbidden);
  const std::size_t nb = body_entry_count(Kind::Babd, 32, 8, 8, 0);
  CHECK(nb == 64 + 3 * 128);
  StructuredMatrix bvp = make(Kind::Babd, 32, 8, 8, 0, std::vector<double>(nb, 1.0), std::vector<double>(64, 0.5), 8, 8);
  CHECK(bvp.at(8, 0) == 1.0 && bvp.at(0, 24) == 0.5 && bvp.at(8, 16) == 0.0);
  // generator determinism and dominance (test_structmat.cpp:83-95)
  StructuredMatrix G1 = generate_random(Kind::Banded, 10, 1, 1, 1, 1, 2.0);
  StructuredMatrix G2 = generate_random(Kind::Banded, 10, 1, 1, 1, 1, 2.0);
  CHECK(G1 == G2);
  for (int i = 0; i < 10; ++i) {
    double off = 0;
    for (int j = 0; j < 10; ++j)
      if (j != i) off += std::fabs(G1.at(i, j));
    CHECK(std::fabs(G1.at(i, i)) >= 2.0 * std::max(off, 1.0) - 1e-12);
  }
  CHECK_THROWS_CODE(generate_random(Kind::Banded, 10, 1, 1, 1, 1, -1.0), Errc::InvalidParameter);
  // plan shapes (test_partition.cpp:21-40)
  PartitionPlan P9 = plan_partition(toeplitz(9), 2);
  CHECK(P9.sep_size == 1 && P9.body_size(0) == 4 && P9.body_size(1) == 4);
  CHECK(P9.sep_count() == 1 && P9.separator_starts[0] == 4);
  CHECK(plan_partition(generate_random(Kind::Banded, 20, 1, 2, 1, 3, 2.0), 3).sep_size == 2);
  PartitionPlan PB = plan_partition(B, 3);
  CHECK(PB.has_corner && PB.sep_count() == 4 && PB.sep_size == 2);
  CHECK_THROWS_CODE(plan_partition(toeplitz(9), 1), Errc::TooManyPartitions);
  // plans tile [0, n) (test_partition.cpp:42-66)
  struct Case { Kind k; int n, m, s, r, p; };
  for (Case c : {Case{Kind::Banded, 37, 1, 2, 3, 4}, Case{Kind::BlockTridiagonal, 36, 3, 1, 1, 3},
                 Case{Kind::Abd, 40, 4, 2, 2, 3}, Case{Kind::Babd, 44, 2, 1, 1, 4}}) {
    StructuredMatrix A = generate_random(c.k, c.n, c.m, c.s, c.r, 11, 2.0);
    PartitionPlan plan = plan_partition(A, c.p);
    std::vector<std::pair<int, int>> spans(plan.body_ranges);
    for (int s0 : plan.separator_starts) spans.emplace_back(s0, s0 + plan.sep_size);
    std::sort(spans.begin(), spans.end());
    int cursor = 0;
    for (auto [b, e] : spans) {
      CHECK(b == cursor);
      cursor = e;
    }
    CHECK(cursor == c.n);
    // extract_block agrees with the dense image (test_partition.cpp:68-95)
    DenseMatrix DA = to_dense(A);
    for (int i = 1; i <= c.p; ++i) {
      PartitionBlock blk = extract_block(A, plan, i);
      auto [b, e] = plan.body_ranges[i - 1];
      for (int x = 0; x < blk.L; ++x)
        for (int y = 0; y < blk.L; ++y) CHECK(blk.body_at(x, y) == DA.at(b + x, b + y));
    }
  }
  CHECK(std::string(strategy_name(Strategy::Lud)) == "lud" && strategy_from_name("cr") == Strategy::CyclicReduction);
  CHECK(!strategy_supports(Strategy::CyclicReduction, Kind::Banded, 2, 1));
  CHECK(strategy_supports(Strategy::Arce, Kind::Babd, 1, 1));
  // STRUCTMAT / VEC round trips, bit-exact (reference io.hpp; tests/test_structmat.cpp round trip)
  for (auto c : std::vector<std::array<int, 5>>{{0, 57, 1, 2, 3}, {1, 48, 4, 1, 1}, {2, 60, 4, 2, 2}, {3, 64, 4, 2, 2},
                                                 {0, 33, 1, 1, 1}}) {
    StructuredMatrix A = generate_random(Kind(c[0]), c[1], c[2], c[3], c[4], 7 + c[1], 2.0);
    const std::string txt = write_matrix(A, {"round trip"});
    CHECK(txt.rfind("STRUCTMAT 1 ", 0) == 0);
    CHECK(parse_matrix(txt) == A);
    CHECK(write_matrix(parse_matrix(txt), {"round trip"}) == txt);
  }
  {
    Vector v = random_vector(41, 3);
    v.push_back(-0.0);
    v.push_back(1e-310);  // subnormal
    const Vector w = parse_vector(write_vector(v, {"c"}));
    CHECK(w.size() == v.size());
    bool same = true;
    for (size_t i = 0; i < v.size(); ++i) same &= std::memcmp(&v[i], &w[i], sizeof(double)) == 0;
    CHECK(same);
    CHECK(format_hex(1.5) == "0x1.8p+0");
  }
  auto errc_of = [](const std::function<void()>& fn) {
    try {
      fn();
    } catch (const Error& e) {
      return int(e.code());
    }
    return -1;
  };
  CHECK(errc_of([] { parse_matrix(""); }) == int(Errc::ParseError));
  CHECK(errc_of([] { parse_matrix("STRUCTMAT 2 banded 3 1 1 1\n"); }) == int(Errc::UnsupportedVersion));
  CHECK(errc_of([] { parse_matrix("STRUCTMAT 1 banded 3 1 1 1\n0x1p+0\n"); }) == int(Errc::ParseError));
  CHECK(errc_of([] { parse_matrix("STRUCTMAT 1 babd 4 2 1 1\n"); }) == int(Errc::ParseError));  // corner shape
  CHECK(errc_of([] { parse_matrix("STRUCTMAT 1 wat 3 1 1 1\n"); }) == int(Errc::ParseError));
  CHECK(errc_of([] { parse_vector("VEC 1 2\n0x1p+0\nabc\n"); }) == int(Errc::ParseError));
  CHECK(errc_of([] { parse_vector("VEC 1 1\n# c\n0x1p+0\n"); }) == -1);
  CHECK(errc_of([] {
          parse_matrix("STRUCTMAT 1 banded 3 1 1 1\n1\n2\n3\n4\n5\n6\n7\n8\n");
        }) == int(Errc::ParseError));  // trailing data
  CHECK(errc_of([] { read_file("/nonexistent/x.mat"); }) == int(Errc::IoError));
}

// ODE windows on the host (reference SPEC.md odeparallel examples)
static IVProblem scalar_ivp(double lambda, double y0, double T) {
  IVProblem P;
  P.L = DenseMatrix(1, 1);
  P.L.at(0, 0) = lambda;
  P.y0 = {y0};
  P.T = T;
  return P;
}

static IVProblem random_ivp(int m, std::uint64_t seed, double T) {
  IVProblem P;
  P.L = DenseMatrix(m, m);
  Vector r = random_vector(m * m + m, seed);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) P.L.at(i, j) = r[i * m + j] - (i == j ? 2.0 : 0.0);
  P.y0 = Vector(r.end() - m, r.end());
  P.g = [m](double t) {
    Vector g(m);
    for (int q = 0; q < m; ++q) g[q] = std::sin((q + 1) * t) + 0.5;
    return g;
  };
  P.T = T;
  return P;
}

static Trajectory host_pipeline(const IVProblem& P, const TimeGrid& G, OdeMethod meth) {
  std::vector<WindowSolution> sols;
  for (int i = 1; i <= G.windows(); ++i) sols.push_back(solve_window_homogeneous(discretize_window(P, G, i, meth)));
  return parallel_update(G, sols, reduced_recursion(sols, P.y0));
}

static Trajectory host_sequential(const IVProblem& P, const TimeGrid& G, OdeMethod meth) {
  Trajectory tr{P.dim(), G.windows(), G.N, P.y0};
  Vector y = P.y0;
  for (int i = 1; i <= G.windows(); ++i) {
    Vector seg = window_forward(discretize_window(P, G, i, meth), y);
    tr.flat.insert(tr.flat.end(), seg.begin(), seg.end());
    y = Vector(seg.end() - P.dim(), seg.end());
  }
  return tr;
}

static void cpu_ode_tests() {
  auto errc_of = [](const std::function<void()>& fn) {
    try {
      fn();
    } catch (const Error& e) {
      return int(e.code());
    }
    return -1;
  };
  TimeGrid G = coarse_mesh(0, 1, 4, 10);
  CHECK(G.windows() == 4 && G.tau[2] == 0.5 && std::fabs(G.h[1] - 0.025) < 1e-17);
  TimeGrid G2 = coarse_mesh({0, 0.1, 1}, 5);
  CHECK(std::fabs(G2.h[0] - 0.02) < 1e-17 && std::fabs(G2.h[1] - 0.18) < 1e-16);
  CHECK(coarse_mesh(0, 1, 1, 1).windows() == 1);
  CHECK(errc_of([] { coarse_mesh(1, 1, 2, 2); }) == int(Errc::InvalidInterval));
  CHECK(errc_of([] { coarse_mesh(0, 1, 0, 2); }) == int(Errc::InvalidInterval));
  CHECK(errc_of([] { coarse_mesh({0, 0.5, 0.5}, 2); }) == int(Errc::InvalidInterval));
  CHECK(std::string(method_name(OdeMethod::Trapezoidal)) == "trap" &&  // src/odeparallel.cpp:10-17
        method_from_name("euler") == OdeMethod::ImplicitEuler && method_from_name("trapezoidal") == OdeMethod::Trapezoidal);
  CHECK(errc_of([] { method_from_name("rk4"); }) == int(Errc::InvalidParameter));
  // scalar lambda = -1, h = 0.1, implicit Euler: diagonal 1.1; w_N = 1.1^-10
  {
    IVProblem P = scalar_ivp(-1.0, 1.0, 1.0);
    WindowSystem W = discretize_window(P, coarse_mesh(0, 1, 1, 10), 1, OdeMethod::ImplicitEuler);
    CHECK(std::fabs(W.diag.at(0, 0) - 1.1) < 1e-15);
    WindowSolution S = solve_window_homogeneous(W);
    CHECK(std::fabs(S.w_tail().at(0, 0) - std::pow(1.1, -10)) < 1e-14);
    CHECK(inf_norm(S.z) == 0.0);  // g = 0 -> z = 0
    // trapezoidal one step h = 0.2: amplification 0.9/1.1
    WindowSystem Wt = discretize_window(scalar_ivp(-1.0, 1.0, 0.2), coarse_mesh(0, 0.2, 1, 1), 1,
                                        OdeMethod::Trapezoidal);
    CHECK(std::fabs(window_forward(Wt, {1.0})[0] - 0.9 / 1.1) < 1e-15);
  }
  // L = 0, g = 1, y0 = 0, implicit Euler: y_n = n h
  {
    IVProblem P = scalar_ivp(0.0, 0.0, 1.0);
    P.g = [](double) { return Vector{1.0}; };
    Trajectory tr = host_sequential(P, coarse_mesh(0, 1, 2, 5), OdeMethod::ImplicitEuler);
    bool ok = true;
    for (int n = 0; n <= 10; ++n) ok &= std::fabs(tr.flat[n] - n * 0.1) < 1e-15;
    CHECK(ok);
  }
  // reduced recursion on a scalar geometric chain: w_N = 0.5, z_N = 1, y0 = 0
  {
    std::vector<WindowSolution> sols(4);
    for (auto& s : sols) {
      s.m = 1, s.N = 1, s.z = {1.0}, s.w = DenseMatrix(1, 1);
      s.w.at(0, 0) = 0.5;
    }
    auto in = reduced_recursion(sols, {0.0});
    CHECK(in[0][0] == 0 && in[1][0] == 1 && in[2][0] == 1.5 && in[3][0] == 1.75);
  }
  // window matrices: M w = v and M z = g (dense residual oracle)
  {
    IVProblem P = random_ivp(3, 77, 1.0);
    for (OdeMethod meth : {OdeMethod::ImplicitEuler, OdeMethod::Trapezoidal}) {
      WindowSystem W = discretize_window(P, coarse_mesh(0, 1, 2, 6), 2, meth);
      WindowSolution S = solve_window_homogeneous(W);
      const DenseMatrix M = W.m_dense();
      CHECK(inf_norm(sub(matmul(M, S.w), W.v_dense())) <= 1e-12);
      Vector r = matvec(M, S.z);
      for (size_t q = 0; q < r.size(); ++q) r[q] -= W.gvec[q];
      CHECK(inf_norm(r) <= 1e-12);
    }
  }
  // parallel / sequential equivalence of the reference's window pipeline
  for (OdeMethod meth : {OdeMethod::ImplicitEuler, OdeMethod::Trapezoidal})
    for (int p : {2, 4, 8})
      for (int m : {1, 3, 6}) {
        IVProblem P = random_ivp(m, 100 + p * 7 + m, 2.0);
        TimeGrid Gp = coarse_mesh(0, 2, p, 25);
        CHECK(rel_err(host_pipeline(P, Gp, meth).flat, host_sequential(P, Gp, meth).flat) <= 1e-12);
      }
}

// ---------------------------------------------------------------- on the GPU
static void gpu_tests() {
  // identity -> x = f, T_p = I
  {
    std::vector<double> d(7, 0.0);
    d.insert(d.end(), 8, 1.0);
    d.insert(d.end(), 7, 0.0);
    StructuredMatrix I = make(Kind::Banded, 8, 1, 1, 1, d);
    ParallelFactorization F = parallel_factor(I, 4, Strategy::Lu);
    CHECK(F.reduced.q == 3 && F.reduced.dim == 3);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) CHECK(std::fabs(F.reduced.T.at(i, j) - (i == j ? 1.0 : 0.0)) < 1e-15);
    Vector f = {1, 2, 3, 4, 5, 6, 7, 8};
    CHECK(rel_err(solve(F, f), f) == 0.0);
  }
  // Toeplitz(-1,2,-1): n=3, f=[1,1,1] -> [1.5, 2, 1.5]; n=9, p=2 -> q=1
  {
    Vector x = solve(parallel_factor(toeplitz(3), 2, Strategy::Lu), {1, 1, 1});
    CHECK(std::fabs(x[0] - 1.5) < 1e-15 && std::fabs(x[1] - 2.0) < 1e-15 && std::fabs(x[2] - 1.5) < 1e-15);
    CHECK(parallel_factor(toeplitz(9), 2, Strategy::Lu).reduced.q == 1);
  }
  // solver equivalence vs a dense LU (SPEC.md acceptance 1): every kind, p in {2,3,4}
  struct Case { Kind k; int n, m, s, r; };
  int seed = 500;
  for (Case c : {Case{Kind::Banded, 120, 1, 1, 1}, Case{Kind::Banded, 131, 1, 3, 2},
                 Case{Kind::BlockTridiagonal, 120, 4, 1, 1}, Case{Kind::BlockTridiagonal, 96, 3, 1, 1},
                 Case{Kind::Abd, 120, 4, 2, 2}, Case{Kind::Babd, 120, 4, 2, 2}, Case{Kind::Babd, 64, 2, 1, 1}}) {
    for (int p : {2, 3, 4}) {
      StructuredMatrix A = generate_random(c.k, c.n, c.m, c.s, c.r, ++seed, 2.0);
      Vector f = random_vector(c.n, seed);
      SolveStats st;
      ParallelFactorization F = parallel_factor(A, p, Strategy::Lu);
      Vector x = solve(F, f, &st);
      Vector want = lu_solve(to_dense(A), f);
      CHECK(rel_err(x, want) <= 1e-10);
      CHECK(residual(A, x, f) <= 1e-10);
      // reduced-size law (SPEC.md acceptance 3)
      CHECK(F.reduced.q == (c.k == Kind::Babd ? p + 1 : p - 1));
      // solve_reduced vs a dense solve of T
      if (!F.reduced.T.empty()) {
        Vector rhs = random_vector(F.reduced.dim, 3);
        CHECK(rel_err(solve_reduced(F, rhs), lu_solve(F.reduced.T, rhs)) <= 1e-10);
      }
      // determinism (SPEC.md acceptance 8): bit-identical on repeat
      CHECK(solve(F, f) == x);
    }
  }
  // residual examples
  {
    StructuredMatrix A = generate_random(Kind::Banded, 50, 1, 2, 2, 9, 3.0);
    Vector f = random_vector(50, 4);
    CHECK(std::fabs(residual(A, Vector(50, 0.0), f) - 1.0) < 1e-15);
    Vector x = solve(parallel_factor(A, 3, Strategy::Lu), f);
    CHECK(residual(A, x, f) <= 1e-10);
    Vector xp = x;
    for (auto& v : xp) v *= 1.0 + 1e-3;
    const double rp = residual(A, xp, f);
    CHECK(rp >= 1e-5 && rp <= 1e-1);
    // matvec vs the dense product
    Vector y = matvec(A, x), yd = matvec(to_dense(A), x);
    CHECK(rel_err(y, yd) <= 1e-15);
    // solve_sequential runs on the GPU too
    CHECK(rel_err(solve_sequential(A, f), x) <= 1e-12);
  }
  // circulant-like (reference permute_corner + LuPivot): rows rotated, wrap in the corner
  {
    const int n = 64;
    std::vector<double> d(3 * n);
    Vector r = random_vector(3 * n, 17);
    for (int i = 0; i < 3 * n; ++i) d[i] = r[i];
    StructuredMatrix C = make(Kind::CirculantLike, n, 1, 1, 1, d);
    auto [B, perm] = permute_corner(C);
    CHECK(B.s == 2 && B.r == 0 && B.corner_canonical() && perm.source[0] == n - 1);
    CHECK(B.at(5, 3) == C.at(4, 3) && B.at(0, n - 1) == C.at(n - 1, n - 1));
    Vector f = random_vector(n, 3);
    Vector want = lu_solve(to_dense(C), f);
    for (Strategy st : {Strategy::LuPivot, Strategy::Qr}) {
      ParallelFactorization F = parallel_factor(C, 4, st);
      CHECK(F.permuted && F.plan.has_corner && F.plan.sep_size == 2);
      CHECK(rel_err(solve(F, f), want) <= 1e-10);
      // the reduced system: q blocks in position order, T dense, solve_reduced consistent
      CHECK(int(F.reduced.positions.size()) == F.reduced.q && F.reduced.T.rows == F.reduced.dim);
      Vector rhs = random_vector(F.reduced.dim, 5);
      CHECK(rel_err(solve_reduced(F, rhs), lu_solve(F.reduced.T, rhs)) <= 1e-10);
    }
  }
  // errors: zero pivot tagged with the partition (test_localfact.cpp:369-385, parfact.cpp:61-68)
  {
    const int n = 3000;
    std::vector<double> d(n - 1, 1.0);
    d.insert(d.end(), n, 4.0);
    d.insert(d.end(), n - 1, 1.0);
    d[n - 1 + 1001] = 0.0;
    d[n - 1 + 1002] = 0.0;
    StructuredMatrix A = make(Kind::Banded, n, 1, 1, 1, d);
    bool ok = false;
    try {
      solve(parallel_factor(A, 3, Strategy::Lu), Vector(n, 1.0));
    } catch (const Error& e) {
      ok = e.code() == Errc::ZeroPivot && e.detail().find("partition 2") != std::string::npos;
    }
    CHECK(ok);
    // ZeroPivot "signals: use LUPivot or QR" (SPEC localfact): both solve the same matrix
    for (Strategy st : {Strategy::LuPivot, Strategy::Qr}) {
      ParallelFactorization Fp = parallel_factor(A, 3, st);
      CHECK(residual(A, solve(Fp, Vector(n, 1.0)), Vector(n, 1.0)) <= 1e-13);
      CHECK(Fp.reduced.q >= 2 && Fp.kept_maps.size() == 3);
    }
    CHECK_THROWS_CODE(parallel_factor(generate_random(Kind::Banded, 30, 1, 2, 1, 5, 2.0), 3, Strategy::CyclicReduction),
                      Errc::UnsupportedKind);
  }
}

static void gpu_ode_tests() {
  // scalar lambda = -1, g = 0, y0 = 1, implicit Euler, p = 4, N = 25: y(1) = 1.01^-100
  {
    IVProblem P = scalar_ivp(-1.0, 1.0, 1.0);
    Trajectory tr = solve_ivp_parallel(P, coarse_mesh(0, 1, 4, 25), OdeMethod::ImplicitEuler);
    CHECK(tr.flat.size() == 101 && std::fabs(tr.endpoint()[0] - std::pow(1.01, -100)) <= 1e-14);
  }
  // L = 0, g = 0, y0 = c: constant trajectory
  {
    IVProblem P;
    P.L = DenseMatrix(2, 2);
    P.y0 = {3.0, -2.0};
    Trajectory tr = solve_ivp_parallel(P, coarse_mesh(0, 1, 3, 7), OdeMethod::Trapezoidal);
    bool ok = true;
    for (int k = 0; k <= 21; ++k) ok &= tr.entry(k) == P.y0;
    CHECK(ok);
  }
  // GPU trajectory vs the host window pipeline and the sequential iteration
  for (OdeMethod meth : {OdeMethod::ImplicitEuler, OdeMethod::Trapezoidal})
    for (int p : {1, 2, 4, 8})
      for (int m : {1, 3, 4, 6, 8}) {
        IVProblem P = random_ivp(m, 300 + p * 11 + m, 2.0);
        TimeGrid Gp = coarse_mesh(0, 2, p, 100);
        const Trajectory got = solve_ivp_parallel(P, Gp, meth);
        CHECK(rel_err(got.flat, host_sequential(P, Gp, meth).flat) <= 1e-12);
        CHECK(rel_err(got.flat, host_pipeline(P, Gp, meth).flat) <= 1e-12);
        if (p == 1) CHECK(solve_ivp_sequential(P, Gp, meth).flat == got.flat);
      }
  // non-uniform mesh
  {
    IVProblem P = random_ivp(4, 9, 1.0);
    TimeGrid Gp = coarse_mesh({0, 0.05, 0.3, 0.31, 1.0}, 40);
    CHECK(rel_err(solve_ivp_parallel(P, Gp, OdeMethod::Trapezoidal).flat,
                  host_sequential(P, Gp, OdeMethod::Trapezoidal).flat) <= 1e-12);
  }
}

int main(int argc, char** argv) {
  const bool cpu = argc < 2 || std::strcmp(argv[1], "--gpu") != 0;
  try {
    if (cpu) {
      cpu_tests();
      cpu_ode_tests();
    } else {
      gpu_tests();
      gpu_ode_tests();
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "uncaught exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s: %d checks, %d failures\n", cpu ? "cpu" : "gpu", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
