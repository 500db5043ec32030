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
    CHECK_THROWS_CODE(parallel_factor(A, 3, Strategy::LuPivot), Errc::UnsupportedStructure);
    CHECK_THROWS_CODE(parallel_factor(generate_random(Kind::Banded, 30, 1, 2, 1, 5, 2.0), 3, Strategy::CyclicReduction),
                      Errc::UnsupportedKind);
  }
}

int main(int argc, char** argv) {
  const bool cpu = argc < 2 || std::strcmp(argv[1], "--gpu") != 0;
  try {
    if (cpu)
      cpu_tests();
    else
      gpu_tests();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "uncaught exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s: %d checks, %d failures\n", cpu ? "cpu" : "gpu", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
