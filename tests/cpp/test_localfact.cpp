// LocalFactorization suite of the reference (proj/tests/test_localfact.cpp,
// doctest) run against this repo's headers and libraries: every factor_* call
// and member operation executes on the GPU (psg_local_*).  ARCE cases are
// left out: the reference's ARCE does not reconstruct its blocks (SURVEY.md
// §0.5) and this library returns UnsupportedStructure for it, which is
// checked instead.  Also: solve_reduced on a ReducedSystem (SPEC.md
// solve_reduced examples), parallel_factor's factor_seconds / reduced.device,
// and materialize_locals against the reduced matrix T.
//   test_localfact --gpu
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "parsol/localfact.hpp"
#include "parsol/parfact.hpp"
#include "parsol/partition.hpp"
#include "parsol/rng.hpp"
#include "parsol/structmat.hpp"

using namespace parsol;

static int g_checks = 0, g_fail = 0;
#define CHECK(cond)                                                                 \
  do {                                                                              \
    ++g_checks;                                                                     \
    if (!(cond)) {                                                                  \
      ++g_fail;                                                                     \
      std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                               \
  } while (0)
#define REQUIRE(cond)                                                                 \
  do {                                                                                \
    ++g_checks;                                                                       \
    if (!(cond)) {                                                                    \
      ++g_fail;                                                                       \
      std::fprintf(stderr, "%s:%d: REQUIRE failed: %s\n", __FILE__, __LINE__, #cond); \
      return;                                                                         \
    }                                                                                 \
  } while (0)
#define CHECK_THROWS_CODE(expr, errc)                                                           \
  do {                                                                                          \
    ++g_checks;                                                                                 \
    bool ok_ = false;                                                                           \
    try {                                                                                       \
      (void)(expr);                                                                             \
    } catch (const Error& e_) {                                                                 \
      ok_ = e_.code() == (errc);                                                                \
    }                                                                                           \
    if (!ok_) {                                                                                 \
      ++g_fail;                                                                                 \
      std::fprintf(stderr, "%s:%d: expected %s from %s\n", __FILE__, __LINE__, #errc, #expr);   \
    }                                                                                           \
  } while (0)

// normwise relative difference (tests/oracles.hpp:61-76 definition)
static double rel_err(const std::vector<double>& got, const std::vector<double>& want) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < got.size(); ++i) {
    num = std::max(num, std::fabs(got[i] - want[i]));
    den = std::max(den, std::fabs(want[i]));
  }
  return den > 0 ? num / den : num;
}
static double rel_err(const DenseMatrix& got, const DenseMatrix& want) { return rel_err(got.a, want.a); }

static Vector random_vector(int n, std::uint64_t seed) {
  SplitMix64 rng(seed, 77);
  Vector v(n);
  for (auto& x : v) x = rng.next_unit();
  return v;
}

static PartitionBlock middle_block(const StructuredMatrix& A) {  // partition 2 of a 3-way split
  return extract_block(A, plan_partition(A, 3), 2);
}

// a banded-kind block with a full L x L envelope holding `body`
static PartitionBlock dense_block(const DenseMatrix& body, const DenseMatrix& b0, const DenseMatrix& c0,
                                  const DenseMatrix& b1, const DenseMatrix& c1, const DenseMatrix& a_right) {
  PartitionBlock P;
  P.index = 2;
  P.kind = Kind::Banded;
  P.m = 1;
  P.s = P.r = 1;
  P.L = body.rows;
  P.k0 = b0.cols;
  P.k1 = b1.cols;
  P.env_s = P.env_r = P.L - 1;
  P.env.assign(std::size_t(P.L) * (2 * P.L - 1), 0.0);
  for (int i = 0; i < P.L; ++i)
    for (int j = 0; j < P.L; ++j) P.body_ref(i, j) = body.at(i, j);
  P.b0 = b0;
  P.c0 = c0;
  P.b1 = b1;
  P.c1 = c1;
  P.a_right = a_right;
  return P;
}

static double reconstruction_error(const PartitionBlock& P, const LocalFactorization& lf) {
  return rel_err(matmul(matmul(lf.dense_F_loc(), lf.dense_T_loc()), lf.dense_G_loc()), P.local_dense());
}

static DenseMatrix tridiag(int L, double lo, double d, double up) {
  DenseMatrix B(L, L);
  for (int i = 0; i < L; ++i) {
    B.at(i, i) = d;
    if (i) B.at(i, i - 1) = lo;
    if (i + 1 < L) B.at(i, i + 1) = up;
  }
  return B;
}

static void identity_body() {
  const DenseMatrix I4 = DenseMatrix::identity(4), z(4, 1);
  const PartitionBlock P = dense_block(I4, z, z, z, z, DenseMatrix::identity(1));
  const LocalFactorization lf = factor_lu(P);
  CHECK(rel_err(lf.dense_N(), I4) == 0.0);
  CHECK(rel_err(lf.dense_S(), I4) == 0.0);
  for (double v : lf.z.a) CHECK(v == 0.0);
  for (double v : lf.w.a) CHECK(v == 0.0);
  CHECK(lf.alpha1.at(0, 0) == 0.0);
  CHECK(lf.alpha2.at(0, 0) == 1.0);
  CHECK(reconstruction_error(P, lf) == 0.0);
}

static void toeplitz_block() {
  DenseMatrix b0(4, 1), c0(4, 1), b1(4, 1), c1(4, 1), ar(1, 1);
  b0.at(0, 0) = c0.at(0, 0) = 1;
  b1.at(3, 0) = c1.at(3, 0) = 1;
  ar.at(0, 0) = 2;
  const PartitionBlock P = dense_block(tridiag(4, -1, 2, -1), b0, c0, b1, c1, ar);
  const LocalFactorization lf = factor_lu(P);
  CHECK(reconstruction_error(P, lf) < 1e-12);
  bool fill = false;
  for (int x = 1; x < 4; ++x) fill |= lf.z.at(x, 0) != 0.0;
  CHECK(fill);
}

static void lu_sparsity() {
  const StructuredMatrix A = generate_random(Kind::Banded, 34, 1, 2, 3, 51, 2.0);
  const PartitionBlock P = middle_block(A);
  const LocalFactorization lf = factor_lu(P);
  CHECK(reconstruction_error(P, lf) < 1e-12);
  for (int t = 0; t < P.k1; ++t)
    for (int x = 0; x < P.L; ++x) {
      if (x < P.L + t - A.r) CHECK(lf.y.at(x, t) == 0.0);
      if (x < P.L + t - A.s) CHECK(lf.v.at(x, t) == 0.0);
    }
  bool zfill = false, wfill = false;
  for (int t = 0; t < P.k0; ++t)
    for (int x = A.s; x < P.L; ++x) {
      zfill |= lf.z.at(x, t) != 0.0;
      wfill |= lf.w.at(x, t) != 0.0;
    }
  CHECK(zfill);
  CHECK(wfill);
}

static void lud_middle_factor() {
  DenseMatrix body(2, 2);
  body.at(0, 0) = 2;
  body.at(1, 1) = 4;
  const DenseMatrix z(2, 1);
  const LocalFactorization lf = factor_lud(dense_block(body, z, z, z, z, DenseMatrix::identity(1)));
  const DenseMatrix S = lf.dense_S();
  CHECK(S.at(0, 0) == 2.0);
  CHECK(S.at(1, 1) == 4.0);
  CHECK(S.at(0, 1) == 0.0);
  CHECK(rel_err(lf.dense_N(), DenseMatrix::identity(2)) == 0.0);

  const StructuredMatrix A = generate_random(Kind::Banded, 30, 1, 1, 1, 52, 2.0);
  const PartitionBlock P = middle_block(A);
  const LocalFactorization lf2 = factor_lud(P);
  CHECK(reconstruction_error(P, lf2) < 1e-12);
  for (int t = 0; t < P.k1; ++t)
    for (int x = 0; x < P.L; ++x)
      if (P.b1.at(x, t) == 0.0) CHECK(lf2.v.at(x, t) == 0.0);
  for (int t = 0; t < P.k0; ++t)
    for (int x = 0; x < P.L; ++x)
      if (P.c0.at(x, t) == 0.0) CHECK(lf2.w.at(x, t) == 0.0);
  bool yfill = false;
  for (int x = 0; x < P.L - 2; ++x) yfill |= lf2.y.at(x, 0) != 0.0;
  CHECK(yfill);
}

static void cyclic_reduction() {
  const StructuredMatrix small = generate_random(Kind::Banded, 5, 1, 1, 1, 3, 2.0);
  REQUIRE(extract_block(small, plan_partition(small, 2), 1).L <= 2);

  const StructuredMatrix A = generate_random(Kind::Banded, 23, 1, 1, 1, 53, 2.0);
  const PartitionBlock P = middle_block(A);
  REQUIRE(P.L == 7);
  const LocalFactorization cr = factor_cyclic_reduction(P);
  CHECK(cr.cr_levels == 3);
  CHECK(reconstruction_error(P, cr) < 1e-12);
  CHECK(cr.v.rows == 0);
  CHECK(cr.w.rows == 0);
  CHECK(cr.y.rows == 0);
  CHECK(cr.z.rows == 0);
  const LocalFactorization lu = factor_lu(P);
  CHECK(rel_err(cr.alpha1, lu.alpha1) < 1e-10);
  CHECK(rel_err(cr.alpha2, lu.alpha2) < 1e-10);
  CHECK(rel_err(cr.beta, lu.beta) < 1e-10);
  CHECK(rel_err(cr.gamma, lu.gamma) < 1e-10);
  const LocalFactorization lud = factor_lud(P);
  CHECK(rel_err(lud.alpha2, lu.alpha2) < 1e-10);
  CHECK(rel_err(lud.beta, lu.beta) < 1e-10);

  const StructuredMatrix tiny = generate_random(Kind::Banded, 7, 1, 1, 1, 54, 2.0);
  const PartitionBlock T1 = extract_block(tiny, plan_partition(tiny, 3), 3);
  REQUIRE(T1.L == 1);
  const LocalFactorization crt = factor_cyclic_reduction(T1);
  CHECK(crt.cr_levels == 0);
  CHECK(reconstruction_error(T1, crt) < 1e-12);

  CHECK_THROWS_CODE(factor_cyclic_reduction(middle_block(generate_random(Kind::Banded, 30, 1, 2, 1, 5, 2.0))),
                    Errc::UnsupportedStructure);
}

static void block_cyclic_reduction() {
  const StructuredMatrix A = generate_random(Kind::BlockTridiagonal, 36, 3, 1, 1, 55, 2.0);
  const PartitionBlock P = middle_block(A);
  const LocalFactorization cr = factor_cyclic_reduction(P);
  const LocalFactorization lu = factor_lu(P);
  CHECK(reconstruction_error(P, cr) < 1e-12);
  CHECK(rel_err(cr.alpha2, lu.alpha2) < 1e-10);
  CHECK(rel_err(cr.gamma, lu.gamma) < 1e-10);
}

static void arce_unsupported() {
  const StructuredMatrix A = generate_random(Kind::Abd, 64, 2, 1, 1, 57, 2.0);
  CHECK_THROWS_CODE(factor_arce(middle_block(A)), Errc::UnsupportedStructure);
  CHECK_THROWS_CODE(factor(Strategy::Arce, middle_block(A)), Errc::UnsupportedStructure);
}

static void lupivot_without_triggers() {
  const StructuredMatrix A = generate_random(Kind::Banded, 34, 1, 1, 2, 59, 2.0);
  const PartitionBlock P = middle_block(A);
  const LocalFactorization piv = factor_lu_pivot(P, 1e-8);
  const LocalFactorization lu = factor_lu(P);
  CHECK(piv.extras.empty());
  CHECK(reconstruction_error(P, piv) < 1e-12);
  CHECK(rel_err(piv.alpha1, lu.alpha1) < 1e-10);
  CHECK(rel_err(piv.alpha2, lu.alpha2) < 1e-10);
  CHECK(rel_err(piv.beta, lu.beta) < 1e-10);
  CHECK(rel_err(piv.gamma, lu.gamma) < 1e-10);
}

static void singular_minor_defers() {
  DenseMatrix body(5, 5);
  body.at(0, 0) = 2, body.at(0, 1) = 1;
  body.at(1, 0) = 1, body.at(1, 1) = 0.5, body.at(1, 2) = 1;  // 0.5 - 1/2 * 1 = 0 after step 1
  body.at(2, 2) = 3, body.at(2, 3) = 1;
  body.at(3, 2) = 1, body.at(3, 3) = 3, body.at(3, 4) = 1;
  body.at(4, 3) = 1, body.at(4, 4) = 3;
  DenseMatrix b0(5, 1), c0(5, 1), b1(5, 1), c1(5, 1), ar(1, 1);
  b0.at(0, 0) = c0.at(0, 0) = 1;
  b1.at(4, 0) = c1.at(4, 0) = 1;
  ar.at(0, 0) = 3;
  const PartitionBlock P = dense_block(body, b0, c0, b1, c1, ar);
  CHECK(std::fabs(body.at(0, 0) * body.at(1, 1) - body.at(0, 1) * body.at(1, 0)) == 0.0);
  const LocalFactorization lf = factor_lu_pivot(P, 1e-8);
  REQUIRE(lf.extras.size() == 1);
  CHECK(lf.extras[0].position == 1);
  CHECK(lf.kept_dim() == 3);
  CHECK(reconstruction_error(P, lf) < 1e-12);
  const LocalFactorization qf = factor_qr(P, 1e-8);
  REQUIRE(qf.extras.size() == 1);
  CHECK(reconstruction_error(P, qf) < 1e-12);
}

static void qr_orthogonality() {
  const DenseMatrix I3 = DenseMatrix::identity(3), z(3, 1);
  const LocalFactorization ilf = factor_qr(dense_block(I3, z, z, z, z, DenseMatrix::identity(1)), 1e-8);
  CHECK(rel_err(matmul(ilf.dense_N(), ilf.dense_S()), I3) < 1e-14);

  const StructuredMatrix A = generate_random(Kind::Banded, 34, 1, 2, 1, 60, 2.0);
  const PartitionBlock P = middle_block(A);
  const LocalFactorization lf = factor_qr(P, 1e-8);
  CHECK(reconstruction_error(P, lf) < 1e-12);
  const DenseMatrix Q = lf.dense_N();
  CHECK(rel_err(matmul(transpose(Q), Q), DenseMatrix::identity(P.L)) < 1e-12);
  const DenseMatrix S = lf.dense_S();
  for (int i = 0; i < P.L; ++i)
    for (int j = 0; j < i; ++j) CHECK(std::fabs(S.at(i, j)) < 1e-13);
  for (int t = 0; t < P.k1; ++t)
    for (int x = 0; x < P.L; ++x) {
      if (x < P.L + t - A.s) CHECK(lf.v.at(x, t) == 0.0);
      if (x < P.L + t - A.r - A.s) CHECK(std::fabs(lf.y.at(x, t)) < 1e-13);
    }
}

static void n_inv_s_inv_compose() {
  const StructuredMatrix A = generate_random(Kind::Banded, 31, 1, 2, 2, 61, 2.0);
  const PartitionBlock P = middle_block(A);
  const Vector rhs = random_vector(P.L, 9);
  const Vector want = lu_solve(P.body_dense(), rhs);
  for (Strategy s : {Strategy::Lu, Strategy::Lud, Strategy::LuPivot, Strategy::Qr}) {
    const LocalFactorization lf = factor(s, P, 1e-8);
    CHECK(rel_err(lf.apply_S_inv(lf.apply_N_inv(rhs)), want) < 1e-10);
  }
  const StructuredMatrix T = generate_random(Kind::Banded, 31, 1, 1, 1, 62, 2.0);
  const PartitionBlock tb = middle_block(T);
  const LocalFactorization cr = factor_cyclic_reduction(tb);
  const Vector rhs2 = random_vector(tb.L, 10);
  CHECK(rel_err(cr.apply_S_inv(cr.apply_N_inv(rhs2)), lu_solve(tb.body_dense(), rhs2)) < 1e-10);
  const LocalFactorization qf = factor_qr(P, 1e-8);
  CHECK(rel_err(matvec(qf.dense_N(), qf.apply_N_inv(rhs)), rhs) < 1e-12);
}

static void zero_pivot() {
  DenseMatrix body(2, 2);
  body.at(0, 1) = body.at(1, 0) = 1;
  const DenseMatrix z(2, 1);
  const PartitionBlock P = dense_block(body, z, z, z, z, DenseMatrix::identity(1));
  CHECK_THROWS_CODE(factor_lu(P), Errc::ZeroPivot);
  CHECK_THROWS_CODE(factor_lud(P), Errc::ZeroPivot);
  const LocalFactorization piv = factor_lu_pivot(P, 1e-10);
  CHECK(reconstruction_error(P, piv) < 1e-12);
  CHECK_THROWS_CODE(factor_lu_pivot(P, 0.0), Errc::InvalidParameter);
}

// condense -> reduced values -> backsolve of one partition reproduces the
// body of a direct solve (phase 1 + 3 of src/parfact.cpp:186-239)
static void condense_backsolve_roundtrip() {
  const StructuredMatrix A = generate_random(Kind::Banded, 60, 1, 2, 2, 63, 2.0);
  const PartitionPlan plan = plan_partition(A, 3);
  const PartitionBlock P = extract_block(A, plan, 2);
  const Vector f = random_vector(A.n, 11);
  const Vector x = lu_solve(to_dense(A), f);
  const int b = plan.body_ranges[1].first, ls = plan.separator_starts[0], rs = plan.separator_starts[1];
  for (Strategy s : {Strategy::Lu, Strategy::Lud, Strategy::LuPivot, Strategy::Qr}) {
    const LocalFactorization lf = factor(s, P, 1e-8);
    const Vector fb(f.begin() + b, f.begin() + b + P.L);
    Vector ghat, kr;
    lf.condense(fb, ghat, kr);
    CHECK(int(kr.size()) == lf.kept_dim());
    Vector xk;
    for (int t = 0; t < P.k0; ++t) xk.push_back(x[ls + t]);
    for (const auto& e : lf.extras) xk.push_back(x[b + e.position]);
    for (int t = 0; t < P.k1; ++t) xk.push_back(x[rs + t]);
    const Vector xb = lf.backsolve(ghat, xk);
    CHECK(rel_err(xb, Vector(x.begin() + b, x.begin() + b + P.L)) < 1e-12);
  }
  Vector g3, k3;
  CHECK_THROWS_CODE(factor_lu(P).condense(Vector(3, 0.0), g3, k3), Errc::DimensionMismatch);
}

// solve_reduced on a ReducedSystem (SPEC.md: T = I -> x = rhs; [[2,1],[1,2]] x = [3,3])
static void solve_reduced_examples() {
  ReducedSystem R;
  R.q = R.dim = 3;
  R.T = DenseMatrix::identity(3);
  const Vector rhs{1.0, -2.0, 3.5};
  CHECK(solve_reduced(R, rhs) == rhs);
  ReducedSystem S;
  S.q = S.dim = 2;
  S.T = DenseMatrix(2, 2);
  S.T.at(0, 0) = S.T.at(1, 1) = 2;
  S.T.at(0, 1) = S.T.at(1, 0) = 1;
  SolveStats st;
  const Vector x = solve_reduced(S, {3.0, 3.0}, &st);
  CHECK(std::fabs(x[0] - 1.0) < 1e-15 && std::fabs(x[1] - 1.0) < 1e-15);
  CHECK(st.reduced_ops == 6);  // the reference's count for dim 2: 2 elimination + 1 forward + 3 backward
  ReducedSystem Z;
  Z.q = Z.dim = 2;
  Z.T = DenseMatrix(2, 2);
  CHECK_THROWS_CODE(solve_reduced(Z, {1.0, 1.0}), Errc::SingularReducedSystem);
  CHECK_THROWS_CODE(solve_reduced(S, {1.0}), Errc::DimensionMismatch);
}

// parallel_factor: factor_seconds filled, reduced usable on its own, and
// materialized locals that assemble into the reduced matrix T
static void parallel_factor_locals() {
  const StructuredMatrix A = generate_random(Kind::Banded, 403, 1, 2, 2, 64, 2.0);
  const int p = 5;
  ParallelFactorization F = parallel_factor(A, p, Strategy::Lu);
  CHECK(F.factor_seconds > 0.0);
  CHECK(F.locals.empty());
  const Vector f = random_vector(A.n, 12);
  const Vector rr = random_vector(F.reduced.dim, 13);
  const Vector x1 = solve_reduced(F.reduced, rr);
  CHECK(rel_err(x1, lu_solve(F.reduced.T, rr)) < 1e-12);
  ReducedSystem no_dense = F.reduced;
  no_dense.T = DenseMatrix();
  CHECK(rel_err(solve_reduced(no_dense, rr), x1) < 1e-12);  // through the device handle
  materialize_locals(F, A);
  REQUIRE(int(F.locals.size()) == p);
  DenseMatrix T(F.reduced.dim, F.reduced.dim);
  const int k = F.plan.sep_size;
  for (int i = 0; i < p; ++i) {
    const LocalFactorization& lf = F.locals[i];
    CHECK(int(F.kept_maps[i].size()) == lf.kept_dim());
    for (int a = 0; a < lf.kept_dim(); ++a)
      for (int b = 0; b < lf.kept_dim(); ++b) T.at(F.kept_maps[i][a], F.kept_maps[i][b]) += lf.kept.at(a, b);
  }
  CHECK(rel_err(T, F.reduced.T) < 1e-14);
  CHECK(k == 2);
  SolveStats st;
  (void)solve(F, f, &st);
  CHECK(st.factor_seconds == 0.0);  // solve never writes it (src/parfact.cpp:233-237)
}

int main(int argc, char** argv) {
  if (argc < 2 || std::strcmp(argv[1], "--gpu") != 0) {
    std::printf("usage: test_localfact --gpu\n");
    return 2;
  }
  identity_body();
  toeplitz_block();
  lu_sparsity();
  lud_middle_factor();
  cyclic_reduction();
  block_cyclic_reduction();
  arce_unsupported();
  lupivot_without_triggers();
  singular_minor_defers();
  qr_orthogonality();
  n_inv_s_inv_compose();
  zero_pivot();
  condense_backsolve_roundtrip();
  solve_reduced_examples();
  parallel_factor_locals();
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
