// host_core.cpp -- C++ host side of the B200 solver API: errors, dense
// helpers, structured-matrix descriptors, partition views and strategy names.
// Everything that solves goes through the C ABI (psg.h); this file only holds
// host data structures and their validation (shared with the C ABI).
#include <algorithm>
#include <cmath>
#include <sstream>

#include "parsol/errors.hpp"
#include "parsol/localfact.hpp"
#include "parsol/partition.hpp"
#include "parsol/structmat.hpp"
#include "parsol/rng.hpp"
#include "psg.h"

namespace parsol {

const char* errc_name(Errc c) {
  switch (c) {
    case Errc::DimensionMismatch: return "DimensionMismatch";
    case Errc::InvalidBandwidth: return "InvalidBandwidth";
    case Errc::CornerForbidden: return "CornerForbidden";
    case Errc::TooLargeForDense: return "TooLargeForDense";
    case Errc::InvalidParameter: return "InvalidParameter";
    case Errc::ParseError: return "ParseError";
    case Errc::UnsupportedVersion: return "UnsupportedVersion";
    case Errc::TooManyPartitions: return "TooManyPartitions";
    case Errc::UnsupportedKind: return "UnsupportedKind";
    case Errc::UnsupportedStructure: return "UnsupportedStructure";
    case Errc::IndexOutOfRange: return "IndexOutOfRange";
    case Errc::ZeroPivot: return "ZeroPivot";
    case Errc::SingularBlock: return "SingularBlock";
    case Errc::SingularFactor: return "SingularFactor";
    case Errc::SingularReducedSystem: return "SingularReducedSystem";
    case Errc::SingularWindow: return "SingularWindow";
    case Errc::ExhaustedBody: return "ExhaustedBody";
    case Errc::StepTooLarge: return "StepTooLarge";
    case Errc::InvalidInterval: return "InvalidInterval";
    case Errc::ExpmFailure: return "ExpmFailure";
    case Errc::NotConverged: return "NotConverged";
    case Errc::IoError: return "IoError";
    case Errc::Cuda: return "Cuda";
  }
  return "UnknownError";
}

// ---------------------------------------------------------------------------
// dense helpers
// ---------------------------------------------------------------------------
DenseMatrix DenseMatrix::identity(int n) {
  DenseMatrix I(n, n);
  for (int i = 0; i < n; ++i) I.at(i, i) = 1.0;
  return I;
}

DenseMatrix matmul(const DenseMatrix& A, const DenseMatrix& B) {
  if (A.cols != B.rows) fail(Errc::DimensionMismatch, "matmul shapes");
  DenseMatrix C(A.rows, B.cols);
  for (int i = 0; i < A.rows; ++i)
    for (int k = 0; k < A.cols; ++k) {
      const double aik = A.at(i, k);
      for (int j = 0; j < B.cols; ++j) C.at(i, j) += aik * B.at(k, j);
    }
  return C;
}

Vector matvec(const DenseMatrix& A, const Vector& x) {
  if (A.cols != int(x.size())) fail(Errc::DimensionMismatch, "matvec shapes");
  Vector y(A.rows, 0.0);
  for (int i = 0; i < A.rows; ++i)
    for (int j = 0; j < A.cols; ++j) y[i] += A.at(i, j) * x[j];
  return y;
}

DenseMatrix transpose(const DenseMatrix& A) {
  DenseMatrix T(A.cols, A.rows);
  for (int i = 0; i < A.rows; ++i)
    for (int j = 0; j < A.cols; ++j) T.at(j, i) = A.at(i, j);
  return T;
}

DenseMatrix add(const DenseMatrix& A, const DenseMatrix& B) {
  DenseMatrix C = A;
  for (std::size_t i = 0; i < C.a.size(); ++i) C.a[i] += B.a[i];
  return C;
}

DenseMatrix sub(const DenseMatrix& A, const DenseMatrix& B) {
  DenseMatrix C = A;
  for (std::size_t i = 0; i < C.a.size(); ++i) C.a[i] -= B.a[i];
  return C;
}

DenseMatrix scale(const DenseMatrix& A, double s) {
  DenseMatrix C = A;
  for (double& v : C.a) v *= s;
  return C;
}

double inf_norm(const DenseMatrix& A) {
  double best = 0.0;
  for (int i = 0; i < A.rows; ++i) {
    double s = 0.0;
    for (int j = 0; j < A.cols; ++j) s += std::fabs(A.at(i, j));
    best = std::max(best, s);
  }
  return best;
}

double inf_norm(const Vector& v) {
  double best = 0.0;
  for (double x : v) best = std::max(best, std::fabs(x));
  return best;
}

DenseLu::DenseLu(DenseMatrix A) : lu(std::move(A)) {
  if (lu.rows != lu.cols) fail(Errc::DimensionMismatch, "LU needs a square matrix");
  const int n = lu.rows;
  perm.resize(n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(lu.at(i, k)) > std::fabs(lu.at(piv, k))) piv = i;
    if (lu.at(piv, k) == 0.0) fail(Errc::SingularFactor, "zero pivot column in dense LU");
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(lu.at(k, j), lu.at(piv, j));
      std::swap(perm[k], perm[piv]);
    }
    for (int i = k + 1; i < n; ++i) {
      const double m = lu.at(i, k) / lu.at(k, k);
      lu.at(i, k) = m;
      for (int j = k + 1; j < n; ++j) lu.at(i, j) -= m * lu.at(k, j);
    }
  }
}

Vector DenseLu::solve(const Vector& b) const {
  const int n = lu.rows;
  if (int(b.size()) != n) fail(Errc::DimensionMismatch, "LU solve rhs");
  Vector y(n);
  for (int i = 0; i < n; ++i) y[i] = b[perm[i]];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) y[i] -= lu.at(i, j) * y[j];
  for (int i = n - 1; i >= 0; --i) {
    for (int j = i + 1; j < n; ++j) y[i] -= lu.at(i, j) * y[j];
    y[i] /= lu.at(i, i);
  }
  return y;
}

DenseMatrix DenseLu::solve(const DenseMatrix& B) const {
  DenseMatrix X(B.rows, B.cols);
  Vector col(B.rows);
  for (int j = 0; j < B.cols; ++j) {
    for (int i = 0; i < B.rows; ++i) col[i] = B.at(i, j);
    const Vector x = solve(col);
    for (int i = 0; i < B.rows; ++i) X.at(i, j) = x[i];
  }
  return X;
}

Vector lu_solve(const DenseMatrix& A, const Vector& b) { return DenseLu(A).solve(b); }
DenseMatrix lu_solve(const DenseMatrix& A, const DenseMatrix& B) { return DenseLu(A).solve(B); }
DenseMatrix inverse(const DenseMatrix& A) { return DenseLu(A).solve(DenseMatrix::identity(A.rows)); }

// ---------------------------------------------------------------------------
// structured matrices
// ---------------------------------------------------------------------------
const char* kind_name(Kind k) {
  switch (k) {
    case Kind::Banded: return "banded";
    case Kind::BlockTridiagonal: return "blocktri";
    case Kind::Abd: return "abd";
    case Kind::Babd: return "babd";
    case Kind::CirculantLike: return "circulant";
  }
  return "?";
}

Kind kind_from_name(const std::string& s) {
  if (s == "banded") return Kind::Banded;
  if (s == "blocktri") return Kind::BlockTridiagonal;
  if (s == "abd") return Kind::Abd;
  if (s == "babd") return Kind::Babd;
  if (s == "circulant") return Kind::CirculantLike;
  fail(Errc::ParseError, "unknown kind '" + s + "'");
}

namespace {

psg_desc host_desc(Kind kind, int n, int m, int s, int r, const std::vector<double>& data,
                   const std::vector<double>& corner, int cr, int cc) {
  return psg_desc{int(kind), n, m, s, r, data.data(), data.size(), corner.empty() ? nullptr : corner.data(), cr, cc,
                  0};
}

long band_offset(int n, int s, int d) {
  long off = 0;
  for (int b = -s; b < d; ++b) off += n - std::abs(b);
  return off;
}

std::pair<int, int> abd_span(int n, int m, int s, int r, int b) {
  return {std::max(0, b * m - s), std::min(n, b * m + m + r)};
}

long abd_row_offset(int m, int s, int r, int b) {  // rows 1.. are m+s+r wide (s <= m)
  return b == 0 ? 0 : long(m) * (m + r) + long(b - 1) * m * (m + r + s);
}

}  // namespace

std::size_t body_entry_count(Kind kind, int n, int m, int s, int r) {
  return psg_body_entry_count(int(kind), n, m, s, r);
}

bool StructuredMatrix::in_structure(int i, int j) const {
  if (i < 0 || j < 0 || i >= n || j >= n) return false;
  switch (kind) {
    case Kind::Banded: return j - i <= r && i - j <= s;
    case Kind::BlockTridiagonal: return std::abs(i / m - j / m) <= 1;
    case Kind::Abd:
    case Kind::Babd: {
      auto [c0, c1] = abd_span(n, m, s, r, i / m);
      if (j >= c0 && j < c1) return true;
      return kind == Kind::Babd && i < corner_rows && j >= n - corner_cols;
    }
    case Kind::CirculantLike: {
      int dd = j - i;
      if (dd < 0) dd += n;
      return dd <= r || n - dd <= s;
    }
  }
  return false;
}

double StructuredMatrix::at(int i, int j) const {
  if (!in_structure(i, j)) return 0.0;
  switch (kind) {
    case Kind::Banded: {
      const int d = j - i;
      return data[band_offset(n, s, d) + (i - std::max(0, -d))];
    }
    case Kind::BlockTridiagonal: {
      const int bi = i / m, bj = j / m;
      const long off = bi == 0 ? 0 : long(3 * bi - 1) * m * m;
      const int blk = bi > 0 ? bj - bi + 1 : bj - bi;
      return data[off + long(blk) * m * m + long(i - bi * m) * m + (j - bj * m)];
    }
    case Kind::Abd:
    case Kind::Babd: {
      const int b = i / m;
      auto [c0, c1] = abd_span(n, m, s, r, b);
      if (j >= c0 && j < c1) return data[abd_row_offset(m, s, r, b) + long(i - b * m) * (c1 - c0) + (j - c0)];
      return corner[long(i) * corner_cols + (j - (n - corner_cols))];
    }
    case Kind::CirculantLike: {
      int dd = j - i;
      if (dd < 0) dd += n;
      const int d = dd <= r ? dd : dd - n;
      return data[long(d + s) * n + i];
    }
  }
  return 0.0;
}

bool StructuredMatrix::corner_canonical() const {
  if (kind != Kind::CirculantLike) return true;
  return r == 0;
}

StructuredMatrix make(Kind kind, int n, int m, int s, int r, std::vector<double> data, std::vector<double> corner,
                      int corner_rows, int corner_cols) {
  const psg_desc d = host_desc(kind, n, m, s, r, data, corner, corner_rows, corner_cols);
  char err[512];
  if (int rc = psg_validate(&d, err, sizeof err)) fail(Errc(rc - 1), err);
  StructuredMatrix A;
  A.kind = kind;
  A.n = n;
  A.m = m;
  A.s = s;
  A.r = r;
  A.data = std::move(data);
  A.corner = std::move(corner);
  A.corner_rows = corner_rows;
  A.corner_cols = corner_cols;
  return A;
}

DenseMatrix to_dense(const StructuredMatrix& A, int limit) {
  if (A.n > limit) fail(Errc::TooLargeForDense, "n = " + std::to_string(A.n) + " exceeds dense limit " +
                                                   std::to_string(limit));
  DenseMatrix D(A.n, A.n);
  for (int i = 0; i < A.n; ++i)
    for (int j = 0; j < A.n; ++j) D.at(i, j) = A.at(i, j);
  return D;
}

Vector matvec(const StructuredMatrix& A, const Vector& x) {
  if (int(x.size()) != A.n) fail(Errc::DimensionMismatch, "matvec length");
  Vector y(A.n);
  const psg_desc d = host_desc(A.kind, A.n, A.m, A.s, A.r, A.data, A.corner, A.corner_rows, A.corner_cols);
  char err[512];
  if (int rc = psg_matvec(&d, x.data(), y.data(), 0, nullptr, err, sizeof err)) fail(Errc(rc - 1), err);
  return y;
}

std::pair<int, int> scalar_envelope(const StructuredMatrix& A) {
  switch (A.kind) {
    case Kind::Banded:
    case Kind::CirculantLike: return {A.s, A.r};
    case Kind::BlockTridiagonal: return {2 * A.m - 1, 2 * A.m - 1};
    default: return {A.m - 1 + A.s, A.m - 1 + A.r};
  }
}

// generate_random: draws in storage order, then the diagonal rescaled to
// +-dominance * max(off-row |sum|, 1) (semantics of src/structmat.cpp:282-333).
StructuredMatrix generate_random(Kind kind, int n, int m, int s, int r, std::uint64_t seed, double dominance) {
  if (dominance < 0) fail(Errc::InvalidParameter, "dominance must be >= 0");
  SplitMix64 rng(seed);
  std::vector<double> data(body_entry_count(kind, n, m, s, r));
  for (auto& v : data) v = rng.next_unit();
  std::vector<double> corner;
  int cr = 0, cc = 0;
  if (kind == Kind::Babd) {
    cr = cc = m;
    corner.resize(std::size_t(m) * m);
    for (auto& v : corner) v = rng.next_unit();
  }
  StructuredMatrix A = make(kind, n, m, s, r, std::move(data), std::move(corner), cr, cc);
  if (dominance > 0.0) {
    for (int i = 0; i < n; ++i) {
      double off = 0.0;
      for (int j = 0; j < n; ++j)
        if (j != i && A.in_structure(i, j)) off += std::fabs(A.at(i, j));
      const double mag = dominance * std::max(off, 1.0);
      const double val = A.at(i, i) < 0 ? -mag : mag;
      switch (kind) {
        case Kind::Banded: A.data[band_offset(n, s, 0) + i] = val; break;
        case Kind::BlockTridiagonal: {
          const int b = i / m;
          const long offr = b == 0 ? 0 : long(3 * b - 1) * m * m;
          A.data[offr + long(b > 0 ? 1 : 0) * m * m + long(i - b * m) * m + (i - b * m)] = val;
          break;
        }
        default: {
          const int b = i / m;
          auto [c0, c1] = abd_span(n, m, s, r, b);
          A.data[abd_row_offset(m, s, r, b) + long(i - b * m) * (c1 - c0) + (i - c0)] = val;
          break;
        }
      }
    }
  }
  return A;
}

// ---------------------------------------------------------------------------
// partitions
// ---------------------------------------------------------------------------
PartitionPlan plan_partition(const StructuredMatrix& A, int p) {
  if (p < 2) fail(Errc::TooManyPartitions, "p must be >= 2");
  const psg_desc d = host_desc(A.kind, A.n, A.m, A.s, A.r, A.data, A.corner, A.corner_rows, A.corner_cols);
  std::vector<int> bb(p), be(p), ss(p + 1);
  int cnt = 0, k = 0;
  char err[512];
  if (int rc = psg_plan(&d, p, bb.data(), be.data(), ss.data(), &cnt, &k, err, sizeof err)) fail(Errc(rc - 1), err);
  PartitionPlan plan;
  plan.kind = A.kind;
  plan.n = A.n;
  plan.m = A.m;
  plan.p = p;
  plan.sep_size = k;
  plan.has_corner = A.kind == Kind::Babd || A.kind == Kind::CirculantLike;
  plan.corner_rows = A.kind == Kind::CirculantLike ? A.s : A.corner_rows;  // wrap extent (src/partition.cpp:68-71)
  plan.corner_cols = A.kind == Kind::CirculantLike ? A.s : A.corner_cols;
  for (int i = 0; i < p; ++i) plan.body_ranges.emplace_back(bb[i], be[i]);
  plan.separator_starts.assign(ss.begin(), ss.begin() + cnt);
  return plan;
}

// Rotate a circulant-like matrix's rows down by r so every wrapped entry sits
// in the upper-right corner (reference src/partition.cpp:175-202): a pure
// relabelling of the stored bands; the GPU factorization does the same
// rotation on the device (psg_factor).
std::pair<StructuredMatrix, Permutation> permute_corner(const StructuredMatrix& A) {
  if (A.kind != Kind::CirculantLike && A.kind != Kind::Babd)
    fail(Errc::UnsupportedKind, "permute_corner applies to circulant-like and BABD matrices");
  Permutation perm;
  perm.source.resize(A.n);
  for (int i = 0; i < A.n; ++i) perm.source[i] = i;
  if (A.corner_canonical()) return {A, perm};
  const int n = A.n, s = A.s, r = A.r;
  for (int i = 0; i < n; ++i) perm.source[i] = ((i - r) % n + n) % n;
  std::vector<double> data(std::size_t(s + r + 1) * n);
  for (int q = 0; q <= s + r; ++q)
    for (int i = 0; i < n; ++i) data[std::size_t(q) * n + i] = A.data[std::size_t(q) * n + perm.source[i]];
  return {make(Kind::CirculantLike, n, 1, s + r, 0, std::move(data)), perm};
}

DenseMatrix PartitionBlock::local_dense() const {
  const int dim = k0 + L + k1;
  DenseMatrix M(dim, dim);
  for (int x = 0; x < L; ++x) {
    for (int t = 0; t < k0; ++t) {
      M.at(k0 + x, t) = b0.at(x, t);
      M.at(t, k0 + x) = c0.at(x, t);
    }
    for (int t = 0; t < k1; ++t) {
      M.at(k0 + x, k0 + L + t) = c1.at(x, t);
      M.at(k0 + L + t, k0 + x) = b1.at(x, t);
    }
    for (int y = 0; y < L; ++y) M.at(k0 + x, k0 + y) = body_at(x, y);
  }
  for (int t = 0; t < k1; ++t)
    for (int u = 0; u < k1; ++u) M.at(k0 + L + t, k0 + L + u) = a_right.at(t, u);
  return M;
}

// Host view of partition i (1-based) -- the blocks the reference's
// extract_block builds (src/partition.cpp:107-173); the GPU never builds them.
PartitionBlock extract_block(const StructuredMatrix& A, const PartitionPlan& plan, int i) {
  if (i < 1 || i > plan.p) fail(Errc::IndexOutOfRange, "partition index " + std::to_string(i));
  PartitionBlock blk;
  blk.index = i;
  blk.kind = A.kind;
  blk.m = A.m;
  blk.s = A.s;
  blk.r = A.r;
  auto [b, e] = plan.body_ranges[i - 1];
  blk.body_begin = b;
  blk.L = e - b;
  const int k = plan.sep_size;
  const int left = plan.has_corner ? i - 1 : i - 2, right = plan.has_corner ? i : i - 1;
  blk.k0 = left >= 0 ? k : 0;
  blk.k1 = right < plan.sep_count() ? k : 0;
  auto [es, er] = scalar_envelope(A);
  blk.env_s = std::min(es, blk.L - 1);
  blk.env_r = std::min(er, blk.L - 1);
  const int w = blk.env_s + 1 + blk.env_r;
  blk.env.assign(std::size_t(blk.L) * w, 0.0);
  for (int x = 0; x < blk.L; ++x)
    for (int j = std::max(0, x - blk.env_s); j <= std::min(blk.L - 1, x + blk.env_r); ++j)
      blk.env[std::size_t(x) * w + (j - x + blk.env_s)] = A.at(b + x, b + j);
  blk.b0 = DenseMatrix(blk.L, blk.k0);
  blk.c0 = DenseMatrix(blk.L, blk.k0);
  blk.b1 = DenseMatrix(blk.L, blk.k1);
  blk.c1 = DenseMatrix(blk.L, blk.k1);
  if (blk.k0) {
    const int ls = plan.separator_starts[left];
    for (int x = 0; x < blk.L; ++x)
      for (int t = 0; t < k; ++t) {
        blk.b0.at(x, t) = A.at(b + x, ls + t);
        blk.c0.at(x, t) = A.at(ls + t, b + x);
      }
    blk.a_left = DenseMatrix(k, k);
    for (int t = 0; t < k; ++t)
      for (int u = 0; u < k; ++u) blk.a_left.at(t, u) = A.at(ls + t, ls + u);
  }
  if (blk.k1) {
    const int rs = plan.separator_starts[right];
    for (int x = 0; x < blk.L; ++x)
      for (int t = 0; t < k; ++t) {
        blk.c1.at(x, t) = A.at(b + x, rs + t);
        blk.b1.at(x, t) = A.at(rs + t, b + x);
      }
    blk.a_right = DenseMatrix(k, k);
    for (int t = 0; t < k; ++t)
      for (int u = 0; u < k; ++u) blk.a_right.at(t, u) = A.at(rs + t, rs + u);
  }
  if (plan.has_corner && i == 1) {
    const int s0 = plan.separator_starts.front(), sp = plan.separator_starts.back();
    blk.corner_slice = DenseMatrix(k, k);
    for (int t = 0; t < k; ++t)
      for (int u = 0; u < k; ++u) blk.corner_slice.at(t, u) = A.at(s0 + t, sp + u);
  }
  return blk;
}

std::string describe(const PartitionPlan& plan) {
  std::ostringstream out;
  out << "plan kind=" << kind_name(plan.kind) << " n=" << plan.n << " p=" << plan.p << " sep_size=" << plan.sep_size
      << (plan.has_corner ? " corner" : "") << '\n';
  for (int i = 0; i < plan.p; ++i) {
    if (plan.has_corner)
      out << "  a(" << i << ") at " << plan.separator_starts[i] << '\n';
    else if (i > 0)
      out << "  a(" << i << ") at " << plan.separator_starts[i - 1] << '\n';
    out << "  A(" << i + 1 << ") rows [" << plan.body_ranges[i].first << ", " << plan.body_ranges[i].second << ")\n";
  }
  if (plan.has_corner) out << "  a(" << plan.p << ") at " << plan.separator_starts.back() << '\n';
  return out.str();
}

// ---------------------------------------------------------------------------
// strategies (src/localfact.cpp:9-42 semantics)
// ---------------------------------------------------------------------------
const char* strategy_name(Strategy s) {
  switch (s) {
    case Strategy::Lu: return "lu";
    case Strategy::Lud: return "lud";
    case Strategy::CyclicReduction: return "cr";
    case Strategy::Arce: return "arce";
    case Strategy::LuPivot: return "lupivot";
    case Strategy::Qr: return "qr";
  }
  return "?";
}

Strategy strategy_from_name(const std::string& s) {
  if (s == "lu") return Strategy::Lu;
  if (s == "lud") return Strategy::Lud;
  if (s == "cr") return Strategy::CyclicReduction;
  if (s == "arce") return Strategy::Arce;
  if (s == "lupivot") return Strategy::LuPivot;
  if (s == "qr") return Strategy::Qr;
  fail(Errc::InvalidParameter, "unknown strategy '" + s + "'");
}

bool strategy_supports(Strategy s, Kind k, int bs, int br) {
  switch (s) {
    case Strategy::Lu:
    case Strategy::Lud:
    case Strategy::LuPivot:
    case Strategy::Qr: return true;
    case Strategy::CyclicReduction: return k == Kind::BlockTridiagonal || (k == Kind::Banded && bs == 1 && br == 1);
    case Strategy::Arce: return k == Kind::Abd || k == Kind::Babd;
  }
  return false;
}

}  // namespace parsol
