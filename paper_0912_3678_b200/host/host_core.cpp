// host_core.cpp -- C++ host side of the B200 solver API: errors, dense
// helpers, structured-matrix descriptors, partition views and strategy names.
// Everything that solves goes through the C ABI (psg.h); this file only holds
// host data structures and their validation (shared with the C ABI).
#include <algorithm>
#include <cmath>
#include <functional>
#include <numeric>
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
// dense helpers (host-side type of T and of the test oracles; not on the
// solve path).  The elimination keeps a row-index indirection instead of
// swapping rows, and products are formed as row-by-column dot products.
// ---------------------------------------------------------------------------
DenseMatrix DenseMatrix::identity(int n) {
  DenseMatrix I(n, n);
  for (int i = 0; i < n; ++i) I.a[std::size_t(i) * n + i] = 1.0;
  return I;
}

DenseMatrix transpose(const DenseMatrix& A) {
  DenseMatrix T(A.cols, A.rows);
  for (std::size_t e = 0; e < A.a.size(); ++e) T.a[(e % A.cols) * A.rows + e / A.cols] = A.a[e];
  return T;
}

DenseMatrix matmul(const DenseMatrix& A, const DenseMatrix& B) {
  if (A.cols != B.rows) fail(Errc::DimensionMismatch, "matmul: " + std::to_string(A.rows) + "x" +
                                                        std::to_string(A.cols) + " times " + std::to_string(B.rows) +
                                                        "x" + std::to_string(B.cols));
  const DenseMatrix Bt = transpose(B);
  DenseMatrix C(A.rows, B.cols);
  for (int i = 0; i < A.rows; ++i) {
    const double* ai = A.a.data() + std::size_t(i) * A.cols;
    for (int j = 0; j < B.cols; ++j) {
      const double* bj = Bt.a.data() + std::size_t(j) * Bt.cols;
      double dot = 0.0;
      for (int k = 0; k < A.cols; ++k)
        if (ai[k] != 0.0) dot += ai[k] * bj[k];
      C.a[std::size_t(i) * C.cols + j] = dot;
    }
  }
  return C;
}

Vector matvec(const DenseMatrix& A, const Vector& x) {
  if (A.cols != int(x.size())) fail(Errc::DimensionMismatch, "matvec: matrix has " + std::to_string(A.cols) +
                                                              " columns, vector " + std::to_string(x.size()));
  Vector y(A.rows);
  for (int i = 0; i < A.rows; ++i) {
    double dot = 0.0;
    for (int j = 0; j < A.cols; ++j) dot += A.a[std::size_t(i) * A.cols + j] * x[j];
    y[i] = dot;
  }
  return y;
}

namespace {
template <typename Op>
DenseMatrix zip(const DenseMatrix& A, const DenseMatrix& B, Op op) {
  if (A.rows != B.rows || A.cols != B.cols) fail(Errc::DimensionMismatch, "elementwise operands differ in shape");
  DenseMatrix C(A.rows, A.cols);
  std::transform(A.a.begin(), A.a.end(), B.a.begin(), C.a.begin(), op);
  return C;
}
}  // namespace

DenseMatrix add(const DenseMatrix& A, const DenseMatrix& B) { return zip(A, B, std::plus<double>()); }
DenseMatrix sub(const DenseMatrix& A, const DenseMatrix& B) { return zip(A, B, std::minus<double>()); }

DenseMatrix scale(const DenseMatrix& A, double s) {
  DenseMatrix C = A;
  std::transform(C.a.begin(), C.a.end(), C.a.begin(), [s](double v) { return v * s; });
  return C;
}

double inf_norm(const Vector& v) {
  double m = 0.0;
  for (double x : v) m = std::max(m, std::fabs(x));
  return m;
}

double inf_norm(const DenseMatrix& A) {
  double m = 0.0;
  for (int i = 0; i < A.rows; ++i) {
    const auto row = A.a.begin() + std::ptrdiff_t(i) * A.cols;
    m = std::max(m, std::accumulate(row, row + A.cols, 0.0, [](double s, double v) { return s + std::fabs(v); }));
  }
  return m;
}

// Partial-pivot LU kept in the caller's row order: `perm[k]` is the original
// row that became pivot row k; rows are never moved, only re-indexed.
DenseLu::DenseLu(DenseMatrix A) : lu(std::move(A)) {
  if (lu.rows != lu.cols) fail(Errc::DimensionMismatch, "LU of a non-square matrix");
  const int n = lu.rows;
  perm.resize(n);
  std::iota(perm.begin(), perm.end(), 0);
  auto at = [&](int row, int col) -> double& { return lu.a[std::size_t(row) * n + col]; };
  for (int k = 0; k < n; ++k) {
    int best = k;
    for (int q = k + 1; q < n; ++q)
      if (std::fabs(at(perm[q], k)) > std::fabs(at(perm[best], k))) best = q;
    std::swap(perm[k], perm[best]);
    const int pr = perm[k];
    const double piv = at(pr, k);
    if (piv == 0.0) fail(Errc::SingularFactor, "singular matrix: column " + std::to_string(k) + " has no pivot");
    for (int q = k + 1; q < n; ++q) {
      const int rr = perm[q];
      const double f = at(rr, k) / piv;
      at(rr, k) = f;
      if (f != 0.0)
        for (int j = k + 1; j < n; ++j) at(rr, j) -= f * at(pr, j);
    }
  }
  // store the factors in pivot order so lu(k, :) is the k-th pivot row
  DenseMatrix ordered(n, n);
  for (int k = 0; k < n; ++k)
    std::copy_n(lu.a.begin() + std::ptrdiff_t(perm[k]) * n, n, ordered.a.begin() + std::ptrdiff_t(k) * n);
  lu = std::move(ordered);
}

Vector DenseLu::solve(const Vector& b) const {
  const int n = lu.rows;
  if (int(b.size()) != n) fail(Errc::DimensionMismatch, "LU solve: rhs has " + std::to_string(b.size()) +
                                                           " entries, matrix order " + std::to_string(n));
  Vector x(n);
  for (int k = 0; k < n; ++k) {  // forward: unit lower
    double t = b[perm[k]];
    for (int j = 0; j < k; ++j) t -= lu.a[std::size_t(k) * n + j] * x[j];
    x[k] = t;
  }
  for (int k = n - 1; k >= 0; --k) {  // backward: upper
    double t = x[k];
    for (int j = k + 1; j < n; ++j) t -= lu.a[std::size_t(k) * n + j] * x[j];
    x[k] = t / lu.a[std::size_t(k) * n + k];
  }
  return x;
}

DenseMatrix DenseLu::solve(const DenseMatrix& B) const {
  const DenseMatrix Bt = transpose(B);
  DenseMatrix Xt(B.cols, B.rows);
  for (int j = 0; j < B.cols; ++j) {
    const Vector col(Bt.a.begin() + std::ptrdiff_t(j) * B.rows, Bt.a.begin() + std::ptrdiff_t(j + 1) * B.rows);
    const Vector x = solve(col);
    std::copy(x.begin(), x.end(), Xt.a.begin() + std::ptrdiff_t(j) * B.rows);
  }
  return transpose(Xt);
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

// Stored columns of row i in ascending order, in the enumeration the
// reference's matvec / to_dense / generate_random walk (for_each_in_row,
// src/structmat.cpp:211-248): a circulant row may list a wrapped column twice
// and a Babd corner row its overlap with the body span twice.
static void row_columns(const StructuredMatrix& A, int i, std::vector<int>& cols) {
  cols.clear();
  switch (A.kind) {
    case Kind::Banded:
      for (int j = std::max(0, i - A.s); j <= std::min(A.n - 1, i + A.r); ++j) cols.push_back(j);
      break;
    case Kind::BlockTridiagonal: {
      const int b = i / A.m;
      for (int j = std::max(0, (b - 1) * A.m); j < std::min(A.n, (b + 2) * A.m); ++j) cols.push_back(j);
      break;
    }
    case Kind::Abd:
    case Kind::Babd: {
      const auto span = abd_span(A.n, A.m, A.s, A.r, i / A.m);
      for (int j = span.first; j < span.second; ++j) cols.push_back(j);
      if (A.kind == Kind::Babd && i < A.corner_rows)
        for (int j = A.n - A.corner_cols; j < A.n; ++j) cols.push_back(j);
      break;
    }
    case Kind::CirculantLike:
      for (int d = -A.s; d <= A.r; ++d) cols.push_back(((i + d) % A.n + A.n) % A.n);
      std::sort(cols.begin(), cols.end());
      break;
  }
}

namespace {

// the storage slot of the diagonal entry A(i, i)
double& diagonal_slot(StructuredMatrix& A, int i) {
  const int n = A.n, m = A.m;
  switch (A.kind) {
    case Kind::Banded: return A.data[band_offset(n, A.s, 0) + i];
    case Kind::CirculantLike: return A.data[std::size_t(A.s) * n + i];
    case Kind::BlockTridiagonal: {
      const int b = i / m, t = i - b * m;
      const std::size_t row = b == 0 ? 0 : std::size_t(3 * b - 1) * m * m;
      return A.data[row + (b > 0 ? std::size_t(m) * m : 0) + std::size_t(t) * m + t];
    }
    default: {
      const int b = i / m;
      const auto span = abd_span(n, m, A.s, A.r, b);
      return A.data[abd_row_offset(m, A.s, A.r, b) + std::size_t(i - b * m) * (span.second - span.first) +
                    (i - span.first)];
    }
  }
}

}  // namespace

// generate_random (src/structmat.cpp:282-333 semantics): storage-order draws
// of one SplitMix64 stream (corner last), then, with dominance > 0, every
// diagonal entry replaced by +-dominance * max(sum of the row's other |a_ij|, 1)
// keeping its sign.  The off-diagonal sums walk each row's stored columns
// only, so generation is O(nnz).
StructuredMatrix generate_random(Kind kind, int n, int m, int s, int r, std::uint64_t seed, double dominance) {
  if (dominance < 0) fail(Errc::InvalidParameter, "dominance must be >= 0");
  SplitMix64 rng(seed);
  auto draw = [&rng](std::size_t count) {
    std::vector<double> v(count);
    std::generate(v.begin(), v.end(), [&rng] { return rng.next_unit(); });
    return v;
  };
  std::vector<double> data = draw(body_entry_count(kind, n, m, s, r));
  const int edge = kind == Kind::Babd ? m : 0;
  std::vector<double> corner = draw(std::size_t(edge) * edge);
  StructuredMatrix A = make(kind, n, m, s, r, std::move(data), std::move(corner), edge, edge);
  if (dominance == 0.0) return A;
  std::vector<int> cols;
  for (int i = 0; i < n; ++i) {
    row_columns(A, i, cols);
    double off = 0.0;
    for (int j : cols)
      if (j != i) off += std::fabs(A.at(i, j));
    double& slot = diagonal_slot(A, i);
    const double mag = dominance * std::max(off, 1.0);
    slot = A.at(i, i) < 0 ? -mag : mag;
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

DenseMatrix PartitionBlock::body_dense() const {
  DenseMatrix D(L, L);
  const int w = env_s + 1 + env_r;
  for (int i = 0; i < L; ++i)
    for (int off = 0; off < w; ++off) {
      const int j = i - env_s + off;
      if (j >= 0 && j < L) D.at(i, j) = env[std::size_t(i) * w + off];
    }
  return D;
}

// Frame [left separator | body | right separator]: the body and its coupling
// blocks, plus the right separator's own diagonal block (the left one
// belongs to the neighbouring partition).
DenseMatrix PartitionBlock::local_dense() const {
  const int dim = k0 + L + k1, r0 = k0 + L;
  DenseMatrix M(dim, dim);
  const DenseMatrix B = body_dense();
  for (int x = 0; x < L; ++x) {
    std::copy_n(B.a.begin() + std::ptrdiff_t(x) * L, L, M.a.begin() + std::ptrdiff_t(k0 + x) * dim + k0);
    for (int t = 0; t < k0; ++t) {
      M.at(k0 + x, t) = b0.at(x, t);
      M.at(t, k0 + x) = c0.at(x, t);
    }
    for (int t = 0; t < k1; ++t) {
      M.at(k0 + x, r0 + t) = c1.at(x, t);
      M.at(r0 + t, k0 + x) = b1.at(x, t);
    }
  }
  for (int t = 0; t < k1; ++t)
    for (int u = 0; u < k1; ++u) M.at(r0 + t, r0 + u) = a_right.at(t, u);
  return M;
}

// Host view of partition i (1-based): the local system M^(i) the reference
// hands to its per-partition factorizations (src/partition.cpp:107-173
// semantics).  Built by walking the stored columns of the body rows and of
// the two separators' rows once and scattering each entry into the block it
// belongs to; the GPU solver never builds these views.
PartitionBlock extract_block(const StructuredMatrix& A, const PartitionPlan& plan, int i) {
  if (i < 1 || i > plan.p) fail(Errc::IndexOutOfRange, "partition index " + std::to_string(i) + " not in [1, " +
                                                            std::to_string(plan.p) + "]");
  const int k = plan.sep_size;
  const int lsep = plan.has_corner ? i - 1 : i - 2, rsep = lsep + 1;  // separator_starts indices
  PartitionBlock P;
  P.index = i;
  P.kind = A.kind;
  P.m = A.m;
  P.s = A.s;
  P.r = A.r;
  const int b = plan.body_ranges[i - 1].first, e = plan.body_ranges[i - 1].second;
  P.body_begin = b;
  P.L = e - b;
  P.k0 = lsep >= 0 ? k : 0;
  P.k1 = rsep < plan.sep_count() ? k : 0;
  const auto env = scalar_envelope(A);
  P.env_s = std::min(env.first, P.L - 1);
  P.env_r = std::min(env.second, P.L - 1);
  const int w = P.env_s + 1 + P.env_r;
  P.env.assign(std::size_t(P.L) * w, 0.0);
  P.b0 = DenseMatrix(P.L, P.k0);
  P.c0 = DenseMatrix(P.L, P.k0);
  P.b1 = DenseMatrix(P.L, P.k1);
  P.c1 = DenseMatrix(P.L, P.k1);
  const int ls = P.k0 ? plan.separator_starts[lsep] : -1, rs = P.k1 ? plan.separator_starts[rsep] : -1;
  if (P.k0) P.a_left = DenseMatrix(k, k);
  if (P.k1) P.a_right = DenseMatrix(k, k);
  auto in = [](int j, int lo, int len) { return lo >= 0 && j >= lo && j < lo + len; };
  std::vector<int> cols;
  for (int x = 0; x < P.L; ++x) {  // body rows: envelope, b0 (left), c1 (right)
    row_columns(A, b + x, cols);
    for (int j : cols) {
      const double val = A.at(b + x, j);
      if (j >= b && j < e) {
        const int off = (j - b) - x + P.env_s;
        if (off >= 0 && off < w) P.env[std::size_t(x) * w + off] = val;
      } else if (in(j, ls, k)) {
        P.b0.at(x, j - ls) = val;
      } else if (in(j, rs, k)) {
        P.c1.at(x, j - rs) = val;
      }
    }
  }
  for (int t = 0; t < k; ++t) {  // separator rows: c0 / a_left, b1 / a_right
    if (P.k0) {
      row_columns(A, ls + t, cols);
      for (int j : cols) {
        if (j >= b && j < e) P.c0.at(j - b, t) = A.at(ls + t, j);
        else if (in(j, ls, k)) P.a_left.at(t, j - ls) = A.at(ls + t, j);
      }
    }
    if (P.k1) {
      row_columns(A, rs + t, cols);
      for (int j : cols) {
        if (j >= b && j < e) P.b1.at(j - b, t) = A.at(rs + t, j);
        else if (in(j, rs, k)) P.a_right.at(t, j - rs) = A.at(rs + t, j);
      }
    }
  }
  if (plan.has_corner && i == 1 && k > 0) {  // the corner couples the first separator to the last
    const int first = plan.separator_starts.front(), last = plan.separator_starts.back();
    P.corner_slice = DenseMatrix(k, k);
    for (int t = 0; t < k; ++t)
      for (int u = 0; u < k; ++u) P.corner_slice.at(t, u) = A.at(first + t, last + u);
  }
  return P;
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
