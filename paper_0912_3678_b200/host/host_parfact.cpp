// host_parfact.cpp -- parallel_factor / solve / solve_reduced / residual /
// solve_sequential of the C++ API (reference proj/include/parsol/parfact.hpp,
// seqref.hpp), each a thin call into the C ABI (psg.h): no CPU fallback.
#include <algorithm>
#include <chrono>
#include <string>

#include "parsol/parfact.hpp"
#include "parsol/seqref.hpp"
#include "psg.h"

namespace parsol {

namespace {

psg_desc host_desc(const StructuredMatrix& A) {
  return psg_desc{int(A.kind), A.n, A.m, A.s, A.r, A.data.data(), A.data.size(),
                  A.corner.empty() ? nullptr : A.corner.data(), A.corner_rows, A.corner_cols, 0};
}

void check(int rc, const char* err) {
  if (rc) fail(Errc(rc - 1), err);
}

void add_stats(SolveStats* st, const psg_stats& s) {
  if (!st) return;
  st->phase1_seconds += s.phase1_seconds;
  st->phase2_seconds += s.phase2_seconds;
  st->phase3_seconds += s.phase3_seconds;
  st->reduced_ops += s.reduced_ops;
  st->certificate = std::max(st->certificate, s.certificate);
  st->fallbacks += s.fallbacks;
}

}  // namespace

ParallelFactorization parallel_factor(const StructuredMatrix& A, int p, Strategy strategy, double tol) {
  const auto t0 = std::chrono::steady_clock::now();
  char err[512];
  ParallelFactorization F;
  F.strategy = strategy;
  if (A.kind == Kind::CirculantLike && !A.corner_canonical()) {  // src/parfact.cpp:29-35
    auto [B, perm] = permute_corner(A);
    F.plan = plan_partition(B, p);
    F.permuted = true;
    F.row_perm = std::move(perm);  // applied on the device by psg_solve
  } else {
    F.plan = plan_partition(A, p);
  }
  psg_handle* h = nullptr;
  const psg_desc d = host_desc(A);
  check(psg_factor(&d, p, int(strategy), tol, nullptr, &h, err, sizeof err), err);
  F.device = std::shared_ptr<psg_handle>(h, psg_release);
  F.n = A.n;
  int q = 0, dim = 0, k = 0, corner = 0;
  psg_reduced_info(h, &q, &dim, &k, &corner);
  ReducedSystem& R = F.reduced;
  R.q = q;
  R.dim = dim;
  R.has_corner = corner != 0;
  // layout in position order: separators and (LuPivot / Qr) adaptive extras (src/parfact.cpp:72-88)
  R.positions.resize(q);
  R.block_sizes.resize(q);
  psg_reduced_layout(h, R.positions.data(), R.block_sizes.data());
  for (int b = 0, off = 0; b < q; ++b) {
    R.offsets.push_back(off);
    off += R.block_sizes[b];
  }
  // kept_maps (src/parfact.cpp:106-127): [left separator | extras by position | right separator]
  F.kept_maps.assign(p, {});
  const auto find_block = [&](int position) {
    return int(std::lower_bound(R.positions.begin(), R.positions.end(), position) - R.positions.begin());
  };
  for (int i = 0; i < p; ++i) {
    const int left = corner ? i : i - 1, right = corner ? i + 1 : i;
    const int nsep = int(F.plan.separator_starts.size());
    std::vector<int>& map = F.kept_maps[i];
    if (left >= 0)
      for (int t = 0; t < k; ++t) map.push_back(R.offsets[find_block(F.plan.separator_starts[left])] + t);
    auto [b, e] = F.plan.body_ranges[i];
    for (int blk = find_block(b); blk < q && R.positions[blk] < e; ++blk) map.push_back(R.offsets[blk]);
    if (right < nsep)
      for (int t = 0; t < k; ++t) map.push_back(R.offsets[find_block(F.plan.separator_starts[right])] + t);
  }
  if (dim <= kDenseReducedLimit) {  // dense image of T for callers and oracles
    R.T = DenseMatrix(dim, dim);
    check(psg_reduced_dense(h, R.T.a.data(), err, sizeof err), err);
  }
  R.device = F.device;
  check(psg_factor_wait(h, nullptr), "factorization failed on the device");
  F.factor_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return F;
}

Vector solve(const ParallelFactorization& F, const Vector& f, SolveStats* stats) {
  if (int(f.size()) != F.n) fail(Errc::DimensionMismatch, "rhs length");
  char err[512];
  Vector x(f.size());
  psg_stats s{};
  check(psg_solve(F.device.get(), f.data(), x.data(), 0, nullptr, stats ? &s : nullptr, err, sizeof err), err);
  add_stats(stats, s);
  return x;
}

void solve_device(const ParallelFactorization& F, const double* f_dev, double* x_dev, SolveStats* stats,
                  void* stream) {
  char err[512];
  psg_stats s{};
  check(psg_solve(F.device.get(), f_dev, x_dev, 1, stream, stats ? &s : nullptr, err, sizeof err), err);
  add_stats(stats, s);
}

Vector solve_reduced(const ParallelFactorization& F, const Vector& rhs, SolveStats* stats) {
  if (int(rhs.size()) != F.reduced.dim) fail(Errc::DimensionMismatch, "reduced rhs length");
  char err[512];
  Vector x(rhs.size());
  psg_stats s{};
  check(psg_solve_reduced(F.device.get(), rhs.data(), x.data(), 0, nullptr, stats ? &s : nullptr, err, sizeof err),
        err);
  if (stats) stats->reduced_ops += s.reduced_ops;
  return x;
}

Vector solve_reduced(const ReducedSystem& R, const Vector& rhs, SolveStats* stats) {
  if (int(rhs.size()) != R.dim) fail(Errc::DimensionMismatch, "reduced rhs length");
  char err[512];
  Vector x(R.dim);
  if (R.T.rows == R.dim && R.T.cols == R.dim) {
    long long ops = 0;
    check(psg_dense_solve(R.dim, R.T.a.data(), rhs.data(), x.data(), &ops, nullptr, err, sizeof err), err);
    if (stats) stats->reduced_ops += ops;
    return x;
  }
  if (!R.device) fail(Errc::InvalidParameter, "reduced system has neither a dense T nor a device factorization");
  psg_stats s{};
  check(psg_solve_reduced(R.device.get(), rhs.data(), x.data(), 0, nullptr, stats ? &s : nullptr, err, sizeof err),
        err);
  if (stats) stats->reduced_ops += s.reduced_ops;
  return x;
}

void materialize_locals(ParallelFactorization& F, const StructuredMatrix& A, int first, int count, double tol) {
  const int p = F.plan.p;
  if (count < 0) count = p - first + 1;
  if (first < 1 || first + count - 1 > p) fail(Errc::IndexOutOfRange, "partition range");
  if (int(F.locals.size()) != p) F.locals.resize(p);
  const StructuredMatrix* work = &A;
  StructuredMatrix rotated;
  if (F.permuted) {
    rotated = permute_corner(A).first;
    work = &rotated;
  }
  for (int i = first; i < first + count; ++i) {
    try {
      F.locals[i - 1] = factor(F.strategy, extract_block(*work, F.plan, i), tol);
    } catch (const Error& e) {
      fail(e.code(), "partition " + std::to_string(i) + ": " + e.detail());
    }
  }
}

double residual(const StructuredMatrix& A, const Vector& x, const Vector& f) {
  if (int(x.size()) != A.n || int(f.size()) != A.n) fail(Errc::DimensionMismatch, "residual lengths");
  char err[512];
  double out = 0;
  const psg_desc d = host_desc(A);
  check(psg_residual(&d, x.data(), f.data(), 0, nullptr, &out, err, sizeof err), err);
  return out;
}

// No CPU solver in this library: the sequential reference entry point runs
// the GPU partition solver with bodies of ~1023 rows (units of m for blocked kinds).
Vector solve_sequential(const StructuredMatrix& A, const Vector& f) {
  const int unit = A.kind == Kind::Banded ? 1 : A.m;
  const int units = A.n / unit;
  int p = std::max(2, units / 1024);
  // keep the plan feasible for small systems (each body at least one separator wide)
  while (p > 2) {
    const int k_units = A.kind == Kind::Banded ? std::max(A.s, A.r) : 1;
    const long seps = A.kind == Kind::Babd ? p + 1 : p - 1;
    if (units - seps * k_units >= long(p) * std::max(1, k_units)) break;
    p /= 2;
  }
  ParallelFactorization F = parallel_factor(A, p, Strategy::Lu);
  return solve(F, f);
}

}  // namespace parsol
